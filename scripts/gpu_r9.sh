timeout 900 python bench.py > gpurun_out/bench_r9.json 2> gpurun_out/bench_r9.err; tail -3 gpurun_out/bench_r9.err
cat gpurun_out/bench_r9.json
