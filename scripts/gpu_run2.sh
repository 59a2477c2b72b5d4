set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout 600 python bench.py --steps 20 --warmup 3 --cpu-seconds 5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -3 gpurun_out/bench2.err
cat gpurun_out/bench2.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 2 --warmup 3 --blocks 2 --no-cpu > /dev/null 2>&1
