O=gpurun_out/c1; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 300 ./scripts/micro/bulk_warp_bench > $O/bulk_warp.txt 2>&1
timeout 300 ./scripts/micro/stream_bench > $O/stream.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
