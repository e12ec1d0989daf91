timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c3" > gpurun_out/t23.txt 2>&1
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench23.json 2>&1
