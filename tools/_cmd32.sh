timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench32_c3.json 2>&1
timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench32_c5.json 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "c3 or c5 or c2" > gpurun_out/t32.txt 2>&1
