timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "invalid or worked or edge or determinism or c1" > gpurun_out/t28.txt 2>&1
PTUCKER_DEBUG=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench28.json 2> gpurun_out/bench28.err
