timeout 60 python tools/quick_update.py c2 0.01 > gpurun_out/q10.txt 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_unequal_j.py tests/test_gpu_push.py tests/test_gpu_generic.py -x -q > gpurun_out/t10.txt 2>&1
bash tools/seg_sweep.sh c2 "-1"
bash tools/seg_sweep.sh c1 "-1 16"
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench10.json 2> gpurun_out/bench10.err
