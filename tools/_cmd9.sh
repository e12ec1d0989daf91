timeout 60 python tools/quick_update.py c2 0.01 > gpurun_out/q9.txt 2>&1 || exit 1
timeout 60 python tools/quick_update.py c5 0.001 >> gpurun_out/q9.txt 2>&1 || exit 1
timeout 60 python tools/quick_update.py c3 0.005 2 >> gpurun_out/q9.txt 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_unequal_j.py -x -q > gpurun_out/t9.txt 2>&1
bash tools/ab_libs.sh c5 "prod k0 r144"
bash tools/seg_sweep.sh c2 "-1 32"
bash tools/seg_sweep.sh c1 "-1 16"
