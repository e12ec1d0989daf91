timeout 2000 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/t26.txt 2>&1
