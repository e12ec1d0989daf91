python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke25.txt 2>&1; echo "rc=$?" >> gpurun_out/smoke25.txt
timeout 2000 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/t25.txt 2>&1
timeout 400 python bench.py > gpurun_out/bench25.json 2> gpurun_out/bench25.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref25.json 2> gpurun_out/ref25.err
