cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/fs
python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/fs/tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fs/smoke.txt 2>&1
python bench.py > gpurun_out/fs/bench.json 2> gpurun_out/fs/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fs/bench_ref.json 2> gpurun_out/fs/bench_ref.err
