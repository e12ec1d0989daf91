cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/fs
python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/fs/tests.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fs/smoke.txt 2>&1
python bench.py > gpurun_out/fs/bench.json 2> gpurun_out/fs/bench.err
python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fs/bench_c4.json 2> gpurun_out/fs/bench_c4.err
python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --policy F32-C > gpurun_out/fs/bench_c4_f32c.json 2> gpurun_out/fs/bench_c4_f32c.err
tail -3 gpurun_out/fs/tests.txt; cat gpurun_out/fs/smoke.txt | tail -2; cut -c1-400 gpurun_out/fs/bench.json; cut -c1-300 gpurun_out/fs/bench_c4.json
