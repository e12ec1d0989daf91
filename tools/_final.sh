cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
for c in c1 c2 c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/final/bench_all.jsonl
done
timeout 600 python bench.py --config c5 --dtype f64 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/final/bench_all.jsonl
python bench.py > gpurun_out/final/bench_default.json 2> gpurun_out/final/bench_default.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/final/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/final/ncu.log 2>&1
