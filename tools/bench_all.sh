# c1..c5 bench lines (N=1) -> gpurun_out/bench_all.jsonl
cd $GRAFT_REPO_ROOT
for c in c1 c2 c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/bench_all.jsonl
done
