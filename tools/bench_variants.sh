# usage: bash tools/bench_variants.sh "bench args" ...  : c5 bench per argument set (current build)
cd $GRAFT_REPO_ROOT
for a in "$@"; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $a 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('[$a]', d['ms_per_step'], {k: v for k, v in d['roofline']['ms_per_step_by_kernel'].items() if k.startswith('update')})" >> gpurun_out/sweep.txt || echo "[$a] run-fail" >> gpurun_out/sweep.txt
done
