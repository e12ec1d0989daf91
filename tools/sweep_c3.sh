# usage: bash tools/sweep_c3.sh "FLAGS" ... : rebuild update_tc.cu with FLAGS, bench c3 (per-mode) and c5
cd $GRAFT_REPO_ROOT
for fl in "$@"; do
  touch paper_1710_02261_b200/csrc/update_tc.cu
  NVCC_APPEND_FLAGS="$fl" python -c "from paper_1710_02261_b200 import build; build.build()" > /dev/null 2>&1 || { echo "[$fl] build-fail" >> gpurun_out/sweep.txt; continue; }
  for c in c3 c5; do
    timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('[$fl $c]', d['ms_per_step'], {k: v for k, v in d['roofline']['ms_per_step_by_kernel'].items() if k.startswith('update')})" >> gpurun_out/sweep.txt || echo "[$fl $c] run-fail" >> gpurun_out/sweep.txt
  done
done
