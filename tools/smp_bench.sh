cd $GRAFT_REPO_ROOT
for fl in "$@"; do
  touch paper_1710_02261_b200/csrc/smp.cu
  NVCC_APPEND_FLAGS="$fl" python -c "from paper_1710_02261_b200 import build; build.build()" > /dev/null 2>&1 || { echo "[$fl] build-fail" >> gpurun_out/sweep.txt; continue; }
  for rep in 1 2; do
  timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('[$fl]', d['ms_per_step'], {k: v for k, v in d['roofline']['ms_per_step_by_kernel'].items() if k.startswith('update')})" >> gpurun_out/sweep.txt
  done
done
