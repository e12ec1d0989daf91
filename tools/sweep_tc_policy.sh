# usage: bash tools/sweep_tc_policy.sh POLICY "FLAGS1" ...  (as sweep_tc.sh with bench --policy)
cd $GRAFT_REPO_ROOT
pol=$1; shift
for fl in "$@"; do
  touch paper_1710_02261_b200/csrc/update_tc.cu
  NVCC_APPEND_FLAGS="$fl" python -c "from paper_1710_02261_b200 import build; build.build()" > gpurun_out/sweep_build.log 2>&1 || { echo "$fl build-fail" >> gpurun_out/sweep.txt; continue; }
  timeout 300 python bench.py --steps 5 --warmup 3 --policy $pol 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('[$pol $fl]', d['ms_per_step'], d['roofline']['ms_per_step_by_kernel']['update_m0'])" >> gpurun_out/sweep.txt || echo "[$fl] run-fail" >> gpurun_out/sweep.txt
done
