# usage: bash tools/sweep_tc.sh "FLAGS1" "FLAGS2" ...  (nvcc -D flags for update_tc.cu; c5 bench per variant)
cd $GRAFT_REPO_ROOT
for fl in "$@"; do
  touch paper_1710_02261_b200/csrc/update_tc.cu
  NVCC_APPEND_FLAGS="$fl" python -c "from paper_1710_02261_b200 import build; build.build()" > gpurun_out/sweep_build.log 2>&1 || { echo "$fl build-fail" >> gpurun_out/sweep.txt; continue; }
  grep -A3 "k_update_tcILi10ELb1ELi1E" paper_1710_02261_b200/_obj/update_tc.ptxas.txt | grep spill | head -1 | sed "s/^/[$fl] /" >> gpurun_out/sweep.txt
  timeout 300 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('[$fl]', d['ms_per_step'], d['roofline']['ms_per_step_by_kernel']['update_m0'])" >> gpurun_out/sweep.txt || echo "[$fl] run-fail" >> gpurun_out/sweep.txt
done
