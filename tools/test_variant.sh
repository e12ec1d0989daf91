# usage: bash tools/test_variant.sh "FLAGS" ...  : build update_tc.cu with FLAGS, run the f32 mode-update parity test + c5 bench
cd $GRAFT_REPO_ROOT
for fl in "$@"; do
  touch paper_1710_02261_b200/csrc/update_tc.cu
  NVCC_APPEND_FLAGS="$fl" python -c "from paper_1710_02261_b200 import build; build.build()" > /dev/null 2>&1 || { echo "[$fl] build-fail" >> gpurun_out/sweep.txt; continue; }
  r=$(timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "mode_update_f32" 2>&1 | grep -E "passed|failed|Error" | tail -2 | tr '\n' ' ')
  echo "[$fl] test: $r" >> gpurun_out/sweep.txt
  timeout 300 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('[$fl]', d['ms_per_step'], d['roofline']['ms_per_step_by_kernel']['update_m0'])" >> gpurun_out/sweep.txt || echo "[$fl] run-fail" >> gpurun_out/sweep.txt
done
