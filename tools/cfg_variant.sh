# usage: bash tools/cfg_variant.sh CONFIG "FLAGS" ...  : rebuild every object with FLAGS, bench CONFIG
cd $GRAFT_REPO_ROOT
cfg=$1; shift
for fl in "$@"; do
  NVCC_APPEND_FLAGS="$fl" python -c "from paper_1710_02261_b200 import build; build.build(force=True)" > /dev/null 2>&1 || { echo "[$fl] build-fail" >> gpurun_out/sweep.txt; continue; }
  timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('[$cfg $fl]', d['ms_per_step'], d['roofline']['frac'], d['roofline']['ms_per_step_by_kernel'])" >> gpurun_out/sweep.txt || echo "[$fl] run-fail" >> gpurun_out/sweep.txt
done
