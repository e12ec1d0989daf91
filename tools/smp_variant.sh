# usage: bash tools/smp_variant.sh "FLAGS" ... : rebuild smp.cu with FLAGS; c3 bench + c3 parity (f32) + fullsize c3
cd $GRAFT_REPO_ROOT
for fl in "$@"; do
  touch paper_1710_02261_b200/csrc/smp.cu
  NVCC_APPEND_FLAGS="$fl" python -c "from paper_1710_02261_b200 import build; build.build()" > /dev/null 2>&1 || { echo "[$fl] build-fail" >> gpurun_out/sweep.txt; continue; }
  timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('[$fl]', d['ms_per_step'], {k: v for k, v in d['roofline']['ms_per_step_by_kernel'].items() if k.startswith('update')})" >> gpurun_out/sweep.txt
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -s -k "c3" 2>&1 | grep -E "worst|passed|failed|max row" | head -8 | sed "s/^/[$fl] /" >> gpurun_out/sweep.txt
done
