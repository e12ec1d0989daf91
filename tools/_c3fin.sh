cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c3f
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_all.py -m gpu -q -x -k "not c5_full_all_rows and not c2_full" 2>&1 | tail -4 > gpurun_out/c3f/tests.txt
for c in c3 c2 c1; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 \
   | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('[$c]', round(d['ms_per_step'],4), round(r['frac'],4), r['ms_per_step_by_kernel'])" >> gpurun_out/c3f/ab.txt
done
