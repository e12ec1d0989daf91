# usage: bash tools/seg_sweep.sh CONFIG "seg1 seg2 ..."  : ms per iteration for each seg_len
cd $GRAFT_REPO_ROOT
cfg=$1
for sl in $2; do
  timeout 300 python bench.py --config $cfg --seg-len $sl --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 \
    | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('[$cfg seg $sl]', round(d['ms_per_step'],4), 'frac', round(r['frac'],4), r['ms_per_step_by_kernel'], 'launches', d['gpu_launches'])" >> gpurun_out/seg.txt \
    || echo "[$cfg seg $sl] run-fail" >> gpurun_out/seg.txt
done
