# usage: bash tools/ab_libs.sh CONFIG "name1 name2 ..." [extra bench args]
# A/B of experiment builds (python -m paper_1710_02261_b200.build --variant NAME -D...):
# bench CONFIG once per variant library (PTUCKER_LIB) plus the product build ("prod").
cd $GRAFT_REPO_ROOT
cfg=$1; names=$2; shift 2
for v in $names; do
  if [ "$v" = prod ]; then lib=""; else lib=paper_1710_02261_b200/_variants/$v/libptucker.so; fi
  PTUCKER_LIB=$lib timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>gpurun_out/ab_$v.err | tail -1 \
    | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('[$cfg $v]', round(d['ms_per_step'],4), 'frac', round(r['frac'],4), r['ms_per_step_by_kernel'])" >> gpurun_out/ab.txt \
    || echo "[$cfg $v] run-fail" >> gpurun_out/ab.txt
done
