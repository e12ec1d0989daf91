cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/full
for a in "c4 F32-C2" "c4 auto"; do set -- $a
  timeout 600 python bench.py --config $1 --policy $2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 \
   | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('[$1 $2]', round(d['ms_per_step'],4), round(r['frac'],4), r['ms_per_step_by_kernel'])" >> gpurun_out/full/c4.txt
done
python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/full/tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full/smoke.txt 2>&1
python bench.py > gpurun_out/full/bench.json 2> gpurun_out/full/bench.err
