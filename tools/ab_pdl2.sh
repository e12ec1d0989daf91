# PDL trigger placement A/B: product build (late trigger) with pdl = 0 / 1, variant pdl_early
# (trigger at kernel start) with pdl = 1; then the PDL bit-identity tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pdl2
run() {  # cfg name lib pdl
  PTUCKER_LIB=$3 timeout 600 python bench.py --config $1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --opt pdl=$4 2>>gpurun_out/pdl2/err.txt | tail -1 \
   | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('[$1 $2 pdl=$4]', round(d['ms_per_step'],4), 'frac', round(r['frac'],4), r['ms_per_step_by_kernel'])" >> gpurun_out/pdl2/ab.txt 2>&1
}
E=paper_1710_02261_b200/_variants/pdl_early/libptucker.so
for c in c2 c1 c2 c3; do
  run $c late "" 0
  run $c late "" 1
  run $c early $E 1
done
python -m pytest tests/test_gpu_parity.py -m gpu -q -k pdl 2>&1 | tail -3 > gpurun_out/pdl2/tests.txt
