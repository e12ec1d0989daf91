# PDL A/B: per config, bench lines with option pdl = 0 and 1 (alternating), then the GPU suite
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pdl
for c in c1 c2 c3 c5; do
  for rep in 1 2; do
    for v in 0 1; do
      timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --opt pdl=$v 2>>gpurun_out/pdl/err.txt | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$c pdl=$v rep$rep', round(d['ms_per_step'],4), 'frac', round(r['frac'],4), r.get('ms_per_step_by_kernel'))" >> gpurun_out/pdl/ab.txt 2>&1
    done
  done
done
python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pdl/tests.txt
