cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/kahan
for c in "c5 0.001 0" "c2 0.01 1"; do python - $c >> gpurun_out/kahan/quick.txt 2>&1 <<'PY'
import sys; sys.path.insert(0,'.')
import numpy as np, torch
from gen import synth
from oracle import oracle as orc
from paper_1710_02261_b200 import ptucker as pt
torch.cuda.set_device(0)
name, scale, n = sys.argv[1], float(sys.argv[2]), int(sys.argv[3])
cfg = synth.small(name, scale); coords, vals = synth.generate(cfg); N = len(cfg.dims)
pt.ptucker_init(coords, vals, cfg.dims, [cfg.J]*N, cfg.lam, 0); pt.ptucker_set_option("l0_group", 0)
pt.ptucker_update_mode(n); a = pt.ptucker_get_factor(n).astype(np.float64)
m = orc.init_model(cfg.dims, [cfg.J]*N, seed=0, prec=0); orc.update_mode(orc.Tensor(coords, vals, cfg.dims), m, n, cfg.lam)
den = np.linalg.norm(m.A(n), axis=1); err = np.linalg.norm(a - m.A(n), axis=1)[den > 0] / den[den > 0]
print(f"{name}@{scale} mode {n} l0_group 0: max row rel err {err.max():.2e}", flush=True)
PY
done
for l in 1 0; do
  timeout 600 python bench.py --config c5 --l0-group $l --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 \
   | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('[c5 l0_group $l]', round(d['ms_per_step'],4), round(r['frac'],4), r['ms_per_step_by_kernel'])" >> gpurun_out/kahan/ab.txt
done
for m in 0 1 2; do timeout 600 python tools/l0_row_errors.py c5 1.0 $m 0 "1,0" >> gpurun_out/kahan/rows.txt 2>&1; done
