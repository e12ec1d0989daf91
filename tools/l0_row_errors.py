"""GPU row errors of the tensor-core update for each level-0 grouping (l0_group 1, 2, 5),
over ALL rows of one mode update from the init state, against the FP64 oracle from the
identical stored state (the per-row criterion of BASELINE.json's north star).

    python tools/l0_row_errors.py [config] [scale] [mode] [sweeps] [groups]

sweeps (default 0): FP64 oracle sweeps applied to the init state before the comparison
(a mid-trajectory state); groups (default "1,2,5"): the l0_group values to run.
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from gen import synth  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_1710_02261_b200 import ptucker as pt  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else 'c5'
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
n = int(sys.argv[3]) if len(sys.argv) > 3 else 0
sweeps = int(sys.argv[4]) if len(sys.argv) > 4 else 0
groups = [int(x) for x in sys.argv[5].split(",")] if len(sys.argv) > 5 else [1, 2, 5]
torch.cuda.set_device(0)
cfg = synth.small(name, scale) if scale < 1 else synth.CONFIGS[name]
coords, vals = synth.generate(cfg)
N = len(cfg.dims)
t0 = time.time()
t = orc.Tensor(coords, vals, cfg.dims)
m = orc.init_model(cfg.dims, [cfg.J] * N, seed=0, prec=0)
for _ in range(sweeps):
    for k in range(N):
        orc.update_mode(t, m, k, cfg.lam)
m32 = orc.Model(m.G.astype(np.float32).astype(np.float64), [a.astype(np.float32).astype(np.float64) for a in m.factors])
ref = m32.copy() if hasattr(m32, 'copy') else orc.Model(m32.G.copy(), [a.copy() for a in m32.factors])
orc.update_mode(t, ref, n, cfg.lam)
a_ref = ref.A(n)
print(f"{name} scale {scale} mode {n} after {sweeps} sweeps: {cfg.dims[n]} rows, {len(vals)} entries; "
      f"oracle {time.time() - t0:.1f} s")
den = np.linalg.norm(a_ref, axis=1)
nz = den > 0
for g in groups:
    pt.ptucker_finalize()
    pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * N, cfg.lam, 0)
    pt.ptucker_set_option("l0_group", g)
    pt.ptucker_set_core(m32.G.astype(np.float32))
    for k in range(N):
        pt.ptucker_set_factor(k, m32.A(k).astype(np.float32))
    pt.ptucker_update_mode(n)
    a = pt.ptucker_get_factor(n).astype(np.float64)
    err = np.linalg.norm(a - a_ref, axis=1)[nz] / den[nz]
    q = [np.quantile(err, 1 - 10.0 ** -k) for k in (2, 3, 4, 5) if 10 ** k <= err.size]
    print(f"  l0_group {g}: max {err.max():.2e}  quantiles 1-1e-2.. {' '.join(f'{z:.2e}' for z in q)}  "
          f"median {np.median(err):.2e}  rows > 1e-5: {(err > 1e-5).sum()}", flush=True)
pt.ptucker_finalize()
