"""One mode update of a reduced config against the oracle (a quick kernel check):
    python tools/quick_update.py CONFIG SCALE [mode]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from gen import synth  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_1710_02261_b200 import ptucker as pt  # noqa: E402

torch.cuda.set_device(0)
name, scale = sys.argv[1], float(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cfg = synth.small(name, scale)
coords, vals = synth.generate(cfg)
N = len(cfg.dims)
pt.ptucker_set_option("seg_len", 256)
pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * N, cfg.lam, 0)
t0 = time.time()
pt.ptucker_update_mode(n)
a = pt.ptucker_get_factor(n).astype(np.float64)
dt = time.time() - t0
m = orc.init_model(cfg.dims, [cfg.J] * N, seed=0, prec=0)
orc.update_mode(orc.Tensor(coords, vals, cfg.dims), m, n, cfg.lam)
den = np.linalg.norm(m.A(n), axis=1)
err = np.linalg.norm(a - m.A(n), axis=1)[den > 0] / den[den > 0]
print(f"{name}@{scale} mode {n}: max row rel err {err.max():.2e} ({dt:.2f} s)", flush=True)
