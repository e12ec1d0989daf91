"""Time ptucker_core_scores (Approx, Eq. 13) on a config for each scores kernel variant.
    python tools/time_scores.py [config] [scale]"""
import sys
import time
import torch
sys.path.insert(0, '.')
from gen import synth
from paper_1710_02261_b200 import ptucker as pt

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
cfg = synth.small(name, scale) if scale < 1 else synth.config(name)
coords, vals = synth.generate(cfg)
torch.cuda.set_device(0)
pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * len(cfg.dims), cfg.lam, 0)
pt.ptucker_sweep()
ref = None
for v in (0,):
    R = pt.ptucker_core_scores()
    pt.ptucker_synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        R = pt.ptucker_core_scores()
    pt.ptucker_synchronize()
    dt = (time.perf_counter() - t0) / 3 * 1e3
    if ref is None:
        ref = R
    print(f"{name} scale {scale} approx_kernel {v}: {dt:.2f} ms per scores call; max |R - R_v0| / max|R| = "
          f"{abs(R - ref).max() / abs(ref).max():.2e}")
