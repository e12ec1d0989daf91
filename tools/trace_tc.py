"""Per-phase clock trace of the tensor-core update kernel (CTA 0, lane 0 of each of its
4 warps, first 64 entries of its first slice group).  Phases per entry:
0 start, 1 after cp.async issue + coordinate loads, 2 after cp.async wait, 3 after
building the next A tile, 4 after arriving (MMA issued by the last arriver),
5 after waiting for this entry's MMA, 6 after TMEM loads + level 0, 7 after B/c."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from gen import synth
from paper_1710_02261_b200 import ptucker as pt

torch.cuda.set_device(0)
cfg = synth.small("c5", float(sys.argv[1]) if len(sys.argv) > 1 else 0.1)
coords, vals = synth.generate(cfg)
pt.ptucker_init(coords, vals, cfg.dims, [10] * 3, cfg.lam, 0)
pt.ptucker_update_mode(0)
pt.ptucker_set_option("trace", 1)
pt.ptucker_update_mode(1)
pt.ptucker_synchronize()
tr = pt.ptucker_debug_trace(4 * 512).reshape(4, 64, 8)
names = ["issue/coords", "cp.wait", "build A", "arrive", "mma wait", "tmem+L0", "B/c", "->next"]
for w in range(4):
    t = tr[w]
    ok = t[:, 0] > 0
    t = t[ok]
    d = np.diff(np.concatenate([t, np.roll(t[:, :1], -1, axis=0)], axis=1), axis=1)[:-1]
    print(f"warp {w}: entries {len(t)}; median cycles per phase: " +
          ", ".join(f"{n} {int(np.median(d[:, i]))}" for i, n in enumerate(names)) +
          f"; per entry {int(np.median(np.diff(t[:, 0])))}")
