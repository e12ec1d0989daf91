"""Per-phase clock trace of the tensor-core update kernel (CTA 0, lane 0 of each of its
4 warps, tiles 64..127 of its sequence).  Phases per tile k:
0 start, 1 after the cp.async issue step (coordinates k+7, rows k+3), 2 after the
cp.async wait for the rows of k+1, 3 after splitting them into the A tile, 4 after
arriving (MMA issued by the last arriver), 5 after waiting for tile k's MMA,
6 after TMEM loads + level 0, 7 after B/c.

    python tools/trace_tc.py [scale] [l0_group]"""
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
if len(sys.argv) > 2:
    pt.ptucker_set_option("l0_group", int(sys.argv[2]))
pt.ptucker_update_mode(0)
pt.ptucker_set_option("trace", 1)
pt.ptucker_update_mode(1)
pt.ptucker_synchronize()
tr = pt.ptucker_debug_trace(4 * 512).reshape(4, 64, 8)
names = ["issue", "cp.wait", "split", "arrive", "mma wait", "tmem+L0", "B/c", "->next"]
for w in range(4):
    t = tr[w]
    ok = t[:, 0] > 0
    t = t[ok]
    d = np.diff(np.concatenate([t, np.roll(t[:, :1], -1, axis=0)], axis=1), axis=1)[:-1]
    print(f"warp {w}: entries {len(t)}; median cycles per phase: " +
          ", ".join(f"{n} {int(np.median(d[:, i]))}" for i, n in enumerate(names)) +
          f"; per entry {int(np.median(np.diff(t[:, 0])))}")
