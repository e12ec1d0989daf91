"""Per-phase clock trace of the tensor-core update kernel (CTA 0, lane 0 of the 4
epilogue warps of pipeline 0, tiles 64..127 of its sequence).  Phases per tile k:
0 start, 1 after level 0 of tile k (TMEM loads + F2F/DFMA), 2 after waiting for
MMA k+1, 3 after the normal equations of tile k, 4 (group end) ..., 4 after the
first TMEM loads of k+1, the A rows of tile k+2 and a0/x of tile k+1.

    python tools/trace_tc.py [scale] [l0_group] [latency]"""
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
full = pt.ptucker_debug_trace(8 * 512)
m = full[4 * 512:4 * 512 + 512].reshape(64, 8)
if len(sys.argv) > 3:  # latency probe: MMA issue -> completion, measured serialised
    pt.ptucker_set_option("trace", 2)
    pt.ptucker_update_mode(2)
    pt.ptucker_synchronize()
    f2 = pt.ptucker_debug_trace(8 * 512)[4 * 512:4 * 512 + 512].reshape(64, 8)
    print("MMA latency (issue -> accumulator ready, serialised): median %d cycles" % np.median(f2[:, 4] - f2[:, 3]))
print("MMA warp (pipeline 0), median cycles: a_full wait %d, acc_empty wait %d, issue %d; per tile %d" % (
    np.median(m[:, 1] - m[:, 0]), np.median(m[:, 2] - m[:, 1]), np.median(m[:, 3] - m[:, 2]),
    np.median(np.diff(m[:, 0]))))
tr = pt.ptucker_debug_trace(4 * 512).reshape(4, 64, 8)[:, :, [0, 1, 2, 3, 4]]
names = ["L0(k)", "wait mma(k+1)", "B/c(k)", "group end+tmem+split+a0", "->next"]
for w in range(4):
    t = tr[w]
    ok = t[:, 0] > 0
    t = t[ok]
    d = np.diff(np.concatenate([t, np.roll(t[:, :1], -1, axis=0)], axis=1), axis=1)[:-1]
    print(f"warp {w}: entries {len(t)}; median cycles per phase: " +
          ", ".join(f"{n} {int(np.median(d[:, i]))}" for i, n in enumerate(names)) +
          f"; per entry {int(np.median(np.diff(t[:, 0])))}")
