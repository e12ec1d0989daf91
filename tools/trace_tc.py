"""Per-phase clock trace of the tensor-core update kernel (CTA 0, lane 0 of the 4
level-0 warps, tiles 64..127).  Phases per tile k: 0 start, 6 after splitting the A rows
of tile k + 4, 1 after waiting for MMA k,
2 after issuing its TMEM loads + reading a0/x,
3 after the TMEM wait, 4 after level 0, 5 after handing delta to the normal-equation
warp.  Also the MMA warp: waits for the A rows and for a free accumulator, issue time.

    python tools/trace_tc.py [scale] [l0_group] [latency]

The marks are compiled in only with -DPT_TRACE (tools/trace_variant.sh builds that way;
the production library has no trace code in the kernel)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from gen import synth
from paper_1710_02261_b200 import ptucker as pt

torch.cuda.set_device(0)
import os
_name = os.environ.get("PT_TRACE_CFG", "c5")
_scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
cfg = synth.small(_name, _scale) if _scale < 1 else synth.config(_name)
coords, vals = synth.generate(cfg)
pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * len(cfg.dims), cfg.lam, 0)
_mode = int(os.environ.get("PT_TRACE_MODE", "1"))
if len(sys.argv) > 2:
    pt.ptucker_set_option("l0_group", int(sys.argv[2]))
import os
if os.environ.get("PT_TRACE_POLICY"):
    pt.ptucker_set_option("policy", int(os.environ["PT_TRACE_POLICY"]))
pt.ptucker_update_mode(0)
pt.ptucker_set_option("trace", 1)
pt.ptucker_update_mode(_mode)
pt.ptucker_synchronize()
full = pt.ptucker_debug_trace(8 * 512)
m = full[4 * 512:4 * 512 + 512].reshape(64, 8)
if len(sys.argv) > 3:  # latency probe: MMA issue -> completion, measured serialised
    pt.ptucker_set_option("trace", 2)
    pt.ptucker_update_mode(2)
    pt.ptucker_synchronize()
    f2 = pt.ptucker_debug_trace(8 * 512)[4 * 512:4 * 512 + 512].reshape(64, 8)
    print("MMA latency (issue -> accumulator ready, serialised): median %d cycles" % np.median(f2[:, 4] - f2[:, 3]))
ld = full[6 * 512:6 * 512 + 512].reshape(64, 8)
print("loader warp, median cycles: raw_empty wait %d, coords wait %d, row gathers %d, coords issue %d; per tile %d" % (
    np.median(ld[:, 1] - ld[:, 0]), np.median(ld[:, 2] - ld[:, 1]), np.median(ld[:, 3] - ld[:, 2]),
    np.median(ld[:, 4] - ld[:, 3]), np.median(np.diff(ld[:, 0]))))
ne = full[5 * 512:5 * 512 + 512].reshape(64, 8)
print("normal-equation warp 8, median cycles: (unused) %d, delta wait %d, B/c %d; per tile %d" % (
    np.median(ne[:, 1] - ne[:, 0]), np.median(ne[:, 2] - ne[:, 1]), np.median(ne[:, 3] - ne[:, 2]),
    np.median(np.diff(ne[:, 0]))))
print("MMA warp (pipeline 0), median cycles: a_full wait %d, acc_empty wait %d, issue %d; per tile %d" % (
    np.median(m[:, 1] - m[:, 0]), np.median(m[:, 2] - m[:, 1]), np.median(m[:, 3] - m[:, 2]),
    np.median(np.diff(m[:, 0]))))
tr = pt.ptucker_debug_trace(4 * 512).reshape(4, 64, 8)[:, :, [0, 7, 6, 1, 2, 3, 4, 5]]
names = ["rows(k+4) wait", "MMA(k) wait + split(k+4)", "acc wait", "ld+a0", "tmem wait", "L0", "handoff", "->next"]
for w in range(4):
    t = tr[w]
    ok = t[:, 0] > 0
    t = t[ok]
    d = np.diff(np.concatenate([t, np.roll(t[:, :1], -1, axis=0)], axis=1), axis=1)[:-1]
    print(f"warp {w}: entries {len(t)}; median cycles per phase: " +
          ", ".join(f"{n} {int(np.median(d[:, i]))}" for i, n in enumerate(names)) +
          f"; per entry {int(np.median(np.diff(t[:, 0])))}")

# ---- critical path of the even tiles 72..120 on the common SM clock
L0 = full[0:512].reshape(64, 8)          # level-0 warp 0: row m = tile 64 + 2m
MM = full[4 * 512:4 * 512 + 512].reshape(64, 8)   # MMA warp: row m = tile 64 + m
NE = full[5 * 512:5 * 512 + 512].reshape(64, 8)   # normal-equation warp 8: row m = iteration 64 + m
KNA = 4
print("tile: split(k) done (level-0 warp, iteration k-4) -> MMA a_full ok -> MMA issued -> L0 acc_full ok -> L0 handoff done -> NE delta ok  (cycles after split)")
for k in range(72, 122, 6):
    if k % 2:
        continue
    j = k - KNA - 64
    if j < 0:
        continue
    t0 = L0[j // 2, 6]
    row = [MM[k - 64, 1], MM[k - 64, 3], L0[(k - 64) // 2, 1], L0[(k - 64) // 2, 5], NE[k - 64, 2]]
    print(k, [int(x - t0) for x in row])
