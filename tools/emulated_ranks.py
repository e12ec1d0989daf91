"""Per-rank update time of a row-partitioned c5 run, each rank emulated on one GPU in turn
(the exact code path of an N-GPU run minus the NCCL all-gather): the projected N-GPU
iteration is max over ranks of the rank's update time plus the all-gather.
    python tools/emulated_ranks.py [world ...]"""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, '.')
from gen import synth
from paper_1710_02261_b200 import ptucker as pt

torch.cuda.set_device(0)
cfg = synth.config("c5")
coords, vals = synth.generate(cfg)
worlds = [int(w) for w in sys.argv[1:]] or [2, 4, 8]
for world in worlds:
    per_rank = []
    for r in range(world):
        pt.ptucker_finalize()
        pt.ptucker_set_option("emulate_world", world)
        pt.ptucker_set_option("emulate_rank", r)
        pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * 3, cfg.lam, 0)
        for _ in range(2):
            pt.ptucker_sweep()
        pt.ptucker_synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            pt.ptucker_sweep()
            pt.ptucker_error()
        pt.ptucker_synchronize()
        per_rank.append((time.perf_counter() - t0) / 3 * 1e3)
    pt.ptucker_finalize()
    pt.ptucker_set_option("emulate_world", 1)
    pt.ptucker_set_option("emulate_rank", 0)
    mx = max(per_rank)
    print(f"world {world}: per-rank ms per iteration (no all-gather) min {min(per_rank):.3f} max {mx:.3f}; "
          f"projected entries/s {cfg.nnz / (mx / 1e3):.3e} + all-gather of 3 x 40 MB per iteration", flush=True)
