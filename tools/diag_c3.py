"""Per-mode worst row error of one mode update (oracle-made init state) for c3 at a
given scale, with the small-mode tables on/off."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from gen import synth
from oracle import oracle as orc
from paper_1710_02261_b200 import ptucker as pt
from test_gpu_parity import oracle_state, push_state, row_rel_err

torch.cuda.set_device(0)
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.005
cfg = synth.small("c3", scale)
T64 = int(sys.argv[2]) if len(sys.argv) > 2 else 1
coords, vals = synth.generate(cfg)
t = orc.Tensor(coords, vals, cfg.dims)
for sweeps in (0, 1):
    s0 = oracle_state(orc, t, cfg, sweeps)
    refs = []
    for n in range(4):
        m = s0.copy(); orc.update_mode(t, m, n, cfg.lam); refs.append(m.A(n).copy())
    for smp in (1, 0):
        pt.ptucker_finalize()
        pt.ptucker_init(coords, vals, cfg.dims, [10] * 4, cfg.lam, 0)
        pt.ptucker_set_option("smp", smp)
        pt.ptucker_set_option("smp_table", T64)
        out = []
        for n in range(4):
            push_state(pt, s0, np.float32)
            pt.ptucker_update_mode(n)
            e = row_rel_err(pt.ptucker_get_factor(n), refs[n])
            row_ptr, _ = t.mode_index(n)
            lens = np.diff(row_ptr)[np.linalg.norm(refs[n], axis=1) > 0]
            i = int(np.argmax(e))
            out.append(f"mode {n}: max {e.max():.2e} (row len {lens[i]}) p99 {np.quantile(e, .99):.2e}")
        print(f"scale {scale} sweeps {sweeps} smp {smp}: " + "; ".join(out), flush=True)
