import sys, time, os
sys.path.insert(0,'.')
import numpy as np, torch
from gen import synth
from paper_1710_02261_b200 import ptucker as pt
torch.cuda.set_device(0)
cfg = synth.config('c5')
coords, vals = synth.generate(cfg)
pc = torch.from_numpy(coords).pin_memory().numpy(); pv = torch.from_numpy(vals).pin_memory().numpy()
for rep in range(int(os.environ.get('PT_INIT_REPS', '2'))):
    t0 = time.perf_counter()
    pt.ptucker_init(pc, pv, cfg.dims, [10]*3, cfg.lam, 0)
    pt.ptucker_synchronize()
    print("init", time.perf_counter() - t0, flush=True)
