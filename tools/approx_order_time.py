"""P-Tucker-Approx on the order-scaling workload (N-way, I = 100, |Omega| = 10^3,
J = 3; the shapes of the paper's Approx/Cache experiments): per-iteration device
time of the sweep for plain P-Tucker and for Approx (p = 0.2) with the sparse-core delta, and of
the scoring + truncation step.

    python tools/approx_order_time.py [orders] [iterations]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from gen import synth  # noqa: E402
from paper_1710_02261_b200 import ptucker as pt  # noqa: E402

torch.cuda.set_device(0)
orders = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [6, 8, 10]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 8
stream = torch.cuda.Stream()   # a real stream: the library's kernels and the events on it
torch.cuda.set_stream(stream)


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for N in orders:
    cfg = synth.order(N)
    coords, vals = synth.generate(cfg)
    for label, approx, sparse in (("P-Tucker", 0, 0), ("Approx dense", 1, 0), ("Approx sparse", 1, -1)):
        pt.ptucker_finalize()
        pt.ptucker_set_option("seg_len", 256)
        pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * N, cfg.lam, 0)
        pt.ptucker_set_stream(stream.cuda_stream)
        pt.ptucker_set_option("sparse_core", sparse)
        pt.ptucker_set_option("graph", 0)
        sweeps, scores = [], []
        for _ in range(iters):
            sweeps.append(timed(pt.ptucker_sweep))
            pt.ptucker_error()
            if approx:
                scores.append(timed(lambda: pt.ptucker_truncate_core(0.2)))
        print(f"order {N} {label:14s} sweep ms per iteration: " + " ".join(f"{x:.3f}" for x in sweeps) +
              (f" | scores+truncation ms: " + " ".join(f"{x:.3f}" for x in scores) if scores else "") +
              f" | core nnz {pt.ptucker_core_nnz()}", flush=True)
