"""Small end-to-end run for compute-sanitizer (one tool per gpurun call, B200_PROFILING.md):
init, two sweeps, the fused and literal errors, Approx scores + truncation and the final
QR on c1 (fp64 ALU kernel), c3 at 0.002 (order 4: SMP tables, heavy rows) and c5 at 1e-4
(tensor-core kernel).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [configs]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from gen import synth  # noqa: E402
from paper_1710_02261_b200 import ptucker as pt  # noqa: E402

torch.cuda.set_device(0)
names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c1", "c3@0.002", "c5@0.0001"]
for spec in names:
    name, _, sc = spec.partition("@")
    cfg = synth.config(name) if not sc else synth.small(name, float(sc))
    coords, vals = synth.generate(cfg)
    N = len(cfg.dims)
    pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * N, cfg.lam, 0)
    for _ in range(2):
        pt.ptucker_sweep()
    e = pt.ptucker_error()
    el = pt.ptucker_error_literal()
    pt.ptucker_truncate_core(0.2)
    pt.ptucker_sweep()
    pt.ptucker_orthogonalize()
    e2 = pt.ptucker_error()
    pt.ptucker_finalize()
    print(f"{spec}: error {e:.6g} (literal {el:.6g}), after Approx + QR {e2:.6g}", flush=True)
print("sanitize run done")
