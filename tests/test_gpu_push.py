"""S5 (replica refresh, Fig. 3 caption P:517-518) through the library's multi-GPU push
exchange: the ranks are processes on ONE GPU (tests/push_worker.py), each updating its
nnz-balanced row block and storing every solved row into the other ranks' replicas
(CUDA IPC, ptucker_open_peers); host barriers order the modes.  After full sweeps
every rank holds the whole factors, bit-identical to a single-rank run (rows are
independent), and the per-rank SSE partials add up to the single-rank error.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from gen import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name,scale,world", [("c5", 0.0005, 2), ("c3", 0.005, 2), ("c2", 0.01, 3),
                                                   ("c4", 0.001, 2)])
def test_push_exchange_bit_identical(tmp_path, name, scale, world):
    import torch
    assert torch.cuda.is_available()
    from paper_1710_02261_b200 import build, ptucker as pt
    build.build()
    sweeps = 2
    cfg = synth.small(name, scale)
    coords, vals = synth.generate(cfg)
    N = len(cfg.dims)
    pt.ptucker_finalize()
    pt.ptucker_set_option("seg_len", -1)      # the workers' (default) automatic S
    pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * N, cfg.lam, 0)
    for _ in range(sweeps):
        pt.ptucker_sweep()
    ref = [pt.ptucker_get_factor(n).copy() for n in range(N)]
    e_ref = pt.ptucker_error()
    pt.ptucker_finalize()
    port = _port()
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "push_worker.py"), str(r), str(world),
                               str(port), name, str(scale), str(sweeps), str(tmp_path / f"r{r}.npz")],
                              cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(world)]
    outs = [p.communicate(timeout=600)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), "\n".join(o[-3000:] for o in outs)
    sse = 0.0
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        b = d["bounds"]
        assert b.shape == (N, world + 1) and np.all(b[:, -1] == np.array(cfg.dims))
        for n in range(N):
            assert np.array_equal(d[f"arr_{n}"], ref[n]), (r, n)   # the whole replica, not only the own block
        sse += float(d["sse"][-1])
    assert abs(np.sqrt(sse) - e_ref) <= 1e-9 * e_ref
