"""The N>1 path's host logic on CPU with world-size-2 `gloo` (no GPU needed):
rows of each mode split by the library's ptucker_partition_rows (the same function
ptucker_init uses for its row blocks), each rank updating only its block with the
oracle, the blocks exchanged (the all-gather the library does with NCCL), the SSE
partials all-reduced -- and the result must equal the single-process sweep bit for
bit (rows are independent).  Also the NCCL unique-id bootstrap
bytes travel through torch.distributed unchanged."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from gen import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        from paper_1710_02261_b200 import ptucker as pt
        pt.load()
        cfg = synth.small("c3", 0.002)
        coords, vals = synth.generate(cfg)
        t = orc.Tensor(coords, vals, cfg.dims)
        N, J = len(cfg.dims), cfg.J
        m = orc.init_model(cfg.dims, [J] * N, seed=0, prec=0)
        sse_total = None
        for n in range(N):
            row_ptr, perm = t.mode_index(n)
            b = pt.ptucker_partition_rows(row_ptr, world)
            r0, r1 = int(b[rank]), int(b[rank + 1])
            before = m.A(n).copy()
            for i in range(r0, r1):
                orc.update_row(t, m, n, i, cfg.lam)
            mine = torch.from_numpy(m.A(n)[r0:r1].copy())
            # all-gather-v of the row blocks
            sizes = [int(b[g + 1] - b[g]) for g in range(world)]
            maxr = max(sizes)
            padded = torch.zeros((maxr, J), dtype=torch.float64)
            padded[: r1 - r0] = mine
            bufs = [torch.zeros_like(padded) for _ in range(world)]
            dist.all_gather(bufs, padded)
            full = torch.cat([bufs[g][: sizes[g]] for g in range(world)]).numpy()
            # rows outside this rank's block were untouched locally
            assert np.array_equal(m.A(n)[:r0], before[:r0]) and np.array_equal(m.A(n)[r1:], before[r1:])
            m.A(n)[:] = full
            if n == N - 1:
                # error: per-row SSE identity over this rank's rows, all-reduced
                local = 0.0
                for i in range(r0, r1):
                    B, c, s2 = orc.row_system(t, m, n, i)
                    a = m.A(n)[i]
                    local += s2 - a @ c - cfg.lam * a @ a
                s = torch.tensor([local], dtype=torch.float64)
                dist.all_reduce(s)
                sse_total = float(s[0])
        # NCCL unique id bytes through torch.distributed (rank 0 creates them)
        obj = [pt.ptucker_get_unique_id() if rank == 0 else None]
        try:
            dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        except Exception as e:  # NCCL may be unable to create an id without a GPU/network
            uid = repr(e)
        if rank == 0:
            q.put(("r0", m.A_all.copy(), sse_total, uid))
        else:
            q.put(("r1", uid))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_rank_sweep_matches_single_process(orc):
    from paper_1710_02261_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0 = [o for o in out if o[0] == "r0"][0]
    r1 = [o for o in out if o[0] == "r1"][0]
    _, A_dist, sse_dist, uid0 = r0
    assert uid0 == r1[1]                      # both ranks hold the same bootstrap bytes
    # single-process reference sweep
    cfg = synth.small("c3", 0.002)
    coords, vals = synth.generate(cfg)
    t = orc.Tensor(coords, vals, cfg.dims)
    m = orc.init_model(cfg.dims, [cfg.J] * 4, seed=0, prec=0)
    for n in range(4):
        orc.update_mode(t, m, n, cfg.lam)
    assert np.array_equal(A_dist, m.A_all)    # bit-identical (F9)
    sse = orc.sse(t, m)
    assert abs(sse_dist - sse) <= 1e-9 * sse
