"""One rank of the two-process push-exchange test (tests/test_gpu_push.py): both ranks
run on the same GPU as separate processes with no NCCL communicator (emulate_world),
open each other's replicas by CUDA IPC and push their solved rows; the ranks are ordered
by a host barrier (gloo) between modes -- no kernel of one rank waits on the other.

    python tests/push_worker.py RANK WORLD PORT CONFIG SCALE SWEEPS OUT.npz
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    rank, world, port = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    name, scale, sweeps, out = sys.argv[4], float(sys.argv[5]), int(sys.argv[6]), sys.argv[7]
    import torch
    import torch.distributed as dist
    from gen import synth
    from paper_1710_02261_b200 import ptucker as pt
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    cfg = synth.small(name, scale)
    coords, vals = synth.generate(cfg)
    N = len(cfg.dims)
    pt.ptucker_set_option("seg_len", -1)
    pt.ptucker_set_option("emulate_world", world)
    pt.ptucker_set_option("emulate_rank", rank)
    pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * N, cfg.lam, 0)
    hs = [None] * world
    dist.all_gather_object(hs, pt.ptucker_peer_handles())
    pt.ptucker_open_peers(b"".join(hs), world)
    info = pt.ptucker_info()
    assert info["exchange"] == "push" and info["peers"] == world - 1, info
    dist.barrier()
    sse = []
    for _ in range(sweeps):
        for n in range(N):
            pt.ptucker_update_mode(n)
            pt.ptucker_synchronize()
            dist.barrier()          # every rank's pushes of mode n landed before mode n + 1
        sse.append(pt.ptucker_error() ** 2)
    np.savez(out, *[pt.ptucker_get_factor(n) for n in range(N)], sse=np.array(sse),
             bounds=np.stack([pt.ptucker_get_partition(n) for n in range(N)]))
    dist.barrier()
    pt.ptucker_finalize()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
