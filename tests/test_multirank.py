"""World-size-2 gloo tests of the multi-GPU plumbing (CPU): batch sharding is
a partition of the global batch with the same signal bytes as one rank would
generate, and the filter broadcast delivers rank 0's buffers bit-exactly.
The device path (NCCL over NVLink) uses the same functions (bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_12718_b200 import dist as pdist
        from paper_2506_12718_b200 import workload
        import oracle

        cfg = workload.Config(0, "t", 3, [243], 4, "uniform", "cnormal")
        first, per = pdist.shard(cfg.batch, rank)
        mine = workload.signals(cfg, first, per)
        # filter: rank 0 prepares (oracle on CPU stands in for the device), others receive
        n = cfg.total
        if rank == 0:
            O = oracle.Oracle()
            op = O.plan(cfg.radix, cfg.dims)
            ghat = op.prepare_filter(op.filter_from_impulse(workload.impulse(cfg)))
            buf = torch.from_numpy(ghat.view(np.float64).copy())
            kern = torch.from_numpy((ghat / n).view(np.float64).copy())
        else:
            buf = torch.zeros(2 * n, dtype=torch.float64)
            kern = torch.zeros(2 * n, dtype=torch.float64)
        pdist.broadcast_filter_tensors([buf, kern])
        t = pdist.max_over_ranks(1.0 + rank)
        gathered = [torch.zeros(per * n * 2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(mine.view(np.float64).reshape(-1).copy()))
        out[rank] = (buf.numpy().copy(), kern.numpy().copy(), t,
                     [g.numpy().copy() for g in gathered], first, per)
    finally:
        dist.destroy_process_group()


def test_sharding_and_filter_broadcast_gloo():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    from paper_2506_12718_b200 import workload
    cfg = workload.Config(0, "t", 3, [243], 4, "uniform", "cnormal")
    r0, r1 = out[0], out[1]
    assert np.array_equal(r0[0], r1[0]) and np.array_equal(r0[1], r1[1])
    assert r0[2] == r1[2] == 2.0                      # max over ranks
    assert (r0[4], r0[5], r1[4], r1[5]) == (0, 4, 4, 4)  # fixed per-rank batch
    whole = workload.signals(cfg, 0, 8).view(np.float64).reshape(2, -1)
    assert np.array_equal(r0[3][0], whole[0]) and np.array_equal(r0[3][1], whole[1])
