"""World-size-2 gloo tests of the multi-GPU plumbing (CPU): batch sharding is
a partition of the FIXED global batch (batch / G per rank)
with the same signal bytes as one rank would generate, and the filter
broadcast delivers rank 0's buffers bit-exactly.  The device path (NCCL over
NVLink) uses the same functions (bench.py)."""
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

        cfg = workload.Config(0, "t", 3, [243], 5, "uniform", "cnormal")
        first, per = pdist.shard(cfg.batch, world, rank)
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
        gathered = [None] * world
        dist.all_gather_object(gathered, (first, mine.copy()))
        out[rank] = (buf.numpy().copy(), kern.numpy().copy(), t, gathered, first, per)
    finally:
        dist.destroy_process_group()


def test_sharding_and_filter_broadcast_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    for attempt in range(3):
        # the free port found here can be taken again before gloo binds it: try another one
        try:
            mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
            break
        except Exception as e:
            if attempt == 2 or not ("EADDRINUSE" in str(e) or "address already in use" in str(e).lower()):
                raise
    from paper_2506_12718_b200 import workload
    cfg = workload.Config(0, "t", 3, [243], 5, "uniform", "cnormal")
    r0, r1 = out[0], out[1]
    assert np.array_equal(r0[0], r1[0]) and np.array_equal(r0[1], r1[1])
    assert r0[2] == r1[2] == 2.0                      # max over ranks
    assert (r0[4], r0[5], r1[4], r1[5]) == (0, 3, 3, 2)  # global batch 5 split 3 + 2
    # the shards, concatenated in rank order, are the global batch exactly once
    whole = workload.signals(cfg, 0, cfg.batch)
    got = np.concatenate([m for _, m in sorted(r0[3], key=lambda fm: fm[0])])
    assert np.array_equal(got, whole)


@pytest.mark.parametrize("batch", [0, 1, 3, 8, 16, 64, 4096, 4097])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_partitions_the_global_batch(batch, world):
    from paper_2506_12718_b200 import dist as pdist
    owner = np.full(batch, -1)
    counts = []
    for r in range(world):
        first, cnt = pdist.shard(batch, world, r)
        counts.append(cnt)
        assert (owner[first:first + cnt] == -1).all()
        owner[first:first + cnt] = r
    assert (owner >= 0).all()                    # covered exactly once
    assert sum(counts) == batch and max(counts) - min(counts) <= 1
    assert list(owner) == sorted(owner)         # contiguous, rank order


def test_baseline_partitions_and_bytes():
    """config 2 64/G, config 3 16/G, config 4 8/G (one volume per
    GPU at 8), config 5 4096/G (512 at 8); config 1 runs replicas."""
    from paper_2506_12718_b200 import dist as pdist
    from paper_2506_12718_b200 import workload
    for idx, per8 in [(2, 8), (3, 2), (4, 1), (5, 512)]:
        cfg = workload.get_config(idx)
        assert pdist.shard(cfg.batch, 8, 7)[1] == per8
        assert workload.shard_count(cfg, 8) == per8
        S = workload.signal_bytes(cfg)
        assert workload.bytes_per_conv(cfg, 8) == 2 * S + S / per8
        assert workload.bytes_per_conv(cfg, 8, weak=True) == 2 * S + S / cfg.batch
    c1 = workload.get_config(1)
    assert workload.shard_count(c1, 8) == 100   # replicas: the 100-call sequence per GPU
    with pytest.raises(ValueError):
        pdist.shard(4, 2, 2)
