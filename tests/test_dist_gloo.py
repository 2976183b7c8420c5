"""Multi-process host logic on CPU (gloo, world_size 2): NCCL unique-id broadcast, the
max-over-ranks timing rule, the rank <-> mesh mapping (R20) and shard reconstruction of the
seeded inputs (all_gather(shard_layer(x)) == x)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import synth
        from paper_2412_07210_b200 import broadcast_unique_id
        uid = broadcast_unique_id()
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        # max over ranks: each rank reports a different time
        t = bench.max_over_ranks(10.0 + rank, world, torch.device("cpu"))
        # mesh 2x1 (M=2 shards) and 1x2 (N=2 replicas): shards of one unit reassemble
        recon = {}
        for M in (1, 2):
            m, n = bench.rank_coords(rank, M)
            u = synth.Unit("u", 1001, ((990, 11),))
            a = synth.shard_anchor(u, 3, M, m, torch.device("cpu"))
            parts = [None] * world
            dist.all_gather_object(parts, (m, n, a))
            recon[M] = parts
        out[rank] = dict(ids=ids, t=t, recon=recon)
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_host_logic():
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    r0, r1 = out[0], out[1]
    assert r0["ids"][0] == r0["ids"][1] == r1["ids"][0] and len(r0["ids"][0]) == 128
    assert r0["t"] == r1["t"] == 11.0
    import synth
    u = synth.Unit("u", 1001, ((990, 11),))
    # M = 2: rank r holds shard m = r; concatenated and unpadded == the M = 1 shard
    parts = sorted(r0["recon"][2], key=lambda p: p[0])
    assert [p[0] for p in parts] == [0, 1] and [p[1] for p in parts] == [0, 0]
    full = torch.cat([p[2] for p in parts])[:1001]
    assert parts[1][2][1001 - 501:].abs().sum() == 0          # zero-padded tail
    # M = 1, N = 2: both replicas hold the identical anchor (kinds 0-2 use n = 0)
    p1 = r0["recon"][1]
    assert [p[1] for p in p1] == [0, 1] and torch.equal(p1[0][2], p1[1][2])
    # the norm segment (1 + N(0, 0.02^2)) sits at the same flat offsets in both layouts
    assert (full[990:1001] > 0.5).all() and (p1[0][2][990:1001] > 0.5).all()
