"""Multi-rank parity worker (launched by tests/test_gpu_multirank.py under torchrun).

Every rank syncs its shards of L units through the C ABI (NCCL comms of the M x N mesh).
Rank 0 regenerates every rank's seeded inputs (synth/, same Philox streams), runs the fp64
oracle for the whole mesh, gathers all ranks' outputs and compares; all ranks check the
cross-rank invariants (identical anchors along a sync row, local == rne(anchor) bitwise).

usage: torchrun --nproc-per-node K tests/mp_parity_worker.py MxN dtype config [peer|nccl]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2412_07210_b200 import EditSync, broadcast_unique_id  # noqa: E402
from tests import parity  # noqa: E402


def inputs_of(units, M, m, n, dtype, dev, plant, recipe, salt=0):
    anc = [synth.shard_anchor(u, i, M, m, dev, recipe) for i, u in enumerate(units)]
    mom = [synth.shard_momentum(u, i, M, m, dev, recipe) for i, u in enumerate(units)]
    loc = [synth.shard_local(u, i, M, m, n, anc[i], dtype, dev, recipe, plant.get((i, n), 1.0), salt)
           for i, u in enumerate(units)]
    return loc, anc, mom


def grad_of(u, i, M, m, n, dtype, dev):
    # a seeded per-rank gradient shard (kind 5), zero in the padded tail
    numel = synth.shard_numel(u.numel, M)
    g = synth._randn(numel, synth.seed_of(5, i, m, n), dev).mul_(1e-3)
    g[max(0, min(numel, u.numel - m * numel)):] = 0
    return g.to(dtype)


def warm_check(units, M, N, m_idx, n_idx, rank, world, dtype, dtype_s, dev, s, mesh, algo, local_rank):
    """Warm-up gradient all-reduce (Alg. 1 l.422-424) vs the oracle's mean over the sync row.
    algo "peer" exercises the peer-memory variant (EDIT_WARMUP_ALGO=peer), "nccl" the default."""
    os.environ["EDIT_WARMUP_ALGO"] = "peer" if algo == "peer" else "nccl"
    grads = [grad_of(u, i, M, m_idx, n_idx, dtype, dev) for i, u in enumerate(units)]
    for i in range(len(units)):
        s.warmup_allreduce(i, grads[i])
    torch.cuda.synchronize()
    mine = {"rank": rank, "g": [parity.to_oracle_local(g) for g in grads]}
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(mine, gathered, dst=0)
    if rank == 0:
        by_rank = {g["rank"]: g for g in gathered}
        for i, u in enumerate(units):
            for m in range(M):
                inp = np.stack([parity.to_oracle_local(grad_of(u, i, M, m, n, dtype, dev)) for n in range(N)])
                ref = oracle.allreduce_mean(inp)
                for n in range(N):
                    r = n * M + m
                    got = by_rank[r]["g"][i]
                    parity.assert_local_close(got, ref, f"warm {mesh} unit {i} rank {r}")
                    assert np.array_equal(got, by_rank[m]["g"][i]), "sync row members differ"
        print(f"PARITY OK warm {mesh} {dtype_s} {algo} unit: {len(units)} units", flush=True)
    s.close()
    dist.barrier(device_ids=[local_rank])
    return 0


def run_case(mesh, dtype_s, config, algo="peer", api="unit"):
    # api -- unit: edit_layer_sync x L; round: edit_sync_round; reg: registered locals + round;
    # gather: fused shard all-gather + round; sched: prefetch scheduler (depth 1);
    # schedpart: registered locals + scheduler in partition mode (8 CTAs, unit 0 full grid);
    # graph: EDIT_GRAPH=1 round captured into a CUDA graph, the checked round is a replay
    M, N = (int(x) for x in mesh.split("x"))
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    assert world == M * N
    local_rank = int(os.environ["LOCAL_RANK"])
    dev = torch.device("cuda", local_rank)
    m_idx, n_idx = rank % M, rank // M
    dtype = torch.bfloat16 if dtype_s == "bf16" else torch.float32
    recipe = synth.Recipe()
    cfg = oracle.Config()
    plant = {}
    seed_ema = True
    if config == "toy":
        # BASELINE configs[0]: 4 layers x 64K fp32 params, replica 1 planted (x4) in every unit
        units = synth.toy_units(4, 65536)
        plant = {(i, 1): 4.0 for i in range(4)} if N > 1 else {}
    elif config == "toy_clip":
        units = synth.toy_units(4, 65536)
        cfg = oracle.Config(clip_threshold=0.3)
    elif config == "ragged":
        units = [synth.Unit("a", 1_000_003, ((999_000, 1003),)), synth.Unit("b", 7, ()),
                 synth.Unit("c", 3 * 65536 + 5, ())]
        seed_ema = False
    elif config == "rollback":
        units = synth.toy_units(2, 40_000)
        plant = {(i, n): 4.0 for i in range(2) for n in range(N)}       # every replica anomalous
    elif config == "nan":
        units = [synth.Unit("a", 300_001, ()), synth.Unit("b", 9, ())]
        seed_ema = False
    elif config == "warm":
        units = [synth.Unit("a", 1_000_003, ()), synth.Unit("b", 13, ()), synth.Unit("c", 65_536, ())]
        seed_ema = False
    elif config == "many_small":
        # 20 small units: the round API syncs them as two unit groups (kMaxGroup = 16); a planted
        # replica in unit 3, every replica planted (rollback) in unit 5
        sizes = [7, 65539, 1000, 300_001, 8, 123_457, 4096, 77_777]
        units = [synth.Unit(f"s{i}", sizes[i % 8] + i, ()) for i in range(20)]
        plant = {(3, 1): 4.0, **{(5, n): 4.0 for n in range(N)}}
    elif config == "llama350m_sample":
        all_units = synth.llama_units("350M")
        units = [all_units[0], all_units[1], all_units[33]]
    else:
        raise SystemExit(f"unknown config {config}")
    numel = [synth.shard_numel(u.numel, M) for u in units]
    uid = broadcast_unique_id()
    if api == "graph":
        os.environ["EDIT_GRAPH"] = "1"   # read at init: device-side mailbox sequence numbers
    s = EditSync(numel, shard_dim=M, sync_dim=N, rank=rank, device=dev, param_dtype=dtype,
                 outer_lr=cfg.outer_lr, outer_momentum=cfg.outer_momentum, clip_threshold=cfg.clip_threshold,
                 clip_eps=cfg.clip_eps, anomaly_threshold=cfg.anomaly_threshold, ema_alpha=cfg.ema_alpha,
                 ema_warmup_rounds=cfg.ema_warmup_rounds, flags=cfg.flags, unique_id=uid, algo=algo)
    os.environ.pop("EDIT_GRAPH", None)
    ema0 = [[oracle.Ema() for _ in range(N)] for _ in units]
    if seed_ema:
        mu = np.array([[synth.ema_seed(u, n, recipe)[0] for n in range(N)] for u in units])
        s.set_ema(mu, 0.1 * mu, recipe.ema_warmup_rounds)
        ema0 = [[oracle.Ema(mu[i, n], 0.1 * mu[i, n], recipe.ema_warmup_rounds) for n in range(N)]
                for i in range(len(units))]

    if config == "warm":
        return warm_check(units, M, N, m_idx, n_idx, rank, world, dtype, dtype_s, dev, s, mesh, algo, local_rank)
    loc, anc, mom = inputs_of(units, M, m_idx, n_idx, dtype, dev, plant, recipe)
    guards = []
    if config == "ragged":
        # guard zones around every buffer: no kernel (local or peer) may write outside a shard
        G = 64
        for lst in (loc, anc, mom):
            for i, t in enumerate(lst):
                big = torch.full((t.numel() + 2 * G,), 7.25, dtype=t.dtype, device=dev)
                big[G:G + t.numel()].copy_(t)
                guards.append((big, G, t.numel()))
                lst[i] = big[G:G + t.numel()]
    if config == "nan" and n_idx == N - 1:
        loc[0][1234 % loc[0].numel()] = float("nan")   # replica N-1 has a NaN param (R9)
    full = None
    if api == "gather":                # NEXT-2: fused write-back -> shard-group all-gather
        full = [torch.zeros(M * n_, dtype=dtype, device=dev) for n_ in numel]
        s.register_gather(full)
    if api in ("sched", "schedpart"):  # a8 prefetch scheduler; schedpart: partition mode
        if api == "schedpart":
            s.register_locals(loc)
            s.set_partition(8, 1)
        stream = torch.cuda.current_stream(dev)
        s.begin_round(loc, anc, mom, 1, stream)
        for i in range(len(units)):
            s.acquire(i, stream)
        s.end_round(stream)
    elif api == "graph":               # EDIT_GRAPH=1: captured round, then a REPLAY is checked
        saved = [x.clone() for x in loc + anc + mom]
        state0 = s.get_state()
        s.sync_round(loc, anc, mom)    # capture + first launch (results discarded)
        torch.cuda.synchronize()
        for x, y in zip(loc + anc + mom, saved):
            x.copy_(y)                 # same buffers -> the next call replays the graph
        s.set_state(state0)
        s.sync_round(loc, anc, mom)
    elif api in ("round", "reg", "gather"):
        if api == "reg":
            s.register_locals(loc)     # peer path reads the members' locals directly
        s.sync_round(loc, anc, mom)
    else:
        for i in range(len(units)):
            s.layer_sync(i, loc[i], anc[i], mom[i])
    torch.cuda.synchronize()
    mine = {"rank": rank, "loc": [parity.to_oracle_local(x) for x in loc],
            "anc": [x.cpu().numpy() for x in anc], "mom": [x.cpu().numpy() for x in mom],
            "stats": [s.stats(i) for i in range(len(units))],
            "ema": s.get_state(),
            "full": [parity.to_oracle_local(f) for f in full] if full is not None else None}
    for big, G, n_ in guards:
        assert (big[:G] == 7.25).all() and (big[G + n_:] == 7.25).all(), f"rank {rank}: write outside a shard"
    # invariant: local == rne(anchor) bitwise on every rank (R16)
    for i in range(len(units)):
        assert torch.equal(loc[i], anc[i].to(dtype)), f"rank {rank} unit {i}: local != rne(anchor)"
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(mine, gathered, dst=0)
    ok = True
    if rank == 0:
        by_rank = {g["rank"]: g for g in gathered}
        # R6: every rank keeps all N replicas' EMA and updates them identically
        for r in range(world):
            assert np.array_equal(by_rank[r]["ema"], by_rank[0]["ema"]), f"EMA state of rank {r} differs"
        for i, u in enumerate(units):
            # regenerate every rank's inputs for unit i (seeded, rank-independent)
            locs, ancs, moms = [], [], []
            for m in range(M):
                a = synth.shard_anchor(u, i, M, m, dev, recipe)
                ancs.append(a.cpu().numpy())
                moms.append(synth.shard_momentum(u, i, M, m, dev, recipe).cpu().numpy())
                row = []
                for n in range(N):
                    l = synth.shard_local(u, i, M, m, n, a, dtype, dev, recipe, plant.get((i, n), 1.0))
                    if config == "nan" and n == N - 1 and i == 0:
                        l[1234 % l.numel()] = float("nan")
                    row.append(parity.to_oracle_local(l))
                locs.append(row)
            o_loc, o_anc, o_mom, o_ema, out = oracle.sync_unit(cfg, np.array(locs), np.stack(ancs), np.stack(moms),
                                                               ema0[i])
            for r in range(world):
                m, n = r % M, r // M
                g = by_rank[r]
                tag = f"{config} {mesh} unit {i} rank {r} (m={m}, n={n})"
                parity.assert_outcome(g["stats"][i], out, o_ema, tag)
                parity.assert_f32_close(g["anc"][i], o_anc[m], tag + " anchor")
                parity.assert_f32_close(g["mom"][i], o_mom[m], tag + " momentum")
                parity.assert_local_close(g["loc"][i], o_loc[m, n], tag + " local")
                # sync-row identity: bitwise identical anchors across the N replicas of shard m
                g0 = by_rank[m]
                assert np.array_equal(g["anc"][i], g0["anc"][i]), tag + " anchors differ across the sync row"
            if api == "gather" and M > 1:
                # every rank's gathered module == its shard group's new locals, bitwise
                for r in range(world):
                    m, n = r % M, r // M
                    f = by_rank[r]["full"][i]
                    nl = numel[i]
                    for q in range(M):
                        assert np.array_equal(f[q * nl:(q + 1) * nl], by_rank[n * M + q]["loc"][i]), \
                            f"gathered module of rank {r}, shard {q}, unit {i}"
            if config == "toy" and N > 1:
                assert out.anomalous[1] and not out.rollback
            if config == "rollback":
                assert out.rollback
            if config == "toy_clip":
                assert out.beta < 1.0
            if config == "nan" and i == 0:
                # the replica with a NaN param is excluded; alone (N == 1) that is a rollback
                assert out.anomalous[N - 1] and out.rollback == (N == 1)
        print(f"PARITY OK {config} {mesh} {dtype_s} {algo} {api}: {len(units)} units", flush=True)
    s.close()
    dist.barrier(device_ids=[local_rank])
    return 0 if ok else 1


def main():
    # usage: worker.py MESH dtype:config:algo:api [dtype:config:algo:api ...]
    #    or: worker.py MESH dtype config [algo [api]]        (one case)
    mesh = sys.argv[1]
    if len(sys.argv) > 2 and ":" in sys.argv[2]:
        cases = [a.split(":") for a in sys.argv[2:]]
    else:
        cases = [sys.argv[2:]]
    local_rank = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local_rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    rc = 0
    for c in cases:
        rc |= run_case(mesh, *c)
    dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
