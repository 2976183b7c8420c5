"""A-EDiT with real ranks (§3.3), launched by
tests/test_gpu_aedit.py under torchrun.

Every rank runs whole "inner steps" of a different length (a sleep kernel: rank r takes
base x (1 + 1.5 r / (K-1)) ms per step), asks its own time trigger (Trigger.time, the
library's edit_trigger_*) at every step boundary, and enters the collective sync
(edit_sync_round through the C ABI) once its own time since the last sync reaches tau_time.
Ranks therefore complete DIFFERENT numbers of inner steps per round; the early ones wait
inside the sync's first exchange.  Measured per rank and round: the wait = (the last rank's
arrival) - (own arrival) on the node's monotonic clock, and the device time of the round.
Checked: the paper's bound "no worker will wait longer than the single step time of the
slowest worker", and oracle parity of the first round's sync (rank 0 regenerates
every rank's inputs from the gathered step counts) plus the cross-rank invariants every round.

usage: worker.py MESH ROUNDS OUT_JSON
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2412_07210_b200 import EditSync, Trigger, broadcast_unique_id  # noqa: E402
from tests import parity  # noqa: E402

BASE_STEP_MS = 20.0
TAU_TIME_S = 0.4


def main():
    mesh, rounds, out_path = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    M, N = (int(x) for x in mesh.split("x"))
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local_rank = int(os.environ["LOCAL_RANK"])
    assert world == M * N
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist.init_process_group("nccl", device_id=dev)
    m_idx, n_idx = rank % M, rank // M
    dtype = torch.bfloat16
    recipe = synth.Recipe()
    units = [synth.Unit("a", 2_000_003, ()), synth.Unit("b", 65_536, ()), synth.Unit("c", 1_000_000, ((999_000, 1000),))]
    numel = [synth.shard_numel(u.numel, M) for u in units]
    cfg = oracle.Config()
    s = EditSync(numel, shard_dim=M, sync_dim=N, rank=rank, device=dev, param_dtype=dtype,
                 unique_id=broadcast_unique_id())
    mu = np.array([[synth.ema_seed(u, n, recipe)[0] for n in range(N)] for u in units])
    s.set_ema(mu, 0.1 * mu, recipe.ema_warmup_rounds)
    ema0 = [[oracle.Ema(mu[i, n], 0.1 * mu[i, n], recipe.ema_warmup_rounds) for n in range(N)]
            for i in range(len(units))]
    anc = [synth.shard_anchor(u, i, M, m_idx, dev, recipe) for i, u in enumerate(units)]
    mom = [synth.shard_momentum(u, i, M, m_idx, dev, recipe) for i, u in enumerate(units)]
    loc = [torch.empty(n_, dtype=dtype, device=dev) for n_ in numel]

    # calibrate the sleep kernel: cycles per ms on this GPU
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    torch.cuda._sleep(20_000_000)
    torch.cuda.synchronize()
    cyc_per_ms = 20_000_000 / ((time.perf_counter() - t0) * 1e3)
    step_ms = BASE_STEP_MS * (1.0 + 1.5 * rank / max(1, world - 1))

    def inner_step():
        torch.cuda._sleep(int(step_ms * cyc_per_ms))

    # the sync alone (every rank arrives together): reference for the device time of a round
    alone = []
    for r in range(4):
        for i, u in enumerate(units):
            loc[i].copy_(synth.shard_local(u, i, M, m_idx, n_idx, anc[i], dtype, dev, recipe, 1.0, 9000 + r))
        saved = ([a.clone() for a in anc], [x.clone() for x in mom], s.get_state())
        dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.sync_round(loc, anc, mom)
        e1.record()
        torch.cuda.synchronize()
        if r > 0:
            alone.append(e0.elapsed_time(e1))
        for a, b in zip(anc, saved[0]):
            a.copy_(b)
        for a, b in zip(mom, saved[1]):
            a.copy_(b)
        s.set_state(saved[2])

    dist.barrier(device_ids=[local_rank])
    t_start = time.perf_counter()   # CLOCK_MONOTONIC: comparable across the node's processes
    trig = Trigger.time(TAU_TIME_S, 0, 0.0)
    step = 0
    recs = []
    for rnd in range(rounds):
        steps = 0
        while not trig.sync_now(step + 1, time.perf_counter() - t_start):
            inner_step()
            torch.cuda.synchronize()   # a whole step: the trigger is asked only at step boundaries
            step += 1
            steps += 1
        # the local after `steps` inner steps of this round (seeded by the step count)
        for i, u in enumerate(units):
            loc[i].copy_(synth.shard_local(u, i, M, m_idx, n_idx, anc[i], dtype, dev, recipe, 1.0,
                                           1000 * (rnd + 1) + steps))
        torch.cuda.synchronize()
        arrive = time.perf_counter() - t_start
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.sync_round(loc, anc, mom)
        e1.record()
        torch.cuda.synchronize()
        release = time.perf_counter() - t_start
        trig.mark_synced(release)
        recs.append({"round": rnd, "steps": steps, "arrive_s": arrive, "release_s": release,
                     "device_round_ms": e0.elapsed_time(e1)})
        # invariants every round: local == rne(anchor)
        for i in range(len(units)):
            assert torch.equal(loc[i], anc[i].to(dtype)), f"rank {rank} round {rnd} unit {i}"
        if rnd == 0:
            first = {"loc_in_steps": steps, "anc": [a.cpu().numpy() for a in anc], "mom": [x.cpu().numpy() for x in mom],
                     "loc": [parity.to_oracle_local(x) for x in loc], "stats": [s.stats(i) for i in range(len(units))]}
    mine = {"rank": rank, "step_ms": step_ms, "recs": recs, "first": first, "alone_ms": alone,
            "anc_last": [a.cpu().numpy() for a in anc]}
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(mine, gathered, dst=0)
    rc = 0
    if rank == 0:
        by = {g["rank"]: g for g in gathered}
        slowest_step = max(g["step_ms"] for g in gathered)
        t_alone = float(np.median([t for g in gathered for t in g["alone_ms"]]))
        rounds_out = []
        for rnd in range(rounds):
            arr = [by[r]["recs"][rnd]["arrive_s"] for r in range(world)]
            last = max(arr)
            waits = [1e3 * (last - a) for a in arr]
            dev_ms = [by[r]["recs"][rnd]["device_round_ms"] for r in range(world)]
            steps = [by[r]["recs"][rnd]["steps"] for r in range(world)]
            rounds_out.append({"round": rnd, "steps_per_rank": steps, "wait_ms_per_rank": waits,
                               "device_round_ms_per_rank": dev_ms, "max_wait_ms": max(waits),
                               "bound_ms": slowest_step})
            # no worker waits longer than one step of the slowest worker (host-clock
            # arrival differences; 2 ms allowance for the host-side step bookkeeping)
            assert max(waits) <= slowest_step + 2.0, (rnd, waits, slowest_step)
            # the early ranks' wait is spent inside the sync (device time ~ wait + round alone)
            for r in range(world):
                assert dev_ms[r] <= waits[r] + t_alone + 5.0 + 0.5 * t_alone, (rnd, r, dev_ms[r], waits[r], t_alone)
            # anchors identical along each sync row every round
        for r in range(world):
            m = r % M
            for i in range(len(units)):
                assert np.array_equal(by[r]["anc_last"][i], by[m]["anc_last"][i]), f"row anchors differ, rank {r}"
        # oracle parity of round 0 (ranks had completed different numbers of inner steps)
        for i, u in enumerate(units):
            locs, ancs, moms = [], [], []
            for m in range(M):
                a = synth.shard_anchor(u, i, M, m, dev, recipe)   # the seeded initial anchor of shard m
                ancs.append(a.cpu().numpy())
                moms.append(synth.shard_momentum(u, i, M, m, dev, recipe).cpu().numpy())
                row = []
                for n in range(N):
                    st = by[n * M + m]["recs"][0]["steps"]
                    l = synth.shard_local(u, i, M, m, n, a, dtype, dev, recipe, 1.0, 1000 + st)
                    row.append(parity.to_oracle_local(l))
                locs.append(row)
            o_loc, o_anc, o_mom, o_ema, out = oracle.sync_unit(cfg, np.array(locs), np.stack(ancs), np.stack(moms),
                                                               ema0[i])
            for r in range(world):
                m, n = r % M, r // M
                f = by[r]["first"]
                tag = f"A-EDiT round 0 unit {i} rank {r}"
                parity.assert_outcome(f["stats"][i], out, o_ema, tag)
                parity.assert_f32_close(f["anc"][i], o_anc[m], tag + " anchor")
                parity.assert_f32_close(f["mom"][i], o_mom[m], tag + " momentum")
                parity.assert_local_close(f["loc"][i], o_loc[m, n], tag + " local")
        res = {"mesh": mesh, "tau_time_s": TAU_TIME_S, "step_ms_per_rank": [by[r]["step_ms"] for r in range(world)],
               "t_round_alone_ms": t_alone, "rounds": rounds_out,
               "note": "wait = last arrival - own arrival (node monotonic clock); bound = slowest worker's step "
                       "(PAPER.md P:149)"}
        with open(out_path, "w") as f:
            json.dump(res, f, indent=1)
        print("AEDIT OK", json.dumps(res), flush=True)
    s.close()
    dist.barrier(device_ids=[local_rank])
    dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
