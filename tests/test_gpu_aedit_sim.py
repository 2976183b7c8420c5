"""A-EDiT time-triggered sync on ONE GPU (§3.3): the
members of a simulated M x N mesh (tests/sim_mesh.py) run real inner steps of different
lengths and sync through the library's production N > 1 kernels.

Each member k is a host thread with its own CUDA stream.  Its inner step is a sleep kernel of
base x (1 + 1.5 k / (K-1)) ms on that stream; at every whole-step boundary it asks its own
time trigger (Trigger.time, the library's edit_trigger_*) and, once its time since the last
sync reaches tau_time, arrives at the collective sync (a host barrier standing in for the
first exchange every real rank blocks in).  When the last member arrives the round runs for
the whole mesh (edit_sync_round on every member, step-major, tests/sim/edit_sim.cpp) with each
member's local drawn from ITS inner-step count.  Checked:
  - the members really completed different numbers of inner steps per round;
  - P:149 "no worker will wait longer than the single step time of the slowest worker":
    max over members of (last arrival - own arrival) <= the slowest member's step (+ 3 ms of
    host bookkeeping);
  - oracle parity of round 0 (every member's inputs regenerated from the step counts) and the
    cross-member invariants every round (anchors identical along a sync row, local ==
    rne(anchor)).
The multi-process version with real ranks is tests/test_gpu_aedit.py (needs >= 2 GPUs)."""
import json
import os
import threading
import time

import numpy as np
import pytest
import torch

import oracle
import synth
from tests import parity

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2412_07210_b200 import Trigger  # noqa: E402
from tests.sim_mesh import SimMesh  # noqa: E402

DEV = torch.device("cuda", 0)
BASE_STEP_MS = 20.0
TAU_TIME_S = 0.3
ROUNDS = 3


@pytest.mark.parametrize("mesh", ["1x2", "1x4", "2x2"])
def test_aedit_time_trigger_simulated_mesh(mesh):
    M, N = (int(x) for x in mesh.split("x"))
    K = M * N
    dtype = torch.bfloat16
    recipe = synth.Recipe()
    units = [synth.Unit("a", 2_000_003, ()), synth.Unit("b", 65_536, ()), synth.Unit("c", 1_000_000, ((999_000, 1000),))]
    numel = [synth.shard_numel(u.numel, M) for u in units]
    cfg = oracle.Config()
    sim = SimMesh(numel, M, N, DEV, dtype)
    try:
        mu = np.array([[synth.ema_seed(u, n, recipe)[0] for n in range(N)] for u in units])
        for e in sim.members:
            e.set_ema(mu, 0.1 * mu, recipe.ema_warmup_rounds)
        ema0 = [[oracle.Ema(mu[i, n], 0.1 * mu[i, n], recipe.ema_warmup_rounds) for n in range(N)]
                for i in range(len(units))]
        anc = [[synth.shard_anchor(u, i, M, k % M, DEV, recipe) for i, u in enumerate(units)] for k in range(K)]
        mom = [[synth.shard_momentum(u, i, M, k % M, DEV, recipe) for i, u in enumerate(units)] for k in range(K)]
        loc = [[torch.empty(n_, dtype=dtype, device=DEV) for n_ in numel] for _ in range(K)]
        o_anc0 = [[anc[m][i].cpu().numpy() for m in range(M)] for i in range(len(units))]
        o_mom0 = [[mom[m][i].cpu().numpy() for m in range(M)] for i in range(len(units))]

        # sleep-kernel calibration: cycles per ms
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        torch.cuda._sleep(20_000_000)
        torch.cuda.synchronize()
        cyc_per_ms = 20_000_000 / ((time.perf_counter() - t0) * 1e3)
        step_ms = [BASE_STEP_MS * (1.0 + 1.5 * k / max(1, K - 1)) for k in range(K)]
        streams = [torch.cuda.Stream(DEV) for _ in range(K)]

        state = {"round": 0, "arrive": [0.0] * K, "steps": [0] * K, "recs": [], "err": None, "first": None}
        t_start = [0.0]

        def run_round():
            """Barrier action: the last member arrived; sync the whole mesh."""
            try:
                rnd = state["round"]
                for k in range(K):
                    m, n = k % M, k // M
                    for i, u in enumerate(units):
                        loc[k][i].copy_(synth.shard_local(u, i, M, m, n, anc[k][i], dtype, DEV, recipe, 1.0,
                                                          1000 * (rnd + 1) + state["steps"][k]))
                torch.cuda.synchronize()
                t_in = time.perf_counter() - t_start[0]
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                sim.sync_round(loc, anc, mom)
                e1.record()
                torch.cuda.synchronize()
                arr = state["arrive"]
                waits = [1e3 * (max(arr) - a) for a in arr]
                state["recs"].append({"round": rnd, "steps_per_member": list(state["steps"]),
                                      "wait_ms_per_member": waits, "max_wait_ms": max(waits),
                                      "bound_ms": max(step_ms), "device_round_ms": e0.elapsed_time(e1),
                                      "host_bookkeeping_ms": 1e3 * (t_in - max(arr))})
                for k in range(K):
                    for i in range(len(units)):
                        assert torch.equal(loc[k][i], anc[k][i].to(dtype)), f"member {k} round {rnd} unit {i}"
                        assert torch.equal(anc[k][i], anc[k % M][i]), f"row anchors differ, member {k}"
                if rnd == 0:
                    state["first"] = {"steps": list(state["steps"]),
                                      "anc": [[a.cpu().numpy() for a in row] for row in anc],
                                      "mom": [[x.cpu().numpy() for x in row] for row in mom],
                                      "loc": [[parity.to_oracle_local(x) for x in row] for row in loc],
                                      "stats": [[sim.members[k].stats(i) for i in range(len(units))]
                                                for k in range(K)]}
                state["round"] += 1
            except BaseException as exc:  # reported by the main thread
                state["err"] = exc

        barrier = threading.Barrier(K, action=run_round)

        def worker(k):
            trig = Trigger.time(TAU_TIME_S, 0, 0.0)
            step = 0
            with torch.cuda.stream(streams[k]):
                for _ in range(ROUNDS):
                    steps = 0
                    while not trig.sync_now(step + 1, time.perf_counter() - t_start[0]):
                        torch.cuda._sleep(int(step_ms[k] * cyc_per_ms))
                        streams[k].synchronize()  # a whole step: the trigger is asked at step boundaries
                        step += 1
                        steps += 1
                    state["steps"][k] = steps
                    state["arrive"][k] = time.perf_counter() - t_start[0]
                    barrier.wait(timeout=120)
                    trig.mark_synced(time.perf_counter() - t_start[0])

        threads = [threading.Thread(target=worker, args=(k,)) for k in range(K)]
        t_start[0] = time.perf_counter()
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout=300)
        if state["err"] is not None:
            raise state["err"]
        recs = state["recs"]
        assert len(recs) == ROUNDS
        # the time trigger produced different inner-step counts across the members
        assert any(len(set(r["steps_per_member"])) > 1 for r in recs), recs
        for r in recs:
            # P:149 (host-clock arrivals; 3 ms allowance for the threads' step bookkeeping)
            assert r["max_wait_ms"] <= r["bound_ms"] + 3.0, r
        # oracle parity of round 0 (members had completed different numbers of inner steps)
        f = state["first"]
        for i, u in enumerate(units):
            locs = []
            for m in range(M):
                a = torch.from_numpy(o_anc0[i][m]).to(DEV)
                row = []
                for n in range(N):
                    l_ = synth.shard_local(u, i, M, m, n, a, dtype, DEV, recipe, 1.0, 1000 + f["steps"][n * M + m])
                    row.append(parity.to_oracle_local(l_))
                locs.append(row)
            o_loc, o_anc, o_mom, o_ema, out = oracle.sync_unit(cfg, np.array(locs), np.stack(o_anc0[i]),
                                                               np.stack(o_mom0[i]), ema0[i])
            for k in range(K):
                m, n = k % M, k // M
                tag = f"A-EDiT (simulated {mesh}) round 0 unit {i} member {k}"
                parity.assert_outcome(f["stats"][k][i], out, o_ema, tag)
                parity.assert_f32_close(f["anc"][k][i], o_anc[m], tag + " anchor")
                parity.assert_f32_close(f["mom"][k][i], o_mom[m], tag + " momentum")
                parity.assert_local_close(f["loc"][k][i], o_loc[m, n], tag + " local")
        dest = os.environ.get("EDIT_AEDIT_LOG")
        if dest:
            with open(dest.replace("{mesh}", "sim" + mesh), "w") as fh:
                json.dump({"mesh": mesh, "simulated": True, "tau_time_s": TAU_TIME_S, "step_ms_per_member": step_ms,
                           "rounds": recs}, fh, indent=1)
    finally:
        sim.close()
