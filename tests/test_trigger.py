"""When-to-sync logic (host only, CPU): EDiT's step trigger (Alg. 1 l.408) and A-EDiT's time
trigger (§3.3), through the C ABI (edit_trigger_*)."""
import pytest

from paper_2412_07210_b200 import EditSyncError, Trigger
from paper_2412_07210_b200.build import build

build()


def test_edit_step_trigger_matches_algorithm_1():
    tau, t_warm = 4, 5
    trig = Trigger.steps(tau, t_warm)
    got = [s for s in range(0, 25) if trig.sync_now(s)]
    # Alg. 1 l.408: (t*tau + p) > t_warm and p == 0, with s = t*tau + p
    assert got == [s for s in range(0, 25) if s > t_warm and s % tau == 0] == [8, 12, 16, 20, 24]
    assert [trig.in_warmup(s) for s in range(8)] == [True] * 6 + [False] * 2


def simulate_aedit(step_times, tau_time, rounds, t_warm=0):
    """Discrete-event run of A-EDiT: each worker asks its own trigger at every step boundary;
    a worker that must sync waits at the barrier until every worker arrived."""
    K = len(step_times)
    trig = [Trigger.time(tau_time, t_warm, 0.0) for _ in range(K)]
    clock = [0.0] * K
    step = [0] * K
    waits, steps_per_round = [], []
    for _ in range(rounds):
        arrive, done = [None] * K, [0] * K
        for k in range(K):
            while True:
                if trig[k].sync_now(step[k], clock[k]):
                    arrive[k] = clock[k]
                    break
                clock[k] += step_times[k]   # one whole inner step (never preempted)
                step[k] += 1
                done[k] += 1
        release = max(arrive)
        waits.append([release - a for a in arrive])
        steps_per_round.append(done)
        for k in range(K):
            clock[k] = release
            trig[k].mark_synced(release)
    return waits, steps_per_round, trig


def test_aedit_wait_bound_and_variable_inner_steps():
    step_times = [1.0, 2.3, 1.7, 0.45]
    waits, steps, trig = simulate_aedit(step_times, tau_time=10.0, rounds=6)
    # "no worker will wait longer than the single step time of the slowest worker"
    assert max(max(w) for w in waits) <= max(step_times) + 1e-12
    # faster workers do more inner steps: each completes ceil(tau_time / step_time) steps,
    # within +-1 for the rounding of the accumulated clock
    import math
    for r in steps:
        assert all(abs(a - math.ceil(10.0 / t)) <= 1 for a, t in zip(r, step_times))
    assert steps[0] == [math.ceil(10.0 / t) for t in step_times]
    assert all(t.syncs == 6 for t in trig)


def test_aedit_no_sync_during_warmup_and_clock_starts_after_it():
    trig = Trigger.time(5.0, t_warm=3, start_time_s=0.0)
    # steps 0..3 are warm-up: never sync, and the time base follows the clock
    assert not any(trig.sync_now(s, 100.0 * s) for s in range(4))
    assert not trig.sync_now(4, 300.0 + 4.9)
    assert trig.sync_now(5, 300.0 + 5.0)


def test_trigger_argument_errors():
    with pytest.raises(EditSyncError):
        Trigger(2)
    with pytest.raises(EditSyncError):
        Trigger.steps(0)
    with pytest.raises(EditSyncError):
        Trigger.time(0.0)
    with pytest.raises(EditSyncError):
        Trigger.steps(4, t_warm=-1)
