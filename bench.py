#!/usr/bin/env python
"""EDiT layer-wise sync benchmark (BASELINE.json metric: "EDiT sync GB/s of params/round
and % HBM+NVLink roofline at 1/2/4/8 B200").

One step = one full sync round (Alg. 2 for every one of the 34 sync units of a
Llama-shaped model) over this rank's shards, through the C ABI.
Workload at N = 1: Llama-7B-shaped shards on a 1 x 1 mesh (the largest single-GPU
configuration of BASELINE.json; 71.3 GB of local/anchor/momentum, far above L2).  With
--gpus N the default mesh is 1 x N (every rank keeps a full 7B replica: weak scaling).

Between steps, outside the timed region, every local is redrawn as
cast(anchor - D) with a fresh inner-loop displacement D (synth/), so each timed round
syncs a realistic pseudo-gradient (clip active, anomaly test live).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl edit|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402

NOMINAL_HBM_GBS = 8000.0       # BASELINE.md roofline definition (nominal)
NOMINAL_NVL_GBS = 900.0        # per direction per GPU (nominal)
MEASURED_NVL_GBS = 770.0       # peer copy per direction, B200_PROFILING.md (measured on this pool)
METRIC = "EDiT sync GB/s of params/round and % HBM+NVLink roofline at 1/2/4/8 B200"


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "_fallback": True}


def max_over_ranks(t_ms: float, world: int, device) -> float:
    """Multi-GPU timing rule: every number is the max over ranks (device-timed per rank)."""
    if world <= 1:
        return t_ms
    tt = torch.tensor([t_ms], device=device, dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return float(tt.item())


def x_bytes(n_f32: int) -> float:
    return 4.0 * n_f32


def rank_coords(rank: int, M: int) -> tuple[int, int]:
    """(shard index m, sync index n) of a rank: rank = n*M + m (R20, include/edit_sync.h)."""
    return rank % M, rank // M


def parse_mesh(s: str | None, world: int) -> tuple[int, int]:
    if not s:
        return 1, world
    m, n = (int(x) for x in s.lower().split("x"))
    if m * n != world:
        raise SystemExit(f"mesh {s} needs {m * n} ranks, have {world}")
    return m, n


class Clocks:
    """nvidia-smi sampler run DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.idx = device_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *exc):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()

    def summary(self) -> dict:
        self.f.flush()
        rows = []
        with open(self.f.name) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        pw = [float(r[3]) for r in rows if r[3].replace(".", "").isdigit()]
        capped = sum(1 for r in rows if r[8].lower() == "active")
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows),
                "power_w": statistics.median(pw) if pw else None,
                "power_cap_frac": capped / len(rows)}


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_cpu_baseline(model: str, dtype, target_s: float = 12.0) -> dict:
    """The oracle (as it stands) on this host's cores, on a bounded sample of the workload:
    whole decoder-unit shards of the 1 x 1 mesh (layer 0, 1, ...) until ~target_s of CPU work."""
    import oracle
    from tests import parity
    oracle.set_threads(os.cpu_count() or 1)
    units = synth.llama_units(model)
    dev = torch.device("cuda", torch.cuda.current_device())
    total_t, total_n, done = 0.0, 0, []
    for i in range(1, len(units) - 1):
        u = units[i]
        a = synth.shard_anchor(u, i, 1, 0, dev)
        m = synth.shard_momentum(u, i, 1, 0, dev)
        l = synth.shard_local(u, i, 1, 0, 0, a, dtype, dev)
        L, A, Mo = parity.to_oracle_local(l)[None, None], a.cpu().numpy()[None], m.cpu().numpy()[None]
        del a, m, l
        mu, sg, cnt = synth.ema_seed(u, 0)
        t0 = time.perf_counter()
        oracle.sync_unit(oracle.Config(), L, A, Mo, [oracle.Ema(mu, sg, cnt)])
        total_t += time.perf_counter() - t0
        total_n += u.numel
        done.append(u.name)
        if total_t >= target_s or len(done) >= 8:
            break
    # the same oracle on ONE thread (threads = 1 and os.cpu_count()), on a 16M-param
    # prefix of the first sampled unit (timing only; a prefix is a smaller unit of the same kind)
    cores = oracle.get_threads()
    u = units[1]
    sub = min(u.numel, 16_000_000)
    a = synth.shard_anchor(u, 1, 1, 0, dev)
    m = synth.shard_momentum(u, 1, 1, 0, dev)
    l = synth.shard_local(u, 1, 1, 0, 0, a, dtype, dev)
    L1 = parity.to_oracle_local(l)[None, None, :sub].copy()
    A1, M1 = a.cpu().numpy()[None, :sub].copy(), m.cpu().numpy()[None, :sub].copy()
    del a, m, l
    oracle.set_threads(1)
    t0 = time.perf_counter()
    oracle.sync_unit(oracle.Config(), L1, A1, M1, [oracle.Ema()])
    t1 = time.perf_counter() - t0
    oracle.set_threads(cores)
    one = {"value": 4.0 * sub / t1 / 1e9, "unit": "GB/s", "cores": 1,
           "sample": f"{sub} params (prefix of {u.name}), {t1:.1f} s on 1 thread"}
    return {"value": 4.0 * total_n / total_t / 1e9, "unit": "GB/s", "cores": cores, "kind": "oracle",
            "threads_1": one, "host_cpu": _cpu_model(),
            "sample": f"1 sync of the Llama-{model} shards {done[0]}..{done[-1]} ({len(done)} decoder units, "
                      f"{total_n} params, 1x1 mesh, {'bf16' if dtype == torch.bfloat16 else 'f32'} local): "
                      f"{total_t:.1f} s on {oracle.get_threads()} threads; fp32 pseudo-gradient bytes / s"}


def reference_arm(args) -> None:
    """--impl reference: the fp64 CPU oracle as it stands, on this host's cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from tests import parity
    oracle.set_threads(os.cpu_count() or 1)
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    M, N = 1, 1
    u = synth.llama_units(args.model)[1]
    x = args.ref_sample
    sub = synth.Unit(u.name + f"[:{x}]", x, ())
    gen_dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
    a = synth.shard_anchor(sub, 1, M, 0, gen_dev)
    m = synth.shard_momentum(sub, 1, M, 0, gen_dev)
    A, Mo = a.cpu().numpy()[None], m.cpu().numpy()[None]
    ema = [oracle.Ema(*synth.ema_seed(sub, 0)[:2], 10)]
    times = []
    for step in range(args.warmup + args.steps):
        L = parity.to_oracle_local(synth.shard_local(sub, 1, M, 0, 0, torch.from_numpy(A[0]).to(gen_dev), dtype,
                                                     gen_dev, round_salt=step))[None, None]
        t0 = time.perf_counter()
        L, A, Mo, ema, _ = oracle.sync_unit(oracle.Config(), L, A, Mo, ema)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
    total = sum(times)
    value = 4.0 * x * len(times) / total / 1e9
    cores = oracle.get_threads()
    line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"llama-{args.model} shards, 1x1 mesh: bounded sample of {x} params of the "
                                   "layer-0 shard per step (oracle throughput; same metric/unit)",
                       "model_shape": args.model, "param_dtype": args.dtype},
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": "oracle",
                             "sample": f"{x} params of the Llama-{args.model} layer-0 shard per step"},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="edit", choices=["edit", "reference"])
    ap.add_argument("--model", default="7B", choices=list(synth.LLAMA))
    ap.add_argument("--mesh", default=None, help="MxN shard x sync mesh (default 1xN)")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--algo", default="peer", choices=["peer", "nccl"], help="N > 1 exchange of Eq. 3")
    ap.add_argument("--e2e-units", default=None,
                    help="unit indices timed through the host-buffer API (default 1..6, or 1..3 at >= 4 GPUs "
                         "to bound the pinned host memory of the node)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-sample", type=int, default=4_000_000)
    ap.add_argument("--overlap-tokens", default="8192,65536",
                    help="tokens/GPU of the synthetic forward(s) for the prefetch-overlap measurement, comma "
                         "list (0 = skip); 8,192 = SURVEY 8d default, 65,536 = the paper's 1024 seqs x 4096 / 64")
    ap.add_argument("--partition", default="-1,0,32",
                    help="scheduler partition modes to measure (comma list: -1 = auto, the library default; "
                         "0 = full grids; > 0 = that many SMs)")
    ap.add_argument("--full-units", type=int, default=2,
                    help="partition mode: units before this index keep full grids (embedding + first layer)")
    ap.add_argument("--overlap-steps", type=int, default=4)
    ap.add_argument("--warmup-allreduce", action="store_true", help="NEXT-3 measurement (N > 1)")
    ap.add_argument("--gather", action="store_true", help="NEXT-2 fused shard all-gather measurement (M > 1)")
    ap.add_argument("--no-register", action="store_true",
                    help="peer path: do not register the locals for direct IPC reads (stage a copy)")
    ap.add_argument("--anomaly-rate", type=float, default=0.0,
                    help="probability that a (unit, replica) is planted anomalous in a round (SURVEY 8d: 3B config)")
    ap.add_argument("--anomaly-sweep", default=None,
                    help="comma list of anomaly rates timed after the main loop (e.g. 0,0.125,0.25,0.5,1)")
    ap.add_argument("--sequential", action="store_true",
                    help="time per-unit edit_layer_sync calls on one stream instead of edit_sync_round")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: W >= 3

    if args.impl == "reference":
        return reference_arm(args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2412_07210_b200 import EditSync, broadcast_unique_id

    M, N = parse_mesh(args.mesh, world)
    m_idx, n_idx = rank_coords(rank, M)
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    b_l = 2 if dtype == torch.bfloat16 else 4
    units = synth.llama_units(args.model)
    numel = [synth.shard_numel(u.numel, M) for u in units]
    P_r = sum(numel)
    uid = broadcast_unique_id() if world > 1 else None
    sync = EditSync(numel, shard_dim=M, sync_dim=N, rank=rank, device=dev, param_dtype=dtype, unique_id=uid,
                    algo=args.algo)
    # EMA seeded at the expected module norm of each replica (synth recipe, R8)
    import numpy as np
    mu = np.array([[synth.ema_seed(u, n)[0] for n in range(N)] for u in units])
    sync.set_ema(mu, 0.1 * mu, synth.Recipe().ema_warmup_rounds)

    anchors, moms, locs = [], [], []
    for i, u in enumerate(units):
        a = synth.shard_anchor(u, i, M, m_idx, dev)
        anchors.append(a)
        moms.append(synth.shard_momentum(u, i, M, m_idx, dev))
        locs.append(torch.empty(numel[i], dtype=dtype, device=dev))
    torch.cuda.synchronize()
    registered = N > 1 and args.algo == "peer" and not args.no_register
    if registered:
        sync.register_locals(locs)   # members read each other's locals directly (no staging copy)

    # NVLink / NCCL calibration in the same job, outside every timed region:
    # the library's peer-pull probe (every member of the sync row pulling from all the others
    # at once, the AG pattern) and torch/NCCL all-reduce bus bandwidth over all ranks
    calib = None
    if N > 1 and args.algo == "peer":
        probe = sync.nvlink_probe(256 << 20, 5)
        pt = torch.tensor([probe, -probe], device=dev, dtype=torch.float64)
        dist.all_reduce(pt, op=dist.ReduceOp.MIN)
        x = torch.empty(64 << 20, dtype=torch.float32, device=dev)  # 256 MiB
        for _ in range(2):
            dist.all_reduce(x)
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        for _ in range(5):
            dist.all_reduce(x)
        c1.record()
        torch.cuda.synchronize()
        t_ar = max_over_ranks(c0.elapsed_time(c1) / 5, world, dev)
        del x
        calib = {"nvlink_allpull_GBps_min_over_ranks": float(pt[0]), "nvlink_allpull_GBps_max_over_ranks": -float(pt[1]),
                 "nvlink_probe": "edit_sync_nvlink_probe: each sync-row member pulls 256 MiB from every other member "
                                 "at once, 5 reps, CUDA events (per-direction ingress)",
                 "nccl_allreduce_busbw_GBps": 2.0 * (world - 1) / world * x_bytes(64 << 20) / (t_ar * 1e-3) / 1e9,
                 "nccl_allreduce": f"torch.distributed all_reduce fp32 256 MiB over {world} ranks, 5 reps, max over ranks"}
        torch.cuda.empty_cache()

    planted = {"replicas": 0, "rounds": 0}

    def redraw(step: int) -> None:
        # "tau inner steps" of every worker, outside the timed region; --anomaly-rate r plants
        # anomalous replicas (x4 displacement) per (unit, replica, round) with probability r
        plants = synth.anomaly_plants(len(units), N, args.anomaly_rate, step)
        planted["replicas"] += len(plants)
        planted["rounds"] += 1
        for i, u in enumerate(units):
            locs[i].copy_(synth.shard_local(u, i, M, m_idx, n_idx, anchors[i], dtype, dev,
                                            plant=plants.get((i, n_idx), 1.0), round_salt=step))

    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local_rank])

    def run_round():
        if args.sequential:
            for i in range(len(units)):
                sync.layer_sync(i, locs[i], anchors[i], moms[i], stream)
        else:  # edit_sync_round: units pipelined over the library's lanes
            sync.sync_round(locs, anchors, moms, stream)

    # profiling events on from the warm-up on (with EDIT_GRAPH=1 the profiled round is the graph
    # that the timed steps replay, so it is captured here, outside the timed region)
    sync.set_profiling(True)
    for w in range(args.warmup):
        redraw(w + 1)
        barrier()
        run_round()
        torch.cuda.synchronize()
    sync.profile_collect()  # drop the warm-up rounds' phase times
    step_ms = []
    phase_ms = {k: 0.0 for k in sync.PHASES}
    phase_busy_ms = {k: 0.0 for k in sync.PHASES}
    k4_elems = 0
    launches0 = sync.kernel_launches
    clocks = Clocks(local_rank)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clocks:
        for s in range(args.steps):
            redraw(args.warmup + s + 1)
            barrier()
            torch.cuda.synchronize()
            ev0.record(stream)
            run_round()
            ev1.record(stream)
            torch.cuda.synchronize()
            t = ev0.elapsed_time(ev1)
            prof = sync.profile_collect()
            for k, v in prof["ms"].items():
                phase_ms[k] += v
            for k, v in prof["busy_ms"].items():
                phase_busy_ms[k] += v
            k4_elems += prof["elements"]
            step_ms.append(max_over_ranks(t, world, dev))
    launches = sync.kernel_launches - launches0
    clk = clocks.summary()
    # SURVEY 8d (3B config): the same timed round at several anomaly rates; throughput should
    # not depend on the rate except through the cheaper rollback write (every replica flagged)
    anomaly_sweep = None
    if args.anomaly_sweep:
        anomaly_sweep = []
        rate0 = args.anomaly_rate
        for ri, rate in enumerate(float(x) for x in args.anomaly_sweep.split(",")):
            args.anomaly_rate = rate
            ts, fl, rb = [], 0, 0
            for s in range(args.steps + 1):      # first round untimed
                redraw(20000 + 100 * ri + s)
                barrier()
                torch.cuda.synchronize()
                ev0.record(stream)
                run_round()
                ev1.record(stream)
                torch.cuda.synchronize()
                if s > 0:
                    ts.append(max_over_ranks(ev0.elapsed_time(ev1), world, dev))
                    for i in range(len(units)):
                        st_i = sync.stats(i)
                        fl += int(sum(st_i.anomalous[:N]))
                        rb += int(st_i.rollback)
            ms = sum(ts) / len(ts)
            anomaly_sweep.append({"rate": rate, "ms_per_round": ms,
                                  "value_GBps": world * 4.0 * P_r / (ms * 1e-3) / 1e9,
                                  "flagged_per_round": fl / len(ts), "rollbacks_per_round": rb / len(ts),
                                  "units_x_replicas": len(units) * N})
        args.anomaly_rate = rate0
    # the same kernels once more, isolated: per-unit calls on one stream (no lane overlap),
    # outside the timed region -- each kernel's own duration for the isolated roofline
    iso_ms = {k: 0.0 for k in sync.PHASES}
    iso_elems = 0
    for s in range(2):
        redraw(5000 + s)
        barrier()
        torch.cuda.synchronize()
        for i in range(len(units)):
            sync.layer_sync(i, locs[i], anchors[i], moms[i], stream)
        torch.cuda.synchronize()
        prof = sync.profile_collect()
        for k, v in prof["ms"].items():
            iso_ms[k] += v
        iso_elems += prof["elements"]
    sync.set_profiling(False)
    # every unit's outcome of the last round (checks nothing rolled back unexpectedly)
    rollbacks = sum(int(sync.stats(i).rollback) for i in range(len(units)))
    betas = [sync.stats(i).beta for i in (0, 1, len(units) - 1)]
    flagged = sum(int(sum(sync.stats(i).anomalous[:N])) for i in range(len(units)))
    anomaly = {"rate": args.anomaly_rate, "planted_replicas_per_round": planted["replicas"] / max(1, planted["rounds"]),
               "flagged_last_round": flagged, "rollbacks_last_round": rollbacks,
               "units_x_replicas": len(units) * N}

    total_ms = sum(step_ms)
    ms_per_step = total_ms / len(step_ms)
    bytes_per_rank_round = 4.0 * P_r
    value = world * bytes_per_rank_round * len(step_ms) / (total_ms * 1e-3) / 1e9

    peaks = measured_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    b_hbm = 16 + 2 * b_l                        # algorithmic HBM B/param
    b_nvl = 8.0 * (N - 1) / N                   # NCCL bus bytes per direction per param
    k4_ms = phase_ms["outer_update"]
    k4_launches = args.steps * len(units)
    # dominant kernel: K4 (outer_update; N == 1 or NCCL exchange) or, on the peer-memory path,
    # ag_update (pulls Dbar over NVLink while applying K4's update).  Its algorithmic bytes:
    # HBM 16 + 2 b_l (20 B bf16) and, on the peer path, NVLink 4 (N-1)/N B/param in.
    peer = N > 1 and args.algo == "peer"
    k4_name = "ag_update (RS'd Dbar pull + Nesterov + write-back)" if peer else "outer_update (K4)"
    k4_hbm_B = b_hbm
    k4_nvl_B = 4.0 * (N - 1) / N if peer else 0.0
    t_hbm = k4_hbm_B / hbm_peak
    t_nvl = k4_nvl_B / MEASURED_NVL_GBS
    if k4_ms > 0 and t_nvl > t_hbm:
        k4_bound, k4_peak, k4_B = "nvlink", MEASURED_NVL_GBS, k4_nvl_B
    else:
        k4_bound, k4_peak, k4_B = "hbm", hbm_peak, k4_hbm_B
    # live achieved = the dominant kernel's algorithmic bytes over the time its launches were
    # running (union of the units' intervals: with several lanes, launches of different units
    # overlap, and the per-launch sum would count shared time twice)
    k4_busy = phase_busy_ms["outer_update"]
    k4_achieved = k4_B * k4_elems / (k4_busy * 1e-3) / 1e9 if k4_busy > 0 else None
    k4_achieved_sum = k4_B * k4_elems / (k4_ms * 1e-3) / 1e9 if k4_ms > 0 else None
    k4_iso = k4_B * iso_elems / (iso_ms["outer_update"] * 1e-3) / 1e9 if iso_ms["outer_update"] > 0 else None
    k1_B = (2 * b_l + 4) if (peer and not registered) else (b_l + 4 + (4 if (N > 1 and not peer) else 0))
    k1_iso = k1_B * iso_elems / (iso_ms["pg_norm"] * 1e-3) / 1e9 if iso_ms["pg_norm"] > 0 else None
    if peer:
        b_nvl = 6.0 * (N - 1) / N if b_l == 2 else 8.0 * (N - 1) / N  # bytes the peer path moves
    t_roof_nom = max(P_r * b_hbm / (NOMINAL_HBM_GBS * 1e9), P_r * (8.0 * (N - 1) / N) / (NOMINAL_NVL_GBS * 1e9)) * 1e3
    t_roof_meas = max(P_r * b_hbm / (hbm_peak * 1e9), P_r * (8.0 * (N - 1) / N) / (MEASURED_NVL_GBS * 1e9)) * 1e3
    # the bytes THIS dataflow must move per param (not the algorithmic minimum), bf16 local:
    # N == 1: 6 + 20 = 26; peer path: 6 (+2 staging copy unless registered) + RS (2 + 8/N) +
    # AG 22 in HBM and 6(N-1)/N over NVLink; the NCCL path is not modelled
    design = None
    if N == 1:
        d_hbm, d_nvl = (b_l + 4) + (16 + 2 * b_l), 0.0                      # K1 + K4
    elif peer:
        # K1 (+ staging copy) + RS (anchor + local slices, served peer reads, Dbar slice) +
        # AG (Dbar own + served, anchor, momentum in; momentum, anchor, local out)
        d_hbm = (b_l + 4) + (0 if registered else b_l) + (b_l + 8.0 / N) + (20 + b_l)
        d_nvl = (b_l + 4) * (N - 1) / N
    else:
        d_hbm = d_nvl = None
    if d_hbm is not None:
        # every member pulling from the others at once: the live probe of this run, else the
        # round-1 measurement (profiles/r1_a2a_peer_pull_2gpu.txt)
        nvl_bidir = calib["nvlink_allpull_GBps_min_over_ranks"] if calib else 673.0
        t_bound = max(P_r * d_hbm / (hbm_peak * 1e9), P_r * d_nvl / (nvl_bidir * 1e9)) * 1e3
        design = {"hbm_B_per_param": d_hbm, "nvlink_B_per_param_per_dir": d_nvl,
                  "hbm_achieved_GBps": P_r * d_hbm / (ms_per_step * 1e-3) / 1e9,
                  "nvlink_achieved_GBps": P_r * d_nvl / (ms_per_step * 1e-3) / 1e9,
                  "t_bound_ms": t_bound, "frac": t_bound / ms_per_step,
                  "peaks": f"HBM {hbm_peak} GB/s (MEASURED_PEAKS), NVLink {nvl_bidir:.1f} GB/s per direction "
                           "with every member pulling (" + ("measured in this run" if calib else "round-1 probe") + ")"}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tinfo = json.load(f)
        key = (f"ag_update_{args.dtype}" if peer else f"outer_update_{args.dtype}_{'S' if N > 1 else 'local'}")
        if key in tinfo:
            traffic = tinfo[key]["dram_bytes_per_elem"] * k4_elems / k4_launches

    # a8: layer-wise prefetch -- hidden fraction h = 1 - (t_fwd+sync - t_fwd) / t_sync,
    # t_sync = the full-speed round alone; swept over forward sizes and partition modes
    overlap = None
    tokens_list = [int(x) for x in str(args.overlap_tokens).split(",") if int(x) > 0]
    parts = [int(x) for x in str(args.partition).split(",")]
    if tokens_list:
        from synth.forward import SyntheticForward

        def timed_clk(fn, nsteps, redraw_first=True):
            c = Clocks(local_rank)
            with c:
                t = timed(fn, nsteps, redraw_first)
            k = c.summary()
            return t, {"sm_mhz": k["sm_mhz"], "power_w": k.get("power_w"),
                       "power_cap_frac": k.get("power_cap_frac"), "samples": k["samples"]}

        def timed(fn, nsteps, redraw_first=True):
            ts = []
            for s in range(nsteps + 1):          # first one untimed (warm-up)
                if redraw_first:
                    redraw(1000 + s)
                barrier()
                torch.cuda.synchronize()
                ev0.record(stream)
                fn()
                ev1.record(stream)
                torch.cuda.synchronize()
                t = ev0.elapsed_time(ev1)
                t = max_over_ranks(t, world, dev)
                if s > 0:
                    ts.append(t)
            return sum(ts) / len(ts)

        t_sync_alone, clk_sync = timed_clk(run_round, args.overlap_steps)

        def sched_only():                       # the scheduled round with no forward
            sync.begin_round(locs, anchors, moms, 1, stream)
            for u in range(len(units)):
                sync.acquire(u, stream)
            sync.end_round(stream)

        t_sync_sched = {}
        for sms in parts:                       # the partitioned sync alone, per SM count
            sync.set_partition(sms, args.full_units)
            t, k = timed_clk(sched_only, args.overlap_steps)
            t_sync_sched[str(sms)] = {"ms": t, "clocks": k}
        sync.set_partition(-1, args.full_units)
        runs = []
        for tokens in tokens_list:
            fwd = SyntheticForward(args.model, units, tokens, dev)

            def forward_only():
                for u in range(len(units)):
                    fwd.unit(u, locs[u])

            def fwd_and_sync(depth):
                def run():
                    sync.begin_round(locs, anchors, moms, depth, stream)
                    for u in range(len(units)):
                        sync.acquire(u, stream)
                        fwd.unit(u, locs[u])
                    sync.end_round(stream)
                return run

            def once(fn, redraw_first, k=[0]):
                k[0] += 1
                if redraw_first:
                    redraw(3000 + k[0])
                barrier()
                torch.cuda.synchronize()
                ev0.record(stream)
                fn()
                ev1.record(stream)
                torch.cuda.synchronize()
                return max_over_ranks(ev0.elapsed_time(ev1), world, dev)

            t_fwd, clk_fwd = timed_clk(forward_only, args.overlap_steps, redraw_first=False)
            for sms in parts:
                sync.set_partition(sms, args.full_units)
                for depth in (1, 2):
                    # warm-up rounds: the auto mode (-1) tunes itself over its first 12 rounds
                    for _ in range(13 if sms == -1 else 1):
                        once(fwd_and_sync(depth), True)
                    # paired measurement: the forward alone and forward + sync back to back, the
                    # exposed sync time = the median of the pair differences (the forward runs
                    # at the power cap and drifts by more than t_sync between separate runs)
                    c = Clocks(local_rank)
                    diffs, tb, tf = [], [], []
                    with c:
                        for _ in range(args.overlap_steps):
                            a_ = once(forward_only, False)
                            b_ = once(fwd_and_sync(depth), True)
                            diffs.append(b_ - a_)
                            tf.append(a_)
                            tb.append(b_)
                    k = c.summary()
                    exposed = statistics.median(diffs)
                    runs.append({"tokens_per_gpu": tokens, "partition_sms": sms, "depth": depth,
                                 "t_fwd_ms": statistics.mean(tf), "t_fwd_plus_sync_ms": statistics.mean(tb),
                                 "exposed_ms_median_pair": exposed, "exposed_ms_pairs": diffs,
                                 "clocks_fwd": clk_fwd,
                                 "clocks_pairs": {"sm_mhz": k["sm_mhz"], "power_w": k.get("power_w"),
                                                  "power_cap_frac": k.get("power_cap_frac"), "samples": k["samples"]},
                                 "fwd_tflops": fwd.flops_per_round() / (t_fwd * 1e-3) / 1e12,
                                 "plan": sync.sched_plan() if sms == -1 else None,
                                 "hidden_fraction": 1.0 - exposed / t_sync_alone})
            sync.set_partition(-1, args.full_units)
            del fwd
            torch.cuda.empty_cache()
        best = {}
        for r in runs:
            k = r["tokens_per_gpu"]
            if k not in best or r["hidden_fraction"] > best[k]["hidden_fraction"]:
                best[k] = r
        default = {str(r["tokens_per_gpu"]): r for r in runs if r["partition_sms"] == -1 and r["depth"] == 1}
        head = best[tokens_list[0]]
        overlap = {"tokens_per_gpu": head["tokens_per_gpu"], "t_sync_ms": t_sync_alone, "clocks_sync": clk_sync,
                   "t_sync_sched_alone_ms_by_partition": t_sync_sched,
                   "t_fwd_ms": head["t_fwd_ms"], "best": {str(k): v for k, v in best.items()},
                   "default_settings": default, "runs": runs,
                   "full_units": args.full_units,
                   "note": ("synthetic forward (bf16 GEMMs of each unit, weights = the synced local) on the "
                            "compute stream; syncs on the library's side streams; acquire(u) before forward(u); "
                            "partition_sms > 0: edit_sched_set_partition (units >= full_units on that many "
                            "persistent TMA CTAs, one per SM; -1 = auto, the library default: per unit the fewest SMs that "
                            "finish its sync within the forward it overlaps, measured in the previous round); "
                            "h = 1 - exposed / t_sync_alone, exposed = median over pairs of (fwd+sync) - (fwd alone) run back to "
                            "back; the auto mode is measured after its 12 tuning rounds")}

    # NEXT-3: warm-up gradient all-reduce (mean over the sync group) of a full set of bf16
    # gradient shards, library path vs torch.distributed/NCCL all_reduce on the same group
    warm = None
    if args.warmup_allreduce and N > 1:
        grads = [torch.randn(numel[i], device=dev).mul_(1e-3).to(dtype) for i in range(len(units))]
        row = [n * M + m_idx for n in range(N)]
        groups = [dist.new_group([n * M + m for n in range(N)]) for m in range(M)]
        my_group = groups[m_idx]

        def lib_warm(algo):
            def run():
                os.environ["EDIT_WARMUP_ALGO"] = algo   # read per call by the library
                for i in range(len(units)):
                    sync.warmup_allreduce(i, grads[i], stream)
            return run

        def lib_warm_round(algo):
            def run():
                os.environ["EDIT_WARMUP_ALGO"] = algo
                sync.warmup_allreduce_round(grads, stream)
            return run

        def torch_warm():
            for i in range(len(units)):
                dist.all_reduce(grads[i], op=dist.ReduceOp.AVG, group=my_group)

        res = {}
        algo0 = os.environ.get("EDIT_WARMUP_ALGO")
        variants = [("library", lib_warm("nccl")), ("library_peer", lib_warm("peer")),
                    ("library_round_nccl", lib_warm_round("nccl")), ("library_round_peer", lib_warm_round("peer")),
                    ("torch_nccl", torch_warm)]
        for name, fn in variants:
            ts = []
            for s_ in range(4):
                barrier()
                torch.cuda.synchronize()
                ev0.record(stream)
                fn()
                ev1.record(stream)
                torch.cuda.synchronize()
                t = max_over_ranks(ev0.elapsed_time(ev1), world, dev)
                if s_ > 0:
                    ts.append(t)
            res[name] = sum(ts) / len(ts)
        if algo0 is None:
            os.environ.pop("EDIT_WARMUP_ALGO", None)
        else:
            os.environ["EDIT_WARMUP_ALGO"] = algo0
        warm = {"ms_per_round": res, "params_per_rank": P_r, "sync_row": row,
                "GBps_of_grad_bytes_per_gpu": {k: P_r * b_l / (v * 1e-3) / 1e9 for k, v in res.items()},
                "note": "all units' bf16 gradient shards averaged over the sync group (Alg. 1 l.422-424); "
                        "library = per-unit edit_warmup_allreduce on the caller stream, library_round = "
                        "edit_warmup_allreduce_round (units pipelined over the lanes); nccl / peer = "
                        "EDIT_WARMUP_ALGO"}
        del grads

    # NEXT-2: fused write-back -> shard-group all-gather (M > 1): a round with the gathered
    # modules filled by the update kernels vs a round followed by an NCCL all-gather per unit
    gather = None
    if args.gather and M > 1:
        full = [torch.empty(M * numel[i], dtype=dtype, device=dev) for i in range(len(units))]
        col = [n_idx * M + q for q in range(M)]
        sgroups = [dist.new_group([n * M + q for q in range(M)]) for n in range(N)]
        my_sgroup = sgroups[n_idx]

        def round_then_allgather():
            run_round()
            for i in range(len(units)):
                dist.all_gather_into_tensor(full[i], locs[i], group=my_sgroup)

        def timed_g(fn):
            ts = []
            for s_ in range(4):
                redraw(7000 + s_)
                barrier()
                torch.cuda.synchronize()
                ev0.record(stream)
                fn()
                ev1.record(stream)
                torch.cuda.synchronize()
                t = max_over_ranks(ev0.elapsed_time(ev1), world, dev)
                if s_ > 0:
                    ts.append(t)
            return sum(ts) / len(ts)

        t_sep = timed_g(round_then_allgather)
        sync.register_gather(full)
        t_fused = timed_g(run_round)
        gather = {"t_round_plus_nccl_allgather_ms": t_sep, "t_round_fused_gather_ms": t_fused,
                  "t_round_ms": ms_per_step, "shard_group": col,
                  "note": "Alg. 1 l.411 all-gather of the freshly synced module within the shard group"}

    # e2e: same metric through the host-buffer C-ABI call (pinned host buffers; H2D of
    # local/anchor/momentum and D2H of the three results inside the timed region)
    e2e = None
    if not args.no_e2e:
        spec = args.e2e_units or ("1,2,3,4,5,6" if world <= 2 else "1,2,3")
        idx = [int(x) for x in spec.split(",") if x.strip()]
        h_loc = [locs[i].cpu().pin_memory() for i in idx]
        h_anc = [anchors[i].cpu().pin_memory() for i in idx]
        h_mom = [moms[i].cpu().pin_memory() for i in idx]
        e_ms = []
        for s in range(args.warmup + args.steps):
            barrier()
            torch.cuda.synchronize()
            ev0.record(stream)
            for j, i in enumerate(idx):
                sync.layer_sync_host(i, h_loc[j], h_anc[j], h_mom[j], stream)
            sync.host_wait(stream)
            ev1.record(stream)
            torch.cuda.synchronize()
            t = ev0.elapsed_time(ev1)
            t = max_over_ranks(t, world, dev)
            if s >= args.warmup:
                e_ms.append(t)
        n_e = sum(numel[i] for i in idx)
        e2e = {"value": world * 4.0 * n_e * len(e_ms) / (sum(e_ms) * 1e-3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": (8 + b_l) * n_e, "d2h_bytes_per_step": (8 + b_l) * n_e,
               "units": [units[i].name for i in idx],
               "note": "host-buffer edit_layer_sync_host (CPU-offloaded anchor/momentum, P:123) over the "
                       "listed units per step; pinned host memory, copies overlapped across units"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_cpu_baseline(args.model, dtype)
        # labelled extrapolation (by parameter count) of one full round of this config
        cpu["extrapolated_full_round_s"] = 4.0 * P_r / (cpu["value"] * 1e9)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step,
            "ms_per_step_median": statistics.median(step_ms), "ms_per_step_min": min(step_ms),
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"llama-{args.model}-shaped shards, {M}x{N} shard x sync mesh, full sync round "
                                   f"of {len(units)} units ({P_r} params/rank), {args.dtype} local + f32 "
                                   "anchor/momentum",
                       "mesh": f"{M}x{N}", "params_per_rank": P_r, "param_dtype": args.dtype,
                       "exchange": (args.algo + (" (registered locals)" if registered else "") if N > 1
                                    else "none (N = 1)"),
                       "api": "edit_layer_sync x L (sequential)" if args.sequential else
                       f"edit_sync_round ({os.environ.get('EDIT_LANES', '4' if N > 1 else '2')} lanes"
                       + (", CUDA-graph replay" if os.environ.get("EDIT_GRAPH", "0") != "0" else "")
                       + (f", unit groups <= {os.environ.get('EDIT_GROUP_NUMEL', '67108864')} elements"
                          if (N > 1 and args.algo == "peer" and os.environ.get("EDIT_GROUP_NUMEL", "1") != "0") else "")
                       + ")",
                       "l2": "inputs (%.1f GB/rank) larger than L2" % (P_r * (b_l + 8) / 1e9),
                       "inner_steps": "locals redrawn as cast(anchor - D) between steps, outside the timed region",
                       "anomaly_rate": args.anomaly_rate},
            "roofline": {"bound": k4_bound, "kernel": k4_name, "achieved": k4_achieved, "peak": k4_peak,
                         "unit": "GB/s", "frac": (k4_achieved / k4_peak) if k4_achieved else None,
                         "traffic": traffic if k4_bound == "hbm" else None,
                         "algorithmic_bytes_per_param": k4_B,
                         "peak_source": ("MEASURED_PEAKS.json hbm_gbs (measured)" if "_fallback" not in peaks
                                         else "fallback 6650 GB/s") if k4_bound == "hbm" else
                         "B200_PROFILING.md measured peer copy 770 GB/s per direction",
                         "hbm_achieved_GBps": (k4_hbm_B * k4_elems / (k4_busy * 1e-3) / 1e9) if k4_busy > 0 else None,
                         "timing": "CUDA events around every launch on its lane stream, union of the launches' "
                                   "intervals over the timed region",
                         "frac_vs_live_allpull": ((k4_achieved / calib["nvlink_allpull_GBps_min_over_ranks"])
                                                  if (calib and k4_achieved and k4_bound == "nvlink") else None),
                         "busy_ms_per_step": k4_busy / args.steps, "launch_sum_ms_per_step": k4_ms / args.steps,
                         "achieved_per_launch_sum": k4_achieved_sum},
            "roofline_isolated": {
                "note": "same kernels, per-unit calls on one stream (no lane overlap), 2 rounds outside the timed "
                        "region; achieved = algorithmic bytes / the kernel's own CUDA-event time",
                "dominant": {"kernel": k4_name, "bound": k4_bound, "achieved": k4_iso, "peak": k4_peak,
                             "frac": (k4_iso / k4_peak) if k4_iso else None},
                "pg_norm": {"bytes_per_param": k1_B, "achieved": k1_iso, "peak": hbm_peak,
                            "frac": (k1_iso / hbm_peak) if k1_iso else None},
                "phases_ms_per_round": {k: v / 2 for k, v in iso_ms.items()}},
            "design_bound": design,
            "sync_roofline": {"t_roof_ms_nominal": t_roof_nom, "frac_nominal": t_roof_nom / ms_per_step,
                              "t_roof_ms_measured": t_roof_meas, "frac_measured": t_roof_meas / ms_per_step,
                              "bound": "hbm" if N == 1 else "nvlink", "hbm_B_per_param": b_hbm,
                              "nvlink_B_per_param_per_dir_bus_convention": 8.0 * (N - 1) / N,
                              "nvlink_B_per_param_per_dir_moved": b_nvl,
                              "note": "T_roof per BASELINE.md: max(P_r*(16+2b_l)/HBM, P_r*8(N-1)/N/NVLink); "
                                      "the peer path moves (b_l+4)(N-1)/N B/param, below the fp32 bus convention"},
            "phases_ms_per_step": {k: v / args.steps for k, v in phase_ms.items()},
            "phases_busy_ms_per_step": {k: v / args.steps for k, v in phase_busy_ms.items()},
            "per_gpu_GBps": bytes_per_rank_round / (ms_per_step * 1e-3) / 1e9,
            "rollbacks_last_round": rollbacks, "beta_sample": betas, "anomaly": anomaly,
            "anomaly_sweep": anomaly_sweep,
            "gpu_launches": launches, "clocks": clk, "e2e": e2e, "cpu_baseline": cpu, "overlap": overlap,
            "warmup_allreduce": warm, "fused_gather": gather, "calibration": calib,
        }
        print(json.dumps(line), flush=True)
    sync.close()
    if world > 1:
        dist.barrier(device_ids=[local_rank])
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
