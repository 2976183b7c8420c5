"""Thin ctypes binding of libedit_sync.so (include/edit_sync.h).

Argument marshalling only: every step of the sync runs in the library's CUDA
kernels and NCCL calls.  There is no CPU fallback -- if the shared library is
missing this module raises on import of the handle.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os

import numpy as np
import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libedit_sync.so")

MAX_SYNC = 8
UNIQUE_ID_BYTES = 128
EDIT_BF16, EDIT_F32 = 0, 1
ALGOS = {"peer": 0, "nccl": 1}
NO_AE, NO_WA, NO_GC = 1, 2, 4

EXPORTED = ("edit_sync_get_unique_id", "edit_sync_workspace_bytes", "edit_sync_init", "edit_layer_sync",
            "edit_layer_sync_host", "edit_sync_host_wait", "edit_sync_round", "edit_sync_register_locals",
            "edit_warmup_allreduce", "edit_warmup_allreduce_round", "edit_sync_register_gather", "edit_sched_begin_round", "edit_sched_acquire",
            "edit_sched_end_round", "edit_sched_set_partition", "edit_sched_get_plan",
            "edit_sync_stats", "edit_sync_get_state", "edit_sync_set_state", "edit_sync_kernel_launches",
            "edit_sync_nvlink_probe",
            "edit_sync_set_profiling", "edit_sync_profile_collect", "edit_trigger_create", "edit_trigger_sync_now",
            "edit_trigger_in_warmup", "edit_trigger_mark_synced", "edit_trigger_syncs", "edit_trigger_destroy",
            "edit_sync_destroy", "edit_sync_last_error", "edit_sync_version")

_STATUS = {0: "EDIT_OK", 1: "EDIT_ERR_INVALID_ARG", 2: "EDIT_ERR_CUDA", 3: "EDIT_ERR_NCCL",
           4: "EDIT_ERR_STATE", 5: "EDIT_ERR_NO_MEMORY"}


class EditSyncError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [("shard_dim", ctypes.c_int32), ("sync_dim", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("device", ctypes.c_int32), ("num_layers", ctypes.c_int32), ("param_dtype", ctypes.c_int32),
                ("layer_numel", ctypes.POINTER(ctypes.c_int64)), ("outer_lr", ctypes.c_float),
                ("outer_momentum", ctypes.c_float), ("clip_threshold", ctypes.c_float),
                ("clip_eps", ctypes.c_float), ("anomaly_threshold", ctypes.c_float),
                ("ema_alpha", ctypes.c_float), ("ema_warmup_rounds", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("algo", ctypes.c_int32)]


class LayerStatsC(ctypes.Structure):
    _fields_ = [("round", ctypes.c_int64), ("G", ctypes.c_double * MAX_SYNC), ("z", ctypes.c_double * MAX_SYNC),
                ("w", ctypes.c_double * MAX_SYNC), ("anomalous", ctypes.c_int32 * MAX_SYNC),
                ("G_bar", ctypes.c_double), ("beta", ctypes.c_double), ("rollback", ctypes.c_int32),
                ("num_sync", ctypes.c_int32), ("ema_mu", ctypes.c_double * MAX_SYNC),
                ("ema_sigma", ctypes.c_double * MAX_SYNC), ("ema_count", ctypes.c_int64 * MAX_SYNC)]


EMA_DTYPE = np.dtype([("mu", np.float64), ("sigma", np.float64), ("count", np.int64), ("reserved", np.int64)])

_lib = None


def load_library() -> ctypes.CDLL:
    """Load libedit_sync.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(python -m paper_2412_07210_b200.build); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, I64, S = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int
    lib.edit_sync_get_unique_id.argtypes, lib.edit_sync_get_unique_id.restype = [P], S
    lib.edit_sync_workspace_bytes.argtypes = [ctypes.POINTER(Config), ctypes.POINTER(ctypes.c_size_t)]
    lib.edit_sync_workspace_bytes.restype = S
    lib.edit_sync_init.argtypes = [ctypes.POINTER(Config), P, P, ctypes.c_size_t, ctypes.POINTER(P)]
    lib.edit_sync_init.restype = S
    lib.edit_layer_sync.argtypes, lib.edit_layer_sync.restype = [P, I32, P, P, P, P], S
    lib.edit_layer_sync_host.argtypes, lib.edit_layer_sync_host.restype = [P, I32, P, P, P, P], S
    lib.edit_sync_host_wait.argtypes, lib.edit_sync_host_wait.restype = [P, P], S
    lib.edit_sync_round.argtypes, lib.edit_sync_round.restype = [P, P, P, P, P], S
    lib.edit_sync_register_locals.argtypes, lib.edit_sync_register_locals.restype = [P, P], S
    lib.edit_warmup_allreduce.argtypes, lib.edit_warmup_allreduce.restype = [P, I32, P, P], S
    lib.edit_warmup_allreduce_round.argtypes, lib.edit_warmup_allreduce_round.restype = [P, P, P], S
    lib.edit_sync_register_gather.argtypes, lib.edit_sync_register_gather.restype = [P, P], S
    lib.edit_sched_begin_round.argtypes, lib.edit_sched_begin_round.restype = [P, P, P, P, I32, P], S
    lib.edit_sched_acquire.argtypes, lib.edit_sched_acquire.restype = [P, I32, P], S
    lib.edit_sched_end_round.argtypes, lib.edit_sched_end_round.restype = [P, P], S
    lib.edit_sched_set_partition.argtypes, lib.edit_sched_set_partition.restype = [P, I32, I32], S
    lib.edit_sched_get_plan.argtypes, lib.edit_sched_get_plan.restype = [P, P, P, P], S
    lib.edit_sync_stats.argtypes = [P, I32, ctypes.POINTER(LayerStatsC)]
    lib.edit_sync_stats.restype = S
    lib.edit_sync_get_state.argtypes = [P, P, ctypes.POINTER(ctypes.c_size_t)]
    lib.edit_sync_get_state.restype = S
    lib.edit_sync_set_state.argtypes, lib.edit_sync_set_state.restype = [P, P, ctypes.c_size_t], S
    lib.edit_sync_set_profiling.argtypes, lib.edit_sync_set_profiling.restype = [P, I32], S
    lib.edit_sync_profile_collect.argtypes = [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                              ctypes.POINTER(I64), ctypes.POINTER(I64)]
    lib.edit_sync_profile_collect.restype = S
    lib.edit_sync_kernel_launches.argtypes, lib.edit_sync_kernel_launches.restype = [P], I64
    lib.edit_sync_nvlink_probe.argtypes = [P, I64, I32, ctypes.POINTER(ctypes.c_double)]
    lib.edit_sync_nvlink_probe.restype = S
    lib.edit_sync_destroy.argtypes, lib.edit_sync_destroy.restype = [P], S
    D = ctypes.c_double
    lib.edit_trigger_create.argtypes = [I32, I64, D, I64, D, ctypes.POINTER(P)]
    lib.edit_trigger_create.restype = S
    lib.edit_trigger_sync_now.argtypes, lib.edit_trigger_sync_now.restype = [P, I64, D], I32
    lib.edit_trigger_in_warmup.argtypes, lib.edit_trigger_in_warmup.restype = [P, I64], I32
    lib.edit_trigger_mark_synced.argtypes, lib.edit_trigger_mark_synced.restype = [P, D], S
    lib.edit_trigger_syncs.argtypes, lib.edit_trigger_syncs.restype = [P], I64
    lib.edit_trigger_destroy.argtypes, lib.edit_trigger_destroy.restype = [P], S
    lib.edit_sync_last_error.argtypes, lib.edit_sync_last_error.restype = [], ctypes.c_char_p
    lib.edit_sync_version.argtypes, lib.edit_sync_version.restype = [], ctypes.c_char_p
    _lib = lib
    return lib


def _check(status: int) -> None:
    if status != 0:
        raise EditSyncError(status, load_library().edit_sync_last_error().decode())


def get_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * UNIQUE_ID_BYTES)()
    _check(load_library().edit_sync_get_unique_id(buf))
    return bytes(buf)


def broadcast_unique_id(group=None) -> bytes:
    """Rank 0 creates the NCCL id; every rank of `group` receives it (torch.distributed)."""
    import torch.distributed as dist
    obj = [get_unique_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


@dataclasses.dataclass
class LayerStats:
    round: int
    G: np.ndarray
    z: np.ndarray
    w: np.ndarray
    anomalous: np.ndarray
    G_bar: float
    beta: float
    rollback: bool
    ema_mu: np.ndarray
    ema_sigma: np.ndarray
    ema_count: np.ndarray


_DTYPES = {torch.bfloat16: EDIT_BF16, torch.float32: EDIT_F32}


class EditSync:
    """One rank's handle: EDiT layer-wise sync (Alg. 2) over an M x N mesh.

    layer_numel: per-rank padded shard length of every sync unit.
    Hyperparameter defaults are the paper's (R19): nu=0.8, mu=0.85,
    phi=10, delta=3, alpha=0.02, eps=1e-6 (R12), W=10 (R8).
    """

    def __init__(self, layer_numel, *, shard_dim: int = 1, sync_dim: int = 1, rank: int = 0,
                 device=None, param_dtype=torch.bfloat16, outer_lr: float = 0.8,
                 outer_momentum: float = 0.85, clip_threshold: float = 10.0, clip_eps: float = 1e-6,
                 anomaly_threshold: float = 3.0, ema_alpha: float = 0.02, ema_warmup_rounds: int = 10,
                 flags: int = 0, unique_id: bytes | None = None, algo: str = "peer"):
        self._lib = load_library()
        self._h = None
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        if dev.type != "cuda":
            raise ValueError("EditSync runs on a CUDA device only (no CPU fallback)")
        self.device = dev
        self.layer_numel = [int(x) for x in layer_numel]
        self.num_layers = len(self.layer_numel)
        self.shard_dim, self.sync_dim, self.rank = int(shard_dim), int(sync_dim), int(rank)
        self.param_dtype = param_dtype
        if param_dtype not in _DTYPES:
            raise TypeError("param_dtype must be torch.bfloat16 or torch.float32")
        self._numel_arr = (ctypes.c_int64 * max(1, self.num_layers))(*self.layer_numel)
        self._cfg = Config(self.shard_dim, self.sync_dim, self.rank, dev.index or 0, self.num_layers,
                           _DTYPES[param_dtype], self._numel_arr, outer_lr, outer_momentum, clip_threshold,
                           clip_eps, anomaly_threshold, ema_alpha, int(ema_warmup_rounds), int(flags),
                           ALGOS[algo])
        self.algo = algo
        nbytes = ctypes.c_size_t()
        _check(self._lib.edit_sync_workspace_bytes(ctypes.byref(self._cfg), ctypes.byref(nbytes)))
        # workspace from torch's allocator (256-byte aligned by the caching allocator)
        self.workspace = torch.empty(nbytes.value, dtype=torch.uint8, device=dev)
        idbuf = None
        if self.shard_dim * self.sync_dim > 1:
            if unique_id is None or len(unique_id) != UNIQUE_ID_BYTES:
                raise ValueError("a multi-rank mesh needs the 128-byte unique id (broadcast_unique_id)")
            idbuf = (ctypes.c_uint8 * UNIQUE_ID_BYTES).from_buffer_copy(unique_id)
        h = ctypes.c_void_p()
        with torch.cuda.device(dev):
            _check(self._lib.edit_sync_init(ctypes.byref(self._cfg), idbuf, self.workspace.data_ptr(),
                                            nbytes.value, ctypes.byref(h)))
        self._h = h

    # ------------------------------------------------------------------ sync
    def layer_sync(self, layer: int, local: torch.Tensor, anchor: torch.Tensor, momentum: torch.Tensor,
                   stream: torch.cuda.Stream | None = None) -> None:
        """Enqueue Sync() of one unit on `stream` (default: torch's current stream)."""
        n = self.layer_numel[layer] if 0 <= layer < self.num_layers else -1
        for name, t, dt in (("local", local, self.param_dtype), ("anchor", anchor, torch.float32),
                            ("momentum", momentum, torch.float32)):
            if t.device != self.device or t.dtype != dt or not t.is_contiguous() or t.numel() != n:
                raise ValueError(f"{name}: need a contiguous {dt} tensor of {n} elements on {self.device}, "
                                 f"got {t.dtype} {tuple(t.shape)} on {t.device}")
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(self._lib.edit_layer_sync(self._h, int(layer), local.data_ptr(), anchor.data_ptr(),
                                         momentum.data_ptr(), st.cuda_stream))

    def layer_sync_host(self, layer: int, local: torch.Tensor, anchor: torch.Tensor, momentum: torch.Tensor,
                        stream: torch.cuda.Stream | None = None) -> None:
        """Host-buffer variant (CPU-offloaded anchor/momentum): pinned CPU tensors in,
        results copied back in place.  Call host_wait() before touching them."""
        n = self.layer_numel[layer] if 0 <= layer < self.num_layers else -1
        for name, t, dt in (("local", local, self.param_dtype), ("anchor", anchor, torch.float32),
                            ("momentum", momentum, torch.float32)):
            if t.device.type != "cpu" or t.dtype != dt or not t.is_contiguous() or t.numel() != n:
                raise ValueError(f"{name}: need a contiguous host {dt} tensor of {n} elements")
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(self._lib.edit_layer_sync_host(self._h, int(layer), local.data_ptr(), anchor.data_ptr(),
                                              momentum.data_ptr(), st.cuda_stream))

    def host_wait(self, stream: torch.cuda.Stream | None = None) -> None:
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(self._lib.edit_sync_host_wait(self._h, st.cuda_stream))

    # ------------------------------------------------ prefetch scheduler (a8)
    def begin_round(self, locals_, anchors, momenta, depth: int = 1, stream=None) -> None:
        """Start a layer-wise prefetched round: syncs run on a side stream, unit u+depth
        is enqueued when the forward acquires unit u."""
        a, b, c = self._check_round(locals_, anchors, momenta)
        self._round_refs = (list(locals_), list(anchors), list(momenta))  # keep alive for the round
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(self._lib.edit_sched_begin_round(self._h, a, b, c, int(depth), st.cuda_stream))

    def acquire(self, layer: int, stream=None) -> None:
        """The forward of unit `layer` may use its params after this (stream-ordered)."""
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(self._lib.edit_sched_acquire(self._h, int(layer), st.cuda_stream))

    def end_round(self, stream=None) -> None:
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(self._lib.edit_sched_end_round(self._h, st.cuda_stream))
        self._round_refs = None

    def set_partition(self, sms: int, full_units: int = 2) -> None:
        """Scheduler partition mode (edit_sched_set_partition): units >= full_units sync on
        persistent TMA CTAs (one per SM) while the forward keeps the other SMs.  sms = -1
        (default): sized per unit from the measured forward; > 0: fixed; 0: full grids."""
        _check(self._lib.edit_sched_set_partition(self._h, int(sms), int(full_units)))

    PLAN_CANDIDATES = ("serial", "partition x1.0 depth>=2", "partition x1.6 depth>=2", "partition x1.0")

    def sched_plan(self) -> dict:
        """The scheduler's last-round plan (edit_sched_get_plan): the auto mode's candidate,
        the SMs each unit's sync got (0 full grid, -1 serial), median round ms per candidate."""
        cand = ctypes.c_int32()
        sms = (ctypes.c_int32 * self.num_layers)()
        med = (ctypes.c_double * 4)()
        _check(self._lib.edit_sched_get_plan(self._h, ctypes.byref(cand), sms, med))
        c = cand.value
        return {"candidate": self.PLAN_CANDIDATES[c] if 0 <= c < 4 else "fixed", "sms_per_unit": list(sms),
                "median_round_ms": dict(zip(self.PLAN_CANDIDATES, list(med)))}

    def _check_round(self, locals_, anchors, momenta):
        L = self.num_layers
        if not (len(locals_) == len(anchors) == len(momenta) == L):
            raise ValueError(f"need {L} units")
        for u in range(L):
            for name, t, dt in (("local", locals_[u], self.param_dtype), ("anchor", anchors[u], torch.float32),
                                ("momentum", momenta[u], torch.float32)):
                if t.device != self.device or t.dtype != dt or not t.is_contiguous() or \
                        t.numel() != self.layer_numel[u]:
                    raise ValueError(f"unit {u} {name}: wrong device/dtype/shape")
        arr = lambda ts: (ctypes.c_void_p * L)(*[t.data_ptr() for t in ts])
        return arr(locals_), arr(anchors), arr(momenta)

    def warmup_allreduce(self, layer: int, grad: torch.Tensor, stream=None) -> None:
        """Warm-up phase (Alg. 1 l.422-424): grad <- mean over the sync row, in place."""
        n = self.layer_numel[layer] if 0 <= layer < self.num_layers else -1
        if grad.device != self.device or grad.dtype != self.param_dtype or not grad.is_contiguous() or \
                grad.numel() != n:
            raise ValueError(f"grad: need a contiguous {self.param_dtype} tensor of {n} elements on {self.device}")
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(self._lib.edit_warmup_allreduce(self._h, int(layer), grad.data_ptr(), st.cuda_stream))

    def warmup_allreduce_round(self, grads, stream=None) -> None:
        """The warm-up all-reduce of every unit in one call, pipelined over the lanes."""
        L = self.num_layers
        if len(grads) != L:
            raise ValueError(f"need {L} gradient tensors")
        for u, g in enumerate(grads):
            if g.device != self.device or g.dtype != self.param_dtype or not g.is_contiguous() or \
                    g.numel() != self.layer_numel[u]:
                raise ValueError(f"unit {u} grad: wrong device/dtype/shape")
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        arr = (ctypes.c_void_p * L)(*[g.data_ptr() for g in grads])
        _check(self._lib.edit_warmup_allreduce_round(self._h, arr, st.cuda_stream))

    def register_gather(self, full_bufs) -> None:
        """NEXT-2: per unit a buffer of M * layer_numel elements that every sync fills with the
        whole module (each shard-group member stores its updated shard into it).  Collective."""
        L = self.num_layers
        if len(full_bufs) != L:
            raise ValueError(f"need {L} units")
        for u, t in enumerate(full_bufs):
            if t.device != self.device or t.dtype != self.param_dtype or not t.is_contiguous() or \
                    t.numel() != self.shard_dim * self.layer_numel[u]:
                raise ValueError(f"unit {u} gather buffer: need {self.shard_dim * self.layer_numel[u]} "
                                 f"{self.param_dtype} elements on {self.device}")
        self._gather = list(full_bufs)
        arr = (ctypes.c_void_p * L)(*[t.data_ptr() for t in full_bufs])
        _check(self._lib.edit_sync_register_gather(self._h, arr))

    def register_locals(self, locals_) -> None:
        """Peer path: let the sync row read these local buffers directly (CUDA IPC); they must
        stay allocated until close().  Collective."""
        L = self.num_layers
        if len(locals_) != L:
            raise ValueError(f"need {L} units")
        for u, t in enumerate(locals_):
            if t.device != self.device or t.dtype != self.param_dtype or not t.is_contiguous() or \
                    t.numel() != self.layer_numel[u]:
                raise ValueError(f"unit {u} local: wrong device/dtype/shape")
        self._registered = list(locals_)
        arr = (ctypes.c_void_p * L)(*[t.data_ptr() for t in locals_])
        _check(self._lib.edit_sync_register_locals(self._h, arr))

    def sync_round(self, locals_, anchors, momenta, stream=None) -> None:
        """One full round (all units), pipelined over the library's lanes (edit_sync_round)."""
        a, b, c = self._check_round(locals_, anchors, momenta)
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(self._lib.edit_sync_round(self._h, a, b, c, st.cuda_stream))

    # ------------------------------------------------------------- queries
    def stats(self, layer: int) -> LayerStats:
        s = LayerStatsC()
        _check(self._lib.edit_sync_stats(self._h, int(layer), ctypes.byref(s)))
        N = self.sync_dim
        return LayerStats(round=s.round, G=np.array(s.G[:N]), z=np.array(s.z[:N]), w=np.array(s.w[:N]),
                          anomalous=np.array(s.anomalous[:N], dtype=bool), G_bar=s.G_bar, beta=s.beta,
                          rollback=bool(s.rollback), ema_mu=np.array(s.ema_mu[:N]),
                          ema_sigma=np.array(s.ema_sigma[:N]), ema_count=np.array(s.ema_count[:N]))

    def get_state(self) -> np.ndarray:
        """EMA state [L, N] (mu, sigma, count)."""
        out = np.zeros((self.num_layers, self.sync_dim), dtype=EMA_DTYPE)
        nb = ctypes.c_size_t(out.nbytes)
        _check(self._lib.edit_sync_get_state(self._h, out.ctypes.data, ctypes.byref(nb)))
        return out

    def set_state(self, state: np.ndarray) -> None:
        st = np.ascontiguousarray(state, dtype=EMA_DTYPE).reshape(self.num_layers, self.sync_dim)
        _check(self._lib.edit_sync_set_state(self._h, st.ctypes.data, st.nbytes))

    def set_ema(self, mu, sigma, count) -> None:
        """Seed the EMA of every (unit, replica): arrays broadcastable to [L, N]."""
        st = np.zeros((self.num_layers, self.sync_dim), dtype=EMA_DTYPE)
        st["mu"], st["sigma"], st["count"] = mu, sigma, count
        self.set_state(st)

    PHASES = ("pg_norm", "gather_decide", "allreduce", "dbar_norm_gather", "outer_update")

    def set_profiling(self, enable: bool) -> None:
        _check(self._lib.edit_sync_set_profiling(self._h, 1 if enable else 0))

    def profile_collect(self) -> dict:
        """Per-phase CUDA-event ms summed over the syncs since the last collect, and per-phase
        busy ms (union of the units' intervals: overlapping lanes counted once)."""
        ms = (ctypes.c_double * len(self.PHASES))()
        busy = (ctypes.c_double * len(self.PHASES))()
        syncs, elems = ctypes.c_int64(), ctypes.c_int64()
        _check(self._lib.edit_sync_profile_collect(self._h, ms, busy, ctypes.byref(syncs), ctypes.byref(elems)))
        return {"ms": dict(zip(self.PHASES, list(ms))), "busy_ms": dict(zip(self.PHASES, list(busy))),
                "syncs": syncs.value, "elements": elems.value}

    def nvlink_probe(self, bytes_per_peer: int = 256 << 20, reps: int = 5) -> float:
        """Per-direction NVLink ingress GB/s of this rank with the whole sync row pulling from
        each other at once (collective over the row; edit_sync_nvlink_probe)."""
        out = ctypes.c_double()
        _check(self._lib.edit_sync_nvlink_probe(self._h, int(bytes_per_peer), int(reps), ctypes.byref(out)))
        return out.value

    @property
    def kernel_launches(self) -> int:
        return int(self._lib.edit_sync_kernel_launches(self._h))

    def close(self) -> None:
        if self._h is not None:
            self._lib.edit_sync_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class Trigger:
    """When to sync: EDiT's step trigger (Alg. 1 l.408) or A-EDiT's time trigger (§3.3).

    Trigger.steps(tau, t_warm) / Trigger.time(tau_time_s, t_warm, start_time_s).  Ask
    sync_now(step, now) at the start of every inner step; call mark_synced(now) after the sync."""

    def __init__(self, kind: int, tau_steps: int = 1, tau_time_s: float = 0.0, t_warm: int = 0,
                 start_time_s: float = 0.0):
        self._lib = load_library()
        h = ctypes.c_void_p()
        _check(self._lib.edit_trigger_create(int(kind), int(tau_steps), float(tau_time_s), int(t_warm),
                                             float(start_time_s), ctypes.byref(h)))
        self._h = h

    @classmethod
    def steps(cls, tau: int, t_warm: int = 0) -> "Trigger":
        return cls(0, tau_steps=tau, t_warm=t_warm)

    @classmethod
    def time(cls, tau_time_s: float, t_warm: int = 0, start_time_s: float = 0.0) -> "Trigger":
        return cls(1, tau_time_s=tau_time_s, t_warm=t_warm, start_time_s=start_time_s)

    def sync_now(self, step: int, now_s: float = 0.0) -> bool:
        return bool(self._lib.edit_trigger_sync_now(self._h, int(step), float(now_s)))

    def in_warmup(self, step: int) -> bool:
        return bool(self._lib.edit_trigger_in_warmup(self._h, int(step)))

    def mark_synced(self, now_s: float = 0.0) -> None:
        _check(self._lib.edit_trigger_mark_synced(self._h, float(now_s)))

    @property
    def syncs(self) -> int:
        return int(self._lib.edit_trigger_syncs(self._h))

    def __del__(self):
        try:
            if self._h:
                self._lib.edit_trigger_destroy(self._h)
                self._h = None
        except Exception:
            pass
