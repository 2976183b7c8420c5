"""EDiT sync oracle -- TEST INFRASTRUCTURE ONLY.

A plain fp64 CPU implementation of Sync() (Alg. 2) and the
equations of Section 3.2 (Eq. 1-5), written in C
(``oracle/edit_oracle.c``) and wrapped here with ctypes + numpy.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It shares
no code with the CUDA path in ``paper_2412_07210_b200/`` and never imports it.
"""
from __future__ import annotations

import ctypes
import dataclasses
import math
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "edit_oracle.c")
_LIB = os.path.join(_HERE, "libedit_oracle.so")
_lock = threading.Lock()
_lib = None

MAX_SYNC = 8
NO_AE, NO_WA, NO_GC = 1, 2, 4


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C99 + OpenMP).  EDIT_ORACLE_LIB=<path> loads a
    prebuilt copy instead (tests/test_oracle_mutations.py: deliberately broken oracles)."""
    override = os.environ.get("EDIT_ORACLE_LIB")
    if override:
        return override
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Cfg(ctypes.Structure):
    _fields_ = [("outer_lr", ctypes.c_double), ("outer_momentum", ctypes.c_double),
                ("clip_threshold", ctypes.c_double), ("clip_eps", ctypes.c_double),
                ("anomaly_threshold", ctypes.c_double), ("ema_alpha", ctypes.c_double),
                ("ema_warmup_rounds", ctypes.c_int64), ("flags", ctypes.c_uint32),
                ("pad_", ctypes.c_uint32)]


class _Ema(ctypes.Structure):
    _fields_ = [("mu", ctypes.c_double), ("sigma", ctypes.c_double), ("count", ctypes.c_int64)]


class _Outcome(ctypes.Structure):
    _fields_ = [("G", ctypes.c_double * MAX_SYNC), ("z", ctypes.c_double * MAX_SYNC),
                ("anomalous", ctypes.c_int32 * MAX_SYNC), ("w", ctypes.c_double * MAX_SYNC),
                ("G_bar", ctypes.c_double), ("beta", ctypes.c_double),
                ("rollback", ctypes.c_int32), ("pad_", ctypes.c_int32)]


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P, D, I64, I32, U32 = ctypes.c_void_p, ctypes.c_double, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32
            lib.oracle_sq_norm.argtypes, lib.oracle_sq_norm.restype = [P, I64], D
            lib.oracle_is_anomaly.argtypes = [D, ctypes.POINTER(_Ema), ctypes.POINTER(_Cfg), ctypes.POINTER(D)]
            lib.oracle_is_anomaly.restype = ctypes.c_int
            lib.oracle_ema_update.argtypes, lib.oracle_ema_update.restype = [ctypes.POINTER(_Ema), D, D], None
            lib.oracle_penalty_weights.argtypes = [P, I32, U32, P]
            lib.oracle_penalty_weights.restype = ctypes.c_int
            lib.oracle_clip_beta.argtypes, lib.oracle_clip_beta.restype = [D, D, D, U32], D
            lib.oracle_outer_nesterov.argtypes, lib.oracle_outer_nesterov.restype = [P, P, P, I64, D, D], None
            lib.oracle_sync_unit.argtypes = [ctypes.POINTER(_Cfg), I32, I32, I64, I32, P, P, P, P,
                                             ctypes.POINTER(_Ema), ctypes.POINTER(_Outcome)]
            lib.oracle_sync_unit.restype = ctypes.c_int
            lib.oracle_f32_to_bf16_rne.argtypes, lib.oracle_f32_to_bf16_rne.restype = [ctypes.c_float], ctypes.c_uint16
            lib.oracle_bf16_to_f64.argtypes, lib.oracle_bf16_to_f64.restype = [ctypes.c_uint16], D
            lib.oracle_allreduce_mean.argtypes, lib.oracle_allreduce_mean.restype = [I32, I64, I32, P, P], None
            lib.oracle_set_threads.argtypes, lib.oracle_set_threads.restype = [ctypes.c_int], None
            lib.oracle_get_threads.argtypes, lib.oracle_get_threads.restype = [], ctypes.c_int
            _lib = lib
    return _lib


@dataclasses.dataclass
class Config:
    """Hyperparameters "as the paper states them" (R19): nu, mu, phi,
    delta, alpha; eps (value unstated, R12) and W (R8)."""
    outer_lr: float = 0.8
    outer_momentum: float = 0.85
    clip_threshold: float = 10.0
    clip_eps: float = 1e-6
    anomaly_threshold: float = 3.0
    ema_alpha: float = 0.02
    ema_warmup_rounds: int = 10
    flags: int = 0

    def _c(self) -> _Cfg:
        return _Cfg(self.outer_lr, self.outer_momentum, self.clip_threshold, self.clip_eps,
                    self.anomaly_threshold, self.ema_alpha, int(self.ema_warmup_rounds),
                    int(self.flags), 0)


@dataclasses.dataclass
class Ema:
    mu: float = 0.0
    sigma: float = 0.0
    count: int = 0


# ---------------------------------------------------------------- primitives
def set_threads(n: int) -> None:
    _load().oracle_set_threads(int(n))


def get_threads() -> int:
    return int(_load().oracle_get_threads())


def l2_norm(x) -> float:
    """sqrt(sum x_i^2) (the G of Alg. 2 l.443)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return math.sqrt(_load().oracle_sq_norm(x.ctypes.data, x.size))


def is_anomaly(G: float, ema: Ema, cfg: Config) -> tuple[bool, float]:
    """IsAnomaly of Alg. 2 l.444. Returns (flag, z)."""
    z = ctypes.c_double()
    e = _Ema(ema.mu, ema.sigma, ema.count)
    f = _load().oracle_is_anomaly(float(G), ctypes.byref(e), ctypes.byref(cfg._c()), ctypes.byref(z))
    return bool(f), z.value


def ema_update(ema: Ema, G: float, alpha: float = 0.02) -> Ema:
    """Eq. 1; skipped for infinite G."""
    e = _Ema(ema.mu, ema.sigma, ema.count)
    _load().oracle_ema_update(ctypes.byref(e), float(G), float(alpha))
    return Ema(e.mu, e.sigma, e.count)


def penalty_weights(G, flags: int = 0) -> tuple[np.ndarray, bool]:
    """Eq. 2 + the gamma == 0 rollback test (Alg. 2 l.447-448)."""
    G = np.ascontiguousarray(np.asarray(G, dtype=np.float64))
    w = np.zeros_like(G)
    rb = _load().oracle_penalty_weights(G.ctypes.data, G.size, int(flags), w.ctypes.data)
    return w, bool(rb)


def clip_beta(G_bar: float, phi: float = 10.0, eps: float = 1e-6, flags: int = 0) -> float:
    """Eq. 4."""
    return float(_load().oracle_clip_beta(float(G_bar), float(phi), float(eps), int(flags)))


def outer_nesterov(a, m, g, nu: float, mu: float) -> tuple[np.ndarray, np.ndarray]:
    """OuterOpt = Nesterov momentum, descent along g (R1, R2)."""
    a = np.array(a, dtype=np.float64)
    m = np.array(m, dtype=np.float64)
    g = np.ascontiguousarray(np.asarray(g, dtype=np.float64))
    _load().oracle_outer_nesterov(a.ctypes.data, m.ctypes.data, g.ctypes.data, a.size, float(nu), float(mu))
    return a, m


def f32_to_bf16_bits(x) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 (bit patterns), elementwise."""
    lib = _load()
    x = np.asarray(x, dtype=np.float32).ravel()
    return np.array([lib.oracle_f32_to_bf16_rne(float(v)) for v in x], dtype=np.uint16)


def bf16_bits_to_f64(h) -> np.ndarray:
    lib = _load()
    h = np.asarray(h, dtype=np.uint16).ravel()
    return np.array([lib.oracle_bf16_to_f64(int(v)) for v in h], dtype=np.float64)


# ------------------------------------------------------------ whole Alg. 2
@dataclasses.dataclass
class Outcome:
    G: np.ndarray
    z: np.ndarray
    anomalous: np.ndarray
    w: np.ndarray
    G_bar: float
    beta: float
    rollback: bool


def sync_unit(cfg: Config, locals_, anchors, momenta, ema: list[Ema]):
    """One Sync() (Alg. 2) of one module over the whole M x N mesh.

    locals_  : [M, N, numel] float32, or uint16 bf16 bit patterns
    anchors  : [M, numel] float32  (identical across each sync row)
    momenta  : [M, numel] float32
    ema      : N Ema records of this module (one per sync replica, R6)
    Returns (new_locals, new_anchors, new_momenta, new_ema, Outcome).
    Inputs are not modified.
    """
    loc = np.ascontiguousarray(locals_)
    if loc.ndim != 3:
        raise ValueError("locals must be [M, N, numel]")
    M, N, numel = loc.shape
    if loc.dtype == np.uint16:
        is_bf16 = 1
    elif loc.dtype == np.float32:
        is_bf16 = 0
    else:
        raise TypeError(f"locals dtype {loc.dtype}: need float32 or uint16 (bf16 bits)")
    anc = np.array(anchors, dtype=np.float32, copy=True).reshape(M, numel)
    mom = np.array(momenta, dtype=np.float32, copy=True).reshape(M, numel)
    out_loc = np.empty_like(loc)
    if len(ema) != N:
        raise ValueError("need one Ema per sync replica")
    e = (_Ema * MAX_SYNC)(*[_Ema(x.mu, x.sigma, x.count) for x in ema])
    o = _Outcome()
    rc = _load().oracle_sync_unit(ctypes.byref(cfg._c()), M, N, numel, is_bf16, loc.ctypes.data,
                                  anc.ctypes.data, mom.ctypes.data, out_loc.ctypes.data, e, ctypes.byref(o))
    if rc != 0:
        raise RuntimeError("oracle_sync_unit failed")
    new_ema = [Ema(e[i].mu, e[i].sigma, e[i].count) for i in range(N)]
    out = Outcome(G=np.array(o.G[:N]), z=np.array(o.z[:N]), anomalous=np.array(o.anomalous[:N], dtype=bool),
                  w=np.array(o.w[:N]), G_bar=o.G_bar, beta=o.beta, rollback=bool(o.rollback))
    return out_loc, anc, mom, new_ema, out


def allreduce_mean(grads) -> np.ndarray:
    """Warm-up gradient sync (Alg. 1 l.422-424): mean over the N members, rounded to the
    stored type.  grads: [N, numel] float32 or uint16 (bf16 bits)."""
    g = np.ascontiguousarray(grads)
    if g.ndim != 2 or g.dtype not in (np.float32, np.uint16):
        raise TypeError("grads must be [N, numel] float32 or uint16 (bf16 bits)")
    out = np.empty(g.shape[1], dtype=g.dtype)
    _load().oracle_allreduce_mean(g.shape[0], g.shape[1], int(g.dtype == np.uint16), g.ctypes.data, out.ctypes.data)
    return out
