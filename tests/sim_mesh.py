"""TEST INFRASTRUCTURE: a simulated M x N mesh on one GPU (tests/sim/libedit_sim.so).

K = M*N member handles live in this process on one device; the shim wires them like
edit_sync_init wires real ranks (mailboxes, peer buffers, registered locals, gather buffers)
and drives them through the library's own enqueue functions, one stream per member, so the
N > 1 production kernels (K1 + folded norm exchange + K2, RS + folded Dbar-norm exchange,
AG + update, the fused shard all-gather, the peer warm-up) run and can be compared with the
whole-mesh oracle on a 1-GPU box.  Each member is exposed as an EditSync object (the product
binding: stats / get_state / set_state / set_ema go through the product C ABI)."""
from __future__ import annotations

import ctypes
import os

import torch

from paper_2412_07210_b200 import edit_sync as es

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


def load():
    global _lib
    if _lib is None:
        import importlib.util
        spec = importlib.util.spec_from_file_location("sim_build", os.path.join(_HERE, "sim", "build.py"))
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        es.load_library()  # the product library first (the shim links against it)
        lib = ctypes.CDLL(mod.build())
        P, I32, S = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int
        lib.edit_sim_create.argtypes, lib.edit_sim_create.restype = [ctypes.POINTER(es.Config), P, ctypes.c_size_t, P], S
        lib.edit_sim_register_locals.argtypes, lib.edit_sim_register_locals.restype = [P, S, P], S
        lib.edit_sim_register_gather.argtypes, lib.edit_sim_register_gather.restype = [P, S, P], S
        lib.edit_sim_layer_sync.argtypes, lib.edit_sim_layer_sync.restype = [P, S, I32, P, P, P, P], S
        lib.edit_sim_round.argtypes, lib.edit_sim_round.restype = [P, S, P, P, P, P], S
        lib.edit_sim_warmup_allreduce.argtypes, lib.edit_sim_warmup_allreduce.restype = [P, S, I32, P, P], S
        lib.edit_sim_warmup_allreduce_round.argtypes, lib.edit_sim_warmup_allreduce_round.restype = [P, S, P, P], S
        _lib = lib
    return _lib


def _ptrs(ts):
    return (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


class SimMesh:
    """members[k] = rank k (m = k % M, n = k // M, R20)."""

    def __init__(self, layer_numel, M, N, device, param_dtype=torch.bfloat16, outer_lr=0.8, outer_momentum=0.85,
                 clip_threshold=10.0, clip_eps=1e-6, anomaly_threshold=3.0, ema_alpha=0.02, ema_warmup_rounds=10,
                 flags=0):
        self.lib = load()
        self.M, self.N, self.K = M, N, M * N
        self.device = torch.device(device)
        self.layer_numel = [int(x) for x in layer_numel]
        L = len(self.layer_numel)
        self._numel_arr = (ctypes.c_int64 * max(1, L))(*self.layer_numel)
        self._cfg = es.Config(M, N, 0, self.device.index or 0, L, es._DTYPES[param_dtype], self._numel_arr, outer_lr,
                              outer_momentum, clip_threshold, clip_eps, anomaly_threshold, ema_alpha,
                              int(ema_warmup_rounds), int(flags), 0)
        plib = es.load_library()
        # the members' exchange kernels wait on each other from different streams of this one
        # context; the library's step-major enqueue keeps every wait satisfiable, and a short
        # exchange timeout turns any unforeseen non-concurrency into a fast test failure (the
        # first timeout poisons the handles: later exchanges return at once) instead of a hang
        os.environ.setdefault("EDIT_XCHG_TIMEOUT_S", "60")
        nbytes = ctypes.c_size_t()
        es._check(plib.edit_sync_workspace_bytes(ctypes.byref(self._cfg), ctypes.byref(nbytes)))
        self.workspaces = [torch.empty(nbytes.value, dtype=torch.uint8, device=self.device) for _ in range(self.K)]
        self._h = (ctypes.c_void_p * self.K)()
        with torch.cuda.device(self.device):
            rc = self.lib.edit_sim_create(ctypes.byref(self._cfg), _ptrs(self.workspaces), nbytes.value, self._h)
        if rc != 0:
            for h in self._h:
                if h:
                    plib.edit_sync_destroy(h)
            es._check(rc)
        self.members = []
        for k in range(self.K):
            e = es.EditSync.__new__(es.EditSync)  # product binding around an existing handle
            e._lib, e._h, e.device = plib, ctypes.c_void_p(self._h[k]), self.device
            e.layer_numel, e.num_layers = self.layer_numel, L
            e.shard_dim, e.sync_dim, e.rank, e.param_dtype, e.algo = M, N, k, param_dtype, "peer"
            e.workspace = self.workspaces[k]
            e._owned_by_sim = True
            self.members.append(e)
        self.streams = [torch.cuda.Stream(self.device) for _ in range(self.K)]

    # ---------------------------------------------------------------- helpers
    def _fork(self, members):
        cur = torch.cuda.current_stream(self.device)
        for k in members:
            self.streams[k].wait_stream(cur)

    def _join(self, members):
        cur = torch.cuda.current_stream(self.device)
        for k in members:
            cur.wait_stream(self.streams[k])

    def _handles(self, members):
        return (ctypes.c_void_p * len(members))(*[self._h[k] for k in members])

    def _streams(self, members):
        return (ctypes.c_void_p * len(members))(*[self.streams[k].cuda_stream for k in members])

    # ---------------------------------------------------------------- API
    def layer_sync(self, layer, locals_, anchors, momenta, members=None):
        """edit_layer_sync of unit `layer` on every member (or the given subset); buffers [K]."""
        members = list(range(self.K)) if members is None else list(members)
        self._fork(members)
        rc = self.lib.edit_sim_layer_sync(self._handles(members), len(members), int(layer),
                                          _ptrs([locals_[k] for k in members]), _ptrs([anchors[k] for k in members]),
                                          _ptrs([momenta[k] for k in members]), self._streams(members))
        self._join(members)
        es._check(rc)

    def sync_round(self, locals_, anchors, momenta):
        """edit_sync_round on every member; buffers [K][L]."""
        members = list(range(self.K))
        flat = lambda xs: _ptrs([t for row in xs for t in row])
        self._fork(members)
        rc = self.lib.edit_sim_round(self._handles(members), self.K, flat(locals_), flat(anchors), flat(momenta),
                                     self._streams(members))
        self._join(members)
        es._check(rc)

    def warmup_allreduce(self, layer, grads):
        members = list(range(self.K))
        self._fork(members)
        rc = self.lib.edit_sim_warmup_allreduce(self._handles(members), self.K, int(layer), _ptrs(grads),
                                                self._streams(members))
        self._join(members)
        es._check(rc)

    def warmup_allreduce_round(self, grads):
        """grads [K][L]: every unit of every member, pipelined over each member's lanes."""
        members = list(range(self.K))
        self._fork(members)
        rc = self.lib.edit_sim_warmup_allreduce_round(self._handles(members), self.K,
                                                      _ptrs([t for row in grads for t in row]), self._streams(members))
        self._join(members)
        es._check(rc)

    def register_locals(self, locals_):
        self._reg = locals_
        es._check(self.lib.edit_sim_register_locals(self._handles(range(self.K)), self.K,
                                                    _ptrs([t for row in locals_ for t in row])))

    def register_gather(self, bufs):
        self._gather = bufs
        es._check(self.lib.edit_sim_register_gather(self._handles(range(self.K)), self.K,
                                                    _ptrs([t for row in bufs for t in row])))

    def close(self):
        if not self.members:
            return
        try:
            torch.cuda.synchronize(self.device)
        except Exception:
            pass
        for e in self.members:
            e.close()
        self.members = []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
