"""Oracle parity of the N > 1 path on ONE GPU: a simulated M x N mesh (tests/sim_mesh.py).

The K members of a mesh run in this process on cuda:0, each with its own handle and stream,
through the library's production enqueue sequence (K1 with the folded norm exchange and K2,
RS with the folded Dbar-norm exchange, AG + update, the fused shard all-gather barrier, the
peer warm-up), with every member's mailbox and peer buffers wired as on a real node.  Rank 0
of a real run would regenerate every rank's inputs (synth/); here the test does, runs the
fp64 oracle (oracle/) for the whole mesh, and compares every member element by element
(tolerances of tests/parity.py, R17), plus the cross-rank invariants: anchors bitwise
identical along a sync row, local == rne(anchor), identical EMA state on every member.

PAPER.md: Eq. 1-5, Alg. 2 l.442-455, the mesh of P:61."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from tests import parity

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2412_07210_b200 import NO_WA, EditSyncError  # noqa: E402
from tests.sim_mesh import SimMesh  # noqa: E402

DEV = torch.device("cuda", 0)
DTYPES = {"bf16": torch.bfloat16, "f32": torch.float32}


def _units(config):
    """(units, oracle cfg, plant {(unit, n): factor}, seed_ema, nan_unit)."""
    cfg, plant, seed_ema, nan_unit = oracle.Config(), {}, True, None
    if config == "toy":          # BASELINE configs[0]: 4 layers x 64K fp32, replica 1 planted x4
        units = synth.toy_units(4, 65536)
        plant = {(i, 1): 4.0 for i in range(4)}
    elif config == "toy_clip":   # phi = 0.3: beta ~ 0.59 (Eq. 4 active)
        units = synth.toy_units(4, 65536)
        cfg = oracle.Config(clip_threshold=0.3)
    elif config == "ragged":     # ragged tails, a 7-element unit, several tiles per slice
        units = [synth.Unit("a", 1_000_003, ((999_000, 1003),)), synth.Unit("b", 7, ()),
                 synth.Unit("c", 3 * 65536 + 5, ())]
        seed_ema = False
    elif config == "rollback":   # every replica anomalous -> Alg. 2 l.449
        units = synth.toy_units(2, 40_000)
        plant = {(i, n): 4.0 for i in range(2) for n in range(8)}
    elif config == "nan":        # replica N-1 holds a NaN param in unit 0 (R9)
        units = [synth.Unit("a", 300_001, ()), synth.Unit("b", 9, ())]
        seed_ema, nan_unit = False, 0
    elif config == "nowa":       # NO_WA ablation: uniform weights over the finite G
        units = synth.toy_units(2, 65536)
        cfg = oracle.Config(flags=NO_WA)
        plant = {(0, 0): 4.0}
    elif config == "wrap":       # enough tiles that every persistent RS/AG CTA wraps its ring
        units = [synth.Unit("big", 16_000_003, ())]
    elif config == "many_small":  # 20 small units: two groups (kMaxGroup = 16) in the round API;
        # a planted replica in unit 3, every replica planted (rollback) in unit 5
        sizes = [7, 65539, 1000, 300_001, 8, 123_457, 4096, 77_777]
        units = [synth.Unit(f"s{i}", sizes[i % 8] + i, ()) for i in range(20)]
        plant = {(3, 1): 4.0, **{(5, n): 4.0 for n in range(8)}}
    elif config == "llama7b_layer0":  # a full-size 7B decoder unit (202,383,360 params)
        units = [synth.llama_units("7B")[1]]
    elif config == "llama350m":  # 350M-shaped units: embedding, decoder layer 0, head
        all_units = synth.llama_units("350M")
        units = [all_units[0], all_units[1], all_units[33]]
    else:
        raise ValueError(config)
    return units, cfg, plant, seed_ema, nan_unit


class MeshCase:
    def __init__(self, mesh, dtype_s, config, lanes=None):
        self.M, self.N = (int(x) for x in mesh.split("x"))
        M, N = self.M, self.N
        self.K = M * N
        self.mesh, self.dtype_s, self.config = mesh, dtype_s, config
        self.dtype = DTYPES[dtype_s]
        self.units, self.cfg, plant, seed_ema, self.nan_unit = _units(config)
        self.plant = {k: v for k, v in plant.items() if k[1] < N}
        self.recipe = synth.Recipe()
        self.numel = [synth.shard_numel(u.numel, M) for u in self.units]
        self.full = None
        if lanes is not None:
            os.environ["EDIT_LANES"] = str(lanes)
        try:
            c = self.cfg
            self.sim = SimMesh(self.numel, M, N, DEV, self.dtype, outer_lr=c.outer_lr, outer_momentum=c.outer_momentum,
                               clip_threshold=c.clip_threshold, clip_eps=c.clip_eps,
                               anomaly_threshold=c.anomaly_threshold, ema_alpha=c.ema_alpha,
                               ema_warmup_rounds=c.ema_warmup_rounds, flags=c.flags)
        finally:
            os.environ.pop("EDIT_LANES", None)
        L = len(self.units)
        self.ema0 = [[oracle.Ema() for _ in range(N)] for _ in range(L)]
        if seed_ema:
            mu = np.array([[synth.ema_seed(u, n, self.recipe)[0] for n in range(N)] for u in self.units])
            for e in self.sim.members:
                e.set_ema(mu, 0.1 * mu, self.recipe.ema_warmup_rounds)
            self.ema0 = [[oracle.Ema(mu[i, n], 0.1 * mu[i, n], self.recipe.ema_warmup_rounds) for n in range(N)]
                         for i in range(L)]
        # every member's inputs (rank k: m = k % M, n = k // M)
        self.loc, self.anc, self.mom = [], [], []
        for k in range(self.K):
            m, n = k % M, k // M
            a = [synth.shard_anchor(u, i, M, m, DEV, self.recipe) for i, u in enumerate(self.units)]
            mo = [synth.shard_momentum(u, i, M, m, DEV, self.recipe) for i, u in enumerate(self.units)]
            lo = [synth.shard_local(u, i, M, m, n, a[i], self.dtype, DEV, self.recipe, self.plant.get((i, n), 1.0))
                  for i, u in enumerate(self.units)]
            if self.nan_unit is not None and n == N - 1:
                lo[self.nan_unit][1234 % lo[self.nan_unit].numel()] = float("nan")
            self.anc.append(a)
            self.mom.append(mo)
            self.loc.append(lo)
        # the oracle's inputs, taken before the sync (as a real rank 0 would regenerate them)
        self.o_in = []
        for i in range(L):
            locs = np.stack([np.stack([parity.to_oracle_local(self.loc[n * M + m][i]) for n in range(N)])
                             for m in range(M)])
            ancs = np.stack([self.anc[m][i].cpu().numpy() for m in range(M)])
            moms = np.stack([self.mom[m][i].cpu().numpy() for m in range(M)])
            self.o_in.append((locs, ancs, moms))

    def run(self, api):
        L = len(self.units)
        self.full = None
        if api == "reg":
            self.sim.register_locals(self.loc)
        if api == "gather":
            self.full = [[torch.zeros(self.M * n_, dtype=self.dtype, device=DEV) for n_ in self.numel]
                         for _ in range(self.K)]
            self.sim.register_gather(self.full)
        if api in ("round", "reg", "gather"):
            self.sim.sync_round(self.loc, self.anc, self.mom)
        elif api == "unit":
            for i in range(L):
                self.sim.layer_sync(i, [x[i] for x in self.loc], [x[i] for x in self.anc], [x[i] for x in self.mom])
        else:
            raise ValueError(api)
        torch.cuda.synchronize()

    def check(self, api="unit"):
        M, N, K = self.M, self.N, self.K
        st = [e.get_state() for e in self.sim.members]
        for k in range(K):  # R6: every member keeps all N replicas' EMA, updated identically
            assert np.array_equal(st[k], st[0]), f"EMA state of member {k} differs"
        outs = []
        for i, u in enumerate(self.units):
            locs, ancs, moms = self.o_in[i]
            o_loc, o_anc, o_mom, o_ema, out = oracle.sync_unit(self.cfg, locs, ancs, moms, self.ema0[i])
            outs.append(out)
            for k in range(K):
                m, n = k % M, k // M
                tag = f"{self.config} {self.mesh} {self.dtype_s} {api} unit {i} member {k} (m={m}, n={n})"
                parity.assert_outcome(self.sim.members[k].stats(i), out, o_ema, tag)
                anc = self.anc[k][i].cpu().numpy()
                parity.assert_f32_close(anc, o_anc[m], tag + " anchor")
                parity.assert_f32_close(self.mom[k][i].cpu().numpy(), o_mom[m], tag + " momentum")
                parity.assert_local_close(parity.to_oracle_local(self.loc[k][i]), o_loc[m, n], tag + " local")
                assert np.array_equal(anc, self.anc[m][i].cpu().numpy()), tag + " anchors differ along the sync row"
                assert torch.equal(self.loc[k][i], self.anc[k][i].to(self.dtype)), tag + " local != rne(anchor)"
            if self.full is not None and M > 1:  # NEXT-2: gathered module == the shard group's locals
                nl = self.numel[i]
                for k in range(K):
                    n = k // M
                    f = self.full[k][i]
                    for q in range(M):
                        assert torch.equal(f[q * nl:(q + 1) * nl], self.loc[n * M + q][i]), \
                            f"gathered module of member {k}, shard {q}, unit {i}"
        return outs

    def close(self):
        self.sim.close()


# (mesh, dtype, config, api): every N > 1 feature on 1-GPU-runnable simulated meshes,
# including the 8-rank meshes of BASELINE.json (1x8, 2x4, 4x2) no test box has GPUs for
CASES = [
    ("2x2", "f32", "toy", "unit"), ("2x2", "f32", "toy", "round"), ("2x2", "f32", "toy_clip", "unit"),
    ("1x2", "bf16", "ragged", "unit"), ("1x2", "bf16", "ragged", "reg"), ("2x1", "bf16", "ragged", "round"),
    ("1x4", "bf16", "ragged", "round"), ("1x8", "bf16", "ragged", "reg"), ("2x4", "bf16", "ragged", "round"),
    ("4x2", "bf16", "ragged", "unit"), ("8x1", "bf16", "ragged", "round"),
    ("1x2", "bf16", "rollback", "unit"), ("2x2", "bf16", "rollback", "round"), ("1x8", "bf16", "rollback", "reg"),
    ("1x2", "bf16", "nan", "unit"), ("1x4", "bf16", "nan", "round"), ("2x4", "f32", "nan", "reg"),
    ("1x4", "bf16", "nowa", "unit"), ("2x2", "bf16", "nowa", "reg"),
    ("2x1", "bf16", "ragged", "gather"), ("2x2", "f32", "toy", "gather"), ("4x2", "bf16", "ragged", "gather"),
    ("2x4", "bf16", "rollback", "gather"),
    ("1x8", "bf16", "llama350m", "reg"), ("2x4", "bf16", "llama350m", "round"), ("4x2", "f32", "llama350m", "gather"),
    ("1x2", "bf16", "wrap", "reg"), ("1x4", "f32", "wrap", "unit"),
]


@pytest.mark.parametrize("mesh,dtype,config,api", CASES, ids=["-".join(c) for c in CASES])
def test_sim_mesh_parity(mesh, dtype, config, api):
    c = MeshCase(mesh, dtype, config)
    try:
        c.run(api)
        outs = c.check(api)
    finally:
        c.close()
    M, N = c.M, c.N
    if config == "toy":           # the planted replica gets w = 0 exactly and the rest is normal
        for o in outs:
            assert o.anomalous[1] and o.w[1] == 0.0 and not o.rollback
    if config == "toy_clip":
        assert all(o.beta < 1.0 for o in outs)
    if config == "rollback":
        assert all(o.rollback for o in outs)
    if config == "nan":
        assert outs[0].anomalous[N - 1] and outs[0].rollback == (N == 1)
    if config == "nowa" and N > 1:
        assert outs[0].anomalous[0] and np.allclose(outs[0].w[1:], 1.0 / (N - 1))


TMA_CASES = [("2x2", "f32", "toy", "unit"), ("1x4", "bf16", "ragged", "round"), ("1x2", "bf16", "wrap", "reg"),
             ("2x4", "bf16", "nan", "gather"), ("1x8", "bf16", "rollback", "round")]


@pytest.mark.parametrize("mesh,dtype,config,api", TMA_CASES, ids=["-".join(c) for c in TMA_CASES])
def test_sim_mesh_parity_tma_peer_kernels(mesh, dtype, config, api):
    # the persistent TMA RS / AG pipelines at full grids (EDIT_PEER_KERNELS=tma; the default
    # full-speed kernels are the LDG ones, the TMA ones also serve the scheduler's partition mode)
    os.environ["EDIT_PEER_KERNELS"] = "tma"
    try:
        c = MeshCase(mesh, dtype, config)
    finally:
        os.environ.pop("EDIT_PEER_KERNELS", None)
    try:
        c.run(api)
        c.check(api)
    finally:
        c.close()


@pytest.mark.parametrize("mesh,dtype,config,api", TMA_CASES[:3], ids=["-".join(c) for c in TMA_CASES[:3]])
def test_sim_mesh_parity_ldg_reduce_scatter(mesh, dtype, config, api):
    # EDIT_PEER_KERNELS=ldgall: the LDG full-grid reduce-scatter variant as well
    os.environ["EDIT_PEER_KERNELS"] = "ldgall"
    try:
        c = MeshCase(mesh, dtype, config)
    finally:
        os.environ.pop("EDIT_PEER_KERNELS", None)
    try:
        c.run(api)
        c.check(api)
    finally:
        c.close()


def test_sim_mesh_two_rounds_and_ring_wrap_small_grid():
    # EDIT_PEER_KERNELS=tma, EDIT_PEER_CTAS=8: a 1M-element unit needs ~15 RS tiles and ~30 AG
    # tiles per CTA, so both mbarrier rings wrap several times; then a second round on the
    # updated state
    os.environ["EDIT_PEER_CTAS"] = "8"
    os.environ["EDIT_PEER_KERNELS"] = "tma"   # the persistent TMA pipelines (partition mode's kernels)
    try:
        c = MeshCase("1x4", "bf16", "ragged")
    finally:
        os.environ.pop("EDIT_PEER_CTAS", None)
        os.environ.pop("EDIT_PEER_KERNELS", None)
    try:
        c.run("round")
        c.check("round")
        # round 2: fresh locals from the updated anchors (oracle state == GPU state within R17;
        # take the GPU's, which is bitwise identical along each row, as the next inputs)
        L = len(c.units)
        ema_gpu = c.sim.members[0].get_state()
        c.ema0 = [[oracle.Ema(float(ema_gpu[i, n]["mu"]), float(ema_gpu[i, n]["sigma"]), int(ema_gpu[i, n]["count"]))
                   for n in range(c.N)] for i in range(L)]
        for k in range(c.K):
            m, n = k % c.M, k // c.M
            for i, u in enumerate(c.units):
                c.loc[k][i].copy_(synth.shard_local(u, i, c.M, m, n, c.anc[k][i], c.dtype, DEV, c.recipe, 1.0, 1))
        c.o_in = []
        for i in range(L):
            locs = np.stack([np.stack([parity.to_oracle_local(c.loc[n * c.M + m][i]) for n in range(c.N)])
                             for m in range(c.M)])
            c.o_in.append((locs, np.stack([c.anc[m][i].cpu().numpy() for m in range(c.M)]),
                           np.stack([c.mom[m][i].cpu().numpy() for m in range(c.M)])))
        c.run("round")
        c.check("round")
        assert c.sim.members[0].stats(0).round == 2
    finally:
        c.close()


def test_sim_mesh_alternating_caller_streams():
    # edit_layer_sync on a different caller stream per unit, no host sync in between: every
    # call reuses lane 0's exchange buffers, so each must be ordered after the previous one
    # (include/edit_sync.h, "Stream order"); results must still match the oracle exactly
    c = MeshCase("1x4", "bf16", "ragged")
    try:
        other = [torch.cuda.Stream(DEV) for _ in range(c.K)]
        base = c.sim.streams
        for i in range(len(c.units)):
            c.sim.streams = other if i % 2 else base
            c.sim.layer_sync(i, [x[i] for x in c.loc], [x[i] for x in c.anc], [x[i] for x in c.mom])
        c.sim.streams = base
        torch.cuda.synchronize()
        c.check("unit")
    finally:
        c.close()


@pytest.mark.parametrize("mesh,dtype,api", [("1x2", "bf16", "unit"), ("1x2", "f32", "unit"), ("2x2", "bf16", "unit"),
                                            ("1x4", "f32", "unit"), ("2x4", "bf16", "unit"), ("1x8", "bf16", "unit"),
                                            ("1x2", "bf16", "round"), ("1x4", "bf16", "round"),
                                            ("2x4", "f32", "round"), ("1x8", "bf16", "round")])
def test_sim_mesh_warmup_allreduce(mesh, dtype, api):
    # NEXT-3 (Alg. 1 l.422-424): grad <- mean over the sync row, peer-memory kernels, against
    # oracle.allreduce_mean; bit-identical along every row
    M, N = (int(x) for x in mesh.split("x"))
    units = [synth.Unit("a", 1_000_003, ()), synth.Unit("b", 13, ()), synth.Unit("c", 65_536, ())]
    numel = [synth.shard_numel(u.numel, M) for u in units]
    dt = DTYPES[dtype]
    sim = SimMesh(numel, M, N, DEV, dt)
    try:
        grads = []
        for k in range(M * N):
            m, n = k % M, k // M
            row = []
            for i, u in enumerate(units):
                g = synth._randn(numel[i], synth.seed_of(5, i, m, n), DEV).mul_(1e-3)
                g[max(0, min(numel[i], u.numel - m * numel[i])):] = 0
                row.append(g.to(dt))
            grads.append(row)
        inputs = [[parity.to_oracle_local(g) for g in row] for row in grads]
        if api == "round":   # every unit in one call, pipelined over the lanes
            sim.warmup_allreduce_round(grads)
        else:
            for i in range(len(units)):
                sim.warmup_allreduce(i, [grads[k][i] for k in range(M * N)])
        torch.cuda.synchronize()
        for i in range(len(units)):
            for m in range(M):
                ref = oracle.allreduce_mean(np.stack([inputs[n * M + m][i] for n in range(N)]))
                for n in range(N):
                    got = parity.to_oracle_local(grads[n * M + m][i])
                    parity.assert_local_close(got, ref, f"warm {mesh} unit {i} member {n * M + m}")
                    assert np.array_equal(got, parity.to_oracle_local(grads[m][i])), "sync row members differ"
    finally:
        sim.close()


def test_sim_mesh_silent_peer_poisons_instead_of_applying_stale_data():
    # a peer that stops syncing must not let the others apply stale data.  1x2
    # mesh, member 1 never calls: member 0's norm exchange times out (EDIT_XCHG_TIMEOUT_S),
    # it writes nothing, and every later call returns EDIT_ERR_STATE
    os.environ["EDIT_XCHG_TIMEOUT_S"] = "0.5"
    try:
        c = MeshCase("1x2", "bf16", "toy")
    finally:
        os.environ.pop("EDIT_XCHG_TIMEOUT_S", None)
    try:
        before = [t.clone() for t in (c.loc[0][0], c.anc[0][0], c.mom[0][0])]
        c.sim.layer_sync(0, [c.loc[0][0]], [c.anc[0][0]], [c.mom[0][0]], members=[0])
        torch.cuda.synchronize()
        with pytest.raises(EditSyncError, match="EDIT_ERR_STATE"):
            c.sim.members[0].stats(0)
        for t, b in zip((c.loc[0][0], c.anc[0][0], c.mom[0][0]), before):
            assert torch.equal(t, b), "a timed-out member wrote its buffers"
        with pytest.raises(EditSyncError, match="EDIT_ERR_STATE"):
            c.sim.layer_sync(1, [c.loc[0][1]], [c.anc[0][1]], [c.mom[0][1]], members=[0])
        assert c.sim.members[1].stats(0).round == 0  # the silent member: untouched, healthy
    finally:
        c.close()


# Unit groups (internal.h GroupArgs): edit_sync_round syncs runs of consecutive small units with
# one K1 / RS / AG launch and one exchange message per phase.  (mesh, dtype, config, api,
# EDIT_GROUP_NUMEL): the default cap (32 Mi elements) groups every unit of these configs; 300,000
# splits "ragged" into {a} + {b, c}; 0 turns groups off (the single-unit round path).
GROUP_CASES = [
    ("1x4", "bf16", "many_small", "round", None), ("1x2", "f32", "many_small", "reg", None),
    ("2x4", "bf16", "many_small", "round", None), ("1x8", "bf16", "many_small", "reg", None),
    ("2x2", "bf16", "many_small", "round", None), ("1x2", "bf16", "ragged", "round", "300000"),
    ("1x4", "bf16", "ragged", "round", "0"), ("2x2", "f32", "toy", "round", "0"), ("1x8", "bf16", "nan", "reg", "0"),
]


@pytest.mark.parametrize("mesh,dtype,config,api,cap", GROUP_CASES, ids=["-".join(map(str, c)) for c in GROUP_CASES])
def test_sim_mesh_unit_groups(mesh, dtype, config, api, cap):
    if cap is not None:
        os.environ["EDIT_GROUP_NUMEL"] = cap
    try:
        c = MeshCase(mesh, dtype, config)
    finally:
        os.environ.pop("EDIT_GROUP_NUMEL", None)
    try:
        c.run(api)
        outs = c.check(api)
        if config == "many_small":
            N = c.N
            assert outs[3].anomalous[1] and outs[3].w[1] == 0.0 and not outs[3].rollback
            assert outs[5].rollback and all(outs[5].anomalous[:N])
            assert not any(o.rollback for i, o in enumerate(outs) if i != 5)
        # a second round through the same groups (tickets re-armed, mailbox sequence advanced)
        _next_round_inputs(c, 7)
        c.run(api)
        c.check(api)
        assert c.sim.members[0].stats(0).round == 2
    finally:
        c.close()


@pytest.mark.parametrize("mesh", ["1x2", "2x2"])
def test_sim_mesh_full_size_7b_unit_bench_launch_config(mesh):
    # BASELINE's 7B workload at full size on the N > 1 path, in the launch configuration
    # bench.py times (defaults: TMA RS on 148 persistent CTAs -- every CTA's ring wraps ~80
    # times at 1x2 --, LDG AG full grid), every element against the whole-mesh oracle
    c = MeshCase(mesh, "bf16", "llama7b_layer0")
    try:
        c.run("reg")
        outs = c.check("reg")
        assert outs[0].beta < 1.0 and not outs[0].rollback   # G ~ 28.5 > phi = 10: the clip is active
    finally:
        c.close()


def _next_round_inputs(c, salt):
    """Fresh locals from the updated anchors; the oracle continues from the GPU's EMA state
    (bitwise identical on every member) and the current anchors / momenta."""
    L = len(c.units)
    ema_gpu = c.sim.members[0].get_state()
    c.ema0 = [[oracle.Ema(float(ema_gpu[i, n]["mu"]), float(ema_gpu[i, n]["sigma"]), int(ema_gpu[i, n]["count"]))
               for n in range(c.N)] for i in range(L)]
    for k in range(c.K):
        m, n = k % c.M, k // c.M
        for i, u in enumerate(c.units):
            c.loc[k][i].copy_(synth.shard_local(u, i, c.M, m, n, c.anc[k][i], c.dtype, DEV, c.recipe, 1.0, salt))
    c.o_in = []
    for i in range(L):
        locs = np.stack([np.stack([parity.to_oracle_local(c.loc[n * c.M + m][i]) for n in range(c.N)])
                         for m in range(c.M)])
        c.o_in.append((locs, np.stack([c.anc[m][i].cpu().numpy() for m in range(c.M)]),
                       np.stack([c.mom[m][i].cpu().numpy() for m in range(c.M)])))
