"""Single-GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, on
seeded synthetic inputs (synth/), mesh 1 x 1 (N = 1: the two-pass path).

Multi-rank parity lives in tests/test_gpu_multirank.py."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from tests import parity

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes too; every test here is -m gpu
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2412_07210_b200 import EditSync  # noqa: E402
from paper_2412_07210_b200.build import build  # noqa: E402

build()
DEV = torch.device("cuda", 0)
DTYPES = {"bf16": torch.bfloat16, "f32": torch.float32}


def _cfg_kwargs(cfg: oracle.Config):
    return dict(outer_lr=cfg.outer_lr, outer_momentum=cfg.outer_momentum, clip_threshold=cfg.clip_threshold,
                clip_eps=cfg.clip_eps, anomaly_threshold=cfg.anomaly_threshold, ema_alpha=cfg.ema_alpha,
                ema_warmup_rounds=cfg.ema_warmup_rounds, flags=cfg.flags)


class Case:
    """One rank (1 x 1 mesh) holding L units, with the oracle's mirror of its state."""

    def __init__(self, units, dtype, cfg=oracle.Config(), recipe=synth.Recipe(), plant=None):
        self.units, self.dtype, self.cfg, self.recipe = units, dtype, cfg, recipe
        self.sync = EditSync([u.numel for u in units], param_dtype=dtype, device=DEV, **_cfg_kwargs(cfg))
        self.anchor = [synth.shard_anchor(u, i, 1, 0, DEV, recipe) for i, u in enumerate(units)]
        self.mom = [synth.shard_momentum(u, i, 1, 0, DEV, recipe) for i, u in enumerate(units)]
        plant = plant or {}
        self.local = [synth.shard_local(u, i, 1, 0, 0, self.anchor[i], dtype, DEV, recipe, plant.get(i, 1.0))
                      for i, u in enumerate(units)]
        # oracle mirror (CPU, fp32 storage as the GPU)
        self.o_anchor = [a.cpu().numpy().copy() for a in self.anchor]
        self.o_mom = [m.cpu().numpy().copy() for m in self.mom]
        self.o_local = [parity.to_oracle_local(l) for l in self.local]
        self.o_ema = [[oracle.Ema()] for _ in units]

    def seed_ema(self, mu, sigma, count):
        self.sync.set_ema(np.asarray(mu)[:, None], np.asarray(sigma)[:, None], count)
        self.o_ema = [[oracle.Ema(float(mu[i]), float(sigma[i]), int(count))] for i in range(len(self.units))]

    def new_round(self, salt, plant=None):
        """Next round from the ORACLE's state (oracle -> GPU only): both sides get identical
        anchor/momentum and the same fresh locals cast(anchor - D).  (Drawing each side's
        locals from its own anchor would let a 1-ulp fp32 anchor difference flip the bf16
        rounding of the input and test the input, not the sync.)  The GPU keeps its own EMA."""
        plant = plant or {}
        for i, u in enumerate(self.units):
            p = plant.get(i, 1.0)
            self.anchor[i].copy_(torch.from_numpy(self.o_anchor[i]))
            self.mom[i].copy_(torch.from_numpy(self.o_mom[i]))
            self.local[i] = synth.shard_local(u, i, 1, 0, 0, self.anchor[i], self.dtype, DEV, self.recipe, p, salt)
            self.o_local[i] = parity.to_oracle_local(self.local[i])

    def run_and_check(self, what=""):
        for i in range(len(self.units)):
            self.sync.layer_sync(i, self.local[i], self.anchor[i], self.mom[i])
        torch.cuda.synchronize()
        for i in range(len(self.units)):
            loc, anc, mom, ema, out = oracle.sync_unit(self.cfg, self.o_local[i][None, None], self.o_anchor[i][None],
                                                       self.o_mom[i][None], self.o_ema[i])
            self.o_anchor[i], self.o_mom[i], self.o_local[i], self.o_ema[i] = anc[0], mom[0], loc[0, 0], ema
            tag = f"{what} unit {i} ({self.units[i].numel})"
            st = self.sync.stats(i)
            parity.assert_outcome(st, out, ema, tag)
            parity.assert_f32_close(self.anchor[i].cpu().numpy(), anc[0], tag + " anchor")
            parity.assert_f32_close(self.mom[i].cpu().numpy(), mom[0], tag + " momentum")
            parity.assert_local_close(parity.to_oracle_local(self.local[i]), loc[0, 0], tag + " local")
            # invariant: local == rne(anchor) bitwise on the GPU side (R16)
            assert torch.equal(self.local[i], self.anchor[i].to(self.dtype)), tag
        return out


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("numel", [1, 7, 8, 1000, 3 * 65536 + 5, 3_000_017])
def test_parity_single_unit_two_rounds(dtype, numel):
    units = [synth.Unit("u", numel, ())]
    c = Case(units, DTYPES[dtype], cfg=oracle.Config(clip_threshold=0.05))
    c.run_and_check("round1")
    c.new_round(1)
    c.run_and_check("round2")
    assert c.sync.stats(0).round == 2


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_parity_multi_unit_with_norm_segments_and_empty_unit(dtype):
    units = [synth.Unit("a", 70_001, ((69_000, 1001),)), synth.Unit("empty", 0, ()),
             synth.Unit("b", 1_048_576, ((0, 512),)), synth.Unit("c", 13, ())]
    c = Case(units, DTYPES[dtype])
    c.run_and_check()


@pytest.mark.parametrize("flags", [oracle.NO_AE, oracle.NO_WA, oracle.NO_GC,
                                   oracle.NO_AE | oracle.NO_WA | oracle.NO_GC])
def test_parity_ablation_flags(flags):
    units = [synth.Unit("u", 200_003, ())]
    c = Case(units, torch.bfloat16, cfg=oracle.Config(flags=flags, clip_threshold=0.1))
    out = c.run_and_check(f"flags={flags}")
    if flags & oracle.NO_GC:
        assert out.beta == 1.0


def test_decisions_bit_exact_seeded_ema():
    # z drawn in U[-2, 2.95] u U[3.05, 10] through the seeded (mu, sigma): N = 1, so a
    # flagged unit takes the rollback branch, an unflagged one the full update.
    rng = np.random.default_rng(42)
    units = [synth.Unit(f"u{i}", int(n), ()) for i, n in enumerate(rng.integers(1000, 300_000, 16))]
    c = Case(units, torch.bfloat16)
    G = np.array([oracle.l2_norm(c.o_anchor[i].astype(np.float64) - parity.local_as_f32(c.o_local[i]))
                  for i in range(len(units))])
    z = np.where(rng.random(len(units)) < 0.5, rng.uniform(-2, 2.95, len(units)), rng.uniform(3.05, 10, len(units)))
    sigma = 0.1 * G
    c.seed_ema(G - z * sigma, sigma, 10)
    c.run_and_check("seeded")
    flagged = [bool(c.sync.stats(i).anomalous[0]) for i in range(len(units))]
    assert flagged == list(z > 3.0)
    assert any(flagged) and not all(flagged)


def test_rollback_is_exact_and_nan_is_excluded():
    units = [synth.Unit("u", 100_000, ()), synth.Unit("v", 4097, ())]
    c = Case(units, torch.bfloat16)
    c.local[0][12345] = float("nan")       # non-finite params: always excluded (R9)
    c.o_local[0] = parity.to_oracle_local(c.local[0])
    anchor0, mom0 = c.anchor[0].clone(), c.mom[0].clone()
    c.run_and_check("nan")
    st = c.sync.stats(0)
    assert st.rollback and st.anomalous[0] and math.isinf(st.G[0])
    assert torch.equal(c.anchor[0], anchor0) and torch.equal(c.mom[0], mom0)
    assert torch.equal(c.local[0], anchor0.to(torch.bfloat16))
    assert not c.sync.stats(1).rollback


def test_deterministic_bitwise():
    units = [synth.Unit("u", 2_000_003, ())]
    outs = []
    for _ in range(2):
        c = Case(units, torch.bfloat16)
        c.sync.layer_sync(0, c.local[0], c.anchor[0], c.mom[0])
        torch.cuda.synchronize()
        outs.append((c.local[0].clone(), c.anchor[0].clone(), c.mom[0].clone(), c.sync.stats(0)))
    for x, y in zip(outs[0][:3], outs[1][:3]):
        assert torch.equal(x, y)
    assert (outs[0][3].G == outs[1][3].G).all() and outs[0][3].beta == outs[1][3].beta


def test_argument_errors():
    s = EditSync([16], device=DEV)
    t = torch.zeros(16, device=DEV)
    with pytest.raises(ValueError):
        s.layer_sync(0, t, t, t)                         # local must be bf16
    with pytest.raises(ValueError):
        s.layer_sync(1, t.bfloat16(), t, t.clone())      # layer out of range
    # misaligned pointer straight through the C ABI -> EDIT_ERR_INVALID_ARG
    assert s._lib.edit_layer_sync(s._h, 0, t.data_ptr() + 2, t.data_ptr(), t.data_ptr(), None) == 1


@pytest.mark.parametrize("unit_index", [0, 1, 33])
def test_full_size_7b_units_bench_launch_config(unit_index):
    # BASELINE.json's N = 1 bench workload: 7B-shaped shards, 1 x 1 mesh, bf16 locals,
    # steady-state momentum, seeded EMA (clip active: G ~ 28 > phi = 10).
    units = synth.llama_units("7B")
    u = units[unit_index]
    c = Case([u], torch.bfloat16, recipe=synth.Recipe())
    mu, sigma, cnt = synth.ema_seed(u, 0)
    c.seed_ema([mu], [sigma], cnt)
    out = c.run_and_check(f"7B {u.name}")
    assert out.beta < 1.0 and not out.rollback


def test_host_buffer_variant_matches_oracle():
    # edit_layer_sync_host: pinned host shards in, results copied back (CPU offload)
    units = [synth.Unit("a", 300_001, ()), synth.Unit("b", 65_536, ()), synth.Unit("c", 1_000_003, ())]
    c = Case(units, torch.bfloat16)
    h_loc = [l.cpu().pin_memory() for l in c.local]
    h_anc = [a.cpu().pin_memory() for a in c.anchor]
    h_mom = [m.cpu().pin_memory() for m in c.mom]
    for i in range(len(units)):
        c.sync.layer_sync_host(i, h_loc[i], h_anc[i], h_mom[i])
    c.sync.host_wait()
    torch.cuda.synchronize()
    for i in range(len(units)):
        loc, anc, mom, ema, out = oracle.sync_unit(c.cfg, c.o_local[i][None, None], c.o_anchor[i][None],
                                                   c.o_mom[i][None], c.o_ema[i])
        parity.assert_outcome(c.sync.stats(i), out, ema, f"host unit {i}")
        parity.assert_f32_close(h_anc[i].numpy(), anc[0], "host anchor")
        parity.assert_f32_close(h_mom[i].numpy(), mom[0], "host momentum")
        parity.assert_local_close(parity.to_oracle_local(h_loc[i]), loc[0, 0], "host local")


@pytest.mark.parametrize("depth", [1, 2, 5])
def test_prefetch_scheduler_round_matches_oracle_and_orders_forward(depth):
    # a8: syncs on the library side stream, the "forward" of unit u (on the caller's
    # stream) must see unit u's SYNCED params; results identical to direct layer_sync.
    units = [synth.Unit(f"u{i}", n, ()) for i, n in enumerate([3_000_017, 65_536, 1_000_000, 7, 2_500_000])]
    c = Case(units, torch.bfloat16)
    stream = torch.cuda.current_stream(DEV)
    seen = []
    c.sync.begin_round(c.local, c.anchor, c.mom, depth, stream)
    for i in range(len(units)):
        c.sync.acquire(i, stream)
        seen.append(c.local[i].float().sum())          # the forward reads unit i
        torch.cuda._sleep(200_000)                      # ~0.1 ms of "compute" per unit
    c.sync.end_round(stream)
    torch.cuda.synchronize()
    for i in range(len(units)):
        assert torch.equal(seen[i], c.local[i].float().sum()), f"forward of unit {i} did not see the synced params"
    # outputs vs oracle
    for i in range(len(units)):
        loc, anc, mom, ema, out = oracle.sync_unit(c.cfg, c.o_local[i][None, None], c.o_anchor[i][None],
                                                   c.o_mom[i][None], c.o_ema[i])
        parity.assert_outcome(c.sync.stats(i), out, ema, f"sched unit {i}")
        parity.assert_f32_close(c.anchor[i].cpu().numpy(), anc[0], "sched anchor")
        parity.assert_f32_close(c.mom[i].cpu().numpy(), mom[0], "sched momentum")
        parity.assert_local_close(parity.to_oracle_local(c.local[i]), loc[0, 0], "sched local")


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("sms,full_units", [(1, 0), (8, 1), (148, 2)])
def test_prefetch_scheduler_partition_mode_matches_oracle(dtype, sms, full_units):
    # edit_sched_set_partition: units >= full_units sync through the persistent TMA K1/K4 on
    # <= sms CTAs; same results as the oracle (R17), forward ordering kept, rollback exact
    units = [synth.Unit(f"u{i}", n, ()) for i, n in enumerate([3_000_017, 7, 4096 * 37 + 3, 1_000_000, 65_536])]
    c = Case(units, DTYPES[dtype], plant={3: 4.0})
    mu = np.array([synth.ema_seed(u, 0, c.recipe)[0] for u in units])
    c.seed_ema(mu, 0.1 * mu, c.recipe.ema_warmup_rounds)   # unit 3 planted x4: flagged -> rollback
    c.sync.set_partition(sms, full_units)
    stream = torch.cuda.current_stream(DEV)
    seen = []
    c.sync.begin_round(c.local, c.anchor, c.mom, 1, stream)
    for i in range(len(units)):
        c.sync.acquire(i, stream)
        seen.append(c.local[i].float().sum())
        torch.cuda._sleep(100_000)
    c.sync.end_round(stream)
    torch.cuda.synchronize()
    for i in range(len(units)):
        assert torch.equal(seen[i], c.local[i].float().sum()), f"forward of unit {i} did not see the synced params"
        loc, anc, mom, ema, out = oracle.sync_unit(c.cfg, c.o_local[i][None, None], c.o_anchor[i][None],
                                                   c.o_mom[i][None], c.o_ema[i])
        tag = f"partition sms={sms} unit {i}"
        parity.assert_outcome(c.sync.stats(i), out, ema, tag)
        parity.assert_f32_close(c.anchor[i].cpu().numpy(), anc[0], tag + " anchor")
        parity.assert_f32_close(c.mom[i].cpu().numpy(), mom[0], tag + " momentum")
        parity.assert_local_close(parity.to_oracle_local(c.local[i]), loc[0, 0], tag + " local")
        assert torch.equal(c.local[i], c.anchor[i].to(DTYPES[dtype])), tag
        if i == 3:
            assert out.rollback and np.array_equal(c.anchor[i].cpu().numpy(), c.o_anchor[i])
    c.sync.set_partition(0, 2)                               # full grids
    c.sync.set_partition(-1, 2)                              # back to the default (auto)
    with pytest.raises(Exception):
        c.sync.set_partition(-2, 0)


def test_prefetch_scheduler_argument_errors():
    from paper_2412_07210_b200 import EditSyncError
    units = [synth.Unit("a", 1000, ()), synth.Unit("b", 2000, ())]
    c = Case(units, torch.bfloat16)
    with pytest.raises(EditSyncError):
        c.sync.acquire(0)                                # no active round
    c.sync.begin_round(c.local, c.anchor, c.mom, 1)
    with pytest.raises(EditSyncError):
        c.sync.acquire(1)                                # out of order
    c.sync.acquire(0)
    c.sync.end_round()
    torch.cuda.synchronize()
    assert c.sync.stats(1).round == 1


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_round_api_matches_oracle_and_sequential_bitwise(dtype):
    # edit_sync_round (units over 2 lanes) == oracle, and == per-unit calls bit for bit
    units = [synth.Unit(f"u{i}", n, ()) for i, n in enumerate([1_000_003, 65_536, 7, 2_000_000, 300_001])]
    c = Case(units, DTYPES[dtype])
    seq = Case(units, DTYPES[dtype])
    c.sync.sync_round(c.local, c.anchor, c.mom)
    for i in range(len(units)):
        seq.sync.layer_sync(i, seq.local[i], seq.anchor[i], seq.mom[i])
    torch.cuda.synchronize()
    for i in range(len(units)):
        assert torch.equal(c.local[i], seq.local[i]) and torch.equal(c.anchor[i], seq.anchor[i])
        assert torch.equal(c.mom[i], seq.mom[i])
        loc, anc, mom, ema, out = oracle.sync_unit(c.cfg, c.o_local[i][None, None], c.o_anchor[i][None],
                                                   c.o_mom[i][None], c.o_ema[i])
        parity.assert_outcome(c.sync.stats(i), out, ema, f"round unit {i}")
        parity.assert_f32_close(c.anchor[i].cpu().numpy(), anc[0], "round anchor")
        parity.assert_f32_close(c.mom[i].cpu().numpy(), mom[0], "round momentum")
        parity.assert_local_close(parity.to_oracle_local(c.local[i]), loc[0, 0], "round local")


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_round_api_graph_replay_matches_oracle(dtype, monkeypatch):
    # EDIT_GRAPH=1: the round is captured once per buffer set and replayed; three rounds on the
    # same buffers (two replays) plus one on new buffers (a second capture) == oracle, and the
    # first round == the non-graph path bit for bit
    units = [synth.Unit(f"u{i}", n, ()) for i, n in enumerate([1_000_003, 65_536, 7, 2_000_000])]
    monkeypatch.setenv("EDIT_GRAPH", "1")
    c = Case(units, DTYPES[dtype])
    monkeypatch.delenv("EDIT_GRAPH")
    ref = Case(units, DTYPES[dtype])
    ref.sync.sync_round(ref.local, ref.anchor, ref.mom)
    for r in range(4):
        if r > 0:
            for i, u in enumerate(units):   # next round from the oracle's state, in place
                c.anchor[i].copy_(torch.from_numpy(c.o_anchor[i]))
                c.mom[i].copy_(torch.from_numpy(c.o_mom[i]))
                c.local[i].copy_(synth.shard_local(u, i, 1, 0, 0, c.anchor[i], c.dtype, DEV, c.recipe, 1.0, r))
                c.o_local[i] = parity.to_oracle_local(c.local[i])
        if r == 3:                          # new buffers -> a second captured graph
            c.local = [x.clone() for x in c.local]
        c.sync.sync_round(c.local, c.anchor, c.mom)
        torch.cuda.synchronize()
        for i in range(len(units)):
            if r == 0:
                assert torch.equal(c.local[i], ref.local[i]) and torch.equal(c.anchor[i], ref.anchor[i])
                assert torch.equal(c.mom[i], ref.mom[i])
            loc, anc, mom, ema, out = oracle.sync_unit(c.cfg, c.o_local[i][None, None], c.o_anchor[i][None],
                                                       c.o_mom[i][None], c.o_ema[i])
            c.o_anchor[i], c.o_mom[i], c.o_local[i], c.o_ema[i] = anc[0], mom[0], loc[0, 0], ema
            tag = f"graph round {r} unit {i}"
            parity.assert_outcome(c.sync.stats(i), out, ema, tag)
            parity.assert_f32_close(c.anchor[i].cpu().numpy(), anc[0], tag + " anchor")
            parity.assert_f32_close(c.mom[i].cpu().numpy(), mom[0], tag + " momentum")
            parity.assert_local_close(parity.to_oracle_local(c.local[i]), loc[0, 0], tag + " local")
            assert c.sync.stats(i).round == r + 1


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("numel", [1, 9, 1000, 65_543, 2_000_001])
def test_no_writes_outside_the_shards(dtype, numel):
    # guard zones around every buffer (compute-sanitizer is closed on this pool): the sync
    # and the host-buffer path must not touch a single element outside [0, numel)
    g = 64
    dt = DTYPES[dtype]
    units = [synth.Unit("u", numel, ())]
    c = Case(units, dt)
    guarded = []
    for t in (c.local[0], c.anchor[0], c.mom[0]):
        big = torch.full((numel + 2 * g,), 7.25, dtype=t.dtype, device=DEV)
        big[g:g + numel].copy_(t)
        guarded.append(big)
    loc, anc, mom = (b[g:g + numel] for b in guarded)
    c.sync.layer_sync(0, loc, anc, mom)
    c.sync.sync_round([loc], [anc], [mom])
    torch.cuda.synchronize()
    for b in guarded:
        assert (b[:g] == 7.25).all() and (b[g + numel:] == 7.25).all()
    assert torch.equal(loc, anc.to(dt))


def test_ema_checkpoint_resume_roundtrip():
    # edit_sync_get_state / set_state: a resumed handle continues exactly like the original
    units = [synth.Unit("a", 100_003, ()), synth.Unit("b", 4099, ())]
    a = Case(units, torch.bfloat16)
    a.run_and_check("r1")
    state = a.sync.get_state()
    assert (state["count"] == 1).all()
    b = EditSync([u.numel for u in units], param_dtype=torch.bfloat16, device=DEV)
    b.set_state(state)
    assert np.array_equal(b.get_state(), state)
    a.new_round(1)
    locs = [l.clone() for l in a.local]
    ancs = [x.clone() for x in a.anchor]
    moms = [x.clone() for x in a.mom]
    for i in range(len(units)):
        b.layer_sync(i, locs[i], ancs[i], moms[i])
    a.run_and_check("r2")
    torch.cuda.synchronize()
    for i in range(len(units)):
        assert torch.equal(locs[i], a.local[i]) and torch.equal(ancs[i], a.anchor[i])
        sa, sb = a.sync.stats(i), b.stats(i)
        assert (sa.G == sb.G).all() and sa.beta == sb.beta and (sa.ema_mu == sb.ema_mu).all()
    sa_, sb_ = a.sync.get_state(), b.get_state()
    for f in ("mu", "sigma", "count"):
        assert np.array_equal(sa_[f], sb_[f])
