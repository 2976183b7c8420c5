"""Pins of the oracle to things other than itself (CPU only).

Each test states what fixes the expected value: a value printed in SPEC.md /
worked by hand (tests/golden/*.json, cited), a closed form, an invariant of
PAPER.md Alg. 2 / Eq. 1-5, or a special case that reduces to a library routine
(numpy, scipy, torch.optim.SGD).
"""
import math

import numpy as np
import pytest
import torch

import oracle
from oracle import NO_AE, NO_GC, NO_WA, Config, Ema


def _f(x):
    return math.inf if x == "inf" else float(x)


# ------------------------------------------------------------ SPEC values
def test_l2_norm_spec_values(golden):
    g = golden("spec_examples.json")
    for case in g["l2_norm"]:
        assert oracle.l2_norm(case["x"]) == case["expect"], case["cite"]


def test_module_norm_from_shard_norms(golden):
    # Module norm assembled from shard sums of squares: build two
    # shards with norms 3 and 4 and run the full oracle on an M=2 mesh.
    c = golden("spec_examples.json")["module_norm_from_shards"]
    anchors = np.zeros((2, 2), np.float32)
    locals_ = np.zeros((2, 1, 2), np.float32)
    locals_[0, 0] = [-3.0, 0.0]     # ||anchor - local|| = 3 on shard 0
    locals_[1, 0] = [0.0, -4.0]     # = 4 on shard 1
    _, _, _, _, out = oracle.sync_unit(Config(), locals_, anchors, np.zeros((2, 2), np.float32), [Ema()])
    assert out.G[0] == c["expect"], c["cite"]


def test_ema_update_spec_values(golden):
    for c in golden("spec_examples.json")["ema_update"]:
        e = oracle.ema_update(Ema(c["mu"], c["sigma"], 0), _f(c["G"]), c["alpha"])
        assert abs(e.mu - c["expect_mu"]) <= c["tol"] + 1e-15, c["cite"]
        assert abs(e.sigma - c["expect_sigma"]) <= max(c["tol"], 1e-15), c["cite"]


def test_ema_sigma_uses_new_mean():
    # Eq. 1 uses mu_{t+1} inside sigma_{t+1}: 0.02*0.98^2 (new mean)
    # vs 0.02*1.0^2 (old mean) -> 0.138593 vs 0.141421.
    e = oracle.ema_update(Ema(1.0, 0.0, 0), 2.0, 0.02)
    assert abs(e.sigma - math.sqrt(0.02) * 0.98) < 1e-15
    assert abs(e.sigma - math.sqrt(0.02)) > 1e-3


def test_ema_mean_closed_form():
    # Constant G from mu_0 = 0: mu_t = G (1 - (1-alpha)^t) (geometric series of Eq. 1).
    G, alpha = 3.7, 0.02
    e = Ema()
    for t in range(1, 200):
        e = oracle.ema_update(e, G, alpha)
        assert abs(e.mu - G * (1 - (1 - alpha) ** t)) < 1e-12
        assert e.count == t


def test_is_anomaly_spec_values(golden):
    for c in golden("spec_examples.json")["is_anomaly"]:
        cfg = Config(anomaly_threshold=c["delta"], ema_warmup_rounds=c["W"])
        flag, z = oracle.is_anomaly(c["G"], Ema(c["mu"], c["sigma"], c["count"]), cfg)
        assert flag == c["expect"], c["cite"]
        if "expect_z" in c:
            assert abs(z - c["expect_z"]) < 1e-12


def test_is_anomaly_strict_and_nonfinite():
    cfg = Config(anomaly_threshold=3.0, ema_warmup_rounds=10)
    # z == delta exactly is not an anomaly (strict ">"; R10)
    assert oracle.is_anomaly(1.75, Ema(1.0, 0.25, 10), cfg)[0] is False
    assert oracle.is_anomaly(1.75 + 1e-12, Ema(1.0, 0.25, 10), cfg)[0] is True
    # non-finite G is always flagged (R9), even in warm-up and with NO_AE
    for G in (math.nan, math.inf):
        assert oracle.is_anomaly(G, Ema(0, 0, 0), cfg)[0] is True
        assert oracle.is_anomaly(G, Ema(1, 1, 99), Config(flags=NO_AE))[0] is True
    # NO_AE disables the z-test for finite G
    assert oracle.is_anomaly(100.0, Ema(1.0, 0.1, 10), Config(flags=NO_AE))[0] is False


def test_penalty_weights_spec_values(golden):
    for c in golden("spec_examples.json")["penalty_weights"]:
        w, rb = oracle.penalty_weights([_f(x) for x in c["G"]])
        assert not rb
        np.testing.assert_allclose(w, c["expect"], atol=c["tol"], rtol=0, err_msg=c["cite"])


def test_penalty_weights_vs_scipy_softmax():
    from scipy.special import softmax
    rng = np.random.default_rng(0)
    for _ in range(200):
        n = rng.integers(1, 9)
        G = rng.uniform(0, 40, n)
        w, rb = oracle.penalty_weights(G)
        assert not rb
        np.testing.assert_allclose(w, softmax(-G), rtol=1e-12, atol=1e-300)
        assert abs(w.sum() - 1.0) < 1e-12 and (w >= 0).all()        # simplex
        # shifting every norm by a constant leaves Eq. 2 unchanged
        np.testing.assert_allclose(oracle.penalty_weights(G + 7.5)[0], w, rtol=1e-12)


def test_penalty_weights_large_norms_no_underflow():
    # exp(-1000) underflows in fp64; Eq. 2 is still [e^0, e^-1]/(1 + e^-1) (R11)
    w, rb = oracle.penalty_weights([1000.0, 1001.0])
    assert not rb
    np.testing.assert_allclose(w, [1 / (1 + math.exp(-1)), math.exp(-1) / (1 + math.exp(-1))], rtol=1e-14)


def test_penalty_weights_rollback_and_uniform():
    w, rb = oracle.penalty_weights([math.inf, math.inf, math.inf])
    assert rb and (w == 0).all()                                   # Alg. 2 l.448
    w, rb = oracle.penalty_weights([1.0, math.inf, 5.0, 2.0], flags=NO_WA)
    assert not rb
    np.testing.assert_array_equal(w, [1 / 3, 0, 1 / 3, 1 / 3])


def test_clip_spec_values(golden):
    for c in golden("spec_examples.json")["clip_pseudo"]:
        b = oracle.clip_beta(c["G_bar"], c["phi"], c["eps"])
        assert abs(b - c["expect_beta"]) <= c["tol"], c["cite"]


def test_clip_bound_and_continuity():
    rng = np.random.default_rng(1)
    for _ in range(1000):
        gbar = rng.uniform(0, 100)
        b = oracle.clip_beta(gbar, 10.0, 1e-6)
        assert 0 < b <= 1.0
        assert b * gbar <= 10.0 * (1 + 1e-15)                      # ||Delta_hat|| <= phi
    assert oracle.clip_beta(50.0, flags=NO_GC) == 1.0
    phi, eps = 10.0, 1e-6
    lo, hi = oracle.clip_beta(phi + eps - 1e-9, phi, eps), oracle.clip_beta(phi + eps + 1e-9, phi, eps)
    assert abs(lo - hi) < 1e-9


def test_outer_nesterov_two_steps(golden):
    c = golden("spec_examples.json")["outer_nesterov_two_steps"]
    a, m = np.array([c["a0"]]), np.array([c["m0"]])
    for i, g in enumerate(c["g"]):
        a, m = oracle.outer_nesterov(a, m, [g], nu=c["nu"], mu=c["mu"])
        assert abs(abs(a[0]) - c["expect_abs_anchor"][i]) < c["tol"], c["cite"]
        assert abs(m[0] - c["expect_m"][i]) < c["tol"]
        assert a[0] < 0  # descent along Delta = anchor - local (R1)


def test_outer_nesterov_vs_torch_sgd():
    # R2: torch.optim.SGD(nesterov=True, dampening=0) with grad = Delta_hat.
    rng = np.random.default_rng(2)
    a0 = rng.normal(size=257)
    p = torch.tensor(a0, dtype=torch.float64, requires_grad=True)
    opt = torch.optim.SGD([p], lr=0.8, momentum=0.85, nesterov=True)
    a, m = a0.copy(), np.zeros_like(a0)
    for _ in range(5):
        g = rng.normal(size=257)
        p.grad = torch.tensor(g, dtype=torch.float64)
        opt.step()
        a, m = oracle.outer_nesterov(a, m, g, nu=0.8, mu=0.85)
        np.testing.assert_allclose(a, p.detach().numpy(), rtol=0, atol=1e-14)  # torch fuses (FMA): few ulp of the O(1-10) terms


def test_bf16_rounding_vs_torch():
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.normal(0, 0.02, 3000), rng.normal(1, 0.02, 1000),
                        rng.uniform(-1e-30, 1e-30, 100)]).astype(np.float32)
    # exact ties: 1 + 2^-8 -> 1 (even), 1 + 3*2^-8 -> 1 + 2^-6 (even)
    ties = np.array([1 + 2 ** -8, 1 + 3 * 2 ** -8, -(1 + 2 ** -8), 3.0e38, np.inf, -np.inf, 0.0, -0.0],
                    dtype=np.float32)
    x = np.concatenate([x, ties])
    ours = oracle.f32_to_bf16_bits(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(ours, ref)
    assert np.isnan(oracle.bf16_bits_to_f64(oracle.f32_to_bf16_bits(np.array([np.nan], np.float32))))[0]


def test_bf16_widening_vs_torch_all_patterns():
    # oracle_bf16_to_f64 (the oracle's only way to read a bf16 local) against torch's
    # bf16 -> fp64 conversion over every one of the 65,536 bit patterns (NaNs: both NaN)
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ours = oracle.bf16_bits_to_f64(bits)
    ref = torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).to(torch.float64).numpy()
    nan = np.isnan(ref)
    assert (np.isnan(ours) == nan).all()
    np.testing.assert_array_equal(ours[~nan], ref[~nan])
    # signed zeros and infinities keep their sign
    np.testing.assert_array_equal(np.signbit(ours[~nan]), np.signbit(ref[~nan]))


def test_bf16_sync_unit_reads_locals_like_torch():
    # a whole Sync() with bf16 locals against one computed from torch-widened locals in plain
    # numpy: NO_AE|NO_WA|NO_GC, nu = 1, mu = 0 -> anchor' = mean_n local_n (R1), so every bit
    # of the widening shows up in the result
    rng = np.random.default_rng(41)
    M, N, numel = 2, 3, 4099
    anchors = rng.normal(0, 0.02, (M, numel)).astype(np.float32)
    loc32 = (anchors[:, None, :] - rng.normal(0, 2e-3, (M, N, numel))).astype(np.float32)
    loc = torch.from_numpy(loc32).to(torch.bfloat16)
    bits = loc.view(torch.int16).numpy().view(np.uint16)
    cfg = oracle.Config(outer_lr=1.0, outer_momentum=0.0, flags=oracle.NO_AE | oracle.NO_WA | oracle.NO_GC)
    _, anc, _, _, _ = oracle.sync_unit(cfg, bits, anchors, np.zeros_like(anchors), [oracle.Ema()] * N)
    ref = loc.to(torch.float64).numpy().mean(axis=1)
    np.testing.assert_allclose(anc, ref.astype(np.float32), rtol=0, atol=2e-9)


# ----------------------------------------------------- App. C worked example
def test_appc_worked_example_primitives(golden):
    c = golden("appc_worked_example.json")
    a = np.array(c["anchor"])
    d = [a - np.array(l) for l in c["locals"]]
    G = [oracle.l2_norm(x) for x in d]
    np.testing.assert_allclose(G, c["expect"]["G"], atol=1e-15)
    w, rb = oracle.penalty_weights(G)
    np.testing.assert_allclose(w, c["expect"]["w"], atol=c["tol"])
    dbar = w[0] * d[0] + w[1] * d[1]
    np.testing.assert_allclose(dbar, c["expect"]["delta_bar"], atol=c["tol"])
    gbar = oracle.l2_norm(dbar)
    beta = oracle.clip_beta(gbar, c["phi"], c["eps"])
    assert abs(gbar - c["expect"]["G_bar"]) < c["tol"] and abs(beta - c["expect"]["beta"]) < c["tol"]
    a1, m1 = oracle.outer_nesterov(a, np.zeros(2), beta * dbar, nu=c["nu"], mu=c["mu"])
    np.testing.assert_allclose(m1, c["expect"]["m1"], atol=c["tol"])
    np.testing.assert_allclose(a1, c["expect"]["a1"], atol=c["tol"])


def test_appc_worked_example_whole_sync(golden):
    c = golden("appc_worked_example.json")
    cfg = Config(outer_lr=c["nu"], outer_momentum=c["mu"], clip_threshold=c["phi"], clip_eps=c["eps"])
    anchors = np.array([c["anchor"]], np.float32)
    locals_ = np.array([c["locals"]], np.float32)              # [M=1, N=2, 2]
    loc, anc, mom, ema, out = oracle.sync_unit(cfg, locals_, anchors, np.zeros((1, 2), np.float32),
                                               [Ema(), Ema()])
    # fp32-stored inputs (1.3 is not exact in fp32) -> ~1e-7 relative differences
    np.testing.assert_allclose(out.G, c["expect"]["G"], rtol=3e-7)
    np.testing.assert_allclose(out.w, c["expect"]["w"], rtol=3e-7)
    assert abs(out.beta - c["expect"]["beta"]) < 3e-7 and abs(out.G_bar - c["expect"]["G_bar"]) < 3e-7
    # absolute: the fp32 input error (~5e-8 on 1.3) is not scaled down by the cancellation in Delta_bar[0]
    np.testing.assert_allclose(anc[0], c["expect"]["a1"], rtol=0, atol=1e-7)
    np.testing.assert_allclose(mom[0], c["expect"]["m1"], rtol=0, atol=1e-7)
    np.testing.assert_array_equal(loc[0, 0], anc[0])
    np.testing.assert_array_equal(loc[0, 1], anc[0])
    assert all(e.count == 1 for e in ema) and not out.rollback


def test_allreduce_mean_spec_values(golden):
    for c in golden("spec_examples.json")["all_reduce_mean"]:
        got = oracle.allreduce_mean(np.array(c["grads"], np.float32))
        np.testing.assert_array_equal(got, np.array(c["expect"], np.float32), err_msg=c["cite"])


def test_allreduce_mean_vs_numpy_and_identical_inputs():
    rng = np.random.default_rng(31)
    g = rng.normal(0, 1e-3, (5, 1001)).astype(np.float32)
    np.testing.assert_allclose(oracle.allreduce_mean(g), g.astype(np.float64).mean(0), rtol=6e-8, atol=1e-12)
    same = np.repeat(g[:1], 4, axis=0)                     # identical inputs -> that input
    np.testing.assert_array_equal(oracle.allreduce_mean(same), g[0])
    gb = oracle.f32_to_bf16_bits(g).reshape(g.shape)
    gw = torch.from_numpy(gb.view(np.int16).copy()).view(torch.bfloat16).to(torch.float64).numpy()  # torch widening
    ref = torch.from_numpy(gw.mean(0).astype(np.float32)).to(
        torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(oracle.allreduce_mean(gb), ref)
