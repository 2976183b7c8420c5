"""Whole-Sync() invariants of the oracle (CPU only).

Special cases of Alg. 2 that reduce to plain averaging / a library routine,
brute force on tiny inputs, and structural invariants.
"""
import math

import numpy as np
import pytest
import torch
from scipy.special import softmax

import oracle
from oracle import NO_AE, NO_GC, NO_WA, Config, Ema


def _rand_mesh(M, N, numel, seed, bf16=False, scale=2e-3):
    rng = np.random.default_rng(seed)
    anchors = rng.normal(0, 0.02, (M, numel)).astype(np.float32)
    momenta = rng.normal(0, 5e-4, (M, numel)).astype(np.float32)
    locals_ = (anchors[:, None, :] - rng.normal(0, scale, (M, N, numel))).astype(np.float32)
    if bf16:
        locals_ = oracle.f32_to_bf16_bits(locals_).reshape(M, N, numel)
    return locals_, anchors, momenta


def _as_f64(locals_):
    # widen with torch (independent of the oracle's own oracle_bf16_to_f64, which is pinned
    # separately against torch over all 65,536 bit patterns in test_oracle_pins.py)
    if locals_.dtype == np.uint16:
        return torch.from_numpy(locals_.view(np.int16).copy()).view(torch.bfloat16).to(torch.float64).numpy()
    return locals_.astype(np.float64)


@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_plain_averaging_special_case(N):
    # NO_AE|NO_WA|NO_GC, mu = 0, nu = 1: one EDiT round = Post Local SGD
    # parameter averaging (sign reading R1): anchor' = mean_n local_n.
    locals_, anchors, momenta = _rand_mesh(2, N, 1000, seed=N)
    cfg = Config(outer_lr=1.0, outer_momentum=0.0, flags=NO_AE | NO_WA | NO_GC)
    loc, anc, mom, _, out = oracle.sync_unit(cfg, locals_, anchors, momenta, [Ema()] * N)
    mean = locals_.astype(np.float64).mean(axis=1)
    np.testing.assert_allclose(anc, mean.astype(np.float32), rtol=0, atol=2e-9)
    np.testing.assert_allclose(out.w, np.full(N, 1 / N))
    # momentum' = mu*m + Delta_bar = mean_n(anchor - local_n)
    np.testing.assert_allclose(mom, (anchors - mean).astype(np.float32), rtol=0, atol=2e-9)


def test_partial_outer_lr_interpolates():
    # NO_WA|NO_GC, mu = 0: anchor' = (1 - nu) anchor + nu mean(local)
    locals_, anchors, momenta = _rand_mesh(1, 3, 777, seed=11)
    nu = 0.7
    cfg = Config(outer_lr=nu, outer_momentum=0.0, flags=NO_WA | NO_GC)
    _, anc, _, _, _ = oracle.sync_unit(cfg, locals_, anchors, momenta, [Ema()] * 3)
    ref = (1 - nu) * anchors.astype(np.float64) + nu * locals_.astype(np.float64).mean(axis=1)
    np.testing.assert_allclose(anc, ref, rtol=1.2e-7, atol=1e-12)  # fp32 store: <= 1/2 ulp


def test_all_equal_workers():
    # identical Delta on every worker -> w = 1/N, Delta_bar = Delta,
    # Delta_hat = Delta min(phi/(||Delta|| + eps), 1)
    M, N, numel = 2, 4, 500
    rng = np.random.default_rng(5)
    anchors = rng.normal(0, 0.02, (M, numel)).astype(np.float32)
    one = (anchors - rng.normal(0, 0.3, (M, numel))).astype(np.float32)
    locals_ = np.repeat(one[:, None, :], N, axis=1)
    cfg = Config(clip_threshold=1.0)
    _, anc, mom, _, out = oracle.sync_unit(cfg, locals_, anchors, np.zeros((M, numel), np.float32), [Ema()] * N)
    np.testing.assert_allclose(out.w, 0.25, rtol=1e-15)
    delta = anchors.astype(np.float64) - one.astype(np.float64)
    G = np.linalg.norm(delta)
    np.testing.assert_allclose(out.G, G, rtol=1e-13)
    assert abs(out.G_bar - G) < 1e-12 * G
    beta = min(1.0 / (G + 1e-6), 1.0)
    assert beta < 1.0 and abs(out.beta - beta) < 1e-15
    np.testing.assert_allclose(mom, (beta * delta).astype(np.float32), rtol=0, atol=1e-8)


def test_brute_force_vs_library_composition():
    # Tiny mesh, bf16 locals, EMA in warm-up: compose Alg. 2 from library
    # routines (numpy norm, scipy softmax, torch.optim.SGD(nesterov)) and compare.
    M, N, numel = 2, 3, 37
    locals_, anchors, momenta = _rand_mesh(M, N, numel, seed=7, bf16=True, scale=0.05)
    cfg = Config(clip_threshold=0.4)
    loc, anc, mom, ema, out = oracle.sync_unit(cfg, locals_, anchors, momenta, [Ema()] * N)
    L = _as_f64(locals_)
    d = anchors[:, None, :].astype(np.float64) - L                      # [M, N, k]
    G = np.array([np.linalg.norm(d[:, n, :]) for n in range(N)])
    np.testing.assert_allclose(out.G, G, rtol=1e-14)
    w = softmax(-G)
    np.testing.assert_allclose(out.w, w, rtol=1e-13)
    dbar = np.einsum("n,mnk->mk", w, d)
    gbar = np.linalg.norm(dbar)
    beta = min(cfg.clip_threshold / (gbar + cfg.clip_eps), 1.0)
    assert abs(out.G_bar - gbar) < 1e-14 * gbar and abs(out.beta - beta) < 1e-14
    for m in range(M):
        p = torch.tensor(anchors[m].astype(np.float64), requires_grad=True)
        opt = torch.optim.SGD([p], lr=cfg.outer_lr, momentum=cfg.outer_momentum, nesterov=True)
        opt.state[p]["momentum_buffer"] = torch.tensor(momenta[m].astype(np.float64))
        p.grad = torch.tensor(beta * dbar[m])
        opt.step()
        # fp64 results agree to ~1 ulp (torch may fuse); after the fp32 store <= 1 fp32 ulp
        np.testing.assert_allclose(anc[m], p.detach().numpy(), rtol=1.2e-7, atol=1e-30)
        np.testing.assert_allclose(mom[m], opt.state[p]["momentum_buffer"].numpy(), rtol=1.2e-7, atol=1e-30)
        ref_local = torch.from_numpy(anc[m]).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
        for n in range(N):
            np.testing.assert_array_equal(loc[m, n], ref_local)
    # EMA from mu=sigma=0 after one finite G: mu = alpha G, sigma = sqrt(alpha) (1-alpha) G
    for n in range(N):
        assert abs(ema[n].mu - 0.02 * G[n]) < 1e-15
        assert abs(ema[n].sigma - math.sqrt(0.02) * 0.98 * G[n]) < 1e-15


def test_planted_anomaly_excluded():
    # Replica 1's Delta is 4x larger; with seeded EMA its z ~ 30 > delta -> G = inf,
    # w = 0, EMA untouched, Delta_bar = weighted sum over the others.
    M, N, numel = 2, 3, 4096
    rng = np.random.default_rng(9)
    anchors = rng.normal(0, 0.02, (M, numel)).astype(np.float32)
    disp = rng.normal(0, 2e-3, (M, N, numel))
    disp[:, 1, :] *= 4.0
    locals_ = (anchors[:, None, :] - disp).astype(np.float32)
    d = anchors[:, None, :].astype(np.float64) - locals_.astype(np.float64)
    G = np.array([np.linalg.norm(d[:, n]) for n in range(N)])
    mu0 = 2e-3 * math.sqrt(M * numel)
    ema0 = [Ema(mu0, 0.1 * mu0, 10) for _ in range(N)]
    loc, anc, mom, ema, out = oracle.sync_unit(Config(), locals_, anchors, np.zeros((M, numel), np.float32), ema0)
    assert list(out.anomalous) == [False, True, False]
    assert out.G[1] == math.inf and out.w[1] == 0.0
    assert ema[1] == ema0[1]                                  # Eq. 1 skipped for infinite G
    assert ema[0].count == 11 and ema[2].count == 11
    w = softmax(-G[[0, 2]])
    np.testing.assert_allclose(out.w[[0, 2]], w, rtol=1e-13)
    dbar = w[0] * d[:, 0] + w[1] * d[:, 2]
    assert abs(out.G_bar - np.linalg.norm(dbar)) < 1e-12


def test_rollback_exact():
    # all workers anomalous -> theta_{t+1,0} = theta_t bitwise, momentum and EMA unchanged
    M, N, numel = 2, 2, 300
    locals_, anchors, momenta = _rand_mesh(M, N, numel, seed=13, bf16=True)
    ema0 = [Ema(1e-6, 1e-7, 50), Ema(1e-6, 1e-7, 50)]       # any realistic G is z >> 3
    loc, anc, mom, ema, out = oracle.sync_unit(Config(), locals_, anchors, momenta, ema0)
    assert out.rollback and all(out.anomalous) and (out.w == 0).all()
    np.testing.assert_array_equal(anc, anchors)
    np.testing.assert_array_equal(mom, momenta)
    assert ema == ema0
    ref = torch.from_numpy(anchors).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    for n in range(N):
        np.testing.assert_array_equal(loc[:, n], ref)


def test_nonfinite_replica_always_excluded():
    # NaN in one replica's params: flagged even in EMA warm-up (R9); outputs finite
    M, N, numel = 1, 3, 100
    locals_, anchors, momenta = _rand_mesh(M, N, numel, seed=17)
    locals_[0, 2, 5] = np.nan
    loc, anc, mom, ema, out = oracle.sync_unit(Config(flags=NO_AE), locals_, anchors, momenta, [Ema()] * N)
    assert list(out.anomalous) == [False, False, True] and not out.rollback
    assert np.isfinite(anc).all() and np.isfinite(mom).all() and np.isfinite(loc).all()
    # same result as running the two healthy replicas alone (N=2)
    loc2, anc2, mom2, _, _ = oracle.sync_unit(Config(flags=NO_AE), locals_[:, :2], anchors, momenta, [Ema()] * 2)
    np.testing.assert_array_equal(anc, anc2)
    np.testing.assert_array_equal(mom, mom2)


def test_pad_and_shard_invariance():
    # Module norm is shard-independent (R5): the same module unsharded (M=1)
    # or ceil-split over M=3 with a zero-padded tail gives the same G,
    # G_bar, beta and the same updated params.
    P, N = 1001, 2
    rng = np.random.default_rng(21)
    full_a = rng.normal(0, 0.02, P).astype(np.float32)
    full_m = rng.normal(0, 5e-4, P).astype(np.float32)
    full_l = (full_a[None] - rng.normal(0, 0.05, (N, P))).astype(np.float32)
    cfg = Config(clip_threshold=1.0)
    l1, a1, m1, _, o1 = oracle.sync_unit(cfg, full_l[None], full_a[None], full_m[None], [Ema()] * N)
    M = 3
    numel = -(-P // M)
    pad = M * numel - P
    sh = lambda x: np.concatenate([x, np.zeros(x.shape[:-1] + (pad,), x.dtype)], -1)
    A = sh(full_a).reshape(M, numel)
    Mo = sh(full_m).reshape(M, numel)
    L = sh(full_l).reshape(N, M, numel).transpose(1, 0, 2).copy()
    l3, a3, m3, _, o3 = oracle.sync_unit(cfg, L, A, Mo, [Ema()] * N)
    np.testing.assert_allclose(o3.G, o1.G, rtol=1e-14)
    assert abs(o3.G_bar - o1.G_bar) < 1e-14 * o1.G_bar and abs(o3.beta - o1.beta) < 1e-14
    np.testing.assert_allclose(a3.reshape(-1)[:P], a1[0], rtol=0, atol=1e-9)
    np.testing.assert_allclose(m3.reshape(-1)[:P], m1[0], rtol=0, atol=1e-9)
    assert (a3.reshape(-1)[P:] == 0).all() and (m3.reshape(-1)[P:] == 0).all()
    assert (l3.transpose(1, 0, 2).reshape(N, -1)[:, P:] == 0).all()


def test_sync_row_identity_and_determinism():
    # every replica of a sync row ends with the same local, and the
    # result does not depend on the oracle's thread count
    locals_, anchors, momenta = _rand_mesh(2, 4, 200_000, seed=23, bf16=True)
    outs = []
    for t in (1, 4):
        oracle.set_threads(t)
        outs.append(oracle.sync_unit(Config(), locals_, anchors, momenta, [Ema()] * 4))
    oracle.set_threads(0)
    (la, aa, ma, _, oa), (lb, ab, mb, _, ob) = outs
    np.testing.assert_array_equal(aa, ab)
    np.testing.assert_array_equal(ma, mb)
    np.testing.assert_array_equal(la, lb)
    assert (oa.G == ob.G).all() and oa.G_bar == ob.G_bar
    for n in range(1, 4):
        np.testing.assert_array_equal(la[:, n], la[:, 0])


def test_clip_never_increases_norm():
    rng = np.random.default_rng(29)
    for phi in (0.01, 0.1, 1.0, 100.0):
        locals_, anchors, _ = _rand_mesh(1, 2, 500, seed=int(phi * 100), scale=0.01)
        cfg = Config(clip_threshold=phi, outer_lr=1.0, outer_momentum=0.0)
        _, _, mom, _, out = oracle.sync_unit(cfg, locals_, anchors, np.zeros((1, 500), np.float32), [Ema()] * 2)
        # with mu = 0, momentum' = Delta_hat
        nh = np.linalg.norm(mom.astype(np.float64))
        assert nh <= out.G_bar * (1 + 1e-6) and nh <= phi * (1 + 1e-6)


def test_empty_unit():
    loc, anc, mom, ema, out = oracle.sync_unit(Config(), np.zeros((1, 2, 0), np.float32),
                                               np.zeros((1, 0), np.float32), np.zeros((1, 0), np.float32),
                                               [Ema()] * 2)
    assert (out.G == 0).all() and out.G_bar == 0 and out.beta == 1.0 and not out.rollback
    np.testing.assert_allclose(out.w, 0.5)
