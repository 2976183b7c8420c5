"""Randomized pins of the oracle's penalty primitives (SPEC acceptance #3: 10^4 random
cases of the penalty unit suite), each against an independent formulation."""
import math

import numpy as np
from scipy.special import softmax

import oracle
from oracle import NO_WA, Config, Ema

RNG = np.random.default_rng(20241210)
CASES = 10_000


def test_weights_random_cases():
    for _ in range(CASES // 10):
        n = int(RNG.integers(1, 9))
        G = RNG.uniform(0, 60, n)
        inf = RNG.random(n) < 0.2
        G[inf] = math.inf
        w, rb = oracle.penalty_weights(G)
        finite = ~np.isinf(G)
        assert rb == (not finite.any())
        if rb:
            assert (w == 0).all()
            continue
        assert (w[~finite] == 0).all() and abs(w.sum() - 1) < 1e-12                    # simplex
        np.testing.assert_allclose(w[finite], softmax(-G[finite]), rtol=1e-12)        # Eq. 2
        wu, _ = oracle.penalty_weights(G, NO_WA)
        np.testing.assert_allclose(wu[finite], 1.0 / finite.sum(), rtol=1e-15)


def test_ema_and_anomaly_random_cases():
    cfg = Config(anomaly_threshold=3.0, ema_warmup_rounds=10)
    for _ in range(CASES // 4):
        mu, sigma, G = RNG.uniform(0.1, 50), RNG.uniform(0, 5), RNG.uniform(0, 80)
        count = int(RNG.integers(0, 20))
        e = Ema(mu, sigma, count)
        flag, z = oracle.is_anomaly(G, e, cfg)
        if count < 10 or sigma == 0:
            assert flag is False and math.isnan(z)
        else:
            assert abs(z - (G - mu) / sigma) <= 1e-12 * max(1.0, abs(z))
            assert flag == ((G - mu) / sigma > 3.0)
        a = RNG.uniform(0.001, 1.0)
        e2 = oracle.ema_update(e, G, a)
        # Eq. 1 as an incremental mean/variance update: mu' - mu = a (G - mu); and since
        # G - mu' = (1-a)(G - mu):  sigma'^2 = (1-a) (sigma^2 + a (1-a) (G - mu)^2)
        assert abs((e2.mu - mu) - a * (G - mu)) <= 1e-12 * max(1.0, abs(G))
        ref = (1 - a) * (sigma ** 2 + a * (1 - a) * (G - mu) ** 2)
        assert abs(e2.sigma ** 2 - ref) <= 1e-10 * max(1.0, ref)
        assert e2.count == count + 1


def test_clip_random_cases():
    for _ in range(CASES // 4):
        gbar, phi, eps = RNG.uniform(0, 100), RNG.uniform(0.01, 50), 10.0 ** RNG.uniform(-9, -3)
        b = oracle.clip_beta(gbar, phi, eps)
        assert 0 < b <= 1.0
        assert b * gbar <= phi * (1 + 1e-15)
        if gbar + eps <= phi:
            assert b == 1.0
        else:
            assert abs(b * (gbar + eps) - phi) <= 1e-12 * phi                            # Eq. 4
