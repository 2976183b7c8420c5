"""Helpers for CUDA-vs-oracle parity (tolerances of BASELINE.json north_star, R17).

* decisions (anomaly flags, rollback, EMA counts): bit-exact
* fp32 anchor / momentum (and fp32 local): max-abs <= 1e-5 x max|ref| per tensor
* bf16 local: |gpu - ref| <= 1 bf16 ulp of ref, or <= 1e-5 x max|ref| (R17: near zero a
  bf16 ulp is below the fp32 arithmetic error)
* scalars (G, w, G_bar, beta, EMA mu/sigma): relative 1e-5 (fp32 streaming sums vs fp64)
"""
from __future__ import annotations

import numpy as np
import torch

REL = 1e-5


def to_oracle_local(t: torch.Tensor) -> np.ndarray:
    """A local shard as the oracle takes it: fp32 values or bf16 bit patterns."""
    t = t.detach().cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16).copy()
    return t.numpy().astype(np.float32, copy=True)


def local_as_f32(x: np.ndarray) -> np.ndarray:
    if x.dtype == np.uint16:
        return (x.astype(np.uint32) << 16).view(np.float32)
    return x


def bf16_ulp(ref_f32: np.ndarray) -> np.ndarray:
    e = (ref_f32.view(np.uint32) >> 23) & 0xFF
    e = np.maximum(e.astype(np.int64), 1)
    return np.ldexp(1.0, (e - 127 - 7).astype(np.int32))


def assert_f32_close(gpu: np.ndarray, ref: np.ndarray, what: str) -> None:
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    assert gpu.shape == ref.shape, what
    if ref.size == 0:
        return
    scale = float(np.max(np.abs(ref)))
    err = float(np.max(np.abs(gpu - ref)))
    assert np.isfinite(gpu).all() == np.isfinite(ref).all(), f"{what}: finiteness differs"
    assert err <= REL * max(scale, 1e-30), f"{what}: max-abs {err:.3e} > 1e-5 x {scale:.3e}"


def assert_local_close(gpu: np.ndarray, ref: np.ndarray, what: str) -> None:
    if ref.dtype != np.uint16:
        return assert_f32_close(gpu, ref, what)
    g = local_as_f32(gpu).astype(np.float64)
    r32 = local_as_f32(ref)
    r = r32.astype(np.float64)
    if r.size == 0:
        return
    scale = float(np.max(np.abs(r)))
    diff = np.abs(g - r)
    ok = (diff <= bf16_ulp(r32)) | (diff <= REL * scale)
    assert ok.all(), f"{what}: {int((~ok).sum())} bf16 elements beyond 1 ulp (max diff {diff.max():.3e})"


def assert_scalar_close(gpu, ref, what, rel=REL) -> None:
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    fin = np.isfinite(ref)
    assert (np.isfinite(gpu) == fin).all(), f"{what}: finiteness {gpu} vs {ref}"
    assert (gpu[~fin] == ref[~fin]).all() or np.isnan(ref[~fin]).all(), f"{what}: {gpu} vs {ref}"
    np.testing.assert_allclose(gpu[fin], ref[fin], rtol=rel, atol=1e-12, err_msg=what)


def assert_outcome(stats, out, ema_ref, what: str) -> None:
    """GPU edit_layer_stats_t vs oracle Outcome + EMA."""
    assert list(stats.anomalous) == list(out.anomalous), f"{what}: anomaly decisions differ"
    assert stats.rollback == out.rollback, f"{what}: rollback decision differs"
    assert_scalar_close(stats.G, out.G, f"{what} G")
    assert_scalar_close(stats.w, out.w, f"{what} w")
    z_ref = np.asarray(out.z)
    assert (np.isnan(stats.z) == np.isnan(z_ref)).all(), f"{what}: z applied differently"
    fin = ~np.isnan(z_ref)
    np.testing.assert_allclose(stats.z[fin], z_ref[fin], rtol=1e-4, atol=1e-4, err_msg=f"{what} z")
    if not out.rollback:
        assert_scalar_close([stats.G_bar], [out.G_bar], f"{what} G_bar")
        assert_scalar_close([stats.beta], [out.beta], f"{what} beta")
    assert list(stats.ema_count) == [e.count for e in ema_ref], f"{what}: EMA counts differ"
    assert_scalar_close(stats.ema_mu, [e.mu for e in ema_ref], f"{what} ema mu")
    assert_scalar_close(stats.ema_sigma, [e.sigma for e in ema_ref], f"{what} ema sigma")
