"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NONE of the method's arithmetic (no pseudo-gradient, norm,
weight, clip or outer update): it only draws the tensors a worker would hold
after tau inner steps, shaped like the paper's Llama models, plus the EMA seed.
Recipe:

* Unit partition (R4): embedding; 32 decoder layers, each flattened as
  q,k,v,o,gate,up,down,input_norm,post_attn_norm (HF registration order);
  final_norm + lm_head.  Shapes from PAPER.md Table 2, vocab 79,800,
  untied embeddings.
* A unit of P_u params is ceil-split over the M shard ranks, zero-padded at the
  tail ("sharded uniformly").
* anchor  ~ N(0, 0.02^2) on matrix segments, 1 + N(0, 0.02^2) on RMSNorm segments.
* momentum ~ N(0, (5e-4)^2) ("steady") or zeros ("zero", first round; R3).
* "inner-loop displacement" of replica n: D_n = s_n (rho c + sqrt(1-rho^2) e_n),
  c, e_n ~ N(0,1), rho = 0.5, s = 2e-3, s_n = s (1 + 0.01 n) x plant[n];
  the local the worker holds is cast_dtype(anchor - D_n) (pad tail 0).
* EMA seed of replica n: mu = s_n sqrt(P_u), sigma = 0.1 mu, count = W.
Seeds: 20241210 + 1000003 kind + 10007 u + 101 m + n  (kind 0 anchor, 1 momentum,
2 common c, 3 per-replica e_n).  kinds 0-2 use n = 0 so a sync row shares them.
"""
from __future__ import annotations

import dataclasses
import math

import torch

# PAPER.md Table 2: hidden size, FFN size; 32 layers, vocab 79,800.
LLAMA = {
    "350M": (768, 2048),
    "1B": (1536, 4096),
    "3B": (2560, 6912),
    "7B": (4096, 11008),
}
N_LAYERS = 32
VOCAB = 79800

KIND_ANCHOR, KIND_MOMENTUM, KIND_COMMON, KIND_REPLICA, KIND_ANOMALY = 0, 1, 2, 3, 4


def seed_of(kind: int, u: int, m: int, n: int) -> int:
    return 20241210 + 1000003 * kind + 10007 * u + 101 * m + n


@dataclasses.dataclass(frozen=True)
class Unit:
    name: str
    numel: int                      # P_u, unsharded
    norm_segments: tuple            # ((offset, length), ...) RMSNorm weights


def llama_units(model: str) -> list[Unit]:
    """The 34 sync units of a Llama model of PAPER.md Table 2 (R4)."""
    h, inter = LLAMA[model]
    units = [Unit("embed", VOCAB * h, ())]
    dec = 4 * h * h + 3 * h * inter
    for i in range(N_LAYERS):
        units.append(Unit(f"layer{i}", dec + 2 * h, ((dec, 2 * h),)))
    units.append(Unit("head", h + VOCAB * h, ((0, h),)))
    return units


def toy_units(n_units: int = 4, numel: int = 65536) -> list[Unit]:
    """BASELINE.json configs[0]: 4 layers x 64K fp32 params."""
    return [Unit(f"toy{i}", numel, ()) for i in range(n_units)]


def shard_numel(P_u: int, M: int) -> int:
    """Per-rank shard length: ceil-split with zero pad."""
    return -(-P_u // M)


def _randn(numel: int, seed: int, device, generator_cache: dict | None = None) -> torch.Tensor:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return torch.randn(numel, generator=g, device=device, dtype=torch.float32)


@dataclasses.dataclass
class Recipe:
    s: float = 2e-3
    rho: float = 0.5
    anchor_std: float = 0.02
    momentum_std: float = 5e-4
    momentum: str = "steady"        # or "zero"
    ema_warmup_rounds: int = 10


def shard_anchor(unit: Unit, u: int, M: int, m: int, device, recipe: Recipe = Recipe()) -> torch.Tensor:
    numel = shard_numel(unit.numel, M)
    lo = m * numel
    valid = max(0, min(numel, unit.numel - lo))
    a = _randn(numel, seed_of(KIND_ANCHOR, u, m, 0), device).mul_(recipe.anchor_std)
    for off, ln in unit.norm_segments:
        s0, s1 = max(off, lo), min(off + ln, lo + valid)
        if s1 > s0:
            a[s0 - lo:s1 - lo] += 1.0
    a[valid:] = 0.0
    return a


def shard_momentum(unit: Unit, u: int, M: int, m: int, device, recipe: Recipe = Recipe()) -> torch.Tensor:
    numel = shard_numel(unit.numel, M)
    valid = max(0, min(numel, unit.numel - m * numel))
    if recipe.momentum == "zero":
        return torch.zeros(numel, device=device, dtype=torch.float32)
    mom = _randn(numel, seed_of(KIND_MOMENTUM, u, m, 0), device).mul_(recipe.momentum_std)
    mom[valid:] = 0.0
    return mom


def replica_scale(n: int, recipe: Recipe = Recipe(), plant: float = 1.0) -> float:
    return recipe.s * (1.0 + 0.01 * n) * plant


def shard_local(unit: Unit, u: int, M: int, m: int, n: int, anchor: torch.Tensor, dtype, device,
                recipe: Recipe = Recipe(), plant: float = 1.0, round_salt: int = 0) -> torch.Tensor:
    """The local shard replica n holds after tau inner steps: cast(anchor - D_n).

    round_salt != 0 draws a fresh displacement (later rounds of a benchmark)."""
    numel = anchor.numel()
    valid = max(0, min(numel, unit.numel - m * numel))
    c = _randn(numel, seed_of(KIND_COMMON, u, m, 0) + 7919 * round_salt, device)
    e = _randn(numel, seed_of(KIND_REPLICA, u, m, n) + 7919 * round_salt, device)
    sn = replica_scale(n, recipe, plant)
    disp = c.mul_(recipe.rho).add_(e, alpha=math.sqrt(1.0 - recipe.rho ** 2)).mul_(sn)
    disp[valid:] = 0.0
    out = anchor.to(torch.float32) - disp
    return out.to(dtype)


def anomaly_plants(num_units: int, N: int, rate: float, round_salt: int = 0, factor: float = 4.0) -> dict:
    """Planted anomalies for an anomaly-rate run: replica n of unit u is
    planted (its displacement x factor, z ~ 30) with probability `rate`, one Bernoulli draw per
    (unit, replica, round) from a CPU generator seeded by (KIND_ANOMALY, u, n, round) -- the
    same decisions on every rank.  Returns {(u, n): factor}."""
    out = {}
    if rate <= 0.0:
        return out
    for u in range(num_units):
        for n in range(N):
            g = torch.Generator()
            g.manual_seed(seed_of(KIND_ANOMALY, u, 0, n) + 7919 * round_salt)
            if torch.rand((), generator=g).item() < rate:
                out[(u, n)] = factor
    return out


def ema_seed(unit: Unit, n: int, recipe: Recipe = Recipe()) -> tuple[float, float, int]:
    """EMA seed of replica n for this unit: expected module norm s_n sqrt(P_u)."""
    mu = replica_scale(n, recipe) * math.sqrt(unit.numel)
    return mu, 0.1 * mu, recipe.ema_warmup_rounds
