"""Are the oracle's pins strong enough?  Mutation testing of oracle/edit_oracle.c (CPU only).

Each mutant is the oracle with ONE plausible mistake -- a dropped term, a wrong sign, a wrong
index or bound, an off-by-one -- compiled to its own .so and loaded through EDIT_ORACLE_LIB by
a fresh pytest run of the pin suites (test_oracle_pins / _invariants / _randomized).  Every
mutant must make at least one pin fail; a surviving mutant means a part of the oracle that
nothing independent of the oracle checks."""
import os
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "edit_oracle.c")
PINS = ["tests/test_oracle_pins.py", "tests/test_oracle_invariants.py", "tests/test_oracle_randomized.py"]

# (name, exact source text, replacement) -- each names the passage / reading it breaks
MUTANTS = [
    ("bf16 widening: low mantissa bit flipped (R16)",
     "uint32_t u = ((uint32_t)h) << 16;", "uint32_t u = ((uint32_t)h) << 16; u ^= 0x10000u;"),
    ("bf16 rounding: truncation instead of RNE (R16)",
     "u += 0x7fffu + lsb;", "u += 0u * lsb;"),
    ("sum of squares: last element of each chunk dropped",
     "for (int64_t k = lo; k < hi; ++k) s += x[k] * x[k];", "for (int64_t k = lo; k + 1 < hi; ++k) s += x[k] * x[k];"),
    ("IsAnomaly: >= instead of strict > (P:90, R10)",
     "return z > cfg->anomaly_threshold;", "return z >= cfg->anomaly_threshold;"),
    ("IsAnomaly: warm-up one round too long (R8)",
     "if (s->count < cfg->ema_warmup_rounds) return 0;", "if (s->count <= cfg->ema_warmup_rounds) return 0;"),
    ("IsAnomaly: non-finite G let through during the warm-up (R9)",
     "  if (!isfinite(G)) return 1;\n  if (cfg->flags & ORACLE_NO_AE)", "  if (cfg->flags & ORACLE_NO_AE)"),
    ("Eq. 1: sigma with the OLD mu (P:94, R7)",
     "alpha * (G - mu_new) * (G - mu_new);", "alpha * (G - s->mu) * (G - s->mu);"),
    ("Eq. 1: alpha and (1 - alpha) swapped in mu",
     "double mu_new = alpha * G + (1.0 - alpha) * s->mu;", "double mu_new = (1.0 - alpha) * G + alpha * s->mu;"),
    ("Eq. 2: exp(+G) instead of exp(-G) (P:102)",
     "w[i] = isfinite(G[i]) ? exp(-(G[i] - Gmin)) / gamma : 0.0;", "w[i] = isfinite(G[i]) ? exp((G[i] - Gmin)) / gamma : 0.0;"),
    ("Eq. 2: normaliser counts one term twice",
     "if (isfinite(G[i])) gamma += exp(-(G[i] - Gmin));", "if (isfinite(G[i])) gamma += (i == 0 ? 2.0 : 1.0) * exp(-(G[i] - Gmin));"),
    ("NO_WA: 1/N instead of 1/#finite (R15)",
     "w[i] = isfinite(G[i]) ? 1.0 / (double)nfinite : 0.0;", "w[i] = isfinite(G[i]) ? 1.0 / (double)n : 0.0;"),
    ("Eq. 4: max instead of min (P:113)", "return b < 1.0 ? b : 1.0;", "return b > 1.0 ? b : 1.0;"),
    ("Eq. 4: eps dropped (P:116)", "double b = phi / (G_bar + eps);", "double b = phi / (G_bar + 0.0 * eps);"),
    ("Nesterov: old momentum in the step (R2)",
     "a[k] = a[k] - nu * (g[k] + mu * m_new);", "a[k] = a[k] - nu * (g[k] + mu * m[k]);"),
    ("Nesterov: momentum term dropped", "double m_new = mu * m[k] + g[k];", "double m_new = g[k];"),
    ("Alg. 2 l.442: Delta sign flipped in Eq. 3 (R1)",
     "s += w[n] * ((double)anchors[(size_t)m * numel + k] - LOCAL(m, n, k));",
     "s += w[n] * (LOCAL(m, n, k) - (double)anchors[(size_t)m * numel + k]);"),
    ("P:98: module norm from shard 0 only (R5)", "sumsq += oracle_sq_norm(delta, numel);",
     "if (m == 0) sumsq += oracle_sq_norm(delta, numel);"),
    ("R13: G_bar from shard 0 only", "for (int m = 0; m < M; ++m) gbar_sq += oracle_sq_norm(dbar + (size_t)m * numel, numel);",
     "for (int m = 0; m < 1; ++m) gbar_sq += oracle_sq_norm(dbar + (size_t)m * numel, numel);"),
    ("Eq. 3: flagged replicas not excluded (R9)", "if (w[n] == 0.0) continue;\n", ""),
    ("Eq. 5: beta not applied", "for (int64_t k = 0; k < numel; ++k) g[k] = beta * g[k];", ""),
    ("Alg. 2 l.446: EMA updated for flagged replicas (P:98)",
     "    oracle_ema_update(&ema[n], G[n], cfg->ema_alpha);\n    out->G[n] = G[n];",
     "    if (flagged) { double G0 = sqrt(-1.0); (void)G0; }\n    oracle_ema_update(&ema[n], flagged ? out->z[n] * ema[n].sigma + ema[n].mu : G[n], cfg->ema_alpha);\n    out->G[n] = G[n];"),
    ("Alg. 2 l.449: rollback writes anchor + momentum step (R14)",
     "float a = anchors[(size_t)m * numel + k];", "float a = anchors[(size_t)m * numel + k] - momenta[(size_t)m * numel + k];"),
    ("warm-up mean: divides by N - 1 (S:313-321)", "float m = (float)(s / (double)N);",
     "float m = (float)(s / (double)(N > 1 ? N - 1 : 1));"),
]


def _build(tmp, i, text, repl):
    src = open(SRC).read()
    assert src.count(text) == 1, f"mutant {i}: pattern not unique in edit_oracle.c: {text!r}"
    path = os.path.join(tmp, f"mut{i}.c")
    with open(path, "w") as f:
        f.write(src.replace(text, repl))
    lib = os.path.join(tmp, f"libmut{i}.so")
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-w", "-o", lib, path, "-lm"])
    return lib


def _killed(lib):
    env = dict(os.environ, EDIT_ORACLE_LIB=lib, OMP_NUM_THREADS="2")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu", *PINS], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    return r.returncode != 0, r.stdout[-600:]


def test_every_oracle_mutant_is_killed_by_a_pin():
    with tempfile.TemporaryDirectory() as tmp:
        libs = [_build(tmp, i, t, r) for i, (_, t, r) in enumerate(MUTANTS)]
        with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
            results = list(ex.map(_killed, libs))
    survivors = [MUTANTS[i][0] for i, (killed, _) in enumerate(results) if not killed]
    assert not survivors, f"{len(survivors)} oracle mutants survive every pin: {survivors}"


def test_unmutated_oracle_passes_the_pins_through_the_override():
    # control: the same harness with the real source must pass (so a kill means the mutation)
    with tempfile.TemporaryDirectory() as tmp:
        lib = _build(tmp, 99, "#define ORACLE_CHUNK 65536", "#define ORACLE_CHUNK 65536")
        killed, tail = _killed(lib)
    assert not killed, tail
