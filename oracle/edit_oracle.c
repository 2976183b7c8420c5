/*
 * oracle/edit_oracle.c -- TEST INFRASTRUCTURE ONLY (not part of the product path).
 *
 * A plain, slow, obviously-correct fp64 CPU implementation of EDiT's layer-wise
 * model synchronisation with the pseudo-gradient penalty, i.e. Sync() of
 * Algorithm 2 (App. A.1) together with the equations of
 * Section 3.2: Eq. 1 (EMA), Eq. 2 (weights),
 * Eq. 3 (weighted sum), Eq. 4-5 (clip) and the outer
 * optimizer (Nesterov momentum, P:161 / P:496).
 *
 * Who may use this file: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs.  It shares no code, header, table or
 * constant with the CUDA path (paper_2412_07210_b200/csrc), and neither imports
 * the other.
 *
 * Everything is computed in fp64 ("the oracle is fp64").  The only
 * reductions are sums of squares (fixed 65536-element chunks whose partial sums
 * are added in index order, so the result does not depend on the thread count)
 * and the n-ordered weighted sum of Eq. 3.  Readings of places where the paper
 * is silent or inconsistent are tagged R1..R20 and listed in DESIGN.md
 * ("Readings of the paper").
 *
 * Parity pins: see tests/test_oracle_*.py.  Parts the paper itself does not pin
 * ("parity unpinned" by the paper, pinned only by the readings): the sign of the
 * pseudo-gradient (R1), the Nesterov form (R2), the EMA initialisation and
 * warm-up length (R8), the unit partition (R4).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_MAX_SYNC 8
#define ORACLE_CHUNK 65536

/* Ablation flags of Section 4.5: w/o AE, w/o WA, w/o GC. */
#define ORACLE_NO_AE 1u
#define ORACLE_NO_WA 2u
#define ORACLE_NO_GC 4u

typedef struct {
  double outer_lr;          /* nu     (0.8 FineWeb-Edu / 1.0 in-house)    */
  double outer_momentum;    /* mu     (0.85 / 0.8)                         */
  double clip_threshold;    /* phi    (10)                                 */
  double clip_eps;          /* epsilon ("a small positive constant")       */
  double anomaly_threshold; /* delta  ("typically set to 3")                */
  double ema_alpha;         /* alpha  ("commonly assigned a value of 0.02") */
  int64_t ema_warmup_rounds;/* "a warm-up period", length unstated (R8)    */
  uint32_t flags;           /* ORACLE_NO_AE | ORACLE_NO_WA | ORACLE_NO_GC          */
  uint32_t pad_;
} oracle_cfg_t;

/* EMA statistics of one (worker, module): mu_t, sigma_t + rounds seen. */
typedef struct {
  double mu;
  double sigma;
  int64_t count;
} oracle_ema_t;

/* What one Sync() of one module decided (one record per sync group row). */
typedef struct {
  double G[ORACLE_MAX_SYNC];          /* module-level ||Delta|| per worker, +inf if flagged */
  double z[ORACLE_MAX_SYNC];          /* EMA z-score, NaN when the test was not applied     */
  int32_t anomalous[ORACLE_MAX_SYNC]; /* 1 if G was set to infinity                          */
  double w[ORACLE_MAX_SYNC];          /* Eq. 2 weights                                       */
  double G_bar;                       /* ||Delta_bar|| (Eq. 4), module level                 */
  double beta;                        /* clip coefficient (Eq. 4)                            */
  int32_t rollback;                   /* Alg. 2 l.448-449 taken                              */
  int32_t pad_;
} oracle_outcome_t;

void oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int oracle_get_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ---------------------------------------------------------------------------
 * Number formats.  Inputs arrive as they are stored (fp32, or bf16 bit
 * patterns); the oracle widens them to fp64 exactly.  Outputs are rounded
 * fp64 -> fp32 by the C cast (round-to-nearest-even) and, for a bf16 local,
 * fp32 -> bf16 round-to-nearest-even (R16).
 * ------------------------------------------------------------------------- */
double oracle_bf16_to_f64(uint16_t h) {
  uint32_t u = ((uint32_t)h) << 16;
  float f;
  memcpy(&f, &u, sizeof f);
  return (double)f;
}

uint16_t oracle_f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, sizeof u);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu) != 0u) {
    return (uint16_t)((u >> 16) | 0x0040u); /* NaN stays a (quiet) NaN */
  }
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb; /* round half to even on the 16 dropped bits */
  return (uint16_t)(u >> 16);
}

/* ---------------------------------------------------------------------------
 * ||x||_2^2 with fixed 65536-element chunks added in index order.
 * SPEC S:45-53 l2_norm: sqrt(sum x_i^2), 0 for an empty vector.
 * ------------------------------------------------------------------------- */
double oracle_sq_norm(const double* x, int64_t n) {
  if (n <= 0) return 0.0;
  int64_t nchunks = (n + ORACLE_CHUNK - 1) / ORACLE_CHUNK;
  double* part = (double*)calloc((size_t)nchunks, sizeof(double));
  if (!part) return NAN;
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < nchunks; ++c) {
    int64_t lo = c * ORACLE_CHUNK, hi = lo + ORACLE_CHUNK < n ? lo + ORACLE_CHUNK : n;
    double s = 0.0;
    for (int64_t k = lo; k < hi; ++k) s += x[k] * x[k];
    part[c] = s;
  }
  double total = 0.0;
  for (int64_t c = 0; c < nchunks; ++c) total += part[c];
  free(part);
  return total;
}

/* ---------------------------------------------------------------------------
 * IsAnomaly (Alg. 2 l.444).
 *   z = (G - mu) / sigma; anomalous iff z > delta (strict, R10).
 *   No worker is flagged during the EMA warm-up period: count < W (R8).
 *   sigma == 0 leaves z undefined -> not flagged (R8).
 *   A non-finite G (NaN/Inf parameters) is always flagged, also during warm-up
 *   and under NO_AE (R9).  *z_out is NaN whenever the z-test is not applied.
 * ------------------------------------------------------------------------- */
int oracle_is_anomaly(double G, const oracle_ema_t* s, const oracle_cfg_t* cfg, double* z_out) {
  *z_out = NAN;
  if (!isfinite(G)) return 1;
  if (cfg->flags & ORACLE_NO_AE) return 0;
  if (s->count < cfg->ema_warmup_rounds) return 0;
  if (!(s->sigma > 0.0)) return 0;
  double z = (G - s->mu) / s->sigma;
  *z_out = z;
  return z > cfg->anomaly_threshold;
}

/* ---------------------------------------------------------------------------
 * EMA statistics update, Eq. 1:
 *   mu'    = alpha G + (1 - alpha) mu
 *   sigma' = sqrt((1 - alpha) sigma^2 + alpha (G - mu')^2)     (uses the NEW mu, R7)
 * "The update of Equation 1 will be skipped if G is infinite".
 * ------------------------------------------------------------------------- */
void oracle_ema_update(oracle_ema_t* s, double G, double alpha) {
  if (!isfinite(G)) return;
  double mu_new = alpha * G + (1.0 - alpha) * s->mu;
  double var_new = (1.0 - alpha) * s->sigma * s->sigma + alpha * (G - mu_new) * (G - mu_new);
  s->mu = mu_new;
  s->sigma = sqrt(var_new);
  s->count += 1;
}

/* ---------------------------------------------------------------------------
 * Weighted averaging, Eq. 2, and the gamma == 0 test of
 * Alg. 2 l.447-448:
 *   w_i = exp(-G_i) / sum_j exp(-G_j),   gamma = sum_j exp(-G_j).
 * Written with the common factor exp(G_min) cancelled (R11), which is the same
 * number mathematically but does not underflow for realistic norms (G ~ 28 for
 * a 7B layer); an infinite G contributes exp(-inf) = 0.  gamma == 0 (rollback)
 * iff no G is finite.  NO_WA: uniform 1/#finite over the finite G.
 * Returns 1 for rollback (w all zero), else 0.
 * ------------------------------------------------------------------------- */
int oracle_penalty_weights(const double* G, int32_t n, uint32_t flags, double* w) {
  int nfinite = 0;
  double Gmin = INFINITY;
  for (int i = 0; i < n; ++i) {
    w[i] = 0.0;
    if (isfinite(G[i])) {
      nfinite += 1;
      if (G[i] < Gmin) Gmin = G[i];
    }
  }
  if (nfinite == 0) return 1;
  if (flags & ORACLE_NO_WA) {
    for (int i = 0; i < n; ++i) w[i] = isfinite(G[i]) ? 1.0 / (double)nfinite : 0.0;
    return 0;
  }
  double gamma = 0.0;
  for (int i = 0; i < n; ++i)
    if (isfinite(G[i])) gamma += exp(-(G[i] - Gmin));
  for (int i = 0; i < n; ++i) w[i] = isfinite(G[i]) ? exp(-(G[i] - Gmin)) / gamma : 0.0;
  return 0;
}

/* ---------------------------------------------------------------------------
 * Clip coefficient, Eq. 4: beta = min(phi / (G_bar + eps), 1).
 * NO_GC: beta = 1.
 * ------------------------------------------------------------------------- */
double oracle_clip_beta(double G_bar, double phi, double eps, uint32_t flags) {
  if (flags & ORACLE_NO_GC) return 1.0;
  double b = phi / (G_bar + eps);
  return b < 1.0 ? b : 1.0;
}

/* ---------------------------------------------------------------------------
 * OuterOpt = Nesterov momentum, in the form of
 * torch.optim.SGD(nesterov=True, dampening=0) with "gradient" Delta_hat (R2),
 * and descent along Delta = anchor - local (R1):
 *   m' = mu m + g ;   a' = a - nu (g + mu m')
 * ------------------------------------------------------------------------- */
void oracle_outer_nesterov(double* a, double* m, const double* g, int64_t n, double nu, double mu) {
  for (int64_t k = 0; k < n; ++k) {
    double m_new = mu * m[k] + g[k];
    a[k] = a[k] - nu * (g[k] + mu * m_new);
    m[k] = m_new;
  }
}

/* ---------------------------------------------------------------------------
 * One Sync() (Alg. 2) of one module l for ONE model sync group row... for the
 * whole M x N mesh at once (M shard ranks x N sync replicas).
 *
 *   locals_in  [M][N][numel]  theta_{t,tau}^{(i,l)}: bf16 bits (local_is_bf16)
 *                             or fp32, shard m of replica n (ceil-split,
 *                             zero-padded tail, R4/R5)
 *   anchors    [M][numel] f32 theta_t^{(i,l)} (identical across a sync row),
 *                             updated in place
 *   momenta    [M][numel] f32 outer momentum (sharded like the params),
 *                             updated in place
 *   locals_out [M][N][numel]  theta_{t+1,0}^{(i,l)} in the local dtype
 *   ema        [N]            EMA of replica n for this module (R6), in/out
 *   out                       the decisions (one record: they are identical on
 *                             every rank because every norm is module-level)
 * Returns 0, or -1 on bad arguments / allocation failure.
 * ------------------------------------------------------------------------- */
int oracle_sync_unit(const oracle_cfg_t* cfg, int32_t M, int32_t N, int64_t numel,
                     int32_t local_is_bf16, const void* locals_in, float* anchors,
                     float* momenta, void* locals_out, oracle_ema_t* ema,
                     oracle_outcome_t* out) {
  if (!cfg || M < 1 || N < 1 || N > ORACLE_MAX_SYNC || numel < 0) return -1;
  const uint16_t* lb = (const uint16_t*)locals_in;
  const float* lf = (const float*)locals_in;
  memset(out, 0, sizeof *out);
  for (int n = 0; n < ORACLE_MAX_SYNC; ++n) out->z[n] = NAN;

  size_t len = (size_t)(numel > 0 ? numel : 1);
  double* delta = (double*)malloc(len * sizeof(double));
  double* dbar = (double*)malloc((size_t)M * len * sizeof(double));
  if (!delta || !dbar) { free(delta); free(dbar); return -1; }

#define LOCAL(m, n, k)                                                                  \
  (local_is_bf16 ? oracle_bf16_to_f64(lb[(((size_t)(m) * N + (n)) * numel) + (k)])      \
                 : (double)lf[(((size_t)(m) * N + (n)) * numel) + (k)])

  /* Alg. 2 l.442-443: Delta = anchor - local (sign: R1) and
   * G = ||Delta||_2 over the whole module = sqrt(sum over the M shards of the
   * shard sums of squares) ("one scalar communication in the model shard
   * groups"; R5). */
  double G[ORACLE_MAX_SYNC];
  for (int n = 0; n < N; ++n) {
    double sumsq = 0.0;
    for (int m = 0; m < M; ++m) {
#pragma omp parallel for schedule(static)
      for (int64_t k = 0; k < numel; ++k)
        delta[k] = (double)anchors[(size_t)m * numel + k] - LOCAL(m, n, k);
      sumsq += oracle_sq_norm(delta, numel);
    }
    G[n] = sqrt(sumsq);
  }

  /* Alg. 2 l.444-446: IsAnomaly -> G = inf; then Eq. 1 for every finite G. */
  for (int n = 0; n < N; ++n) {
    double z;
    int flagged = oracle_is_anomaly(G[n], &ema[n], cfg, &z);
    out->z[n] = z;
    if (flagged) {
      G[n] = INFINITY;
      out->anomalous[n] = 1;
    }
    oracle_ema_update(&ema[n], G[n], cfg->ema_alpha);
    out->G[n] = G[n];
  }

  /* Alg. 2 l.447-451: gamma, rollback test, weights (Eq. 2). */
  double w[ORACLE_MAX_SYNC];
  int rollback = oracle_penalty_weights(G, N, cfg->flags, w);
  for (int n = 0; n < N; ++n) out->w[n] = w[n];
  out->rollback = rollback;

  if (rollback) {
    /* Alg. 2 l.449: theta_{t+1,0} = theta_t; anchor and momentum unchanged (R14). */
    out->beta = 1.0;
    out->G_bar = 0.0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n)
        for (int64_t k = 0; k < numel; ++k) {
          size_t i = (((size_t)m * N + n) * numel) + k;
          float a = anchors[(size_t)m * numel + k];
          if (local_is_bf16) ((uint16_t*)locals_out)[i] = oracle_f32_to_bf16_rne(a);
          else ((float*)locals_out)[i] = a;
        }
    free(delta);
    free(dbar);
    return 0;
  }

  /* Eq. 3 / Alg. 2 l.452: Delta_bar = sum_j w_j Delta_j, summed in j order.
   * A worker with w_j == 0 is excluded (its Delta may be non-finite, R9). */
  for (int m = 0; m < M; ++m)
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < numel; ++k) {
      double s = 0.0;
      for (int n = 0; n < N; ++n) {
        if (w[n] == 0.0) continue;
        s += w[n] * ((double)anchors[(size_t)m * numel + k] - LOCAL(m, n, k));
      }
      dbar[(size_t)m * numel + k] = s;
    }

  /* Eq. 4: G_bar = ||Delta_bar|| over the whole module (R13); beta. */
  double gbar_sq = 0.0;
  for (int m = 0; m < M; ++m) gbar_sq += oracle_sq_norm(dbar + (size_t)m * numel, numel);
  double G_bar = sqrt(gbar_sq);
  double beta = oracle_clip_beta(G_bar, cfg->clip_threshold, cfg->clip_eps, cfg->flags);
  out->G_bar = G_bar;
  out->beta = beta;

  /* Eq. 5: Delta_hat = beta Delta_bar; Alg. 2 l.454: theta_{t+1} = OuterOpt(theta_t,
   * Delta_hat); l.455: theta_{t+1,0} = theta_{t+1} (stored, then rounded, R16). */
  for (int m = 0; m < M; ++m) {
    double* g = dbar + (size_t)m * numel; /* reused as Delta_hat */
    for (int64_t k = 0; k < numel; ++k) g[k] = beta * g[k];
    double* a = delta; /* reused as the fp64 anchor of shard m */
    double* mom = (double*)malloc(len * sizeof(double));
    if (!mom) { free(delta); free(dbar); return -1; }
    for (int64_t k = 0; k < numel; ++k) {
      a[k] = (double)anchors[(size_t)m * numel + k];
      mom[k] = (double)momenta[(size_t)m * numel + k];
    }
    oracle_outer_nesterov(a, mom, g, numel, cfg->outer_lr, cfg->outer_momentum);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < numel; ++k) {
      float a32 = (float)a[k];
      anchors[(size_t)m * numel + k] = a32;
      momenta[(size_t)m * numel + k] = (float)mom[k];
      for (int n = 0; n < N; ++n) {
        size_t i = (((size_t)m * N + n) * numel) + k;
        if (local_is_bf16) ((uint16_t*)locals_out)[i] = oracle_f32_to_bf16_rne(a32);
        else ((float*)locals_out)[i] = a32;
      }
    }
    free(mom);
  }
#undef LOCAL
  free(delta);
  free(dbar);
  return 0;
}

/* ---------------------------------------------------------------------------
 * Warm-up phase gradient synchronisation (Alg. 1 l.422-424):
 *   "If the current step t is within the warmup phase, an additional all-reduce
 *    operation will be performed within each model sync group to synchronize
 *    gradients across all workers" -- read as the MEAN over the N members (SPEC
 *    S:313-321 all_reduce_mean; the shard group's reduce-scatter averages too).
 * grads [N][numel] as stored (bf16 bits or fp32); out [numel] in the same type:
 *   out[k] = round_to_dtype( (1/N) * sum_n grads[n][k] )   (fp64 sum in n order)
 * ------------------------------------------------------------------------- */
void oracle_allreduce_mean(int32_t N, int64_t numel, int32_t is_bf16, const void* grads, void* out) {
  const uint16_t* gb = (const uint16_t*)grads;
  const float* gf = (const float*)grads;
  for (int64_t k = 0; k < numel; ++k) {
    double s = 0.0;
    for (int n = 0; n < N; ++n)
      s += is_bf16 ? oracle_bf16_to_f64(gb[(size_t)n * numel + k]) : (double)gf[(size_t)n * numel + k];
    float m = (float)(s / (double)N);
    if (is_bf16) ((uint16_t*)out)[k] = oracle_f32_to_bf16_rne(m);
    else ((float*)out)[k] = m;
  }
}
