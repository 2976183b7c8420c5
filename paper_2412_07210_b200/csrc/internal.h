// Internal declarations shared by api.cpp and kernels.cu (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "edit_sync.h"

namespace edit {

constexpr int kThreads = 256;   // threads per CTA of the streaming kernels
constexpr int kMaxCtas = 2048;  // upper bound of a streaming grid (per-CTA partial slots)
constexpr int kMaxRanks = EDIT_MAX_SYNC * EDIT_MAX_SHARD;

// Per-unit device scratch: partial sums, gathered scalars, the PreMulSum weight and
// the rollback decision of the unit's last sync.  One per unit so that the scalar
// chains of different units never share a slot.
struct alignas(256) LayerScratch {
  double send1;               // this rank's ||Delta_shard||^2            (K1 output)
  double gsq;                 // N == 1: G^2 of the module (= G_bar^2)    (K2 output)
  double send2;               // this rank's ||Dbar_shard||^2             (K3 output)
  double pad0;
  double recv1[kMaxRanks];    // gathered send1 of all K ranks, index n*M + m
  double recv2[EDIT_MAX_SHARD];  // gathered send2 of the M shard ranks
  float w;                    // own Eq. 2 weight: the PreMulSum scalar
  int32_t rollback;           // Alg. 2 l.448
  uint32_t counter1;          // last-CTA tickets
  uint32_t counter2;
  double cta1[kMaxCtas];      // per-CTA partials of K1
  double cta2[kMaxCtas];      // per-CTA partials of K3
};

struct DecideArgs {
  const double* parts;        // [M*N] gathered per-rank partial sums of squares
  int32_t M, N, my_n;
  edit_ema_t* ema;            // [N] EMA of this unit
  edit_layer_stats_t* rec;    // outcome record of this unit
  float* w_out;
  int32_t* rollback_out;
  double* gsq_out;
  double alpha, delta;
  int64_t warmup;
  uint32_t flags;
};

struct UpdateArgs {
  void* local;                // T*
  float* anchor;
  float* momentum;
  const float* dbar;          // N > 1: the all-reduced Dbar shard (nullptr for N == 1)
  int64_t n;
  const double* gparts;       // partial sums of ||Dbar||^2 to combine in order
  int32_t n_gparts;
  const int32_t* rollback;
  float nu, mu;
  double phi, eps;
  uint32_t flags;
  edit_layer_stats_t* rec;
};

// Launchers (kernels.cu).  Each returns the number of kernels launched.
int launch_pg_norm(int dtype, const void* local, const float* anchor, float* S, int64_t n,
                   LayerScratch* scr, int grid, cudaStream_t st);
int launch_sumsq(const float* x, int64_t n, LayerScratch* scr, int grid, cudaStream_t st);
int launch_decide(const DecideArgs& a, cudaStream_t st);
int launch_update(int dtype, const UpdateArgs& a, int grid, cudaStream_t st);

// Max co-resident CTAs of each streaming kernel (for grid sizing).
struct Occupancy {
  int pg_norm[2][2];  // [dtype][write_S]
  int sumsq;
  int update[2][2];   // [dtype][from_S]
};
cudaError_t query_occupancy(Occupancy* occ);

}  // namespace edit
