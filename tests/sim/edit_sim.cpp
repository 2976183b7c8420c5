// edit_sim.cpp -- TEST INFRASTRUCTURE ONLY: a simulated M x N mesh on ONE GPU.
//
// The driver's GPU tests run on a 1-GPU box, where no multi-rank torchrun can exercise the
// N > 1 path.  This shim builds the K = M*N member handles of a mesh in one process on one
// device with the library's own create_local() (libedit_sync.so, paper_2412_07210_b200/csrc),
// wires them the way edit_sync_init wires real ranks -- every member's mailbox and peer
// buffers, registered locals and gather buffers -- but with plain device pointers instead of
// CUDA IPC mappings, and drives them through the library's own enqueue_units() /
// enqueue_warmup(): the production plan/step sequence (K1 + folded norm exchange + K2,
// RS + folded Dbar-norm exchange, AG + update, the NEXT-2 gather barrier, the warm-up
// kernels), launched on K streams.  Inside a unit the steps are enqueued step-major across
// the members, so a member's exchange never waits behind another member's later step.
//
// What it does not cover: NCCL (communicator setup, the EDIT_ALGO_NCCL / EDIT_XCHG=nccl
// baselines) and CUDA IPC -- the multi-rank tests (tests/test_gpu_multirank.py) do.
#include <vector>

#include "handle.h"

using namespace edit;

extern "C" {

// K member handles of an M x N mesh (cfg->rank is ignored: member k is rank k).  workspaces:
// K device buffers of edit_sync_workspace_bytes(cfg) each.  Peer exchange only (N > 1).
edit_status_t edit_sim_create(const edit_sync_config_t* cfg, void* const* workspaces, size_t ws_bytes,
                              edit_sync_t* out) {
  if (!cfg || !workspaces || !out) return fail(EDIT_ERR_INVALID_ARG, "null argument");
  const int M = cfg->shard_dim, N = cfg->sync_dim, K = M * N;
  if (N > 1 && cfg->algo != EDIT_ALGO_PEER) return fail(EDIT_ERR_INVALID_ARG, "the simulated mesh runs the peer path");
  for (int k = 0; k < K; ++k) out[k] = nullptr;
  for (int k = 0; k < K; ++k) {
    edit_sync_config_t c = *cfg;
    c.rank = k;
    edit_sync_t h = nullptr;
    const edit_status_t st = create_local(&c, workspaces[k], ws_bytes, &h);
    out[k] = h;
    if (st != EDIT_OK) return st;
    if (K > 1 && !h->dev_xchg) return fail(EDIT_ERR_INVALID_ARG, "the simulated mesh needs the mailbox exchange");
    h->simulated = true;
    h->ready = true;
  }
  const int nl = (int)out[0]->lanes.size();
  for (int k = 0; k < K; ++k) {
    edit_sync_t h = out[k];
    if ((int)h->lanes.size() != nl) return fail(EDIT_ERR_INVALID_ARG, "members disagree on EDIT_LANES");
    for (int li = 0; li < nl && K > 1; ++li) {
      Lane& ln = h->lanes[li];
      for (int r = 0; r < K; ++r) ln.mp.box[r] = out[r]->lanes[li].mailbox;
      if (h->peer)
        for (int j = 0; j < N; ++j) {
          const Lane& o = out[j * M + h->shard_idx]->lanes[li];  // member j of my sync row
          ln.pp.L[j] = o.Lown;
          ln.pp.D[j] = o.Down;
        }
    }
  }
  return EDIT_OK;
}

// locals: [K][L] device pointers (row k = member k), as edit_sync_register_locals per rank.
edit_status_t edit_sim_register_locals(edit_sync_t const* hs, int K, void* const* locals) {
  const int L = hs[0]->cfg.num_layers, M = hs[0]->M, N = hs[0]->N;
  for (int k = 0; k < K; ++k) {
    edit_sync_t h = hs[k];
    if (!h->peer) continue;
    h->reg_local.assign(locals + (size_t)k * L, locals + (size_t)(k + 1) * L);
    h->reg_peer.assign(L, std::vector<const void*>(N, nullptr));
    for (int u = 0; u < L; ++u)
      for (int j = 0; j < N; ++j) h->reg_peer[u][j] = locals[(size_t)(j * M + h->shard_idx) * L + u];
  }
  return EDIT_OK;
}

// bufs: [K][L] device pointers of M * layer_numel[u] elements, as edit_sync_register_gather.
edit_status_t edit_sim_register_gather(edit_sync_t const* hs, int K, void* const* bufs) {
  const int L = hs[0]->cfg.num_layers, M = hs[0]->M;
  if (M == 1) return EDIT_OK;
  for (int k = 0; k < K; ++k) {
    edit_sync_t h = hs[k];
    h->reg_gather.assign(L, std::vector<void*>(M, nullptr));
    for (int u = 0; u < L; ++u)
      for (int q = 0; q < M; ++q) h->reg_gather[u][q] = bufs[(size_t)(h->sync_idx * M + q) * L + u];
  }
  return EDIT_OK;
}

// edit_layer_sync on each of the nh given members (a subset leaves the others silent: the
// exchange-timeout test).  locals/anchors/momenta/streams: [nh].
edit_status_t edit_sim_layer_sync(edit_sync_t const* hs, int nh, int32_t layer, void* const* locals,
                                  float* const* anchors, float* const* momenta, void* const* streams) {
  return enqueue_units(hs, nh, 1, &layer, locals, anchors, momenta, reinterpret_cast<const cudaStream_t*>(streams),
                       false);
}

// edit_sync_round on each member (units dealt over the lanes).  [nh][L] pointer arrays.
edit_status_t edit_sim_round(edit_sync_t const* hs, int nh, void* const* locals, float* const* anchors,
                             float* const* momenta, void* const* streams) {
  const int L = hs[0]->cfg.num_layers;
  std::vector<int32_t> layers(L);
  for (int u = 0; u < L; ++u) layers[u] = u;
  return enqueue_units(hs, nh, L, layers.data(), locals, anchors, momenta,
                       reinterpret_cast<const cudaStream_t*>(streams), true);
}

// edit_warmup_allreduce (peer-memory variant) on each member.  grads/streams: [nh].
edit_status_t edit_sim_warmup_allreduce(edit_sync_t const* hs, int nh, int32_t layer, void* const* grads,
                                        void* const* streams) {
  return enqueue_warmup(hs, nh, layer, grads, reinterpret_cast<const cudaStream_t*>(streams), true);
}

// edit_warmup_allreduce_round (peer-memory variant) on each member: every unit, pipelined over
// the lanes.  grads: [nh][L]; streams: [nh].
edit_status_t edit_sim_warmup_allreduce_round(edit_sync_t const* hs, int nh, void* const* grads,
                                              void* const* streams) {
  return enqueue_warmup_units(hs, nh, hs[0]->cfg.num_layers, grads, reinterpret_cast<const cudaStream_t*>(streams),
                              true);
}

}  // extern "C"
