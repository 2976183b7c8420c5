// trigger.cpp -- WHEN a rank syncs (host logic, no device work): the EDiT step trigger of
// Alg. 1 l.408 ("if (t*tau + p) > t_warm and p == 0") and the A-EDiT time trigger of §3.3
// ("we set a fixed time interval tau_time, and let each worker update locally until
// surpassing this specified time threshold.  Then, a parameter synchronization ensues").
//
// A-EDiT needs no extra communication: every rank decides from its own clock at whole-step
// boundaries and then enters the (collective) sync; ranks that reach the
// threshold first wait inside the sync's first collective for the others, which are at most
// one step away -- "no worker will wait longer than the single step time of the slowest
// worker".  The time base restarts when the sync completes on this rank.
#include <math.h>

#include <new>

#include "edit_sync.h"

struct edit_trigger {
  int32_t kind = EDIT_TRIGGER_STEPS;
  int64_t tau = 1;
  double tau_time = 0.0;
  int64_t t_warm = 0;
  double last_sync = 0.0;  // A-EDiT: time base of the current inner loop
  int64_t syncs = 0;
};

extern "C" {

edit_status_t edit_trigger_create(int32_t kind, int64_t tau_steps, double tau_time_s, int64_t t_warm,
                                  double start_time_s, edit_trigger_t* out) {
  if (!out) return EDIT_ERR_INVALID_ARG;
  *out = nullptr;
  if (kind != EDIT_TRIGGER_STEPS && kind != EDIT_TRIGGER_TIME) return EDIT_ERR_INVALID_ARG;
  if (kind == EDIT_TRIGGER_STEPS && tau_steps < 1) return EDIT_ERR_INVALID_ARG;
  if (kind == EDIT_TRIGGER_TIME && !(tau_time_s > 0.0 && isfinite(tau_time_s))) return EDIT_ERR_INVALID_ARG;
  if (t_warm < 0 || !isfinite(start_time_s)) return EDIT_ERR_INVALID_ARG;
  edit_trigger* t = new (std::nothrow) edit_trigger();
  if (!t) return EDIT_ERR_NO_MEMORY;
  t->kind = kind;
  t->tau = tau_steps;
  t->tau_time = tau_time_s;
  t->t_warm = t_warm;
  t->last_sync = start_time_s;
  *out = t;
  return EDIT_OK;
}

int32_t edit_trigger_in_warmup(edit_trigger_t t, int64_t step) {
  // Alg. 1 l.422: "if (t*tau + p) <= t_warm": synchronous mini-batch phase
  return (t && step <= t->t_warm) ? 1 : 0;
}

int32_t edit_trigger_sync_now(edit_trigger_t t, int64_t step, double now_s) {
  if (!t || step <= t->t_warm) {
    // the local-SGD clock starts when the warm-up ends
    if (t) t->last_sync = now_s;
    return 0;
  }
  if (t->kind == EDIT_TRIGGER_STEPS) return (step % t->tau) == 0 ? 1 : 0;  // p == 0
  return (now_s - t->last_sync) >= t->tau_time ? 1 : 0;
}

edit_status_t edit_trigger_mark_synced(edit_trigger_t t, double now_s) {
  if (!t) return EDIT_ERR_INVALID_ARG;
  t->last_sync = now_s;
  t->syncs += 1;
  return EDIT_OK;
}

int64_t edit_trigger_syncs(edit_trigger_t t) { return t ? t->syncs : -1; }

edit_status_t edit_trigger_destroy(edit_trigger_t t) {
  delete t;
  return EDIT_OK;
}

}  // extern "C"
