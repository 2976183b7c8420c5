"""A/B of the a8 overlap (layer-wise prefetch behind a synthetic forward, as bench.py measures
it) for a given library build: 7B-shaped 1x1 round, all 34 units, h per partition setting.
usage: python tools/overlap_ab.py PKGROOT [--tokens 65536] [--sms -1,16,32,64] [--depth 1]"""
import argparse
import os
import sys

ap = argparse.ArgumentParser()
ap.add_argument("pkgroot")
ap.add_argument("--tokens", type=int, default=65536)
ap.add_argument("--sms", default="-1,16,32,64")
ap.add_argument("--depth", type=int, default=1)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--full-units", type=int, default=2)
args = ap.parse_args()
sys.path.insert(0, os.path.abspath(args.pkgroot))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(1, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from synth.forward import SyntheticForward  # noqa: E402
from paper_2412_07210_b200 import EditSync  # noqa: E402
import paper_2412_07210_b200 as pkg  # noqa: E402

dev = torch.device("cuda", 0)
units = synth.llama_units("7B")
numel = [u.numel for u in units]
s = EditSync(numel, device=dev)
import numpy as np  # noqa: E402
mu = np.array([[synth.ema_seed(u, 0)[0]] for u in units])
s.set_ema(mu, 0.1 * mu, 10)
anc = [synth.shard_anchor(u, i, 1, 0, dev) for i, u in enumerate(units)]
mom = [synth.shard_momentum(u, i, 1, 0, dev) for i, u in enumerate(units)]
loc = [torch.empty(n, dtype=torch.bfloat16, device=dev) for n in numel]
st = torch.cuda.current_stream(dev)
fwd = SyntheticForward("7B", units, args.tokens, dev)


def redraw(k):
    for i, u in enumerate(units):
        loc[i].copy_(synth.shard_local(u, i, 1, 0, 0, anc[i], torch.bfloat16, dev, round_salt=k))


def timed_once(fn, redraw_first=True, k=[0]):
    k[0] += 1
    if redraw_first:
        redraw(500 + k[0])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def timed(fn, redraw_first=True):
    ts = []
    for r in range(args.reps + 1):
        if redraw_first:
            redraw(100 + r)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    return sum(ts) / len(ts)


t_sync = timed(lambda: s.sync_round(loc, anc, mom, st))


def fwd_only():
    for u in range(len(units)):
        fwd.unit(u, loc[u])


t_fwd = timed(fwd_only, False)
print("lib", pkg.__file__, "tokens", args.tokens, "t_sync", round(t_sync, 2), "t_fwd", round(t_fwd, 1), flush=True)
for sms in [int(x) for x in args.sms.split(",")]:
    try:
        s.set_partition(sms, args.full_units)
    except Exception as e:
        print("sms", sms, "unsupported:", e)
        continue

    def both():
        s.begin_round(loc, anc, mom, args.depth, st)
        for u in range(len(units)):
            s.acquire(u, st)
            fwd.unit(u, loc[u])
        s.end_round(st)
    # paired: forward alone and forward + sync back to back, several pairs; the exposed time
    # is the median of the per-pair differences (the forward runs at the power cap, so its
    # own time drifts by more than t_sync between separate measurements)
    diffs, tb, tf = [], [], []
    for r in range(args.reps + 1):
        a_ = timed_once(fwd_only, False)
        b_ = timed_once(both, True)
        if r:
            diffs.append(b_ - a_)
            tb.append(b_)
            tf.append(a_)
    diffs.sort()
    ex = diffs[len(diffs) // 2]
    print(f"sms {sms:4d} depth {args.depth}: fwd {sum(tf) / len(tf):8.1f}  fwd+sync {sum(tb) / len(tb):8.1f} ms  "
          f"exposed(median pair) {ex:6.1f} ms  h {1 - ex / t_sync:6.3f}  diffs {[round(x, 1) for x in diffs]}", flush=True)
s.close()
