"""A/B of the prefetch scheduler's partition mode alone (no forward): per-round time of a
7B-shaped 1x1 round restricted to `--units` decoder units, for fixed SM counts and lanes.
usage: python tools/sched_ab.py PKGROOT [--units 8] [--sms 8,16,32]   (PKGROOT holds the package)"""
import argparse
import os
import sys

ap = argparse.ArgumentParser()
ap.add_argument("pkgroot")
ap.add_argument("--units", type=int, default=8)
ap.add_argument("--sms", default="0,8,16,32,64")
ap.add_argument("--reps", type=int, default=4)
args = ap.parse_args()
sys.path.insert(0, os.path.abspath(args.pkgroot))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(1, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2412_07210_b200 import EditSync  # noqa: E402
import paper_2412_07210_b200 as pkg  # noqa: E402

dev = torch.device("cuda", 0)
units = synth.llama_units("7B")[1:1 + args.units]
numel = [u.numel for u in units]
s = EditSync(numel, device=dev)
anc = [synth.shard_anchor(u, i, 1, 0, dev) for i, u in enumerate(units)]
mom = [synth.shard_momentum(u, i, 1, 0, dev) for i, u in enumerate(units)]
loc = [synth.shard_local(u, i, 1, 0, 0, anc[i], torch.bfloat16, dev) for i, u in enumerate(units)]
st = torch.cuda.current_stream(dev)
P = sum(numel)
print("lib", pkg.__file__, "lanes", os.environ.get("EDIT_LANES", "default"))
for sms in [int(x) for x in args.sms.split(",")]:
    s.set_partition(sms, 0)
    ts = []
    for r in range(args.reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.begin_round(loc, anc, mom, 1, st)
        for u in range(len(units)):
            s.acquire(u, st)
        s.end_round(st)
        e1.record(st)
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    print(f"sms {sms:4d}: {ms:8.3f} ms  {26.0 * P / ms / 1e6:7.0f} GB/s  {26.0 * P / ms / 1e6 / max(sms, 1):6.1f} GB/s/SM")
s.close()
