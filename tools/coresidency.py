"""Can the sync's streaming kernels co-reside with the forward's GEMMs on B200?

Runs a bf16 GEMM loop (the synthetic forward's largest GEMM shape) on stream A and the
library's N = 1 sync of one 7B unit in a loop on stream B, alone and together, with and
without a cap on... nothing: just measures both throughputs.  Dev tool, not product."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2412_07210_b200 import EditSync  # noqa: E402

dev = torch.device("cuda", 0)
T, h, I = 8192, 4096, 11008
x = torch.randn(T, h, device=dev, dtype=torch.bfloat16)
w = torch.randn(I, h, device=dev, dtype=torch.bfloat16)
u = synth.llama_units("7B")[1]
s = EditSync([u.numel], device=dev)
a = synth.shard_anchor(u, 1, 1, 0, dev)
m = synth.shard_momentum(u, 1, 1, 0, dev)
l = synth.shard_local(u, 1, 1, 0, 0, a, torch.bfloat16, dev)
sa, sb = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
NG, NS = 60, 20


def gemm_loop():
    with torch.cuda.stream(sa):
        for _ in range(NG):
            torch.matmul(x, w.t())


def sync_loop():
    for _ in range(NS):
        s.layer_sync(0, l, a, m, sb)


def timed(fns):
    torch.cuda.synchronize()
    e = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for k in ("a", "b")}
    e["a"][0].record(sa)
    e["b"][0].record(sb)
    for f in fns:
        f()
    e["a"][1].record(sa)
    e["b"][1].record(sb)
    torch.cuda.synchronize()
    return e["a"][0].elapsed_time(e["a"][1]), e["b"][0].elapsed_time(e["b"][1])


timed([gemm_loop, sync_loop])  # warm-up
g_alone, _ = timed([gemm_loop])
_, s_alone = timed([sync_loop])
g_both, s_both = timed([gemm_loop, sync_loop])
fl = 2 * T * h * I * NG
print(f"gemm alone {g_alone:.1f} ms ({fl / g_alone / 1e9:.0f} TF/s); sync alone {s_alone:.1f} ms "
      f"({26 * u.numel * NS / s_alone / 1e9:.0f} GB/s)")
print(f"together: gemm {g_both:.1f} ms, sync {s_both:.1f} ms; serial sum {g_alone + s_alone:.1f}; "
      f"overlap gain {(g_alone + s_alone - max(g_both, s_both)) / s_alone:.2f} of the sync time")
