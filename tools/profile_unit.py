"""Run the sync of a few Llama-7B-shaped units on one GPU (1 x 1 mesh) -- the bench's
launch configuration -- for ncu captures (`ncu -k regex:outer_update ...`)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2412_07210_b200 import EditSync  # noqa: E402

dtype = torch.bfloat16 if (len(sys.argv) < 2 or sys.argv[1] == "bf16") else torch.float32
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda", 0)
u = synth.llama_units("7B")[1]
s = EditSync([u.numel], param_dtype=dtype, device=dev)
mu = synth.ema_seed(u, 0)[0]
s.set_ema([[mu]], [[0.1 * mu]], 10)
a = synth.shard_anchor(u, 1, 1, 0, dev)
m = synth.shard_momentum(u, 1, 1, 0, dev)
for r in range(reps):
    l = synth.shard_local(u, 1, 1, 0, 0, a, dtype, dev, round_salt=r)
    s.layer_sync(0, l, a, m)
    torch.cuda.synchronize()
print("profile_unit done", s.stats(0).beta, s.kernel_launches)
