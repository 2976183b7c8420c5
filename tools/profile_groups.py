"""ncu target: the unit-group kernels (group_norm / group_rs / group_ag) on ONE GPU, driven
through the simulated 1x2 mesh of tests/sim (two members on one device, so "NVLink" reads are
local HBM reads) with Llama-350M-shaped units -- for dram bytes per element and SASS evidence.
  ncu --set full --kernel-name regex:group_ -c 6 python tools/profile_groups.py
Not product code (test infrastructure drives it)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from tests.sim_mesh import SimMesh  # noqa: E402

dev = torch.device("cuda", 0)
units = synth.llama_units("350M")
numel = [u.numel for u in units]
sim = SimMesh(numel, 1, 2, dev, torch.bfloat16)
loc, anc, mom = [], [], []
for k in range(2):
    a = [synth.shard_anchor(u, i, 1, 0, dev) for i, u in enumerate(units)]
    anc.append(a)
    mom.append([synth.shard_momentum(u, i, 1, 0, dev) for i, u in enumerate(units)])
    loc.append([synth.shard_local(u, i, 1, 0, k, a[i], torch.bfloat16, dev) for i, u in enumerate(units)])
torch.cuda.synchronize()
for r in range(2):
    sim.sync_round(loc, anc, mom)
    torch.cuda.synchronize()
print("groups profiled:", sum(u.numel for u in units), "params per member")
sim.close()
