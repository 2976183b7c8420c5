"""Multi-rank parity over NCCL / NVLink peer memory (needs >= 2 GPUs; a mesh skips when the
box has fewer GPUs than ranks).

One torchrun per mesh runs every case of that mesh (tests/mp_parity_worker.py): rank 0
compares every rank's outputs with the fp64 oracle for the whole M x N mesh and checks the
cross-rank invariants.  Cases = (dtype, config, exchange algo, API):
  unit   edit_layer_sync per unit           round  edit_sync_round (2 lanes)
  reg    registered locals + round (peer)   gather fused shard all-gather + round (NEXT-2)
  sched  prefetch scheduler (a8)            schedpart  scheduler in partition mode (8 CTAs)
  graph  EDIT_GRAPH=1 round (captured CUDA graph; the checked round is a replay)
configs: ragged units, toy (BASELINE configs[0]: 4 x 64K fp32, replica 1 planted x4),
toy_clip, rollback (every replica anomalous), nan (one replica with a NaN param),
llama350m_sample, warm (NEXT-3 warm-up gradient all-reduce)."""
import os
import subprocess
import sys
from collections import defaultdict

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

ALGOS = ["peer", "nccl"]
UNIT_CASES = [
    ("1x2", "bf16", "ragged"), ("2x1", "bf16", "ragged"), ("1x2", "f32", "toy"), ("1x2", "bf16", "rollback"),
    ("1x2", "bf16", "nan"), ("2x2", "f32", "toy"), ("2x2", "f32", "toy_clip"), ("1x4", "bf16", "ragged"),
    ("2x2", "bf16", "rollback"), ("1x4", "bf16", "nan"), ("1x8", "bf16", "llama350m_sample"),
    ("2x4", "bf16", "ragged"), ("4x2", "bf16", "toy"), ("4x2", "f32", "toy_clip"), ("1x8", "bf16", "nan"),
]
ROUND_CASES = [("1x2", "bf16", "ragged"), ("2x2", "f32", "toy"), ("1x4", "bf16", "nan"), ("2x1", "bf16", "ragged"),
               ("2x4", "bf16", "toy"), ("1x8", "bf16", "ragged")]
REG_CASES = [("1x2", "bf16", "ragged"), ("2x2", "f32", "toy"), ("1x4", "bf16", "nan"), ("1x2", "f32", "rollback"),
             ("4x2", "bf16", "ragged"), ("1x8", "bf16", "toy")]
WARM_CASES = [("1x2", "bf16"), ("1x2", "f32"), ("2x2", "bf16"), ("1x4", "f32"), ("2x4", "bf16"), ("1x8", "bf16")]
GATHER_CASES = [("2x1", "bf16", "ragged"), ("2x2", "f32", "toy"), ("4x1", "bf16", "ragged"),
                ("2x2", "bf16", "rollback"), ("2x4", "bf16", "ragged"), ("4x2", "f32", "toy")]


def _core_cases(mesh):
    """The default subset (every feature once per mesh); EDIT_TEST_FULL=1 runs every case."""
    M, N = (int(x) for x in mesh.split("x"))
    c = [("bf16", "ragged", "peer", "unit"), ("f32", "toy", "nccl", "unit"), ("bf16", "nan", "peer", "round"),
         ("f32", "toy_clip", "peer", "unit")]
    c += [("bf16", "ragged", "peer", "schedpart"), ("bf16", "toy", "nccl", "sched"), ("bf16", "ragged", "peer", "graph")]
    if N > 1:
        c += [("bf16", "ragged", "peer", "reg"), ("bf16", "warm", "peer", "unit"), ("bf16", "rollback", "nccl", "round")]
    if M > 1:
        c += [("bf16", "ragged", "peer", "gather")]
    return c


def _mesh_cases():
    if not os.environ.get("EDIT_TEST_FULL"):
        meshes = sorted({m for m, *_ in UNIT_CASES + ROUND_CASES + REG_CASES + WARM_CASES + GATHER_CASES})
        return {m: _core_cases(m) for m in meshes}
    by_mesh = defaultdict(list)
    for algo in ALGOS:
        for mesh, dt, cfg in UNIT_CASES:
            by_mesh[mesh].append((dt, cfg, algo, "unit"))
        for mesh, dt, cfg in ROUND_CASES:
            by_mesh[mesh].append((dt, cfg, algo, "round"))
        for mesh, dt in WARM_CASES:
            by_mesh[mesh].append((dt, "warm", algo, "unit"))
        for mesh, dt, cfg in GATHER_CASES:
            by_mesh[mesh].append((dt, cfg, algo, "gather"))
    for mesh, dt, cfg in REG_CASES:
        by_mesh[mesh].append((dt, cfg, "peer", "reg"))
        by_mesh[mesh].append((dt, cfg, "peer", "schedpart"))
        by_mesh[mesh].append((dt, cfg, "nccl", "sched"))
        by_mesh[mesh].append((dt, cfg, "peer", "graph"))
        by_mesh[mesh].append((dt, cfg, "nccl", "graph"))
    return dict(sorted(by_mesh.items()))


MESH_CASES = _mesh_cases()


def _ngpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("mesh", list(MESH_CASES))
def test_multirank_parity(mesh):
    M, N = (int(x) for x in mesh.split("x"))
    if _ngpus() < M * N:
        pytest.skip(f"needs {M * N} GPUs, have {_ngpus()}")
    cases = MESH_CASES[mesh]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={M * N}",
           "--master-addr=127.0.0.1", "--master-port=29611", os.path.join(ROOT, "tests", "mp_parity_worker.py"),
           mesh] + [":".join(c) for c in cases]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=120 + 45 * len(cases))
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    for dt, cfg, algo, api in cases:
        assert f"PARITY OK {cfg} {mesh} {dt} {algo} {api}" in r.stdout, (cfg, dt, algo, api, r.stdout[-3000:])
