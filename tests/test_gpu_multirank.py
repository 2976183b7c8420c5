"""Multi-rank parity over NCCL (needs >= 2 GPUs; each case skips when the box has fewer).

Launches tests/mp_parity_worker.py under torchrun; rank 0 compares every rank's outputs
with the fp64 oracle for the whole M x N mesh."""
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

CASES = [
    ("1x2", "bf16", "ragged"), ("2x1", "bf16", "ragged"), ("1x2", "f32", "toy"), ("1x2", "bf16", "rollback"),
    ("1x2", "bf16", "nan"), ("2x2", "f32", "toy"), ("2x2", "f32", "toy_clip"), ("1x4", "bf16", "ragged"),
    ("2x2", "bf16", "rollback"), ("1x4", "bf16", "nan"), ("1x8", "bf16", "llama350m_sample"),
    ("2x4", "bf16", "ragged"), ("4x2", "bf16", "toy"), ("4x2", "f32", "toy_clip"), ("1x8", "bf16", "nan"),
]
ALGOS = ["peer", "nccl"]
ROUND_CASES = [("1x2", "bf16", "ragged"), ("2x2", "f32", "toy"), ("1x4", "bf16", "nan"), ("2x1", "bf16", "ragged"),
               ("2x4", "bf16", "toy"), ("1x8", "bf16", "ragged")]


def _ngpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _run(mesh, dtype, config, algo, api):
    M, N = (int(x) for x in mesh.split("x"))
    if _ngpus() < M * N:
        pytest.skip(f"needs {M * N} GPUs, have {_ngpus()}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={M * N}",
           "--master-addr=127.0.0.1", "--master-port=29611", os.path.join(ROOT, "tests", "mp_parity_worker.py"),
           mesh, dtype, config, algo, api]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert f"PARITY OK {config} {mesh} {dtype} {algo} {api}" in r.stdout


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("mesh,dtype,config", CASES)
def test_multirank_parity(mesh, dtype, config, algo):
    _run(mesh, dtype, config, algo, "unit")


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("mesh,dtype,config", ROUND_CASES)
def test_multirank_parity_round_api(mesh, dtype, config, algo):
    # edit_sync_round: units pipelined over two lanes (own comms / exchange buffers each)
    _run(mesh, dtype, config, algo, "round")


@pytest.mark.parametrize("mesh,dtype,config", [("1x2", "bf16", "ragged"), ("2x2", "f32", "toy"), ("1x4", "bf16", "nan"),
                                               ("1x2", "f32", "rollback"), ("4x2", "bf16", "ragged"),
                                               ("1x8", "bf16", "toy")])
def test_multirank_parity_registered_locals(mesh, dtype, config):
    # peer path reading the members' registered local buffers directly (no staging copy)
    _run(mesh, dtype, config, "peer", "reg")


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("mesh,dtype", [("1x2", "bf16"), ("1x2", "f32"), ("2x2", "bf16"), ("1x4", "f32"),
                                        ("2x4", "bf16"), ("1x8", "bf16")])
def test_warmup_allreduce_parity(mesh, dtype, algo):
    # NEXT-3: the warm-up phase's gradient all-reduce over the sync group (Alg. 1 l.422-424)
    _run(mesh, dtype, "warm", algo, "unit")


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("mesh,dtype,config", [("2x1", "bf16", "ragged"), ("2x2", "f32", "toy"), ("4x1", "bf16", "ragged"),
                                               ("2x2", "bf16", "rollback"), ("2x4", "bf16", "ragged"),
                                               ("4x2", "f32", "toy")])
def test_fused_shard_allgather_parity(mesh, dtype, config, algo):
    # NEXT-2: the update kernel also writes the new local into every shard-group member's
    # full-module buffer; each rank's gathered module must equal its group's new locals
    _run(mesh, dtype, config, algo, "gather")
