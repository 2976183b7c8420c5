"""bench.py's driver contract on CPU: the reference arm (the fp64 oracle on the host cores)
prints ONE JSON line with the keys the driver reads; the GPU arm refuses a WORLD_SIZE that
does not match --gpus.  (The GPU arm itself is exercised on the B200 boxes.)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=e,
                          capture_output=True, text=True, timeout=600)


def test_reference_arm_prints_one_contract_line():
    r = _run(["--impl", "reference", "--steps", "2", "--warmup", "3", "--ref-sample", "50000"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 3
    assert d["unit"] == "GB/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"] and "model" not in d["config"]


def test_reference_arm_nonzero_rank_exits_silently():
    r = _run(["--impl", "reference", "--steps", "1", "--ref-sample", "1000"], env={"RANK": "1"})
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_warmup_floor_and_world_size_check():
    # W >= 3 is enforced; a --gpus that disagrees with WORLD_SIZE is refused before any GPU work
    r = _run(["--gpus", "2", "--steps", "1", "--warmup", "1"], env={"WORLD_SIZE": "1"})
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stderr + r.stdout)
