"""Upper bound on the hidden fraction h of the layer-wise sync behind a tensor-bound forward on
one B200, from measured constants, next to the measured h.

A tensor-bound forward loses the SM time the sync occupies, whichever SMs run it.  Streaming
through an SM is capped at ~100 GB/s per SM (profiles/r1_sm_stream_bench_v*.txt), so the sync
costs at least  SMB = P_r * B_sm / (100 GB/s)  SM-seconds, i.e. SMB / 148 seconds of whole-GPU
forward time; the units the forward reaches before any GEMM (embedding, layer 1) are exposed.

    h <= 1 - (SMB / 148 + t_exposed) / t_sync

B_sm = bytes per param that pass through the SMs of one rank (bf16 local, b_l = 2):
  N = 1: K1 6 + K4 20 = 26;
  peer path: K1 6 + RS (anchor slice 4/N + N local slices b_l + D write 4/N) + AG 22.
Power (both workloads at the 1000 W cap) lowers the real h further; it is not modelled.

usage: python tools/overlap_bound.py [profiles/r1_*.json ...]
"""
from __future__ import annotations

import json
import sys

PER_SM_GBS = 100.0
SMS = 148


def sm_bytes_per_param(N: int, b_l: int = 2) -> float:
    if N == 1:
        return 6.0 + 20.0                                   # K1 + K4
    rs = 4.0 / N + b_l * 1.0 + 4.0 / N                      # anchor slice + N locals' slices + D write
    ag = 4.0 + 8.0 + 10.0                                   # D pull + anchor, momentum read + 3 writes
    return (b_l + 4.0) + rs + ag                            # K1 reads local + anchor


def bound(P_r: float, N: int, t_sync_ms: float, t_exposed_ms: float) -> float:
    smb = P_r * sm_bytes_per_param(N) / (PER_SM_GBS * 1e9)  # SM-seconds
    return 1.0 - (smb / SMS * 1e3 + t_exposed_ms) / t_sync_ms


def main(paths):
    for p in paths:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        o = d.get("overlap")
        if not o:
            continue
        mesh = d["config"]["mesh"]
        N = int(mesh.split("x")[1])
        P_r = d["config"]["params_per_rank"]
        t_sync = o["t_sync_ms"]
        t_exposed = t_sync * (2.0 / 34.0) * 1.5           # embedding (~1.6 decoder units) + layer 1
        hb = bound(P_r, N, t_sync, t_exposed)
        best = {k: round(v["hidden_fraction"], 2) for k, v in o.get("best", {}).items()}
        print(f"{p}: mesh {mesh}, t_sync {t_sync:.1f} ms, SM bytes/param {sm_bytes_per_param(N):.1f}, "
              f"h bound {hb:.2f}, measured best {best}")


if __name__ == "__main__":
    main(sys.argv[1:] or ["profiles/r1_bench_1gpu_final2.json", "profiles/r1_bench_1x2_partition.json",
                          "profiles/r1_b4b_7B_1x4.json"])
