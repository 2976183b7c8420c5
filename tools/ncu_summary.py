"""Summarise an ncu report (--set full) of the sync kernels into profiles/.

usage: python tools/ncu_summary.py gpurun_out/X.ncu-rep NUMEL_PER_LAUNCH out.json [label]
Writes per-kernel duration, DRAM bytes read/write, achieved GB/s, % of DRAM peak,
registers, grid, occupancy; and merges dram bytes/element into profiles/ncu_traffic.json
(bench.py reports it as roofline.traffic)."""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIELDS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
          "launch__occupancy_limit_registers", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
          "lts__t_sector_hit_rate.pct"]
SCALE = {"us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1.0, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0,
         "Tbyte": 1e12}


def key_of(name: str) -> str:
    m = re.search(r"(pg_norm_kernel|outer_update_kernel|sumsq_kernel|decide_kernel|ag_update_tma_kernel|rs_tma_kernel)"
                  r"<?([^>]*)>?", name)
    if not m:
        return name[:40]
    base = m.group(1).replace("_kernel", "")
    args = m.group(2)
    dt = "bf16" if "bfloat16" in args else ("f32" if "float" in args else "")
    parts = [a.strip() for a in args.split(",")]
    flag = parts[1] if len(parts) > 1 else ""
    if base == "outer_update":
        return f"outer_update_{dt}_{'S' if flag in ('1', 'true') else 'local'}"
    if base in ("ag_update_tma", "rs_tma"):
        return f"{base.replace('_tma', '')}_{dt}"
    if base == "pg_norm":
        return f"pg_norm_{dt}_{'S' if flag in ('1', 'true') else 'noS'}"
    return base


def main():
    rep, numel, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    label = sys.argv[4] if len(sys.argv) > 4 else os.path.basename(rep)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        k = key_of(name)
        d = {"kernel": name}
        for f in FIELDS:
            if f in hdr:
                i = hdr.index(f)
                v = r[i].replace(",", "")
                try:
                    d[f] = float(v) * SCALE.get(units[i], 1.0)
                except ValueError:
                    d[f] = v
        t = d.get("gpu__time_duration.sum")
        rb, wb = d.get("dram__bytes_read.sum", 0.0), d.get("dram__bytes_write.sum", 0.0)
        d["dram_bytes_per_elem"] = (rb + wb) / numel
        d["dram_GBps"] = (rb + wb) / t / 1e9 if t else None
        res.setdefault(k, []).append(d)
    summary = {"report": label, "numel_per_launch": numel, "kernels": res}
    with open(out, "w") as f:
        json.dump(summary, f, indent=1)
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for k, lst in res.items():
        traffic[k] = {"dram_bytes_per_elem": sum(x["dram_bytes_per_elem"] for x in lst) / len(lst),
                      "source": label}
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1)
    for k, lst in res.items():
        for x in lst:
            print(f"{k:28s} {x['gpu__time_duration.sum']*1e6:9.1f} us  dram {x['dram_bytes_per_elem']:.3f} B/elem "
                  f"{x['dram_GBps']:.0f} GB/s  dram% {x.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')}"
                  f"  regs {x.get('launch__registers_per_thread')} grid {x.get('launch__grid_size')}")


if __name__ == "__main__":
    main()
