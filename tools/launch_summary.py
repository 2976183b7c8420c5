"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into profiles/.

usage: python tools/launch_summary.py gpurun_out/launches.csv profiles/rN_launches.md "command"
Keeps every launch of the library's kernels (edit::...) as a compact CSV next to the
summary, and reports each sync kernel's count, mean duration and share of the sync step.
(ncu serialises launches and runs them cold-cache: compare SHARES, not absolutes.)"""
import collections
import csv
import os
import sys

SCALE = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}


def main():
    src, out_md, cmd = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
    with open(src) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    ours, other = [], collections.Counter()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ms = float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1e-6)
        name = r["Kernel Name"]
        if "edit::" in name:
            short = name.split("(")[0].replace("void ", "").replace("edit::<unnamed>::", "")
            ours.append((int(r["ID"]), short, r["Grid Size"], r["Block Size"], ms))
        else:
            other[name.split("<")[0].split("(")[0][:60]] += ms
    agg = collections.defaultdict(list)
    for _, k, *_rest, ms in ours:
        agg[k].append(ms)
    total = sum(sum(v) for v in agg.values())
    csv_out = os.path.splitext(out_md)[0] + ".csv"
    with open(csv_out, "w") as f:
        f.write("id,kernel,grid,block,ms\n")
        for i, k, g, b, ms in ours:
            f.write(f'{i},"{k}","{g}","{b}",{ms:.6f}\n')
    with open(out_md, "w") as f:
        f.write(f"# ncu launch list: `{cmd}`\n\n")
        f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` (serialised, cold-cache; compare shares).\n")
        f.write(f"All {len(ours)} launches of the library's kernels are in `{os.path.basename(csv_out)}`.\n\n")
        f.write("| kernel | launches | mean us | total ms | share of sync kernels |\n|---|---|---|---|---|\n")
        for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
            f.write(f"| `{k}` | {len(v)} | {1e3 * sum(v) / len(v):.1f} | {sum(v):.2f} | {100 * sum(v) / total:.1f} % |\n")
        f.write(f"\nOther (non-library) kernels in the same run, e.g. the synthetic input redraw between steps "
                f"(outside the timed region): {sum(other.values()):.1f} ms total.\n")
    print(open(out_md).read())


if __name__ == "__main__":
    main()
