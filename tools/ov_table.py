"""Summarise bench.py overlap blocks: python tools/ov_table.py file.json ..."""
import json
import sys

for f in sys.argv[1:]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    o = d["overlap"]
    sched = {k: round(v["ms"], 1) for k, v in o["t_sync_sched_alone_ms_by_partition"].items()}
    print(f"{f}: t_sync {o['t_sync_ms']:.1f} ms, sched-alone by sms {sched}")
    for r in o["runs"]:
        print(f"  tok {r['tokens_per_gpu']:6d} sms {r['partition_sms']:3d} d{r['depth']} fwd {r['t_fwd_ms']:7.1f} "
              f"both {r['t_fwd_plus_sync_ms']:7.1f} h {r['hidden_fraction']:+.3f} "
              f"W {r['clocks_fwd_plus_sync']['power_w']}")
