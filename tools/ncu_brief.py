"""Brief per-kernel summary of an ncu report: `ncu -i R --page raw --csv | python tools/ncu_brief.py`."""
import csv
import sys

rows = list(csv.reader([l for l in sys.stdin if l.startswith('"')]))
h = rows[0]
KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_bytes.sum"]
for r in rows[2:]:
    if len(r) < len(h):
        continue
    d = dict(zip(h, r))
    print("##", d.get("Kernel Name", "?")[:70])
    for k in KEYS:
        if k in d:
            print(f"  {k} = {d[k]}")
    st = [(float(v.replace(",", "")), k) for k, v in d.items()
          if k.startswith("smsp__average_warp_latency_issue_stalled_") or
          (k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"))]
    st = [x for x in st if x[0] > 0]
    for v, k in sorted(st, reverse=True)[:8]:
        print(f"  {k} = {v:g}")
