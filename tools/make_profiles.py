"""Summarise ncu captures from gpurun_out/ into profiles/ (tracked).

    python tools/make_profiles.py r01 C5=gpurun_out/prof_c5g.ncu-rep C1=gpurun_out/prof_c1g.ncu-rep ...
                                  [--launches gpurun_out/launches_c5.csv]

Writes profiles/ncu_summary_<round>.json (per workload: kernel, duration,
dram read/write bytes per launch, throughputs, registers, occupancy, issue
activity, instruction mix per output pixel) and profiles/ncu_<round>_<W>.txt
(the same as text), plus profiles/launches_<round>.txt from a launch list.
bench.py reads dram_bytes from the JSON for roofline.traffic.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PX = {"C1": 3840 * 2160, "C2": 50 * 64 * 128, "C3": 4096 * 4096, "C4": 8192 * 224 * 224, "C5": 8192 * 224 * 224}
KEYS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "l1tex_throughput_pct": ("l1tex__throughput.avg.pct_of_peak_sustained_active", 1),
    "fp64_pipe_pct": ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1),
    "registers": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
    "warp_instructions": ("smsp__inst_executed.sum", 1),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-3, "us": 1, "ms": 1e3,
              "s": 1e6}


def ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def summarise(rep, px):
    rows = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))
    out = {"kernel": d.get("Kernel Name", "?"), "report": os.path.basename(rep)}
    for name, (metric, _) in KEYS.items():
        if metric not in d or d[metric] == "":
            continue
        v = float(d[metric].replace(",", ""))
        if name.startswith("dram_") and name.endswith("bytes"):
            v *= UNIT_SCALE.get(u.get(metric, "byte"), 1)
        if name == "duration_us":
            v *= UNIT_SCALE.get(u.get(metric, "us"), 1)
        out[name] = v
    if "dram_read_bytes" in out and "dram_write_bytes" in out:
        out["dram_bytes"] = int(out["dram_read_bytes"] + out["dram_write_bytes"])
    src = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    if len(src) > 2 and px:
        h = src[1]
        iS, iE = h.index("Source"), h.index("Instructions Executed")
        mix = Counter()
        for r in src[2:]:
            if r[iE].isdigit():
                t = r[iS].strip().split()
                op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "?")).split(".")[0]
                mix[op] += int(r[iE])
        total = sum(mix.values())
        out["thread_instructions_per_px"] = round(total * 32 / px, 1)
        out["top_opcodes_per_px"] = {k: round(v * 32 / px, 1) for k, v in mix.most_common(12)}
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[k]) for k in d
              if re.match(r"smsp__pcsamp_warps_issue_stalled_[a-z_]+$", k) and not k.endswith("not_issued")
              and d[k] not in ("", "0")}
    out["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
    return out


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = {}
    for r in rows[hi + 1:]:
        v = float(r[iv].replace(",", "")) * {"ns": 1e-3, "us": 1, "ms": 1e3}.get(r[iu], 1)
        agg.setdefault(r[ik], []).append(v)
    total = sum(sum(v) for v in agg.values())
    lines = [f"{'launches':>8} {'mean_us':>10} {'share':>6}  kernel"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{len(v):>8} {sum(v) / len(v):>10.1f} {sum(v) / total:>6.1%}  {k[:110]}")
    return "\n".join(lines)


def main():
    rnd = sys.argv[1]
    items = [a for a in sys.argv[2:] if "=" in a]
    launch = sys.argv[sys.argv.index("--launches") + 1] if "--launches" in sys.argv else None
    out_dir = os.environ.get("PROFILES_DIR", os.path.join(ROOT, "profiles"))
    os.makedirs(out_dir, exist_ok=True)
    path = os.path.join(out_dir, f"ncu_summary_{rnd}.json")
    summary = json.load(open(path)) if os.path.exists(path) else {}
    for item in items:
        w, rep = item.rsplit("=", 1)
        s = summarise(rep, PX.get(w.split("[")[0]))
        summary[w] = s
        with open(os.path.join(out_dir, f"ncu_{rnd}_{w}.txt"), "w") as f:
            f.write(json.dumps(s, indent=1) + "\n")
        print(w, s.get("kernel"), s.get("duration_us"), s.get("dram_bytes"))
    with open(path, "w") as f:
        json.dump(summary, f, indent=1)
    if launch:
        with open(os.path.join(out_dir, f"launches_{rnd}.txt"), "w") as f:
            f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none ({os.path.basename(launch)})\n")
            f.write(launches(launch) + "\n")


if __name__ == "__main__":
    main()
