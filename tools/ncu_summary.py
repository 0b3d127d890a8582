"""Summarise an ncu --set full report: time, DRAM bytes, throughput, pipes, stalls, per-opcode mix."""
import csv, io, subprocess, sys, re
from collections import Counter

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [dict(zip(rows[0], r)) for r in rows[2:]], dict(zip(rows[0], rows[1]))

def main(rep, px=None):
    recs, units = raw(rep)
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum",
            "launch__grid_size", "launch__occupancy_limit_registers"]
    for r in recs:
        for k in keys:
            if k in r:
                print(f"  {k:60s} {r[k]} {units.get(k,'')}")
        stalls = {k: float(r[k]) for k in r if re.match(r"smsp__average_warp_latency_issue_stalled_.*_per_warp_active.pct$|smsp__pcsamp_warps_issue_stalled_[a-z_]+$", k) and r[k] not in ("", "0")}
        for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:10]:
            print(f"  stall {k:70s} {v}")
    if px:
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr = rows[1]; data = rows[2:]
        iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        c, st = Counter(), Counter()
        for r in data:
            if not r[iE].isdigit(): continue
            t = r[iS].strip().split()
            op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            c[op] += int(r[iE]); st[op] += int(r[iW] or 0)
        tot = sum(c.values())
        print(f"  thread-instr per px: {tot*32/px:.1f}")
        for k, v in c.most_common(18):
            print(f"    {k:10s} {v*32/px:6.1f}/px  stall-samples {st[k]}")

if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None)
