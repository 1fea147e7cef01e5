"""Summarise an ncu report (dev tool): key SOL metrics, stall reasons, hottest SASS lines.

usage: ncu_summary.py REPORT [TOP] [LAUNCH_INDEX ...]   (default: every profiled launch)
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
only = [int(x) for x in sys.argv[3:]]


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


want = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
        "Compute (SM) Throughput", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Executed Ipc Active", "Issue Slots Busy", "No Eligible", "Warp Cycles Per Issued Instruction",
        "L2 Hit Rate", "L1/TEX Hit Rate", "Mem Busy", "Max Bandwidth", "Dynamic Shared Memory Per Block"]
raw_keys = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
            "lts__t_sector_hit_rate.pct", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
            "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "smsp__inst_executed.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed_op_shared_ld.sum"]

det = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
h = raw[0]
ids = sorted({int(r[0]) for r in det[1:] if r and r[0].isdigit()})
for kid in ids:
    if only and kid not in only:
        continue
    name = next(r[4] for r in det[1:] if r and r[0] == str(kid))
    print(f"== launch {kid}: {name[:110]}")
    for r in det[1:]:
        if r and r[0] == str(kid) and len(r) > 14 and r[12] in want:
            print(f"  {r[12]:40s} {r[14]:>12s} {r[13]}")
    d = dict(zip(h, raw[2 + ids.index(kid)]))
    for k in raw_keys:
        if k in d:
            print(f"  {k:50s} {d[k]}")
    st = [(float(d[k].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for k in d
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
          and d[k].replace(",", "").replace(".", "").isdigit()]
    tot = sum(x for x, _ in st) or 1
    print("  stalls:", ", ".join(f"{n} {100*x/tot:.0f}%" for x, n in sorted(st, reverse=True)[:8]))
    src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass",
                                          "--filter-mode", "per-launch-config" if False else "global",
                                          "--launch-skip", str(kid), "--launch-count", "1"))))
    if len(src) < 2:
        continue
    hh = src[1] if "Source" in src[1] else src[0]
    try:
        i_s, i_src = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source")
    except ValueError:
        continue
    rows = []
    for r in src[2:]:
        try:
            rows.append((int(r[i_s]), r[0][-5:], r[i_src]))
        except Exception:
            pass
    t = sum(x[0] for x in rows) or 1
    for x in sorted(rows, reverse=True)[:top]:
        print(f"  {100*x[0]/t:5.1f}% {x[1]} {x[2][:100]}")
