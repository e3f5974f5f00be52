"""Summarise ncu exports: launch list shares (--launches csv) and one capture's
key metrics (--rep .ncu-rep).  Used to write profiles/*.md."""
import csv
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            u = d["Metric Unit"]
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                  "msecond": 1e3}.get(u, 1.0)
            out.append((d["Kernel Name"].split("(")[0], d["Grid Size"], v))
    agg = defaultdict(lambda: [0, 0.0])
    for k, g, v in out:
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {v[0]} | {v[1]:.1f} | {v[1] / tot:.3f} |")
    print(f"\ntotal device time {tot / 1e3:.2f} ms over {len(out)} launches")
    return out


def capture(path, keys=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    iS, iM, iU, iV = (h.index(x) for x in ("Section Name", "Metric Name", "Metric Unit",
                                           "Metric Value"))
    want = keys or {"Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate",
                    "L2 Hit Rate", "Compute (SM) Throughput", "Executed Ipc Active",
                    "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy",
                    "Registers Per Thread", "Grid Size", "Block Size", "No Eligible",
                    "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
                    "L2 Cache Throughput", "L1/TEX Cache Throughput", "Executed Instructions"}
    print("| metric | value |\n|---|---|")
    for row in r[1:]:
        if row[iM] in want:
            print(f"| {row[iM]} | {row[iV]} {row[iU]} |")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    hdr = next(csv.reader([raw[0]]))
    vals = next(csv.reader([raw[2]]))
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
              "smsp__average_warp_latency_issue_stalled_long_scoreboard",
              "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"):
        if m in hdr:
            print(f"| {m} | {vals[hdr.index(m)]} |")


def stalls(path, top=12):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    hdr = next(csv.reader([out[0]]))
    vals = next(csv.reader([out[2]]))
    items = []
    for name, v in zip(hdr, vals):
        if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
            try:
                items.append((float(v.replace(",", "")), name[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(x for x, _ in items) or 1
    print("| stall reason | share of samples |\n|---|---|")
    for v, n in sorted(items, reverse=True)[:top]:
        print(f"| {n} | {v / tot:.3f} |")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    elif sys.argv[1] == "--rep":
        capture(sys.argv[2])
        stalls(sys.argv[2])
