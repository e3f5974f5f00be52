"""Issue-rate roofline of one relaxation launch: the ncu --set full capture's
executed IPC and issue-slot use against the measured per-SM issue peak
(tools/micro/pipes) -> profiles/relax_issue.json, read by bench.py.

  python tools/issue_summary.py <capture.ncu-rep> <pipes.json> <workload> [label]"""
import csv
import json
import subprocess
import sys
from pathlib import Path


def details(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    iM, iU, iV = (h.index(x) for x in ("Metric Name", "Metric Unit", "Metric Value"))
    return {row[iM]: (float(row[iV].replace(",", "")), row[iU]) for row in r[1:]
            if row[iV].replace(",", "").replace(".", "", 1).isdigit()}


def main(rep, pipes, workload, label="heaviest k_relax_tile launch"):
    d = details(rep)
    pk = json.loads(Path(pipes).read_text().strip().splitlines()[-1])
    ipc = d["Executed Ipc Active"][0]
    peak = pk["int32_warp_ops_per_clk_sm"]  # 4 issue slots per SM, measured 3.93 on IADD3/LOP3
    rec = {"workload": workload, "launch": label,
           "ipc": ipc, "issue_slots_busy": d["Issue Slots Busy"][0] / 100.0,
           "peak_ipc_measured": peak, "frac": ipc / peak,
           "instructions": d["Executed Instructions"][0],
           "duration_us": d["Duration"][0] * (1e3 if d["Duration"][1] == "ms" else 1.0),
           "red_shared_peak_per_clk_sm": pk["red_shared_warp_per_clk_sm"],
           "source": f"{Path(rep).name} (ncu --set full) + {Path(pipes).name}"}
    out = Path("profiles/relax_issue.json")
    db = json.loads(out.read_text()) if out.exists() else {}
    db[workload] = rec
    out.write_text(json.dumps(db, indent=1) + "\n")
    print(json.dumps(rec))


if __name__ == "__main__":
    main(*sys.argv[1:])
