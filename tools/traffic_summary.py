"""Per-launch DRAM traffic of k_relax_tile from an ncu metrics CSV
(tools/gpu_traffic.sh) -> profiles/relax_traffic.json entry for bench.py."""
import csv
import json
import sys
from collections import defaultdict
from pathlib import Path

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9,
        "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}


def main(path, workload, out):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(dict)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1)
            per[d["ID"]][d["Metric Name"]] = v
    n = len(per)
    rd = sum(x.get("dram__bytes_read.sum", 0) for x in per.values())
    wr = sum(x.get("dram__bytes_write.sum", 0) for x in per.values())
    t = sum(x.get("gpu__time_duration.sum", 0) for x in per.values())
    rec = {"workload": workload, "kernel": "k_relax_tile", "launches": n,
           "dram_read_bytes": rd, "dram_write_bytes": wr,
           "dram_bytes_per_launch": (rd + wr) / max(n, 1),
           "ncu_seconds_total": t, "source": Path(path).name}
    p = Path(out)
    d = json.loads(p.read_text()) if p.exists() else {}
    d[workload] = rec
    p.write_text(json.dumps(d, indent=1) + "\n")
    print(json.dumps(rec))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "profiles/relax_traffic.json")
