"""Enumeration time (family build) of the full-lattice configs, min over repeats."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_11722_b200 import named_graph  # noqa: E402
from paper_1905_11722_b200._native import DeviceFamily, DeviceGraph  # noqa: E402

out = {}
for name, g in [("unet8", named_graph("unet", skip_len=8)),
                ("c5p03", named_graph("random-dag", depth=516, edge_prob=0.3, seed=0)),
                ("c5p02", named_graph("random-dag", depth=516, edge_prob=0.2, seed=0)),
                ("densenet", named_graph("densenet161"))]:
    dg = DeviceGraph(g, 0)
    best = None
    for _ in range(4):
        fam = DeviceFamily(dg, "full", 2_000_000)
        t = fam.timings()["enumerate_ms"]
        best = t if best is None else min(best, t)
        F = fam.size
        fam.close()
    out[name] = {"enumerate_ms": round(best, 3), "F": F}
    dg.close()
print(json.dumps(out), flush=True)
