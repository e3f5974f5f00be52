"""Per-level work profile of one exact solve: width, predecessor range,
comparable pairs P, transitions X, mean |frontier| of the level's members and
the pair density P / (width · predecessors) — the numbers that decide which
relaxation kernel a level wants.  Prints one JSON line per level."""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_11722_b200 import named_graph  # noqa: E402
from paper_1905_11722_b200._native import DeviceFamily, DeviceGraph  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="unet")
ap.add_argument("--skip-len", type=int, default=8)
ap.add_argument("--edge-prob", type=float, default=0.3)
a = ap.parse_args()
g = (named_graph("unet", skip_len=a.skip_len) if a.workload == "unet" else
     named_graph(a.workload) if a.workload in ("pspnet", "resnet50", "densenet161") else
     named_graph("random-dag", depth=516, edge_prob=a.edge_prob, seed=0))
dg = DeviceGraph(g)
fam = DeviceFamily(dg, "full", 2_000_000)
fam.solve([2 * g.total_memory], "minimize")
st = fam.member_stats(0)
pc = np.array([bin(m).count("1") for m in fam.masks()])
start = 0
for lvl in range(g.n + 1):
    idx = np.nonzero(pc == lvl)[0]
    if not len(idx):
        continue
    w = len(idx)
    P = int(st["pairs"][idx].sum())
    X = int(st["trans"][idx].sum())
    print(json.dumps({"level": lvl, "width": w, "preds": int(idx[0]), "P": P, "X": X,
                      "density": P / max(1, w * int(idx[0])), "X_per_P": X / max(1, P),
                      "flen_mean": float(st["flen"][idx].mean())}))
fam.close()
dg.close()
