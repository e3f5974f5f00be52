"""Enumeration (K1) time of the named lattices, best of 3 (family build only)."""
import sys
sys.path.insert(0, "/root/repo")
from paper_1905_11722_b200 import named_graph  # noqa: E402
from paper_1905_11722_b200._native import DeviceFamily, DeviceGraph  # noqa: E402

for name, kw in (("random-dag", dict(depth=516, edge_prob=0.2, seed=0)),
                 ("random-dag", dict(depth=516, edge_prob=0.3, seed=0)),
                 ("unet", dict(skip_len=8)), ("densenet161", {})):
    g = named_graph(name, **kw)
    dg = DeviceGraph(g)
    best, F = 1e9, 0
    for _ in range(3):
        f = DeviceFamily(dg, "full", 2_000_000)
        best = min(best, f.timings()["enumerate_ms"])
        F = f.size
        f.close()
    dg.close()
    print(name, kw, "F", F, "enumerate_ms", round(best, 3), flush=True)
