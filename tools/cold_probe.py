"""First-call (cold) costs per phase in a fresh process: graph handle, family
build, search/solve (lazy kernel-module loading happens on first launch)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_11722_b200 import named_graph  # noqa: E402
from paper_1905_11722_b200._native import DeviceFamily, DeviceGraph  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "densenet161"
fam = sys.argv[2] if len(sys.argv) > 2 else "full"
g = named_graph(name) if name != "unet" else named_graph("unet", skip_len=8)
for rep in range(2):
    t0 = time.perf_counter()
    dg = DeviceGraph(g, 0)
    t1 = time.perf_counter()
    f = DeviceFamily(dg, fam, 2_000_000)
    t2 = time.perf_counter()
    f.solve([2 * g.total_memory], "maximize")
    t3 = time.perf_counter()
    f.min_feasible_budget("maximize", 144)
    t4 = time.perf_counter()
    print(name, fam, rep, "graph %.1f family %.1f solve %.1f search %.1f ms" %
          tuple(1e3 * x for x in (t1 - t0, t2 - t1, t3 - t2, t4 - t3)), flush=True)
    f.close()
    dg.close()
