import sys, time
sys.path.insert(0, '.')
from paper_1905_11722_b200 import memory_centric_plan, named_graph, Solver
g = named_graph("densenet161")
for fam in ("full", "pruned", "full"):
    ts = []
    for _ in range(8):
        t0 = time.perf_counter(); memory_centric_plan(g, fam); ts.append(round((time.perf_counter() - t0) * 1e3, 1))
    print(fam, ts, flush=True)
s = Solver(g, "full")
ts = []
for _ in range(8):
    t0 = time.perf_counter(); s.min_feasible_budget("maximize"); ts.append(round((time.perf_counter() - t0) * 1e3, 1))
print("resident full", ts, s.timings())
