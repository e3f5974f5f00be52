import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_1905_11722_b200 import Solver, named_graph
g = named_graph("unet", skip_len=3)
s = Solver(g, "full")
for k in (1, 2, 4, 8, 16, 32, 64):
    best = 1e9
    for _ in range(5):
        t0 = time.perf_counter(); b, p = s.min_feasible_budget("minimize", k); best = min(best, time.perf_counter() - t0)
    print(k, b, round(best * 1e3, 3), "ms", s.last_search if hasattr(s, "last_search") else "", flush=True)
