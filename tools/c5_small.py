import sys, os
sys.path.insert(0, "/root/repo")
from paper_1905_11722_b200 import Solver, named_graph
out = []
for p in (0.4, 0.3, 0.2):
    g = named_graph("random-dag", depth=516, edge_prob=p, seed=0); s = Solver(g, "full")
    best = 1e9
    for _ in range(3):
        pl = s.plan(2 * g.total_memory); best = min(best, s.timings()["relax_ms"])
    out.append(f"p={p} relax {best:.3f} ({pl.objective_value},{pl.stats.transitions})")
    s.close()
g = named_graph("unet", skip_len=8); s = Solver(g, "full"); best = 1e9
for _ in range(3):
    pl = s.plan(2 * g.total_memory); best = min(best, s.timings()["relax_ms"])
out.append(f"unet8 relax {best:.3f}")
print(os.environ.get("REMAT_MIN_CHUNKS"), " | ".join(out), flush=True)
