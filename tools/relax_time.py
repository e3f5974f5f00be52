import sys
sys.path.insert(0, "/root/repo")
from paper_1905_11722_b200 import Solver, named_graph
for name, kw in (("random-dag", dict(depth=516, edge_prob=0.2, seed=0)), ("random-dag", dict(depth=516, edge_prob=0.3, seed=0)), ("unet", dict(skip_len=8))):
    g = named_graph(name, **kw); s = Solver(g, "full")
    best = 1e9
    for _ in range(3):
        p = s.plan(2 * g.total_memory); t = s.timings(); best = min(best, t["relax_ms"])
    print(name, kw, "relax_ms", round(best, 3), p.objective_value, p.stats.transitions)
    s.close()
