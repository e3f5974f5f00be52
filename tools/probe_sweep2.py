import sys, time
sys.path.insert(0, '.')
from paper_1905_11722_b200 import Solver, named_graph
for name, g, fam, obj, ks in [("unet c=6 full min", named_graph("unet", skip_len=6), "full", "minimize", (1, 2, 3, 4)),
                              ("unet c=8 full min", named_graph("unet", skip_len=8), "full", "minimize", (1, 2, 4, 8)),
                              ("unet c=4 full min", named_graph("unet", skip_len=4), "full", "minimize", (1, 2, 4, 8)),
                              ("pspnet full max", named_graph("pspnet"), "full", "maximize", (1, 2, 4, 8)),
                              ("pspnet full min", named_graph("pspnet"), "full", "minimize", (1, 2, 4, 8)),
                              ("c5 p0.3 full min", named_graph("random-dag", depth=516, edge_prob=0.3), "full", "minimize", (1, 2, 4, 8))]:
    s = Solver(g, fam)
    out = []
    for k in ks:
        s.min_feasible_budget(obj, k)
        ts = []
        for _ in range(2):
            t0 = time.perf_counter(); s.min_feasible_budget(obj, k); ts.append(time.perf_counter() - t0)
        out.append(f"k={k}: {min(ts) * 1e3:.1f} ms")
    print(name, "F", s.dev.size, " | ".join(out), flush=True)
    s.close()
