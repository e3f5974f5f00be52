import sys, os, time
sys.path.insert(0, os.getcwd())
from paper_1905_11722_b200 import named_graph, Solver
g = named_graph("densenet161")
for fam in ("pruned",):
    s = Solver(g, fam)
    for obj in ("minimize", "maximize"):
        for k in (8, 32, 144):
            s.min_feasible_budget(obj, k)
            t0 = time.perf_counter(); b, p = s.min_feasible_budget(obj, k); t1 = time.perf_counter()
            print(os.environ.get("REMAT_SMALL_FAMILY"), fam, obj, "probes", k, "b", b, round((t1 - t0) * 1e3, 1), "ms")
    t0 = time.perf_counter(); s.plan(2 * g.total_memory); t1 = time.perf_counter()
    print("single minimize solve at 2M(V)", round((t1 - t0) * 1e3, 1), "ms")
    s.close()
