import sys, os, time
sys.path.insert(0, os.getcwd())
from paper_1905_11722_b200 import named_graph, Solver, liveness_pass, simulate, vanilla_schedule
g = named_graph("resnet50")
vp = simulate(g, liveness_pass(g, vanilla_schedule(g))).peak_live_memory
for rep in range(3):
    t0 = time.perf_counter(); s = Solver(g, "pruned"); t1 = time.perf_counter()
    p = s.plan(vp // 2); t2 = time.perf_counter()
    print("C1 build", round((t1 - t0) * 1e3, 3), "ms solve", round((t2 - t1) * 1e3, 3), "ms", s.timings(), p.stats)
    s.close()
g = named_graph("densenet161")
for rep in range(4):
    s = Solver(g, "pruned"); t1 = time.perf_counter()
    b, p = s.min_feasible_budget("maximize"); t2 = time.perf_counter()
    print("C3 search", round((t2 - t1) * 1e3, 3), "ms", s.timings())
    s.close()
