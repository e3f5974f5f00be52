import sys, time, os
sys.path.insert(0, '/root/repo')
from paper_1905_11722_b200 import named_graph, Solver
from paper_1905_11722_b200.sweep import budget_sweep
import json
rec = json.load(open('/root/repo/tests/golden/bench_configs.json'))['data'][0]
b = rec['budgets']
g = named_graph("pspnet")
for fam in ("pruned", "full"):
    for k in range(3):
        t0 = time.perf_counter(); ps = budget_sweep(g, b, fam); t1 = time.perf_counter()
        print(fam, "sweep", k, round((t1-t0)*1e3, 1), "ms")
    s = Solver(g, fam)
    for k in range(3):
        t0 = time.perf_counter(); ps = s.plans(b); t1 = time.perf_counter()
        print(fam, "resident", k, round((t1-t0)*1e3, 1), "ms", s.timings())
    s.close()
g = named_graph("densenet161")
from paper_1905_11722_b200 import memory_centric_plan
for k in range(3):
    t0 = time.perf_counter(); memory_centric_plan(g, "pruned"); t1 = time.perf_counter()
    print("C3 pruned", round((t1-t0)*1e3, 1))
