"""Phase split of the small configs (C1 dp_plan, C3 memory-centric searches)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_11722_b200 import (PlanRequest, Solver, dp_plan, liveness_pass,  # noqa: E402
                                   memory_centric_plan, named_graph, simulate, vanilla_schedule)


def best(fn, k=5):
    fn()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


g = named_graph("resnet50")
b = simulate(g, liveness_pass(g, vanilla_schedule(g))).peak_live_memory // 2
print("C1 dp_plan ms", best(lambda: dp_plan(PlanRequest(g, b, "pruned"))))
s = Solver(g, "pruned")
print("C1 Solver.plan ms", best(lambda: s.plan(b)), json.dumps(s.timings()))
print("  F", s.dev.size)
s.close()
g = named_graph("densenet161")
for fam in ("pruned", "full"):
    print("C3", fam, "memory_centric ms", best(lambda: memory_centric_plan(g, fam), 3))
    s = Solver(g, fam)
    print("  F", s.dev.size)
    print("  search ms", best(lambda: s.min_feasible_budget("maximize"), 3), json.dumps(s.timings()))
    s.close()
