"""One C1 solve (ResNet-50 pruned family, B = half the vanilla peak) for ncu."""
import os
import sys

sys.path.insert(0, os.getcwd())
from paper_1905_11722_b200 import Solver, liveness_pass, named_graph, simulate, vanilla_schedule  # noqa: E402

g = named_graph("resnet50")
vp = simulate(g, liveness_pass(g, vanilla_schedule(g))).peak_live_memory
s = Solver(g, "pruned")
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    p = s.plan(vp // 2)
print(p.objective_value, s.timings())
s.close()
