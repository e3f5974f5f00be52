import sys, os
sys.path.insert(0, os.getcwd())
from paper_1905_11722_b200 import named_graph, Solver, liveness_pass, simulate, vanilla_schedule
g = named_graph("resnet50")
vp = simulate(g, liveness_pass(g, vanilla_schedule(g))).peak_live_memory
s = Solver(g, "pruned"); p = s.plan(vp // 2); print(p.objective_value); s.close()
