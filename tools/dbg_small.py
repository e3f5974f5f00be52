import sys, os
sys.path.insert(0, os.getcwd())
from oracle import oracle as orc
from paper_1905_11722_b200 import named_graph, Solver, dp_plan, PlanRequest
g = named_graph("unet", skip_len=2)
rb, ref = orc.min_feasible_budget(g, "full", "maximize")
print("ref", rb, ref["objective_value"], ref["stats"])
s = Solver(g, "full")
for k in (1, 8, 48):
    b, p = s.min_feasible_budget("maximize", k)
    print("probes", k, b, p.objective_value, p.stats)
for bb in (rb, rb + 1, 2 * g.total_memory):
    p = s.plan(bb, "maximize"); r = orc.dp_plan(g, bb, "full", "maximize")
    print("single", bb, p.objective_value, r["objective_value"], p.stats.states_visited, r["stats"]["states_visited"])
ps = s.plans([rb, rb + 1, 2 * g.total_memory] * 4, "maximize")
print("batched", [(p.objective_value, p.stats.states_visited) for p in ps])
for bb in (rb, 2 * g.total_memory):
    p = s.plan(bb, "minimize"); r = orc.dp_plan(g, bb, "full", "minimize")
    print("min", bb, p.objective_value, r["objective_value"], p.stats.states_visited, r["stats"]["states_visited"])
