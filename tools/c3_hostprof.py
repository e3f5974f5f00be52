import sys, time, cProfile, pstats
sys.path.insert(0, '.')
from paper_1905_11722_b200 import memory_centric_plan, named_graph
g = named_graph("densenet161")
for _ in range(3): memory_centric_plan(g, "full")
pr = cProfile.Profile(); pr.enable()
for _ in range(5): memory_centric_plan(g, "full")
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
