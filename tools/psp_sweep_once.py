"""One C4 full-family PSPNet 64-budget sweep (for ncu)."""
import os
import sys

sys.path.insert(0, os.getcwd())
from paper_1905_11722_b200 import Solver, named_graph  # noqa: E402
from paper_1905_11722_b200.sweep import sweep_budgets  # noqa: E402

g = named_graph("pspnet")
s = Solver(g, "full")
ps = s.plans(sweep_budgets(55, 385))
print(sum(p.stats.transitions for p in ps))
