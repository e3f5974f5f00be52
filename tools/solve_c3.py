"""One C3 memory-centric search (DenseNet-161, pruned family) for ncu."""
import os
import sys

sys.path.insert(0, os.getcwd())
from paper_1905_11722_b200 import memory_centric_plan, named_graph  # noqa: E402

g = named_graph("densenet161")
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    p = memory_centric_plan(g, "pruned")
print(p.objective_value)
