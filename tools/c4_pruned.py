"""C4 pruned-family 64-budget sweep (PSPNet) wall time, best of 5."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
from paper_1905_11722_b200 import Solver, named_graph  # noqa: E402
from paper_1905_11722_b200.sweep import sweep_budgets  # noqa: E402

g = named_graph("pspnet")
s = Solver(g, "pruned")
bs = sweep_budgets(55, 385)
best = 1e9
for _ in range(5):
    t0 = time.perf_counter()
    ps = s.plans(bs)
    best = min(best, (time.perf_counter() - t0) * 1e3)
t = s.timings()
print(f"C4 pruned 64-budget sweep: best {best:.2f} ms, relax {t['relax_ms']:.3f} ms, "
      f"launches {t['relax_launches']}, X={sum(p.stats.transitions for p in ps)}", flush=True)
