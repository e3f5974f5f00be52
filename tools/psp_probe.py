import json, os, sys, time, hashlib
sys.path.insert(0, '/root/repo')
from paper_1905_11722_b200 import Solver, named_graph
from paper_1905_11722_b200.sweep import sweep_budgets
g = named_graph("pspnet"); s = Solver(g, "full"); bs = sweep_budgets(55, 385)
best = None
for _ in range(3):
    ps = s.plans(bs); tm = s.timings()
    best = tm["relax_ms"] if best is None else min(best, tm["relax_ms"])
sig = hashlib.md5(str([(p.objective_value, p.stats.transitions, p.stats.table_entries) for p in ps]).encode()).hexdigest()[:12]
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("REMAT_")}, "psp_relax_ms": best, "sig": sig}))
