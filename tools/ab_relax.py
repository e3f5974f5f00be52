"""A/B of library builds on the relaxation workloads: relax time (best of 3)
and a signature of every plan (objective, stats, chain) so variants are
checked against each other.  REMAT_B200_LIB selects the build.
  python tools/ab_relax.py [case ...]   (cases: c5p2 c5p3 c5p4 unet8 psp64 dn)"""
import hashlib
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_11722_b200 import Solver, named_graph  # noqa: E402
from paper_1905_11722_b200.sweep import sweep_budgets  # noqa: E402

CASES = {
    "c5p2": (lambda: named_graph("random-dag", depth=516, edge_prob=0.2, seed=0), None, "minimize"),
    "c5p3": (lambda: named_graph("random-dag", depth=516, edge_prob=0.3, seed=0), None, "minimize"),
    "c5p4": (lambda: named_graph("random-dag", depth=516, edge_prob=0.4, seed=0), None, "minimize"),
    "unet8": (lambda: named_graph("unet", skip_len=8), None, "minimize"),
    "psp64": (lambda: named_graph("pspnet"), sweep_budgets(55, 385), "minimize"),
}
names = sys.argv[1:] or list(CASES)
out = {"lib": os.path.basename(os.environ.get("REMAT_B200_LIB", "libremat_b200.so"))}
for name in names:
    mk, budgets, obj = CASES[name]
    g = mk()
    s = Solver(g, "full")
    bs = budgets or [2 * g.total_memory]
    best = None
    for _ in range(3):
        ps = s.plans(bs)
        tm = s.timings()
        if best is None or tm["relax_ms"] < best:
            best = tm["relax_ms"]
    sig = [(p.objective_value, p.stats.transitions, p.stats.table_entries, p.stats.states_visited,
            list(p.sequence.chain) if p.feasible else None) for p in ps]
    out[name] = {"relax_ms": round(best, 3), "sig": hashlib.md5(str(sig).encode()).hexdigest()[:12]}
    s.close()
print(json.dumps(out), flush=True)
