"""A/B of the relaxation variants (REMAT_PM and tuning knobs) on the long-frontier
workloads, with a parity check of every solve against the other mode's."""
import hashlib
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_11722_b200 import Solver, named_graph  # noqa: E402
from paper_1905_11722_b200.sweep import sweep_budgets  # noqa: E402

cases = [("unet8", named_graph("unet", skip_len=8), None),
         ("unet5", named_graph("unet", skip_len=5), None),
         ("psp_full64", named_graph("pspnet"), sweep_budgets(55, 385))]
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("REMAT_")}}
for name, g, budgets in cases:
    s = Solver(g, "full")
    bs = budgets or [2 * g.total_memory]
    best = None
    for _ in range(4):
        t0 = time.perf_counter()
        ps = s.plans(bs)
        dt = time.perf_counter() - t0
        tm = s.timings()
        if best is None or tm["relax_ms"] < best[0]:
            best = (tm["relax_ms"], dt * 1e3, tm["relax_launches"])
    sig = [(p.objective_value, p.stats.transitions, p.stats.table_entries, p.stats.states_visited,
            list(p.sequence.chain) if p.feasible else None) for p in ps]
    out[name] = {"relax_ms": round(best[0], 3), "solve_ms": round(best[1], 3),
                 "launches": best[2], "X": sum(p.stats.transitions for p in ps),
                 "sig": hashlib.md5(str(sig).encode()).hexdigest()[:12]}
    s.close()
print(json.dumps(out), flush=True)
