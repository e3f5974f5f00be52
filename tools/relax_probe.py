"""Relaxation time of the bench workloads (min over repeats), for A/B runs of
kernel knobs set through the environment."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_11722_b200 import Solver, named_graph  # noqa: E402

cases = [("unet8", named_graph("unet", skip_len=8), 5),
         ("c5p03", named_graph("random-dag", depth=516, edge_prob=0.3, seed=0), 5)]
if "--big" in sys.argv:
    cases.append(("c5p02", named_graph("random-dag", depth=516, edge_prob=0.2, seed=0), 2))
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("REMAT_")}}
for name, g, rep in cases:
    s = Solver(g, "full")
    best = None
    for _ in range(rep):
        t0 = time.perf_counter()
        p = s.plan(2 * g.total_memory)
        dt = time.perf_counter() - t0
        tm = s.timings()
        if best is None or tm["relax_ms"] < best[0]:
            best = (tm["relax_ms"], dt * 1e3)
    out[name] = {"relax_ms": round(best[0], 3), "solve_ms": round(best[1], 3),
                 "X": p.stats.transitions, "t*": p.objective_value}
    s.close()
print(json.dumps(out), flush=True)
