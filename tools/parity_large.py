"""Parity at sizes beyond the test suite (minutes of oracle time), recorded as
evidence: every field of the GPU plan against the 16-thread oracle."""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from _util import assert_plan_matches  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_1905_11722_b200 import Solver, named_graph  # noqa: E402

th = len(os.sched_getaffinity(0))
cases = [
    ("C5 random-dag n=516 p=0.25 full, B=2M(V)", named_graph("random-dag", depth=516, edge_prob=0.25), "full", "minimize", "top"),
    ("C5 random-dag n=516 p=0.3 full, B_min search", named_graph("random-dag", depth=516, edge_prob=0.3), "full", "minimize", "bmin"),
    ("U-Net c=8 full, maximize, B=2M(V)", named_graph("unet", skip_len=8), "full", "maximize", "top"),
    ("U-Net c=6 full, B_min search", named_graph("unet", skip_len=6), "full", "minimize", "bmin"),
    ("PSPNet full, memory-centric B_min search", named_graph("pspnet"), "full", "maximize", "bmin"),
]
for name, g, fam, obj, kind in cases:
    s = Solver(g, fam)
    t0 = time.perf_counter()
    if kind == "top":
        b = 2 * g.total_memory
        plan = s.plan(b, obj)
        tg = time.perf_counter() - t0
        t1 = time.perf_counter()
        ref = orc.dp_plan(g, b, fam, obj, nthreads=th)
    else:
        b, plan = s.min_feasible_budget(obj)
        tg = time.perf_counter() - t0
        t1 = time.perf_counter()
        rb, ref = orc.min_feasible_budget(g, fam, obj, nthreads=th)
        assert rb == b, (name, rb, b)
    tc = time.perf_counter() - t1
    assert_plan_matches(plan, ref, name)
    print(f"{name}: F={s.dev.size} budget={b} t*={plan.objective_value} "
          f"transitions={plan.stats.transitions} -- identical (GPU {tg * 1e3:.1f} ms, "
          f"oracle {tc:.1f} s on {th} threads)", flush=True)
    s.close()
