"""Wall time vs device time of the small-config calls (C1, C2 search, C3):
how much of each call is host-side (planning, launches, syncs)."""
import sys
import time
sys.path.insert(0, "/root/repo")
import torch  # noqa: E402
from paper_1905_11722_b200 import (PlanRequest, Solver, dp_plan, memory_centric_plan,  # noqa: E402
                                   min_feasible_budget, named_graph)
from paper_1905_11722_b200._native import kernel_launches  # noqa: E402

cases = [("C1", lambda g: dp_plan(PlanRequest(g, 6929, "pruned")), named_graph("resnet50")),
         ("C2", lambda g: min_feasible_budget(g, "full"), named_graph("unet", skip_len=3)),
         ("C3p", lambda g: memory_centric_plan(g, "pruned"), named_graph("densenet161")),
         ("C3f", lambda g: memory_centric_plan(g, "full"), named_graph("densenet161"))]
for name, fn, g in cases:
    fn(g)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        n0 = kernel_launches()
        t0 = time.perf_counter()
        fn(g)
        dt = time.perf_counter() - t0
        best = min(best, dt)
        nl = kernel_launches() - n0
    print(name, f"wall {best*1e3:.2f} ms, launches {nl}", flush=True)
