"""Phase times of the small-family BASELINE configs (C1 ResNet-50 pruned
dp_plan, C3 DenseNet-161 memory-centric search): wall time of the public call
and the device phases of every solve it issued (k-ary probe rounds)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
from paper_1905_11722_b200 import Solver, named_graph  # noqa: E402

for name, fam, kind in (("resnet50", "pruned", "c1"), ("densenet161", "pruned", "c3"),
                        ("densenet161", "full", "c3")):
    g = named_graph(name)
    s = Solver(g, fam)
    for rep in range(3):
        t0 = time.perf_counter()
        if kind == "c1":
            p = s.plan(6929)
            rounds = [s.timings()]
        else:
            b, p = s.min_feasible_budget("maximize")
            rounds = [s.timings()]
        dt = (time.perf_counter() - t0) * 1e3
    t = rounds[-1]
    print(f"{name} {fam} {kind}: wall {dt:.2f} ms, F={s.size if hasattr(s, 'size') else '?'}, last solve: "
          f"relax {t['relax_ms']:.3f} finish {t['finish_ms']:.3f} total {t['total_ms']:.3f} ms, "
          f"relax launches {t['relax_launches']}, kernels {t['kernel_launches']}", flush=True)
    s.close()
