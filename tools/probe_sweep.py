"""B_min search time vs probes per round (the k of the k-ary search)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_11722_b200 import Solver, named_graph  # noqa: E402

for name, g, fam, obj, ks in [("unet c=3 full min", named_graph("unet", skip_len=3), "full", "minimize", (4, 8, 16, 32, 64)),
                              ("unet c=6 full min", named_graph("unet", skip_len=6), "full", "minimize", (4, 8, 16, 32)),
                              ("pspnet full max", named_graph("pspnet"), "full", "maximize", (8, 16, 32, 64, 144)),
                              ("pspnet pruned min", named_graph("pspnet"), "pruned", "minimize", (8, 16, 32, 64, 144)),
                              ("resnet pruned min", named_graph("resnet50"), "pruned", "minimize", (8, 16, 32, 64, 144)),
                              ("densenet pruned max", named_graph("densenet161"), "pruned", "maximize", (48, 96, 144, 256))]:
    s = Solver(g, fam)
    out = []
    for k in ks:
        s.min_feasible_budget(obj, k)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            s.min_feasible_budget(obj, k)
            ts.append(time.perf_counter() - t0)
        out.append(f"k={k}: {min(ts) * 1e3:.1f} ms")
    print(name, "F", s.dev.size, " | ".join(out), flush=True)
    s.close()
