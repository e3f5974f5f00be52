"""B_min search time vs probes per round (k-ary search) on the BASELINE
search configs: C3 DenseNet-161 memory-centric (both families), C2 U-Net
skip 3, C1 ResNet-50 pruned."""
import sys
import time
sys.path.insert(0, "/root/repo")
from paper_1905_11722_b200 import Solver, named_graph  # noqa: E402

for name, g, fam, obj, ks in [
        ("C3 pruned max", named_graph("densenet161"), "pruned", "maximize", (144, 296, 592, 1024)),
        ("C3 full max", named_graph("densenet161"), "full", "maximize", (144, 296, 592, 1024)),
        ("C2 full min", named_graph("unet", skip_len=3), "full", "minimize", (2, 4, 8, 16, 32)),
        ("C1 pruned min", named_graph("resnet50"), "pruned", "minimize", (16, 32, 64, 144))]:
    s = Solver(g, fam)
    out, ref = [], None
    for k in ks:
        b, p = s.min_feasible_budget(obj, k)
        ref = ref or (b, p.objective_value)
        assert (b, p.objective_value) == ref
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            s.min_feasible_budget(obj, k)
            ts.append(time.perf_counter() - t0)
        out.append(f"k={k}: {min(ts) * 1e3:.2f} ms ({s.last_search['probes']} probes)")
    print(name, "F", s.dev.size, "2M(V)", 2 * g.total_memory, " | ".join(out), flush=True)
    s.close()
