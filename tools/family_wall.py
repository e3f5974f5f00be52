"""Wall time of a family build (C-ABI remat_family_create) against its device phases."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_11722_b200 import named_graph  # noqa: E402
from paper_1905_11722_b200._native import DeviceFamily, DeviceGraph  # noqa: E402

for name, g in [("densenet", named_graph("densenet161")), ("unet8", named_graph("unet", skip_len=8)),
                ("resnet", named_graph("resnet50"))]:
    dg = DeviceGraph(g, 0)
    for fam in ("full", "pruned"):
        if name == "resnet" and fam == "full":
            continue
        ws = []
        for _ in range(6):
            t0 = time.perf_counter()
            f = DeviceFamily(dg, fam, 2_000_000)
            ws.append(round((time.perf_counter() - t0) * 1e3, 2))
            t = f.timings()
            f.close()
        print(name, fam, "wall ms", ws, "enumerate", round(t["enumerate_ms"], 3), "precompute",
              round(t["precompute_ms"], 3), flush=True)
    dg.close()

# the public-API pattern: a fresh graph handle (stream) per call
g = named_graph("densenet161")
for fam in ("full", "pruned"):
    ws, wg = [], []
    for _ in range(6):
        t0 = time.perf_counter()
        dg = DeviceGraph(g, 0)
        t1 = time.perf_counter()
        f = DeviceFamily(dg, fam, 2_000_000)
        t2 = time.perf_counter()
        f.close()
        dg.close()
        t3 = time.perf_counter()
        ws.append(round((t2 - t1) * 1e3, 2))
        wg.append((round((t1 - t0) * 1e3, 2), round((t3 - t2) * 1e3, 2)))
    print("fresh handle", fam, "family ms", ws, "graph create / close ms", wg, flush=True)

# the memory_centric_plan pattern: family build, 144-probe search, close
for fam in ("full", "pruned"):
    ws, ss = [], []
    for _ in range(6):
        dg = DeviceGraph(g, 0)
        t1 = time.perf_counter()
        f = DeviceFamily(dg, fam, 2_000_000)
        t2 = time.perf_counter()
        f.min_feasible_budget("maximize", 144)
        t3 = time.perf_counter()
        f.close()
        dg.close()
        ws.append(round((t2 - t1) * 1e3, 2))
        ss.append(round((t3 - t2) * 1e3, 2))
    print("after search", fam, "family ms", ws, "search ms", ss, flush=True)
