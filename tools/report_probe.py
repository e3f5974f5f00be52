import sys, os, time
sys.path.insert(0, os.getcwd())
from paper_1905_11722_b200 import named_graph, build_report
import cProfile, pstats
for name, kw in [("unet", {"skip_len": 3}), ("densenet161", {}), ("resnet50", {})]:
    g = named_graph(name, **kw)
    build_report(g)
    t0 = time.perf_counter(); r = build_report(g); t1 = time.perf_counter()
    print(name, kw, "report", round((t1 - t0) * 1e3, 1), "ms")
    if name == "densenet161":
        pr = cProfile.Profile(); pr.enable(); build_report(g); pr.disable()
        pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
