"""One exact-DP solve of a bench workload (for ncu / compute-sanitizer runs)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_11722_b200 import PlanRequest, dp_plan, named_graph  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="unet")
ap.add_argument("--skip-len", type=int, default=8)
ap.add_argument("--edge-prob", type=float, default=0.3)
ap.add_argument("--repeat", type=int, default=1)
a = ap.parse_args()
if a.workload == "unet":
    g = named_graph("unet", skip_len=a.skip_len)
else:
    g = named_graph("random-dag", depth=516, edge_prob=a.edge_prob)
for _ in range(a.repeat):
    p = dp_plan(PlanRequest(g, 2 * g.total_memory, "full"))
print("t*", p.objective_value, "transitions", p.stats.transitions)
