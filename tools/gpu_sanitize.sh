#!/bin/bash
# compute-sanitizer memcheck + racecheck on small exact-DP solves (both key widths)
mkdir -p gpurun_out
cat > /tmp/san.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
from paper_1905_11722_b200 import named_graph, Solver, dp_plan, PlanRequest
from paper_1905_11722_b200.shard import loopback_plans
g = named_graph("unet", skip_len=2)
s = Solver(g, "full")
print(s.plans([2 * g.total_memory, 200]), flush=True)
print(s.min_feasible_budget("maximize")[0])
s.close()
g = named_graph("random-dag", depth=64, edge_prob=0.4, seed=0)
print(dp_plan(PlanRequest(g, 2 * g.total_memory, "full")).objective_value)
print(loopback_plans(g, [100], 3)[0].objective_value)
g = named_graph("resnet50")  # chain-like pruned family: one predecessor per warp, split tiles
print(dp_plan(PlanRequest(g, 6929, "pruned")).objective_value)
g = named_graph("densenet161")  # chain lattice: single-block enumeration runs
print(dp_plan(PlanRequest(g, 2 * g.total_memory, "full", "maximize")).objective_value)
# round 2: 16-target tiles (U-Net minimize above), pm cluster kernel (>= 8 budgets),
# every level exchanged in the loopback, the sparse-cell path (FLOP costs:
# global cells; forced on U-Net c=2 with shared-memory cells)
g = named_graph("unet", skip_len=2)
s = Solver(g, "full")
print([p.objective_value for p in s.plans(list(range(150, 150 + 16 * 20, 20)))])
s.close()
os.environ["REMAT_SHARD_REPLICATE"] = "0"
print(loopback_plans(g, [2 * g.total_memory], 2)[0].objective_value)
del os.environ["REMAT_SHARD_REPLICATE"]
# round 2 (late): wide bitsets (W = 5) through the per-level tile kernel:
# tile-intersection subset test, one-class pair terms over padded 16-byte rows
import random
from paper_1905_11722_b200.graph import graph_from_document
rng = random.Random(3)
doc = {"nodes": [{"id": f"r{i}", "compute_cost": 3, "memory_cost": 5} for i in range(300)],
       "edges": [[f"r{i}", f"r{j}"] for i in range(300) for j in range(i + 1, 300) if rng.random() < 0.33]}
g3 = graph_from_document(doc)
s = Solver(g3, "full", 30_000)
print("wide", s.size if hasattr(s, "size") else "", [p.objective_value for p in s.plans([2 * g3.total_memory, g3.total_memory])])
s.close()
import json
rec = json.load(open("tests/golden/large_costs.json"))["data"][5]
g2 = graph_from_document(rec["graph"])
print(dp_plan(PlanRequest(g2, 2 * g2.total_memory, "full")).objective_value)
os.environ["REMAT_FORCE_SPARSE"] = "1"
os.environ["REMAT_SPARSE_CELLS"] = "1024"
print(dp_plan(PlanRequest(g, 2 * g.total_memory, "full", "maximize")).objective_value)
PY
timeout 1200 compute-sanitizer --tool memcheck --leak-check no python /tmp/san.py > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck.log
REMAT_FORCE_WIDE=1 timeout 1200 compute-sanitizer --tool memcheck python /tmp/san.py > gpurun_out/memcheck_wide.log 2>&1; echo "rc=$?" >> gpurun_out/memcheck_wide.log
timeout 1800 compute-sanitizer --tool racecheck python /tmp/san.py > gpurun_out/racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck.log
timeout 1200 compute-sanitizer --tool synccheck python /tmp/san.py > gpurun_out/synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/synccheck.log
tail -n 3 gpurun_out/memcheck.log gpurun_out/memcheck_wide.log gpurun_out/racecheck.log gpurun_out/synccheck.log
