"""Fixed cost of the level-sharded exchange on ONE GPU: the same solve through
Solver (no exchange) and through LevelShardedSolver on a one-rank
communicator with REMAT_SHARD_EXCHANGE=1 (pack, a real ncclAllGather, status
OR, unpack for every exchanged level).  Prints relax ms of both, the number of
exchanged levels and the cost per exchanged level."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29611")
os.environ["REMAT_SHARD_EXCHANGE"] = "1"
import torch.distributed as dist  # noqa: E402

dist.init_process_group("gloo", rank=0, world_size=1)
from paper_1905_11722_b200 import Solver, named_graph  # noqa: E402
from paper_1905_11722_b200.shard import LevelShardedSolver  # noqa: E402

p = float(sys.argv[1]) if len(sys.argv) > 1 else 0.2
g = named_graph("random-dag", depth=516, edge_prob=p, seed=0)
b = 2 * g.total_memory
out = {"workload": f"C5 random-dag n=516 p={p}", "replicate_tests": os.environ.get("REMAT_SHARD_REPLICATE", "default")}
s = Solver(g, "full")
ref = None
best = 1e9
for _ in range(3):
    ref = s.plan(b)
    best = min(best, s.timings()["relax_ms"])
out["single_relax_ms"] = best
ls = LevelShardedSolver(g, "full")
best, got = 1e9, None
for _ in range(3):
    got = ls.plan(b)
    best = min(best, ls.timings()["relax_ms"])
out["sharded_1rank_relax_ms"] = best
out["same_plan"] = (got.objective_value, got.stats.transitions) == (ref.objective_value, ref.stats.transitions)
# exchanged levels under the replicate threshold
thr = int(os.environ.get("REMAT_SHARD_REPLICATE", 4 << 20))
import numpy as np  # noqa: E402
pc = np.array([bin(m).count("1") for m in s.family.masks])
starts = np.searchsorted(pc, np.arange(g.n + 2))
ex = sum(1 for l in range(1, g.n + 1) if starts[l + 1] > starts[l]
         and (starts[l + 1] - starts[l]) * starts[l] > thr)
out["exchanged_levels"] = ex
out["us_per_exchanged_level"] = 1e3 * (out["sharded_1rank_relax_ms"] - out["single_relax_ms"]) / max(ex, 1)
print(json.dumps(out))
ls.close()
s.close()
dist.destroy_process_group()
