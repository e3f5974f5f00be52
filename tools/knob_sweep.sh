#!/bin/bash
# one pass of relax_probe (+ the C4 sweep) per library variant
# (paper_1905_11722_b200/libremat_b200*.so, built with make EXTRA=-D... OUT=...).
# The planner constants it was used to sweep (tasks per SM, split rounds,
# small-level threshold) are now fixed in relax_impl.cuh / relax.cu.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
probe() { timeout 300 python tools/relax_probe.py --big; timeout 300 python - <<'PY'
import sys, time
sys.path.insert(0, '.')
from paper_1905_11722_b200 import Solver, named_graph, liveness_pass, simulate, vanilla_schedule
from paper_1905_11722_b200.sweep import sweep_budgets
g = named_graph("pspnet")
vp = simulate(g, liveness_pass(g, vanilla_schedule(g))).peak_live_memory
s = Solver(g, "full"); bmin, _ = s.min_feasible_budget("minimize")
b = sweep_budgets(bmin, vp if vp > bmin else 2 * g.total_memory, 64)
s.plans(b); t0 = time.perf_counter(); s.plans(b); print("C4 full sweep ms", round((time.perf_counter() - t0) * 1e3, 1))
PY
}
for lib in paper_1905_11722_b200/libremat_b200*.so; do echo "== $lib"; REMAT_B200_LIB=$PWD/$lib probe; done
