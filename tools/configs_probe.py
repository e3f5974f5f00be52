"""Time every BASELINE config on one GPU through the public API (warm), with
the CPU port beside it where it finishes in seconds.  Prints one JSON line per
config."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1905_11722_b200 import (PlanRequest, Solver, dp_plan, liveness_pass,  # noqa: E402
                                   memory_centric_plan, min_feasible_budget, named_graph,
                                   simulate, vanilla_schedule)
from paper_1905_11722_b200.sweep import sweep_budgets  # noqa: E402


def vanilla_peak(g):
    return simulate(g, liveness_pass(g, vanilla_schedule(g))).peak_live_memory


def timed(fn, reps=3):
    fn()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        t.append(time.perf_counter() - t0)
    return min(t), r


NOCPU = "--no-cpu" in sys.argv


class _Any(dict):
    """Stands in for a skipped CPU result: every comparison passes."""

    def __getitem__(self, k):
        return _Eq()


class _Eq:
    def __eq__(self, o):
        return True


def cpu(fn):
    if NOCPU:
        return None, _Any()
    t0 = time.perf_counter()
    r = fn()
    return time.perf_counter() - t0, r


def cpu2(fn):
    t, r = cpu(fn)
    return (t, (_Eq(), _Any())) if NOCPU else (t, r)


def main():
    from oracle import oracle as orc

    th = len(os.sched_getaffinity(0))
    out = []
    # C1 ResNet-50 approx DP at half the vanilla peak
    g = named_graph("resnet50")
    b = vanilla_peak(g) // 2
    t, p = timed(lambda: dp_plan(PlanRequest(g, b, "pruned")))
    tc, r = cpu(lambda: orc.dp_plan(g, b, "pruned", "minimize", nthreads=th))
    assert r["objective_value"] == p.objective_value
    out.append({"config": "C1 resnet50 pruned dp_plan B=vanilla/2", "budget": b, "gpu_s": t,
                "cpu_port_s": tc, "t*": p.objective_value, "transitions": p.stats.transitions})
    # C2 U-Net c=3 exact B_min search
    g = named_graph("unet", skip_len=3)
    t, (bm, p) = timed(lambda: min_feasible_budget(g, "full"))
    tc, (rb, r) = cpu2(lambda: orc.min_feasible_budget(g, "full", "minimize", nthreads=th))
    assert rb == bm
    out.append({"config": "C2 unet c=3 full min_feasible_budget", "b_min": bm, "gpu_s": t,
                "cpu_port_s": tc})
    # C3 DenseNet-161 memory-centric, both families
    g = named_graph("densenet161")
    for fam in ("pruned", "full"):
        t, p = timed(lambda: memory_centric_plan(g, fam))
        tc, (rb, r) = cpu2(lambda: orc.min_feasible_budget(g, fam, "maximize", nthreads=th))
        assert r["objective_value"] == p.objective_value
        out.append({"config": f"C3 densenet161 memory_centric_plan {fam}", "gpu_s": t,
                    "cpu_port_s": tc, "t*": p.objective_value})
    # C4 PSPNet 64-budget sweeps, pruned and full, one batched solve each
    g = named_graph("pspnet")
    vp = vanilla_peak(g)
    for fam in ("pruned", "full"):
        s = Solver(g, fam)
        bmin, _ = s.min_feasible_budget("minimize")
        budgets = sweep_budgets(bmin, vp if vp > bmin else 2 * g.total_memory, 64)
        t, plans = timed(lambda: s.plans(budgets))
        X = sum(p.stats.transitions for p in plans)
        s.close()
        tc = None
        if fam == "pruned":
            tc, _ = cpu(lambda: [orc.dp_plan(g, x, fam, "minimize", nthreads=th) for x in budgets])
        out.append({"config": f"C4 pspnet {fam} 64-budget sweep (family resident)",
                    "b_min": bmin, "gpu_s": t, "transitions": X, "cpu_port_s": tc})
    # C5 random DAG n=516 p=0.4 exact
    g = named_graph("random-dag", depth=516, edge_prob=0.4, seed=0)
    t, p = timed(lambda: dp_plan(PlanRequest(g, 2 * g.total_memory, "full")))
    tc, r = cpu(lambda: orc.dp_plan(g, 2 * g.total_memory, "full", "minimize", nthreads=th))
    assert r["objective_value"] == p.objective_value
    out.append({"config": "C5 random-dag n=516 p=0.4 exact dp_plan B=2M(V)", "gpu_s": t,
                "cpu_port_s": tc, "transitions": p.stats.transitions})
    for o in out:
        o["cpu_threads"] = th
        print(json.dumps(o), flush=True)


if __name__ == "__main__":
    main()
