"""Seeded differential fuzzing of the CUDA solver against the CPU oracle on
graphs larger than the reference goldens (n = 12..60): uniform and varied
costs (the probe and bare-RED candidate paths), activation-sized memories
(wide keys), both families and objectives, batches of 1..64 budgets (the
multi-CTA level path and the one-CTA-per-budget solver), every field."""

from __future__ import annotations

import random

import pytest

from _util import assert_plan_matches
from paper_1905_11722_b200 import Solver
from paper_1905_11722_b200.graph import graph_from_document

pytestmark = pytest.mark.gpu


def _graph(rng: random.Random):
    n = rng.randint(12, 60)
    p = rng.choice([0.08, 0.15, 0.3, 0.6])
    kind = rng.choice(["uniform", "conv", "wide", "mixed"])
    nodes = []
    for i in range(n):
        if kind == "uniform":
            t, m = 1, 1
        elif kind == "conv":
            t, m = rng.choice([1, 10]), rng.choice([1, 2, 4, 8, 16])
        elif kind == "wide":
            t, m = rng.randint(0, 30), rng.randint(1, 1 << 40)
        else:
            t, m = rng.randint(0, 5), rng.randint(1, 50)
        nodes.append({"id": f"v{i}", "compute_cost": t, "memory_cost": m})
    # a backbone chain keeps lattices manageable; random forward edges on top
    edges = [[f"v{i}", f"v{i + 1}"] for i in range(n - 1) if rng.random() < 0.85]
    edges += [[f"v{i}", f"v{j}"] for i in range(n) for j in range(i + 2, min(n, i + 12))
              if rng.random() < p]
    return graph_from_document({"nodes": nodes, "edges": edges}), kind


@pytest.mark.parametrize("seed", range(160))
def test_fuzz_against_oracle(seed):
    from oracle import oracle as orc

    rng = random.Random(1000 + seed)
    done = 0
    while done < 3:
        g, kind = _graph(rng)
        try:
            F = len(orc.family(g, "full", 5_000))
        except RuntimeError:
            continue  # lattice beyond the fuzz budget
        done += 1
        for fam in ("full", "pruned"):
            s = Solver(g, fam, 5_000)
            top = 2 * g.total_memory
            nb = rng.choice([1, 5, 64])
            budgets = sorted({rng.randint(0, top) for _ in range(nb)} | {top})
            for obj in ("minimize", "maximize"):
                plans = s.plans(budgets, obj)
                for b, plan in zip(budgets, plans):
                    ref = orc.dp_plan(g, b, fam, obj, cap=5_000)
                    assert_plan_matches(plan, ref, (seed, kind, g.n, F, fam, obj, b))
            b_min, plan = s.min_feasible_budget("minimize")
            ref_b, ref = orc.min_feasible_budget(g, fam, "minimize", cap=5_000)
            assert b_min == ref_b
            assert_plan_matches(plan, ref, (seed, kind, fam, "bmin"))
            s.close()


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_level_sharding_loopback_against_oracle(seed):
    """The level-sharded exchange (pack, all-gather, unpack per level) with
    2..5 replicas on one device, on the fuzz graphs: every field equals the
    oracle's, both objectives, pruned and full families."""
    from oracle import oracle as orc
    from paper_1905_11722_b200.shard import loopback_plans

    rng = random.Random(5000 + seed)
    done = 0
    while done < 2:
        g, kind = _graph(rng)
        try:
            orc.family(g, "full", 5_000)
        except RuntimeError:
            continue
        done += 1
        world = rng.randint(2, 5)
        top = 2 * g.total_memory
        budgets = sorted({rng.randint(0, top) for _ in range(3)} | {top})
        for fam in ("full", "pruned"):
            for obj in ("minimize", "maximize"):
                plans = loopback_plans(g, budgets, world, fam, obj, 5_000)
                for b, plan in zip(budgets, plans):
                    ref = orc.dp_plan(g, b, fam, obj, cap=5_000)
                    assert_plan_matches(plan, ref, (seed, kind, world, fam, obj, b))


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_one_cta_per_budget_minimize(seed):
    """Minimize batches with a budget for every SM and more run whole in the
    one-CTA-per-budget solver (k_solve_small, 64-item steps over long
    frontiers): every field equals the oracle's."""
    from oracle import oracle as orc

    rng = random.Random(9000 + seed)
    while True:
        g, kind = _graph(rng)
        try:
            F = len(orc.family(g, "full", 1_000))
        except RuntimeError:
            continue
        break
    top = 2 * g.total_memory
    budgets = sorted([rng.randint(0, top) for _ in range(159)] + [top])  # repeats allowed
    for fam in ("full", "pruned"):
        s = Solver(g, fam, 1_000)
        plans = s.plans(budgets, "minimize")
        for b, plan in zip(budgets, plans):
            ref = orc.dp_plan(g, b, fam, "minimize", cap=1_000)
            assert_plan_matches(plan, ref, (seed, kind, g.n, F, fam, b))
        s.close()
