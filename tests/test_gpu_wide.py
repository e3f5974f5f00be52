"""Differential tests of the wide-bitset relaxation (W = 6..9 words: the
tile-intersection subset test, the one-class pair terms over padded 16-byte
mask rows, interior/boundary masks) against the CPU oracle, on dense random
DAGs of 380..520 nodes (families of 5..13 k members, so wide levels run as
per-level tile launches) with uniform costs of random magnitude (one weight
class, coefficients != 1) and with two or three cost classes."""

from __future__ import annotations

import random

import pytest

from _util import assert_plan_matches
from paper_1905_11722_b200 import Solver
from paper_1905_11722_b200.graph import graph_from_document

pytestmark = pytest.mark.gpu


def _dense_dag(rng: random.Random):
    n = rng.randint(380, 520)
    p = rng.choice([0.3, 0.32, 0.35])
    kind = rng.choice(["one-class", "one-class", "two-class", "three-class"])
    if kind == "one-class":
        tv, mv = rng.randint(1, 7), rng.randint(1, 9)
    nodes = []
    for i in range(n):
        if kind == "one-class":
            t, m = tv, mv
        elif kind == "two-class":
            t, m = rng.choice([(1, 2), (3, 5)])
        else:
            t, m = rng.choice([(1, 1), (2, 4), (0, 3)])
        nodes.append({"id": f"r{i}", "compute_cost": t, "memory_cost": m})
    edges = [[f"r{i}", f"r{j}"] for i in range(n) for j in range(i + 1, n) if rng.random() < p]
    return graph_from_document({"nodes": nodes, "edges": edges}), kind, p


@pytest.mark.parametrize("seed", range(8))
def test_wide_dense_dags_against_oracle(seed):
    from oracle import oracle as orc

    rng = random.Random(7000 + seed)
    done = 0
    while done < 1:
        g, kind, p = _dense_dag(rng)
        try:
            F = len(orc.family(g, "full", 30_000))
        except RuntimeError:
            continue  # lattice beyond the test budget
        done += 1
        s = Solver(g, "full", 30_000)
        top = 2 * g.total_memory
        budgets = sorted({top, rng.randint(top // 2, top)})
        plans = s.plans(budgets, "minimize")
        for b, plan in zip(budgets, plans):
            ref = orc.dp_plan(g, b, "full", "minimize", cap=30_000)
            assert_plan_matches(plan, ref, (seed, kind, p, g.n, F, b))
        s.close()
