"""Budget sweeps sharded across GPUs (BASELINE config C4).

Independent budgets of a sweep go to separate GPUs, one process per GPU
(``torch.distributed``): each rank builds the family once on its own device,
solves its contiguous share of the budgets in one batched launch sequence, and
the ranks exchange the finished ``PlanResult`` objects (host-side gather; there
is no data-path collective — the budgets never interact).
"""

from __future__ import annotations

from typing import Callable, Sequence

from .graph import DEFAULT_LATTICE_CAP


def sweep_budgets(b_min: int, top: int, count: int = 64) -> list[int]:
    """B_k = B_min + ⌊k·(top − B_min)/(count−1)⌋, k = 0…count−1."""
    if count < 2 or top <= b_min:
        return [b_min] * max(count, 1)
    return [b_min + (k * (top - b_min)) // (count - 1) for k in range(count)]


def shard(items: Sequence, world: int, rank: int) -> list:
    """Contiguous, balanced share of ``items`` for ``rank`` (first ranks take the
    remainder), so concatenating the shards in rank order restores the input."""
    n = len(items)
    q, r = divmod(n, world)
    lo = rank * q + min(rank, r)
    hi = lo + q + (1 if rank < r else 0)
    return list(items[lo:hi])


def _dist():
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return dist
    except Exception:
        pass
    return None


def budget_sweep(g, budgets: Sequence[int], family: str = "pruned",
                 objective: str = "minimize", lattice_cap: int = DEFAULT_LATTICE_CAP,
                 solve: Callable | None = None, group=None) -> list:
    """Plans for every budget, in input order, computed across all ranks.

    ``solve(g, budgets, family, objective, lattice_cap) -> list[PlanResult]``
    defaults to one resident ``Solver`` on this rank's GPU."""
    dist = _dist()
    world = dist.get_world_size(group) if dist else 1
    rank = dist.get_rank(group) if dist else 0
    mine = shard(list(budgets), world, rank)
    if solve is None:
        from .planner import Solver

        def solve(g, bs, family, objective, cap):
            if not bs:
                return []
            s = Solver(g, family, cap)
            try:
                return s.plans(bs, objective)
            finally:
                s.close()

    local = solve(g, mine, family, objective, lattice_cap)
    if world == 1:
        return local
    gathered: list = [None] * world
    dist.all_gather_object(gathered, local, group=group)
    return [p for part in gathered for p in part]


def min_feasible_budget_sharded(g, family: str = "full", objective: str = "minimize",
                                lattice_cap: int = DEFAULT_LATTICE_CAP, probes_per_rank: int = 8,
                                solve: Callable | None = None, group=None):
    """``min_feasible_budget`` (reference planner.py:271-297) with the probes of
    every search round spread over the ranks (one probe batch per
    GPU per round).  Feasibility is monotone in the budget, so
    any probe order finds the reference's B_min; the returned plan is the
    solve at B_min.  Each rank keeps one family resident for the whole search;
    a round exchanges only (budget, feasible) pairs.

    ``solve(g, budgets, family, objective, cap) -> list of plans`` with a
    ``feasible`` attribute or key (default: this rank's GPU ``Solver``)."""
    dist = _dist()
    world = dist.get_world_size(group) if dist else 1
    rank = dist.get_rank(group) if dist else 0
    solver = None
    if solve is None:
        from .planner import Solver

        solver = Solver(g, family, lattice_cap)

        def solve(g, bs, family, objective, cap):
            return solver.plans(bs, objective) if bs else []

    def feasible(p):
        return p["feasible"] if isinstance(p, dict) else p.feasible

    try:
        hi = 2 * g.total_memory            # always feasible
        lo = 2 * max(g.memory_costs) - 1   # no stage fits below 2·max_v M_v
        best = None                        # (budget, plan) of the smallest feasible probe
        while hi - lo > 1:
            k = world * probes_per_rank
            probes = sorted({lo + (hi - lo) * q // (k + 1) for q in range(1, k + 1)} - {lo, hi})
            if not probes:
                probes = [lo + (hi - lo) // 2]
            mine = shard(probes, world, rank)
            got = list(zip(mine, (feasible(p) for p in solve(g, mine, family, objective,
                                                              lattice_cap))))
            if world > 1:
                parts: list = [None] * world
                dist.all_gather_object(parts, got, group=group)
                got = [x for part in parts for x in part]
            ok = [b for b, f in got if f]
            if ok:
                hi = min(ok)
                below = [b for b, _ in got if b < hi]
                lo = max(below) if below else lo
            else:
                lo = max(b for b, _ in got)
        plan = solve(g, [hi], family, objective, lattice_cap)[0]
        return hi, plan
    finally:
        if solver is not None:
            solver.close()
