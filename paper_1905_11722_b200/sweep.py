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
