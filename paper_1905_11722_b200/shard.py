"""Exact DP with every wavefront level sharded across GPUs (BASELINE config C5;
SURVEY §8(e)).

One process per GPU (``torch.distributed``).  Every rank builds the same
family on its own device; in the level loop (inside libremat_b200) rank r
relaxes its contiguous share of each level's targets and the ranks then
all-gather the finished level over NVLink with NCCL (one ``ncclAllGather`` per
level).  Each rank ends with the whole DP table and returns the same
``PlanResult`` a single GPU would (the reference's ``dp_plan``,
``pkg/src/remat/planner.py:214-223``).

``loopback_plans`` runs the identical exchange with ``world`` replicas on one
device (device copies instead of NCCL) — the single-GPU test form.
"""

from __future__ import annotations

import time

from .graph import DEFAULT_LATTICE_CAP
from .planner import FAMILIES, OBJECTIVES, _result


def _dist(group=None):
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        raise RuntimeError("level sharding needs an initialised torch.distributed process group")
    return dist


def exchange_unique_id(group=None, make=None) -> bytes:
    """Rank 0 draws an NCCL unique id (``make``, default ncclGetUniqueId);
    every rank of ``group`` receives it."""
    dist = _dist(group)
    if make is None:
        from ._native import Comm

        make = Comm.unique_id
    box = [make() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0,
                               group=group)
    return box[0]


_COMMS: dict = {}


def communicator(device: int, group=None):
    """This process's NCCL communicator for ``group`` on ``device``, created
    once (ncclCommInitRank is collective and slow) and reused by every solve."""
    dist = _dist(group)
    key = (id(group) if group is not None else None, device, dist.get_world_size(group))
    comm = _COMMS.get(key)
    if comm is None or comm.handle is None:
        from ._native import Comm

        uid = exchange_unique_id(group)
        comm = Comm(uid, dist.get_world_size(group), dist.get_rank(group), device)
        _COMMS[key] = comm
    return comm


class LevelShardedSolver:
    """A (graph, family) resident on this rank's GPU, solved level-sharded."""

    def __init__(self, g, family: str = "full", lattice_cap: int = DEFAULT_LATTICE_CAP,
                 device: int | None = None, group=None):
        if family not in FAMILIES:
            raise ValueError(f"family must be one of {FAMILIES}, got {family!r}")
        if family == "full" and lattice_cap < g.n + 1:
            raise ValueError(f"cap must be at least n+1 = {g.n + 1}, got {lattice_cap}")
        from ._native import DeviceFamily, DeviceGraph

        self.graph, self.family_name = g, family
        self.dg = DeviceGraph(g, device)
        self.dev = DeviceFamily(self.dg, family, lattice_cap)
        self.comm = communicator(self.dg.device, group)

    def plans(self, budgets, objective: str = "minimize"):
        if objective not in OBJECTIVES:
            raise ValueError(f"objective must be one of {OBJECTIVES}, got {objective!r}")
        budgets = list(budgets)
        for b in budgets:
            if b < 0:
                raise ValueError("budget must be non-negative")
        t0 = time.perf_counter()
        raw = self.dev.solve_level_sharded(self.comm, budgets, objective)
        wall = time.perf_counter() - t0
        return [_result(r, b, self.family_name, objective, wall) for r, b in zip(raw, budgets)]

    def plan(self, budget: int, objective: str = "minimize"):
        return self.plans([budget], objective)[0]

    def timings(self) -> dict:
        return self.dev.timings()

    def close(self):
        self.dev.close()  # the communicator is shared (see communicator())
        self.dg.close()


def loopback_plans(g, budgets, world: int, family: str = "full", objective: str = "minimize",
                   lattice_cap: int = DEFAULT_LATTICE_CAP, device: int | None = None):
    """Level-sharded plans with ``world`` replicas on ONE device."""
    from ._native import DeviceFamily, DeviceGraph, solve_loopback

    dg = DeviceGraph(g, device)
    fams = [DeviceFamily(dg, family, lattice_cap) for _ in range(world)]
    try:
        t0 = time.perf_counter()
        raw = solve_loopback(fams, list(budgets), objective)
        wall = time.perf_counter() - t0
        return [_result(r, b, family, objective, wall) for r, b in zip(raw, budgets)]
    finally:
        for f in fams:
            f.close()
        dg.close()
