"""Planners for the budget-constrained recomputation problem (drop-in for
reference ``pkg/src/remat/planner.py``).

Same entry points, dataclasses, validation order and errors as the reference:
``dp_plan`` (planner.py:214), ``min_feasible_budget`` (271) and
``memory_centric_plan`` (300).  The work — family enumeration, pair constants,
the (lower set, overhead) DP, reconstruction and the plan's figures — runs on
the GPU through ``libremat_b200.so``; this module only marshals arguments and
builds the result objects.

``Solver`` keeps one graph + family resident in HBM so several budgets (a
sweep, a search, or the two solves of ``report.build_report``) share the
enumeration and precompute, the way the reference shares its
``TransitionIndex`` inside ``min_feasible_budget`` (planner.py:283-284).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

from .graph import DEFAULT_LATTICE_CAP, ComputationGraph
from .lattice import LowerSetFamily
from .strategy import LowerSetSequence, StrategyEvaluation

FAMILIES = ("full", "pruned")
OBJECTIVES = ("minimize", "maximize")

DEFAULT_DFS_STATE_CAP = 10_000_000
SMALL_FAMILY = 1100  # csrc/relax.cu kSmallFamily: one CTA per budget


class PlannerError(RuntimeError):
    """Planner invariant violation or unusable configuration (planner.py:36-37)."""


class SearchCapExceeded(PlannerError):
    """The exhaustive search visited more states than allowed (planner.py:40-41)."""


@dataclass(frozen=True)
class PlanRequest:
    graph: ComputationGraph
    budget: int
    family: str = "full"
    objective: str = "minimize"
    lattice_cap: int = DEFAULT_LATTICE_CAP

    def __post_init__(self):
        if self.budget < 0:
            raise ValueError("budget must be non-negative")
        if self.family not in FAMILIES:
            raise ValueError(f"family must be one of {FAMILIES}, got {self.family!r}")
        if self.objective not in OBJECTIVES:
            raise ValueError(f"objective must be one of {OBJECTIVES}, got {self.objective!r}")


@dataclass
class SearchStats:
    states_visited: int = 0
    table_entries: int = 0
    transitions: int = 0
    dominated_skipped: int = 0
    wall_time_s: float = 0.0


@dataclass(frozen=True)
class PlanResult:
    feasible: bool
    sequence: LowerSetSequence | None
    evaluation: StrategyEvaluation | None
    objective_value: int | None
    budget: int | None
    family: str
    objective: str
    stats: SearchStats


def _result(unpacked, budget, family: str, objective: str, wall: float) -> PlanResult:
    info, chain, cached, stages = unpacked
    st = info.stats
    stats = SearchStats(st.states_visited, st.table_entries, st.transitions,
                        st.dominated_skipped, wall)
    if info.status < 0:  # a failed self-check is the reference's assert, never "infeasible"
        raise AssertionError(f"plan for budget {budget} failed the reference self-check "
                             "(planner.py:206-210)")
    if info.status != 0:
        return PlanResult(False, None, None, None, budget, family, objective, stats)
    prev = 0
    segments = []
    for m in chain:
        segments.append(m & ~prev)
        prev = m
    seq = LowerSetSequence(tuple(chain), tuple(segments), tuple(cached))
    ev = StrategyEvaluation(info.overhead, tuple(stages), info.peak_memory, info.cached_total)
    return PlanResult(True, seq, ev, info.objective_value, budget, family, objective, stats)


class Solver:
    """One (graph, family) resident on a GPU, solved for any number of budgets."""

    def __init__(self, g, family: str = "full", lattice_cap: int = DEFAULT_LATTICE_CAP,
                 device: int | None = None):
        if family not in FAMILIES:
            raise ValueError(f"family must be one of {FAMILIES}, got {family!r}")
        if family == "full" and lattice_cap < g.n + 1:
            raise ValueError(f"cap must be at least n+1 = {g.n + 1}, got {lattice_cap}")
        from ._native import DeviceFamily, DeviceGraph

        self.graph = g
        self.family_name = family
        self.dg = DeviceGraph(g, device)
        self.dev = DeviceFamily(self.dg, family, lattice_cap)

    @property
    def family(self) -> LowerSetFamily:
        return LowerSetFamily._from_device(self.dev)

    def plans(self, budgets, objective: str = "minimize") -> list[PlanResult]:
        if objective not in OBJECTIVES:
            raise ValueError(f"objective must be one of {OBJECTIVES}, got {objective!r}")
        budgets = list(budgets)
        for b in budgets:
            if b < 0:
                raise ValueError("budget must be non-negative")
        t0 = time.perf_counter()
        raw = self.dev.solve(budgets, objective)
        wall = time.perf_counter() - t0
        return [_result(r, b, self.family_name, objective, wall) for r, b in zip(raw, budgets)]

    def plan(self, budget: int, objective: str = "minimize") -> PlanResult:
        return self.plans([budget], objective)[0]

    def min_feasible_budget(self, objective: str = "minimize",
                            probes_per_round: int | None = None) -> tuple[int, PlanResult]:
        if objective not in OBJECTIVES:
            raise ValueError(f"objective must be one of {OBJECTIVES}, got {objective!r}")
        if probes_per_round is None:
            # small families: maximize rounds run one budget per CTA (144 probes
            # cost what one does); minimize rounds spread every probe over CTAs.
            # Larger families fill the GPU with fewer probes: a round of k
            # probes costs ~k solves, so the search narrows to binary as the
            # family grows (measured on the B200: tools/probe_sweep2.py,
            # tools/search_sweep.py: DenseNet-161 maximize 18.0 ms at 144 probes,
            # 20.5 / 31.9 ms at 296 / 592)
            if self.dev.size <= SMALL_FAMILY:
                probes_per_round = 144 if objective == "maximize" else 32
            elif self.dev.size <= 15_000:
                probes_per_round = 4
            elif self.dev.size <= 40_000:
                probes_per_round = 2
            else:
                probes_per_round = 1
        t0 = time.perf_counter()
        bmin, raw, search = self.dev.min_feasible_budget(objective, probes_per_round)
        wall = time.perf_counter() - t0
        self.last_search = search
        return bmin, _result(raw, bmin, self.family_name, objective, wall)

    def timings(self) -> dict:
        return self.dev.timings()

    def close(self):
        self.dev.close()
        self.dg.close()


def dp_plan(req: PlanRequest) -> PlanResult:
    """Best plan within the requested family and budget (planner.py:214-223).

    ``minimize`` gives the least-overhead feasible plan, ``maximize`` the
    overhead-maximising one; an infeasible budget gives ``feasible=False``."""
    s = Solver(req.graph, req.family, req.lattice_cap)
    try:
        return s.plan(req.budget, req.objective)
    finally:
        s.close()


def min_feasible_budget(
    g,
    family: str = "full",
    objective: str = "minimize",
    lattice_cap: int = DEFAULT_LATTICE_CAP,
) -> tuple[int, PlanResult]:
    """Smallest integer budget with any feasible plan, and the plan at it
    (planner.py:271-297).  Feasibility is monotone in the budget, so the GPU's
    batched k-ary search returns the reference's binary-search answer."""
    s = Solver(g, family, lattice_cap)
    try:
        return s.min_feasible_budget(objective)
    finally:
        s.close()


def dfs_exhaustive_plan(req: PlanRequest, state_cap: int = DEFAULT_DFS_STATE_CAP) -> PlanResult:
    """Exhaustive depth-first search over every chain of the family — the
    reference's exponential optimality oracle (planner.py:226-268), kept on the
    host by design (n <= ~12, nothing for a GPU to do).  The
    family comes from the device; pair constants are the reference definitions
    (planner.py:104-131).  Raises ``SearchCapExceeded`` past ``state_cap``
    visited states."""
    from .graph import boundary, delta_minus, delta_plus, memory_of, time_of
    from .lattice import all_lower_sets, pruned_lower_sets
    from .strategy import make_sequence, peak_memory

    g = req.graph
    fam = all_lower_sets(g, req.lattice_cap) if req.family == "full" else pruned_lower_sets(g)
    masks = list(fam.masks)
    bound = [boundary(g, m) for m in masks]
    base = []
    for m in masks:
        out = delta_plus(g, m)
        base.append(memory_of(g, out & ~m) + memory_of(g, delta_minus(g, out) & ~m))
    nxt = [[] for _ in masks]
    for i, lo in enumerate(masks):
        for j in range(i + 1, len(masks)):
            hi = masks[j]
            if lo & ~hi:
                continue
            seg = hi & ~lo
            nxt[i].append((j, 2 * memory_of(g, seg) + base[j], time_of(g, seg & ~bound[j]),
                           memory_of(g, bound[j] & ~lo)))
    stats = SearchStats()
    t0 = time.perf_counter()
    minimize = req.objective == "minimize"
    full = len(masks) - 1
    best = None
    trail: list[int] = []
    # explicit stack: (cell, t, m, next successor position)
    stack = [(0, 0, 0, 0)]
    stats.states_visited = 1  # the root visit counts (planner.py:242-246)
    if stats.states_visited > state_cap:
        raise SearchCapExceeded(f"exhaustive search exceeded {state_cap} states")
    while stack:
        i, t, m, k = stack[-1]
        if i == full:
            if best is None or (t < best[0] if minimize else t > best[0]):
                best = (t, trail.copy())
            stack.pop()
            if trail:
                trail.pop()
            continue
        if k == len(nxt[i]):
            stack.pop()
            if trail:
                trail.pop()
            continue
        stack[-1] = (i, t, m, k + 1)
        j, fixed, dt, dm = nxt[i][k]
        stats.transitions += 1
        if m + fixed > req.budget:
            continue
        stats.states_visited += 1
        if stats.states_visited > state_cap:
            raise SearchCapExceeded(f"exhaustive search exceeded {state_cap} states")
        trail.append(j)
        stack.append((j, t + dt, m + dm, 0))
    stats.wall_time_s = time.perf_counter() - t0
    if best is None:
        return PlanResult(False, None, None, None, req.budget, req.family, req.objective, stats)
    t_star, path = best
    seq = make_sequence(g, [masks[j] for j in path])
    ev = peak_memory(g, seq)
    # the reference's asserts (planner.py:265-266)
    if ev.overhead != t_star or ev.peak_memory > req.budget:
        raise AssertionError("exhaustive search produced an inconsistent plan")
    return PlanResult(True, seq, ev, t_star, req.budget, req.family, req.objective, stats)


def memory_centric_plan(g, family: str = "full",
                        lattice_cap: int = DEFAULT_LATTICE_CAP) -> PlanResult:
    """Overhead-maximising plan at the minimal feasible budget (planner.py:300-313)."""
    _, plan = min_feasible_budget(g, family, "maximize", lattice_cap)
    return plan
