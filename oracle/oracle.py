"""ctypes wrapper of the CPU oracle (``oracle/remat_oracle.c``).

TEST INFRASTRUCTURE ONLY — the parity checker and the CPU baseline ("port").
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  The product package
(``paper_1905_11722_b200``) never does.

Results come back as plain dicts whose keys mirror the reference ``PlanResult``
fields (``pkg/src/remat/planner.py:61-79``).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libremat_oracle.so"

OK, INFEASIBLE = 0, 1
ERR_ARG, ERR_LATTICE, ERR_NOMEM, ERR_ASSERT, ERR_PLANNER, ERR_SIM = -1, -2, -3, -4, -5, -6


class _Graph(C.Structure):
    _fields_ = [
        ("n", C.c_int), ("w", C.c_int),
        ("preds", C.c_void_p), ("succs", C.c_void_p),
        ("tcost", C.c_void_p), ("mcost", C.c_void_p),
    ]


class _Stats(C.Structure):
    _fields_ = [(k, C.c_int64) for k in
                ("states_visited", "table_entries", "transitions", "dominated_skipped")]


class _Plan(C.Structure):
    _fields_ = [
        ("feasible", C.c_int32),
        ("t_star", C.c_int64), ("cached_total", C.c_int64), ("peak", C.c_int64),
        ("overhead", C.c_int64),
        ("k", C.c_int32),
        ("chain", C.c_void_p), ("stage_memory", C.c_void_p),
        ("stats", _Stats),
        ("family_size", C.c_int64), ("pairs_expanded", C.c_int64),
    ]


class _Sim(C.Structure):
    _fields_ = [
        ("peak", C.c_int64), ("total_forward", C.c_int64), ("recompute", C.c_int64),
        ("backward_count", C.c_int64), ("err_idx", C.c_int64),
        ("err_code", C.c_int32), ("err_v", C.c_int32), ("err_w", C.c_int32),
    ]


_lib = None

# OpenMP barriers spin by default; with any other process on the box that
# turns into scheduler-quantum stalls.  Must be set before libgomp loads.
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")


def build() -> Path:
    """Compile the oracle with the Makefile next to this file."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        L.orc_family.argtypes = [C.POINTER(_Graph), C.c_int, C.c_int64, C.POINTER(C.c_int64),
                                 C.c_void_p, C.c_int64]
        L.orc_dp_plan.argtypes = [C.POINTER(_Graph), C.c_int, C.c_int64, C.c_int64, C.c_int,
                                  C.c_int, C.POINTER(_Plan)]
        L.orc_min_feasible_budget.argtypes = [C.POINTER(_Graph), C.c_int, C.c_int64, C.c_int,
                                              C.c_int, C.POINTER(C.c_int64), C.POINTER(_Plan),
                                              C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.orc_evaluate.argtypes = [C.POINTER(_Graph), C.c_int, C.c_void_p, C.POINTER(C.c_int64),
                                   C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.orc_simulate.argtypes = [C.POINTER(_Graph), C.c_int64, C.c_void_p, C.c_void_p,
                                   C.POINTER(_Sim)]
        _lib = L
    return _lib


class Packed:
    """A graph packed for the oracle (keeps the numpy buffers alive)."""

    def __init__(self, g):
        n = g.n
        w = max(1, (n + 63) // 64)
        self.n, self.w = n, w
        self.preds = np.zeros((n, w), dtype=np.uint64)
        self.succs = np.zeros((n, w), dtype=np.uint64)
        for v in range(n):
            for k in range(w):
                self.preds[v, k] = (g.preds[v] >> (64 * k)) & 0xFFFFFFFFFFFFFFFF
                self.succs[v, k] = (g.succs[v] >> (64 * k)) & 0xFFFFFFFFFFFFFFFF
        self.t = np.ascontiguousarray(g.compute_costs, dtype=np.int64)
        self.m = np.ascontiguousarray(g.memory_costs, dtype=np.int64)
        self.total_memory = int(self.m.sum())
        self.c = _Graph(n, w, self.preds.ctypes.data, self.succs.ctypes.data,
                        self.t.ctypes.data, self.m.ctypes.data)


def _words_to_int(row) -> int:
    out = 0
    for k, x in enumerate(row):
        out |= int(x) << (64 * k)
    return out


_FAM = {"full": 0, "pruned": 1}
_OBJ = {"minimize": 0, "maximize": 1}


def _threads(nthreads):
    if nthreads is None:
        return len(os.sched_getaffinity(0))
    return int(nthreads)


def family(g, name="full", cap=2_000_000):
    p = g if isinstance(g, Packed) else Packed(g)
    size = C.c_int64(0)
    rc = lib().orc_family(C.byref(p.c), _FAM[name], cap, C.byref(size), None, 0)
    if rc:
        raise RuntimeError(f"oracle family rc={rc}")
    buf = np.zeros((size.value, p.w), dtype=np.uint64)
    rc = lib().orc_family(C.byref(p.c), _FAM[name], cap, C.byref(size), buf.ctypes.data,
                          size.value)
    if rc:
        raise RuntimeError(f"oracle family rc={rc}")
    return [_words_to_int(r) for r in buf]


def _plan_dict(p: Packed, plan: _Plan, chain, stage, budget, fam, obj):
    stats = {k: int(getattr(plan.stats, k)) for k, _ in _Stats._fields_}
    if not plan.feasible:
        return {"feasible": False, "budget": budget, "family": fam, "objective": obj,
                "stats": stats, "family_size": int(plan.family_size)}
    k = plan.k
    return {
        "feasible": True,
        "objective_value": int(plan.t_star),
        "chain": [_words_to_int(chain[s]) for s in range(k)],
        "per_stage_memory": [int(x) for x in stage[:k]],
        "peak_memory": int(plan.peak),
        "overhead": int(plan.overhead),
        "cached_total": int(plan.cached_total),
        "budget": budget,
        "family": fam,
        "objective": obj,
        "stats": stats,
        "family_size": int(plan.family_size),
    }


def _new_plan(p: Packed):
    chain = np.zeros((p.n + 1, p.w), dtype=np.uint64)
    stage = np.zeros(p.n + 1, dtype=np.int64)
    plan = _Plan()
    plan.chain = chain.ctypes.data
    plan.stage_memory = stage.ctypes.data
    return plan, chain, stage


def _check(rc):
    if rc in (OK, INFEASIBLE):
        return
    names = {ERR_ARG: "ValueError", ERR_LATTICE: "LatticeTooLargeError", ERR_NOMEM: "MemoryError",
             ERR_ASSERT: "AssertionError", ERR_PLANNER: "PlannerError"}
    raise RuntimeError(f"oracle failed: {names.get(rc, rc)}")


def dp_plan(g, budget, family="full", objective="minimize", cap=2_000_000, nthreads=None):
    p = g if isinstance(g, Packed) else Packed(g)
    plan, chain, stage = _new_plan(p)
    rc = lib().orc_dp_plan(C.byref(p.c), _FAM[family], cap, int(budget), _OBJ[objective],
                           _threads(nthreads), C.byref(plan))
    _check(rc)
    return _plan_dict(p, plan, chain, stage, budget, family, objective)


def min_feasible_budget(g, family="full", objective="minimize", cap=2_000_000, nthreads=None):
    p = g if isinstance(g, Packed) else Packed(g)
    plan, chain, stage = _new_plan(p)
    b = C.c_int64(0)
    probes = C.c_int64(0)
    ptrans = C.c_int64(0)
    rc = lib().orc_min_feasible_budget(C.byref(p.c), _FAM[family], cap, _OBJ[objective],
                                       _threads(nthreads), C.byref(b), C.byref(plan),
                                       C.byref(probes), C.byref(ptrans))
    _check(rc)
    d = _plan_dict(p, plan, chain, stage, b.value, family, objective)
    d["probes"] = probes.value
    d["probe_transitions"] = ptrans.value
    return b.value, d


def evaluate(g, chain):
    p = g if isinstance(g, Packed) else Packed(g)
    k = len(chain)
    buf = np.zeros((max(k, 1), p.w), dtype=np.uint64)
    for s, m in enumerate(chain):
        for q in range(p.w):
            buf[s, q] = (m >> (64 * q)) & 0xFFFFFFFFFFFFFFFF
    stage = np.zeros(max(k, 1), dtype=np.int64)
    ovh, peak, cached = C.c_int64(), C.c_int64(), C.c_int64()
    rc = lib().orc_evaluate(C.byref(p.c), k, buf.ctypes.data, C.byref(ovh), stage.ctypes.data,
                            C.byref(peak), C.byref(cached))
    if rc:
        raise ValueError(f"oracle evaluate rc={rc}")
    return {"overhead": ovh.value, "per_stage_memory": [int(x) for x in stage[:k]],
            "peak_memory": peak.value, "cached_total": cached.value}


SIM_KIND = {"F": 0, "B": 1, "FREE_fwd": 2, "FREE_grad": 3}


def simulate(g, ops):
    """``ops``: int32 array [S][2] of (kind, node).  Returns a dict, or a dict
    with ``error=(idx, code, v, w)`` for a simulation fault."""
    p = g if isinstance(g, Packed) else Packed(g)
    ops = np.ascontiguousarray(ops, dtype=np.int32).reshape(-1, 2)
    trace = np.zeros(max(len(ops), 1), dtype=np.int64)
    res = _Sim()
    rc = lib().orc_simulate(C.byref(p.c), len(ops), ops.ctypes.data, trace.ctypes.data,
                            C.byref(res))
    if rc == ERR_SIM:
        return {"error": (int(res.err_idx), int(res.err_code), int(res.err_v), int(res.err_w))}
    if rc:
        raise ValueError(f"oracle simulate rc={rc}")
    return {"peak_live_memory": res.peak, "trace": [int(x) for x in trace[:len(ops)]],
            "total_forward_cost": res.total_forward, "recompute_cost": res.recompute,
            "backward_count": res.backward_count}
