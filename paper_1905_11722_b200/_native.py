"""ctypes binding of ``libremat_b200.so`` (the C-ABI in ``include/remat_b200.h``).

There is no fallback: if the library is missing or no CUDA device is visible,
every solver entry point raises.  Build it with ``python -c "import
__graft_entry__ as g; g.build()"`` (or ``make -C paper_1905_11722_b200/csrc``).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .graph import GraphError, array_to_masks, masks_to_array, pack_graph

# REMAT_B200_LIB: an alternative build of the same library (A/B runs of kernel variants)
LIB_PATH = Path(os.environ.get("REMAT_B200_LIB") or
                Path(__file__).resolve().parent / "libremat_b200.so")

OK, INFEASIBLE = 0, 1
ERR_VALUE, ERR_LATTICE, ERR_CUDA, ERR_NOMEM, ERR_INTERNAL, ERR_RANGE, ERR_SIM = (
    -1, -2, -3, -4, -5, -6, -7)

FAMILY_CODE = {"full": 0, "pruned": 1}
OBJECTIVE_CODE = {"minimize": 0, "maximize": 1}


class NativeError(RuntimeError):
    """A CUDA / device failure inside libremat_b200.so."""


class Stats(C.Structure):
    _fields_ = [(k, C.c_int64) for k in
                ("states_visited", "table_entries", "transitions", "dominated_skipped")]


class PlanInfo(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("k", C.c_int32), ("budget", C.c_int64),
        ("objective_value", C.c_int64), ("peak_memory", C.c_int64), ("overhead", C.c_int64),
        ("cached_total", C.c_int64), ("stats", Stats),
    ]


class SimInfo(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("err_code", C.c_int32), ("err_index", C.c_int64),
        ("err_v", C.c_int32), ("err_w", C.c_int32),
        ("peak_live_memory", C.c_int64), ("total_forward_cost", C.c_int64),
        ("recompute_cost", C.c_int64), ("backward_count", C.c_int64),
    ]


class Timings(C.Structure):
    _fields_ = [
        ("enumerate_ms", C.c_float), ("precompute_ms", C.c_float), ("relax_ms", C.c_float),
        ("finish_ms", C.c_float), ("total_ms", C.c_float),
        ("relax_launches", C.c_int64), ("kernel_launches", C.c_int64),
        ("comparable_pairs", C.c_int64),
    ]


_lib = None
_lock = threading.Lock()

_P = C.c_void_p
_I32, _I64 = C.c_int32, C.c_int64


def lib():
    """Load the library (once).  Raises ImportError if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: the CUDA extension must be built "
                "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
        L = C.CDLL(str(LIB_PATH))
        L.remat_last_error.restype = C.c_char_p
        L.remat_kernel_launch_count.restype = C.c_int64
        sigs = {
            "remat_abi_version": [],
            "remat_device_count": [C.POINTER(_I32)],
            "remat_graph_create": [_I32, _I32, _P, _P, _P, _P, C.POINTER(_P)],
            "remat_graph_free": [_P],
            "remat_graph_stream": [_P, C.POINTER(_P)],
            "remat_family_create": [_P, _I32, _I64, C.POINTER(_P)],
            "remat_family_size": [_P, C.POINTER(_I64)],
            "remat_family_masks": [_P, _I64, _I64, _P],
            "remat_family_free": [_P],
            "remat_family_timings": [_P, C.POINTER(Timings)],
            "remat_family_member_stats": [_P, _I32, _I64, _I64, _P, _P, _P, _P],
            "remat_solve": [_P, _P, _I32, _I32, _P, _P, _P, _P],
            "remat_min_feasible_budget": [_P, _I32, _I32, C.POINTER(_I64), C.POINTER(PlanInfo),
                                          _P, _P, _P, C.POINTER(_I64), C.POINTER(_I64)],
            "remat_evaluate": [_P, _I32, _P, C.POINTER(_I64), _P, C.POINTER(_I64),
                               C.POINTER(_I64), _P],
            "remat_simulate": [_P, _I32, _P, _P, _P, _P],
            "remat_schedule_build": [_P, _I32, _P, _P, _P, _P, _I32, _I64, _P, _P, _P, _P, _P],
            "remat_schedule_vanilla": [_P, _I32, _I64, C.POINTER(_I64), _P, _P, _P],
            "remat_schedule_streams": [_P, _I32, _P, _P, _P, _I32, _I64, _P, _P, _P, _P],
            "remat_comm_unique_id": [_P],
            "remat_comm_create": [_P, _I32, _I32, _I32, C.POINTER(_P)],
            "remat_comm_free": [_P],
            "remat_level_partition": [_I64, _I64, _I32, _I32, C.POINTER(_I64), C.POINTER(_I64)],
            "remat_solve_level_sharded": [_P, _P, _P, _I32, _I32, _P, _P, _P, _P],
            "remat_solve_level_sharded_loopback": [_P, _I32, _P, _I32, _I32, _P, _P, _P, _P],
        }
        for name, args in sigs.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        _lib = L
        return _lib


def exported_symbols() -> list[str]:
    return [
        "remat_abi_version", "remat_last_error", "remat_device_count",
        "remat_kernel_launch_count", "remat_graph_create", "remat_graph_free",
        "remat_graph_stream", "remat_family_create", "remat_family_size",
        "remat_family_masks", "remat_family_free", "remat_family_timings",
        "remat_family_member_stats", "remat_solve",
        "remat_min_feasible_budget", "remat_evaluate", "remat_simulate",
        "remat_schedule_build", "remat_schedule_vanilla", "remat_schedule_streams",
        "remat_comm_unique_id", "remat_comm_create", "remat_comm_free", "remat_level_partition",
        "remat_solve_level_sharded", "remat_solve_level_sharded_loopback",
    ]


def check(rc: int, cap: int | None = None) -> int:
    if rc >= 0:
        return rc
    msg = (lib().remat_last_error() or b"").decode()
    if rc == ERR_LATTICE:
        from .lattice import LatticeTooLargeError

        raise LatticeTooLargeError(cap if cap is not None else -1)
    if rc == ERR_VALUE:
        raise ValueError(msg)
    if rc == ERR_RANGE:
        raise GraphError(msg)
    if rc == ERR_NOMEM:
        raise MemoryError(msg)
    if rc == ERR_INTERNAL:
        if "self-check" in msg:  # the reference's own asserts (planner.py:206-210)
            raise AssertionError(msg)
        from .planner import PlannerError

        raise PlannerError(msg)
    raise NativeError(msg or f"libremat_b200 error {rc}")


def device_count() -> int:
    c = _I32(0)
    rc = lib().remat_device_count(C.byref(c))
    if rc < 0:
        return 0
    return c.value


def kernel_launches() -> int:
    return int(lib().remat_kernel_launch_count())


def default_device() -> int:
    env = os.environ.get("REMAT_DEVICE")
    if env is not None:
        return int(env)
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:
        pass
    return 0


def _live(h, what: str):
    if h is None:
        raise ValueError(f"{what} is closed")
    return h


class DeviceGraph:
    """A graph resident on one GPU (owns a ``remat_graph_t``).  Calls on one
    handle are serialised (its stream and scratch buffers are shared)."""

    def __init__(self, g, device: int | None = None):
        packed = getattr(g, "packed", None)
        n, w, preds, succs, tcost, mcost = packed if packed is not None else pack_graph(g)
        self.lock = threading.Lock()
        self.graph = g
        self.n, self.w = n, w
        self.device = default_device() if device is None else device
        h = _P()
        check(lib().remat_graph_create(self.device, n, preds.ctypes.data, succs.ctypes.data,
                                       tcost.ctypes.data, mcost.ctypes.data, C.byref(h)))
        self.handle = h

    def stream(self) -> int:
        s = _P()
        check(lib().remat_graph_stream(_live(self.handle, "graph handle"), C.byref(s)))
        return s.value or 0

    def close(self):
        if getattr(self, "handle", None):
            lib().remat_graph_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- evaluation / simulation -------------------------------------------------

    def evaluate(self, chain: list[int]):
        k = len(chain)
        buf = masks_to_array(chain, self.w) if k else np.zeros((1, self.w), dtype=np.uint64)
        stage = np.zeros(max(k, 1), dtype=np.int64)
        cached = np.zeros((max(k, 1), self.w), dtype=np.uint64)
        ovh, peak, ctot = _I64(), _I64(), _I64()
        with self.lock:
            check(lib().remat_evaluate(_live(self.handle, "graph handle"), k, buf.ctypes.data,
                                       C.byref(ovh), stage.ctypes.data, C.byref(peak),
                                       C.byref(ctot), cached.ctypes.data))
        return ovh.value, [int(x) for x in stage[:k]], peak.value, ctot.value, \
            array_to_masks(cached[:k])

    # -- K7 schedules (csrc/schedule.cu) -----------------------------------------

    def simulate(self, schedules: list[np.ndarray], want_trace: bool = True):
        offs = np.zeros(len(schedules) + 1, dtype=np.int64)
        for s, ops in enumerate(schedules):
            offs[s + 1] = offs[s] + len(ops)
        flat = np.concatenate([np.asarray(o, dtype=np.int32).reshape(-1, 2) for o in schedules]
                              + [np.zeros((1, 2), dtype=np.int32)])
        infos = (SimInfo * len(schedules))()
        trace = np.zeros(max(int(offs[-1]), 1), dtype=np.int64)
        with self.lock:
            check(lib().remat_simulate(_live(self.handle, "graph handle"), len(schedules),
                                       offs.ctypes.data, flat.ctypes.data, C.addressof(infos),
                                       trace.ctypes.data if want_trace else None))
        return infos, offs, trace

    def build(self, seqs, flags: int):
        """Canonical schedules of ``seqs`` (LowerSetSequence-like: chain,
        segments, cached), + liveness (flags & 1), + simulation (flags & 2).
        Returns (ops per plan, SimInfo per plan or [], trace per plan or [])."""
        ks = np.array([len(q.chain) for q in seqs], dtype=np.int32)
        chains = masks_to_array([m for q in seqs for m in q.chain], self.w)
        segs = masks_to_array([m for q in seqs for m in q.segments], self.w)
        cached = masks_to_array([m for q in seqs for m in q.cached], self.w)
        nb = len(seqs)
        cap = 6 * self.n * nb
        offs = np.zeros(nb + 1, dtype=np.int64)
        ops = np.zeros((max(cap, 1), 2), dtype=np.int32)
        status = np.zeros(nb, dtype=np.int32)
        infos = (SimInfo * nb)()
        trace = np.zeros(max(cap, 1), dtype=np.int64) if flags & 2 else None
        with self.lock:
            check(lib().remat_schedule_build(
                _live(self.handle, "graph handle"), nb, ks.ctypes.data, chains.ctypes.data,
                segs.ctypes.data, cached.ctypes.data, flags, cap, offs.ctypes.data,
                ops.ctypes.data, status.ctypes.data, C.addressof(infos),
                trace.ctypes.data if trace is not None else None))
        if (status != OK).any():
            # the reference's own assert (schedule.py:111)
            raise AssertionError("stage targets are not live: the sequence is inconsistent")
        outs = [ops[offs[b]:offs[b + 1]] for b in range(nb)]
        if not flags & 2:
            return outs, [], []
        return outs, list(infos), [trace[offs[b]:offs[b + 1]] for b in range(nb)]

    def vanilla(self, flags: int):
        cap = 6 * self.n
        ops = np.zeros((cap, 2), dtype=np.int32)
        nops = _I64()
        info = SimInfo()
        trace = np.zeros(cap, dtype=np.int64) if flags & 2 else None
        with self.lock:
            check(lib().remat_schedule_vanilla(
                _live(self.handle, "graph handle"), flags, cap, C.byref(nops), ops.ctypes.data,
                C.byref(info), trace.ctypes.data if trace is not None else None))
        m = nops.value
        return ops[:m], info, (trace[:m] if trace is not None else None)

    def streams(self, schedules: list[np.ndarray], events: list[int], flags: int):
        """liveness (flags & 1) and/or simulate (flags & 2) of encoded streams.
        Returns (liveness outputs or [], SimInfo per stream or [], traces or [])."""
        ns = len(schedules)
        offs = np.zeros(ns + 1, dtype=np.int64)
        for s, o in enumerate(schedules):
            offs[s + 1] = offs[s] + len(o)
        flat = np.concatenate([np.asarray(o, dtype=np.int32).reshape(-1, 2) for o in schedules]
                              + [np.zeros((1, 2), dtype=np.int32)])
        ev = np.asarray(events, dtype=np.int64)
        cap = 2 * int(offs[-1]) + 1
        out_offs = np.zeros(ns + 1, dtype=np.int64)
        out = np.zeros((cap, 2), dtype=np.int32)
        infos = (SimInfo * ns)()
        trace = np.zeros(cap, dtype=np.int64) if flags & 2 else None
        with self.lock:
            check(lib().remat_schedule_streams(
                _live(self.handle, "graph handle"), ns, offs.ctypes.data, flat.ctypes.data,
                ev.ctypes.data, flags, cap, out_offs.ctypes.data, out.ctypes.data,
                C.addressof(infos), trace.ctypes.data if trace is not None else None))
        o = out_offs if flags & 1 else offs
        outs = [out[out_offs[s]:out_offs[s + 1]] for s in range(ns)] if flags & 1 else []
        if not flags & 2:
            return outs, [], []
        return outs, list(infos), [trace[o[s]:o[s + 1]] for s in range(ns)]


class Comm:
    """An NCCL communicator inside libremat_b200 (level sharding)."""

    ID_BYTES = 128

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * Comm.ID_BYTES)()
        check(lib().remat_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, uid: bytes, world: int, rank: int, device: int):
        buf = (C.c_uint8 * Comm.ID_BYTES).from_buffer_copy(uid)
        h = _P()
        check(lib().remat_comm_create(buf, world, rank, device, C.byref(h)))
        self.handle, self.world, self.rank, self.device = h, world, rank, device

    def close(self):
        if getattr(self, "handle", None):
            lib().remat_comm_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def level_partition(level_start: int, width: int, world: int, rank: int) -> tuple[int, int]:
    """Targets [begin, end) of a level owned by ``rank`` (host-only)."""
    a, b = _I64(), _I64()
    check(lib().remat_level_partition(level_start, width, world, rank, C.byref(a), C.byref(b)))
    return a.value, b.value


def solve_loopback(fams: list["DeviceFamily"], budgets: list[int], objective: str):
    """Level-sharded solve with ``len(fams)`` replicas on one device."""
    arr = (_P * len(fams))(*[f.handle for f in fams])
    f0 = fams[0]
    return f0._solve_with(
        lambda *a: lib().remat_solve_level_sharded_loopback(arr, len(fams), *a), budgets,
        objective)


def words_to_int(row) -> int:
    out = 0
    for k, x in enumerate(row):
        out |= int(x) << (64 * k)
    return out


class DeviceFamily:
    """A lower-set family + per-member precompute resident on the GPU."""

    def __init__(self, dg: DeviceGraph, family: str, cap: int):
        self.dg = dg
        self.family = family
        self.cap = cap
        h = _P()
        check(lib().remat_family_create(_live(dg.handle, "graph handle"), FAMILY_CODE[family],
                                        int(cap), C.byref(h)), cap=cap)
        self.handle = h
        sz = _I64()
        check(lib().remat_family_size(h, C.byref(sz)))
        self.size = sz.value

    def close(self):
        if getattr(self, "handle", None):
            lib().remat_family_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def masks(self, start: int = 0, count: int | None = None) -> list[int]:
        if count is None:
            count = self.size - start
        buf = np.zeros((max(count, 1), self.dg.w), dtype=np.uint64)
        check(lib().remat_family_masks(_live(self.handle, "family handle"), start, count,
                                       buf.ctypes.data))
        return array_to_masks(buf[:count])

    def member_stats(self, b: int = 0) -> dict:
        """Per-member |frontier| and |cell| of the last solve's budget ``b``,
        plus transitions and comparable-pair counts accumulated per relaxation
        tile on the tile's first target (sums over whole levels are exact;
        numpy arrays of length F)."""
        F = self.size
        out = {"flen": np.zeros(F, np.int32), "cells": np.zeros(F, np.int32),
               "trans": np.zeros(F, np.uint64), "pairs": np.zeros(F, np.uint64)}
        check(lib().remat_family_member_stats(
            _live(self.handle, "family handle"), b, 0, F, out["flen"].ctypes.data,
            out["cells"].ctypes.data, out["trans"].ctypes.data, out["pairs"].ctypes.data))
        return out

    def timings(self) -> dict:
        t = Timings()
        check(lib().remat_family_timings(_live(self.handle, "family handle"), C.byref(t)))
        return {k: getattr(t, k) for k, _ in Timings._fields_}

    def _alloc(self, nb: int):
        rows = self.dg.n + 1
        return (np.zeros((nb, rows, self.dg.w), dtype=np.uint64),
                np.zeros((nb, rows, self.dg.w), dtype=np.uint64),
                np.zeros((nb, rows), dtype=np.int64))

    MAX_BATCH = 256  # budgets per device solve (DP tables scale with the batch)

    def solve(self, budgets: list[int], objective: str):
        """Batched dp over ``budgets``: list of (PlanInfo, chain, cached, stages)."""
        if not budgets:
            return []
        if len(budgets) > self.MAX_BATCH:
            out = []
            for k in range(0, len(budgets), self.MAX_BATCH):
                out += self.solve(budgets[k:k + self.MAX_BATCH], objective)
            return out
        nb = len(budgets)
        b = np.asarray([min(int(x), 2**62) for x in budgets], dtype=np.int64)
        infos = (PlanInfo * nb)()
        chain, cached, stage = self._alloc(nb)
        check(lib().remat_solve(_live(self.handle, "family handle"), b.ctypes.data, nb,
                                OBJECTIVE_CODE[objective],
                                C.addressof(infos), chain.ctypes.data, cached.ctypes.data,
                                stage.ctypes.data))
        return [self._unpack(infos[i], chain[i], cached[i], stage[i]) for i in range(nb)]

    def _solve_with(self, fn, budgets: list[int], objective: str):
        nb = len(budgets)
        b = np.asarray([min(int(x), 2**62) for x in budgets], dtype=np.int64)
        infos = (PlanInfo * nb)()
        chain, cached, stage = self._alloc(nb)
        check(fn(b.ctypes.data, nb, OBJECTIVE_CODE[objective], C.addressof(infos),
                 chain.ctypes.data, cached.ctypes.data, stage.ctypes.data))
        return [self._unpack(infos[i], chain[i], cached[i], stage[i]) for i in range(nb)]

    def solve_level_sharded(self, comm: "Comm", budgets: list[int], objective: str):
        """``solve`` with every level's targets split over the communicator's ranks."""
        return self._solve_with(
            lambda *a: lib().remat_solve_level_sharded(_live(self.handle, "family handle"),
                                                       _live(comm.handle, "communicator"), *a),
            budgets, objective)

    def min_feasible_budget(self, objective: str, probes_per_round: int = 8):
        info = PlanInfo()
        chain, cached, stage = self._alloc(1)
        bmin, probes, ptrans = _I64(), _I64(), _I64()
        check(lib().remat_min_feasible_budget(_live(self.handle, "family handle"),
                                              OBJECTIVE_CODE[objective],
                                              probes_per_round, C.byref(bmin), C.byref(info),
                                              chain.ctypes.data, cached.ctypes.data,
                                              stage.ctypes.data, C.byref(probes),
                                              C.byref(ptrans)))
        return bmin.value, self._unpack(info, chain[0], cached[0], stage[0]), {
            "probes": probes.value, "probe_transitions": ptrans.value}

    @staticmethod
    def _unpack(info, chain, cached, stage):
        k = info.k if info.status == OK else 0
        return (info, array_to_masks(chain[:k]), array_to_masks(cached[:k]),
                [int(x) for x in stage[:k]])
