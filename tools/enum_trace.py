"""Per-level phase times of the enumeration kernel (K1) on the C5 lattices:
scatter / emit / rank per level (slowest block) and the barrier gap, from
globaltimer stamps of a REMAT_ENUM_TRACE build:

  make -C paper_1905_11722_b200/csrc OUT=$PWD/build_trace/libremat_b200.so \
       OBJDIR=/tmp/obj_trace EXTRA=-DREMAT_ENUM_TRACE
  python tools/enum_trace.py"""
import ctypes as C, os, sys, json
import numpy as np
sys.path.insert(0, "/root/repo")
os.environ["REMAT_B200_LIB"] = "/root/repo/build_trace/libremat_b200.so"
from paper_1905_11722_b200 import named_graph
from paper_1905_11722_b200._native import DeviceFamily, DeviceGraph, lib
for p in (0.2, 0.3):
    g = named_graph("random-dag", depth=516, edge_prob=p, seed=0)
    dg = DeviceGraph(g)
    f = DeviceFamily(dg, "full", 2_000_000)
    f = DeviceFamily(dg, "full", 2_000_000)
    buf = np.zeros(600 * 148 * 4, dtype=np.uint64)
    L = C.CDLL(os.environ["REMAT_B200_LIB"])
    assert L.remat_debug_enum_trace(buf.ctypes.data_as(C.c_void_p)) == 0
    t = buf.reshape(600, 148, 4).astype(np.int64)
    lv = [k for k in range(600) if t[k, :, 0].max() > 0]
    t0 = t[lv[0], :, 0].min()
    res = []
    for k in lv:
        a = t[k]
        start = a[:, 0].min()
        # phase durations on the slowest block, and the level's span
        scat = (a[:, 1] - a[:, 0]).max() / 1e3
        emit = (a[:, 2] - a[:, 1]).max() / 1e3
        rank = (a[:, 3] - a[:, 2]).max() / 1e3
        done = a[:, 3].max()
        nxt = t[k + 1, :, 0].min() if (k + 1) in lv else done
        res.append((k, scat, emit, rank, (done - start) / 1e3, (nxt - done) / 1e3))
    arr = np.array([r[1:] for r in res])
    print(p, "levels", len(res), "sum us: scatter %.0f emit %.0f rank %.0f level-span %.0f barrier-gap %.0f" % tuple(arr.sum(0)))
    for r in res[::60]: print("  k=%d scat %.1f emit %.1f rank %.1f span %.1f gap %.1f" % r)
    f.close(); dg.close()
