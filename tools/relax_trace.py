"""Per-level times of the cooperative multi-level relaxation (k_relax_levels)
on C5 p=0.4 (one such launch per solve): per level, the span of the slowest
block's virtual CTAs and the barrier gap, from globaltimer stamps of a
REMAT_RELAX_TRACE build (W=9 instantiation):

  make -C paper_1905_11722_b200/csrc OUT=$PWD/build_rt/libremat_b200.so \\
       OBJDIR=/tmp/obj_rt EXTRA=-DREMAT_RELAX_TRACE
  python tools/relax_trace.py"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
os.environ.setdefault("REMAT_B200_LIB", "/root/repo/build_rt/libremat_b200.so")
from paper_1905_11722_b200 import Solver, named_graph  # noqa: E402

p = float(sys.argv[1]) if len(sys.argv) > 1 else 0.4
g = named_graph("random-dag", depth=516, edge_prob=p, seed=0)
s = Solver(g, "full")
s.plan(2 * g.total_memory)
s.plan(2 * g.total_memory)
print("relax_ms", s.timings()["relax_ms"], "launches", s.timings()["relax_launches"])
buf = np.zeros(600 * 296 * 4, dtype=np.uint64)
assert C.CDLL(os.environ["REMAT_B200_LIB"]).remat_debug_relax_trace(buf.ctypes.data_as(C.c_void_p)) == 0
t = buf.reshape(600, 296, 4).astype(np.int64)
lv = [l for l in range(600) if t[l, :, 0].max() > 0]
spans, gaps, imb = [], [], []
for l in lv:
    a = t[l]
    ok = a[:, 0] > 0
    start, end = a[ok, 0].min(), a[ok, 1].max()
    work = a[ok, 1] - a[ok, 0]
    spans.append((end - start) / 1e3)
    imb.append((work.max() - np.median(work)) / 1e3)
    if l + 1 in lv:
        gaps.append((t[l + 1, t[l + 1, :, 0] > 0, 0].min() - end) / 1e3)
spans, gaps, imb = map(np.array, (spans, gaps, imb))
print(f"levels {len(lv)}: level span sum {spans.sum():.0f} us (mean {spans.mean():.1f}), "
      f"barrier gap sum {gaps.sum():.0f} us (mean {gaps.mean():.1f}), "
      f"slowest-minus-median block mean {imb.mean():.1f} us")
for l in lv[::50]:
    a = t[l]
    ok = a[:, 0] > 0
    w = (a[ok, 1] - a[ok, 0]) / 1e3
    print(f"  level {l}: span {(a[ok, 1].max() - a[ok, 0].min()) / 1e3:.1f} us, block work "
          f"min {w.min():.1f} med {np.median(w):.1f} max {w.max():.1f}")
