"""Group an ncu SASS source-page export into straight-line blocks with their
share of executed instructions and stall samples (reads /tmp/sass.csv)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "/tmp/sass.csv")))
h = rows[1]
data = rows[2:]
iA, iS, iW, iE = (h.index("Address"), h.index("Source"),
                  h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"))
tot_e = sum(float(r[iE] or 0) for r in data)
tot_w = sum(float(r[iW] or 0) for r in data)
print("total inst", tot_e, "samples", tot_w)
blocks, cur = [], None
for r in data:
    e = float(r[iE] or 0)
    w = float(r[iW] or 0)
    if cur is None or abs(e - cur["e0"]) > 0.2 * max(cur["e0"], 1):
        cur = {"start": r[iA][-5:], "e0": e, "n": 0, "E": 0, "W": 0, "ops": []}
        blocks.append(cur)
    cur["n"] += 1
    cur["E"] += e
    cur["W"] += w
    cur["ops"].append(r[iS].strip()[:40])
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
for b in blocks:
    if b["E"] / tot_e > thr or b["W"] / tot_w > thr:
        print(f"{b['start']} n={b['n']:4d} inst={b['E'] / tot_e * 100:5.1f}% "
              f"stall={b['W'] / tot_w * 100:5.1f}%  per-exec={b['e0']:.0f}  {b['ops'][0]} | {b['ops'][-1]}")
