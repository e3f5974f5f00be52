"""Per-source-line profile of one kernel: align an ncu SASS source-page export
(Address/Source/Instructions Executed/Warp Stall Sampling columns) with the
nvdisasm -g listing of the same cubin (same instruction order), and sum the
executed instructions and stall samples per CUDA source line.

  python tools/sass_lines.py <ncu_sass.csv> <nvdisasm -g listing> <function substring> [min%]"""
import collections
import csv
import re
import sys

csvf, lst, fn = sys.argv[1:4]
thr = float(sys.argv[4]) if len(sys.argv) > 4 else 0.3
lines = open(lst).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith("//---") and fn in l)
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith("//---")), len(lines))
cur, instr = None, []
for l in lines[start:end]:
    m = re.search(r'//## File ".*/(\S+)", line (\d+)', l)
    if m:
        cur = (m.group(1), int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        instr.append(cur)
rows = list(csv.reader(open(csvf)))
h, data = rows[1], rows[2:]
iE, iW = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
assert len(instr) == len(data), (len(instr), len(data))
agg, st = collections.Counter(), collections.Counter()
for c, r in zip(instr, data):
    agg[c] += float(r[iE] or 0)
    st[c] += float(r[iW] or 0)
tot, tw = sum(agg.values()), sum(st.values())
srcs = {}
for c in sorted(k for k in agg if k):
    if agg[c] / tot * 100 < thr and st[c] / tw * 100 < thr:
        continue
    f, ln = c
    if f not in srcs:
        try:
            srcs[f] = open(f"paper_1905_11722_b200/csrc/{f}").read().split("\n")
        except OSError:
            srcs[f] = []
    text = srcs[f][ln - 1].strip()[:80] if ln - 1 < len(srcs[f]) else ""
    print(f"{f}:{ln:5d} inst {agg[c] / tot * 100:5.1f}%  stall {st[c] / tw * 100:5.1f}%  {text}")
