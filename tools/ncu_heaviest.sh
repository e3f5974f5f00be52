#!/bin/bash
# ncu: launch list of the relax kernels of one solve, then a --set full
# capture of the heaviest launch of kernel $1.  Extra args go to solve_once.py.
mkdir -p gpurun_out
K=${1:-k_relax_pm}; TAG=${2:-pm}; shift 2
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ --csv \
  --log-file gpurun_out/launches_$TAG.csv python tools/solve_once.py "$@" > /dev/null 2>&1
IDX=$(python - "$K" gpurun_out/launches_$TAG.csv <<'PY'
import csv, sys
k, path = sys.argv[1], sys.argv[2]
rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))]
seen, best, bi = {}, -1, 0
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum": continue
    name = r["Kernel Name"]
    if k not in name: continue
    idx = int(r["ID"])
    v = float(r["Metric Value"].replace(",", ""))
    if v > best: best, bi = v, idx
kidx = sorted({int(r["ID"]) for r in rows if k in r["Kernel Name"]}).index(bi)
print(kidx)
PY
)
echo "heaviest $K launch index $IDX"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $IDX -c 1 -o gpurun_out/prof_$TAG -f python tools/solve_once.py "$@" > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
