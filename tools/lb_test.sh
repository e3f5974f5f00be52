cd $GRAFT_REPO_ROOT
for LB in 3 4; do
  sed -i "s/__launch_bounds__(kThreads, [0-9])\n    k_relax_tile/X/" paper_1905_11722_b200/csrc/relax.cu
  python - <<PY
import re
p='paper_1905_11722_b200/csrc/relax.cu'
s=open(p).read()
s=re.sub(r'__launch_bounds__\(kThreads, \d\)\n    k_relax_tile', '__launch_bounds__(kThreads, $LB)\n    k_relax_tile', s)
open(p,'w').write(s)
PY
  make -s -j16 -C paper_1905_11722_b200/csrc > /dev/null 2>&1
  echo "LB=$LB"
  timeout 300 python bench.py --no-cpu --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('unet', d['ms_per_step'], d['config']['phase_ms'])"
  timeout 300 python bench.py --no-cpu --steps 10 --workload random-dag --edge-prob 0.3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', d['ms_per_step'], d['config']['phase_ms'])"
  timeout 300 python bench.py --no-cpu --steps 3 --workload random-dag --edge-prob 0.2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5p02', d['ms_per_step'], d['config']['phase_ms'])"
done
