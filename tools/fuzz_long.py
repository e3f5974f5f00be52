"""Long differential fuzz run (seeds beyond the test suite's): python tools/fuzz_long.py A B"""
import importlib.util
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
spec = importlib.util.spec_from_file_location("fz", ROOT / "tests" / "test_gpu_fuzz.py")
m = importlib.util.module_from_spec(spec)
spec.loader.exec_module(m)
a, b = int(sys.argv[1]), int(sys.argv[2])
t0 = time.time()
for seed in range(a, b):
    m.test_fuzz_against_oracle(seed)
    if seed % 50 == 0:
        print("seed", seed, "ok", round(time.time() - t0, 1), flush=True)
for seed in range(a, a + (b - a) // 4):
    m.test_fuzz_level_sharding_loopback_against_oracle(seed)
print("all ok", b - a, "seeds", round(time.time() - t0, 1))
# wide bitsets (tests/test_gpu_wide.py) and the one-CTA-per-budget minimize
# solver, seeds beyond the suite's: FUZZ_WIDE=<count>
import os  # noqa: E402

nw = int(os.environ.get("FUZZ_WIDE", "0"))
if nw:
    spec2 = importlib.util.spec_from_file_location("wd", ROOT / "tests" / "test_gpu_wide.py")
    wd = importlib.util.module_from_spec(spec2)
    spec2.loader.exec_module(wd)
    for seed in range(a, a + nw):
        wd.test_wide_dense_dags_against_oracle(seed)
        m.test_fuzz_one_cta_per_budget_minimize(seed)
    print("wide + one-CTA minimize ok", nw, "seeds", round(time.time() - t0, 1))
