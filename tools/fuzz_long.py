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
