"""bench.py's output contract: the reference arm on CPU (single process and
under torchrun with 2 gloo ranks: rank 0 alone prints), and our arm's JSON
line on the GPU."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _lines(out: str) -> list[dict]:
    return [json.loads(x) for x in out.splitlines() if x.startswith("{")]


def _env():
    env = dict(os.environ)
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    return env


def test_reference_arm_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--skip-len", "3",
                        "--steps", "1", "--warmup", "1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600, env=_env())
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = _lines(r.stdout)
    assert BASE_KEYS <= set(line)
    assert line["impl"] == "reference"
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["value"] == line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["config"]["transitions_per_step"] > 0
    py = line["cpu_baseline"]["python_reference"]
    if (ROOT / "oracle" / "_ref" / "remat").is_dir():
        assert py["kind"] == "reference" and py["cores"] == 1 and py["value"] > 0


def test_reference_arm_under_torchrun_prints_once():
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(_free_port()), "bench.py", "--gpus", "2", "--impl", "reference",
                        "--skip-len", "3", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600, env=_env())
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = _lines(r.stdout)
    assert line["impl"] == "reference" and line["n_gpus"] == 2


@pytest.mark.gpu
def test_our_arm_line():
    r = subprocess.run([sys.executable, "bench.py", "--skip-len", "3", "--steps", "3",
                        "--warmup", "3", "--no-cpu", "--no-configs"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600, env=_env())
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = _lines(r.stdout)
    assert BASE_KEYS <= set(line)
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["gpu_launches"] > 0
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(line["roofline"])
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(line["clocks"])


@pytest.mark.gpu
def test_our_arm_configs_are_timed_and_bit_exact():
    """Every BASELINE config rides in the bench line, each checked against its
    committed golden (reference or pinned-oracle outputs)."""
    r = subprocess.run([sys.executable, "bench.py", "--skip-len", "3", "--steps", "1",
                        "--warmup", "3", "--no-cpu"], cwd=ROOT, capture_output=True, text=True,
                       timeout=900, env=_env())
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = _lines(r.stdout)
    cfgs = line["configs"]
    assert len(cfgs) >= 8
    for c in cfgs:
        assert "error" not in c, c
        assert not c["parity"].startswith("MISMATCH"), c
    c5 = cfgs[0]
    assert "p=0.2" in c5["config"] and c5["transitions"] > 10**10
    assert c5["roofline"]["frac"] > 0
