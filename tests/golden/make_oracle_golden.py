"""Golden fixtures for instances the Python reference cannot solve in a
practical time, made by the PINNED C oracle (oracle/remat_oracle.c).

The oracle restates the reference solver (planner.py / lattice.py /
strategy.py) and is itself checked against the reference's own outputs on
every fixture in this directory (tests/test_oracle.py).  The north-star
"largest graph" — C5, ``TopologySpec("random-dag", 516, seed=0,
edge_prob=0.2)`` (reference benchmarks.py:90-99; F = 199,048 lower sets,
1.9·10¹⁰ transitions per solve) — would take the Python reference weeks
(SURVEY §6), so its golden comes from the oracle:

    python tests/golden/make_oracle_golden.py [--threads T] [--only NAME]

Writes tests/golden/oracle_large.json (the graph document + the oracle's
``dp_plan`` at 2·M(V), the binary-search ``min_feasible_budget`` and the
memory-centric plan at B_min).  Several minutes per solve on 8 host threads.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REPO))

from oracle import oracle as orc  # noqa: E402  (test infrastructure)
from paper_1905_11722_b200 import named_graph  # noqa: E402
from paper_1905_11722_b200.graph import graph_to_document  # noqa: E402

OUT = Path(__file__).resolve().parent / "oracle_large.json"

CASES = {
    # name: (named_graph kwargs, runs)
    "c5_p02": ({"name": "random-dag", "depth": 516, "edge_prob": 0.2, "seed": 0},
               ("dp_2mv", "mfb_min", "dp_max_bmin")),
    "c5_p03": ({"name": "random-dag", "depth": 516, "edge_prob": 0.3, "seed": 0},
               ("dp_2mv", "mfb_min")),
    # the bench headline (BASELINE configs[1]): U-Net skip 8, exact, B = 2·M(V)
    "unet_c8": ({"name": "unet", "skip_len": 8}, ("dp_2mv",)),
    # C4 (BASELINE configs[3]) on the FULL family: the 64-budget PSPNet sweep
    # (budgets of bench_configs.json, whose pruned-family plans are reference
    # outputs); 1.5e11 transitions in all
    "pspnet_full_sweep": ({"name": "pspnet"}, ("dp_sweep",)),
}


def hexed(plan: dict) -> dict:
    out = dict(plan)
    if plan.get("feasible"):
        out["chain"] = [format(m, "x") for m in plan["chain"]]
    out.pop("probes", None)
    out.pop("probe_transitions", None)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=None)
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    data = json.loads(OUT.read_text())["data"] if OUT.exists() else []
    done = {r["name"] for r in data}
    for name, (kw, runs) in CASES.items():
        if args.only and name != args.only:
            continue
        if name in done and not args.only:
            continue
        kw = dict(kw)
        g = named_graph(kw.pop("name"), **kw)
        p = orc.Packed(g)
        rec = {"name": name, "kw": CASES[name][0], "graph": graph_to_document(g), "runs": []}
        b_min = None
        for run in runs:
            t0 = time.time()
            if run == "dp_2mv":
                plan = orc.dp_plan(p, 2 * g.total_memory, "full", "minimize", nthreads=args.threads)
                rec["runs"].append({"kind": "dp", "plan": hexed(plan)})
            elif run == "mfb_min":
                b_min, plan = orc.min_feasible_budget(p, "full", "minimize", nthreads=args.threads)
                rec["runs"].append({"kind": "mfb", "family": "full", "objective": "minimize",
                                    "b_min": b_min, "plan": hexed(plan),
                                    "probes": plan["probes"]})
            elif run == "dp_sweep":
                sweep = json.loads((OUT.parent / "bench_configs.json").read_text())["data"]
                budgets = next(r for r in sweep if r["name"] == "pspnet_sweep")["budgets"]
                for b in budgets:
                    plan = orc.dp_plan(p, b, "full", "minimize", nthreads=args.threads)
                    rec["runs"].append({"kind": "dp", "plan": hexed(plan)})
            elif run == "dp_max_bmin":
                # memory_centric_plan (planner.py:300-313) = the maximize DP at B_min
                plan = orc.dp_plan(p, b_min, "full", "maximize", nthreads=args.threads)
                rec["runs"].append({"kind": "dp", "plan": hexed(plan)})
            print(f"{name} {run}: {time.time() - t0:.1f} s", flush=True)
        data = [r for r in data if r["name"] != name] + [rec]
        OUT.write_text(json.dumps({
            "generator": "tests/golden/make_oracle_golden.py",
            "pinned_by": "oracle/remat_oracle.c, checked against the reference goldens "
                         "(tests/test_oracle.py)",
            "data": data}, separators=(",", ":")))


if __name__ == "__main__":
    main()
