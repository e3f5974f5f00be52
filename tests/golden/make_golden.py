"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container only (it imports the read-only reference package at
/root/reference/pkg/src; the GPU box does not have it):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--slow]

Every fixture stores the graph as the reference's own ``graph_to_document``
(index order) plus the reference's outputs for it.  Node sets are written as
hex strings.  ``--slow`` adds the named-shape cases whose reference solve takes
minutes (C3 DenseNet-161, C5 random-dag n=516 p=0.5); ``--xslow`` writes
named_xslow.json (C5 p=0.4, memory-centric U-Net; ~10 min); ``--bench`` writes
bench_configs.json (the C4 PSPNet 64-budget sweep that bench.py checks).

Fixtures (all keyed on reference call sites, file:line under pkg/src/remat):
  dp_corpus.json     dp_plan (planner.py:214) on seeded random DAGs, both
                     families and objectives, budgets across [0, 3·M(V)]
  mfb_corpus.json    min_feasible_budget (271) / memory_centric_plan (300)
  lattice.json       all_lower_sets / pruned_lower_sets (lattice.py:59, 87)
  sim_corpus.json    build_schedule / vanilla_schedule / liveness_pass /
                     simulate (schedule.py:88-254), incl. fault cases
  reports.json       build_report (report.py:82) CSV for the 6 snapshot specs
  named.json         named-shape configs (C1-C5 at reference-solvable size)
"""

from __future__ import annotations

import json
import os
import random
import sys
import time
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from remat.benchmarks import (  # noqa: E402
    TopologySpec, articulation_points, chen_baseline_plan, generate,
)
from remat.graph import graph_from_document, graph_to_document  # noqa: E402
from remat.lattice import all_lower_sets, pruned_lower_sets  # noqa: E402
from remat.planner import (  # noqa: E402
    PlanRequest, dp_plan, memory_centric_plan, min_feasible_budget,
)
from remat.report import build_report  # noqa: E402
from remat.schedule import (  # noqa: E402
    BackwardCompute, ForwardCompute, Free, SimulationError, ValueRef,
    build_schedule, liveness_pass, simulate, vanilla_schedule,
)
from remat.strategy import make_sequence  # noqa: E402

REPO = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REPO))
from paper_1905_11722_b200 import benchmarks as ours  # noqa: E402  (named-shape docs)

OUT = Path(__file__).resolve().parent


def random_graph(rng: random.Random, n: int, p: float, lo: int = 1, hi: int = 5):
    """Same construction as the reference's tests/conftest.py:36-47."""
    nodes = [
        {"id": f"r{i}", "kind": "other", "compute_cost": rng.randint(lo, hi),
         "memory_cost": rng.randint(lo, hi)}
        for i in range(n)
    ]
    edges = [[f"r{i}", f"r{j}"] for i in range(n) for j in range(i + 1, n) if rng.random() < p]
    return graph_from_document({"nodes": nodes, "edges": edges})


def hx(m: int) -> str:
    return format(m, "x")


def plan_json(plan) -> dict:
    s = plan.stats
    d = {
        "feasible": plan.feasible,
        "budget": plan.budget,
        "family": plan.family,
        "objective": plan.objective,
        "stats": {
            "states_visited": s.states_visited,
            "table_entries": s.table_entries,
            "transitions": s.transitions,
            "dominated_skipped": s.dominated_skipped,
        },
    }
    if plan.feasible:
        ev = plan.evaluation
        d.update(
            objective_value=plan.objective_value,
            chain=[hx(m) for m in plan.sequence.chain],
            segments=[hx(m) for m in plan.sequence.segments],
            cached=[hx(m) for m in plan.sequence.cached],
            overhead=ev.overhead,
            per_stage_memory=list(ev.per_stage_memory),
            peak_memory=ev.peak_memory,
            cached_total=ev.cached_total,
        )
    return d


def budgets(g, count=6):
    top = 3 * g.total_memory
    if top <= 8:
        return list(range(top + 1))
    return sorted({round(i * top / (count - 1)) for i in range(count)})


def dp_corpus():
    rng = random.Random(0xB200)
    out = []
    for gi in range(120):
        n = rng.randint(1, 9)
        g = random_graph(rng, n, rng.random(), 1, rng.choice([1, 3, 5, 10]))
        M = g.total_memory
        bs = sorted(set(budgets(g, 5)) | {2 * M, M, rng.randint(0, 2 * M)})
        cases = []
        for b in bs:
            for fam in ("full", "pruned"):
                for obj in ("minimize", "maximize"):
                    cases.append(plan_json(dp_plan(PlanRequest(g, b, fam, obj))))
        out.append({"graph": graph_to_document(g), "cases": cases})
    # conv-style costs closer to the named shapes (T in {1,10}, M powers of 2)
    for gi in range(40):
        n = rng.randint(8, 13)
        p = 0.15 + 0.45 * rng.random()
        nodes = [
            {"id": f"c{i}", "kind": "conv" if rng.random() < 0.4 else "other",
             "memory_cost": rng.choice([1, 2, 4, 8, 16])}
            for i in range(n)
        ]
        edges = [[f"c{i}", f"c{j}"] for i in range(n) for j in range(i + 1, n) if rng.random() < p]
        g = graph_from_document({"nodes": nodes, "edges": edges})
        bmin, _ = min_feasible_budget(g, "full")
        M = g.total_memory
        cases = []
        for b in sorted({bmin - 1, bmin, bmin + 1, (bmin + 2 * M) // 2, 2 * M}):
            for fam in ("full", "pruned"):
                for obj in ("minimize", "maximize"):
                    cases.append(plan_json(dp_plan(PlanRequest(g, b, fam, obj))))
        out.append({"graph": graph_to_document(g), "cases": cases})
    return out


def large_costs_corpus():
    """FLOP-valued compute costs (T_v up to 10^12, so T(V) far above 2^24:
    the solver's sparse-cell path) with byte-like memory costs; dp_plan at
    budgets around B_min and 2·M(V), both families and objectives, and the
    B_min searches (planner.py:214-223, 271-297)."""
    rng = random.Random(0xF10B5)
    out = []
    for gi in range(36):
        n = rng.randint(3, 13)
        p = 0.15 + 0.6 * rng.random()
        nodes = []
        for i in range(n):
            conv = rng.random() < 0.5
            t = rng.randint(10**9, 10**12) if conv else rng.choice([0, rng.randint(10**6, 10**9)])
            nodes.append({"id": f"f{i}", "kind": "conv" if conv else "other", "compute_cost": t,
                          "memory_cost": rng.choice([1, 2, 3, 4, 8, 16]) * rng.choice([1, 1024, 4096])})
        edges = [[f"f{i}", f"f{j}"] for i in range(n) for j in range(i + 1, n) if rng.random() < p]
        g = graph_from_document({"nodes": nodes, "edges": edges})
        M = g.total_memory
        bmin, _ = min_feasible_budget(g, "full")
        cases = []
        for b in sorted({max(0, bmin - 1), bmin, bmin + 1, (bmin + 2 * M) // 2, 2 * M}):
            for fam in ("full", "pruned"):
                for obj in ("minimize", "maximize"):
                    cases.append(plan_json(dp_plan(PlanRequest(g, b, fam, obj))))
        mfb = []
        for fam in ("full", "pruned"):
            for obj in ("minimize", "maximize"):
                b, plan = min_feasible_budget(g, fam, obj)
                mfb.append({"family": fam, "objective": obj, "b_min": b, "plan": plan_json(plan)})
        out.append({"graph": graph_to_document(g), "cases": cases, "mfb": mfb})
    # byte-valued memory so large that no 64-bit key holds (m << IB) | i:
    # M(V) ~ 2^55-2^57 on lattices of hundreds of members (small and
    # FLOP-valued compute costs)
    for gi in range(12):
        n = rng.randint(9, 13)
        p = 0.05 + 0.25 * rng.random()
        flops = gi % 2 == 1
        nodes = [{"id": f"h{i}", "kind": "other",
                  "compute_cost": rng.randint(10**9, 10**11) if flops else rng.randint(0, 10),
                  "memory_cost": rng.randint(10**15, 2 * 10**16)} for i in range(n)]
        edges = [[f"h{i}", f"h{j}"] for i in range(n) for j in range(i + 1, n) if rng.random() < p]
        g = graph_from_document({"nodes": nodes, "edges": edges})
        M = g.total_memory
        bmin, _ = min_feasible_budget(g, "full")
        cases = []
        for b in sorted({bmin, (bmin + 2 * M) // 2, 2 * M}):
            for fam in ("full", "pruned"):
                for obj in ("minimize", "maximize"):
                    cases.append(plan_json(dp_plan(PlanRequest(g, b, fam, obj))))
        out.append({"graph": graph_to_document(g), "cases": cases,
                    "mfb": [{"family": "full", "objective": "minimize", "b_min": bmin,
                             "plan": plan_json(min_feasible_budget(g, "full")[1])}]})
    # a named shape with FLOP-scale costs: the U-Net (skip 2), conv nodes
    # ~10^10-10^11 and the rest ~10^9, all distinct
    doc = ours.unet_document(2)
    for nd in doc["nodes"]:
        base = 10**10 if nd.get("kind") == "conv" else 10**9
        nd["compute_cost"] = base * rng.randint(1, 9) + rng.randint(0, 10**6)
    g = graph_from_document(doc)
    M = g.total_memory
    bmin, _ = min_feasible_budget(g, "full")
    cases = [plan_json(dp_plan(PlanRequest(g, b, fam, "minimize")))
             for b in (bmin, 2 * M) for fam in ("full", "pruned")]
    out.append({"graph": graph_to_document(g), "cases": cases,
                "mfb": [{"family": "full", "objective": "minimize", "b_min": bmin,
                         "plan": plan_json(min_feasible_budget(g, "full")[1])}]})
    return out


def mfb_corpus():
    rng = random.Random(0x5EA4C4)
    out = []
    for gi in range(60):
        g = random_graph(rng, rng.randint(1, 9), 0.2 + 0.6 * rng.random(), 1, rng.choice([1, 5, 10]))
        cases = []
        for fam in ("full", "pruned"):
            for obj in ("minimize", "maximize"):
                b, plan = min_feasible_budget(g, fam, obj)
                cases.append({"b_min": b, "plan": plan_json(plan)})
            cases.append({"memory_centric": True, "plan": plan_json(memory_centric_plan(g, fam))})
        out.append({"graph": graph_to_document(g), "cases": cases})
    return out


def lattice_corpus():
    rng = random.Random(0x1A77)
    out = []
    for gi in range(60):
        g = random_graph(rng, rng.randint(1, 11), rng.random())
        out.append({
            "graph": graph_to_document(g),
            "full": [hx(m) for m in all_lower_sets(g).masks],
            "pruned": [hx(m) for m in pruned_lower_sets(g).masks],
        })
    return out


def sched_json(sched):
    out = []
    for ins in sched:
        if isinstance(ins, ForwardCompute):
            out.append(["F", ins.node])
        elif isinstance(ins, BackwardCompute):
            out.append(["B", ins.node])
        else:
            out.append([f"FREE_{ins.ref.kind}", ins.ref.node])
    return out


def sim_json(g, sched):
    try:
        r = simulate(g, sched)
    except SimulationError as exc:
        return {"error": str(exc)}
    return {
        "peak_live_memory": r.peak_live_memory,
        "trace": list(r.trace),
        "total_forward_cost": r.total_forward_cost,
        "recompute_cost": r.recompute_cost,
        "backward_count": r.backward_count,
    }


def sim_corpus():
    rng = random.Random(0x51A1)
    out = []
    for gi in range(80):
        g = random_graph(rng, rng.randint(1, 9), 0.2 + 0.6 * rng.random())
        fam = all_lower_sets(g)
        chain, cur = [], 0
        while cur != g.full_mask:
            cur = rng.choice([m for m in fam.masks if m | cur == m and m != cur])
            chain.append(cur)
        seq = make_sequence(g, chain)
        entries = []
        for name, sched in (
            ("canonical", build_schedule(g, seq)),
            ("vanilla", vanilla_schedule(g)),
        ):
            live = liveness_pass(g, sched)
            entries.append({"kind": name, "schedule": sched_json(sched), "result": sim_json(g, sched),
                            "liveness_schedule": sched_json(live), "liveness_result": sim_json(g, live)})
        # a corrupted schedule: drop or duplicate one instruction
        sched = build_schedule(g, seq)
        bad = list(sched)
        pos = rng.randrange(len(bad))
        if rng.random() < 0.5:
            del bad[pos]
        else:
            bad.insert(pos, bad[pos])
        entries.append({"kind": "corrupted", "schedule": sched_json(bad), "result": sim_json(g, bad)})
        out.append({"graph": graph_to_document(g), "chain": [hx(m) for m in chain], "entries": entries})
    return out


SNAPSHOT_SPECS = (
    TopologySpec("chain", 12),
    TopologySpec("skip-chain", 10),
    TopologySpec("resnet-like", 3, cost_model="conv-weighted"),
    TopologySpec("densenet-like", 5, cost_model="conv-weighted"),
    TopologySpec("unet-like", 3, cost_model="conv-weighted"),
    TopologySpec("random-dag", 8, seed=7, edge_prob=0.4),
)


def reports():
    out = []
    for spec in SNAPSHOT_SPECS:
        g = generate(spec)
        entry = {"spec": {"family": spec.family, "depth": spec.depth, "seed": spec.seed,
                          "edge_prob": spec.edge_prob, "cost_model": spec.cost_model},
                 "graph": graph_to_document(g), "csv": build_report(g).to_csv(), "plans": []}
        for fam in ("full", "pruned"):
            b, tc = min_feasible_budget(g, fam, "minimize")
            mc = dp_plan(PlanRequest(g, b, fam, "maximize"))
            entry["plans"].append({"family": fam, "b_min": b, "tc": plan_json(tc), "mc": plan_json(mc)})
        chen = chen_baseline_plan(g)
        entry["chen"] = {"points": articulation_points(g), "plan": plan_json(chen),
                         "table": build_report(g).render_table()}
        out.append(entry)
    # Chen baseline on more archetype shapes (benchmarks.py:136-222)
    rng = random.Random(0xC4E)
    for fam in ("chain", "skip-chain", "resnet-like", "densenet-like", "unet-like", "random-dag"):
        for seed in range(4):
            spec = TopologySpec(fam, rng.randint(3, 60), seed=seed,
                                edge_prob=rng.choice([0.1, 0.3, 0.6]))
            g = generate(spec)
            out.append({"spec": {"family": fam, "depth": spec.depth, "seed": seed,
                                 "edge_prob": spec.edge_prob, "cost_model": spec.cost_model},
                        "graph": graph_to_document(g),
                        "chen": {"points": articulation_points(g),
                                 "plan": plan_json(chen_baseline_plan(g))}})
    return out


def vanilla_peak(g) -> int:
    return simulate(g, liveness_pass(g, vanilla_schedule(g))).peak_live_memory


def named(slow: bool):
    out = []

    def add(name, kw, g, runs):
        rec = {"name": name, "kw": kw, "graph": graph_to_document(g), "runs": []}
        for r in runs:
            t0 = time.perf_counter()
            kind = r[0]
            if kind == "dp":
                _, fam, obj, b = r
                res = {"kind": "dp", "plan": plan_json(dp_plan(PlanRequest(g, b, fam, obj)))}
            elif kind == "mfb":
                _, fam, obj = r
                b, plan = min_feasible_budget(g, fam, obj)
                res = {"kind": "mfb", "family": fam, "objective": obj, "b_min": b, "plan": plan_json(plan)}
            else:
                _, fam = r
                res = {"kind": "mc", "family": fam, "plan": plan_json(memory_centric_plan(g, fam))}
            res["ref_seconds"] = round(time.perf_counter() - t0, 3)
            rec["runs"].append(res)
            print(f"  {name} {kw} {r}: {res['ref_seconds']}s", flush=True)
        out.append(rec)

    # C1: ResNet-50, pruned, minimize, budget = floor(vanilla_peak / 2)
    g = graph_from_document(ours.resnet50_document())
    vp = vanilla_peak(g)
    add("resnet50", {"vanilla_peak": vp}, g,
        [("dp", "pruned", "minimize", vp // 2), ("mfb", "pruned", "minimize")])
    # C2: U-Net, full family, at 2M(V) and via the B_min search
    for c in (1, 2, 3):
        g = graph_from_document(ours.unet_document(c))
        runs = [("dp", "full", "minimize", 2 * g.total_memory)]
        if c <= 2 or slow:
            runs.append(("mfb", "full", "minimize"))
        runs.append(("mfb", "pruned", "minimize"))
        add("unet", {"skip_len": c}, g, runs)
    # C4: PSPNet pruned budget points
    g = graph_from_document(ours.pspnet_document())
    vp = vanilla_peak(g)
    b, _ = min_feasible_budget(g, "pruned")
    pts = sorted({b, b + (vp - b) // 3 if vp > b else b, vp if vp > b else 2 * g.total_memory})
    add("pspnet", {"vanilla_peak": vp}, g, [("dp", "pruned", "minimize", x) for x in pts])
    # C5 (small): random-dag n=64 exact, uniform costs
    g = generate(TopologySpec("random-dag", 64, seed=0, edge_prob=0.4))
    add("random-dag", {"depth": 64, "seed": 0, "edge_prob": 0.4}, g,
        [("dp", "full", "minimize", 2 * g.total_memory), ("mfb", "full", "minimize")])
    if slow:
        g = graph_from_document(ours.densenet161_document())
        add("densenet161", {}, g, [("mc", "pruned"), ("mc", "full")])
        g = generate(TopologySpec("random-dag", 516, seed=0, edge_prob=0.5))
        add("random-dag", {"depth": 516, "seed": 0, "edge_prob": 0.5}, g,
            [("dp", "full", "minimize", 2 * g.total_memory)])
    return out


def cli_corpus():
    """The reference CLI's own outputs (cli.py): plan JSON (byte-stable),
    simulate summary / trace / schedule text, report table + CSV, exit codes
    and stderr, for a handful of graphs and flag combinations."""
    import contextlib
    import io
    import tempfile

    from remat.cli import main as ref_main

    out = []
    with tempfile.TemporaryDirectory() as td:
        def run(argv):
            so, se = io.StringIO(), io.StringIO()
            with contextlib.redirect_stdout(so), contextlib.redirect_stderr(se):
                code = ref_main(argv)
            return code, so.getvalue(), se.getvalue()

        graphs = {}
        for name, gen in [("chain3", ["--family", "chain", "--depth", "3"]),
                          ("dense4", ["--family", "densenet-like", "--depth", "4"]),
                          ("skip9", ["--family", "skip-chain", "--depth", "9", "--skip", "3",
                                     "--cost-model", "conv-weighted"]),
                          ("rand8", ["--family", "random-dag", "--depth", "8", "--seed", "3",
                                     "--edge-prob", "0.4"]),
                          ("unet5", ["--family", "unet-like", "--depth", "5",
                                     "--cost-model", "conv-weighted"])]:
            path = os.path.join(td, name + ".json")
            code, _, _ = run(["gen", *gen, "--out", path])
            graphs[name] = (path, open(path).read())
            out.append({"argv": ["gen", *gen], "code": code, "files": {"out": graphs[name][1]}})
        for name, (path, text) in graphs.items():
            for algo in ("exact", "approx", "dfs", "chen"):
                for budget in ("min", "0", "7", "40"):
                    for obj in ("time", "memory"):
                        if algo == "chen" and obj == "memory":
                            continue
                        if algo == "dfs" and name in ("unet5", "dense4") and budget == "min":
                            continue
                        argv = ["plan", "--graph", "@" + name, "--budget", budget, "--algo", algo,
                                "--objective", obj]
                        code, so, se = run([a if a[0] != "@" else path for a in argv])
                        out.append({"argv": argv, "code": code, "stdout": so, "stderr": se})
            plan_path = os.path.join(td, "plan.json")
            run(["plan", "--graph", path, "--budget", "min", "--out", plan_path])
            plan_text = open(plan_path).read()
            for live in ("on", "off"):
                tr, sc = os.path.join(td, "t.json"), os.path.join(td, "s.txt")
                code, so, se = run(["simulate", "--graph", path, "--plan", plan_path,
                                    "--liveness", live, "--trace", tr, "--schedule", sc])
                out.append({"argv": ["simulate", "--graph", "@" + name, "--plan", "@plan",
                                     "--liveness", live, "--trace", "@trace", "--schedule",
                                     "@schedule"],
                            "plan": plan_text, "code": code, "stdout": so, "stderr": se,
                            "files": {"trace": open(tr).read(), "schedule": open(sc).read()}})
            csv_path = os.path.join(td, "r.csv")
            code, so, se = run(["report", "--graph", path, "--csv", csv_path])
            out.append({"argv": ["report", "--graph", "@" + name, "--csv", "@csv"], "code": code,
                        "stdout": so, "stderr": se, "files": {"csv": open(csv_path).read()}})
        for name in graphs:
            graphs[name] = graphs[name][1]
    return [{"graphs": graphs, "runs": out}]


def named_xslow():
    """Reference runs that take many minutes in the build container: C5 at
    p=0.4 (F=3,293, ~440 s of TransitionIndex) and memory-centric U-Net."""
    out = []
    g = generate(TopologySpec("random-dag", 516, seed=0, edge_prob=0.4))
    rec = {"name": "random-dag", "kw": {"depth": 516, "seed": 0, "edge_prob": 0.4},
           "graph": graph_to_document(g), "runs": []}
    t0 = time.perf_counter()
    b = 2 * g.total_memory
    rec["runs"].append({"kind": "dp", "plan": plan_json(dp_plan(PlanRequest(g, b, "full"))),
                        "ref_seconds": round(time.perf_counter() - t0, 3)})
    print(f"  C5 p=0.4: {rec['runs'][-1]['ref_seconds']}s", flush=True)
    out.append(rec)
    g = graph_from_document(ours.unet_document(2))
    rec = {"name": "unet", "kw": {"skip_len": 2}, "graph": graph_to_document(g), "runs": []}
    t0 = time.perf_counter()
    rec["runs"].append({"kind": "mc", "family": "full",
                        "plan": plan_json(memory_centric_plan(g, "full")),
                        "ref_seconds": round(time.perf_counter() - t0, 3)})
    out.append(rec)
    return out


def bench_configs():
    """Reference outputs for the bench.py workloads the reference finishes:
    C4 — PSPNet, pruned family, the 64-budget sweep B_k = B_min +
    ⌊k·(V_peak − B_min)/63⌋, each budget one dp_plan."""
    out = []
    g = graph_from_document(ours.pspnet_document())
    vp = vanilla_peak(g)
    b_min, _ = min_feasible_budget(g, "pruned")
    top = vp if vp > b_min else 2 * g.total_memory
    budgets = [b_min + (k * (top - b_min)) // 63 for k in range(64)]
    rec = {"name": "pspnet_sweep", "kw": {"vanilla_peak": vp, "b_min": b_min},
           "graph": graph_to_document(g), "budgets": budgets, "runs": []}
    t0 = time.perf_counter()
    for b in budgets:
        rec["runs"].append({"kind": "dp", "plan": plan_json(dp_plan(PlanRequest(g, b, "pruned")))})
    rec["ref_seconds"] = round(time.perf_counter() - t0, 3)
    print(f"  C4 sweep: {rec['ref_seconds']}s", flush=True)
    out.append(rec)
    return out


def loader_corpus():
    """graph_from_document (graph.py:185-262) on shuffled documents — node and
    edge order permuted, input nodes, duplicate edges, default costs — and on
    malformed documents: the reference's index order or its error message."""
    from remat.graph import GraphError

    rng = random.Random(0x10AD)
    out = []
    for trial in range(300):
        n = rng.randint(1, 24)
        nodes = []
        for i in range(n):
            e = {"id": f"n{i}", "memory_cost": rng.randint(1, 9)}
            if rng.random() < 0.5:
                e["compute_cost"] = rng.randint(0, 12)
            if rng.random() < 0.3:
                e["kind"] = rng.choice(["conv", "relu", "add"])
            if rng.random() < 0.12:
                e["is_input"] = True
            nodes.append(e)
        p = rng.choice([0.1, 0.3, 0.6])
        edges = [[f"n{i}", f"n{j}"] for i in range(n) for j in range(i + 1, n) if rng.random() < p]
        if edges and rng.random() < 0.3:
            edges.append(list(rng.choice(edges)))  # a duplicate edge
        rng.shuffle(nodes)
        rng.shuffle(edges)
        if trial % 10 == 9 and edges:  # a back edge: cycle
            a, b = rng.choice(edges)
            edges.append([b, a])
        doc = {"nodes": nodes, "edges": edges}
        try:
            out.append({"doc": doc, "graph": graph_to_document(graph_from_document(doc))})
        except GraphError as exc:
            out.append({"doc": doc, "error": str(exc)})
    bad = [
        [], {"nodes": 3}, {"nodes": [], "edges": {}}, {"nodes": [3]}, {"nodes": [{"id": ""}]},
        {"nodes": [{"id": 7}]}, {"nodes": [{"id": "a", "memory_cost": 1}], "edges": [["a"]]},
        {"nodes": [{"id": "a", "memory_cost": 1}], "edges": [["a", "z"]]},
        {"nodes": [{"id": "a", "memory_cost": 1}], "edges": [["z", "a"]]},
        {"nodes": [{"id": "a", "memory_cost": 1, "kind": 5}]},
        {"nodes": [{"id": "a", "memory_cost": 1, "compute_cost": -1}]},
        {"nodes": [{"id": "a", "memory_cost": 1, "compute_cost": 1.5}]},
        {"nodes": [{"id": "a", "memory_cost": 2**62}, {"id": "b", "memory_cost": 2**62}]},
        {"nodes": [{"id": "a", "memory_cost": 1}], "edges": [["a", "a"]]},
        {"nodes": [{"id": "a", "memory_cost": 1}, {"id": "a", "memory_cost": 1}], "edges": 5},
    ]
    for doc in bad:
        try:
            out.append({"doc": doc, "graph": graph_to_document(graph_from_document(doc))})
        except GraphError as exc:
            out.append({"doc": doc, "error": str(exc)})
    return out


def dump(name: str, obj) -> None:
    path = OUT / name
    path.write_text(json.dumps(obj, separators=(",", ":")) + "\n")
    print(f"wrote {path} ({path.stat().st_size} bytes)")


def main() -> None:
    slow = "--slow" in sys.argv
    only = [a for a in sys.argv[1:] if not a.startswith("--")]
    jobs = {
        "dp_corpus.json": dp_corpus,
        "mfb_corpus.json": mfb_corpus,
        "lattice.json": lattice_corpus,
        "sim_corpus.json": sim_corpus,
        "reports.json": reports,
        "named.json": lambda: named(slow),
        "cli.json": cli_corpus,
        "loader.json": loader_corpus,
        "large_costs.json": large_costs_corpus,
    }
    if "--xslow" in sys.argv:
        jobs = {"named_xslow.json": named_xslow}
    if "--bench" in sys.argv:
        jobs = {"bench_configs.json": bench_configs}
    for fname, fn in jobs.items():
        if only and fname not in only:
            continue
        t0 = time.perf_counter()
        dump(fname, {"generator": "tests/golden/make_golden.py", "reference": "remat 0.1.0",
                     "data": fn()})
        print(f"  {fname}: {time.perf_counter() - t0:.1f}s")


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    main()
