"""Host-side logic (CPU only): the graph format, generators, request
validation, schedule construction, and that the C-ABI library loads and
exports every symbol declared in include/remat_b200.h (no device calls)."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

from _util import golden, h, load
from paper_1905_11722_b200 import (
    GraphError,
    LowerSetSequence,
    PlanRequest,
    TopologySpec,
    build_schedule,
    dump_graph,
    generate,
    graph_from_document,
    graph_to_document,
    liveness_pass,
    load_graph,
    named_graph,
    vanilla_schedule,
)
from paper_1905_11722_b200.graph import boundary, pack_graph, words_to_mask
from paper_1905_11722_b200.schedule import (
    BackwardCompute,
    ForwardCompute,
    Free,
    ScheduleError,
    ValueRef,
    encode,
    schedule_from_text,
    schedule_to_text,
)

ROOT = Path(__file__).resolve().parents[1]


def test_chen_chain_matches_reference():
    """Articulation points and the Chen sqrt(n) chain (host-only part of
    chen_baseline_plan, reference benchmarks.py:136-222)."""
    from paper_1905_11722_b200 import articulation_points, chen_chain

    for rec in golden("reports.json"):
        g = load(rec["graph"])
        assert articulation_points(g) == rec["chen"]["points"], rec["spec"]
        chain, npts = chen_chain(g)
        assert chain == [h(x) for x in rec["chen"]["plan"]["chain"]], rec["spec"]
        assert npts == rec["chen"]["plan"]["stats"]["states_visited"]


# --- graph format ------------------------------------------------------------

def test_golden_graph_documents_round_trip():
    for name in ("dp_corpus.json", "lattice.json", "sim_corpus.json", "named.json", "reports.json"):
        for rec in golden(name):
            g = load(rec["graph"])
            assert graph_to_document(g) == rec["graph"]


def test_loader_matches_reference_on_shuffled_and_malformed_documents():
    """graph_from_document against the reference's own loader (golden
    loader.json): index order of permuted documents with input nodes and
    duplicate edges, and the first error of malformed ones."""
    for rec in golden("loader.json"):
        if "error" in rec:
            with pytest.raises(GraphError) as ei:
                graph_from_document(rec["doc"])
            assert str(ei.value) == rec["error"], rec["doc"]
        else:
            assert graph_to_document(graph_from_document(rec["doc"])) == rec["graph"]


def test_loader_reindexes_in_reverse_dfs_postorder():
    # a shuffled diamond loads as a, c, b, d
    doc = {"nodes": [{"id": x, "memory_cost": 1} for x in "dcba"],
           "edges": [["a", "b"], ["a", "c"], ["b", "d"], ["c", "d"]]}
    g = graph_from_document(doc)
    assert [x.id for x in g.nodes] == ["a", "c", "b", "d"]
    assert load_graph(dump_graph(g)) == g


def test_loader_validation_messages():
    with pytest.raises(GraphError, match="duplicate node id"):
        graph_from_document({"nodes": [{"id": "a", "memory_cost": 1}] * 2})
    with pytest.raises(GraphError, match="dangling edge endpoint"):
        graph_from_document({"nodes": [{"id": "a", "memory_cost": 1}], "edges": [["a", "b"]]})
    with pytest.raises(GraphError, match="cycle detected"):
        graph_from_document({"nodes": [{"id": x, "memory_cost": 1} for x in "ab"],
                             "edges": [["a", "b"], ["b", "a"]]})
    with pytest.raises(GraphError, match="memory cost is required"):
        graph_from_document({"nodes": [{"id": "a"}]})
    with pytest.raises(GraphError, match="must be >= 1"):
        graph_from_document({"nodes": [{"id": "a", "memory_cost": 0}]})
    with pytest.raises(GraphError, match="must be an integer"):
        graph_from_document({"nodes": [{"id": "a", "memory_cost": True}]})
    with pytest.raises(GraphError, match="no intermediate nodes"):
        graph_from_document({"nodes": [{"id": "a", "memory_cost": 1, "is_input": True}]})
    with pytest.raises(GraphError, match="invalid JSON"):
        load_graph("{")
    g = graph_from_document({"nodes": [{"id": "x", "memory_cost": 1, "is_input": True},
                                       {"id": "c", "kind": "conv", "memory_cost": 2}],
                             "edges": [["x", "c"]]})
    assert g.n == 1 and g.compute_costs == (10,)


def test_pack_graph_round_trips_masks():
    g = named_graph("random-dag", depth=130, edge_prob=0.1)
    n, w, preds, succs, t, m = pack_graph(g)
    assert w == 3
    for v in range(n):
        assert words_to_mask(preds[v]) == g.preds[v]
        assert words_to_mask(succs[v]) == g.succs[v]


# --- generators --------------------------------------------------------------

def test_archetypes_match_reference_snapshot_graphs():
    for rec in golden("reports.json"):
        sp = rec["spec"]
        spec = TopologySpec(sp["family"], sp["depth"], seed=sp["seed"],
                            edge_prob=sp["edge_prob"], cost_model=sp["cost_model"])
        assert graph_to_document(generate(spec)) == rec["graph"]


def test_named_shapes_sizes():
    # node counts of PAPER.md:327-333 and the SURVEY Appendix B prototypes
    u = named_graph("unet", skip_len=3)
    assert (u.n, u.total_time, u.total_memory) == (61, 268, 440)
    assert named_graph("resnet50").n == 176
    d = named_graph("densenet161")
    assert (d.n, d.total_time, d.total_memory) == (566, 2006, 337489)
    p = named_graph("pspnet")
    assert (p.n, p.total_time) == (384, 1410)
    assert named_graph("random-dag", depth=516).n == 516


def test_named_shape_lattice_sizes_with_oracle():
    from oracle import oracle as orc

    assert len(orc.family(named_graph("unet", skip_len=1))) == 276
    assert len(orc.family(named_graph("unet", skip_len=2))) == 1006
    assert len(orc.family(named_graph("pspnet"))) == 11181
    assert len(orc.family(named_graph("random-dag", depth=516, edge_prob=0.4))) == 3293


def test_named_graph_rejects_unknown():
    with pytest.raises(ValueError, match="unknown named shape"):
        named_graph("vgg19")


# --- planner request validation (reference planner.py:52-58) -------------------

def test_plan_request_validation_order():
    g = named_graph("unet", skip_len=1)
    with pytest.raises(ValueError, match="non-negative"):
        PlanRequest(g, budget=-1, family="nope")
    with pytest.raises(ValueError, match="family"):
        PlanRequest(g, budget=1, family="everything")
    with pytest.raises(ValueError, match="objective"):
        PlanRequest(g, budget=1, objective="fastest")


# --- schedules (host construction) ---------------------------------------------

def _seq(g, chain):
    prev, segs, cached, acc = 0, [], [], 0
    for m in chain:
        segs.append(m & ~prev)
        acc |= boundary(g, m)
        cached.append(acc)
        prev = m
    return LowerSetSequence(tuple(chain), tuple(segs), tuple(cached))


def _enc(ops):
    kind = {"F": 0, "B": 1, "FREE_fwd": 2, "FREE_grad": 3}
    return [[kind[k], v] for k, v in ops]


def test_schedule_text_round_trip():
    from paper_1905_11722_b200.schedule import decode

    for rec in golden("sim_corpus.json")[:40]:
        g = load(rec["graph"])
        for e in rec["entries"]:
            sched = decode(_enc(e["schedule"]))
            assert encode(sched).tolist() == _enc(e["schedule"])
            assert schedule_from_text(g, schedule_to_text(g, sched)) == sched
    g = named_graph("unet", skip_len=1)
    with pytest.raises(ScheduleError, match="unknown node id"):
        schedule_from_text(g, "F zzz\n")
    with pytest.raises(ScheduleError, match="cannot parse"):
        schedule_from_text(g, "COMPUTE x\n")
    assert encode([ForwardCompute(1), BackwardCompute(2), Free(ValueRef("grad", 3))]).tolist() == [
        [0, 1], [1, 2], [3, 3]]


# --- the C-ABI library --------------------------------------------------------

def _header_symbols():
    text = (ROOT / "include" / "remat_b200.h").read_text()
    return sorted(set(re.findall(r"REMAT_API\s+[\w\s\*]+?\b(remat_\w+)\s*\(", text)))


def test_header_declares_the_bound_symbols():
    from paper_1905_11722_b200 import _native

    assert _header_symbols() == sorted(_native.exported_symbols())


def test_library_loads_and_exports_every_symbol():
    lib_path = ROOT / "paper_1905_11722_b200" / "libremat_b200.so"
    if not lib_path.exists():
        pytest.fail("libremat_b200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(lib_path))
    for name in _header_symbols():
        assert hasattr(lib, name), name
    from paper_1905_11722_b200 import _native

    assert _native.lib().remat_abi_version() == 1


def test_library_contains_sm100a_code():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf",
                          str(ROOT / "paper_1905_11722_b200" / "libremat_b200.so")],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_oracle_import_in_product_package():
    pkg = ROOT / "paper_1905_11722_b200"
    for p in pkg.rglob("*.py"):
        assert not re.search(r"^\s*(from|import)\s+oracle", p.read_text(), re.M), p


# --- C-ABI argument validation (runs before any device work) -------------------

def _raw_graph(n, tcost=1, mcost=1):
    import numpy as np

    from paper_1905_11722_b200.graph import graph_from_document

    doc = {"nodes": [{"id": f"v{i}", "compute_cost": tcost, "memory_cost": mcost}
                     for i in range(n)],
           "edges": [[f"v{i}", f"v{i + 1}"] for i in range(n - 1)]}
    return graph_from_document(doc)


def test_graph_size_limits_are_reported_not_crashed():
    from paper_1905_11722_b200._native import DeviceGraph
    from paper_1905_11722_b200.graph import GraphError

    with pytest.raises(ValueError, match="above 2048 nodes"):
        DeviceGraph(_raw_graph(2049))
    with pytest.raises(GraphError, match="below 2\\^61"):
        DeviceGraph(_raw_graph(4, mcost=1 << 60))


def test_chen_chain_matches_reference_reports():
    """The Chen baseline's chain and candidate count (host-only:
    articulation points from component counts, benchmarks.py:136-211)
    against the reference's report goldens."""
    from paper_1905_11722_b200.benchmarks import articulation_points, chen_chain

    n = 0
    for rec in golden("reports.json"):
        g = load(rec["graph"])
        chain, npoints = chen_chain(g)
        ref = rec["chen"]["plan"]
        assert npoints == ref["stats"]["states_visited"], rec.get("spec")
        assert articulation_points(g) == rec["chen"]["points"], rec.get("spec")
        assert [format(m, "x") for m in chain] == ref["chain"], rec.get("spec")
        n += 1
    assert n >= 6
