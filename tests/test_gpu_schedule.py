"""GPU simulator (K7) and strategy evaluation against the reference's outputs."""

from __future__ import annotations

import pytest

from _util import golden, h, load
from paper_1905_11722_b200 import (
    BackwardCompute,
    ForwardCompute,
    Free,
    SequenceError,
    SimulationError,
    ValueRef,
    build_schedule,
    liveness_pass,
    make_sequence,
    overhead,
    peak_memory,
    simulate,
    simulate_many,
    stage_memories,
    vanilla_schedule,
)
from paper_1905_11722_b200.graph import boundary, graph_from_document
from paper_1905_11722_b200.schedule import encode, plan_schedules
from paper_1905_11722_b200.strategy import LowerSetSequence

pytestmark = pytest.mark.gpu


def _decode(ops):
    out = []
    for kind, v in ops:
        if kind == "F":
            out.append(ForwardCompute(v))
        elif kind == "B":
            out.append(BackwardCompute(v))
        else:
            out.append(Free(ValueRef(kind.split("_")[1], v)))
    return out


def _check(rep, ref):
    if "error" in ref:
        assert isinstance(rep, SimulationError)
        assert str(rep) == ref["error"]
        return
    assert not isinstance(rep, Exception), rep
    assert rep.peak_live_memory == ref["peak_live_memory"]
    assert list(rep.trace) == ref["trace"]
    assert rep.total_forward_cost == ref["total_forward_cost"]
    assert rep.recompute_cost == ref["recompute_cost"]
    assert rep.backward_count == ref["backward_count"]


def test_simulator_matches_reference_corpus():
    for rec in golden("sim_corpus.json"):
        g = load(rec["graph"])
        scheds, refs = [], []
        for e in rec["entries"]:
            scheds.append(_decode(e["schedule"]))
            refs.append(e["result"])
            if "liveness_schedule" in e:
                scheds.append(_decode(e["liveness_schedule"]))
                refs.append(e["liveness_result"])
        for rep, ref in zip(simulate_many(g, scheds), refs):
            _check(rep, ref)


def test_make_sequence_and_evaluation_match_reference():
    for rec in golden("dp_corpus.json")[:60]:
        g = load(rec["graph"])
        for case in rec["cases"]:
            if not case["feasible"]:
                continue
            chain = [h(x) for x in case["chain"]]
            seq = make_sequence(g, chain)
            assert list(seq.segments) == [h(x) for x in case["segments"]]
            assert list(seq.cached) == [h(x) for x in case["cached"]]
            ev = peak_memory(g, seq)
            assert ev.overhead == case["overhead"] == overhead(g, seq)
            assert list(ev.per_stage_memory) == case["per_stage_memory"]
            assert tuple(case["per_stage_memory"]) == stage_memories(g, seq)
            assert ev.peak_memory == case["peak_memory"]
            assert ev.cached_total == case["cached_total"]


def _chain3():
    ids = ["n0", "n1", "n2"]
    return graph_from_document({
        "nodes": [{"id": x, "kind": "other", "compute_cost": 1, "memory_cost": 1} for x in ids],
        "edges": [["n0", "n1"], ["n1", "n2"]],
    })


def _diamond():
    return graph_from_document({
        "nodes": [{"id": x, "kind": "other", "compute_cost": 1, "memory_cost": 1} for x in "abcd"],
        "edges": [["a", "b"], ["a", "c"], ["b", "d"], ["c", "d"]],
    })


def test_known_answers():
    # reference tests/test_strategy.py:66-80 and test_schedule.py:133-182
    g = _chain3()
    seq = make_sequence(g, [0b1, g.full_mask])
    assert stage_memories(g, seq) == (3, 5)
    d = _diamond()
    a = 1 << d.index_of["a"]
    ev = peak_memory(d, make_sequence(d, [a, d.full_mask]))
    assert ev.per_stage_memory == (4, 7) and ev.overhead == 3 and ev.cached_total == 1
    one = make_sequence(g, [g.full_mask])
    assert overhead(g, one) == 3 and peak_memory(g, one).peak_memory == 6
    rep = simulate(g, vanilla_schedule(g))
    assert rep.peak_live_memory == 5 and rep.recompute_cost == 0 and rep.backward_count == 3
    rep = simulate(d, build_schedule(d, make_sequence(d, [a, d.full_mask])))
    assert rep.recompute_cost == 3 and rep.peak_live_memory == 7 and rep.backward_count == 4
    assert rep.trace[-1] == 0


def test_simulation_errors():
    g = _chain3()
    with pytest.raises(SimulationError, match="reads non-live value fwd:n0"):
        simulate(g, [ForwardCompute(0), Free(ValueRef("fwd", 0)), ForwardCompute(1)])
    with pytest.raises(SimulationError, match="double free"):
        simulate(g, [ForwardCompute(0), Free(ValueRef("fwd", 0)), Free(ValueRef("fwd", 0))])
    with pytest.raises(SimulationError, match="before gradient grad:n2"):
        simulate(g, [ForwardCompute(0), ForwardCompute(1), ForwardCompute(2), BackwardCompute(1)])


def test_sequence_errors():
    g = _chain3()
    with pytest.raises(SequenceError, match="not a lower set"):
        make_sequence(g, [0b010, g.full_mask])
    with pytest.raises(SequenceError, match="strictly increasing"):
        make_sequence(g, [0b011, 0b011, g.full_mask])
    with pytest.raises(SequenceError, match="end at the full node set"):
        make_sequence(g, [0b001])
    with pytest.raises(SequenceError, match="at least one"):
        make_sequence(g, [])


def test_liveness_never_worse_on_device():
    for rec in golden("sim_corpus.json")[:30]:
        g = load(rec["graph"])
        seq = make_sequence(g, [h(x) for x in rec["chain"]])
        sched = build_schedule(g, seq)
        before, after = simulate_many(g, [sched, liveness_pass(g, sched)])
        assert after.peak_live_memory <= before.peak_live_memory
        assert before.peak_live_memory == peak_memory(g, seq).peak_memory


def _enc(ops):
    kind = {"F": 0, "B": 1, "FREE_fwd": 2, "FREE_grad": 3}
    return [[kind[k], v] for k, v in ops]


def _seq(g, chain):
    prev, segs, cached, acc = 0, [], [], 0
    for m in chain:
        segs.append(m & ~prev)
        acc |= boundary(g, m)
        cached.append(acc)
        prev = m
    return LowerSetSequence(tuple(chain), tuple(segs), tuple(cached))


def test_device_builders_match_reference():
    """K7 build_schedule / vanilla_schedule / liveness_pass on the device,
    instruction for instruction against the reference (sim_corpus.json)."""
    for rec in golden("sim_corpus.json"):
        g = load(rec["graph"])
        seq = _seq(g, [h(x) for x in rec["chain"]])
        canon, van = rec["entries"][0], rec["entries"][1]
        sched = build_schedule(g, seq)
        assert encode(sched).tolist() == _enc(canon["schedule"])
        assert encode(liveness_pass(g, sched)).tolist() == _enc(canon["liveness_schedule"])
        vs = vanilla_schedule(g)
        assert encode(vs).tolist() == _enc(van["schedule"])
        assert encode(liveness_pass(g, vs)).tolist() == _enc(van["liveness_schedule"])


def test_batched_build_liveness_simulate_matches_reference():
    """plan_schedules: many plans of one graph built, rewritten and simulated
    in one device batch, equal to the reference's per-plan results."""
    by_graph = {}
    for rec in golden("sim_corpus.json"):
        by_graph.setdefault(str(rec["graph"]), []).append(rec)
    for recs in by_graph.values():
        g = load(recs[0]["graph"])
        seqs = [_seq(g, [h(x) for x in r["chain"]]) for r in recs]
        plain, preps = plan_schedules(g, seqs, liveness=False)
        live, lreps = plan_schedules(g, seqs, liveness=True)
        for r, ps, pr, ls, lr in zip(recs, plain, preps, live, lreps):
            canon = r["entries"][0]
            assert encode(ps).tolist() == _enc(canon["schedule"])
            assert encode(ls).tolist() == _enc(canon["liveness_schedule"])
            _check(pr, canon["result"])
            _check(lr, canon["liveness_result"])


def test_simulator_matches_oracle_on_named_graphs_and_mutations():
    """Parallel simulation against the oracle's sequential replay: canonical
    and liveness schedules of DP plans on the named shapes, and random
    mutations of them (dropped, duplicated and swapped instructions) that
    fault at arbitrary points."""
    import random

    import numpy as np

    from oracle import oracle as orc
    from paper_1905_11722_b200 import Solver, named_graph
    from paper_1905_11722_b200.schedule import decode

    rng = random.Random(5)
    for g in (named_graph("densenet161"), named_graph("pspnet"), named_graph("unet", skip_len=3)):
        s = Solver(g, "pruned")
        b, plan = s.min_feasible_budget("minimize")
        s.close()
        scheds = [build_schedule(g, plan.sequence)]
        scheds.append(liveness_pass(g, scheds[0]))
        scheds.append(vanilla_schedule(g))
        for _ in range(24):
            ops = encode(rng.choice(scheds[:3])).tolist()
            for _ in range(rng.randint(1, 3)):
                i = rng.randrange(len(ops))
                op = rng.choice(["drop", "dup", "swap"])
                if op == "drop":
                    ops.pop(i)
                elif op == "dup":
                    ops.insert(i, list(ops[i]))
                else:
                    j = rng.randrange(len(ops))
                    ops[i], ops[j] = ops[j], ops[i]
            scheds.append(decode(ops))
        for rep, sc in zip(simulate_many(g, scheds), scheds):
            ref = orc.simulate(g, np.asarray(encode(sc)))
            if "error" in ref:
                assert isinstance(rep, SimulationError), ref
                idx = int(str(rep).split()[1].rstrip(":"))
                assert idx == ref["error"][0], (str(rep), ref)
            else:
                assert not isinstance(rep, Exception), rep
                assert rep.peak_live_memory == ref["peak_live_memory"]
                assert list(rep.trace) == ref["trace"]
                assert rep.recompute_cost == ref["recompute_cost"]
                assert rep.total_forward_cost == ref["total_forward_cost"]
                assert rep.backward_count == ref["backward_count"]
