"""Shared helpers for the parity tests: golden fixture loading and field-by-field
comparison of a PlanResult (ours) with a reference plan record (golden JSON, made
by tests/golden/make_golden.py from the reference itself) or an oracle dict."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

from paper_1905_11722_b200.graph import graph_from_document

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def golden(name: str):
    return json.loads((GOLDEN / name).read_text())["data"]


def load(doc):
    return graph_from_document(doc)


def h(x: str) -> int:
    return int(x, 16)


STAT_KEYS = ("states_visited", "table_entries", "transitions", "dominated_skipped")


def stats_of(plan) -> dict:
    return {k: getattr(plan.stats, k) for k in STAT_KEYS}


def assert_plan_matches(plan, ref: dict, ctx=""):
    """``plan``: our PlanResult; ``ref``: golden record (hex masks) or oracle dict."""
    assert plan.feasible == ref["feasible"], ctx
    assert stats_of(plan) == ref["stats"], (ctx, stats_of(plan), ref["stats"])
    if not plan.feasible:
        assert plan.sequence is None and plan.evaluation is None and plan.objective_value is None
        return
    conv = (lambda x: h(x)) if isinstance(ref["chain"][0], str) else (lambda x: x)
    assert plan.objective_value == ref["objective_value"], ctx
    assert list(plan.sequence.chain) == [conv(x) for x in ref["chain"]], ctx
    if "segments" in ref:
        assert list(plan.sequence.segments) == [conv(x) for x in ref["segments"]], ctx
        assert list(plan.sequence.cached) == [conv(x) for x in ref["cached"]], ctx
    ev = plan.evaluation
    assert ev.overhead == ref["overhead"], ctx
    assert list(ev.per_stage_memory) == list(ref["per_stage_memory"]), ctx
    assert ev.peak_memory == ref["peak_memory"], ctx
    assert ev.cached_total == ref["cached_total"], ctx
