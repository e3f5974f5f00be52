"""Lower-set sequences and their two functionals (drop-in for reference
``pkg/src/remat/strategy.py``).

``make_sequence`` validates on the host (argument checking, as the reference
does) and derives the segments; the cache sets U_i and both functionals —
Eq. 1 overhead and Eq. 2 per-stage memory — are computed on the GPU by the
evaluation kernels (csrc/evaluate.cu), the same ones that score DP plans.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable

from .graph import NodeSet, bits, is_lower_set


class SequenceError(ValueError):
    """A chain of node sets does not form a valid plan (strategy.py:36-37)."""


@dataclass(frozen=True)
class LowerSetSequence:
    chain: tuple[NodeSet, ...]
    segments: tuple[NodeSet, ...]
    cached: tuple[NodeSet, ...]  # U_i after each stage

    @property
    def k(self) -> int:
        return len(self.chain)


@dataclass(frozen=True)
class StrategyEvaluation:
    overhead: int
    per_stage_memory: tuple[int, ...]
    peak_memory: int
    cached_total: int


def _validate(g, masks: tuple[NodeSet, ...]) -> tuple[NodeSet, ...]:
    """strategy.py:74-85 checks, in the reference's order."""
    if not masks:
        raise SequenceError("sequence must contain at least one lower set")
    prev = 0
    segments = []
    for mask in masks:
        if not is_lower_set(g, mask):
            names = ", ".join(g.id_of(v) for v in bits(mask))
            raise SequenceError(f"not a lower set: {{{names}}}")
        if prev | mask != mask or prev == mask:
            raise SequenceError("chain is not strictly increasing")
        segments.append(mask & ~prev)
        prev = mask
    if masks[-1] != g.full_mask:
        raise SequenceError("sequence must end at the full node set")
    return tuple(segments)


def _device_graph(g):
    from .graph import device_graph

    return device_graph(g)


def make_sequence(g, chain: Iterable[NodeSet]) -> LowerSetSequence:
    masks = tuple(chain)
    segments = _validate(g, masks)
    _, _, _, _, cached = _device_graph(g).evaluate(list(masks))
    return LowerSetSequence(masks, segments, tuple(cached))


def _evaluate(g, seq: LowerSetSequence) -> StrategyEvaluation:
    ovh, stages, peak, ctot, _ = _device_graph(g).evaluate(list(seq.chain))
    return StrategyEvaluation(ovh, tuple(stages), peak, ctot)


def overhead(g, seq: LowerSetSequence) -> int:
    """T(V \\ U_k), checked on device against the stage-wise sum (strategy.py:89-101)."""
    return _evaluate(g, seq).overhead


def stage_memories(g, seq: LowerSetSequence) -> tuple[int, ...]:
    """Per-stage backward memory, Eq. 2 (strategy.py:104-117)."""
    return _evaluate(g, seq).per_stage_memory


def peak_memory(g, seq: LowerSetSequence) -> StrategyEvaluation:
    """Overhead, per-stage memory, peak and final cache size (strategy.py:120-128)."""
    return _evaluate(g, seq)
