"""Synthetic graphs for parity tests and the bench configs.

Two groups:

* The reference's six structural archetypes (``pkg/src/remat/benchmarks.py:26-133``:
  ``TopologySpec`` + ``generate``).  They must produce byte-identical graph
  documents because the reference's frozen report snapshots
  (``pkg/tests/data/report_*.csv``) are keyed on them.
* Op-level "named shapes" for the configs in BASELINE.json (the reference has
  none; SURVEY §7 step 0 / Appendix B gives the recipes).  Node kinds drive the
  loader's default compute cost (conv = 10, else 1; reference graph.py:172-174)
  and memory costs are integer activation sizes.
"""

from __future__ import annotations

import random
from dataclasses import dataclass

from .graph import ComputationGraph, graph_from_document

FAMILIES = ("chain", "skip-chain", "resnet-like", "densenet-like", "unet-like", "random-dag")
COST_MODELS = ("uniform", "conv-weighted")


@dataclass(frozen=True)
class TopologySpec:
    family: str
    depth: int
    skip: int = 2
    seed: int = 0
    edge_prob: float = 0.5
    cost_model: str = "uniform"

    def __post_init__(self):
        if self.family not in FAMILIES:
            raise ValueError(f"unknown family {self.family!r}; expected one of {FAMILIES}")
        if self.cost_model not in COST_MODELS:
            raise ValueError(f"unknown cost model {self.cost_model!r}")
        if self.depth < 1:
            raise ValueError("depth must be at least 1")
        if self.family == "skip-chain" and self.skip < 2:
            raise ValueError("skip distance must be at least 2")


def _archetype(spec: TopologySpec):
    d = spec.depth
    f = spec.family
    if f in ("chain", "skip-chain"):
        nodes = [(f"v{i}", "other" if i % 2 else "conv", 1) for i in range(d)]
        edges = [(f"v{i}", f"v{i + 1}") for i in range(d - 1)]
        if f == "skip-chain":
            edges += [(f"v{i}", f"v{i + spec.skip}") for i in range(d - spec.skip)]
        return nodes, edges
    if f == "resnet-like":
        nodes, edges, prev = [("stem", "conv", 2)], [], "stem"
        for b in range(d):
            c1, c2, add = f"b{b}c1", f"b{b}c2", f"b{b}add"
            nodes += [(c1, "conv", 2), (c2, "conv", 2), (add, "other", 2)]
            edges += [(prev, c1), (c1, c2), (c2, add), (prev, add)]
            prev = add
        return nodes, edges
    if f == "densenet-like":
        nodes = [(f"d{i}", "conv", 1) for i in range(d)]
        edges = [(f"d{j}", f"d{i}") for i in range(d) for j in range(i)]
        return nodes, edges
    if f == "unet-like":
        nodes = [(f"e{l}", "conv", 2 ** (d - l)) for l in range(d + 1)]
        nodes += [(f"u{l}", "conv", 2 ** (d - l)) for l in range(d - 1, -1, -1)]
        edges = [(f"e{l}", f"e{l + 1}") for l in range(d)]
        edges.append((f"e{d}", f"u{d - 1}"))
        edges += [(f"u{l + 1}", f"u{l}") for l in range(d - 1)]
        edges += [(f"e{l}", f"u{l}") for l in range(d)]
        return nodes, edges
    # random-dag: edges first, then kinds, from one seeded stream
    rng = random.Random(spec.seed)
    edges = [
        (f"r{i}", f"r{j}")
        for i in range(d)
        for j in range(i + 1, d)
        if rng.random() < spec.edge_prob
    ]
    nodes = [(f"r{i}", "conv" if rng.random() < 0.3 else "other", 1) for i in range(d)]
    return nodes, edges


def generate_document(spec: TopologySpec) -> dict:
    nodes, edges = _archetype(spec)
    out = []
    for nid, kind, width in nodes:
        e = {"id": nid, "kind": kind}
        if spec.cost_model == "uniform":
            e["compute_cost"] = 1
            e["memory_cost"] = 1
        else:
            e["memory_cost"] = width
        out.append(e)
    return {"nodes": out, "edges": [list(e) for e in edges]}


def generate(spec: TopologySpec) -> ComputationGraph:
    return graph_from_document(generate_document(spec))


# --------------------------------------------------------------------------
# Op-level named shapes (SURVEY Appendix B recipes)
# --------------------------------------------------------------------------

class _Doc:
    def __init__(self):
        self.nodes: list[dict] = []
        self.edges: list[list[str]] = []
        self._count: dict[str, int] = {}

    def add(self, kind: str, mem: int, *inputs: str, tag: str = "") -> str:
        k = self._count.get(kind, 0)
        self._count[kind] = k + 1
        nid = tag or f"{kind}{k}"
        self.nodes.append({"id": nid, "kind": kind, "memory_cost": max(1, int(mem))})
        self.edges.extend([src, nid] for src in inputs)
        return nid

    def document(self) -> dict:
        return {"nodes": self.nodes, "edges": self.edges}


def unet_document(skip_len: int = 3) -> dict:
    """Op-level U-Net with "copy-and-crop" skip branches of ``skip_len`` nodes.

    n = 49 + 4·skip_len.  Widths 2^(4-l) at encoder/decoder level l, pools half,
    concats double, bottleneck 1, output map 1 (c=3 gives
    n=61, T(V)=268, M(V)=440, |L_G|=2,726).  ``skip_len`` is the lattice-size knob.
    """
    if skip_len < 1:
        raise ValueError("skip_len must be >= 1")
    d = _Doc()
    levels = 4
    crops: list[str] = []
    prev: str | None = None
    for l in range(levels):
        w = 2 ** (levels - l)
        c1 = d.add("conv", w, *([prev] if prev else []), tag=f"enc{l}_conv1")
        r1 = d.add("relu", w, c1, tag=f"enc{l}_relu1")
        c2 = d.add("conv", w, r1, tag=f"enc{l}_conv2")
        r2 = d.add("relu", w, c2, tag=f"enc{l}_relu2")
        src = r2
        for k in range(skip_len):
            src = d.add("crop", w, src, tag=f"enc{l}_crop{k}")
        crops.append(src)
        prev = d.add("pool", w // 2, r2, tag=f"enc{l}_pool")
    x = prev
    for k, kind in enumerate(("conv", "relu", "conv", "relu")):
        x = d.add(kind, 1, x, tag=f"mid_{kind}{k}")
    for l in range(levels - 1, -1, -1):
        w = 2 ** (levels - l)
        up = d.add("conv", w, x, tag=f"dec{l}_up")
        cat = d.add("concat", 2 * w, up, crops[l], tag=f"dec{l}_concat")
        c1 = d.add("conv", w, cat, tag=f"dec{l}_conv1")
        r1 = d.add("relu", w, c1, tag=f"dec{l}_relu1")
        c2 = d.add("conv", w, r1, tag=f"dec{l}_conv2")
        x = d.add("relu", w, c2, tag=f"dec{l}_relu2")
    d.add("conv", 1, x, tag="out_conv")
    return d.document()


def _mib(batch: int, c: int, h: int, w: int) -> int:
    """Activation size in MiB of fp32, rounded up (>= 1)."""
    return max(1, -(-(batch * c * h * w * 4) // (1 << 20)))


def resnet50_document(batch: int = 96) -> dict:
    """Op-level ResNet-50 (n = 176): conv/bn/relu/add nodes, bottleneck stages
    (3, 4, 6, 3) with a projection shortcut on each stage's first block.
    Memory = fp32 activation MiB at ``batch`` × 224²."""
    d = _Doc()
    b = batch
    x = d.add("conv", _mib(b, 64, 112, 112), tag="stem_conv")
    x = d.add("bn", _mib(b, 64, 112, 112), x, tag="stem_bn")
    x = d.add("relu", _mib(b, 64, 112, 112), x, tag="stem_relu")
    x = d.add("pool", _mib(b, 64, 56, 56), x, tag="stem_pool")
    hw = 56
    for s, (blocks, width) in enumerate(zip((3, 4, 6, 3), (64, 128, 256, 512))):
        for k in range(blocks):
            out_hw = hw // 2 if (k == 0 and s > 0) else hw
            p = f"s{s}b{k}"
            a = d.add("conv", _mib(b, width, hw, hw), x, tag=f"{p}_conv1")
            a = d.add("bn", _mib(b, width, hw, hw), a, tag=f"{p}_bn1")
            a = d.add("relu", _mib(b, width, hw, hw), a, tag=f"{p}_relu1")
            a = d.add("conv", _mib(b, width, out_hw, out_hw), a, tag=f"{p}_conv2")
            a = d.add("bn", _mib(b, width, out_hw, out_hw), a, tag=f"{p}_bn2")
            a = d.add("relu", _mib(b, width, out_hw, out_hw), a, tag=f"{p}_relu2")
            a = d.add("conv", _mib(b, 4 * width, out_hw, out_hw), a, tag=f"{p}_conv3")
            a = d.add("bn", _mib(b, 4 * width, out_hw, out_hw), a, tag=f"{p}_bn3")
            short = x
            if k == 0:
                short = d.add("conv", _mib(b, 4 * width, out_hw, out_hw), x, tag=f"{p}_proj")
                short = d.add("bn", _mib(b, 4 * width, out_hw, out_hw), short, tag=f"{p}_projbn")
            a = d.add("add", _mib(b, 4 * width, out_hw, out_hw), a, short, tag=f"{p}_add")
            x = d.add("relu", _mib(b, 4 * width, out_hw, out_hw), a, tag=f"{p}_relu3")
            hw = out_hw
    x = d.add("pool", _mib(b, 2048, 1, 1), x, tag="head_pool")
    x = d.add("flatten", _mib(b, 2048, 1, 1), x, tag="head_flatten")
    x = d.add("fc", _mib(b, 1000, 1, 1), x, tag="head_fc")
    d.add("loss", 1, x, tag="head_loss")
    return d.document()


def densenet161_document() -> dict:
    """Op-level DenseNet-161 (n = 566): BN-ReLU-Conv1×1-BN-ReLU-Conv3×3 layers
    with a running concat, blocks (6, 12, 36, 24), growth 48; memory = channel
    count."""
    d = _Doc()
    x = d.add("conv", 96, tag="stem_conv")
    x = d.add("bn", 96, x, tag="stem_bn")
    x = d.add("relu", 96, x, tag="stem_relu")
    x = d.add("pool", 96, x, tag="stem_pool")
    ch = 96
    for bi, layers in enumerate((6, 12, 36, 24)):
        for li in range(layers):
            p = f"b{bi}l{li}"
            a = d.add("bn", ch, x, tag=f"{p}_bn1")
            a = d.add("relu", ch, a, tag=f"{p}_relu1")
            a = d.add("conv", 192, a, tag=f"{p}_conv1")
            a = d.add("bn", 192, a, tag=f"{p}_bn2")
            a = d.add("relu", 192, a, tag=f"{p}_relu2")
            a = d.add("conv", 48, a, tag=f"{p}_conv3")
            ch += 48
            x = d.add("concat", ch, x, a, tag=f"{p}_concat")
        if bi < 3:
            p = f"t{bi}"
            a = d.add("bn", ch, x, tag=f"{p}_bn")
            a = d.add("relu", ch, a, tag=f"{p}_relu")
            ch //= 2
            a = d.add("conv", ch, a, tag=f"{p}_conv")
            x = d.add("pool", ch, a, tag=f"{p}_pool")
    x = d.add("bn", ch, x, tag="tail_bn")
    x = d.add("relu", ch, x, tag="tail_relu")
    x = d.add("pool", ch, x, tag="tail_pool")
    d.add("fc", 1, x, tag="tail_fc")
    return d.document()


def pspnet_document(memory: str = "uniform") -> dict:
    """Op-level PSPNet (n = 384): dilated ResNet-101 trunk (3, 4, 23, 3),
    4-branch pyramid pooling, main and auxiliary heads, summed losses
    (uniform M=1 gives |L_G| = 11,181)."""
    d = _Doc()
    uni = memory == "uniform"

    def m(c: int, hw: int) -> int:
        return 1 if uni else _mib(2, c, hw, hw)

    x = None
    for k, (c, hw) in enumerate(((64, 357), (64, 357), (128, 357))):
        x = d.add("conv", m(c, hw), *([x] if x else []), tag=f"stem{k}_conv")
        x = d.add("bn", m(c, hw), x, tag=f"stem{k}_bn")
        x = d.add("relu", m(c, hw), x, tag=f"stem{k}_relu")
    x = d.add("pool", m(128, 179), x, tag="stem_pool")
    hw = 179
    aux_src = None
    for s, (blocks, width) in enumerate(zip((3, 4, 23, 3), (64, 128, 256, 512))):
        if s == 1:
            hw = 90
        for k in range(blocks):
            p = f"s{s}b{k}"
            a = x
            for j, c in enumerate((width, width)):
                a = d.add("conv", m(c, hw), a, tag=f"{p}_conv{j}")
                a = d.add("bn", m(c, hw), a, tag=f"{p}_bn{j}")
                a = d.add("relu", m(c, hw), a, tag=f"{p}_relu{j}")
            a = d.add("conv", m(4 * width, hw), a, tag=f"{p}_conv2")
            a = d.add("bn", m(4 * width, hw), a, tag=f"{p}_bn2")
            short = x
            if k == 0:
                short = d.add("conv", m(4 * width, hw), x, tag=f"{p}_proj")
                short = d.add("bn", m(4 * width, hw), short, tag=f"{p}_projbn")
            a = d.add("add", m(4 * width, hw), a, short, tag=f"{p}_add")
            x = d.add("relu", m(4 * width, hw), a, tag=f"{p}_relu")
        if s == 2:
            aux_src = x
    feats = [x]
    for k, bins in enumerate((1, 2, 3, 6)):
        p = f"ppm{k}"
        a = d.add("pool", m(2048, bins), x, tag=f"{p}_pool")
        a = d.add("conv", m(512, bins), a, tag=f"{p}_conv")
        a = d.add("bn", m(512, bins), a, tag=f"{p}_bn")
        a = d.add("relu", m(512, bins), a, tag=f"{p}_relu")
        feats.append(d.add("upsample", m(512, hw), a, tag=f"{p}_up"))
    cat = d.add("concat", m(4096, hw), *feats, tag="ppm_concat")

    def head(src: str, p: str) -> str:
        a = d.add("conv", m(512, hw), src, tag=f"{p}_conv0")
        a = d.add("bn", m(512, hw), a, tag=f"{p}_bn")
        a = d.add("relu", m(512, hw), a, tag=f"{p}_relu")
        a = d.add("dropout", m(512, hw), a, tag=f"{p}_drop")
        a = d.add("conv", m(21, hw), a, tag=f"{p}_conv1")
        a = d.add("upsample", m(21, 713), a, tag=f"{p}_up")
        return d.add("loss", 1, a, tag=f"{p}_loss")

    main = head(cat, "head")
    aux = head(aux_src, "aux")
    d.add("sum", 1, main, aux, tag="total_loss")
    return d.document()


NAMED_SHAPES = ("resnet50", "unet", "densenet161", "pspnet", "random-dag")


def named_graph(name: str, **kw) -> ComputationGraph:
    """Graph for a BASELINE.json config shape: ``resnet50`` (C1), ``unet`` (C2,
    kw ``skip_len``), ``densenet161`` (C3), ``pspnet`` (C4, kw ``memory``),
    ``random-dag`` (C5, kw ``depth``, ``edge_prob``, ``seed``)."""
    if name == "resnet50":
        return graph_from_document(resnet50_document(kw.get("batch", 96)))
    if name == "unet":
        return graph_from_document(unet_document(kw.get("skip_len", 3)))
    if name == "densenet161":
        return graph_from_document(densenet161_document())
    if name == "pspnet":
        return graph_from_document(pspnet_document(kw.get("memory", "uniform")))
    if name == "random-dag":
        return generate(
            TopologySpec(
                "random-dag", kw.get("depth", 516), seed=kw.get("seed", 0),
                edge_prob=kw.get("edge_prob", 0.4),
            )
        )
    raise ValueError(f"unknown named shape {name!r}; expected one of {NAMED_SHAPES}")


# ---------------------------------------------------------------------------
# Chen et al. sqrt(n) segmentation baseline (reference benchmarks.py:136-222)
# ---------------------------------------------------------------------------


def _components(adj: list[int], alive: int) -> int:
    """Connected components of the undirected skeleton restricted to the node
    set ``alive`` (bitmask flood fill: one frontier expansion per BFS layer)."""
    count = 0
    left = alive
    while left:
        seed = left & -left
        comp = frontier = seed
        while frontier:
            grow = 0
            f = frontier
            while f:
                low = f & -f
                grow |= adj[low.bit_length() - 1]
                f ^= low
            frontier = grow & alive & ~comp
            comp |= frontier
        left &= ~comp
        count += 1
    return count


def articulation_points(g: ComputationGraph) -> list[int]:
    """Cut vertices of the undirected skeleton of ``g``, ascending — the set
    the reference's low-link DFS returns (benchmarks.py:136-183), computed
    from the definition instead: v is a cut vertex iff deleting it leaves more
    connected components than its own component contributed (an isolated v
    is not one).  O(n) bitmask flood fills; host-only, off the hot path."""
    n = g.n
    adj = [g.preds[v] | g.succs[v] for v in range(n)]
    full = (1 << n) - 1
    base = _components(adj, full)
    cut = []
    for v in range(n):
        if not adj[v]:
            continue  # isolated: removing it only removes its own component
        if _components(adj, full & ~(1 << v)) > base:
            cut.append(v)
    return cut


def chen_chain(g: ComputationGraph) -> tuple[list[int], int]:
    """The Chen baseline's chain and its candidate count (host-only): candidate
    cuts are articulation-point ancestor closures forming a strictly increasing
    chain; a cut is taken once the running segment reaches isqrt(n) nodes; V
    closes the chain (reference benchmarks.py:196-211)."""
    from math import isqrt

    from .graph import ancestors_closure

    points = articulation_points(g)
    cands, cur = [], 0
    for v in points:
        c = ancestors_closure(g, v)
        if c != g.full_mask and c != cur and (cur & ~c) == 0:
            cands.append(c)
            cur = c
    step = max(1, isqrt(g.n))
    chain, last = [], 0
    for c in cands:
        if c.bit_count() - last >= step:
            chain.append(c)
            last = c.bit_count()
    chain.append(g.full_mask)
    return chain, len(points)


def chen_baseline_plan(g: ComputationGraph, budget: int | None = None):
    """sqrt(n)-segment checkpointing baseline scored with the same plan
    machinery (reference benchmarks.py:186-222); infeasible if a given budget
    is below its peak."""
    from .planner import PlanResult, SearchStats
    from .strategy import make_sequence, peak_memory

    chain, npoints = chen_chain(g)
    stats = SearchStats(states_visited=npoints)
    seq = make_sequence(g, chain)
    ev = peak_memory(g, seq)
    if budget is not None and ev.peak_memory > budget:
        return PlanResult(False, None, None, None, budget, "chen", "baseline", stats)
    return PlanResult(True, seq, ev, ev.overhead, ev.peak_memory if budget is None else budget,
                      "chen", "baseline", stats)
