"""Lower-set families (drop-in for reference ``pkg/src/remat/lattice.py``).

``all_lower_sets`` / ``pruned_lower_sets`` build the family on the GPU (K1 / K2
in csrc/family.cu) and return a ``LowerSetFamily`` that stays resident in HBM;
``.masks`` / ``.index`` materialise Python ints lazily, only when touched.
"""

from __future__ import annotations

from .graph import DEFAULT_LATTICE_CAP, NodeSet


class LatticeTooLargeError(RuntimeError):
    """The graph has more lower sets than the configured cap (lattice.py:21-29)."""

    def __init__(self, cap: int):
        super().__init__(
            f"lattice too large: more than {cap} lower sets; "
            "raise the cap or use the pruned family"
        )
        self.cap = cap


class LowerSetFamily:
    """Ordered, deduplicated lower sets, sorted by (cardinality, bit pattern)
    (lattice.py:32-56).  Device-backed when produced by the builders below."""

    __slots__ = ("_masks", "_index", "_device")

    def __init__(self, masks=None, index=None, device=None):
        self._masks = tuple(masks) if masks is not None else None
        self._index = index
        self._device = device

    @classmethod
    def from_masks(cls, masks) -> "LowerSetFamily":
        ordered = tuple(sorted(set(masks), key=lambda m: (m.bit_count(), m)))
        return cls(ordered, {m: i for i, m in enumerate(ordered)})

    @classmethod
    def _from_device(cls, dev) -> "LowerSetFamily":
        return cls(device=dev)

    @property
    def masks(self) -> tuple[NodeSet, ...]:
        if self._masks is None:
            self._masks = tuple(self._device.masks())
        return self._masks

    @property
    def index(self) -> dict[NodeSet, int]:
        if self._index is None:
            self._index = {m: i for i, m in enumerate(self.masks)}
        return self._index

    @property
    def device(self):
        return self._device

    def __len__(self) -> int:
        if self._masks is None and self._device is not None:
            return self._device.size
        return len(self.masks)

    def __iter__(self):
        return iter(self.masks)

    def __contains__(self, mask: NodeSet) -> bool:
        return mask in self.index

    def __eq__(self, other) -> bool:
        return isinstance(other, LowerSetFamily) and self.masks == other.masks

    def __repr__(self) -> str:
        return f"LowerSetFamily(size={len(self)})"


def _device_graph(g):
    from .graph import device_graph

    return device_graph(g)


def all_lower_sets(g, cap: int = DEFAULT_LATTICE_CAP) -> LowerSetFamily:
    """Every lower set of ``g`` incl. ∅ and V (lattice.py:59-84).

    Raises ``ValueError`` if ``cap < n+1`` and ``LatticeTooLargeError`` when the
    lattice has more than ``cap`` members."""
    if cap < g.n + 1:
        raise ValueError(f"cap must be at least n+1 = {g.n + 1}, got {cap}")
    from ._native import DeviceFamily

    return LowerSetFamily._from_device(DeviceFamily(_device_graph(g), "full", cap))


def pruned_lower_sets(g) -> LowerSetFamily:
    """{closure(v)} ∪ {∅, V} (lattice.py:87-93)."""
    from ._native import DeviceFamily

    return LowerSetFamily._from_device(DeviceFamily(_device_graph(g), "pruned", 0))
