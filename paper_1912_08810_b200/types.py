"""Host-side mirror of the reference data model used by the SSE path.

Same names, fields, validation and error messages as the reference
``negflow`` classes the SSE entry point consumes, so callers (and the
reference's own tests) can hand either kind of object to
:func:`paper_1912_08810_b200.sse.sse_sigma`.  Objects of the reference
package are accepted by duck typing (``.lesser``, ``.greater``, ``.idx``,
``.frequency_map``), see :mod:`paper_1912_08810_b200.compat`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

Array = np.ndarray

FLOPS_PER_CMULADD = 8  # flops.py:16


class SseVariant(Enum):
    """The five Sigma arrangements (sse.py:35-40)."""

    REFERENCE = "reference"
    FISSIONED = "fissioned"
    REDUNDANCY_REMOVED = "redundancy-removed"
    LAYOUT_TRANSFORMED = "layout-transformed"
    BATCHED_FUSED = "batched-fused"


VARIANT_CODES = {
    SseVariant.REFERENCE: 0,
    SseVariant.FISSIONED: 1,
    SseVariant.REDUNDANCY_REMOVED: 2,
    SseVariant.LAYOUT_TRANSFORMED: 3,
    SseVariant.BATCHED_FUSED: 4,
}


def _check_pair(lesser: Array, greater: Array, ndim: int, kind: str) -> None:
    # gf.py:30-34
    if lesser.shape != greater.shape:
        raise ValueError(f"lesser/greater shape mismatch: {lesser.shape} vs {greater.shape}")
    if lesser.ndim != ndim:
        raise ValueError(f"{kind} tensor must be {ndim}-D, got {lesser.ndim}-D")


@dataclass(frozen=True)
class SimParams:
    """Shape fields of the reference SimParams (params.py:24-50)."""

    n_kz: int
    n_qz: int
    n_E: int
    n_w: int
    n_A: int
    n_B: int
    n_orb: int
    bnum: int = 1
    n_3D: int = 3
    eta: float = 1e-3

    @property
    def electron_shape(self) -> tuple[int, int, int, int, int]:
        return (self.n_kz, self.n_E, self.n_A, self.n_orb, self.n_orb)

    @property
    def phonon_shape(self) -> tuple[int, int, int, int, int, int]:
        return (self.n_qz, self.n_w, self.n_A, self.n_B + 1, self.n_3D, self.n_3D)

    @property
    def combined_shape(self) -> tuple[int, int, int, int, int, int]:
        return (self.n_qz, self.n_w, self.n_A, self.n_B, self.n_3D, self.n_3D)

    @property
    def dh_shape(self) -> tuple[int, int, int, int, int]:
        return (self.n_A, self.n_B, self.n_3D, self.n_orb, self.n_orb)

    def replace(self, **kwargs) -> "SimParams":
        from dataclasses import replace

        return replace(self, **kwargs)


# params.py:11-21 soft ranges (warnings only) and the integer count fields
_TYPICAL_RANGES = {"n_kz": (1, 21), "n_qz": (1, 21), "n_E": (700, 1500), "n_w": (10, 100), "n_B": (4, 50),
                   "n_orb": (1, 30)}
_COUNT_FIELDS = ("n_kz", "n_qz", "n_E", "n_w", "n_A", "n_B", "n_orb", "n_3D", "bnum")


@dataclass(frozen=True)
class ValidationReport:
    """Result of :func:`validate` (params.py:71-81)."""

    ok: bool
    violations: tuple[str, ...]
    warnings: tuple[str, ...]


def validate(params: SimParams) -> ValidationReport:
    """The reference's hard invariants and soft ranges of a parameter set (params.py:84-129);
    report-only, never raises."""
    violations: list[str] = []
    warnings: list[str] = []
    ints = {name: isinstance(getattr(params, name), (int, np.integer)) for name in _COUNT_FIELDS}
    for name in _COUNT_FIELDS:
        value = getattr(params, name)
        if not ints[name]:
            violations.append(f"{name} must be an integer, got {value!r}")
        elif value < 1:
            violations.append(f"{name} must be >= 1, got {value}")
    if ints["n_3D"] and params.n_3D != 3:
        violations.append("n_3D must equal 3")
    if ints["n_A"] and ints["bnum"] and params.bnum >= 1 and params.n_A >= 1 and params.n_A % params.bnum != 0:
        violations.append(f"n_A must be divisible by bnum ({params.n_A} % {params.bnum} != 0)")
    if params.n_qz > params.n_kz:
        violations.append(f"n_qz must be <= n_kz ({params.n_qz} > {params.n_kz})")
    if ints["n_A"] and ints["n_B"] and params.n_A % 2 == 1 and params.n_B % 2 == 1:
        violations.append(f"n_A * n_B must be even (got n_A={params.n_A}, n_B={params.n_B})")
    if params.n_w >= params.n_E:
        violations.append(f"n_w must be < n_E ({params.n_w} >= {params.n_E})")
    if not params.eta > 0:
        violations.append(f"eta must be > 0, got {params.eta}")
    for name, (lo, hi) in _TYPICAL_RANGES.items():
        value = getattr(params, name)
        if ints.get(name, isinstance(value, (int, np.integer))) and value >= 1 and not lo <= value <= hi:
            warnings.append(f"{name} outside [{lo},{hi}]: {value}")
    return ValidationReport(ok=not violations, violations=tuple(violations), warnings=tuple(warnings))


@dataclass(frozen=True)
class GreensTensor:
    """Lesser/greater pair; electron 5-D, phonon 6-D (gf.py:37-69)."""

    lesser: Array
    greater: Array

    def __post_init__(self):
        if self.lesser.ndim not in (5, 6):
            raise ValueError("expected a 5-D electron or 6-D phonon tensor")
        _check_pair(self.lesser, self.greater, self.lesser.ndim, self.kind)

    @property
    def kind(self) -> str:
        return "electron" if self.lesser.ndim == 5 else "phonon"


@dataclass(frozen=True)
class SelfEnergyTensor:
    """Scattering self-energy pair, same layouts as GreensTensor (gf.py:72-100)."""

    lesser: Array
    greater: Array

    def __post_init__(self):
        if self.lesser.ndim not in (5, 6):
            raise ValueError("expected a 5-D electron or 6-D phonon tensor")
        _check_pair(self.lesser, self.greater, self.lesser.ndim, self.kind)

    @property
    def kind(self) -> str:
        return "electron" if self.lesser.ndim == 5 else "phonon"


@dataclass(frozen=True)
class CombinedD:
    """Preprocessed phonon input Dc[q,w,a,s,i,j] (sse.py:79-88)."""

    lesser: Array
    greater: Array

    def __post_init__(self):
        if self.lesser.shape != self.greater.shape or self.lesser.ndim != 6:
            raise ValueError("combined phonon tensor must be a matching 6-D pair")


@dataclass(frozen=True)
class NeighborMap:
    """idx[a, s] = atom index of neighbour s of a (device.py:23-66)."""

    idx: Array

    def __post_init__(self):
        idx = np.asarray(self.idx)
        if idx.ndim != 2 or idx.dtype.kind != "i":
            raise ValueError("neighbor map must be a 2-D integer array")

    @property
    def n_A(self) -> int:
        return self.idx.shape[0]

    @property
    def n_B(self) -> int:
        return self.idx.shape[1]

    @property
    def max_reach(self) -> int:
        a = np.arange(self.n_A)[:, None]
        return int(np.max(np.abs(self.idx - a))) if self.idx.size else 0


def build_neighbor_map(n_A: int, n_B: int) -> NeighborMap:
    """1-D chain table, slots a+1, a-1, a+2, a-2, ... reflected at the ends.

    Same table as device.py:105-130 (odd n_B adds an XOR-1 partner slot).
    """
    if n_B >= n_A:
        raise ValueError(f"n_B must be < n_A (got n_B={n_B}, n_A={n_A})")
    if n_B < 1:
        raise ValueError("n_B must be >= 1")
    if n_B % 2 == 1 and n_A % 2 == 1:
        raise ValueError("odd n_B requires an even atom count for a symmetric neighbor map")
    a = np.arange(n_A, dtype=np.int64)
    cols = []
    for m in range(1, n_B // 2 + 1):
        cols.append(np.where(a + m < n_A, a + m, a - m))
        cols.append(np.where(a - m >= 0, a - m, a + m))
    if n_B % 2 == 1:
        cols.append(a ^ 1)
    return NeighborMap(idx=np.stack(cols, axis=1).astype(np.int64))


@dataclass(frozen=True)
class EnergyGrid:
    """Energy grid plus the (offset, weight) frequency map (params.py:132-192)."""

    values: tuple[float, ...]
    frequency_map: tuple[tuple[int, float], ...]
    energy_weight: float

    def __post_init__(self):
        vals = np.asarray(self.values, dtype=float)
        if vals.ndim != 1 or vals.size < 1:
            raise ValueError("energy grid must be a non-empty 1-D sequence")
        if vals.size > 1:  # params.py:151-156
            steps = np.diff(vals)
            if np.any(steps <= 0):
                raise ValueError("energy grid must be strictly increasing")
            if not np.allclose(steps, steps[0], rtol=1e-9, atol=1e-12):
                raise ValueError("energy grid must be uniformly spaced")
        n_e = vals.size
        for w, (off, weight) in enumerate(self.frequency_map):
            if not isinstance(off, (int, np.integer)) or not 0 <= off < n_e:
                raise ValueError(f"frequency offset {off} (index {w}) outside [0, {n_e})")
            if not math.isfinite(weight):
                raise ValueError(f"frequency weight {weight} (index {w}) is not finite")

    @property
    def n_E(self) -> int:
        return len(self.values)

    @property
    def n_w(self) -> int:
        return len(self.frequency_map)

    @property
    def offsets(self) -> tuple[int, ...]:
        return tuple(off for off, _ in self.frequency_map)

    @property
    def weights(self) -> tuple[float, ...]:
        return tuple(w for _, w in self.frequency_map)

    @property
    def max_offset(self) -> int:
        return max(self.offsets) if self.frequency_map else 0


def default_grid(params: SimParams, e_min: float = -1.0, e_max: float = 1.0) -> EnergyGrid:
    """Offsets min(w+1, NE-1), weights 1/(2 pi Nw) (params.py:195-208)."""
    values = (0.0,) if params.n_E == 1 else tuple(np.linspace(e_min, e_max, params.n_E))
    weight = 1.0 / (2.0 * math.pi * params.n_w)
    freq_map = tuple((min(w + 1, params.n_E - 1), weight) for w in range(params.n_w))
    return EnergyGrid(values=values, frequency_map=freq_map, energy_weight=1.0 / (2.0 * math.pi * params.n_E))


@dataclass
class FlopCounter:
    """Per-stage complex multiply-add tally (flops.py:21-41)."""

    stages: dict[str, int] = field(default_factory=dict)

    def add_matmul(self, m: int, k: int, n: int, repeat: int = 1, stage: str = "gemm") -> None:
        self.stages[stage] = self.stages.get(stage, 0) + m * k * n * repeat

    def cmuladds(self, stage: str | None = None) -> int:
        if stage is not None:
            return self.stages.get(stage, 0)
        return sum(self.stages.values())

    def flops(self, stage: str | None = None) -> int:
        return FLOPS_PER_CMULADD * self.cmuladds(stage)
