"""Synthetic SSE inputs.

Two generators:

* ``stream_instance`` replays the reference tests' single-stream recipe
  (``default_rng(seed)``; G<, G>, D<, D>, dH complex normals in that order;
  test_sse.py:32-43, test_acceptance.py:38-39,158-159, cli.py:214-220), used
  for golden-fixture replays at small sizes.
* ``atom_keyed_values`` is the counter-based, atom-keyed generator used at
  paper scale: value(seed, tensor_id, atom, local index) depends on nothing
  else, so the GPU (``sse.fill_synthetic``, libsse ``fill_synthetic_kernel``)
  can fill 95 GB of inputs in place while the host regenerates any atom
  sub-problem bit-exactly for parity checks.  Each real/imaginary part is an
  Irwin-Hall(4) sum of 16-bit digits of a splitmix64 hash, scaled to unit
  variance (integer sum exact, one rounding per product).

Tensor ids: 0 = G<, 1 = G>, 2 = D<, 3 = D>, 4 = dH (scale 0.05, the
``synthesize`` coupling default, device.py:175,226-229).
"""

from __future__ import annotations

import numpy as np

from .types import SimParams, build_neighbor_map, default_grid

G_LESSER, G_GREATER, D_LESSER, D_GREATER, DH = 0, 1, 2, 3, 4
DH_SCALE = 0.05

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_IH_SCALE = float.fromhex("0x1.bb67ae86627e7p-16")  # 1/sqrt((2^32 - 1)/3)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _irwin_hall4(h: np.ndarray, scale: float) -> np.ndarray:
    m = np.uint64(0xFFFF)
    s = (h & m) + ((h >> np.uint64(16)) & m) + ((h >> np.uint64(32)) & m) + (h >> np.uint64(48))
    x = (s.astype(np.int64) - 131070).astype(np.float64) * _IH_SCALE
    return x * scale


def atom_keyed_values(seed: int, tensor_id: int, atoms, outer: int, inner: int, scale: float = 1.0) -> np.ndarray:
    """complex128 [len(atoms), outer, inner] of the atom-keyed generator."""
    atoms = np.asarray(atoms, dtype=np.uint64).reshape(-1)
    k0 = _splitmix64(_splitmix64(np.array([seed], dtype=np.uint64)) ^ np.uint64(tensor_id))
    keys = _splitmix64(k0 ^ atoms)[:, None]  # [A, 1]
    local = np.arange(outer * inner, dtype=np.uint64)[None, :]
    re = _irwin_hall4(_splitmix64(keys ^ (local * np.uint64(2))), scale)
    im = _irwin_hall4(_splitmix64(keys ^ (local * np.uint64(2) + np.uint64(1))), scale)
    return (re + 1j * im).reshape(len(atoms), outer, inner)


def atom_keyed_electron(seed: int, tensor_id: int, p: SimParams, atoms) -> np.ndarray:
    """G slab [Nkz, NE, len(atoms), No, No] (grid-major) for the given atoms."""
    v = atom_keyed_values(seed, tensor_id, atoms, p.n_kz * p.n_E, p.n_orb * p.n_orb)
    return np.ascontiguousarray(
        v.transpose(1, 0, 2).reshape(p.n_kz, p.n_E, len(v), p.n_orb, p.n_orb)
    )


def atom_keyed_phonon(seed: int, tensor_id: int, p: SimParams, atoms) -> np.ndarray:
    """raw D slab [Nqz, Nw, len(atoms), NB+1, 3, 3] for the given atoms."""
    v = atom_keyed_values(seed, tensor_id, atoms, p.n_qz * p.n_w, (p.n_B + 1) * 9)
    return np.ascontiguousarray(v.transpose(1, 0, 2).reshape(p.n_qz, p.n_w, len(v), p.n_B + 1, 3, 3))


def atom_keyed_dh(seed: int, p: SimParams, atoms) -> np.ndarray:
    """dH slab [len(atoms), NB, 3, No, No] (scale 0.05)."""
    v = atom_keyed_values(seed, DH, atoms, 1, p.n_B * 3 * p.n_orb * p.n_orb, DH_SCALE)
    return v.reshape(len(v), p.n_B, 3, p.n_orb, p.n_orb)


def stream_instance(seed: int, p: SimParams, dh_scale: float = 1.0):
    """(G<, G>, D<, D>, dH) drawn from one default_rng(seed) stream."""
    rng = np.random.default_rng(seed)

    def rand(shape):
        return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)

    g_l, g_g = rand(p.electron_shape), rand(p.electron_shape)
    d_l, d_g = rand(p.phonon_shape), rand(p.phonon_shape)
    dh = dh_scale * rand(p.dh_shape)
    return g_l, g_g, d_l, d_g, dh


# BASELINE.json configs (Nqz = Nkz, NB = 4).
CONFIGS = {
    "tiny": SimParams(n_kz=3, n_qz=3, n_E=32, n_w=4, n_A=64, n_B=4, n_orb=4),
    "small": SimParams(n_kz=3, n_qz=3, n_E=256, n_w=16, n_A=1024, n_B=4, n_orb=10),
    "paper": SimParams(n_kz=3, n_qz=3, n_E=706, n_w=70, n_A=4864, n_B=4, n_orb=12),
    "kheavy": SimParams(n_kz=7, n_qz=7, n_E=706, n_w=70, n_A=4864, n_B=4, n_orb=12),
    "large": SimParams(n_kz=5, n_qz=5, n_E=1220, n_w=70, n_A=10240, n_B=4, n_orb=12),
}


def config(name: str):
    """(params, grid, nmap) of a BASELINE config."""
    p = CONFIGS[name]
    return p, default_grid(p), build_neighbor_map(p.n_A, p.n_B)
