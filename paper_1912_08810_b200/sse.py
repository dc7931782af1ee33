"""Drop-in SSE electron self-energy on B200: ``sse_sigma`` and device helpers.

``sse_sigma(variant, g, dc, dh, nmap, grid, counter=None)`` keeps the
signature, argument meaning, array conventions and error behaviour of the
reference entry point ``negflow.sse.sse_sigma`` (sse.py:305-329) and
computes Sigma^{<>} with libsse's sm_100a kernels (K2 operator build, K3
fused DMMA Sigma kernel; K1 layout transforms for LAYOUT_TRANSFORMED).
There is no CPU path: without libsse.so and a B200 it raises.

Device-resident entry points (torch CUDA tensors, used by the bench and the
multi-GPU shard driver) are ``sigma_device``, ``layout_transform``,
``preprocess_D_device`` and ``fill_synthetic``.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from .types import (
    VARIANT_CODES,
    CombinedD,
    FlopCounter,
    SelfEnergyTensor,
    SseVariant,
)

Array = np.ndarray

__all__ = [
    "sse_sigma",
    "sse_pi",
    "sse_pi_chains",
    "pi_tallies",
    "pi_device",
    "sigma_tallies",
    "sigma_device",
    "layout_transform",
    "preprocess_D_device",
    "fill_synthetic",
    "alg_flops",
    "sse_phase",
    "sse_phase_device",
    "alloc_host",
]


def _resolve_variant(variant) -> SseVariant:
    """Accept this package's or the reference's SseVariant (matched by value)."""
    if isinstance(variant, SseVariant):
        return variant
    value = getattr(variant, "value", None)
    for v in SseVariant:
        if value == v.value:
            return v
    raise ValueError(f"unknown variant {variant!r}")


def sigma_tallies(variant: SseVariant, n_kz, n_qz, n_e, n_w, n_a, n_b, n_o) -> dict[str, int]:
    """Complex MAC tallies the reference FlopCounter records for Sigma.

    add_matmul call sites sse.py:159-160 (REFERENCE), 183/213 (FISSIONED),
    231/235/260 (REDUNDANCY_REMOVED / LAYOUT_TRANSFORMED), 289/301
    (BATCHED_FUSED), both polarities.
    """
    base = 2 * 3 * n_a * n_b * n_kz * n_e * n_o**3
    qw = n_qz * n_w
    redundant = variant in (SseVariant.REFERENCE, SseVariant.FISSIONED)
    return {"sigma.dhg": base * (qw if redundant else 1), "sigma.accumulate": base * qw}


def alg_flops(n_kz, n_qz, n_e, n_a, n_b, n_o, offsets) -> int:
    """F_alg = 16 NA NB Nkz Nqz No^3 sum_w max(0, NE - off_w) (both polarities)."""
    terms = sum(max(0, n_e - int(o)) for o in offsets)
    return 16 * n_a * n_b * n_kz * n_qz * n_o**3 * terms


def alloc_host(shape) -> Array:
    """A zero-filled complex128 host array for a call's output (the reference allocates its outputs
    with np.zeros, sse.py:146-147).  Large outputs are anonymous mappings with transparent huge pages
    off: the grid-major [Nkz, NE, NA, No, No] output is written one atom-column chunk at a time, so
    with 2 MB pages the FIRST chunk would fault (and the kernel zero) one huge page per (k, E) row --
    8.5 GB at paper before any other chunk could be staged; 4 KB pages spread the page-zeroing over
    the chunks, under the GPU compute.  SSE_OUT_ALLOC=numpy keeps np.zeros."""
    nbytes = int(np.prod(shape)) * 16
    if nbytes < (1 << 30) or os.environ.get("SSE_OUT_ALLOC", "") == "numpy":
        return np.zeros(shape, dtype=np.complex128)
    import mmap

    buf = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    if hasattr(mmap, "MADV_NOHUGEPAGE"):
        buf.madvise(mmap.MADV_NOHUGEPAGE)
    return np.frombuffer(buf, dtype=np.complex128).reshape(shape)


def _f64(arr: Array) -> Array:
    return np.ascontiguousarray(arr, dtype=np.complex128)


def _ptr(arr: Array):
    return arr.ctypes.data_as(ctypes.c_void_p)


def _default_gpus() -> int:
    return int(os.environ.get("SSE_N_GPUS", "1"))


def sse_sigma(
    variant,
    g,
    dc,
    dh: Array,
    nmap,
    grid,
    counter: FlopCounter | None = None,
    *,
    n_gpus: int | None = None,
    timing: dict | None = None,
) -> SelfEnergyTensor:
    """Electron self-energy Sigma^{<>} (drop-in for sse.py:305-329).

    ``n_gpus`` (default ``$SSE_N_GPUS`` or 1) splits atoms over that many
    devices of this process.  ``timing``, if given, is filled with the
    library's per-call timing (milliseconds, bytes, flops).
    """
    if g.kind != "electron":
        raise ValueError("sse_sigma expects an electron tensor")
    if dc.lesser.shape[2:4] != (nmap.n_A, nmap.n_B):
        raise ValueError("combined phonon tensor does not match the neighbor map")
    var = _resolve_variant(variant)

    g_l, g_g = g.lesser, g.greater
    n_kz, n_e, n_a, n_o, n_o2 = g_l.shape
    n_qz, n_w = dc.lesser.shape[:2]
    n_b = nmap.n_B
    if n_o != n_o2:
        raise ValueError(f"electron blocks must be square, got {n_o}x{n_o2}")
    if n_a != nmap.n_A:
        raise ValueError(f"electron tensor has {n_a} atoms but the neighbor map has {nmap.n_A}")
    if dc.lesser.shape[4:] != (3, 3):
        raise ValueError("combined phonon tensor must end in 3x3 blocks")
    dh = np.asarray(dh)
    if dh.shape != (n_a, n_b, 3, n_o, n_o):
        raise ValueError(f"dH must have shape {(n_a, n_b, 3, n_o, n_o)}, got {dh.shape}")
    fmap = grid.frequency_map
    if len(fmap) < n_w:
        raise ValueError(f"frequency map has {len(fmap)} entries for n_w={n_w}")
    offsets = np.array([int(fmap[w][0]) for w in range(n_w)], dtype=np.int64)
    weights = np.array([float(fmap[w][1]) for w in range(n_w)], dtype=np.float64)

    if counter is not None:
        for stage, n in sigma_tallies(var, n_kz, n_qz, n_e, n_w, n_a, n_b, n_o).items():
            counter.stages[stage] = counter.stages.get(stage, 0) + n

    out_l = alloc_host(g_l.shape)
    out_g = alloc_host(g_g.shape)
    if out_l.size == 0 or dc.lesser.size == 0:
        return SelfEnergyTensor(lesser=out_l, greater=out_g)

    idx = np.ascontiguousarray(nmap.idx, dtype=np.int64)
    if idx.size and (idx.min() < 0 or idx.max() >= n_a):
        raise ValueError(f"neighbor map entries must lie in [0, {n_a})")
    arrays = [_f64(g_l), _f64(g_g), _f64(dc.lesser), _f64(dc.greater), _f64(dh)]
    dims = _lib.SseDims(n_kz, n_qz, n_e, n_w, n_a, n_b, n_o)
    tim = _lib.SseTiming()
    ctx = _lib.context(n_gpus=n_gpus or _default_gpus())
    rc = _lib.load().sse_sigma_c128(
        ctx.handle,
        ctypes.byref(dims),
        VARIANT_CODES[var],
        *[_ptr(a) for a in arrays],
        _ptr(idx),
        _ptr(offsets),
        _ptr(weights),
        _ptr(out_l),
        _ptr(out_g),
        ctypes.byref(tim),
    )
    _lib.check(rc)
    if timing is not None:
        timing.update(tim.as_dict())
    return SelfEnergyTensor(lesser=out_l, greater=out_g)


def pi_tallies(hoist_invariant: bool, n_kz, n_qz, n_e, n_w, n_atoms, n_b, n_o) -> dict[str, int]:
    """Complex MAC tallies of the reference Pi kernel (sse.py:353-386), both chains."""
    per = 2 * n_atoms * n_b * n_kz * n_e * 3 * n_o**3
    return {"pi.m2": per * (1 if hoist_invariant else n_qz * n_w), "pi.m1": per * n_qz * n_w}


def sse_pi(
    g,
    dh: Array,
    nmap,
    grid,
    n_qz: int,
    counter: FlopCounter | None = None,
    hoist_invariant: bool = True,
    point_mask: Array | None = None,
    atom_range: tuple[int, int] | None = None,
    *,
    n_gpus: int | None = None,
    timing: dict | None = None,
):
    """Phonon self-energy Pi^{<>} (drop-in for sse.py:409-428) on FP64 tensor cores.

    Same arguments and conventions as the reference: ``point_mask`` restricts
    the (k, E) reduction and ``atom_range`` the produced atoms (distsim);
    ``hoist_invariant`` only changes the ``counter`` tallies (the reference's
    two arrangements are value-identical, test_sse.py:313-318).  Returns the
    slot-layout tensor [Nqz, Nw, NA, NB+1, 3, 3] (slot 0 = -i sum_s chain,
    slots 1.. = +i chain, sse.py:393-406).
    """
    if g.kind != "electron":
        raise ValueError("sse_pi expects the electron Green's tensor")
    g_l, g_g = g.lesser, g.greater
    n_kz, n_e, n_a, n_o, _ = g_l.shape
    n_b = nmap.n_B
    n_w = grid.n_w
    a_lo, a_hi = atom_range if atom_range is not None else (0, n_a)
    mask = None
    if point_mask is not None:
        mask = np.asarray(point_mask, dtype=bool)
        if mask.shape != (n_kz, n_e):
            raise ValueError(f"point mask must have shape ({n_kz}, {n_e})")
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
    if n_a != nmap.n_A:
        raise ValueError(f"electron tensor has {n_a} atoms but the neighbor map has {nmap.n_A}")
    dh = np.asarray(dh)
    if dh.shape != (n_a, n_b, 3, n_o, n_o):
        raise ValueError(f"dH must have shape {(n_a, n_b, 3, n_o, n_o)}, got {dh.shape}")
    if not 0 <= a_lo <= a_hi <= n_a:
        raise ValueError(f"atom range {atom_range} outside [0, {n_a}]")
    if counter is not None:
        for stage, n in pi_tallies(hoist_invariant, n_kz, n_qz, n_e, n_w, a_hi - a_lo, n_b, n_o).items():
            counter.stages[stage] = counter.stages.get(stage, 0) + n
    shape = (n_qz, n_w, n_a, n_b + 1, 3, 3)
    out_l = np.zeros(shape, dtype=np.complex128)
    out_g = np.zeros(shape, dtype=np.complex128)
    from .types import SelfEnergyTensor as _SE

    if out_l.size == 0 or g_l.size == 0 or a_hi == a_lo or n_w == 0:
        return _SE(lesser=out_l, greater=out_g)
    idx = np.ascontiguousarray(nmap.idx, dtype=np.int64)
    if idx.size and (idx.min() < 0 or idx.max() >= n_a):
        raise ValueError(f"neighbor map entries must lie in [0, {n_a})")
    offsets = np.array([int(o) for o in grid.offsets], dtype=np.int64)
    arrays = [_f64(g_l), _f64(g_g), _f64(dh)]
    dims = _lib.SseDims(n_kz, n_qz, n_e, n_w, n_a, n_b, n_o)
    tim = _lib.SseTiming()
    ctx = _lib.context(n_gpus=n_gpus or _default_gpus())
    rc = _lib.load().sse_pi_c128(
        ctx.handle, ctypes.byref(dims), *[_ptr(a) for a in arrays], _ptr(idx), _ptr(offsets),
        float(grid.energy_weight), _ptr(mask) if mask is not None else None, int(a_lo), int(a_hi),
        _ptr(out_l), _ptr(out_g), ctypes.byref(tim),
    )
    _lib.check(rc)
    if timing is not None:
        timing.update(tim.as_dict())
    return _SE(lesser=out_l, greater=out_g)


def sse_pi_chains(
    g,
    dh: Array,
    nmap,
    grid,
    n_qz: int,
    counter: FlopCounter | None = None,
    hoist_invariant: bool = True,
    point_mask: Array | None = None,
    atom_range: tuple[int, int] | None = None,
    *,
    n_gpus: int | None = None,
):
    """Per-(q,w,a,s,i,j) phonon trace chains before the slot signs (drop-in for sse.py:332-390),
    the entry point distsim's schemes call (distsim.py:24,227,344).

    Computed by the same kernels as :func:`sse_pi` (K5-K7); K7 stores slot 1+s = i*chain as
    (-Im, Re), so the chain is recovered exactly (no rounding) from those slots.  Returns
    (chains_lesser, chains_greater) [Nqz, Nw, NA, NB, 3, 3]; rows outside ``atom_range`` are 0.
    """
    pi = sse_pi(g, dh, nmap, grid, n_qz, counter=counter, hoist_invariant=hoist_invariant,
                point_mask=point_mask, atom_range=atom_range, n_gpus=n_gpus)
    out = []
    for slots in (pi.lesser, pi.greater):
        ch = np.empty(slots.shape[:3] + (slots.shape[3] - 1, 3, 3), dtype=np.complex128)
        ch.real = slots[:, :, :, 1:].imag
        ch.imag = -slots[:, :, :, 1:].real
        out.append(ch)
    return out[0], out[1]


def sse_phase(
    g_e,
    g_ph,
    dh: Array,
    nmap,
    grid,
    n_qz: int,
    *,
    n_gpus: int | None = None,
    device: int | None = None,
    out=None,
    timing: dict | None = None,
):
    """The SSE phase of one Born iteration in one library call.

    Equivalent to the body of ``self_consistent_loop`` (sse.py:532-534)::

        dc = preprocess_D(g_ph, nmap)
        sigma = sse_sigma(variant, g_e, dc, dh, nmap, grid)
        pi = sse_pi(g_e, dh, nmap, grid, n_qz)

    but G is uploaded once for Sigma and Pi and preprocess_D runs on the
    device (libsse ``sse_phase_c128``).  Every arrangement of the reference
    gives the same Sigma here (the kernels are arrangement-independent), so
    there is no variant argument.  Returns ``(sigma, pi)``.  Errors as the
    three reference calls (ValueError for inconsistent shapes or a map that
    is not reverse-closed, device.py:55-57).  ``device`` pins the call to one
    GPU (else ``n_gpus`` devices split the atoms); ``out`` = (Sigma<, Sigma>,
    Pi<, Pi>) C-contiguous complex128 host arrays (e.g. pinned) to fill.
    """
    if g_e.kind != "electron":
        raise ValueError("sse_sigma expects an electron tensor")
    if g_ph.kind != "phonon":
        raise ValueError("preprocess_D expects the phonon Green's tensor")
    g_l, g_g = g_e.lesser, g_e.greater
    n_kz, n_e, n_a, n_o, n_o2 = g_l.shape
    n_b = nmap.n_B
    if n_o != n_o2:
        raise ValueError(f"electron blocks must be square, got {n_o}x{n_o2}")
    if n_a != nmap.n_A:
        raise ValueError(f"electron tensor has {n_a} atoms but the neighbor map has {nmap.n_A}")
    d_l, d_g = g_ph.lesser, g_ph.greater
    if d_l.shape[2:] != (n_a, n_b + 1, 3, 3):
        raise ValueError(f"phonon tensor must be [Nqz, Nw, {n_a}, {n_b + 1}, 3, 3], got {d_l.shape}")
    if d_l.shape[0] != n_qz:
        raise ValueError(f"phonon tensor has {d_l.shape[0]} momenta for n_qz={n_qz}")
    n_w = d_l.shape[1]
    dh = np.asarray(dh)
    if dh.shape != (n_a, n_b, 3, n_o, n_o):
        raise ValueError(f"dH must have shape {(n_a, n_b, 3, n_o, n_o)}, got {dh.shape}")
    fmap = grid.frequency_map
    if len(fmap) < n_w:
        raise ValueError(f"frequency map has {len(fmap)} entries for n_w={n_w}")
    offsets = np.array([int(fmap[w][0]) for w in range(n_w)], dtype=np.int64)
    weights = np.array([float(fmap[w][1]) for w in range(n_w)], dtype=np.float64)
    from .types import SelfEnergyTensor as _SE

    if out is not None:
        sig_l, sig_g, pi_l, pi_g = (np.asarray(o) for o in out)
        for o, shape in ((sig_l, g_l.shape), (sig_g, g_l.shape), (pi_l, d_l.shape), (pi_g, d_l.shape)):
            if o.shape != shape or o.dtype != np.complex128 or not o.flags.c_contiguous:
                raise ValueError(f"out arrays must be C-contiguous complex128 of shape {shape}")
    else:
        sig_l = alloc_host(g_l.shape)
        sig_g = alloc_host(g_l.shape)
        pi_l = np.zeros(d_l.shape, dtype=np.complex128)
        pi_g = np.zeros(d_l.shape, dtype=np.complex128)
    if g_l.size == 0 or d_l.size == 0:
        return _SE(lesser=sig_l, greater=sig_g), _SE(lesser=pi_l, greater=pi_g)
    idx = np.ascontiguousarray(nmap.idx, dtype=np.int64)
    if idx.size and (idx.min() < 0 or idx.max() >= n_a):
        raise ValueError(f"neighbor map entries must lie in [0, {n_a})")
    arrays = [_f64(g_l), _f64(g_g), _f64(d_l), _f64(d_g), _f64(dh)]
    dims = _lib.SseDims(n_kz, n_qz, n_e, n_w, n_a, n_b, n_o)
    tim = _lib.SseTiming()
    ctx = _lib.context(device=device) if device is not None else _lib.context(n_gpus=n_gpus or _default_gpus())
    rc = _lib.load().sse_phase_c128(
        ctx.handle, ctypes.byref(dims), *[_ptr(a) for a in arrays], _ptr(idx), _ptr(offsets), _ptr(weights),
        float(grid.energy_weight), _ptr(sig_l), _ptr(sig_g), _ptr(pi_l), _ptr(pi_g), ctypes.byref(tim),
    )
    _lib.check(rc)
    if timing is not None:
        timing.update(tim.as_dict())
    return _SE(lesser=sig_l, greater=sig_g), _SE(lesser=pi_l, greater=pi_g)


# ---------------------------------------------------------------------------
# device-resident API (torch CUDA tensors, complex128)
# ---------------------------------------------------------------------------


def _dptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("device API expects CUDA tensors")
    if not t.is_contiguous():
        raise ValueError("device API expects contiguous tensors")
    return ctypes.c_void_p(t.data_ptr())


_CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy


def _check_dev(t, shape, name: str, device=None) -> None:
    """A contiguous complex128 CUDA tensor of exactly ``shape`` (on ``device`` if given):
    the C side only sees raw pointers, so a mismatch would be an out-of-bounds access."""
    import torch

    if not getattr(t, "is_cuda", False):
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != torch.complex128:
        raise ValueError(f"{name} must be complex128, got {t.dtype}")
    if tuple(t.shape) != tuple(int(x) for x in shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")


def _stream_ptr(stream):
    """cudaStream_t of a torch stream (default: torch's current stream).

    torch's default stream has handle 0, which libsse would read as "use the
    library's own stream"; map it to cudaStreamLegacy so our kernels stay
    ordered with torch's work and events.
    """
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream or _CUDA_STREAM_LEGACY)


def _device_ctx(t):
    return _lib.context(device=t.device.index if t.device.index is not None else 0)


def _electron_shape(n_kz, n_e, atoms, n_o, atom_major):
    return (atoms, n_kz, n_e, n_o, n_o) if atom_major else (n_kz, n_e, atoms, n_o, n_o)


def _check_slab_args(g_l, g_g, dc_l, dc_g, dh, out_l, out_g, atom_major) -> None:
    """Shapes of a device Sigma call: G slab pair, Dc pair / dH of the owned atoms, Sigma pair."""
    if atom_major:
        g_atoms, n_kz, n_e, n_o = (int(x) for x in g_l.shape[:4])
        o_atoms = int(out_l.shape[0])
    else:
        n_kz, n_e, g_atoms, n_o = (int(x) for x in g_l.shape[:4])
        o_atoms = int(out_l.shape[2])
    dev = g_l.device
    _check_dev(g_l, _electron_shape(n_kz, n_e, g_atoms, n_o, atom_major), "g_l", dev)
    _check_dev(g_g, g_l.shape, "g_g", dev)
    _check_dev(out_l, _electron_shape(n_kz, n_e, o_atoms, n_o, atom_major), "out_l", dev)
    _check_dev(out_g, out_l.shape, "out_g", dev)
    n_qz, n_w, _, n_b = (int(x) for x in dc_l.shape[:4])
    _check_dev(dc_l, (n_qz, n_w, o_atoms, n_b, 3, 3), "dc_l", dev)
    _check_dev(dc_g, dc_l.shape, "dc_g", dev)
    _check_dev(dh, (o_atoms, n_b, 3, n_o, n_o), "dh", dev)


def sigma_device(
    g_l,
    g_g,
    dc_l,
    dc_g,
    dh,
    nmap_rows: Array,
    offsets,
    weights,
    out_l,
    out_g,
    *,
    n_a: int,
    g_atom0: int = 0,
    out_atom0: int = 0,
    atom_major: bool = False,
    stream=None,
    sync_timing: bool = False,
) -> dict | None:
    """Sigma for an owned atom range, all tensors resident on one GPU.

    g_*: [Nkz, NE, gA, No, No] (grid-major) or [gA, Nkz, NE, No, No]
    (atom_major) holding atoms [g_atom0, g_atom0 + gA) — every f(a, s) of
    the owned atoms.  out_*: same layout for the owned atoms
    [out_atom0, out_atom0 + oA).  dc_*: [Nqz, Nw, oA, NB, 3, 3];
    dh: [oA, NB, 3, No, No]; nmap_rows: host int64 [oA, NB] (global ids).
    Launches on ``stream`` (default: torch's current stream) and returns
    without synchronising unless ``sync_timing``.
    """
    if atom_major:
        g_atoms, n_kz, n_e, n_o = g_l.shape[0], g_l.shape[1], g_l.shape[2], g_l.shape[3]
        o_atoms = out_l.shape[0]
    else:
        n_kz, n_e, g_atoms, n_o = g_l.shape[0], g_l.shape[1], g_l.shape[2], g_l.shape[3]
        o_atoms = out_l.shape[2]
    n_qz, n_w, dc_atoms, n_b = dc_l.shape[:4]
    if dc_atoms != o_atoms or dh.shape[0] != o_atoms:
        raise ValueError("Dc/dH rows must match the owned atom count")
    idx = np.ascontiguousarray(nmap_rows, dtype=np.int64)
    if idx.shape != (o_atoms, n_b):
        raise ValueError(f"nmap rows must have shape {(o_atoms, n_b)}")
    _check_slab_args(g_l, g_g, dc_l, dc_g, dh, out_l, out_g, atom_major)
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    wts = np.ascontiguousarray(weights, dtype=np.float64)
    dims = _lib.SseDims(n_kz, n_qz, n_e, n_w, n_a, n_b, n_o)
    gs = _lib.SseSlab(g_atom0, g_atoms, int(atom_major), 0)
    os_ = _lib.SseSlab(out_atom0, o_atoms, int(atom_major), 0)
    tim = _lib.SseTiming()
    ctx = _device_ctx(g_l)
    rc = _lib.load().sse_sigma_device(
        ctx.handle, ctypes.byref(dims), ctypes.byref(gs), ctypes.byref(os_),
        _dptr(g_l), _dptr(g_g), _dptr(dc_l), _dptr(dc_g), _dptr(dh),
        _ptr(idx), _ptr(offs), _ptr(wts), _dptr(out_l), _dptr(out_g),
        _stream_ptr(stream), ctypes.byref(tim) if sync_timing else None,
    )
    _lib.check(rc)
    return tim.as_dict() if sync_timing else None


def sigma_device_scatter(
    g_l, g_g, dc_l, dc_g, dh, nmap_rows: Array, offsets, weights, targets_l, targets_g, pt_lo, *,
    n_a: int, g_atom0: int = 0, out_atom0: int = 0, atom_major: bool = False, stream=None,
    sync_timing: bool = False,
) -> dict | None:
    """:func:`sigma_device` with Sigma written into the (k,E)-point layout buffers of the owners.

    ``targets_*[r]``: device pointers (int) of rank r's [pt_lo[r+1]-pt_lo[r], NA, No, No]
    buffers, valid in this process (CUDA IPC mappings of the peers'); ``pt_lo``: the
    GF phase's point partition (``dist.point_chunks``), length nranks + 1.
    """
    if atom_major:
        g_atoms, n_kz, n_e, n_o = g_l.shape[0], g_l.shape[1], g_l.shape[2], g_l.shape[3]
    else:
        n_kz, n_e, g_atoms, n_o = g_l.shape[0], g_l.shape[1], g_l.shape[2], g_l.shape[3]
    n_qz, n_w, o_atoms, n_b = dc_l.shape[:4]
    if dh.shape[0] != o_atoms:
        raise ValueError("Dc/dH rows must match the owned atom count")
    idx = np.ascontiguousarray(nmap_rows, dtype=np.int64)
    if idx.shape != (o_atoms, n_b):
        raise ValueError(f"nmap rows must have shape {(o_atoms, n_b)}")
    dev = g_l.device
    _check_dev(g_l, _electron_shape(n_kz, n_e, g_atoms, n_o, atom_major), "g_l", dev)
    _check_dev(g_g, g_l.shape, "g_g", dev)
    _check_dev(dc_l, (n_qz, n_w, o_atoms, n_b, 3, 3), "dc_l", dev)
    _check_dev(dc_g, dc_l.shape, "dc_g", dev)
    _check_dev(dh, (o_atoms, n_b, 3, n_o, n_o), "dh", dev)
    nranks = len(targets_l)
    if len(targets_g) != nranks or len(pt_lo) != nranks + 1:
        raise ValueError("one target per rank and nranks + 1 point bounds")
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    wts = np.ascontiguousarray(weights, dtype=np.float64)
    bounds = np.ascontiguousarray(pt_lo, dtype=np.int64)
    tl = (ctypes.c_void_p * nranks)(*[int(x) for x in targets_l])
    tg = (ctypes.c_void_p * nranks)(*[int(x) for x in targets_g])
    dims = _lib.SseDims(n_kz, n_qz, n_e, n_w, n_a, n_b, n_o)
    gs = _lib.SseSlab(g_atom0, g_atoms, int(atom_major), 0)
    os_ = _lib.SseSlab(out_atom0, o_atoms, int(atom_major), 0)
    tim = _lib.SseTiming()
    ctx = _device_ctx(g_l)
    rc = _lib.load().sse_sigma_device_scatter(
        ctx.handle, ctypes.byref(dims), ctypes.byref(gs), ctypes.byref(os_),
        _dptr(g_l), _dptr(g_g), _dptr(dc_l), _dptr(dc_g), _dptr(dh),
        _ptr(idx), _ptr(offs), _ptr(wts), nranks, _ptr(bounds), tl, tg,
        _stream_ptr(stream), ctypes.byref(tim) if sync_timing else None,
    )
    _lib.check(rc)
    return tim.as_dict() if sync_timing else None


def sigma_device_peer(
    sources_l, sources_g, dc_l, dc_g, dh, nmap_rows: Array, offsets, weights, targets_l, targets_g, pt_lo, *,
    n_kz: int, n_e: int, n_a: int, n_o: int, out_atom0: int, device: int, stream=None,
    sync_timing: bool = False,
) -> dict | None:
    """Sigma of owned atoms with G read from, and Sigma written to, the GF point-layout buffers
    of the owner ranks (``sse_sigma_device_peer``): ``sources_*[r]`` / ``targets_*[r]`` are
    device pointers (int) of rank r's [pts_r, NA, No, No] buffers valid in this process."""
    n_qz, n_w, o_atoms, n_b = dc_l.shape[:4]
    if dh.shape[0] != o_atoms:
        raise ValueError("Dc/dH rows must match the owned atom count")
    idx = np.ascontiguousarray(nmap_rows, dtype=np.int64)
    if idx.shape != (o_atoms, n_b):
        raise ValueError(f"nmap rows must have shape {(o_atoms, n_b)}")
    _check_dev(dc_l, (n_qz, n_w, o_atoms, n_b, 3, 3), "dc_l")
    _check_dev(dc_g, dc_l.shape, "dc_g", dc_l.device)
    _check_dev(dh, (o_atoms, n_b, 3, n_o, n_o), "dh", dc_l.device)
    nranks = len(targets_l)
    if not (len(targets_g) == len(sources_l) == len(sources_g) == nranks) or len(pt_lo) != nranks + 1:
        raise ValueError("one source and target per rank and nranks + 1 point bounds")
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    wts = np.ascontiguousarray(weights, dtype=np.float64)
    bounds = np.ascontiguousarray(pt_lo, dtype=np.int64)
    arr = lambda xs: (ctypes.c_void_p * nranks)(*[int(x) for x in xs])  # noqa: E731
    dims = _lib.SseDims(n_kz, n_qz, n_e, n_w, n_a, n_b, n_o)
    os_ = _lib.SseSlab(out_atom0, o_atoms, 1, 0)
    tim = _lib.SseTiming()
    ctx = _lib.context(device=device)
    rc = _lib.load().sse_sigma_device_peer(
        ctx.handle, ctypes.byref(dims), ctypes.byref(os_), arr(sources_l), arr(sources_g),
        _dptr(dc_l), _dptr(dc_g), _dptr(dh), _ptr(idx), _ptr(offs), _ptr(wts), nranks, _ptr(bounds),
        arr(targets_l), arr(targets_g), _stream_ptr(stream), ctypes.byref(tim) if sync_timing else None,
    )
    _lib.check(rc)
    return tim.as_dict() if sync_timing else None


def slab_from_points(sources, pt_lo, out, *, n_kz: int, n_e: int, n_a: int, g_atom0: int,
                     atom_major: bool = True, self_rank: int = -1, stream=None) -> None:
    """Fill the device G slab ``out`` (atoms [g_atom0, g_atom0 + natoms), layout
    [natoms, Nkz, NE, No, No] or grid-major [Nkz, NE, natoms, No, No]) from the GF
    (k,E)-point layout: ``sources[r]`` is rank r's [pts_r, NA, No, No] buffer (device
    pointer valid in this process, a CUDA-IPC-mapped peer read over NVLink),
    ``pt_lo`` the point bounds, ``self_rank`` this rank (reads start at its own points so
    concurrent pulls spread over the owners) (``sse_slab_from_points``)."""
    import torch

    if out.dtype != torch.complex128:
        raise ValueError("out must be complex128")
    shape = tuple(out.shape)
    if len(shape) != 5 or shape[3] != shape[4]:
        raise ValueError("out must be a 5-d slab of square blocks")
    natoms = shape[0] if atom_major else shape[2]
    grid = shape[1:3] if atom_major else shape[0:2]
    if tuple(grid) != (n_kz, n_e):
        raise ValueError(f"slab grid {tuple(grid)} != (Nkz, NE) = {(n_kz, n_e)}")
    nranks = len(sources)
    if len(pt_lo) != nranks + 1:
        raise ValueError("nranks + 1 point bounds")
    bounds = np.ascontiguousarray(pt_lo, dtype=np.int64)
    srcs = (ctypes.c_void_p * nranks)(*[int(x) for x in sources])
    dims = _lib.SseDims(n_kz, 1, n_e, 1, n_a, 1, shape[3])
    slab = _lib.SseSlab(g_atom0, natoms, 1 if atom_major else 0, 0)
    ctx = _lib.context(device=out.device.index or 0)
    _lib.check(_lib.load().sse_slab_from_points(ctx.handle, ctypes.byref(dims), ctypes.byref(slab), nranks,
                                                _ptr(bounds), srcs, self_rank, _dptr(out), _stream_ptr(stream)))


def pi_device_peer(
    sources_l, sources_g, dh, nmap_rows: Array, offsets, energy_weight: float, out_l, out_g, pt_lo, *,
    n_kz: int, n_qz: int, n_e: int, n_a: int, n_o: int, out_atom0: int, stream=None, sync_timing: bool = False,
) -> dict | None:
    """Pi of owned atoms with G read from the GF point-layout buffers of the owner ranks
    (``sse_pi_device_peer``); out_*: device [Nqz, Nw, oA, NB+1, 3, 3]."""
    o_atoms, n_b = dh.shape[0], dh.shape[1]
    idx = np.ascontiguousarray(nmap_rows, dtype=np.int64)
    if idx.shape != (o_atoms, n_b):
        raise ValueError(f"nmap rows must have shape {(o_atoms, n_b)}")
    nranks = len(sources_l)
    if len(sources_g) != nranks or len(pt_lo) != nranks + 1:
        raise ValueError("one source per rank and nranks + 1 point bounds")
    n_w = out_l.shape[1]
    _check_dev(dh, (o_atoms, n_b, 3, n_o, n_o), "dh")
    _check_dev(out_l, (n_qz, n_w, o_atoms, n_b + 1, 3, 3), "out_l", dh.device)
    _check_dev(out_g, out_l.shape, "out_g", dh.device)
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    bounds = np.ascontiguousarray(pt_lo, dtype=np.int64)
    arr = lambda xs: (ctypes.c_void_p * nranks)(*[int(x) for x in xs])  # noqa: E731
    dims = _lib.SseDims(n_kz, n_qz, n_e, n_w, n_a, n_b, n_o)
    os_ = _lib.SseSlab(out_atom0, o_atoms, 1, 0)
    tim = _lib.SseTiming()
    ctx = _device_ctx(out_l)
    rc = _lib.load().sse_pi_device_peer(
        ctx.handle, ctypes.byref(dims), ctypes.byref(os_), arr(sources_l), arr(sources_g), _dptr(dh), _ptr(idx),
        _ptr(offs), float(energy_weight), nranks, _ptr(bounds), _dptr(out_l), _dptr(out_g),
        _stream_ptr(stream), ctypes.byref(tim) if sync_timing else None,
    )
    _lib.check(rc)
    return tim.as_dict() if sync_timing else None


def pi_device(
    g_l, g_g, dh, nmap_rows: Array, offsets, energy_weight: float, pi_l, pi_g, *, n_a: int, n_qz: int,
    g_atom0: int = 0, out_atom0: int = 0, atom_major: bool = False, point_mask=None, stream=None,
) -> None:
    """Pi of an owned atom range, all tensors on one GPU (see sse_pi_device in include/sse.h).

    g_*: slab with the owned atoms and their neighbours ([Nkz, NE, gA, No, No]
    or atom-major); dh [oA, NB, 3, No, No]; pi_* [Nqz, Nw, oA, NB+1, 3, 3].
    """
    if atom_major:
        g_atoms, n_kz, n_e, n_o = g_l.shape[0], g_l.shape[1], g_l.shape[2], g_l.shape[3]
    else:
        n_kz, n_e, g_atoms, n_o = g_l.shape[0], g_l.shape[1], g_l.shape[2], g_l.shape[3]
    o_atoms, n_b = dh.shape[0], dh.shape[1]
    idx = np.ascontiguousarray(nmap_rows, dtype=np.int64)
    if idx.shape != (o_atoms, n_b):
        raise ValueError(f"nmap rows must have shape {(o_atoms, n_b)}")
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    dev = g_l.device
    _check_dev(g_l, _electron_shape(n_kz, n_e, g_atoms, n_o, atom_major), "g_l", dev)
    _check_dev(g_g, g_l.shape, "g_g", dev)
    _check_dev(dh, (o_atoms, n_b, 3, n_o, n_o), "dh", dev)
    _check_dev(pi_l, (n_qz, len(offs), o_atoms, n_b + 1, 3, 3), "pi_l", dev)
    _check_dev(pi_g, pi_l.shape, "pi_g", dev)
    mask = None if point_mask is None else np.ascontiguousarray(point_mask, dtype=np.uint8)
    if mask is not None and mask.shape != (n_kz, n_e):
        raise ValueError(f"point mask must have shape ({n_kz}, {n_e})")
    dims = _lib.SseDims(n_kz, n_qz, n_e, len(offs), n_a, n_b, n_o)
    gs = _lib.SseSlab(g_atom0, g_atoms, int(atom_major), 0)
    os_ = _lib.SseSlab(out_atom0, o_atoms, int(atom_major), 0)
    rc = _lib.load().sse_pi_device(
        _device_ctx(g_l).handle, ctypes.byref(dims), ctypes.byref(gs), ctypes.byref(os_), _dptr(g_l), _dptr(g_g),
        _dptr(dh), _ptr(idx), _ptr(offs), float(energy_weight), _ptr(mask) if mask is not None else None,
        _dptr(pi_l), _dptr(pi_g), _stream_ptr(stream), None,
    )
    _lib.check(rc)


def sse_phase_device(
    g_l, g_g, d_l, d_g, dh, nmap_idx: Array, grid, sig_l, sig_g, pi_l, pi_g, *,
    g_atom0: int = 0, out_atom0: int = 0, atom_major: bool = False, stream=None, sync_timing: bool = False,
) -> dict | None:
    """The SSE phase of a Born iteration (sse.py:532-534: preprocess_D -> sse_sigma -> sse_pi)
    on device-resident torch tensors of one GPU, no host copies (libsse ``sse_phase_device``).

    g_* : G slab [Nkz, NE, gA, No, No] (or atom-major [gA, ...]) of atoms [g_atom0, g_atom0 + gA),
          the owned atoms and all their neighbours; d_*: raw phonon tensors of the same atoms
          [Nqz, Nw, gA, NB+1, 3, 3]; dh: [oA, NB, 3, No, No] of the owned atoms
          [out_atom0, out_atom0 + oA); nmap_idx: the full host map [NA, NB];
    sig_*: Sigma of the owned atoms (G's layout); pi_*: [Nqz, Nw, oA, NB+1, 3, 3].
    A full single-GPU problem is gA = oA = NA.  Launches on ``stream`` (default: torch's current
    stream); returns the library timing when ``sync_timing``.
    """
    idx = np.ascontiguousarray(nmap_idx, dtype=np.int64)
    if idx.ndim != 2:
        raise ValueError("neighbor map must be a 2-D integer array")
    n_a, n_b = idx.shape
    if atom_major:
        g_atoms, n_kz, n_e, n_o = (int(x) for x in g_l.shape[:4])
        o_atoms = int(sig_l.shape[0])
    else:
        n_kz, n_e, g_atoms, n_o = (int(x) for x in g_l.shape[:4])
        o_atoms = int(sig_l.shape[2])
    n_qz, n_w = int(d_l.shape[0]), int(d_l.shape[1])
    dev = g_l.device
    _check_dev(g_l, _electron_shape(n_kz, n_e, g_atoms, n_o, atom_major), "g_l", dev)
    _check_dev(g_g, g_l.shape, "g_g", dev)
    _check_dev(d_l, (n_qz, n_w, g_atoms, n_b + 1, 3, 3), "d_l", dev)
    _check_dev(d_g, d_l.shape, "d_g", dev)
    _check_dev(dh, (o_atoms, n_b, 3, n_o, n_o), "dh", dev)
    _check_dev(sig_l, _electron_shape(n_kz, n_e, o_atoms, n_o, atom_major), "sig_l", dev)
    _check_dev(sig_g, sig_l.shape, "sig_g", dev)
    _check_dev(pi_l, (n_qz, n_w, o_atoms, n_b + 1, 3, 3), "pi_l", dev)
    _check_dev(pi_g, pi_l.shape, "pi_g", dev)
    fmap = grid.frequency_map
    if len(fmap) < n_w:
        raise ValueError(f"frequency map has {len(fmap)} entries for n_w={n_w}")
    offs = np.array([int(fmap[w][0]) for w in range(n_w)], dtype=np.int64)
    wts = np.array([float(fmap[w][1]) for w in range(n_w)], dtype=np.float64)
    dims = _lib.SseDims(n_kz, n_qz, n_e, n_w, n_a, n_b, n_o)
    gs = _lib.SseSlab(g_atom0, g_atoms, int(atom_major), 0)
    os_ = _lib.SseSlab(out_atom0, o_atoms, int(atom_major), 0)
    tim = _lib.SseTiming()
    rc = _lib.load().sse_phase_device(
        _device_ctx(g_l).handle, ctypes.byref(dims), ctypes.byref(gs), ctypes.byref(os_), _dptr(g_l), _dptr(g_g),
        _dptr(d_l), _dptr(d_g), _dptr(dh), _ptr(idx), _ptr(offs), _ptr(wts), float(grid.energy_weight),
        _dptr(sig_l), _dptr(sig_g), _dptr(pi_l), _dptr(pi_g), _stream_ptr(stream),
        ctypes.byref(tim) if sync_timing else None,
    )
    _lib.check(rc)
    return tim.as_dict() if sync_timing else None


def multi_layout(n_gpus: int, nmap_idx: Array) -> list[tuple[int, int, int, int]]:
    """(lo, hi, glo, ghi) per device of the in-library multi-GPU split (``sse_multi_layout``):
    device i owns atoms [lo, hi) and holds the atom-major G slab [glo, ghi) (owned + halo)."""
    idx = np.ascontiguousarray(nmap_idx, dtype=np.int64)
    n_a, n_b = idx.shape
    dims = _lib.SseDims(1, 1, 1, 1, n_a, n_b, 1)
    bounds = np.zeros(4 * n_gpus, dtype=np.int64)
    ctx = _lib.context(n_gpus=n_gpus)
    _lib.check(_lib.load().sse_multi_layout(ctx.handle, ctypes.byref(dims), _ptr(idx), _ptr(bounds)))
    return [tuple(int(x) for x in bounds[4 * i:4 * i + 4]) for i in range(n_gpus)]


def sigma_multi(g_l, g_g, dc_l, dc_g, dh, nmap_idx: Array, grid, out_l, out_g, *, sync_timing: bool = False):
    """Sigma over all devices of this process in ONE library call (``sse_sigma_multi``): lists with
    one tensor per device i (on cuda:i) in the layout of :func:`multi_layout` -- g_* [ghi-glo, Nkz,
    NE, No, No] with the owned atoms filled (the library fills the halos from the owning devices
    by NCCL), dc_* [Nqz, Nw, hi-lo, NB, 3, 3], dh [hi-lo, NB, 3, No, No], out_* [hi-lo, Nkz, NE, No, No]."""
    n = len(g_l)
    idx = np.ascontiguousarray(nmap_idx, dtype=np.int64)
    n_a, n_b = idx.shape
    lay = multi_layout(n, idx)
    _, n_kz, n_e, n_o = (int(x) for x in g_l[0].shape[:4])
    n_qz, n_w = int(dc_l[0].shape[0]), int(dc_l[0].shape[1])
    import torch

    for i, (lo, hi, glo, ghi) in enumerate(lay):
        dev = torch.device("cuda", i)
        if hi <= lo:  # this device owns no atom (more devices than chunks)
            continue
        _check_dev(g_l[i], (ghi - glo, n_kz, n_e, n_o, n_o), f"g_l[{i}]", dev)
        _check_dev(g_g[i], (ghi - glo, n_kz, n_e, n_o, n_o), f"g_g[{i}]", dev)
        _check_dev(dc_l[i], (n_qz, n_w, hi - lo, n_b, 3, 3), f"dc_l[{i}]", dev)
        _check_dev(dc_g[i], (n_qz, n_w, hi - lo, n_b, 3, 3), f"dc_g[{i}]", dev)
        _check_dev(dh[i], (hi - lo, n_b, 3, n_o, n_o), f"dh[{i}]", dev)
        _check_dev(out_l[i], (hi - lo, n_kz, n_e, n_o, n_o), f"out_l[{i}]", dev)
        _check_dev(out_g[i], (hi - lo, n_kz, n_e, n_o, n_o), f"out_g[{i}]", dev)
    fmap = grid.frequency_map
    offs = np.array([int(fmap[w][0]) for w in range(n_w)], dtype=np.int64)
    wts = np.array([float(fmap[w][1]) for w in range(n_w)], dtype=np.float64)
    arr = lambda ts: (ctypes.c_void_p * n)(*[t.data_ptr() if t.numel() else None for t in ts])  # noqa: E731
    dims = _lib.SseDims(n_kz, n_qz, n_e, n_w, n_a, n_b, n_o)
    tim = _lib.SseTiming()
    ctx = _lib.context(n_gpus=n)
    _lib.check(_lib.load().sse_sigma_multi(
        ctx.handle, ctypes.byref(dims), arr(g_l), arr(g_g), arr(dc_l), arr(dc_g), arr(dh), _ptr(idx), _ptr(offs),
        _ptr(wts), arr(out_l), arr(out_g), ctypes.byref(tim) if sync_timing else None))
    return tim.as_dict() if sync_timing else None


def layout_transform(src, dst, to_atom_major: bool, stream=None) -> None:
    """K1 (sse.py:48-55): [Nkz,NE,NA,No,No] <-> [NA,Nkz,NE,No,No] on the GPU.

    Any trailing block works: the phonon tensors [Nqz,Nw,NA,NB+1,3,3] <-> [NA,Nqz,Nw,NB+1,3,3] too.
    """
    if to_atom_major:
        n_kz, n_e, n_a = src.shape[:3]
        want = (n_a, n_kz, n_e) + tuple(src.shape[3:])
    else:
        n_a, n_kz, n_e = src.shape[:3]
        want = (n_kz, n_e, n_a) + tuple(src.shape[3:])
    _check_dev(src, src.shape, "src")
    _check_dev(dst, want, "dst", src.device)
    blk = int(np.prod(src.shape[3:])) * 2
    rc = _lib.load().sse_layout_transform(
        _device_ctx(src).handle, n_kz, n_e, n_a, blk, int(to_atom_major), _dptr(src), _dptr(dst),
        _stream_ptr(stream),
    )
    _lib.check(rc)


def preprocess_D_device(d, dc, nmap_idx: Array, *, d_atom0: int = 0, out_atom0: int = 0,
                        stream=None) -> None:
    """preprocess_D (sse.py:91-115) for one polarity on the GPU, raw D -> Dc.

    d: [Nqz, Nw, dA, NB+1, 3, 3] holding atoms [d_atom0, d_atom0 + dA);
    dc: [Nqz, Nw, oA, NB, 3, 3] for atoms [out_atom0, out_atom0 + oA);
    nmap_idx: the full host map [NA, NB].
    """
    n_qz, n_w, d_atoms, n_slots = d.shape[:4]
    o_atoms = dc.shape[2]
    idx = np.ascontiguousarray(nmap_idx, dtype=np.int64)
    if idx.ndim != 2 or n_slots != idx.shape[1] + 1:
        raise ValueError(
            f"missing neighbor slot: tensor has {n_slots - 1} slots for {idx.shape[-1]} neighbors"
        )
    _check_dev(d, (n_qz, n_w, d_atoms, n_slots, 3, 3), "d")
    _check_dev(dc, (n_qz, n_w, o_atoms, n_slots - 1, 3, 3), "dc", d.device)
    rc = _lib.load().sse_preprocess_D(
        _device_ctx(d).handle, n_qz, n_w, idx.shape[0], idx.shape[1], _ptr(idx), d_atom0, d_atoms,
        out_atom0, o_atoms, _dptr(d), _dptr(dc), _stream_ptr(stream),
    )
    _lib.check(rc)


def fill_synthetic(dst, seed: int, tensor_id: int, atom0: int, natoms: int, outer: int, inner: int,
                   atom_stride: int, outer_stride: int, scale: float = 1.0, stream=None) -> None:
    """Device side of :func:`paper_1912_08810_b200.inputs.atom_keyed_values`."""
    _check_dev(dst, dst.shape, "dst")
    if natoms > 0:  # the last element written must lie inside dst
        last = (natoms - 1) * atom_stride + (outer - 1) * outer_stride + inner - 1
        if min(atom_stride, outer_stride) < 0 or last >= dst.numel():
            raise ValueError(f"fill of {natoms} x {outer} x {inner} values overruns dst ({dst.numel()} elements)")
    rc = _lib.load().sse_fill_synthetic(
        _device_ctx(dst).handle, ctypes.c_uint64(seed), ctypes.c_uint32(tensor_id), atom0, natoms,
        outer, inner, atom_stride, outer_stride, float(scale), _dptr(dst), _stream_ptr(stream),
    )
    _lib.check(rc)


def _host_ptr(a):
    """ctypes pointer of a C-contiguous numpy array or CPU (pinned) torch tensor."""
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("host arrays must be C-contiguous")
        return _ptr(a)
    if getattr(a, "is_cuda", False):
        raise ValueError("host API expects host memory")
    if not a.is_contiguous():
        raise ValueError("host arrays must be contiguous")
    return ctypes.c_void_p(a.data_ptr())


def sigma_host_slab(
    g_l, g_g, dc_l, dc_g, dh, nmap_rows, offsets, weights, out_l, out_g, *,
    n_a: int, g_atom0: int, out_atom0: int, variant=SseVariant.BATCHED_FUSED,
    device: int | None = None, n_gpus: int | None = None,
) -> dict:
    """Host-memory Sigma of an owned atom range (libsse sse_sigma_c128_slab).

    Grid-major host slabs (numpy or pinned torch CPU tensors):
    g_* [Nkz, NE, gA, No, No] for atoms [g_atom0, g_atom0 + gA);
    out_* [Nkz, NE, oA, No, No], dc_* [Nqz, Nw, oA, NB, 3, 3],
    dh [oA, NB, 3, No, No] for atoms [out_atom0, out_atom0 + oA).
    Copies in, computes on the GPU(s) (pipelined), copies Sigma out; returns
    the library's timing.
    """
    n_kz, n_e, g_atoms, n_o = (int(x) for x in g_l.shape[:4])
    o_atoms = int(out_l.shape[2])
    n_qz, n_w, _, n_b = (int(x) for x in dc_l.shape[:4])
    idx = np.ascontiguousarray(nmap_rows, dtype=np.int64)
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    wts = np.ascontiguousarray(weights, dtype=np.float64)
    dims = _lib.SseDims(n_kz, n_qz, n_e, n_w, n_a, n_b, n_o)
    gs = _lib.SseSlab(g_atom0, g_atoms, 0, 0)
    os_ = _lib.SseSlab(out_atom0, o_atoms, 0, 0)
    tim = _lib.SseTiming()
    ctx = _lib.context(device=device) if device is not None else _lib.context(n_gpus=n_gpus or _default_gpus())
    rc = _lib.load().sse_sigma_c128_slab(
        ctx.handle, ctypes.byref(dims), VARIANT_CODES[_resolve_variant(variant)], ctypes.byref(gs),
        ctypes.byref(os_), *[_host_ptr(a) for a in (g_l, g_g, dc_l, dc_g, dh)], _ptr(idx), _ptr(offs),
        _ptr(wts), _host_ptr(out_l), _host_ptr(out_g), ctypes.byref(tim),
    )
    _lib.check(rc)
    return tim.as_dict()


class Profile:
    """CUDA-event profile of libsse launches on one context (per kernel kind).

    with Profile(device=0) as prof: ...  ->  prof.result["sigma"]["ms"], ...
    """

    def __init__(self, device: int | None = 0, n_gpus: int | None = None):
        self.ctx = _lib.context(device=device) if device is not None else _lib.context(n_gpus=n_gpus or 1)
        self.result: dict = {}

    def __enter__(self):
        _lib.check(_lib.load().sse_profile_begin(self.ctx.handle))
        return self

    def __exit__(self, *exc):
        prof = _lib.SseProfile()
        _lib.check(_lib.load().sse_profile_end(self.ctx.handle, ctypes.byref(prof)))
        self.result = prof.as_dict()
        return False
