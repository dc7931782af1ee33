"""C-ABI boundary checks that need no GPU: symbols, loading, error mapping."""

import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from paper_1912_08810_b200 import _lib, build
from paper_1912_08810_b200.sse import sse_sigma
from paper_1912_08810_b200.types import (
    CombinedD,
    GreensTensor,
    SimParams,
    build_neighbor_map,
    default_grid,
)

HEADER = build.HEADERS[1]


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(sse_\w+)\s*\(", text, re.M)))


def test_library_builds_and_is_current():
    build.build()
    assert build.up_to_date()


def test_header_and_binding_agree():
    assert header_functions() == sorted(_lib.EXPORTED)


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    for name in header_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (sse_\w+)", out))
    assert set(header_functions()) <= exported


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


@pytest.mark.parametrize("kernel, dmma", [
    ("_ZN3sse24sigma_dmma_kslide_kernelILi12ELi12ELi2ELi3ELb0EEEvNS_9SigmaArgsE", 162),  # production K3m, odd Nkz (3 momenta)
    ("_ZN3sse24sigma_dmma_kslide_kernelILi12ELi12ELi3ELi2ELb0EEEvNS_9SigmaArgsE", 108),  # K3m momentum pairs
    ("_ZN3sse24sigma_dmma_kslide_kernelILi10ELi12ELi3ELi3ELb1EEEvNS_9SigmaArgsE", 120),  # K3m, No=10 combined
    ("_ZN3sse22sigma_dmma_pipe_kernelILi12EEEvNS_9SigmaArgsE", 108),  # register-pipelined K3 (2 stages x 54)
    ("_ZN3sse17sigma_dmma_kernelILi12EEEvNS_9SigmaArgsE", 54),        # simple K3
    ("_ZN3sse23sigma_dmma_slide_kernelILi12ELi12ELi3EEEvNS_9SigmaArgsE", 54),  # single-momentum sliding-window K3
    ("_ZN3sse15pi_dmma3_kernelILb0ELi12ELi4ELi9ELi3EEEvNS_6PiArgsEi", 108),    # Pi K6 v3 (paper shapes)
    ("_ZN3sse15pi_dmma3_kernelILb0ELi0ELi0ELi6ELi3EEEvNS_6PiArgsEi", 54),      # Pi K6 v3, 6-warp q in warps (small)
    ("_ZN3sse15pi_dmma4_kernelILi12ELi4ELi4ELi4ELi3ELb1EEEvNS_6PiArgsEi", 216),  # Pi K6 v4 split (default: 4-slot ring, 3 CTAs / SM)
    ("_ZN3sse20pi_build_dmma_kernelILi12ELi3EEEvNS_11PiBuildArgsE", 72),       # Pi K5 v2 (W in 3-n-tile groups)
])
def test_fp64_tensor_core_sass_present(kernel, dmma):
    """The Sigma / Pi kernels issue DMMA.8x8x4 (FP64 tensor cores), not a CPU/DFMA fallback."""
    out = subprocess.run(["cuobjdump", "-sass", "-fun", kernel, _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert out.count("DMMA.8x8x4") >= dmma
    if "slide" in kernel or "pi_dmma3" in kernel or "pi_dmma4" in kernel:  # operands staged by the TMA engine (bulk copies + mbarriers)
        assert "UBLKCP.S.G" in out and "SYNCS" in out
    if "pi_build" in kernel:  # V written by a bulk async store (shared -> global)
        assert "UBLKCP.G.S" in out


def test_version_and_no_cpu_fallback():
    lib = _lib.load()
    assert lib.sse_version() == 1
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    handle = ctypes.c_void_p()
    rc = lib.sse_ctx_create(1, ctypes.byref(handle))
    assert rc == _lib.SSE_ECUDA
    assert "no CUDA device" in lib.sse_last_error().decode()
    with pytest.raises(_lib.SseError):
        _lib.Context(1)


def _instance():
    p = SimParams(n_kz=2, n_qz=1, n_E=4, n_w=2, n_A=4, n_B=2, n_orb=2)
    rng = np.random.default_rng(0)
    z = lambda s: rng.standard_normal(s) + 1j * rng.standard_normal(s)  # noqa: E731
    g = GreensTensor(z(p.electron_shape), z(p.electron_shape))
    dc = CombinedD(z(p.combined_shape), z(p.combined_shape))
    return p, g, dc, z(p.dh_shape), build_neighbor_map(4, 2), default_grid(p)


def test_sse_sigma_argument_errors_match_reference():
    """sse.py:315-318, 329: ValueError before any device work."""
    p, g, dc, dh, nmap, grid = _instance()
    from paper_1912_08810_b200.types import SseVariant

    with pytest.raises(ValueError, match="expects an electron tensor"):
        sse_sigma(SseVariant.REFERENCE, GreensTensor(np.zeros((1, 1, 4, 1, 3, 3)), np.zeros((1, 1, 4, 1, 3, 3))),
                  dc, dh, nmap, grid)
    with pytest.raises(ValueError, match="does not match the neighbor map"):
        sse_sigma(SseVariant.REFERENCE, g, dc, dh, build_neighbor_map(4, 1), grid)
    with pytest.raises(ValueError, match="unknown variant"):
        sse_sigma("no-such-variant", g, dc, dh, nmap, grid)
    with pytest.raises(ValueError, match="dH must have shape"):
        sse_sigma(SseVariant.REFERENCE, g, dc, dh[:, :1], nmap, grid)


def test_types_mirror_reference_validation():
    with pytest.raises(ValueError, match="combined phonon tensor must be a matching 6-D pair"):
        CombinedD(np.zeros((1, 1, 1, 1, 3, 3)), np.zeros((1, 1, 1, 2, 3, 3)))
    with pytest.raises(ValueError, match="lesser/greater shape mismatch"):
        GreensTensor(np.zeros((1, 1, 1, 1, 1)), np.zeros((1, 1, 2, 1, 1)))
    from paper_1912_08810_b200.types import EnergyGrid, NeighborMap

    with pytest.raises(ValueError, match="2-D integer"):
        NeighborMap(np.zeros((2, 2)))
    with pytest.raises(ValueError, match="outside"):
        EnergyGrid(values=(0.0, 1.0), frequency_map=((2, 1.0),), energy_weight=1.0)
    # params.py:151-156: the grid itself must be strictly increasing and uniform
    with pytest.raises(ValueError, match="strictly increasing"):
        EnergyGrid(values=(0.0, 1.0, 0.5), frequency_map=((1, 1.0),), energy_weight=1.0)
    with pytest.raises(ValueError, match="uniformly spaced"):
        EnergyGrid(values=(0.0, 1.0, 3.0), frequency_map=((1, 1.0),), energy_weight=1.0)


@pytest.mark.parametrize("kwargs", [
    dict(n_kz=3, n_qz=3, n_E=706, n_w=70, n_A=4864, n_B=4, n_orb=12),   # paper: ok
    dict(n_kz=3, n_qz=3, n_E=32, n_w=4, n_A=64, n_B=4, n_orb=4),        # tiny: ok with warnings
    dict(n_kz=2, n_qz=3, n_E=8, n_w=2, n_A=8, n_B=2, n_orb=2),          # n_qz > n_kz
    dict(n_kz=3, n_qz=2, n_E=4, n_w=4, n_A=5, n_B=3, n_orb=2),          # n_w >= n_E, odd n_A * n_B
    dict(n_kz=3, n_qz=2, n_E=8, n_w=2, n_A=9, n_B=2, n_orb=2, bnum=4),  # n_A % bnum
    dict(n_kz=0, n_qz=1, n_E=8, n_w=2, n_A=8, n_B=2, n_orb=2, eta=0.0),  # count < 1, eta <= 0
])
def test_validate_mirrors_reference(kwargs):
    """SimParams validation (params.py:84-129): the same verdict, violations and warnings as
    the reference's validate() when the reference is importable (build container)."""
    from paper_1912_08810_b200.types import SimParams, validate

    rep = validate(SimParams(**kwargs))
    assert rep.ok == (not rep.violations)
    ref_src = "/root/reference/pkg/src"
    if not os.path.isdir(ref_src):
        return
    sys.path.insert(0, ref_src)
    try:
        from negflow.params import SimParams as RefParams
        from negflow.params import validate as ref_validate

        want = ref_validate(RefParams(**kwargs))
    finally:
        sys.path.remove(ref_src)
    assert (rep.ok, rep.violations, rep.warnings) == (want.ok, want.violations, want.warnings)


def test_sse_phase_argument_errors():
    """The fused SSE phase validates like the three reference calls, before any device work."""
    from paper_1912_08810_b200.sse import sse_phase

    p, g, dc, dh, nmap, grid = _instance()
    rng = np.random.default_rng(1)
    ph = GreensTensor(rng.standard_normal(p.phonon_shape) + 0j, rng.standard_normal(p.phonon_shape) + 0j)
    with pytest.raises(ValueError, match="expects an electron tensor"):
        sse_phase(ph, ph, dh, nmap, grid, p.n_qz)
    with pytest.raises(ValueError, match="phonon"):
        sse_phase(g, g, dh, nmap, grid, p.n_qz)
    with pytest.raises(ValueError, match="momenta"):
        sse_phase(g, ph, dh, nmap, grid, p.n_qz + 1)
    with pytest.raises(ValueError, match="dH must have shape"):
        sse_phase(g, ph, dh[:, :1], nmap, grid, p.n_qz)
    with pytest.raises(ValueError, match="out arrays"):
        sse_phase(g, ph, dh, nmap, grid, p.n_qz, out=(np.zeros(3),) * 4)


def test_alloc_host_is_a_zeroed_writable_array():
    """The drop-in's output allocator (4 KB-page anonymous mapping for >= 1 GiB, np.zeros below)
    returns ordinary zero-filled, writable, C-contiguous complex128 arrays like the reference's
    np.zeros (sse.py:146-147)."""
    from paper_1912_08810_b200.sse import alloc_host

    for shape in ((3, 5, 7), (2, 1024, 1024, 33)):  # small, and just over 1 GiB
        a = alloc_host(shape)
        assert a.shape == shape and a.dtype == np.complex128 and a.flags.c_contiguous and a.flags.writeable
        assert not a[0].any() and not a[-1].any()
        a[-1, ..., -1] = 1 + 2j
        assert a[-1, ..., -1].all()
        del a
