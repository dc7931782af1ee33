"""Parity of the CUDA phonon self-energy Pi (K5-K7, through the C ABI).

Reference: negflow.sse.sse_pi (sse.py:409-428), chains sse.py:332-390, slot
assembly sse.py:393-406.  Golden outputs come from the reference itself
(tests/golden/make_golden.py); larger shapes and the mask/atom-range options
are checked against the oracle (pinned to those goldens by tests/test_oracle.py).
Tolerance: the reference metric <= 1e-10.
"""

import numpy as np
import pytest

from oracle import sse_oracle as orc
from paper_1912_08810_b200 import inputs
from paper_1912_08810_b200.sse import pi_tallies, sse_pi
from paper_1912_08810_b200.types import (
    EnergyGrid,
    FlopCounter,
    GreensTensor,
    NeighborMap,
    SimParams,
    build_neighbor_map,
    default_grid,
)
from tests.golden_cases import load_case

pytestmark = pytest.mark.gpu
TOL = 1e-10
# pi_paperlike_s12: the paper's No = 12, NB = 4, Nw = 70 -> K5 pi_build_dmma_kernel<12> and the
# split K6 v4 (9 lag tiles) against the reference's own sse_pi output
PI_CASES = ["test_tiny_s3", "test_tiny_s4", "cli_tiny_s1", "cli_small_s2", "general_grid_s8", "pi_paperlike_s12"]


def _grid(case):
    n_e = case.p.n_E
    return EnergyGrid(
        values=tuple(np.linspace(-1, 1, n_e)) if n_e > 1 else (0.0,),
        frequency_map=tuple(zip(case.offsets.tolist(), case.weights.tolist())),
        energy_weight=case.meta["energy_weight"],
    )


@pytest.mark.parametrize("name", PI_CASES)
def test_pi_golden_parity(name):
    c = load_case(name)
    assert c.inputs_ok
    counter = FlopCounter()
    out = sse_pi(GreensTensor(c.g_l, c.g_g), c.dh, NeighborMap(c.idx), _grid(c), c.p.n_qz, counter=counter)
    dev = orc.parity_dev(out.lesser, out.greater, c.arrays["pi_l"], c.arrays["pi_g"])
    assert dev <= TOL, (name, dev)
    if name == "pi_paperlike_s12":
        from paper_1912_08810_b200 import _lib

        assert _lib.kernel_name("pi") == "pi_dmma4_kernel<12,4,4,4,3,true>", _lib.kernel_name("pi")
        assert _lib.kernel_name("pi_build") == "pi_build_dmma_kernel<12>"
    p = c.p
    assert counter.stages == pi_tallies(True, p.n_kz, p.n_qz, p.n_E, p.n_w, p.n_A, p.n_B, p.n_orb)


def test_pi_zero_electron_input():
    """test_sse.py:275-281."""
    c = load_case("test_tiny_s3")
    zero = GreensTensor(np.zeros_like(c.g_l), np.zeros_like(c.g_g))
    out = sse_pi(zero, c.dh, NeighborMap(c.idx), _grid(c), c.p.n_qz)
    assert np.all(out.lesser == 0) and np.all(out.greater == 0)


def test_pi_single_point_signs():
    """test_sse.py:284-302: one (k, E) point, slot 0 = -i chain, slot 1 = +i chain."""
    p = SimParams(n_kz=1, n_qz=1, n_E=1, n_w=1, n_A=2, n_B=1, n_orb=1)
    nmap = build_neighbor_map(2, 1)
    w_e = 0.21
    grid = EnergyGrid(values=(0.0,), frequency_map=((0, 1.0),), energy_weight=w_e)
    rng = np.random.default_rng(10)
    z = lambda s: rng.standard_normal(s) + 1j * rng.standard_normal(s)  # noqa: E731
    g = GreensTensor(z(p.electron_shape), z(p.electron_shape))
    dh = z((2, 1, 3, 1, 1))
    out = sse_pi(g, dh, nmap, grid, 1)
    for a in range(2):
        b = int(nmap.idx[a, 0])
        chain = np.array([[w_e * dh[a, 0, i, 0, 0] * g.greater[0, 0, a, 0, 0] * dh[a, 0, j, 0, 0]
                           * g.lesser[0, 0, b, 0, 0] for j in range(3)] for i in range(3)])
        assert np.allclose(out.greater[0, 0, a, 0], -1j * chain, atol=1e-14)
        assert np.allclose(out.greater[0, 0, a, 1], +1j * chain, atol=1e-14)


def test_pi_hoisting_is_value_neutral():
    """test_sse.py:313-318; only the counter tallies differ (sse.py:353-386)."""
    c = load_case("cli_tiny_s1")
    args = (GreensTensor(c.g_l, c.g_g), c.dh, NeighborMap(c.idx), _grid(c), c.p.n_qz)
    c1, c2 = FlopCounter(), FlopCounter()
    a = sse_pi(*args, counter=c1, hoist_invariant=True)
    b = sse_pi(*args, counter=c2, hoist_invariant=False)
    assert np.array_equal(a.lesser, b.lesser) and np.array_equal(a.greater, b.greater)
    assert c1.stages["pi.m1"] == c2.stages["pi.m1"]
    assert c2.stages["pi.m2"] == c1.stages["pi.m2"] * c.p.n_qz * c.p.n_w


@pytest.mark.parametrize("n_kz, n_qz, n_e, n_w, n_a, n_b, n_o", [
    (3, 3, 30, 10, 6, 4, 12),   # the No of the paper configs
    (2, 2, 17, 5, 5, 4, 10),    # No = 10 (small config), 5 atoms (odd) with NB even
    (3, 3, 40, 16, 6, 4, 10),   # the small config's Nw = 16 / Nqz = 3: K6 v3 with q in warps (6 of 9 warps)
    (4, 3, 9, 3, 4, 1, 5),      # NB = 1 (XOR partner slot), Nqz < Nkz
    (2, 2, 13, 5, 5, 2, 8),     # No = 8 (DMMA operand build), NB = 2
    (2, 1, 9, 4, 5, 4, 16),     # No = 16 (largest DMMA orbital count)
    (1, 1, 80, 75, 3, 2, 4),    # Nw = 75: 10 lag tiles (two warp groups per CTA column)
    (2, 2, 9, 3, 14, 6, 4),     # NB = 6: 54 chains, 14 real n-tiles (two n-groups in K6 v3)
    (1, 1, 12, 11, 3, 2, 4),    # Nw close to NE (most E + off >= NE terms dropped)
    (2, 2, 7, 3, 4, 2, 1),      # No = 1: one kappa quad, empty second half stage
    (3, 2, 11, 4, 4, 2, 3),     # No = 3: No^2 = 9, ragged last quad
])
def test_pi_shapes_against_oracle(monkeypatch, n_kz, n_qz, n_e, n_w, n_a, n_b, n_o):
    """Every K6 variant (0 direct, 1 TMA 2-q, 2 TMA half stages, 3 one m-tile per warp) vs the oracle."""
    p = SimParams(n_kz=n_kz, n_qz=n_qz, n_E=n_e, n_w=n_w, n_A=n_a, n_B=n_b, n_orb=n_o)
    g_l, g_g, _, _, dh = inputs.stream_instance(5, p, dh_scale=0.05)
    nmap = build_neighbor_map(n_a, n_b)
    grid = default_grid(p)
    ch_l, ch_g = orc.pi_chains(g_l, g_g, dh, nmap.idx, np.array(grid.offsets), grid.energy_weight, n_qz)
    ref_l, ref_g = orc.pi_from_chains(ch_l, ch_g)
    outs = []
    for choice in ("4", "3", "2", "1", "0"):
        monkeypatch.setenv("SSE_PI_KERNEL", choice)
        out = sse_pi(GreensTensor(g_l, g_g), dh, nmap, grid, n_qz)
        assert orc.parity_dev(out.lesser, out.greater, ref_l, ref_g) <= TOL, choice
        outs.append(out)
    monkeypatch.setenv("SSE_PI_KERNEL", "3")
    monkeypatch.setenv("SSE_PI_PRODUCER", "1")  # v3 with the last releaser refilling
    outs.append(sse_pi(GreensTensor(g_l, g_g), dh, nmap, grid, n_qz))
    monkeypatch.delenv("SSE_PI_PRODUCER")
    for o in outs[1:]:
        assert np.array_equal(outs[0].lesser, o.lesser) and np.array_equal(outs[0].greater, o.greater)
    # the DFMA operand build (K5 v1; the DMMA build serves No % 4 == 0)
    monkeypatch.setenv("SSE_PI_KERNEL", "3")
    monkeypatch.setenv("SSE_PI_BUILD", "0")
    out = sse_pi(GreensTensor(g_l, g_g), dh, nmap, grid, n_qz)
    assert orc.parity_dev(out.lesser, out.greater, ref_l, ref_g) <= TOL


def test_pi_point_mask_and_atom_range():
    """The distributed schemes' options (sse.py:339-364): a (k, E) mask and an atom range."""
    p = SimParams(n_kz=2, n_qz=2, n_E=11, n_w=3, n_A=8, n_B=2, n_orb=3)
    g_l, g_g, _, _, dh = inputs.stream_instance(6, p)
    nmap = build_neighbor_map(p.n_A, p.n_B)
    grid = default_grid(p)
    mask = np.zeros((p.n_kz, p.n_E), dtype=bool)
    mask[:, 3:8] = True
    mask[1, 0] = True
    out = sse_pi(GreensTensor(g_l, g_g), dh, nmap, grid, p.n_qz, point_mask=mask, atom_range=(2, 6))
    ch_l, ch_g = orc.pi_chains(g_l, g_g, dh, nmap.idx, np.array(grid.offsets), grid.energy_weight, p.n_qz,
                               point_mask=mask, atom_range=(2, 6))
    ref_l, ref_g = orc.pi_from_chains(ch_l, ch_g)
    assert orc.parity_dev(out.lesser, out.greater, ref_l, ref_g) <= TOL
    assert np.all(out.lesser[:, :, :2] == 0) and np.all(out.greater[:, :, 6:] == 0)
    with pytest.raises(ValueError, match="point mask must have shape"):
        sse_pi(GreensTensor(g_l, g_g), dh, nmap, grid, p.n_qz, point_mask=mask[:, :5])


def test_pi_rejects_phonon_tensor():
    c = load_case("test_tiny_s3")
    with pytest.raises(ValueError, match="expects the electron Green's tensor"):
        sse_pi(GreensTensor(c.d_l, c.d_g), c.dh, NeighborMap(c.idx), _grid(c), c.p.n_qz)


def test_pi_multi_gpu_bitwise():
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    c = load_case("cli_small_s2")
    args = (GreensTensor(c.g_l, c.g_g), c.dh, NeighborMap(c.idx), _grid(c), c.p.n_qz)
    a = sse_pi(*args, n_gpus=1)
    b = sse_pi(*args, n_gpus=2)
    assert np.array_equal(a.lesser, b.lesser) and np.array_equal(a.greater, b.greater)


def test_pi_device_api_slab_bitwise():
    """Owned-range shard with halo (atom-major) equals the host call bitwise."""
    import torch

    from paper_1912_08810_b200 import sse as dev

    p = SimParams(n_kz=3, n_qz=3, n_E=20, n_w=6, n_A=10, n_B=4, n_orb=12)
    g_l, g_g, _, _, dh = inputs.stream_instance(8, p, dh_scale=0.05)
    nmap = build_neighbor_map(p.n_A, p.n_B)
    grid = default_grid(p)
    full = sse_pi(GreensTensor(g_l, g_g), dh, nmap, grid, p.n_qz)
    lo, hi = 3, 7
    glo, ghi = int(nmap.idx[lo:hi].min()), int(nmap.idx[lo:hi].max()) + 1
    glo, ghi = min(glo, lo), max(ghi, hi)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    gl = cu(np.moveaxis(g_l[:, :, glo:ghi], 2, 0))
    gg = cu(np.moveaxis(g_g[:, :, glo:ghi], 2, 0))
    shape = (p.n_qz, p.n_w, hi - lo, p.n_B + 1, 3, 3)
    pl = torch.zeros(shape, dtype=torch.complex128, device="cuda")
    pg = torch.zeros_like(pl)
    dev.pi_device(gl, gg, cu(dh[lo:hi]), nmap.idx[lo:hi], grid.offsets, grid.energy_weight, pl, pg,
                  n_a=p.n_A, n_qz=p.n_qz, g_atom0=glo, out_atom0=lo, atom_major=True)
    torch.cuda.synchronize()
    assert np.array_equal(pl.cpu().numpy(), full.lesser[:, :, lo:hi])
    assert np.array_equal(pg.cpu().numpy(), full.greater[:, :, lo:hi])


def test_pi_split_lag_tiles_bitwise(monkeypatch):
    """Paper shapes with 9 lag tiles (Nw in 65..72): K6 v4 runs tiles 0..7 with 4 warps per CTA plus a
    tail CTA computing the 9th tile of every q; bitwise equal to the unsplit v4 and to v3."""
    p = SimParams(n_kz=5, n_qz=5, n_E=72, n_w=66, n_A=5, n_B=4, n_orb=12)  # Nqz = 5: two tail q-groups
    g_l, g_g, _, _, dh = inputs.stream_instance(8, p, dh_scale=0.05)
    nmap = build_neighbor_map(p.n_A, p.n_B)
    grid = default_grid(p)
    outs = []
    for kernel, warps in (("4", None), ("4", "5"), ("3", None)):
        monkeypatch.setenv("SSE_PI_KERNEL", kernel)
        if warps:
            monkeypatch.setenv("SSE_PI_V4_WARPS", warps)
        else:
            monkeypatch.delenv("SSE_PI_V4_WARPS", raising=False)
        outs.append(sse_pi(GreensTensor(g_l, g_g), dh, nmap, grid, p.n_qz))
    for o in outs[1:]:
        assert np.array_equal(outs[0].lesser, o.lesser) and np.array_equal(outs[0].greater, o.greater)
    assert np.abs(outs[0].lesser).max() > 0


def test_ctx_trim_then_recompute_bitwise():
    """sse_ctx_trim hands the cached scratch back (Pi operand buffers, staging ring); the next calls
    allocate again and give bit-identical Pi and Sigma."""
    from paper_1912_08810_b200 import _lib
    from paper_1912_08810_b200.sse import sse_sigma
    from paper_1912_08810_b200.types import CombinedD, SseVariant

    p = SimParams(n_kz=3, n_qz=3, n_E=30, n_w=12, n_A=5, n_B=4, n_orb=12)
    g_l, g_g, d_l, d_g, dh = inputs.stream_instance(6, p, dh_scale=0.05)
    nmap = build_neighbor_map(p.n_A, p.n_B)
    grid = default_grid(p)
    dc = CombinedD(*orc.preprocess_D(d_l, d_g, nmap.idx))
    runs = []
    for _ in range(2):
        pi = sse_pi(GreensTensor(g_l, g_g), dh, nmap, grid, p.n_qz)
        sig = sse_sigma(SseVariant.BATCHED_FUSED, GreensTensor(g_l, g_g), dc, dh, nmap, grid)
        runs.append((pi, sig))
        for ctx in list(_lib._contexts.values()):  # whichever contexts the drop-ins used
            ctx.trim()
    (pa, sa), (pb, sb) = runs
    assert np.array_equal(pa.lesser, pb.lesser) and np.array_equal(pa.greater, pb.greater)
    assert np.array_equal(sa.lesser, sb.lesser) and np.array_equal(sa.greater, sb.greater)
