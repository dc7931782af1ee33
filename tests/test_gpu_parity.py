"""Parity of the CUDA path (through the C ABI) with the reference's outputs.

Tolerance: the reference's own metric, max|out - ref| / max(max|ref<|, max|ref>|)
<= 1e-10 in complex128 (BASELINE.json north_star; test_acceptance.py:162-171).
Golden outputs come from the reference itself (tests/golden/make_golden.py).
"""

import numpy as np
import pytest

from oracle import sse_oracle as orc
from paper_1912_08810_b200 import inputs
from paper_1912_08810_b200.sse import sse_sigma
from paper_1912_08810_b200.types import (
    CombinedD,
    EnergyGrid,
    FlopCounter,
    GreensTensor,
    NeighborMap,
    SimParams,
    SseVariant,
    build_neighbor_map,
    default_grid,
)
from tests.golden_cases import criterion5_instances, kat_scalar, load_case, stream_case_names

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _grid(case):
    n_e = case.p.n_E
    return EnergyGrid(
        values=tuple(np.linspace(-1, 1, n_e)) if n_e > 1 else (0.0,),
        frequency_map=tuple(zip(case.offsets.tolist(), case.weights.tolist())),
        energy_weight=1.0,
    )


def _dc(case):
    return CombinedD(*orc.preprocess_D(case.d_l, case.d_g, case.idx))


@pytest.fixture(scope="module", params=stream_case_names())
def case(request):
    c = load_case(request.param)
    assert c.inputs_ok
    return c


@pytest.mark.parametrize("variant", list(SseVariant))
def test_golden_parity_all_variants(case, variant):
    counter = FlopCounter()
    out = sse_sigma(variant, GreensTensor(case.g_l, case.g_g), _dc(case), case.dh, NeighborMap(case.idx),
                    _grid(case), counter=counter)
    dev = orc.parity_dev(out.lesser, out.greater, case.arrays["sigma_l"], case.arrays["sigma_g"])
    assert dev <= TOL, (case.name, variant, dev)
    p = case.p
    assert counter.stages == orc.sigma_tallies(variant.value, p.n_kz, p.n_qz, p.n_E, p.n_w, p.n_A, p.n_B,
                                               p.n_orb)


def test_kat_scalar():
    g_l, g_g, dc_l, dc_g, dh, idx, off, wt, ref_l, ref_g = kat_scalar()
    grid = EnergyGrid(values=(0.0,), frequency_map=((0, 0.37),), energy_weight=1.0)
    out = sse_sigma(SseVariant.REFERENCE, GreensTensor(g_l, g_g), CombinedD(dc_l, dc_g), dh, NeighborMap(idx), grid)
    assert np.max(np.abs(out.lesser - ref_l)) <= 1e-13 * np.max(np.abs(ref_l))
    assert np.max(np.abs(out.greater - ref_g)) <= 1e-13 * np.max(np.abs(ref_g))


def test_criterion5_fifty_instances_all_variants():
    worst = 0.0
    for p, grid, nmap, g_l, g_g, d_l, d_g, dh, ref_l, ref_g in criterion5_instances():
        dc = CombinedD(*orc.preprocess_D(d_l, d_g, nmap.idx))
        for variant in SseVariant:
            out = sse_sigma(variant, GreensTensor(g_l, g_g), dc, dh, nmap, grid)
            worst = max(worst, orc.parity_dev(out.lesser, out.greater, ref_l, ref_g))
    assert worst <= TOL


def test_zero_phonon_input_gives_exact_zero():
    """test_sse.py:165-172."""
    c = load_case("test_tiny_s3")
    zero = CombinedD(np.zeros(c.p.combined_shape, complex), np.zeros(c.p.combined_shape, complex))
    out = sse_sigma(SseVariant.BATCHED_FUSED, GreensTensor(c.g_l, c.g_g), zero, c.dh, NeighborMap(c.idx), _grid(c))
    assert np.all(out.lesser == 0) and np.all(out.greater == 0)


def test_linearity_in_g_and_dc():
    """test_sse.py:253-272 at the kernel's No=12 shape."""
    c = load_case("orb12_s5")
    rng = np.random.default_rng(42)
    z = lambda s: rng.standard_normal(s) + 1j * rng.standard_normal(s)  # noqa: E731
    nmap, grid, dc = NeighborMap(c.idx), _grid(c), _dc(c)
    g2 = GreensTensor(z(c.g_l.shape), z(c.g_g.shape))
    d2 = CombinedD(z(dc.lesser.shape), z(dc.greater.shape))

    def run(g, d):
        return sse_sigma(SseVariant.BATCHED_FUSED, g, d, c.dh, nmap, grid).lesser

    g1 = GreensTensor(c.g_l, c.g_g)
    lhs = run(GreensTensor(c.g_l + g2.lesser, c.g_g + g2.greater), dc)
    rhs = run(g1, dc) + run(g2, dc)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.max(np.abs(rhs))
    lhs = run(g1, CombinedD(dc.lesser + d2.lesser, dc.greater + d2.greater))
    rhs = run(g1, dc) + run(g1, d2)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.max(np.abs(rhs))


def test_deterministic_bitwise():
    c = load_case("orb10_s6")
    args = (GreensTensor(c.g_l, c.g_g), _dc(c), c.dh, NeighborMap(c.idx), _grid(c))
    a = sse_sigma(SseVariant.BATCHED_FUSED, *args)
    b = sse_sigma(SseVariant.BATCHED_FUSED, *args)
    assert np.array_equal(a.lesser, b.lesser) and np.array_equal(a.greater, b.greater)


@pytest.mark.parametrize("name", ["orb10_s6", "orb12_s5", "cli_small_s2", "general_grid_s8", "slide_orb12_s9",
                                  "slide_orb10_s10", "paperlike_w70_s11"])
def test_all_sigma_kernels_bitwise(monkeypatch, name):
    """Every K3 kernel (simple, pipelined, TMA sliding-window) accumulates in the
    same (q, s, w, k-step) order: outputs are bitwise equal (the general grid's
    non-sliding offsets route the TMA choice to the pipelined kernel)."""
    c = load_case(name)
    args = (GreensTensor(c.g_l, c.g_g), _dc(c), c.dh, NeighborMap(c.idx), _grid(c))
    outs = []
    for choice in ("0", "1", "3", "4"):
        monkeypatch.setenv("SSE_SIGMA_KERNEL", choice)
        outs.append(sse_sigma(SseVariant.BATCHED_FUSED, *args))
    for o in outs[1:]:
        assert np.array_equal(outs[0].lesser, o.lesser) and np.array_equal(outs[0].greater, o.greater)
    dev = orc.parity_dev(outs[0].lesser, outs[0].greater, c.arrays["sigma_l"], c.arrays["sigma_g"])
    assert dev <= TOL


@pytest.mark.parametrize("n_e, n_w, n_o, n_a, n_b", [
    (24, 6, 12, 10, 4),    # the smoke shape: 6 offsets < 12 ring stages (pipelined fallback)
    (48, 12, 12, 6, 4),    # sliding-window kernel, one CTA tile, segments of exactly 12 stages
    (64, 20, 12, 5, 4),    # sliding-window kernel, two CTA tiles, window clipped at E = 0
    (25, 12, 12, 5, 4),    # sliding-window tail CTA: 12 rows, interleaved tiles, a partial tile
    (41, 14, 12, 5, 4),    # sliding-window tail CTA: 204 rows (warps with 3 / 2 valid tiles, partial tile)
    (40, 13, 10, 6, 4),    # No = 10: interleaved-K embedding (K' = 20), sliding window with a 72-slot FIFO
    (33, 12, 6, 5, 4),     # No = 6: interleaved K, odd k-step count (3), sliding window
    (19, 12, 2, 5, 2),     # No = 2: interleaved K, one k-step
    (24, 12, 14, 5, 4),    # No = 14: interleaved K (K' = 28), ring too large: pipelined kernel
    (300, 16, 10, 3, 2),   # No = 10 at the small config's NE / Nw: 11 row CTAs per (atom, k), tail CTA
    (31, 16, 4, 7, 4),     # No = 4, ragged last tile
    (30, 14, 12, 9, 6),    # NB = 6 neighbour slots
    (20, 13, 17, 5, 2),    # No = 17 > 16: the DFMA kernel (K3g)
])
def test_kernel_shapes_against_oracle(monkeypatch, n_e, n_w, n_o, n_a, n_b):
    """Shapes that exercise the K3 ring/window logic, checked against the oracle
    (pinned to the reference by tests/test_oracle.py) for every kernel choice."""
    p = SimParams(n_kz=3, n_qz=2, n_E=n_e, n_w=n_w, n_A=n_a, n_B=n_b, n_orb=n_o)
    g_l, g_g, d_l, d_g, dh = inputs.stream_instance(11, p, dh_scale=0.05)
    nmap = build_neighbor_map(p.n_A, p.n_B)
    grid = default_grid(p)
    dc = CombinedD(*orc.preprocess_D(d_l, d_g, nmap.idx))
    off, wt = np.array(grid.offsets), np.array(grid.weights)
    ref_l, ref_g = orc.sigma_batched_fused(g_l, g_g, dc.lesser, dc.greater, dh, nmap.idx, off, wt)
    outs = []
    for choice in ("0", "1", "3", "4"):
        monkeypatch.setenv("SSE_SIGMA_KERNEL", choice)
        out = sse_sigma(SseVariant.BATCHED_FUSED, GreensTensor(g_l, g_g), dc, dh, nmap, grid)
        assert orc.parity_dev(out.lesser, out.greater, ref_l, ref_g) <= TOL, choice
        outs.append(out)
    for o in outs[1:]:
        assert np.array_equal(outs[0].lesser, o.lesser) and np.array_equal(outs[0].greater, o.greater)


@pytest.mark.parametrize("n_kz, n_qz, n_e, n_w, n_o, n_a", [
    (5, 3, 30, 8, 12, 5),   # K3m No = 12, odd Nkz: group {0,1} then one 3-momentum group {2,3,4} (2 row tiles); Nqz < Nkz
    (3, 3, 41, 12, 12, 5),  # the paper's Nkz = Nqz = 3: one 3-momentum launch; 492 rows = 2 full + 1 partial CTA
    (4, 4, 26, 7, 10, 5),   # combined fragments (No = 10): groups {0,1,2}, {3 + 2 padded momenta}
    (1, 1, 20, 8, 12, 5),   # Nkz = 1: a single-momentum launch
    (7, 2, 22, 6, 4, 5),    # No = 4 (kg 3): groups {0,1,2}, {3,4,5}, remainder {6}; Nqz = 2 (most M vectors zero)
    (2, 2, 33, 9, 6, 5),    # No = 6 combined, Nkz = 2: one padded group
])
def test_multi_momentum_groups_against_oracle(monkeypatch, n_kz, n_qz, n_e, n_w, n_o, n_a):
    """K3m's momentum grouping (full groups, remainder launches, padded combined groups, zero M
    vectors for q >= Nqz) against the oracle, and bitwise equal to the single-momentum kernels."""
    p = SimParams(n_kz=n_kz, n_qz=n_qz, n_E=n_e, n_w=n_w, n_A=n_a, n_B=4, n_orb=n_o)
    g_l, g_g, d_l, d_g, dh = inputs.stream_instance(13, p, dh_scale=0.05)
    nmap = build_neighbor_map(p.n_A, p.n_B)
    grid = default_grid(p)
    dc = CombinedD(*orc.preprocess_D(d_l, d_g, nmap.idx))
    off, wt = np.array(grid.offsets), np.array(grid.weights)
    ref_l, ref_g = orc.sigma_batched_fused(g_l, g_g, dc.lesser, dc.greater, dh, nmap.idx, off, wt)
    from paper_1912_08810_b200 import _lib

    outs = []
    for choice in ("4", "1"):
        monkeypatch.setenv("SSE_SIGMA_KERNEL", choice)
        out = sse_sigma(SseVariant.BATCHED_FUSED, GreensTensor(g_l, g_g), dc, dh, nmap, grid)
        if choice == "4":
            assert _lib.kernel_name("sigma").startswith("sigma_dmma_kslide_kernel"), _lib.kernel_name("sigma")
        assert orc.parity_dev(out.lesser, out.greater, ref_l, ref_g) <= TOL, choice
        outs.append(out)
    assert np.array_equal(outs[0].lesser, outs[1].lesser) and np.array_equal(outs[0].greater, outs[1].greater)
    if n_o == 12 and n_kz % 2 == 1 and n_kz >= 3:  # the plain groups of 2 + a 1-momentum remainder agree bitwise
        monkeypatch.setenv("SSE_SIGMA_KERNEL", "4")
        monkeypatch.setenv("SSE_K3M_MT", "3")
        out = sse_sigma(SseVariant.BATCHED_FUSED, GreensTensor(g_l, g_g), dc, dh, nmap, grid)
        assert "<12,12,3,1>" in _lib.kernel_name("sigma"), _lib.kernel_name("sigma")
        assert np.array_equal(outs[0].lesser, out.lesser) and np.array_equal(outs[0].greater, out.greater)


def test_layout_transformed_equals_grid_major_bitwise():
    """K1 round trip is lossless and the atom-major accumulation has the same order."""
    c = load_case("orb12_s5")
    args = (GreensTensor(c.g_l, c.g_g), _dc(c), c.dh, NeighborMap(c.idx), _grid(c))
    a = sse_sigma(SseVariant.BATCHED_FUSED, *args)
    b = sse_sigma(SseVariant.LAYOUT_TRANSFORMED, *args)
    assert np.array_equal(a.lesser, b.lesser) and np.array_equal(a.greater, b.greater)


def test_multi_gpu_split_is_bitwise_identical():
    import torch

    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    c = load_case("cli_small_s2")
    args = (GreensTensor(c.g_l, c.g_g), _dc(c), c.dh, NeighborMap(c.idx), _grid(c))
    a = sse_sigma(SseVariant.BATCHED_FUSED, *args, n_gpus=1)
    for k in range(2, n + 1):
        b = sse_sigma(SseVariant.BATCHED_FUSED, *args, n_gpus=k)
        assert np.array_equal(a.lesser, b.lesser) and np.array_equal(a.greater, b.greater)


def test_timing_and_launch_accounting():
    c = load_case("orb12_s5")
    timing = {}
    sse_sigma(SseVariant.BATCHED_FUSED, GreensTensor(c.g_l, c.g_g), _dc(c), c.dh, NeighborMap(c.idx),
              _grid(c), timing=timing)
    assert timing["kernel_launches"] >= 2
    assert timing["h2d_bytes"] > 2 * c.g_l.nbytes
    assert timing["d2h_bytes"] == 2 * c.g_l.nbytes
    assert timing["flops"] > 0


def test_invalid_neighbor_index_raises_value_error():
    c = load_case("test_tiny_s3")
    bad = c.idx.copy()
    bad[0, 0] = c.p.n_A
    with pytest.raises(ValueError):
        sse_sigma(SseVariant.REFERENCE, GreensTensor(c.g_l, c.g_g), _dc(c), c.dh, NeighborMap(bad), _grid(c))


# ---------------------------------------------------------------------------
# device-resident API
# ---------------------------------------------------------------------------


def _torch():
    import torch

    return torch


def test_device_api_slabs_and_layouts_bitwise():
    """Owned-range shards with halos, grid- and atom-major, equal the full call bitwise."""
    torch = _torch()
    from paper_1912_08810_b200 import sse as dev

    c = load_case("orb12_s5")
    p = c.p
    dc = _dc(c)
    full = sse_sigma(SseVariant.BATCHED_FUSED, GreensTensor(c.g_l, c.g_g), dc, c.dh, NeighborMap(c.idx), _grid(c))
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    for lo, hi in ((0, 3), (3, 6), (2, 4)):
        need = c.idx[lo:hi]
        glo, ghi = int(need.min()), int(need.max()) + 1
        for atom_major in (False, True):
            gl, gg = c.g_l[:, :, glo:ghi], c.g_g[:, :, glo:ghi]
            if atom_major:
                gl, gg = np.moveaxis(gl, 2, 0), np.moveaxis(gg, 2, 0)
            gl, gg = cu(gl), cu(gg)
            shape = (hi - lo, p.n_kz, p.n_E, p.n_orb, p.n_orb) if atom_major else (p.n_kz, p.n_E, hi - lo, p.n_orb, p.n_orb)
            ol = torch.zeros(shape, dtype=torch.complex128, device="cuda")
            og = torch.zeros_like(ol)
            dev.sigma_device(gl, gg, cu(dc.lesser[:, :, lo:hi]), cu(dc.greater[:, :, lo:hi]), cu(c.dh[lo:hi]),
                             need, c.offsets, c.weights, ol, og, n_a=p.n_A, g_atom0=glo, out_atom0=lo,
                             atom_major=atom_major)
            torch.cuda.synchronize()
            got_l, got_g = ol.cpu().numpy(), og.cpu().numpy()
            if atom_major:
                got_l, got_g = np.moveaxis(got_l, 0, 2), np.moveaxis(got_g, 0, 2)
            assert np.array_equal(got_l, full.lesser[:, :, lo:hi])
            assert np.array_equal(got_g, full.greater[:, :, lo:hi])


def test_layout_transform_kernel_bitwise():
    torch = _torch()
    from paper_1912_08810_b200 import sse as dev

    c = load_case("orb10_s6")
    g = torch.from_numpy(c.g_l).cuda()
    am = torch.empty((c.p.n_A, c.p.n_kz, c.p.n_E, c.p.n_orb, c.p.n_orb), dtype=torch.complex128, device="cuda")
    back = torch.empty_like(g)
    dev.layout_transform(g, am, to_atom_major=True)
    dev.layout_transform(am, back, to_atom_major=False)
    torch.cuda.synchronize()
    assert np.array_equal(am.cpu().numpy(), np.moveaxis(c.g_l, 2, 0))
    assert np.array_equal(back.cpu().numpy(), c.g_l)
    # the phonon tensor D[qz, w, atom, neighbour, 3, 3] -> atom-major (north_star item 1)
    d = torch.from_numpy(c.d_l).cuda()
    dam = torch.empty((c.p.n_A, c.p.n_qz, c.p.n_w, c.p.n_B + 1, 3, 3), dtype=torch.complex128, device="cuda")
    dback = torch.empty_like(d)
    dev.layout_transform(d, dam, to_atom_major=True)
    dev.layout_transform(dam, dback, to_atom_major=False)
    torch.cuda.synchronize()
    assert np.array_equal(dam.cpu().numpy(), np.moveaxis(c.d_l, 2, 0))
    assert np.array_equal(dback.cpu().numpy(), c.d_l)


def test_preprocess_D_device_bitwise():
    torch = _torch()
    from paper_1912_08810_b200 import sse as dev

    for name in ("cli_small_s2", "orb10_s6", "orb5_nb1_s7"):
        c = load_case(name)
        ref_l, _ = orc.preprocess_D(c.d_l, c.d_g, c.idx)
        out = torch.empty(ref_l.shape, dtype=torch.complex128, device="cuda")
        dev.preprocess_D_device(torch.from_numpy(c.d_l).cuda(), out, c.idx)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), ref_l), name


def test_preprocess_D_device_missing_slot():
    torch = _torch()
    from paper_1912_08810_b200 import sse as dev

    idx = np.array([[1], [0], [1]], dtype=np.int64)
    d = torch.ones((1, 1, 3, 2, 3, 3), dtype=torch.complex128, device="cuda")
    with pytest.raises(ValueError, match="missing neighbor slot"):
        dev.preprocess_D_device(d, torch.empty((1, 1, 3, 1, 3, 3), dtype=torch.complex128, device="cuda"), idx)


def test_fill_synthetic_matches_host_generator_bitwise():
    torch = _torch()
    from paper_1912_08810_b200 import sse as dev

    p = SimParams(n_kz=2, n_qz=2, n_E=5, n_w=2, n_A=7, n_B=2, n_orb=3)
    g = torch.empty(p.electron_shape, dtype=torch.complex128, device="cuda")
    no2 = p.n_orb**2
    dev.fill_synthetic(g, 11, inputs.G_LESSER, 0, p.n_A, p.n_kz * p.n_E, no2, no2, p.n_A * no2)
    torch.cuda.synchronize()
    host = inputs.atom_keyed_electron(11, inputs.G_LESSER, p, np.arange(p.n_A))
    assert np.array_equal(g.cpu().numpy(), host)
    # a slab of atoms [2, 5) holds the same values as the full tensor
    s = torch.empty((p.n_kz, p.n_E, 3, p.n_orb, p.n_orb), dtype=torch.complex128, device="cuda")
    dev.fill_synthetic(s, 11, inputs.G_LESSER, 2, 3, p.n_kz * p.n_E, no2, no2, 3 * no2)
    torch.cuda.synchronize()
    assert np.array_equal(s.cpu().numpy(), host[:, :, 2:5])
    dh = torch.empty(p.dh_shape, dtype=torch.complex128, device="cuda")
    inner = p.n_B * 3 * no2
    dev.fill_synthetic(dh, 11, inputs.DH, 0, p.n_A, 1, inner, inner, 0, scale=inputs.DH_SCALE)
    torch.cuda.synchronize()
    assert np.array_equal(dh.cpu().numpy(), inputs.atom_keyed_dh(11, p, np.arange(p.n_A)))


# ---------------------------------------------------------------------------
# BASELINE configs at full size: sampled points vs the pointwise oracle
# ---------------------------------------------------------------------------


def _full_scale_points(name, seed, points_per_atom, atoms):
    """Device-resident full-config Sigma; sampled (atom, k, E) blocks vs oracle."""
    torch = _torch()
    from tests.scale_helpers import DeviceProblem, host_point

    prob = DeviceProblem(name, seed)
    prob.run()
    p = prob.p
    rng = np.random.default_rng(seed)
    worst = 0.0
    for a in atoms:
        es = sorted({0, 1, p.n_E - 1, int(prob.offsets.max()), *rng.integers(0, p.n_E, points_per_atom).tolist()})
        for e in es:
            k = int(rng.integers(0, p.n_kz))
            for pol in (0, 1):
                got = prob.sigma_block(pol, k, e, a)
                ref = host_point(prob, pol, k, e, a)
                scale = max(np.max(np.abs(ref)), 1e-300)
                worst = max(worst, float(np.max(np.abs(got - ref)) / scale))
    prob.free()
    torch.cuda.empty_cache()
    return worst


def test_small_config_sampled_points():
    p = inputs.CONFIGS["small"]
    dev = _full_scale_points("small", 0, 6, [0, 1, 2, p.n_A // 2, p.n_A - 2, p.n_A - 1])
    assert dev <= TOL


@pytest.mark.slow
def test_paper_config_sampled_points():
    p = inputs.CONFIGS["paper"]
    dev = _full_scale_points("paper", 0, 4, [0, 1, 2, 2431, p.n_A - 2, p.n_A - 1])
    assert dev <= TOL


def _sharded_points(name, world, ranks, atoms_per_shard=3, points=3, seed=0):
    """Shards of a config too large for one B200, run one after another on cuda:0.

    Each shard is a rank's share of a `world`-way atom sharding (owned atoms + the +-reach halo,
    filled locally from the atom-keyed generator, exactly the slab the multi-GPU run computes);
    sampled blocks of the first / last owned atoms and random ones are checked against the
    pointwise oracle (oracle.sigma_point, pinned to the reference in tests/test_oracle.py).
    """
    torch = _torch()
    from tests.scale_helpers import DeviceProblem, host_point

    rng = np.random.default_rng(seed)
    worst = 0.0
    for r in ranks:
        sh = DeviceProblem(name, seed, world, r, device=0)
        sh.run()
        p = sh.p
        atoms = {sh.lo, sh.hi - 1, *rng.integers(sh.lo, sh.hi, atoms_per_shard - 2).tolist()}
        for a in sorted(atoms):
            for e in sorted({0, p.n_E - 1, int(sh.offsets.max()), *rng.integers(0, p.n_E, points).tolist()}):
                k = int(rng.integers(0, p.n_kz))
                for pol in (0, 1):
                    got = sh.sigma_block(pol, k, e, a)
                    ref = host_point(sh, pol, k, e, a)
                    worst = max(worst, float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300)))
        sh.free()
        del sh
        torch.cuda.empty_cache()
    return worst


@pytest.mark.slow
def test_kheavy_config_sampled_points():
    """Nkz = Nqz = 7 (k - q wrap over 7 momenta), 221.5 GB in total: the first and last of its
    4-way atom shards (55 GB each) on one B200, chain ends included."""
    assert _sharded_points("kheavy", 4, (0, 3)) <= TOL


@pytest.mark.slow
def test_large_config_sampled_points():
    """NA = 10,240, NE = 1,220, Nkz = Nqz = 5, 575.7 GB in total: three of its 8-way atom shards
    (72 GB each; the 8-GPU run's per-GPU share) on one B200, chain ends included."""
    assert _sharded_points("large", 8, (0, 4, 7)) <= TOL


@pytest.mark.parametrize("mode", ["0", "1", "auto"])
def test_host_staging_ring_bitwise(monkeypatch, mode):
    """The pageable-memory staging ring (SSE_HOST_STAGING auto/1: host worker pool packs and
    unpacks pinned double buffers) and direct DMA (0) give the same bits as the device-resident
    call, over many pipeline chunks (ramped chunk sizes, halo columns, both polarities)."""
    torch = _torch()
    from paper_1912_08810_b200 import sse as dev

    p = SimParams(n_kz=3, n_qz=3, n_E=40, n_w=14, n_A=150, n_B=4, n_orb=12)
    g_l, g_g, d_l, d_g, dh = inputs.stream_instance(21, p, dh_scale=0.05)
    nmap = build_neighbor_map(p.n_A, p.n_B)
    grid = default_grid(p)
    dc = CombinedD(*orc.preprocess_D(d_l, d_g, nmap.idx))
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    ref = [torch.zeros(p.electron_shape, dtype=torch.complex128, device="cuda") for _ in range(2)]
    dev.sigma_device(cu(g_l), cu(g_g), cu(dc.lesser), cu(dc.greater), cu(dh), nmap.idx, grid.offsets,
                     grid.weights, ref[0], ref[1], n_a=p.n_A)
    torch.cuda.synchronize()
    ref = [r.cpu().numpy() for r in ref]
    monkeypatch.setenv("SSE_OP_CHUNK_ATOMS", "16")
    if mode != "auto":
        monkeypatch.setenv("SSE_HOST_STAGING", mode)
    timing = {}
    out = sse_sigma(SseVariant.BATCHED_FUSED, GreensTensor(g_l, g_g), dc, dh, nmap, grid, timing=timing)
    assert np.array_equal(out.lesser, ref[0]) and np.array_equal(out.greater, ref[1])
    assert timing["staged"] == (0 if mode == "0" else 3)
    # pinned caller buffers take the direct path in auto mode
    if mode == "auto":
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        o = [torch.empty(p.electron_shape, dtype=torch.complex128, pin_memory=True) for _ in range(2)]
        tim = dev.sigma_host_slab(pin(g_l), pin(g_g), pin(dc.lesser), pin(dc.greater), pin(dh), nmap.idx,
                                  grid.offsets, grid.weights, o[0], o[1], n_a=p.n_A, g_atom0=0, out_atom0=0)
        assert tim["staged"] == 0
        assert np.array_equal(o[0].numpy(), ref[0]) and np.array_equal(o[1].numpy(), ref[1])


def test_in_library_multi_gpu_sigma_bitwise():
    """sse_sigma_multi: one call over all devices of the process, halos exchanged by the library
    with NCCL (ncclCommInitAll) -- equal bit for bit to the single-device call; on one GPU it
    runs the same path without communication."""
    torch = _torch()
    from paper_1912_08810_b200 import sse as dev

    n = torch.cuda.device_count()
    c = load_case("slide_orb12_s9")
    p = c.p
    dc = _dc(c)
    full = sse_sigma(SseVariant.BATCHED_FUSED, GreensTensor(c.g_l, c.g_g), dc, c.dh, NeighborMap(c.idx), _grid(c))
    for ngpu in sorted({1, min(n, 2), n}):
        lay = dev.multi_layout(ngpu, c.idx)
        cu = lambda a, i: torch.from_numpy(np.ascontiguousarray(a)).to(f"cuda:{i}")  # noqa: E731
        g_l, g_g, dl, dg, dh, ol, og = [], [], [], [], [], [], []
        for i, (lo, hi, glo, ghi) in enumerate(lay):
            for src, dst in ((c.g_l, g_l), (c.g_g, g_g)):
                slab = np.full((ghi - glo, p.n_kz, p.n_E, p.n_orb, p.n_orb), np.nan, dtype=np.complex128)
                slab[lo - glo:hi - glo] = np.moveaxis(src[:, :, lo:hi], 2, 0)  # owned atoms only: halo by NCCL
                dst.append(cu(slab, i))
            dl.append(cu(dc.lesser[:, :, lo:hi], i))
            dg.append(cu(dc.greater[:, :, lo:hi], i))
            dh.append(cu(c.dh[lo:hi], i))
            ol.append(torch.zeros((hi - lo, p.n_kz, p.n_E, p.n_orb, p.n_orb), dtype=torch.complex128, device=f"cuda:{i}"))
            og.append(torch.zeros_like(ol[-1]))
        dev.sigma_multi(g_l, g_g, dl, dg, dh, c.idx, _grid(c), ol, og, sync_timing=True)
        for i, (lo, hi, _, _) in enumerate(lay):
            assert np.array_equal(np.moveaxis(ol[i].cpu().numpy(), 0, 2), full.lesser[:, :, lo:hi]), (ngpu, i)
            assert np.array_equal(np.moveaxis(og[i].cpu().numpy(), 0, 2), full.greater[:, :, lo:hi]), (ngpu, i)


def test_device_wrappers_reject_mismatched_tensors():
    """The C side sees raw pointers only, so the device wrappers check every tensor's shape, dtype
    and device before the call (a mismatch raises ValueError instead of an out-of-bounds access)."""
    torch = _torch()
    from paper_1912_08810_b200 import sse as dev

    c = load_case("orb12_s5")
    p = c.p
    dc = _dc(c)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    gl, gg = cu(c.g_l), cu(c.g_g)
    ol = torch.zeros(p.electron_shape, dtype=torch.complex128, device="cuda")
    og = torch.zeros_like(ol)
    args = dict(n_a=p.n_A)
    with pytest.raises(ValueError, match="out_g"):
        dev.sigma_device(gl, gg, cu(dc.lesser), cu(dc.greater), cu(c.dh), c.idx, c.offsets, c.weights, ol,
                         og[:, :, :-1].contiguous(), **args)
    with pytest.raises(ValueError, match="complex128"):
        dev.sigma_device(gl, gg.to(torch.complex64), cu(dc.lesser), cu(dc.greater), cu(c.dh), c.idx, c.offsets,
                         c.weights, ol, og, **args)
    with pytest.raises(ValueError, match="dst"):
        dev.layout_transform(gl, torch.empty((1, 2, 3), dtype=torch.complex128, device="cuda"), to_atom_major=True)
    pi = [torch.zeros((p.n_qz, p.n_w, p.n_A, p.n_B + 1, 3, 3), dtype=torch.complex128, device="cuda") for _ in range(2)]
    with pytest.raises(ValueError, match="pi_g"):
        dev.pi_device(gl, gg, cu(c.dh), c.idx, c.offsets, 0.1, pi[0], pi[1][:, :1].contiguous(), n_a=p.n_A,
                      n_qz=p.n_qz)
    with pytest.raises(ValueError, match="overruns"):
        dev.fill_synthetic(ol, 0, 0, 0, p.n_A + 1, p.n_kz * p.n_E, p.n_orb**2, p.n_orb**2, p.n_A * p.n_orb**2)
