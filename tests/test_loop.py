"""The self-consistent Born loop with the fused SSE phase.

The golden traces (tests/golden/make_loop_golden.py) hold what the reference's
``gf_phase`` returned at each iteration of the reference's own
``self_consistent_loop`` (sse.py:495-535) and the self-energies it was handed.
Replaying the recorded GF outputs through ``paper_1912_08810_b200.loop``
checks every SSE phase against the reference's and the loop bookkeeping
(deltas, iteration count, final record).  The CPU test runs the loop with the
oracle standing in for the device phase (loop logic only); the GPU tests run
``sse_phase`` through libsse and compare it with the three separate calls.
Tolerance: the reference metric <= 1e-10.
"""

import json
import os
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import sse_oracle as orc
from paper_1912_08810_b200 import loop as b200_loop
from paper_1912_08810_b200.types import (
    EnergyGrid,
    GreensTensor,
    NeighborMap,
    SelfEnergyTensor,
    SimParams,
)

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = 1e-10


def _load(preset):
    data = np.load(os.path.join(HERE, f"loop_{preset}.npz"))
    meta = json.loads(str(data["meta"]))
    p = SimParams(**meta["params"])
    grid = EnergyGrid(values=tuple(np.linspace(-1, 1, p.n_E)),
                      frequency_map=tuple(zip(meta["offsets"], meta["weights"])),
                      energy_weight=meta["energy_weight"])
    return data, meta, p, grid, NeighborMap(np.array(data["nmap"]))


def oracle_phase(g_e, g_ph, dh, nmap, grid, n_qz, **_):
    """preprocess_D + sse_sigma + sse_pi on the CPU oracle (test stand-in for sse_phase)."""
    off = np.array(grid.offsets)
    wt = np.array([w for _, w in grid.frequency_map])
    dc_l, dc_g = orc.preprocess_D(g_ph.lesser, g_ph.greater, nmap.idx)
    s_l, s_g = orc.sigma_batched_fused(g_e.lesser, g_e.greater, dc_l, dc_g, dh, nmap.idx, off, wt)
    ch_l, ch_g = orc.pi_chains(g_e.lesser, g_e.greater, dh, nmap.idx, off, grid.energy_weight, n_qz)
    p_l, p_g = orc.pi_from_chains(ch_l, ch_g)
    return SelfEnergyTensor(s_l, s_g), SelfEnergyTensor(p_l, p_g)


def replay(preset, monkeypatch, phase=None):
    data, meta, p, grid, nmap = _load(preset)
    if phase is not None:
        monkeypatch.setattr(b200_loop, "sse_phase", phase)
    calls = []

    def gf_phase(dev, sigma, pi, params, grid_, nmap_, solver="dense", threads=1):
        i = len(calls)
        calls.append(i)
        # the self-energies this GF pass receives are the reference's (iteration i)
        assert orc.parity_dev(sigma.lesser, sigma.greater, data[f"it{i}_sig_in_l"], data[f"it{i}_sig_in_g"]) <= TOL
        assert orc.parity_dev(pi.lesser, pi.greater, data[f"it{i}_pi_in_l"], data[f"it{i}_pi_in_g"]) <= TOL
        return (GreensTensor(data[f"it{i}_ge_l"], data[f"it{i}_ge_g"]),
                GreensTensor(data[f"it{i}_gph_l"], data[f"it{i}_gph_g"]))

    res = b200_loop.self_consistent_loop(
        SimpleNamespace(dH=data["dh"]), nmap, p, grid, max_iter=meta["iterations"], tol=0.0,
        initial_sigma=SelfEnergyTensor(data["it0_sig_in_l"], data["it0_sig_in_g"]),
        initial_pi=SelfEnergyTensor(data["it0_pi_in_l"], data["it0_pi_in_g"]),
        gf_phase=gf_phase, self_energy_cls=SelfEnergyTensor)
    assert len(calls) == meta["recorded"]
    assert (res.iterations, res.converged) == (meta["iterations"], meta["converged"])
    assert res.deltas == meta["deltas"] and res.abs_deltas == meta["abs_deltas"]  # same G, same formula
    assert orc.parity_dev(res.sigma.lesser, res.sigma.greater, data["final_sigma_l"], data["final_sigma_g"]) <= TOL
    assert orc.parity_dev(res.pi.lesser, res.pi.greater, data["final_pi_l"], data["final_pi_g"]) <= TOL
    return res


@pytest.mark.parametrize("preset", ["tiny", "small"])
def test_loop_bookkeeping_replays_reference_trace_cpu(preset, monkeypatch):
    replay(preset, monkeypatch, phase=oracle_phase)


@pytest.mark.gpu
@pytest.mark.parametrize("preset", ["tiny", "small"])
def test_loop_with_device_sse_phase_replays_reference_trace(preset, monkeypatch):
    replay(preset, monkeypatch)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cli_small_s2", "orb12_s5", "orb5_nb1_s7"])
def test_sse_phase_equals_separate_calls_bitwise(name):
    from paper_1912_08810_b200.sse import sse_phase, sse_pi, sse_sigma
    from paper_1912_08810_b200.types import CombinedD, SseVariant
    from tests.golden_cases import load_case

    c = load_case(name)
    assert c.inputs_ok
    grid = EnergyGrid(values=tuple(np.linspace(-1, 1, c.p.n_E)),
                      frequency_map=tuple(zip(c.offsets.tolist(), c.weights.tolist())),
                      energy_weight=c.meta.get("energy_weight", 1.0 / (2 * np.pi * c.p.n_E)))
    nmap = NeighborMap(c.idx)
    g = GreensTensor(c.g_l, c.g_g)
    timing = {}
    sig, pi = sse_phase(g, GreensTensor(c.d_l, c.d_g), c.dh, nmap, grid, c.p.n_qz, timing=timing)
    dc_l, dc_g = orc.preprocess_D(c.d_l, c.d_g, c.idx)
    sep = sse_sigma(SseVariant.BATCHED_FUSED, g, CombinedD(dc_l, dc_g), c.dh, nmap, grid)
    sep_pi = sse_pi(g, c.dh, nmap, grid, c.p.n_qz)
    assert np.array_equal(sig.lesser, sep.lesser) and np.array_equal(sig.greater, sep.greater)
    assert np.array_equal(pi.lesser, sep_pi.lesser) and np.array_equal(pi.greater, sep_pi.greater)
    assert orc.parity_dev(sig.lesser, sig.greater, c.arrays["sigma_l"], c.arrays["sigma_g"]) <= TOL
    if "pi_l" in c.arrays:
        assert orc.parity_dev(pi.lesser, pi.greater, c.arrays["pi_l"], c.arrays["pi_g"]) <= TOL
    # one G upload for both halves: exactly G, raw D and dH in (no Dc, no second G)
    blk = 16 * c.p.n_orb**2
    g_bytes = 2 * c.p.n_kz * c.p.n_E * c.p.n_A * blk
    d_bytes = 2 * c.d_l.size * 16
    dh_bytes = c.dh.size * 16
    assert timing["h2d_bytes"] == g_bytes + d_bytes + dh_bytes


@pytest.mark.gpu
def test_sse_phase_rejects_non_reverse_closed_map():
    from paper_1912_08810_b200.sse import sse_phase
    from tests.golden_cases import load_case

    c = load_case("cli_small_s2")
    idx = c.idx.copy()
    idx[0, 0] = next(b for b in range(1, len(idx)) if 0 not in idx[b])  # edge 0 -> b without b -> 0
    grid = EnergyGrid(values=tuple(np.linspace(-1, 1, c.p.n_E)),
                      frequency_map=tuple(zip(c.offsets.tolist(), c.weights.tolist())), energy_weight=0.1)
    with pytest.raises(ValueError, match="missing neighbor slot"):
        sse_phase(GreensTensor(c.g_l, c.g_g), GreensTensor(c.d_l, c.d_g), c.dh, NeighborMap(idx), grid, c.p.n_qz)


@pytest.mark.gpu
def test_sse_phase_multi_gpu_bitwise():
    """Atoms split over 2 devices of the process (each device reads its own halo)."""
    import torch

    from paper_1912_08810_b200.sse import sse_phase
    from tests.golden_cases import load_case

    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    c = load_case("orb12_s5")
    grid = EnergyGrid(values=tuple(np.linspace(-1, 1, c.p.n_E)),
                      frequency_map=tuple(zip(c.offsets.tolist(), c.weights.tolist())), energy_weight=0.01)
    args = (GreensTensor(c.g_l, c.g_g), GreensTensor(c.d_l, c.d_g), c.dh, NeighborMap(c.idx), grid, c.p.n_qz)
    s1, p1 = sse_phase(*args, n_gpus=1)
    s2, p2 = sse_phase(*args, n_gpus=2)
    for a, b in ((s1, s2), (p1, p2)):
        assert np.array_equal(a.lesser, b.lesser) and np.array_equal(a.greater, b.greater)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["orb12_s5", "baseline_tiny_s0", "cli_small_s2"])
def test_sse_phase_chunked_pipelines_bitwise(name, monkeypatch):
    """Small Sigma and Pi atom chunks (SSE_OP_CHUNK_ATOMS / SSE_PI_CHUNK_ATOMS): the host pipelines'
    chunk ramps and per-chunk Pi downloads give the same bits as one chunk."""
    from paper_1912_08810_b200.sse import sse_phase, sse_pi
    from tests.golden_cases import load_case

    c = load_case(name)
    grid = EnergyGrid(values=tuple(np.linspace(-1, 1, c.p.n_E)),
                      frequency_map=tuple(zip(c.offsets.tolist(), c.weights.tolist())), energy_weight=0.01)
    args = (GreensTensor(c.g_l, c.g_g), GreensTensor(c.d_l, c.d_g), c.dh, NeighborMap(c.idx), grid, c.p.n_qz)
    s1, p1 = sse_phase(*args)
    q1 = sse_pi(args[0], c.dh, args[3], grid, c.p.n_qz)
    monkeypatch.setenv("SSE_OP_CHUNK_ATOMS", "16")  # Sigma chunks of min(16, NA/8): ramps at both ends
    monkeypatch.setenv("SSE_PI_CHUNK_ATOMS", "5")
    s2, p2 = sse_phase(*args)
    q2 = sse_pi(args[0], c.dh, args[3], grid, c.p.n_qz)
    for a, b in ((s1, s2), (p1, p2), (q1, q2)):
        assert np.array_equal(a.lesser, b.lesser) and np.array_equal(a.greater, b.greater)
    assert np.array_equal(p1.lesser, q1.lesser) and np.array_equal(p1.greater, q1.greater)


@pytest.mark.gpu
@pytest.mark.parametrize("preset", ["tiny", "small"])
def test_device_resident_loop_replays_reference_trace(preset):
    """self_consistent_loop_device: G / D handed over as CUDA tensors by a device GF phase (here
    the reference's recorded gf_phase outputs, uploaded), Sigma / Pi kept in HBM between the
    phases (sse_phase_device), every phase and the final record equal to the reference's."""
    import torch

    data, meta, p, grid, nmap = _load(preset)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    calls = []

    def gf_phase_device(sigma, pi, iteration):
        i = len(calls)
        calls.append(i)
        assert sigma.lesser.is_cuda and pi.greater.is_cuda
        assert orc.parity_dev(sigma.lesser.cpu().numpy(), sigma.greater.cpu().numpy(),
                              data[f"it{i}_sig_in_l"], data[f"it{i}_sig_in_g"]) <= TOL
        assert orc.parity_dev(pi.lesser.cpu().numpy(), pi.greater.cpu().numpy(),
                              data[f"it{i}_pi_in_l"], data[f"it{i}_pi_in_g"]) <= TOL
        return (GreensTensor(cu(data[f"it{i}_ge_l"]), cu(data[f"it{i}_ge_g"])),
                GreensTensor(cu(data[f"it{i}_gph_l"]), cu(data[f"it{i}_gph_g"])))

    res = b200_loop.self_consistent_loop_device(
        gf_phase_device, cu(data["dh"]), nmap, p, grid, max_iter=meta["iterations"], tol=0.0,
        initial_sigma=SelfEnergyTensor(cu(data["it0_sig_in_l"]), cu(data["it0_sig_in_g"])),
        initial_pi=SelfEnergyTensor(cu(data["it0_pi_in_l"]), cu(data["it0_pi_in_g"])))
    assert len(calls) == meta["recorded"]
    assert (res.iterations, res.converged) == (meta["iterations"], meta["converged"])
    np.testing.assert_allclose(res.deltas, meta["deltas"], rtol=1e-12)
    np.testing.assert_allclose(res.abs_deltas, meta["abs_deltas"], rtol=1e-12)
    assert orc.parity_dev(res.sigma.lesser.cpu().numpy(), res.sigma.greater.cpu().numpy(),
                          data["final_sigma_l"], data["final_sigma_g"]) <= TOL
    assert orc.parity_dev(res.pi.lesser.cpu().numpy(), res.pi.greater.cpu().numpy(),
                          data["final_pi_l"], data["final_pi_g"]) <= TOL


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cli_small_s2", "orb12_s5", "slide_orb12_s9"])
def test_sse_phase_device_equals_host_phase_bitwise(name):
    """sse_phase_device on CUDA tensors == sse_phase (host arrays) bit for bit, full problem and an
    owned-atom shard with its halo slab (atom-major)."""
    import torch

    from paper_1912_08810_b200.sse import sse_phase, sse_phase_device
    from tests.golden_cases import load_case

    c = load_case(name)
    p, grid = c.p, EnergyGrid(values=tuple(np.linspace(-1, 1, c.p.n_E)),
                              frequency_map=tuple(zip(c.offsets.tolist(), c.weights.tolist())), energy_weight=0.3)
    nmap = NeighborMap(c.idx)
    s_ref, p_ref = sse_phase(GreensTensor(c.g_l, c.g_g), GreensTensor(c.d_l, c.d_g), c.dh, nmap, grid, p.n_qz)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    sig = [torch.empty(p.electron_shape, dtype=torch.complex128, device="cuda") for _ in range(2)]
    pis = [torch.empty(p.phonon_shape, dtype=torch.complex128, device="cuda") for _ in range(2)]
    sse_phase_device(cu(c.g_l), cu(c.g_g), cu(c.d_l), cu(c.d_g), cu(c.dh), c.idx, grid, *sig, *pis)
    torch.cuda.synchronize()
    assert np.array_equal(sig[0].cpu().numpy(), s_ref.lesser) and np.array_equal(sig[1].cpu().numpy(), s_ref.greater)
    assert np.array_equal(pis[0].cpu().numpy(), p_ref.lesser) and np.array_equal(pis[1].cpu().numpy(), p_ref.greater)
    # shard [lo, hi) with the halo slab, atom-major
    lo, hi = 1, p.n_A - 1
    glo, ghi = int(min(lo, c.idx[lo:hi].min())), int(max(hi, c.idx[lo:hi].max() + 1))
    am = lambda a: cu(np.moveaxis(a[:, :, glo:ghi], 2, 0))  # noqa: E731
    sig = [torch.empty((hi - lo, p.n_kz, p.n_E, p.n_orb, p.n_orb), dtype=torch.complex128, device="cuda")
           for _ in range(2)]
    pis = [torch.empty((p.n_qz, p.n_w, hi - lo, p.n_B + 1, 3, 3), dtype=torch.complex128, device="cuda")
           for _ in range(2)]
    sse_phase_device(am(c.g_l), am(c.g_g), cu(c.d_l[:, :, glo:ghi]), cu(c.d_g[:, :, glo:ghi]), cu(c.dh[lo:hi]),
                     c.idx, grid, *sig, *pis, g_atom0=glo, out_atom0=lo, atom_major=True)
    torch.cuda.synchronize()
    assert np.array_equal(np.moveaxis(sig[0].cpu().numpy(), 0, 2), s_ref.lesser[:, :, lo:hi])
    assert np.array_equal(np.moveaxis(sig[1].cpu().numpy(), 0, 2), s_ref.greater[:, :, lo:hi])
    assert np.array_equal(pis[0].cpu().numpy(), p_ref.lesser[:, :, lo:hi])
    assert np.array_equal(pis[1].cpu().numpy(), p_ref.greater[:, :, lo:hi])
