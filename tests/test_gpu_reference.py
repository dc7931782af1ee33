"""The UNMODIFIED reference running on the B200 through patch_reference() (GPU box).

negflow comes from oracle/_ref (bytecode staged by oracle/make_ref.py) or /root/reference.
patch_reference() rebinds the reference's own lookups of sse_sigma, sse_pi, sse_pi_chains and
self_consistent_loop, so the reference's callers -- its Born loop (sse.py:495-535), the simulated
distributed schemes (distsim.py:166-353) -- run their SSE work on libsse.  Each is compared with
the same call unpatched (the reference's CPU path): acceptance criterion 7's setup
(test_acceptance.py:218-250) and the CLI tiny preset's loop.  Tolerance: the reference metric 1e-10.
"""

import numpy as np
import pytest

from oracle.ref import import_negflow, ref_path

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def nf():
    if ref_path() is None:
        pytest.skip("reference not staged (oracle/make_ref.py)")
    return import_negflow()


def _dev(got, ref):
    scale = max(np.max(np.abs(ref.lesser)), np.max(np.abs(ref.greater)), 1e-300)
    return max(np.max(np.abs(got.lesser - ref.lesser)), np.max(np.abs(got.greater - ref.greater))) / scale


def _patched(fn):
    from paper_1912_08810_b200.compat import patch_reference, unpatch_reference

    patch_reference()
    try:
        return fn()
    finally:
        unpatch_reference()


def _instance(nf, params, seed):
    rng = np.random.default_rng(seed)
    rand = lambda s: rng.standard_normal(s) + 1j * rng.standard_normal(s)  # noqa: E731
    grid = nf.params.default_grid(params)
    dev, nmap = nf.device.synthesize(params, seed=seed)
    g = nf.gf.GreensTensor(rand(params.electron_shape), rand(params.electron_shape))
    d = nf.gf.GreensTensor(rand(params.phonon_shape), rand(params.phonon_shape))
    return grid, dev, nmap, g, d


def test_patched_entry_points_route_to_libsse(nf):
    from paper_1912_08810_b200 import _lib

    params = nf.params.SimParams(n_kz=3, n_qz=3, n_E=40, n_w=14, n_A=8, n_B=4, n_orb=12)
    grid, dev, nmap, g, d = _instance(nf, params, 5)
    dc = nf.sse.preprocess_D(d, nmap)
    ref = nf.sse.sse_sigma(nf.sse.SseVariant.BATCHED_FUSED, g, dc, dev.dH, nmap, grid)
    got = _patched(lambda: nf.sse.sse_sigma(nf.sse.SseVariant.BATCHED_FUSED, g, dc, dev.dH, nmap, grid))
    assert type(got) is nf.gf.SelfEnergyTensor
    assert _dev(got, ref) <= TOL
    assert _lib.kernel_name("sigma").startswith("sigma_dmma_kslide_kernel<12")
    ref_pi = nf.sse.sse_pi(g, dev.dH, nmap, grid, params.n_qz)
    got_pi = _patched(lambda: nf.sse.sse_pi(g, dev.dH, nmap, grid, params.n_qz))
    assert _dev(got_pi, ref_pi) <= TOL
    ch = _patched(lambda: nf.distsim.sse_pi_chains(g, dev.dH, nmap, grid, params.n_qz, atom_range=(2, 6)))
    ref_ch = nf.sse.sse_pi_chains(g, dev.dH, nmap, grid, params.n_qz, atom_range=(2, 6))
    scale = max(np.max(np.abs(ref_ch[0])), np.max(np.abs(ref_ch[1])))
    assert max(np.max(np.abs(ch[0] - ref_ch[0])), np.max(np.abs(ch[1] - ref_ch[1]))) <= TOL * scale


@pytest.mark.parametrize("params_kw, schemes", [
    # acceptance criterion 7 (test_acceptance.py:218-250)
    (dict(n_kz=2, n_qz=2, n_E=4, n_w=1, n_A=4, n_B=2, n_orb=2, bnum=2),
     [("omen", 1), ("omen", 2), ("omen", 4), ("omen", 8), ("tiled", (1, 1)), ("tiled", (2, 2)), ("tiled", (1, 4)),
      ("tiled", (2, 1))]),
    # test_distsim.py RICH shape
    (dict(n_kz=2, n_qz=2, n_E=16, n_w=2, n_A=8, n_B=2, n_orb=2, bnum=4), [("omen", 4), ("tiled", (2, 2))]),
])
def test_distributed_schemes_patched_match_reference(nf, params_kw, schemes):
    """run_omen_scheme / run_tiled_scheme with their sse_sigma and sse_pi_chains on the B200: the
    same Sigma / Pi as the single-node reference and the same message ledgers as unpatched."""
    params = nf.params.SimParams(**params_kw)
    grid, dev, nmap, g, d = _instance(nf, params, 7)
    dc = nf.sse.preprocess_D(d, nmap)
    ref_sigma = nf.sse.sse_sigma(nf.sse.SseVariant.REFERENCE, g, dc, dev.dH, nmap, grid)
    ref_pi = nf.sse.sse_pi(g, dev.dH, nmap, grid, params.n_qz)
    for kind, arg in schemes:
        if kind == "omen":
            run = lambda: nf.distsim.run_omen_scheme(g, d, dev.dH, nmap, grid, params, arg)  # noqa: E731
            model = ("omen", arg)
        else:
            run = lambda: nf.distsim.run_tiled_scheme(g, d, dev.dH, nmap, grid, params, *arg)  # noqa: E731
            model = ("tiled", arg[0] * arg[1], *arg)
        sigma, pi, ledger = _patched(run)
        _, _, ref_ledger = run()
        assert _dev(sigma, ref_sigma) <= TOL, (kind, arg)
        assert _dev(pi, ref_pi) <= TOL, (kind, arg)
        assert [(e.round, e.src, e.dst, e.tag, e.bytes) for e in ledger.entries] == \
               [(e.round, e.src, e.dst, e.tag, e.bytes) for e in ref_ledger.entries]
        rows = nf.distsim.compare_ledger_with_model(ledger, params, *model)
        assert max(r["rel_delta"] for r in rows) == 0.0


def test_patched_born_loop_matches_reference(nf):
    """negflow.self_consistent_loop (CLI tiny preset, seeded self-energies) with the SSE phase on
    the B200 (libsse sse_phase) and the reference's own gf_phase: same trajectory and record."""
    p = nf.cli.PRESETS["tiny"]
    dev, nmap = nf.device.synthesize(p, seed=1)
    s0, p0 = nf.sse.seeded_self_energies(p, 0.05)
    ref = nf.sse.self_consistent_loop(dev, nmap, p, max_iter=4, tol=0.0, initial_sigma=s0, initial_pi=p0)
    got = _patched(lambda: nf.self_consistent_loop(dev, nmap, p, max_iter=4, tol=0.0, initial_sigma=s0,
                                                   initial_pi=p0))
    assert type(got) is nf.sse.LoopResult
    assert (got.iterations, got.converged) == (ref.iterations, ref.converged)
    np.testing.assert_allclose(got.deltas, ref.deltas, rtol=1e-8)
    assert _dev(got.sigma, ref.sigma) <= TOL
    assert _dev(got.pi, ref.pi) <= TOL
    assert _dev(got.g_electron, ref.g_electron) <= 1e-9
