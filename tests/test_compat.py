"""patch_reference rebinds the reference's sse_sigma / sse_pi lookups (no GPU needed)."""

import os
import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.fixture
def negflow():
    if not os.path.isdir(REF):
        pytest.skip("reference not present (GPU box)")
    sys.path.insert(0, REF)
    try:
        import negflow  # noqa: F401
        import negflow.cli  # noqa: F401
        import negflow.distsim  # noqa: F401
        import negflow.sse  # noqa: F401
    except Exception as exc:  # pragma: no cover
        pytest.skip(f"reference not importable: {exc}")
    yield sys.modules["negflow"]
    sys.path.remove(REF)


def test_patch_and_unpatch(negflow):
    from paper_1912_08810_b200.compat import patch_reference, unpatch_reference

    mods = [sys.modules[m] for m in ("negflow.sse", "negflow.distsim", "negflow.cli", "negflow")]
    orig = [m.sse_sigma for m in mods]
    orig_pi = [sys.modules[m].sse_pi for m in ("negflow.sse", "negflow.cli", "negflow")]
    patch_reference()
    try:
        for m in mods:
            assert m.sse_sigma.__doc__.startswith("B200 drop-in")
        for m in ("negflow.sse", "negflow.cli", "negflow"):
            assert sys.modules[m].sse_pi.__doc__.startswith("B200 drop-in")
        for m in ("negflow.sse", "negflow.distsim"):
            assert sys.modules[m].sse_pi_chains.__doc__.startswith("B200 drop-in")
        # the reference's own validation still runs first (no device work): wrong kind -> ValueError
        import numpy as np
        from negflow.gf import GreensTensor
        from negflow.sse import CombinedD, SseVariant

        ph = GreensTensor(np.zeros((1, 1, 2, 2, 3, 3), complex), np.zeros((1, 1, 2, 2, 3, 3), complex))
        dc = CombinedD(np.zeros((1, 1, 2, 1, 3, 3), complex), np.zeros((1, 1, 2, 1, 3, 3), complex))
        from negflow.device import build_neighbor_map
        from negflow.params import SimParams, default_grid

        grid = default_grid(SimParams(1, 1, 2, 1, 2, 1, 1))
        with pytest.raises(ValueError, match="expects an electron tensor"):
            negflow.sse.sse_sigma(SseVariant.REFERENCE, ph, dc, np.zeros((2, 1, 3, 1, 1)),
                                  build_neighbor_map(2, 1), grid)
    finally:
        unpatch_reference()
    assert [m.sse_sigma for m in mods] == orig
    assert [sys.modules[m].sse_pi for m in ("negflow.sse", "negflow.cli", "negflow")] == orig_pi


def test_patch_rebinds_self_consistent_loop(negflow):
    from paper_1912_08810_b200.compat import patch_reference, unpatch_reference

    names = ("negflow.sse", "negflow.cli", "negflow")
    orig = [sys.modules[m].self_consistent_loop for m in names]
    patch_reference()
    try:
        for m in names:
            assert sys.modules[m].self_consistent_loop.__doc__.startswith("B200 drop-in")
    finally:
        unpatch_reference()
    assert [sys.modules[m].self_consistent_loop for m in names] == orig
    patch_reference(loop=False)
    try:
        assert [sys.modules[m].self_consistent_loop for m in names] == orig
    finally:
        unpatch_reference()


def test_patched_loop_runs_reference_gf_phase_cpu(negflow, monkeypatch):
    """The rebound loop drives the reference's own gf_phase and LoopResult; the device
    phase is replaced by the CPU oracle here (no GPU), so this checks the wiring."""
    import numpy as np

    import paper_1912_08810_b200.loop as b200_loop
    from negflow.cli import PRESETS
    from negflow.device import synthesize
    from negflow.sse import seeded_self_energies
    from paper_1912_08810_b200.compat import patch_reference, unpatch_reference
    from tests.test_loop import oracle_phase

    p = PRESETS["tiny"]
    dev, nmap = synthesize(p, seed=1)
    s0, p0 = seeded_self_energies(p, 0.05)
    ref = negflow.sse.self_consistent_loop(dev, nmap, p, max_iter=3, tol=0.0, initial_sigma=s0, initial_pi=p0)
    monkeypatch.setattr(b200_loop, "sse_phase", oracle_phase)
    patch_reference()
    try:
        got = negflow.self_consistent_loop(dev, nmap, p, max_iter=3, tol=0.0, initial_sigma=s0, initial_pi=p0)
    finally:
        unpatch_reference()
    assert type(got).__name__ == "LoopResult" and type(got).__module__ == "negflow.sse"
    assert (got.iterations, got.converged) == (ref.iterations, ref.converged)
    scale = max(np.abs(ref.g_electron.lesser).max(), np.abs(ref.g_electron.greater).max())
    assert np.abs(got.g_electron.lesser - ref.g_electron.lesser).max() <= 1e-9 * scale
    assert np.abs(got.g_electron.greater - ref.g_electron.greater).max() <= 1e-9 * scale
