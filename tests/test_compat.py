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
