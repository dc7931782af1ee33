"""Route the reference package's callers to the B200 Sigma.

``negflow`` binds ``sse_sigma`` by name in four places, all looked up at call
time:

* ``negflow.sse.sse_sigma``      called by self_consistent_loop (sse.py:533)
                                 and count_sse_phase (sse.py:449)
* ``negflow.distsim.sse_sigma``  run_omen_scheme / run_tiled_scheme
                                 (distsim.py:24,223,340)
* ``negflow.cli.sse_sigma``      cmd_distsim (cli.py:24-31,222)
* ``negflow.sse_sigma``          the package re-export (__init__.py:16-26)

``patch_reference()`` rebinds all four to a wrapper around
:func:`paper_1912_08810_b200.sse.sse_sigma` that returns the reference's own
``SelfEnergyTensor`` type; ``unpatch_reference()`` restores the originals.
The reference stays read-only.
"""

from __future__ import annotations

import importlib

from .sse import sse_sigma as _b200_sse_sigma

_TARGETS = ("negflow.sse", "negflow.distsim", "negflow.cli", "negflow")
_saved: dict[str, object] = {}


def make_drop_in(self_energy_cls, **kwargs):
    """sse_sigma with the reference signature returning ``self_energy_cls``."""

    def sse_sigma(variant, g, dc, dh, nmap, grid, counter=None):
        out = _b200_sse_sigma(variant, g, dc, dh, nmap, grid, counter=counter, **kwargs)
        return self_energy_cls(lesser=out.lesser, greater=out.greater)

    sse_sigma.__doc__ = "B200 drop-in for negflow.sse.sse_sigma (sse.py:305-329)."
    return sse_sigma


def patch_reference(**kwargs) -> None:
    """Rebind every reference lookup of ``sse_sigma`` to the B200 path."""
    gf = importlib.import_module("negflow.gf")
    drop_in = make_drop_in(gf.SelfEnergyTensor, **kwargs)
    for name in _TARGETS:
        mod = importlib.import_module(name)
        if name not in _saved:
            _saved[name] = getattr(mod, "sse_sigma")
        setattr(mod, "sse_sigma", drop_in)


def unpatch_reference() -> None:
    for name, fn in list(_saved.items()):
        setattr(importlib.import_module(name), "sse_sigma", fn)
        del _saved[name]
