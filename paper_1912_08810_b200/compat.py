"""Route the reference package's callers to the B200 Sigma.

``negflow`` binds ``sse_sigma`` by name in four places, all looked up at call
time:

* ``negflow.sse.sse_sigma``      called by self_consistent_loop (sse.py:533)
                                 and count_sse_phase (sse.py:449)
* ``negflow.distsim.sse_sigma``  run_omen_scheme / run_tiled_scheme
                                 (distsim.py:24,223,340)
* ``negflow.cli.sse_sigma``      cmd_distsim (cli.py:24-31,222)
* ``negflow.sse_sigma``          the package re-export (__init__.py:16-26)

``patch_reference()`` rebinds all four (and, with ``pi=True``, ``sse_pi`` and the
``sse_pi_chains`` that distsim's schemes call) to a wrapper around
:func:`paper_1912_08810_b200.sse.sse_sigma` that returns the reference's own
``SelfEnergyTensor`` type; ``unpatch_reference()`` restores the originals.
The reference stays read-only.

With ``loop=True`` (default) ``self_consistent_loop`` (bound in negflow.sse,
negflow.cli and the package root) is rebound to
:func:`paper_1912_08810_b200.loop.self_consistent_loop`, whose SSE phase is
one device call (G uploaded once, preprocess_D on the GPU); the GF phase
stays the reference's ``gf_phase``.
"""

from __future__ import annotations

import importlib

from .sse import sse_pi as _b200_sse_pi
from .sse import sse_pi_chains as _b200_sse_pi_chains
from .sse import sse_sigma as _b200_sse_sigma

_TARGETS = ("negflow.sse", "negflow.distsim", "negflow.cli", "negflow")
# sse_pi is bound by name in negflow.sse (self_consistent_loop sse.py:534,
# count_sse_phase sse.py:450), negflow.cli (cli.py:223) and the package root.
_PI_TARGETS = ("negflow.sse", "negflow.cli", "negflow")
# sse_pi_chains: called by sse_pi (sse.py:417) and bound by name in negflow.distsim (distsim.py:24;
# run_omen_scheme distsim.py:227, run_tiled_scheme distsim.py:344)
_PI_CHAINS_TARGETS = ("negflow.sse", "negflow.distsim")
# self_consistent_loop: sse.py:495, re-exported at __init__.py:22, bound in cli.py:28
_LOOP_TARGETS = ("negflow.sse", "negflow.cli", "negflow")
_saved: dict[tuple[str, str], object] = {}


def make_drop_in(self_energy_cls, **kwargs):
    """sse_sigma with the reference signature returning ``self_energy_cls``."""

    def sse_sigma(variant, g, dc, dh, nmap, grid, counter=None):
        out = _b200_sse_sigma(variant, g, dc, dh, nmap, grid, counter=counter, **kwargs)
        return self_energy_cls(lesser=out.lesser, greater=out.greater)

    sse_sigma.__doc__ = "B200 drop-in for negflow.sse.sse_sigma (sse.py:305-329)."
    return sse_sigma


def make_pi_drop_in(self_energy_cls, **kwargs):
    """sse_pi with the reference signature returning ``self_energy_cls``."""

    def sse_pi(g, dh, nmap, grid, n_qz, counter=None, hoist_invariant=True, point_mask=None, atom_range=None):
        out = _b200_sse_pi(g, dh, nmap, grid, n_qz, counter=counter, hoist_invariant=hoist_invariant,
                           point_mask=point_mask, atom_range=atom_range, **kwargs)
        return self_energy_cls(lesser=out.lesser, greater=out.greater)

    sse_pi.__doc__ = "B200 drop-in for negflow.sse.sse_pi (sse.py:409-428)."
    return sse_pi


def make_pi_chains_drop_in(**kwargs):
    """sse_pi_chains with the reference signature (a (lesser, greater) pair of chain arrays)."""

    def sse_pi_chains(g, dh, nmap, grid, n_qz, counter=None, hoist_invariant=True, point_mask=None,
                      atom_range=None):
        return _b200_sse_pi_chains(g, dh, nmap, grid, n_qz, counter=counter, hoist_invariant=hoist_invariant,
                                   point_mask=point_mask, atom_range=atom_range, **kwargs)

    sse_pi_chains.__doc__ = "B200 drop-in for negflow.sse.sse_pi_chains (sse.py:332-390)."
    return sse_pi_chains


def make_loop_drop_in(**kwargs):
    """self_consistent_loop with the reference signature, types and GF phase."""
    from .loop import self_consistent_loop as _loop

    def self_consistent_loop(dev, nmap, params, grid=None, max_iter=20, tol=1e-8, variant=None, solver="dense",
                             threads=1, initial_sigma=None, initial_pi=None):
        ref_sse = importlib.import_module("negflow.sse")
        ref_gf = importlib.import_module("negflow.gf")
        return _loop(dev, nmap, params, grid, max_iter, tol,
                     variant if variant is not None else ref_sse.SseVariant.REFERENCE, solver, threads,
                     initial_sigma, initial_pi, gf_phase=ref_sse.gf_phase, self_energy_cls=ref_gf.SelfEnergyTensor,
                     result_cls=ref_sse.LoopResult, **kwargs)

    self_consistent_loop.__doc__ = "B200 drop-in for negflow.sse.self_consistent_loop (sse.py:495-535)."
    return self_consistent_loop


def _bind(name: str, attr: str, fn) -> None:
    mod = importlib.import_module(name)
    if (name, attr) not in _saved:
        _saved[(name, attr)] = getattr(mod, attr)
    setattr(mod, attr, fn)


def patch_reference(pi: bool = True, loop: bool = True, **kwargs) -> None:
    """Rebind every reference lookup of ``sse_sigma`` (``sse_pi``, ``self_consistent_loop``) to the B200 path."""
    gf = importlib.import_module("negflow.gf")
    drop_in = make_drop_in(gf.SelfEnergyTensor, **kwargs)
    for name in _TARGETS:
        _bind(name, "sse_sigma", drop_in)
    if pi:
        pi_drop_in = make_pi_drop_in(gf.SelfEnergyTensor, **kwargs)
        for name in _PI_TARGETS:
            _bind(name, "sse_pi", pi_drop_in)
        chains_drop_in = make_pi_chains_drop_in(**kwargs)
        for name in _PI_CHAINS_TARGETS:
            _bind(name, "sse_pi_chains", chains_drop_in)
    if loop:
        loop_drop_in = make_loop_drop_in(**kwargs)
        for name in _LOOP_TARGETS:
            _bind(name, "self_consistent_loop", loop_drop_in)


def unpatch_reference() -> None:
    for (name, attr), fn in list(_saved.items()):
        setattr(importlib.import_module(name), attr, fn)
        del _saved[(name, attr)]
