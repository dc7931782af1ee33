"""Self-consistent Born loop with the SSE phase in one device call.

Mirror of ``negflow.sse.self_consistent_loop`` (sse.py:495-535): the GF phase
is the caller's (the reference's ``negflow.gf.gf_phase`` by default, CPU);
the SSE phase -- ``preprocess_D`` + ``sse_sigma`` + ``sse_pi``
(sse.py:532-534) -- is one :func:`paper_1912_08810_b200.sse.sse_phase` call:
G^<> uploaded once for Sigma and Pi, the raw phonon tensor reduced on the
device.  Convergence test, iteration order, seeds and the result record are
the reference's (``_gf_change`` sse.py:468-475).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .sse import sse_phase
from .types import SseVariant


@dataclass
class LoopResult:
    """Same fields as ``negflow.sse.LoopResult`` (sse.py:455-465)."""

    g_electron: object
    g_phonon: object
    sigma: object
    pi: object
    iterations: int
    converged: bool
    deltas: list
    abs_deltas: list


def gf_change(old, new) -> tuple[float, float]:
    """(absolute, relative) max change of the lesser/greater pair (sse.py:468-475)."""
    scale = max(float(np.max(np.abs(old.lesser))), float(np.max(np.abs(old.greater))), 1e-300)
    diff = max(
        float(np.max(np.abs(new.lesser - old.lesser))),
        float(np.max(np.abs(new.greater - old.greater))),
    )
    return diff, diff / scale


def self_consistent_loop(
    dev,
    nmap,
    params,
    grid=None,
    max_iter: int = 20,
    tol: float = 1e-8,
    variant=SseVariant.REFERENCE,
    solver: str = "dense",
    threads: int = 1,
    initial_sigma=None,
    initial_pi=None,
    *,
    gf_phase=None,
    self_energy_cls=None,
    result_cls=None,
    n_gpus: int | None = None,
):
    """Alternate GF and SSE phases until the electron GF stops moving (sse.py:495-535).

    ``gf_phase(dev, sigma, pi, params, grid, nmap, solver=, threads=)`` and
    the zero self-energy constructors default to the reference's
    (``negflow.gf``); ``self_energy_cls`` / ``result_cls`` select the types
    handed back (the reference's when patched in).  ``variant`` is accepted
    for signature compatibility: every arrangement gives the same Sigma here.
    """
    SseVariant(variant.value if hasattr(variant, "value") else variant)  # same validation as sse.py:533
    if gf_phase is None or self_energy_cls is None or grid is None:
        import negflow.gf as ref_gf
        import negflow.params as ref_params

        gf_phase = gf_phase or ref_gf.gf_phase
        self_energy_cls = self_energy_cls or ref_gf.SelfEnergyTensor
        grid = grid if grid is not None else ref_params.default_grid(params)
    result_cls = result_cls or LoopResult
    if initial_sigma is not None:
        sigma = initial_sigma
    else:
        sigma = self_energy_cls(lesser=np.zeros(params.electron_shape, dtype=np.complex128),
                                greater=np.zeros(params.electron_shape, dtype=np.complex128))
    if initial_pi is not None:
        pi = initial_pi
    else:
        pi = self_energy_cls(lesser=np.zeros(params.phonon_shape, dtype=np.complex128),
                             greater=np.zeros(params.phonon_shape, dtype=np.complex128))
    g_e = g_ph = None
    prev = None
    deltas: list[float] = []
    abs_deltas: list[float] = []
    for iteration in range(1, max_iter + 1):
        g_e, g_ph = gf_phase(dev, sigma, pi, params, grid, nmap, solver=solver, threads=threads)
        if prev is not None:
            diff, delta = gf_change(prev, g_e)
            deltas.append(delta)
            abs_deltas.append(diff)
            if delta <= tol:
                return result_cls(g_e, g_ph, sigma, pi, iteration, True, deltas, abs_deltas)
        prev = g_e
        s, p = sse_phase(g_e, g_ph, dev.dH, nmap, grid, params.n_qz, n_gpus=n_gpus)
        sigma = self_energy_cls(lesser=s.lesser, greater=s.greater)
        pi = self_energy_cls(lesser=p.lesser, greater=p.greater)
    return result_cls(g_e, g_ph, sigma, pi, max_iter, False, deltas, abs_deltas)
