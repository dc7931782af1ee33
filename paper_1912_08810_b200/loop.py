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


def gf_change_device(old, new) -> tuple[float, float]:
    """gf_change (sse.py:468-475) on device tensors: only the two scalars come back to the host."""
    import torch

    scale = torch.maximum(old.lesser.abs().max(), old.greater.abs().max()).clamp_min(1e-300)
    diff = torch.maximum((new.lesser - old.lesser).abs().max(), (new.greater - old.greater).abs().max())
    d, s = (float(x) for x in torch.stack([diff, scale]).cpu())
    return d, d / s


def self_consistent_loop_device(
    gf_phase_device,
    dh,
    nmap,
    params,
    grid,
    max_iter: int = 20,
    tol: float = 1e-8,
    initial_sigma=None,
    initial_pi=None,
    *,
    self_energy_cls=None,
    greens_cls=None,
    result_cls=None,
):
    """The Born loop with G, D, Sigma and Pi resident in HBM between the phases.

    Same iteration order, convergence test and result record as ``self_consistent_loop``
    (sse.py:495-535), but the SSE phase is :func:`sse.sse_phase_device` on torch CUDA tensors and
    nothing crosses the host link except the two convergence scalars per iteration:

    ``gf_phase_device(sigma, pi, iteration) -> (g_e, g_ph)`` is the (device) GF phase: it receives
    the self-energies as ``self_energy_cls`` pairs of CUDA tensors and returns ``greens_cls`` pairs
    of CUDA tensors (G<> [Nkz, NE, NA, No, No], raw D<> [Nqz, Nw, NA, NB+1, 3, 3]).  ``dh`` is the
    coupling tensor on the device.  The reference's GF phase is a CPU solver (out of scope here);
    any GPU GF phase with this signature plugs in without host copies.
    """
    import torch

    from .sse import sse_phase_device
    from .types import GreensTensor, SelfEnergyTensor

    self_energy_cls = self_energy_cls or SelfEnergyTensor
    greens_cls = greens_cls or GreensTensor
    result_cls = result_cls or LoopResult
    dev = dh.device
    c128 = dict(dtype=torch.complex128, device=dev)
    sigma = initial_sigma or self_energy_cls(lesser=torch.zeros(params.electron_shape, **c128),
                                             greater=torch.zeros(params.electron_shape, **c128))
    pi = initial_pi or self_energy_cls(lesser=torch.zeros(params.phonon_shape, **c128),
                                       greater=torch.zeros(params.phonon_shape, **c128))
    idx = np.ascontiguousarray(nmap.idx, dtype=np.int64)
    g_e = g_ph = prev = None
    deltas: list[float] = []
    abs_deltas: list[float] = []
    for iteration in range(1, max_iter + 1):
        g_e, g_ph = gf_phase_device(sigma, pi, iteration)
        if prev is not None:
            diff, delta = gf_change_device(prev, g_e)
            deltas.append(delta)
            abs_deltas.append(diff)
            if delta <= tol:
                return result_cls(g_e, g_ph, sigma, pi, iteration, True, deltas, abs_deltas)
        prev = g_e
        s = [torch.empty(params.electron_shape, **c128) for _ in range(2)]
        p = [torch.empty(params.phonon_shape, **c128) for _ in range(2)]
        sse_phase_device(g_e.lesser, g_e.greater, g_ph.lesser, g_ph.greater, dh, idx, grid, s[0], s[1], p[0], p[1])
        sigma = self_energy_cls(lesser=s[0], greater=s[1])
        pi = self_energy_cls(lesser=p[0], greater=p[1])
    return result_cls(g_e, g_ph, sigma, pi, max_iter, False, deltas, abs_deltas)
