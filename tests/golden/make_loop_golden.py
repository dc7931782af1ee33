"""Golden trace of the REFERENCE self-consistent Born loop (sse.py:495-535).

Run in the build container (the reference is importable only there):

    python tests/golden/make_loop_golden.py

For the CLI presets ``tiny`` and ``small`` (cli.py:34-35) it synthesizes the
device (device.py:175, seed 1), seeds the self-energies
(``seeded_self_energies``, sse.py:478-492, scale 0.05) and runs the
reference's own ``self_consistent_loop`` for 4 iterations (tol 0: never
converges), recording what its ``gf_phase`` returned at every iteration and
the self-energies it was handed.  The GPU box has no reference GF solver;
tests there replay the recorded GF outputs through the B200 loop
(``paper_1912_08810_b200.loop``) and compare every SSE phase with the
reference's, plus the final ``LoopResult``.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import negflow.sse as ref_sse  # noqa: E402
from negflow.cli import PRESETS  # noqa: E402
from negflow.device import synthesize  # noqa: E402
from negflow.params import default_grid  # noqa: E402

ITERS = 4
SCALE = 0.05


def run(preset: str) -> None:
    p = PRESETS[preset]
    dev, nmap = synthesize(p, seed=1)
    grid = default_grid(p)
    sigma0, pi0 = ref_sse.seeded_self_energies(p, SCALE)
    trace = []
    real_gf = ref_sse.gf_phase

    def recording_gf(dev_, sigma, pi, params, grid_, nmap_, solver="dense", threads=1):
        g_e, g_ph = real_gf(dev_, sigma, pi, params, grid_, nmap_, solver=solver, threads=threads)
        trace.append((sigma.lesser.copy(), sigma.greater.copy(), pi.lesser.copy(), pi.greater.copy(),
                      g_e.lesser.copy(), g_e.greater.copy(), g_ph.lesser.copy(), g_ph.greater.copy()))
        return g_e, g_ph

    ref_sse.gf_phase = recording_gf
    try:
        res = ref_sse.self_consistent_loop(dev, nmap, p, grid, max_iter=ITERS, tol=0.0,
                                           initial_sigma=sigma0, initial_pi=pi0)
    finally:
        ref_sse.gf_phase = real_gf
    arrays = {"dh": dev.dH, "nmap": nmap.idx}
    names = ("sig_in_l", "sig_in_g", "pi_in_l", "pi_in_g", "ge_l", "ge_g", "gph_l", "gph_g")
    for i, rec in enumerate(trace):
        for n, a in zip(names, rec):
            arrays[f"it{i}_{n}"] = a
    arrays["final_sigma_l"], arrays["final_sigma_g"] = res.sigma.lesser, res.sigma.greater
    arrays["final_pi_l"], arrays["final_pi_g"] = res.pi.lesser, res.pi.greater
    meta = {
        "preset": preset, "params": {k: getattr(p, k) for k in ("n_kz", "n_qz", "n_E", "n_w", "n_A", "n_B",
                                                               "n_orb", "bnum")},
        "iterations": res.iterations, "converged": res.converged, "deltas": res.deltas,
        "abs_deltas": res.abs_deltas, "recorded": len(trace), "offsets": list(grid.offsets),
        "weights": [w for _, w in grid.frequency_map], "energy_weight": grid.energy_weight,
    }
    np.savez_compressed(os.path.join(HERE, f"loop_{preset}.npz"), meta=json.dumps(meta), **arrays)
    print(preset, res.iterations, res.converged, res.deltas)


if __name__ == "__main__":
    for preset in ("tiny", "small"):
        run(preset)
