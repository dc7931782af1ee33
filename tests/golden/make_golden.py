"""Generate golden SSE fixtures by running the REFERENCE implementation.

Run in the build container (the reference is importable only there):

    python tests/golden/make_golden.py

It imports ``negflow`` from /root/reference/pkg/src (read-only), draws each
case's inputs with the documented recipe (the same draws the package's
``inputs.stream_instance`` replays), runs the reference's ``sse_sigma``
(REFERENCE and BATCHED_FUSED), ``preprocess_D`` and ``sse_pi``, and stores
the outputs plus a sha256 digest of the inputs in ``tests/golden/*.npz``.
The GPU box has no /root/reference; tests there regenerate the inputs from
the recipe, check the digest, and compare against these stored outputs.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from negflow.device import build_neighbor_map  # noqa: E402
from negflow.gf import GreensTensor  # noqa: E402
from negflow.params import EnergyGrid, SimParams, default_grid  # noqa: E402
from negflow.sse import CombinedD, SseVariant, preprocess_D, sse_pi, sse_sigma  # noqa: E402


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def stream(seed, p, dh_scale):
    rng = np.random.default_rng(seed)

    def rand(shape):
        return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)

    g_l, g_g = rand(p.electron_shape), rand(p.electron_shape)
    d_l, d_g = rand(p.phonon_shape), rand(p.phonon_shape)
    dh = dh_scale * rand((p.n_A, p.n_B, 3, p.n_orb, p.n_orb))
    return g_l, g_g, d_l, d_g, dh


run_case_filter = None  # "only" mode: the names to (re)generate


def run_case(name, p, seed, dh_scale=1.0, grid=None, with_pi=False, store_dc=False, store_bf=True):
    if run_case_filter is not None and name not in run_case_filter:
        return
    grid = grid if grid is not None else default_grid(p)
    nmap = build_neighbor_map(p.n_A, p.n_B)
    g_l, g_g, d_l, d_g, dh = stream(seed, p, dh_scale)
    g = GreensTensor(g_l, g_g)
    dc = preprocess_D(GreensTensor(d_l, d_g), nmap)
    ref = sse_sigma(SseVariant.REFERENCE, g, dc, dh, nmap, grid)
    bf = sse_sigma(SseVariant.BATCHED_FUSED, g, dc, dh, nmap, grid)
    out = {"sigma_l": ref.lesser, "sigma_g": ref.greater}
    if store_bf:  # BATCHED_FUSED output (small cases only, to keep the fixtures small)
        out["bf_l"] = bf.lesser
        out["bf_g"] = bf.greater
    if store_dc:
        out["dc_l"] = dc.lesser
        out["dc_g"] = dc.greater
    if with_pi:
        pi = sse_pi(g, dh, nmap, grid, p.n_qz)
        out["pi_l"] = pi.lesser
        out["pi_g"] = pi.greater
    meta = {
        "name": name,
        "recipe": "stream",
        "seed": seed,
        "dh_scale": dh_scale,
        "params": {k: getattr(p, k) for k in ("n_kz", "n_qz", "n_E", "n_w", "n_A", "n_B", "n_orb")},
        "offsets": [int(o) for o, _ in grid.frequency_map],
        "weights": [float(w) for _, w in grid.frequency_map],
        "energy_weight": grid.energy_weight,
        "nmap": nmap.idx.tolist(),
        "input_sha256": digest(g_l, g_g, d_l, d_g, dh),
        "dc_sha256": digest(dc.lesser, dc.greater),
        "bf_vs_reference": float(
            max(np.max(np.abs(bf.lesser - ref.lesser)), np.max(np.abs(bf.greater - ref.greater)))
            / max(np.max(np.abs(ref.lesser)), np.max(np.abs(ref.greater)), 1e-300)
        ),
    }
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), meta=json.dumps(meta), **out)
    print(f"{name}: {p} -> {sum(v.nbytes for v in out.values()) / 1e6:.2f} MB")


def scalar_kat():
    """test_sse.py:175-197 scalar instance (offset 0, NE = 1, weight 0.37)."""
    p = SimParams(n_kz=1, n_qz=1, n_E=1, n_w=1, n_A=2, n_B=1, n_orb=1, bnum=1)
    nmap = build_neighbor_map(2, 1)
    grid = EnergyGrid(values=(0.0,), frequency_map=((0, 0.37),), energy_weight=1.0)
    rng = np.random.default_rng(9)

    def rand(shape):
        return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)

    g_l, g_g = rand(p.electron_shape), rand(p.electron_shape)
    dh = rand((2, 1, 3, 1, 1))
    dc_l, dc_g = rand((1, 1, 2, 1, 3, 3)), rand((1, 1, 2, 1, 3, 3))
    ref = sse_sigma(SseVariant.REFERENCE, GreensTensor(g_l, g_g), CombinedD(dc_l, dc_g), dh, nmap, grid)
    meta = {
        "name": "kat_scalar",
        "recipe": "kat_scalar",
        "offsets": [0],
        "weights": [0.37],
        "nmap": nmap.idx.tolist(),
        "input_sha256": digest(g_l, g_g, dh, dc_l, dc_g),
    }
    np.savez_compressed(
        os.path.join(HERE, "kat_scalar.npz"), meta=json.dumps(meta), sigma_l=ref.lesser, sigma_g=ref.greater
    )
    print("kat_scalar")


def criterion5():
    """test_acceptance.py:139-177: 50 random instances from default_rng(2024)."""
    rng = np.random.default_rng(2024)

    def rand(shape):
        return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)

    arrays = {}
    metas = []
    instances = 0
    while instances < 50:
        n_kz = int(rng.integers(1, 5))
        n_qz = int(rng.integers(1, n_kz + 1))
        n_e = int(rng.integers(2, 5))
        n_w = int(rng.integers(1, min(4, n_e)))
        n_a = int(rng.choice([2, 4]))
        n_b = int(rng.integers(1, min(3, n_a)))
        n_orb = int(rng.integers(1, 4))
        if n_a % 2 == 1 and n_b % 2 == 1:
            continue
        p = SimParams(n_kz=n_kz, n_qz=n_qz, n_E=n_e, n_w=n_w, n_A=n_a, n_B=n_b, n_orb=n_orb, bnum=1)
        grid = default_grid(p)
        nmap = build_neighbor_map(n_a, n_b)
        g_l, g_g = rand(p.electron_shape), rand(p.electron_shape)
        d_l, d_g = rand(p.phonon_shape), rand(p.phonon_shape)
        dh = rand((n_a, n_b, 3, n_orb, n_orb))
        dc = preprocess_D(GreensTensor(d_l, d_g), nmap)
        ref = sse_sigma(SseVariant.REFERENCE, GreensTensor(g_l, g_g), dc, dh, nmap, grid)
        arrays[f"sigma_l_{instances}"] = ref.lesser
        arrays[f"sigma_g_{instances}"] = ref.greater
        metas.append(
            {
                "params": [n_kz, n_qz, n_e, n_w, n_a, n_b, n_orb],
                "input_sha256": digest(g_l, g_g, d_l, d_g, dh),
            }
        )
        instances += 1
    np.savez_compressed(os.path.join(HERE, "criterion5.npz"), meta=json.dumps(metas), **arrays)
    print("criterion5: 50 instances")


def slide_cases():
    """Shapes that run the production sliding-window Sigma kernel (Nw >= 12, sliding default offsets).

    slide_orb12: No = 12, NB = 4 (the paper's block shape), 480 rows per (atom, k) -> one full and
    one partial 288-row CTA; slide_orb10: No = 10 (the small config's block); paperlike_w70: the
    paper's Nw = 70 and offsets 1..70 with NE = 90, so offsets run past the top energy of the first
    CTAs (empty stages) and each (q, s) segment crosses the stage ring many times.
    """
    run_case("slide_orb12_s9", SimParams(n_kz=3, n_qz=3, n_E=40, n_w=14, n_A=6, n_B=4, n_orb=12), 9,
             dh_scale=0.05, store_bf=False)
    run_case("slide_orb10_s10", SimParams(n_kz=3, n_qz=3, n_E=48, n_w=16, n_A=6, n_B=4, n_orb=10), 10,
             dh_scale=0.05, store_bf=False)
    run_case("paperlike_w70_s11", SimParams(n_kz=3, n_qz=2, n_E=90, n_w=70, n_A=4, n_B=2, n_orb=12), 11,
             dh_scale=0.05, store_bf=False)
    # the paper's Pi shapes (No = 12, NB = 4, Nw = 70: K5 pi_build_dmma_kernel<12> and the split
    # K6 v4 pi_dmma4_kernel<12,4,4,3,4,true>, 9 lag tiles) pinned to the reference's sse_pi
    run_case("pi_paperlike_s12", SimParams(n_kz=2, n_qz=2, n_E=80, n_w=70, n_A=6, n_B=4, n_orb=12), 12,
             dh_scale=0.05, store_bf=False, with_pi=True)


def main():
    if sys.argv[1:] == ["slide"]:
        slide_cases()
        return
    if len(sys.argv) > 2 and sys.argv[1] == "only":  # regenerate named slide cases only
        import inspect

        src = inspect.getsource(slide_cases)
        for name in sys.argv[2:]:
            assert f'"{name}"' in src, name
        globals()["run_case_filter"] = set(sys.argv[2:])
        slide_cases()
        return
    scalar_kat()
    criterion5()
    # test_sse.py TINY instance recipe (seeds 3, 4)
    tiny_test = SimParams(n_kz=3, n_qz=2, n_E=4, n_w=2, n_A=4, n_B=2, n_orb=2, bnum=2)
    run_case("test_tiny_s3", tiny_test, 3, with_pi=True, store_dc=True)
    run_case("test_tiny_s4", tiny_test, 4, with_pi=True)
    # CLI presets (cli.py:34-35)
    run_case("cli_tiny_s1", SimParams(n_kz=3, n_qz=2, n_E=8, n_w=2, n_A=8, n_B=2, n_orb=2, bnum=4), 1,
             with_pi=True)
    run_case("cli_small_s2", SimParams(n_kz=3, n_qz=2, n_E=8, n_w=2, n_A=32, n_B=4, n_orb=2, bnum=4), 2,
             with_pi=True)
    # BASELINE.json configs[0] ("tiny": NA=64, NB=4, No=4, NE=32, Nw=4, Nkz=Nqz=3), dH x 0.05
    base = SimParams(n_kz=3, n_qz=3, n_E=32, n_w=4, n_A=64, n_B=4, n_orb=4)
    run_case("baseline_tiny_s0", base, 0, dh_scale=0.05, store_bf=False)
    # kernel-shape coverage: the No of the larger configs, NB odd (XOR slot), Nqz < Nkz
    run_case("orb12_s5", SimParams(n_kz=2, n_qz=2, n_E=12, n_w=5, n_A=6, n_B=4, n_orb=12), 5, dh_scale=0.05, store_bf=False)
    run_case("orb10_s6", SimParams(n_kz=3, n_qz=2, n_E=10, n_w=3, n_A=6, n_B=3, n_orb=10), 6, dh_scale=0.05, store_bf=False)
    run_case("orb5_nb1_s7", SimParams(n_kz=4, n_qz=3, n_E=9, n_w=4, n_A=4, n_B=1, n_orb=5), 7)
    # general (offset, weight) table: non-monotone offsets incl. 0, varied weights
    p = SimParams(n_kz=2, n_qz=1, n_E=7, n_w=4, n_A=5, n_B=2, n_orb=3)
    grid = EnergyGrid(
        values=tuple(np.linspace(-1, 1, 7)),
        frequency_map=((3, 0.25), (0, -0.5), (6, 1.75), (1, 0.125)),
        energy_weight=0.1,
    )
    run_case("general_grid_s8", p, 8, grid=grid, with_pi=True)
    slide_cases()


if __name__ == "__main__":
    main()
