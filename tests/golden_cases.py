"""Loader for the golden fixtures in tests/golden (see make_golden.py)."""

from __future__ import annotations

import glob
import hashlib
import json
import os

import numpy as np

from paper_1912_08810_b200.inputs import stream_instance
from paper_1912_08810_b200.types import SimParams

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


class Case:
    """One stream-recipe golden case: regenerated inputs + stored reference outputs."""

    def __init__(self, path):
        data = np.load(path)
        self.meta = json.loads(str(data["meta"]))
        self.name = self.meta["name"]
        self.arrays = {k: data[k] for k in data.files if k != "meta"}
        pr = self.meta["params"]
        self.p = SimParams(**pr)
        self.offsets = np.array(self.meta["offsets"], dtype=np.int64)
        self.weights = np.array(self.meta["weights"], dtype=np.float64)
        self.idx = np.array(self.meta["nmap"], dtype=np.int64)
        g_l, g_g, d_l, d_g, dh = stream_instance(self.meta["seed"], self.p, self.meta["dh_scale"])
        self.inputs_ok = digest(g_l, g_g, d_l, d_g, dh) == self.meta["input_sha256"]
        self.g_l, self.g_g, self.d_l, self.d_g, self.dh = g_l, g_g, d_l, d_g, dh

    def __repr__(self):
        return f"Case({self.name})"


def stream_case_names():
    names = []
    for path in sorted(glob.glob(os.path.join(HERE, "*.npz"))):
        name = os.path.splitext(os.path.basename(path))[0]
        if name not in ("kat_scalar", "criterion5") and not name.startswith("loop_"):
            names.append(name)
    return names


def load_case(name) -> Case:
    return Case(os.path.join(HERE, f"{name}.npz"))


def kat_scalar():
    """Inputs of test_sse.py:175-197 and the stored reference output."""
    data = np.load(os.path.join(HERE, "kat_scalar.npz"))
    meta = json.loads(str(data["meta"]))
    rng = np.random.default_rng(9)

    def rand(shape):
        return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)

    g_l, g_g = rand((1, 1, 2, 1, 1)), rand((1, 1, 2, 1, 1))
    dh = rand((2, 1, 3, 1, 1))
    dc_l, dc_g = rand((1, 1, 2, 1, 3, 3)), rand((1, 1, 2, 1, 3, 3))
    assert digest(g_l, g_g, dh, dc_l, dc_g) == meta["input_sha256"]
    idx = np.array(meta["nmap"], dtype=np.int64)
    return g_l, g_g, dc_l, dc_g, dh, idx, np.array([0]), np.array([0.37]), data["sigma_l"], data["sigma_g"]


def criterion5_instances():
    """Replay test_acceptance.py:139-177's generator; yield inputs + stored output."""
    data = np.load(os.path.join(HERE, "criterion5.npz"))
    metas = json.loads(str(data["meta"]))
    rng = np.random.default_rng(2024)

    def rand(shape):
        return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)

    from paper_1912_08810_b200.types import build_neighbor_map, default_grid

    i = 0
    while i < 50:
        n_kz = int(rng.integers(1, 5))
        n_qz = int(rng.integers(1, n_kz + 1))
        n_e = int(rng.integers(2, 5))
        n_w = int(rng.integers(1, min(4, n_e)))
        n_a = int(rng.choice([2, 4]))
        n_b = int(rng.integers(1, min(3, n_a)))
        n_orb = int(rng.integers(1, 4))
        if n_a % 2 == 1 and n_b % 2 == 1:
            continue
        p = SimParams(n_kz=n_kz, n_qz=n_qz, n_E=n_e, n_w=n_w, n_A=n_a, n_B=n_b, n_orb=n_orb)
        g_l, g_g = rand(p.electron_shape), rand(p.electron_shape)
        d_l, d_g = rand(p.phonon_shape), rand(p.phonon_shape)
        dh = rand((n_a, n_b, 3, n_orb, n_orb))
        assert digest(g_l, g_g, d_l, d_g, dh) == metas[i]["input_sha256"]
        grid = default_grid(p)
        nmap = build_neighbor_map(n_a, n_b)
        yield p, grid, nmap, g_l, g_g, d_l, d_g, dh, data[f"sigma_l_{i}"], data[f"sigma_g_{i}"]
        i += 1
