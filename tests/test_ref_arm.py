"""The reference arm of bench.py: the unmodified reference, one (atom, slot) pair at a time.

bench.py --impl reference and the cpu_baseline leg time negflow.sse.sse_sigma(BATCHED_FUSED)
(from oracle/_ref, built by oracle/make_ref.py) on single-pair sub-problems and scale by NA*NB.
These CPU tests check that decomposition against the reference's own full evaluation.
"""

import json
import os

import numpy as np
import pytest

import bench
from oracle import make_ref
from oracle.ref import import_negflow, ref_path
from paper_1912_08810_b200 import inputs


@pytest.fixture(scope="module")
def nf():
    if ref_path() is None:
        pytest.skip("reference not available (run oracle/make_ref.py in the build container)")
    return import_negflow()


def test_pairs_cover_chain_ends_and_every_slot():
    p = inputs.CONFIGS["paper"]
    pairs = bench.sample_pairs(p)
    atoms = {a for a, _ in pairs}
    assert len(pairs) >= 8 and {0, p.n_A - 1} <= atoms
    assert {s for _, s in pairs} == set(range(p.n_B))


def test_pair_sum_equals_reference_full_evaluation(nf):
    """sum_s negflow_pair(a, s) == negflow's own Sigma[:, :, a] of the whole config (tiny)."""
    p, grid, nmap = inputs.config("tiny")
    idx = nmap.idx
    atoms = np.arange(p.n_A)
    g_l = inputs.atom_keyed_electron(0, inputs.G_LESSER, p, atoms)
    g_g = inputs.atom_keyed_electron(0, inputs.G_GREATER, p, atoms)
    d_l = inputs.atom_keyed_phonon(0, inputs.D_LESSER, p, atoms)
    d_g = inputs.atom_keyed_phonon(0, inputs.D_GREATER, p, atoms)
    dh = inputs.atom_keyed_dh(0, p, atoms)
    ref_nmap = nf.device.build_neighbor_map(p.n_A, p.n_B)
    assert np.array_equal(ref_nmap.idx, idx)
    dc = nf.sse.preprocess_D(nf.gf.GreensTensor(d_l, d_g), ref_nmap)
    ref_p = nf.params.SimParams(n_kz=p.n_kz, n_qz=p.n_qz, n_E=p.n_E, n_w=p.n_w, n_A=p.n_A, n_B=p.n_B, n_orb=p.n_orb)
    full = nf.sse.sse_sigma(nf.sse.SseVariant.BATCHED_FUSED, nf.gf.GreensTensor(g_l, g_g), dc, dh, ref_nmap,
                            nf.params.default_grid(ref_p))
    scale = max(np.max(np.abs(full.lesser)), np.max(np.abs(full.greater)))
    for a in (0, 1, p.n_A // 2, p.n_A - 1):
        runs = [bench.negflow_pair(nf, p, idx, a, s) for s in range(p.n_B)]
        got_l = sum(r["sigma_l"] for r in runs)
        got_g = sum(r["sigma_g"] for r in runs)
        dev = max(np.max(np.abs(got_l - full.lesser[:, :, a])), np.max(np.abs(got_g - full.greater[:, :, a])))
        assert dev / scale <= 1e-13, (a, dev / scale)


def test_staged_reference_matches_source():
    """oracle/_ref holds bytecode of exactly the reference's current sources (sha256 manifest)."""
    if not os.path.isdir(make_ref.SRC):
        pytest.skip("/root/reference absent (GPU box): nothing to compare against")
    if not os.path.isfile(make_ref.MANIFEST):
        make_ref.stage()
    with open(make_ref.MANIFEST) as fh:
        manifest = json.load(fh)
    srcs = sorted(f for f in os.listdir(make_ref.SRC) if f.endswith(".py"))
    assert sorted(manifest["files"]) == srcs
    for f in srcs:
        assert manifest["files"][f] == make_ref.sha256(os.path.join(make_ref.SRC, f)), f
    import zipfile

    names = zipfile.ZipFile(make_ref.DST).namelist()
    assert sorted(names) == sorted(f"negflow/{f[:-3]}.pyc" for f in srcs)
    assert not any(n.endswith(".py") for n in names), "no reference source in the repo"
