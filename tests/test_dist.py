"""Multi-rank atom sharding on CPU: world_size-2 gloo halo exchange + sharded Sigma.

The GPU kernel is replaced here by the oracle as each rank's local compute
(test-only); what is tested is the host-side plan, the halo exchange over
torch.distributed and the stitching, which are the same code the NCCL bench
runs.
"""

import os
import socket

import numpy as np
import pytest

from paper_1912_08810_b200 import dist as sdist
from paper_1912_08810_b200 import inputs
from paper_1912_08810_b200.problem import chunk
from paper_1912_08810_b200.types import SimParams, build_neighbor_map


def test_halo_plan_chain_map():
    idx = build_neighbor_map(16, 4).idx
    plans = [sdist.halo_plan(idx, 4, r) for r in range(4)]
    assert [(p.lo, p.hi) for p in plans] == [(0, 4), (4, 8), (8, 12), (12, 16)]
    assert [(p.glo, p.ghi) for p in plans] == [(0, 6), (2, 10), (6, 14), (10, 16)]
    # every receive is matched by exactly one send
    recv = sorted((p.rank, t.peer, t.atom0, t.atom1) for p in plans for t in p.recvs)
    send = sorted((t.peer, p.rank, t.atom0, t.atom1) for p in plans for t in p.sends)
    assert recv == send
    assert plans[1].halo_atoms() == 4


def test_halo_plan_spans_multiple_owners():
    # chunks of 1 atom with reach 2: a halo run crosses two owners
    idx = build_neighbor_map(6, 4).idx
    p = sdist.halo_plan(idx, 6, 2)
    assert (p.glo, p.ghi) == (0, 5)
    assert sorted((t.peer, t.atom0, t.atom1) for t in p.recvs) == [(0, 0, 1), (1, 1, 2), (3, 3, 4), (4, 4, 5)]


def test_chunks_match_reference_partition():
    # distsim._chunks: ceil division, short or empty tails
    assert [chunk(10, 3, r) for r in range(3)] == [(0, 4), (4, 8), (8, 10)]
    assert [chunk(5, 7, r) for r in range(7)][-2:] == [(5, 5), (5, 5)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, p, seed, result_q):
    import torch
    import torch.distributed as dist

    from oracle import sse_oracle as orc

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    idx = build_neighbor_map(p.n_A, p.n_B).idx
    plan = sdist.halo_plan(idx, world, rank)
    n_slab = plan.ghi - plan.glo
    # owner-computes inputs: only owned atoms are generated locally (atom-major slab)
    slabs = []
    for tid in (inputs.G_LESSER, inputs.G_GREATER):
        t = torch.full((n_slab, p.n_kz, p.n_E, p.n_orb, p.n_orb), float("nan"), dtype=torch.complex128)
        own = inputs.atom_keyed_values(seed, tid, np.arange(plan.lo, plan.hi), p.n_kz * p.n_E, p.n_orb**2)
        t[plan.lo - plan.glo:plan.hi - plan.glo] = torch.from_numpy(
            own.reshape(plan.hi - plan.lo, p.n_kz, p.n_E, p.n_orb, p.n_orb))
        slabs.append(t)
    sdist.exchange_halos(slabs, plan)
    # the received halo equals the generator's values for those atoms (bitwise)
    for t, tid in zip(slabs, (inputs.G_LESSER, inputs.G_GREATER)):
        want = inputs.atom_keyed_values(seed, tid, np.arange(plan.glo, plan.ghi), p.n_kz * p.n_E, p.n_orb**2)
        assert np.array_equal(t.numpy().reshape(want.shape), want)
    # local Sigma of owned atoms from the slab (oracle stands in for the kernel)
    g_l = np.ascontiguousarray(np.moveaxis(slabs[0].numpy(), 0, 2))
    g_g = np.ascontiguousarray(np.moveaxis(slabs[1].numpy(), 0, 2))
    sub_idx = np.zeros((n_slab, p.n_B), dtype=np.int64)
    sub_idx[plan.lo - plan.glo:plan.hi - plan.glo] = idx[plan.lo:plan.hi] - plan.glo
    rng = np.random.default_rng(seed + 1)
    shape = (p.n_qz, p.n_w, p.n_A, p.n_B, 3, 3)
    dc_l = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    dc_g = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    dh = inputs.atom_keyed_dh(seed, p, np.arange(p.n_A))
    sl = slice(plan.glo, plan.ghi)
    off, wt = inputs.default_grid(p).offsets, inputs.default_grid(p).weights
    pairs = [(a - plan.glo, s) for a in range(plan.lo, plan.hi) for s in range(p.n_B)]
    out_l, out_g = orc.sigma_batched_fused(g_l, g_g, dc_l[:, :, sl], dc_g[:, :, sl], dh[sl], sub_idx,
                                           np.array(off), np.array(wt), pairs=pairs)
    own = slice(plan.lo - plan.glo, plan.hi - plan.glo)
    parts = [None] * world
    dist.all_gather_object(parts, (plan.lo, plan.hi, out_l[:, :, own], out_g[:, :, own]))
    if rank == 0:
        result_q.put(parts)
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_sigma_matches_single_process():
    import multiprocessing as mp

    from oracle import sse_oracle as orc

    p = SimParams(n_kz=2, n_qz=2, n_E=6, n_w=3, n_A=9, n_B=4, n_orb=3)
    seed, world = 3, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, p, seed, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    parts = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    # single-process reference on the full tensors
    idx = build_neighbor_map(p.n_A, p.n_B).idx
    g_l = inputs.atom_keyed_electron(seed, inputs.G_LESSER, p, np.arange(p.n_A))
    g_g = inputs.atom_keyed_electron(seed, inputs.G_GREATER, p, np.arange(p.n_A))
    rng = np.random.default_rng(seed + 1)
    shape = (p.n_qz, p.n_w, p.n_A, p.n_B, 3, 3)
    dc_l = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    dc_g = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    dh = inputs.atom_keyed_dh(seed, p, np.arange(p.n_A))
    grid = inputs.default_grid(p)
    ref_l, ref_g = orc.sigma_batched_fused(g_l, g_g, dc_l, dc_g, dh, idx, np.array(grid.offsets),
                                           np.array(grid.weights))
    got_l = np.concatenate([x[2] for x in parts], axis=2)
    got_g = np.concatenate([x[3] for x in parts], axis=2)
    assert [(x[0], x[1]) for x in parts] == [(0, 5), (5, 9)]
    # identical per-atom arithmetic on identical inputs: bitwise
    assert np.array_equal(got_l, ref_l) and np.array_equal(got_g, ref_g)


def _a2a_worker(rank, world, port, p, seed, result_q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    idx = build_neighbor_map(p.n_A, p.n_B).idx
    full = inputs.atom_keyed_electron(seed, inputs.G_LESSER, p, np.arange(p.n_A))  # [Nkz, NE, NA, No, No]
    flat = full.reshape(p.n_kz * p.n_E, p.n_A, p.n_orb, p.n_orb)
    ps, pe = sdist.point_chunks(p.n_kz, p.n_E, world)[rank]
    g_pts = torch.from_numpy(np.ascontiguousarray(flat[ps:pe]))
    slab = sdist.points_to_atom_slab(g_pts, idx, p.n_kz, p.n_E)
    plan = sdist.halo_plan(idx, world, rank)
    want = np.moveaxis(full[:, :, plan.glo:plan.ghi], 2, 0)
    ok_fwd = np.array_equal(slab.numpy(), want)
    own = slab[plan.lo - plan.glo:plan.hi - plan.glo] * 2  # stand-in for this rank's Sigma
    back = sdist.atom_slab_to_points(own.contiguous(), idx, p.n_kz, p.n_E)
    ok_back = np.array_equal(back.numpy(), 2 * flat[ps:pe])
    res = [None] * world
    dist.all_gather_object(res, (ok_fwd, ok_back))
    if rank == 0:
        result_q.put(res)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gf_points_to_atom_slabs_all_to_all(world):
    """GF (k, E)-point layout -> atom slabs with halos -> Sigma back, one all-to-all each."""
    import multiprocessing as mp

    p = SimParams(n_kz=2, n_qz=2, n_E=7, n_w=2, n_A=10, n_B=4, n_orb=2)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_a2a_worker, args=(r, world, port, p, 4, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert all(f and b for f, b in res), res


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_a2a_bytes_within_reference_tiled_model(world):
    """the all-to-all volume against the reference's tiled model with T_E = 1, T_A = P
    (comm.dace_volume, comm.py:86-106: 32 Nkz (NE/T_E + 2 Nw)(NA/T_A + NB) No^2 bytes per direction)."""
    from paper_1912_08810_b200.inputs import config

    p, grid, nmap = config("paper")
    model = 32 * p.n_kz * (p.n_E + 2 * p.n_w) * (p.n_A / world + p.n_B) * p.n_orb**2
    for rank in range(world):
        b = sdist.a2a_bytes(nmap.idx, p.n_kz, p.n_E, p.n_orb, world, rank)
        assert b["g_in"] <= model
        assert b["sigma_back"] <= model
    ref = "/root/reference/pkg/src"
    if os.path.isdir(ref):
        import sys

        sys.path.insert(0, ref)
        try:
            from negflow import comm
            from negflow.params import SimParams as RefParams

            rp = RefParams(n_kz=p.n_kz, n_qz=p.n_qz, n_E=p.n_E, n_w=p.n_w, n_A=p.n_A, n_B=p.n_B,
                           n_orb=p.n_orb, bnum=p.bnum)
            plan = comm.dace_volume(rp, 1, world)
            assert abs(plan.per_process_bytes[comm.ELECTRON_G] - model) <= 1e-6 * model
            if world > 1:
                assert comm.optimize_tiles(rp, world).t_e == 1  # the tiling this all-to-all implements
        finally:
            sys.path.remove(ref)


def _phonon_a2a_worker(rank, world, port, p, seed, result_q):
    import torch
    import torch.distributed as dist

    from oracle import sse_oracle as orc

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    idx = build_neighbor_map(p.n_A, p.n_B).idx
    rng = np.random.default_rng(seed)
    shape = (p.n_qz, p.n_w, p.n_A, p.n_B + 1, 3, 3)
    d_full = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    pi_full = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    n_pts = p.n_qz * p.n_w
    ps, pe = sdist.chunk(n_pts, world, rank)
    # D arrives from the phonon GF phase's (q, w) points; preprocess_D on the slab == on the full tensor
    d_pts = torch.from_numpy(np.ascontiguousarray(d_full.reshape(n_pts, *shape[2:])[ps:pe]))
    slab = sdist.phonon_points_to_slab(d_pts, idx, p.n_qz, p.n_w).numpy()
    plan = sdist.halo_plan(idx, world, rank)
    ok_d = np.array_equal(slab, d_full[:, :, plan.glo:plan.ghi])
    ref_l, _ = orc.preprocess_D(d_full, d_full, idx)
    # reverse slots need the full map: evaluate the owned rows from the slab by the same formula
    got = np.empty_like(ref_l[:, :, plan.lo:plan.hi])
    for a in range(plan.lo, plan.hi):
        for s in range(p.n_B):
            b = int(idx[a, s])
            r = int(np.nonzero(idx[b] == a)[0][0])
            got[:, :, a - plan.lo, s] = (slab[:, :, b - plan.glo, 1 + r] - slab[:, :, b - plan.glo, 0]
                                         - slab[:, :, a - plan.glo, 0] + slab[:, :, a - plan.glo, 1 + s])
    ok_pre = np.array_equal(got, ref_l[:, :, plan.lo:plan.hi])
    # Pi of the owned atoms returns to the (q, w) point owners
    lo, hi = sdist.chunk(p.n_A, world, rank)
    back = sdist.pi_to_points(torch.from_numpy(np.ascontiguousarray(pi_full[:, :, lo:hi])), p.n_A, p.n_qz, p.n_w)
    ok_pi = np.array_equal(back.numpy(), pi_full.reshape(n_pts, *shape[2:])[ps:pe])
    res = [None] * world
    dist.all_gather_object(res, (ok_d, ok_pre, ok_pi))
    if rank == 0:
        result_q.put(res)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_phonon_points_to_slab_and_pi_return(world):
    """SURVEY 8f-3, phonon side: raw D from the (q, w)-point layout -> halo'd slabs (preprocess_D
    on them matches the full tensor bitwise), and Pi of the owned atoms back to the point owners."""
    import multiprocessing as mp

    p = SimParams(n_kz=2, n_qz=2, n_E=7, n_w=3, n_A=11, n_B=4, n_orb=2)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_phonon_a2a_worker, args=(r, world, port, p, 6, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert all(all(x) for x in res), res
