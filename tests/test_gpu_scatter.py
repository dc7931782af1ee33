"""Sigma scattered straight into the GF-layout point owners over NVLink.

Two ranks (spawned processes): NCCL with one GPU each, or -- so the path runs on a 1-GPU
box too -- gloo with both processes on cuda:0 (the CUDA-IPC mappings are then same-device
peer memory and the all-to-alls run on host copies).  The peer-scatter epilogue
(``sse_sigma_device_scatter`` into CUDA-IPC-mapped buffers) and the fully fused
variant that also reads G from the owners' point buffers with TMA
(``sse_sigma_device_peer``), and Pi with G read the same way (``sse_pi_device_peer``), must equal, bitwise, Sigma computed into atom slabs
and returned with the NCCL all-to-all (``dist.atom_slab_to_points``); the G slab pulled from the
point owners (``sse_slab_from_points``) must equal the slab filled directly.
"""

import os
import socket

import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, backend="nccl"):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1912_08810_b200 import dist as sdist
    from paper_1912_08810_b200.inputs import default_grid
    from paper_1912_08810_b200.problem import ShardProblem
    from paper_1912_08810_b200.types import SimParams, build_neighbor_map

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    device = rank if backend == "nccl" else 0
    torch.cuda.set_device(device)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", device))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = SimParams(n_kz=3, n_qz=2, n_E=37, n_w=13, n_A=26, n_B=4, n_orb=12)
        idx = build_neighbor_map(p.n_A, p.n_B).idx
        prob = ShardProblem(p, rank=rank, world=world, device=device, seed=3, grid=default_grid(p), idx=idx)
        prob.allocate()
        prob.fill(owned_g_only=False)
        prob.preprocess()
        prob.sigma()

        def to_points(t):  # the all-to-all return path (gloo: on host copies)
            if backend == "nccl":
                return sdist.atom_slab_to_points(t, idx, p.n_kz, p.n_E)
            return sdist.atom_slab_to_points(t.cpu().contiguous(), idx, p.n_kz, p.n_E).to(prob.device)

        ref = [to_points(prob.sig[pol]) for pol in range(2)]
        peer = sdist.PeerPointBuffers(p.n_kz, p.n_E, p.n_A, p.n_orb, device=device)
        for t in peer.tensors:
            t.fill_(float("nan"))
        torch.cuda.synchronize()
        dist.barrier()
        prob.sigma_scatter(peer)
        torch.cuda.synchronize()
        dist.barrier()  # every rank's peer stores have landed
        ok = all(torch.equal(peer.tensors[pol], ref[pol]) for pol in range(2))
        finite = all(bool(torch.isfinite(torch.view_as_real(t)).all()) for t in peer.tensors)
        # fully fused: G read from the point owners too (their GF-layout buffers)
        peer_g = sdist.PeerPointBuffers(p.n_kz, p.n_E, p.n_A, p.n_orb, device=device)
        own = slice(prob.lo - prob.glo, prob.hi - prob.glo)
        for pol in range(2):
            peer_g.tensors[pol].copy_(to_points(prob.g[pol][own].contiguous()))
        for t in peer.tensors:
            t.fill_(float("nan"))
        torch.cuda.synchronize()
        dist.barrier()
        prob.sigma_peer(peer_g, peer)
        torch.cuda.synchronize()
        dist.barrier()
        ok_fused = all(torch.equal(peer.tensors[pol], ref[pol]) for pol in range(2))
        # Pi from the point layout too (K5 reads G2, K6 reads G1 over NVLink) == Pi from the slabs
        prob.pi()
        pi_ref = [t.clone() for t in prob.pi_out]
        for t in prob.pi_out:
            t.fill_(float("nan"))
        prob.pi_peer(peer_g)
        torch.cuda.synchronize()
        ok_pi = all(torch.equal(prob.pi_out[pol], pi_ref[pol]) for pol in range(2))
        ok_fused = ok_fused and ok_pi
        # the whole G slab (owned + halo) pulled from the point owners == the slab filled directly
        g_ref = [t.clone() for t in prob.g]
        for t in prob.g:
            t.fill_(float("nan"))
        torch.cuda.synchronize()
        dist.barrier()
        prob.pull_g(peer_g)
        torch.cuda.synchronize()
        ok_fused = ok_fused and all(torch.equal(prob.g[pol], g_ref[pol]) for pol in range(2))
        dist.barrier()
        peer_g.close()
        peer.close()
        res = [None] * world
        dist.all_gather_object(res, (ok, finite, ok_fused))
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("backend", ["gloo", "nccl"])
def test_peer_scatter_and_gather_equal_all_to_all_bitwise(backend):
    import multiprocessing as mp

    import torch

    if backend == "nccl" and torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (the gloo case runs both ranks on one GPU)")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, backend)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    assert all(ok and fin for ok, fin, _ in res), res
    assert all(fused for _, _, fused in res), res


@pytest.mark.parametrize("world,self_rank,atom_major", [(3, 1, True), (3, -1, False), (1, 0, True)])
def test_slab_from_points_single_process(world, self_rank, atom_major):
    """``sse_slab_from_points`` with every "rank's" point buffer on this GPU: the slab equals the
    tensor sliced directly, for ragged point ranges, a rotated start and both slab layouts."""
    import torch

    from paper_1912_08810_b200 import dist as sdist
    from paper_1912_08810_b200 import sse as dev

    n_kz, n_e, n_a, n_o = 2, 13, 11, 3
    g = torch.randn(n_kz, n_e, n_a, n_o, n_o, dtype=torch.complex128, device="cuda")
    pts = sdist.point_chunks(n_kz, n_e, world)
    flat = g.reshape(n_kz * n_e, n_a, n_o, n_o)
    bufs = [flat[a:b].contiguous() for a, b in pts]
    pt_lo = [a for a, _ in pts] + [pts[-1][1]]
    glo, ghi = 3, 9
    want = g[:, :, glo:ghi]
    if atom_major:
        want = want.permute(2, 0, 1, 3, 4)
    out = torch.full_like(want.contiguous(), float("nan"))
    dev.slab_from_points([b.data_ptr() for b in bufs], pt_lo, out, n_kz=n_kz, n_e=n_e, n_a=n_a, g_atom0=glo,
                         atom_major=atom_major, self_rank=self_rank)
    torch.cuda.synchronize()
    assert torch.equal(out, want.contiguous())
    with pytest.raises(ValueError, match="self_rank"):
        dev.slab_from_points([b.data_ptr() for b in bufs], pt_lo, out, n_kz=n_kz, n_e=n_e, n_a=n_a,
                             g_atom0=glo, atom_major=atom_major, self_rank=world)
