"""Atom-sharded multi-GPU SSE: halo plan and halo exchange (torch.distributed).

One process per GPU.  Rank r owns the contiguous atom chunk [lo, hi)
(problem.chunk, distsim.py:117-120); Sigma of an owned atom needs G at
f(a, s) only (sse.py:151-157), so the single data exchange of an SSE step is
the G halo: every rank receives, from the owners, the atoms of its slab
[glo, ghi) it does not own.  This is the reference tiled scheme's forward
round (distsim.py:253-353, atom halo max(NB//2, max_reach), distsim.py:290)
with T_E = 1, the tiling the reference's own optimiser picks for every
BASELINE config (comm.py:117-137).  Dc, dH and Sigma stay sharded; there is
no reduction, so results are bitwise independent of the rank count.

On NCCL the sends/receives of a step form one batch_isend_irecv group (no
ordering deadlock, NVLink P2P); on gloo (CPU tests) they are posted as
individual isend/irecv.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .problem import chunk


@dataclass(frozen=True)
class Transfer:
    peer: int
    atom0: int
    atom1: int  # exclusive


@dataclass(frozen=True)
class HaloPlan:
    rank: int
    world: int
    lo: int
    hi: int
    glo: int
    ghi: int
    recvs: tuple[Transfer, ...]
    sends: tuple[Transfer, ...]

    def halo_atoms(self) -> int:
        return sum(t.atom1 - t.atom0 for t in self.recvs)


def slab_range(idx: np.ndarray, lo: int, hi: int) -> tuple[int, int]:
    rows = idx[lo:hi]
    return int(min(lo, rows.min())), int(max(hi, rows.max() + 1))


def _split_by_owner(a0: int, a1: int, n_a: int, world: int, peer_self: int) -> list[Transfer]:
    out = []
    size = -(-n_a // world)
    x = a0
    while x < a1:
        owner = x // size
        end = min(a1, (owner + 1) * size)
        if owner != peer_self:
            out.append(Transfer(owner, x, end))
        x = end
    return out


def halo_plan(idx: np.ndarray, world: int, rank: int) -> HaloPlan:
    """Receives and sends of ``rank`` for the G halo of one SSE step."""
    n_a = idx.shape[0]
    slabs = []
    for r in range(world):
        lo, hi = chunk(n_a, world, r)
        slabs.append((lo, hi) + (slab_range(idx, lo, hi) if hi > lo else (lo, hi)))
    lo, hi, glo, ghi = slabs[rank]
    recvs = _split_by_owner(glo, lo, n_a, world, rank) + _split_by_owner(hi, ghi, n_a, world, rank)
    sends = []
    for r, (rlo, rhi, rglo, rghi) in enumerate(slabs):
        if r == rank or rhi <= rlo:
            continue
        for t in _split_by_owner(rglo, rlo, n_a, world, r) + _split_by_owner(rhi, rghi, n_a, world, r):
            if t.peer == rank:
                sends.append(Transfer(r, t.atom0, t.atom1))
    return HaloPlan(rank, world, lo, hi, glo, ghi, tuple(recvs), tuple(sends))


def exchange_halos(slabs, plan: HaloPlan, group=None) -> None:
    """Fill the halo atoms of atom-major slabs [gA, ...] (one per polarity) from their owners."""
    import torch
    import torch.distributed as dist

    def view(t, a0, a1):
        v = t[a0 - plan.glo:a1 - plan.glo]
        return torch.view_as_real(v) if v.is_complex() else v

    ops = []
    for t in slabs:
        for tr in plan.sends:
            ops.append(dist.P2POp(dist.isend, view(t, tr.atom0, tr.atom1), tr.peer, group))
        for tr in plan.recvs:
            ops.append(dist.P2POp(dist.irecv, view(t, tr.atom0, tr.atom1), tr.peer, group))
    if not ops:
        return
    if dist.get_backend(group) == "nccl":
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    else:
        reqs = [op.op(op.tensor, op.peer, group=group) for op in ops]
        for req in reqs:
            req.wait()


def halo_bytes(plan: HaloPlan, bytes_per_atom: int, polarities: int = 2) -> int:
    return polarities * plan.halo_atoms() * bytes_per_atom


# ---------------------------------------------------------------------------
# GF-phase layout <-> SSE atom slabs
#
# The GF phase owns flattened (k, E) points in contiguous chunks
# (distsim._PointLayout, distsim.py:130-150): rank r holds G[points_r, all
# atoms].  The SSE phase needs atom slabs (owned atoms + halo) over all points.
# One all-to-all moves each rank's point rows of every destination's slab
# (halo included: no separate halo round), and one all-to-all returns Sigma to
# the point owners: the tiled scheme's two rounds (distsim.py:300-315) with
# T_E = 1, on NCCL.
# ---------------------------------------------------------------------------


def point_chunks(n_kz: int, n_e: int, world: int) -> list[tuple[int, int]]:
    """Flattened (k, E) ownership of the GF phase (distsim.py:117-120,130-150)."""
    return [chunk(n_kz * n_e, world, r) for r in range(world)]


def _slabs(idx: np.ndarray, world: int):
    out = []
    n_a = idx.shape[0]
    for r in range(world):
        lo, hi = chunk(n_a, world, r)
        glo, ghi = slab_range(idx, lo, hi) if hi > lo else (lo, hi)
        out.append((lo, hi, glo, ghi))
    return out


def points_to_columns(x_pts, ranges, n_pts: int, atom_major: bool, group=None):
    """Point-distributed rows -> this rank's column slab, one all-to-all.

    ``x_pts``: this rank's point rows [pts_r, NA, *blk] (``point_chunks`` of
    ``n_pts``); ``ranges[r] = (c0, c1)``: the atom columns rank r needs
    (its slab with halo, or its owned atoms).  Returns this rank's
    [c1-c0, n_pts, *blk] (``atom_major``) or [n_pts, c1-c0, *blk].
    """
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    pts = [chunk(n_pts, world, r) for r in range(world)]
    blk = tuple(x_pts.shape[2:])
    nblk = int(np.prod(blk)) if blk else 1
    flat = x_pts.reshape(x_pts.shape[0], x_pts.shape[1], nblk)
    send = flat.new_empty(sum(flat.shape[0] * (c1 - c0) * nblk for c0, c1 in ranges))
    pos = 0
    for c0, c1 in ranges:
        n = flat.shape[0] * (c1 - c0) * nblk
        send[pos:pos + n] = flat[:, c0:c1].reshape(-1)
        pos += n
    send_sizes = [flat.shape[0] * (c1 - c0) * nblk for c0, c1 in ranges]
    c0, c1 = ranges[rank]
    width = c1 - c0
    recv_sizes = [(pe - ps) * width * nblk for ps, pe in pts]
    recv = flat.new_empty(sum(recv_sizes))
    _all_to_all(recv, send, recv_sizes, send_sizes, group)
    out = flat.new_empty((width, n_pts, nblk) if atom_major else (n_pts, width, nblk))
    pos = 0
    for (ps, pe), sz in zip(pts, recv_sizes):
        if pe > ps:
            part = recv[pos:pos + sz].view(pe - ps, width, nblk)
            if atom_major:
                out[:, ps:pe] = part.transpose(0, 1)
            else:
                out[ps:pe] = part
        pos += sz
    return out.view(*out.shape[:2], *blk)


def columns_to_points(y, ranges, n_pts: int, n_a: int, atom_major: bool, group=None):
    """This rank's columns ``ranges[rank]`` of every point -> the point owners' rows [pts_r, NA, *blk].

    ``y``: [c1-c0, n_pts, *blk] (``atom_major``) or [n_pts, c1-c0, *blk]; the
    ranges of all ranks must partition [0, NA) (owned atoms).
    """
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    pts = [chunk(n_pts, world, r) for r in range(world)]
    c0, c1 = ranges[rank]
    width = c1 - c0
    blk = tuple(y.shape[2:])
    nblk = int(np.prod(blk)) if blk else 1
    flat = y.reshape(y.shape[0], y.shape[1], nblk)
    send = flat.new_empty(n_pts * width * nblk)
    pos = 0
    for ps, pe in pts:
        n = (pe - ps) * width * nblk
        part = flat[:, ps:pe].transpose(0, 1) if atom_major else flat[ps:pe]
        send[pos:pos + n] = part.reshape(-1)
        pos += n
    send_sizes = [(pe - ps) * width * nblk for ps, pe in pts]
    ps, pe = pts[rank]
    recv_sizes = [(pe - ps) * (r1 - r0) * nblk for r0, r1 in ranges]
    recv = flat.new_empty(sum(recv_sizes))
    _all_to_all(recv, send, recv_sizes, send_sizes, group)
    out = flat.new_empty((pe - ps, n_a, nblk))
    pos = 0
    for (r0, r1), sz in zip(ranges, recv_sizes):
        if r1 > r0:
            out[:, r0:r1] = recv[pos:pos + sz].view(pe - ps, r1 - r0, nblk)
        pos += sz
    return out.view(pe - ps, n_a, *blk)


def halo_ranges(idx: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Each rank's atom slab (owned atoms + every neighbour f(a, s)): the columns it reads."""
    return [(glo, ghi) for (_, _, glo, ghi) in _slabs(idx, world)]


def owned_ranges(n_a: int, world: int) -> list[tuple[int, int]]:
    return [chunk(n_a, world, r) for r in range(world)]


def points_to_atom_slab(g_pts, idx: np.ndarray, n_kz: int, n_e: int, group=None):
    """G: [pts_r, NA, No, No] (this rank's GF points) -> atom-major slab [gA, Nkz, NE, No, No].

    Collective over the group; every rank passes its own point rows.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group)
    slab = points_to_columns(g_pts, halo_ranges(idx, world), n_kz * n_e, True, group)
    return slab.view(slab.shape[0], n_kz, n_e, *g_pts.shape[2:])


def atom_slab_to_points(sig, idx: np.ndarray, n_kz: int, n_e: int, group=None):
    """Owned-atom Sigma [oA, Nkz, NE, No, No] -> this rank's GF points [pts_r, NA, No, No]."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n_a = idx.shape[0]
    y = sig.reshape(sig.shape[0], n_kz * n_e, *sig.shape[3:])
    return columns_to_points(y, owned_ranges(n_a, world), n_kz * n_e, n_a, True, group)


def phonon_points_to_slab(d_pts, idx: np.ndarray, n_qz: int, n_w: int, group=None):
    """Raw D from the phonon GF phase's (q, w) points [pts_r, NA, NB+1, 3, 3] -> this rank's
    grid-major D slab [Nqz, Nw, gA, NB+1, 3, 3] (halo included: preprocess_D reads D at f(a, s))."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    slab = points_to_columns(d_pts, halo_ranges(idx, world), n_qz * n_w, False, group)
    return slab.view(n_qz, n_w, *slab.shape[1:])


def pi_to_points(pi_owned, n_a: int, n_qz: int, n_w: int, group=None):
    """Owned-atom Pi [Nqz, Nw, oA, NB+1, 3, 3] -> the phonon GF phase's (q, w) point owners
    [pts_r, NA, NB+1, 3, 3] (the Pi return of the tiled scheme)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    y = pi_owned.reshape(n_qz * n_w, *pi_owned.shape[2:])
    return columns_to_points(y, owned_ranges(n_a, world), n_qz * n_w, n_a, False, group)


def _all_to_all(recv, send, recv_sizes, send_sizes, group):
    """all_to_all_single on complex tensors (NCCL/gloo see their real view)."""
    import torch
    import torch.distributed as dist

    r = torch.view_as_real(recv).reshape(-1) if recv.is_complex() else recv
    s = torch.view_as_real(send).reshape(-1) if send.is_complex() else send
    f = 2 if recv.is_complex() else 1
    dist.all_to_all_single(r, s, [x * f for x in recv_sizes], [x * f for x in send_sizes], group=group)


def a2a_bytes(idx: np.ndarray, n_kz: int, n_e: int, n_o: int, world: int, rank: int,
              polarities: int = 2) -> dict:
    """Bytes rank ``rank`` receives in the two all-to-alls of one SSE step (G in, Sigma back).

    Own rows are included (they are copied, not sent), matching the reference's
    model that counts a process's whole window (comm.dace_volume, comm.py:86-106).
    """
    blk = n_o * n_o * 16 * polarities
    pts = point_chunks(n_kz, n_e, world)
    slabs = _slabs(idx, world)
    lo, hi, glo, ghi = slabs[rank]
    ps, pe = pts[rank]
    g_in = n_kz * n_e * (ghi - glo) * blk
    sigma_in = (pe - ps) * idx.shape[0] * blk
    return {"g_in": g_in, "sigma_back": sigma_in,
            "g_in_from_peers": g_in - (pe - ps) * (ghi - glo) * blk}


# ---------------------------------------------------------------------------
# Sigma straight into the owners' point-layout buffers (NVLink peer stores)
# ---------------------------------------------------------------------------


class PeerPointBuffers:
    """This rank's GF-layout Sigma buffers [pts_r, NA, No, No] (both polarities), mapped
    into every rank of the group by CUDA IPC, so the Sigma kernel's epilogue can store
    each (k, E, atom) block directly into its owner's buffer over NVLink
    (``sse.sigma_device_scatter``): the return all-to-all fused into the compute.

    Collective over the group (handle exchange); call :meth:`close` on every rank.
    """

    def __init__(self, n_kz: int, n_e: int, n_a: int, n_o: int, device: int, group=None):
        import torch
        import torch.distributed as dist

        from . import _lib

        self.group = group
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        if self.world > 8:
            raise ValueError("peer scatter supports up to 8 ranks")
        self.pts = point_chunks(n_kz, n_e, self.world)
        self.pt_lo = [a for a, _ in self.pts] + [self.pts[-1][1]]
        ps, pe = self.pts[self.rank]
        self.shape = (pe - ps, n_a, n_o, n_o)
        nbytes = max(1, (pe - ps) * n_a * n_o * n_o * 16)
        self._lib = _lib.load()
        self._ctx = _lib.context(device=device)
        self.local = []
        for _ in range(2):
            ptr = _lib._P()
            _lib.check(self._lib.sse_dev_alloc(self._ctx.handle, nbytes, ctypes.byref(ptr)))
            self.local.append(ptr.value)
        handles = []
        for ptr in self.local:
            h = ctypes.create_string_buffer(_lib.IPC_HANDLE_BYTES)
            _lib.check(self._lib.sse_ipc_handle(self._ctx.handle, ctypes.c_void_p(ptr), h))
            handles.append(h.raw)
        everyone = [None] * self.world
        dist.all_gather_object(everyone, handles, group=group)
        self.remote = []  # [pol][rank] device pointers valid in this process
        self._opened = []
        for pol in range(2):
            row = []
            for r in range(self.world):
                if r == self.rank:
                    row.append(self.local[pol])
                    continue
                ptr = _lib._P()
                _lib.check(self._lib.sse_ipc_open(self._ctx.handle, everyone[r][pol], ctypes.byref(ptr)))
                self._opened.append(ptr.value)
                row.append(ptr.value)
            self.remote.append(row)
        dev = torch.device("cuda", device)
        self.tensors = [_wrap_device(ptr, self.shape, dev) for ptr in self.local]

    def close(self) -> None:
        from . import _lib

        import torch.distributed as dist

        for ptr in self._opened:
            _lib.check(self._lib.sse_ipc_close(self._ctx.handle, ctypes.c_void_p(ptr)))
        self._opened = []
        self.tensors = []
        # every peer has unmapped this rank's buffers before they are freed
        dist.barrier(group=self.group)
        for ptr in self.local:
            _lib.check(self._lib.sse_dev_free(self._ctx.handle, ctypes.c_void_p(ptr)))
        self.local = []


class _CudaArray:
    def __init__(self, ptr: int, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<c16", "data": (ptr, False),
                                         "version": 3, "strides": None}


def _wrap_device(ptr: int, shape, device):
    """A torch complex128 view of library-owned device memory (no copy)."""
    import torch

    return torch.as_tensor(_CudaArray(ptr, shape), device=device)
