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


def points_to_atom_slab(g_pts, idx: np.ndarray, n_kz: int, n_e: int, group=None):
    """[pts_r, NA, No, No] (this rank's GF points) -> atom-major slab [gA, Nkz, NE, No, No].

    Collective over the group; every rank passes its own point rows.
    """
    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    pts = point_chunks(n_kz, n_e, world)
    slabs = _slabs(idx, world)
    no2 = g_pts.shape[-1] * g_pts.shape[-2]
    flat = g_pts.reshape(g_pts.shape[0], g_pts.shape[1], no2)
    send = torch.cat([flat[:, glo:ghi].reshape(-1) for (_, _, glo, ghi) in slabs]) if flat.numel() else \
        flat.new_zeros(0)
    send_sizes = [flat.shape[0] * (ghi - glo) * no2 for (_, _, glo, ghi) in slabs]
    lo, hi, glo, ghi = slabs[rank]
    gA = ghi - glo
    recv_sizes = [(pe - ps) * gA * no2 for (ps, pe) in pts]
    recv = flat.new_empty(sum(recv_sizes))
    _all_to_all(recv, send, recv_sizes, send_sizes, group)
    slab = flat.new_empty((gA, n_kz * n_e, no2))
    pos = 0
    for (ps, pe), sz in zip(pts, recv_sizes):
        if pe > ps:
            slab[:, ps:pe] = recv[pos:pos + sz].view(pe - ps, gA, no2).transpose(0, 1)
        pos += sz
    n_o = g_pts.shape[-1]
    return slab.view(gA, n_kz, n_e, n_o, n_o)


def atom_slab_to_points(sig, idx: np.ndarray, n_kz: int, n_e: int, group=None):
    """Owned-atom Sigma [oA, Nkz, NE, No, No] -> this rank's GF points [pts_r, NA, No, No]."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    pts = point_chunks(n_kz, n_e, world)
    slabs = _slabs(idx, world)
    n_a = idx.shape[0]
    oA, n_o = sig.shape[0], sig.shape[-1]
    no2 = n_o * n_o
    flat = sig.reshape(oA, n_kz * n_e, no2)
    import torch

    send = torch.cat([flat[:, ps:pe].transpose(0, 1).reshape(-1) for (ps, pe) in pts])
    send_sizes = [(pe - ps) * oA * no2 for (ps, pe) in pts]
    ps, pe = pts[rank]
    recv_sizes = [(pe - ps) * (hi - lo) * no2 for (lo, hi, _, _) in slabs]
    recv = flat.new_empty(sum(recv_sizes))
    _all_to_all(recv, send, recv_sizes, send_sizes, group)
    out = flat.new_empty((pe - ps, n_a, no2))
    pos = 0
    for (lo, hi, _, _), sz in zip(slabs, recv_sizes):
        if hi > lo:
            out[:, lo:hi] = recv[pos:pos + sz].view(pe - ps, hi - lo, no2)
        pos += sz
    return out.view(pe - ps, n_a, n_o, n_o)


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

        for ptr in self._opened:
            _lib.check(self._lib.sse_ipc_close(self._ctx.handle, ctypes.c_void_p(ptr)))
        self._opened = []
        self.tensors = []
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
