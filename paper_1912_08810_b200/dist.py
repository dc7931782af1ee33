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
