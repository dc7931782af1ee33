"""Device-resident SSE problem of one rank: synthetic inputs, halos, Sigma.

Atom sharding (the reference optimiser's choice
T_E = 1, T_A = P, comm.py:117-137): rank r owns the contiguous atom chunk
[lo, hi) (distsim.py:117-120 ceil division).  Sigma[:, :, a] needs G at the
atoms f(a, .) only (sse.py:151-157), so each rank holds

* G<, G>   atom-major slab [glo, ghi) = owned atoms + the +-reach halo,
           [gA, Nkz, NE, No, No] (each atom one contiguous run, so a halo is
           one contiguous NCCL send/recv);
* D<, D>   raw phonon slab [Nqz, Nw, dA, NB+1, 3, 3] over the same atoms
           (preprocess_D reads D at f(a, s));
* Dc<, Dc> [Nqz, Nw, oA, NB, 3, 3] and dH [oA, NB, 3, No, No] of owned atoms;
* Sigma<, Sigma> atom-major [oA, Nkz, NE, No, No].

Inputs come from the atom-keyed generator (inputs.atom_keyed_values), so a
rank fills only the atoms it owns and receives its halo from the owners.
One SSE step = [halo exchange of G] + preprocess_D (device) + K2 + K3.
"""

from __future__ import annotations

import numpy as np

from . import inputs
from . import sse as dev
from .types import SimParams, build_neighbor_map, default_grid


def chunk(total: int, parts: int, rank: int) -> tuple[int, int]:
    """Contiguous ceil-division chunk (distsim.py:117-120)."""
    size = -(-total // parts)
    return min(rank * size, total), min((rank + 1) * size, total)


class ShardProblem:
    def __init__(self, p: SimParams, rank: int = 0, world: int = 1, device: int = 0, seed: int = 0,
                 grid=None, idx=None):
        import torch

        self.torch = torch
        self.p = p
        self.rank, self.world, self.seed = rank, world, seed
        self.device = torch.device("cuda", device)
        self.grid = grid if grid is not None else default_grid(p)
        self.idx = np.ascontiguousarray(idx if idx is not None else build_neighbor_map(p.n_A, p.n_B).idx)
        self.offsets = np.array(self.grid.offsets[: p.n_w], dtype=np.int64)
        self.weights = np.array(self.grid.weights[: p.n_w], dtype=np.float64)
        self.lo, self.hi = chunk(p.n_A, world, rank)
        rows = self.idx[self.lo:self.hi]
        # G / D slab: owned atoms plus every neighbour they reference
        self.glo = int(min(self.lo, rows.min()))
        self.ghi = int(max(self.hi, rows.max() + 1))
        self.tensors_allocated = False

    # ------------------------------------------------------------------
    @property
    def n_owned(self) -> int:
        return self.hi - self.lo

    @property
    def n_slab(self) -> int:
        return self.ghi - self.glo

    def allocate(self) -> None:
        t, p = self.torch, self.p
        c128 = dict(dtype=t.complex128, device=self.device)
        self.g = [t.empty((self.n_slab, p.n_kz, p.n_E, p.n_orb, p.n_orb), **c128) for _ in range(2)]
        self.d = [t.empty((p.n_qz, p.n_w, self.n_slab, p.n_B + 1, 3, 3), **c128) for _ in range(2)]
        self.dc = [t.empty((p.n_qz, p.n_w, self.n_owned, p.n_B, 3, 3), **c128) for _ in range(2)]
        self.dh = t.empty((self.n_owned, p.n_B, 3, p.n_orb, p.n_orb), **c128)
        self.sig = [t.zeros((self.n_owned, p.n_kz, p.n_E, p.n_orb, p.n_orb), **c128) for _ in range(2)]
        self.pi_out = None
        self.tensors_allocated = True

    def fill(self, owned_g_only: bool) -> None:
        """Generate inputs on the device (atom-keyed, bit-exact with the host)."""
        p = self.p
        if not self.tensors_allocated:
            self.allocate()
        no2 = p.n_orb * p.n_orb
        per_g = p.n_kz * p.n_E * no2
        g_lo, g_hi = (self.lo, self.hi) if owned_g_only else (self.glo, self.ghi)
        for pol, tid in ((0, inputs.G_LESSER), (1, inputs.G_GREATER)):
            view = self.g[pol][g_lo - self.glo:]
            dev.fill_synthetic(view, self.seed, tid, g_lo, g_hi - g_lo, p.n_kz * p.n_E, no2, per_g, no2)
        slots = (p.n_B + 1) * 9
        for pol, tid in ((0, inputs.D_LESSER), (1, inputs.D_GREATER)):
            dev.fill_synthetic(self.d[pol], self.seed, tid, self.glo, self.n_slab, p.n_qz * p.n_w, slots,
                               slots, self.n_slab * slots)
        inner = p.n_B * 3 * no2
        dev.fill_synthetic(self.dh, self.seed, inputs.DH, self.lo, self.n_owned, 1, inner, inner, 0,
                           scale=inputs.DH_SCALE)

    def preprocess(self, stream=None) -> None:
        for pol in range(2):
            dev.preprocess_D_device(self.d[pol], self.dc[pol], self.idx, d_atom0=self.glo,
                                    out_atom0=self.lo, stream=stream)

    def sigma(self, stream=None) -> None:
        dev.sigma_device(
            self.g[0], self.g[1], self.dc[0], self.dc[1], self.dh, self.idx[self.lo:self.hi],
            self.offsets, self.weights, self.sig[0], self.sig[1], n_a=self.p.n_A, g_atom0=self.glo,
            out_atom0=self.lo, atom_major=True, stream=stream,
        )

    def sigma_scatter(self, peer, stream=None) -> None:
        """Sigma of the owned atoms written into the point owners' buffers (dist.PeerPointBuffers)."""
        dev.sigma_device_scatter(
            self.g[0], self.g[1], self.dc[0], self.dc[1], self.dh, self.idx[self.lo:self.hi],
            self.offsets, self.weights, peer.remote[0], peer.remote[1], peer.pt_lo, n_a=self.p.n_A,
            g_atom0=self.glo, out_atom0=self.lo, atom_major=True, stream=stream,
        )

    def sigma_peer(self, peer_g, peer_s, stream=None) -> None:
        """Sigma with G read from the GF point owners (peer_g) and written to them (peer_s):
        no slab, no halo, no return collective (dist.PeerPointBuffers for both)."""
        p = self.p
        dev.sigma_device_peer(
            peer_g.remote[0], peer_g.remote[1], self.dc[0], self.dc[1], self.dh, self.idx[self.lo:self.hi],
            self.offsets, self.weights, peer_s.remote[0], peer_s.remote[1], peer_s.pt_lo, n_kz=p.n_kz, n_e=p.n_E,
            n_a=p.n_A, n_o=p.n_orb, out_atom0=self.lo, device=self.device.index or 0, stream=stream,
        )

    def pull_g(self, peer_g, stream=None) -> None:
        """The G slab (owned atoms + halo) from the GF point owners' buffers (dist.PeerPointBuffers):
        one kernel per polarity reading the peers over NVLink; replaces slab assembly + halo exchange."""
        p = self.p
        for pol in range(2):
            dev.slab_from_points(peer_g.remote[pol], peer_g.pt_lo, self.g[pol], n_kz=p.n_kz, n_e=p.n_E, n_a=p.n_A,
                                 g_atom0=self.glo, atom_major=True, self_rank=peer_g.rank, stream=stream)

    def pi(self, stream=None) -> None:
        """Phonon self-energy Pi of the owned atoms (sse.py:409-428), [Nqz, Nw, oA, NB+1, 3, 3]."""
        t, p = self.torch, self.p
        if self.pi_out is None:
            shape = (p.n_qz, p.n_w, self.n_owned, p.n_B + 1, 3, 3)
            self.pi_out = [t.zeros(shape, dtype=t.complex128, device=self.device) for _ in range(2)]
        dev.pi_device(
            self.g[0], self.g[1], self.dh, self.idx[self.lo:self.hi], self.offsets, self.grid.energy_weight,
            self.pi_out[0], self.pi_out[1], n_a=p.n_A, n_qz=p.n_qz, g_atom0=self.glo, out_atom0=self.lo,
            atom_major=True, stream=stream,
        )

    def phase(self, stream=None) -> None:
        """The SSE phase of a Born iteration in one device call (sse_phase_device, sse.py:532-534):
        preprocess_D + Sigma + Pi of the owned atoms from the resident G / raw D slabs."""
        t, p = self.torch, self.p
        if self.pi_out is None:
            shape = (p.n_qz, p.n_w, self.n_owned, p.n_B + 1, 3, 3)
            self.pi_out = [t.zeros(shape, dtype=t.complex128, device=self.device) for _ in range(2)]
        dev.sse_phase_device(self.g[0], self.g[1], self.d[0], self.d[1], self.dh, self.idx, self.grid, self.sig[0],
                             self.sig[1], self.pi_out[0], self.pi_out[1], g_atom0=self.glo, out_atom0=self.lo,
                             atom_major=True, stream=stream)

    def pi_peer(self, peer_g, stream=None) -> None:
        """Pi of the owned atoms with G read from the GF point owners (dist.PeerPointBuffers)."""
        t, p = self.torch, self.p
        if self.pi_out is None:
            shape = (p.n_qz, p.n_w, self.n_owned, p.n_B + 1, 3, 3)
            self.pi_out = [t.zeros(shape, dtype=t.complex128, device=self.device) for _ in range(2)]
        dev.pi_device_peer(
            peer_g.remote[0], peer_g.remote[1], self.dh, self.idx[self.lo:self.hi], self.offsets,
            self.grid.energy_weight, self.pi_out[0], self.pi_out[1], peer_g.pt_lo, n_kz=p.n_kz, n_qz=p.n_qz,
            n_e=p.n_E, n_a=p.n_A, n_o=p.n_orb, out_atom0=self.lo, stream=stream,
        )

    def step(self, exchange=None, stream=None, with_pi: bool = False) -> None:
        """One SSE evaluation: halo exchange (if any) + preprocess_D + Sigma (+ Pi)."""
        if exchange is not None:
            exchange(self)
        self.preprocess(stream)
        self.sigma(stream)
        if with_pi:
            self.pi(stream)

    def sigma_block(self, pol: int, k: int, e: int, a: int) -> np.ndarray:
        """Sigma[k, e, a] of an owned atom (copied to the host)."""
        return self.sig[pol][a - self.lo, k, e].cpu().numpy()

    def flops(self) -> int:
        p = self.p
        return dev.alg_flops(p.n_kz, p.n_qz, p.n_E, self.n_owned, p.n_B, p.n_orb, self.offsets)

    def free(self) -> None:
        for name in ("g", "d", "dc", "dh", "sig", "pi_out"):
            if hasattr(self, name):
                delattr(self, name)
        self.tensors_allocated = False
