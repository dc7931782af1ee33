"""Full-size parity helpers: device-resident problem + pointwise host oracle.

The GPU computes the whole BASELINE config from device-generated atom-keyed
inputs; the host regenerates only the atoms a sampled output block depends
on (its neighbours' G, the raw D rows of the atom and its neighbours, dH)
and evaluates that block with oracle.sigma_point (the reference's term
order, sse.py:145-161).
"""

from __future__ import annotations

import numpy as np

from oracle import sse_oracle as orc
from paper_1912_08810_b200 import inputs
from paper_1912_08810_b200.problem import ShardProblem


class DeviceProblem(ShardProblem):
    """Rank `rank` of a `world`-way atom sharding, on device `rank`, halo filled locally."""

    def __init__(self, name, seed=0, world=1, rank=0, device=None):
        super().__init__(inputs.CONFIGS[name], rank=rank, world=world, device=rank if device is None else device,
                         seed=seed)

    def launch(self):
        with self.torch.cuda.device(self.device):
            self.fill(owned_g_only=False)
            self.step()

    def run(self):
        self.launch()
        self.torch.cuda.synchronize(self.device)


def run_sharded(name, world, seed=0):
    """All shards of a config, one per GPU, launched concurrently."""
    shards = [DeviceProblem(name, seed, world, r) for r in range(world)]
    for sh in shards:
        sh.launch()
    for sh in shards:
        sh.torch.cuda.synchronize(sh.device)
    return shards


def host_point(prob: ShardProblem, pol: int, k: int, e: int, a: int) -> np.ndarray:
    p, seed, idx = prob.p, prob.seed, prob.idx
    g_tid = inputs.G_LESSER if pol == 0 else inputs.G_GREATER
    d_tid = inputs.D_LESSER if pol == 0 else inputs.D_GREATER
    nbrs = sorted(set(int(b) for b in idx[a]))
    gvals = {
        b: inputs.atom_keyed_values(seed, g_tid, [b], p.n_kz * p.n_E, p.n_orb**2)[0].reshape(
            p.n_kz, p.n_E, p.n_orb, p.n_orb)
        for b in nbrs
    }
    atoms = sorted(set(nbrs) | {a})
    draw = inputs.atom_keyed_values(seed, d_tid, atoms, p.n_qz * p.n_w, (p.n_B + 1) * 9)
    d = {x: draw[i].reshape(p.n_qz, p.n_w, p.n_B + 1, 3, 3) for i, x in enumerate(atoms)}
    # Dc[:, :, a] from the reference formula (sse.py:105-113), pinned in tests/test_oracle.py
    dc_a = orc.preprocess_D_atom(lambda x: d[x], idx, a)
    dh_a = inputs.atom_keyed_dh(seed, p, [a])[0]
    return orc.sigma_point(lambda kk, ee, b: gvals[b][kk, ee], dc_a, dh_a, idx[a], prob.offsets,
                           prob.weights, p.n_kz, p.n_qz, k, e)
