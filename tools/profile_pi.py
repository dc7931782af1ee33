"""Pi kernels on a shard of a BASELINE config (K5 build, K6 DMMA chains, K7 assembly).

    python tools/profile_pi.py [--config paper] [--atoms 64] [--steps 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1912_08810_b200.inputs import config  # noqa: E402
from paper_1912_08810_b200.problem import ShardProblem  # noqa: E402
from paper_1912_08810_b200.sse import Profile  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="paper")
ap.add_argument("--atoms", type=int, default=64)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--nw", type=int, default=0, help="override the number of phonon frequencies")
ap.add_argument("--lib", default=None, help="libsse.so to load instead of the in-tree build (A/B runs)")
args = ap.parse_args()
if args.lib:
    from paper_1912_08810_b200 import _lib
    _lib.LIB_PATH = os.path.abspath(args.lib)
p, grid, nmap = config(args.config)
if args.nw:
    import dataclasses

    from paper_1912_08810_b200.types import default_grid

    p = dataclasses.replace(p, n_w=args.nw)
    grid = default_grid(p)
world = max(1, p.n_A // args.atoms)
prob = ShardProblem(p, rank=world // 2, world=world, seed=0, grid=grid, idx=nmap.idx)
prob.allocate()
prob.fill(owned_g_only=False)
prob.pi()
torch.cuda.synchronize()
with Profile(device=0) as prof:
    for _ in range(args.steps):
        prob.pi()
    torch.cuda.synchronize()
r = prof.result
k6 = r["pi"]
print(f"atoms {prob.n_owned}: K6 {k6['ms'] / k6['launches']:.2f} ms/launch {k6['flops'] / k6['ms'] / 1e9:.2f} TFLOP/s; "
      f"K5 {r['pi_build']['ms'] / max(1, r['pi_build']['launches']):.2f} ms; K7 {r['pi_assemble']['ms'] / max(1, r['pi_assemble']['launches']):.3f} ms")
