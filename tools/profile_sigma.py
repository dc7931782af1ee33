"""Small device-resident SSE step for ncu: a 64-atom shard of a BASELINE config.

    python tools/profile_sigma.py [--config paper] [--atoms 64] [--steps 2]
Runs --steps full steps (preprocess_D, K2, K3 for both polarities) of one
atom shard whose per-atom shapes are the config's; prints the K3 time.
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
ap.add_argument("--lib", default=None, help="libsse.so to load instead of the in-tree build (A/B runs)")
args = ap.parse_args()
if args.lib:
    from paper_1912_08810_b200 import _lib
    _lib.LIB_PATH = os.path.abspath(args.lib)
p, grid, nmap = config(args.config)
world = max(1, p.n_A // args.atoms)
prob = ShardProblem(p, rank=world // 2, world=world, seed=0, grid=grid, idx=nmap.idx)
prob.allocate()
prob.fill(owned_g_only=False)
prob.step()
torch.cuda.synchronize()
with Profile(device=0) as prof:
    for _ in range(args.steps):
        prob.step()
    torch.cuda.synchronize()
s = prof.result["sigma"]
print(f"atoms {prob.n_owned} K3 {s['ms'] / s['launches']:.3f} ms/launch "
      f"{s['flops'] / s['ms'] / 1e9:.2f} TFLOP/s; K2 {prof.result['operator']['ms'] / max(1, prof.result['operator']['launches']):.3f} ms")
