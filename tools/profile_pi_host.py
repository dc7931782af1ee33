"""Pi through the host drop-in (sse_pi_c128) from pinned host memory at paper scale: the G upload
streams under K5/K6 chunk by chunk.

    python tools/profile_pi_host.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1912_08810_b200 import inputs  # noqa: E402
from paper_1912_08810_b200 import sse as dev  # noqa: E402
from paper_1912_08810_b200.inputs import config  # noqa: E402
from paper_1912_08810_b200.types import GreensTensor  # noqa: E402

p, grid, nmap = config("paper")
cuda = torch.device("cuda", 0)
no2 = p.n_orb * p.n_orb
shape = (p.n_kz, p.n_E, p.n_A, p.n_orb, p.n_orb)
g = []
for tid in (inputs.G_LESSER, inputs.G_GREATER):
    t = torch.empty(shape, dtype=torch.complex128, device=cuda)
    dev.fill_synthetic(t, 0, tid, 0, p.n_A, p.n_kz * p.n_E, no2, no2, p.n_A * no2)
    h = torch.empty(shape, dtype=torch.complex128, pin_memory=True)
    h.copy_(t)
    g.append(h)
    del t
dh = torch.empty((p.n_A, p.n_B, 3, p.n_orb, p.n_orb), dtype=torch.complex128, device=cuda)
inner = p.n_B * 3 * no2
dev.fill_synthetic(dh, 0, inputs.DH, 0, p.n_A, 1, inner, inner, 0, scale=inputs.DH_SCALE)
dh_h = dh.cpu().numpy()
torch.cuda.synchronize()
torch.cuda.empty_cache()
gt = GreensTensor(g[0].numpy(), g[1].numpy())
dev.sse_pi(gt, dh_h, nmap, grid, p.n_qz, n_gpus=1)
tim = {}
dev.sse_pi(gt, dh_h, nmap, grid, p.n_qz, n_gpus=1, timing=tim)
print({k: tim[k] for k in ("total_ms", "h2d_bytes", "d2h_bytes", "kernel_launches")})
