"""Small K3m / K5-K7 / staging invocations for compute-sanitizer (memcheck): one process, tiny shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import sse_oracle as orc  # noqa: E402
from paper_1912_08810_b200 import inputs  # noqa: E402
from paper_1912_08810_b200.sse import sse_phase, sse_sigma  # noqa: E402
from paper_1912_08810_b200.types import (CombinedD, GreensTensor, SimParams, SseVariant,  # noqa: E402
                                         build_neighbor_map, default_grid)

for n_kz, n_qz, n_e, n_w, n_o, n_a in ((3, 3, 26, 14, 12, 6), (3, 2, 30, 8, 10, 5), (4, 4, 20, 7, 4, 5)):
    p = SimParams(n_kz=n_kz, n_qz=n_qz, n_E=n_e, n_w=n_w, n_A=n_a, n_B=4, n_orb=n_o)
    g_l, g_g, d_l, d_g, dh = inputs.stream_instance(3, p, dh_scale=0.05)
    nmap = build_neighbor_map(p.n_A, p.n_B)
    grid = default_grid(p)
    dc = CombinedD(*orc.preprocess_D(d_l, d_g, nmap.idx))
    out = sse_sigma(SseVariant.BATCHED_FUSED, GreensTensor(g_l, g_g), dc, dh, nmap, grid)
    ref = orc.sigma_batched_fused(g_l, g_g, dc.lesser, dc.greater, dh, nmap.idx, np.array(grid.offsets),
                                  np.array(grid.weights))
    dev = orc.parity_dev(out.lesser, out.greater, *ref)
    s, pi = sse_phase(GreensTensor(g_l, g_g), GreensTensor(d_l, d_g), dh, nmap, grid, n_qz)
    print(f"No={n_o} Nkz={n_kz}: sigma dev {dev:.2e}, phase ok", flush=True)
    assert dev <= 1e-10
print("SANITIZE_OK")
