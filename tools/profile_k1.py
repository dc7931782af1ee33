"""HBM-bound kernels at paper scale: K1 layout transform (grid <-> atom major G, one polarity,
23.7 GB each way) and preprocess_D (raw D -> Dc), achieved GB/s vs the measured HBM copy peak.

    python tools/profile_k1.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1912_08810_b200 import inputs  # noqa: E402
from paper_1912_08810_b200 import sse as dev  # noqa: E402
from paper_1912_08810_b200.inputs import config  # noqa: E402

p, grid, nmap = config("paper")
cuda = torch.device("cuda", 0)
no2 = p.n_orb * p.n_orb
src = torch.empty((p.n_kz, p.n_E, p.n_A, p.n_orb, p.n_orb), dtype=torch.complex128, device=cuda)
dev.fill_synthetic(src, 0, inputs.G_LESSER, 0, p.n_A, p.n_kz * p.n_E, no2, no2, p.n_A * no2)
dst = torch.empty((p.n_A, p.n_kz, p.n_E, p.n_orb, p.n_orb), dtype=torch.complex128, device=cuda)
back = torch.empty_like(src)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = {}
nbytes = src.numel() * 16
for name, fn in (("to_atom_major", lambda: dev.layout_transform(src, dst, True)),
                 ("to_grid_major", lambda: dev.layout_transform(dst, back, False))):
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    res[name] = {"ms": ms, "GB/s": 2 * nbytes / ms / 1e6}
assert torch.equal(src, back)  # lossless round trip (test_sse.py:231-236)
del dst, back
slots = (p.n_B + 1) * 9
d = torch.empty((p.n_qz, p.n_w, p.n_A, p.n_B + 1, 3, 3), dtype=torch.complex128, device=cuda)
dev.fill_synthetic(d, 0, inputs.D_LESSER, 0, p.n_A, p.n_qz * p.n_w, slots, slots, p.n_A * slots)
dc = torch.empty((p.n_qz, p.n_w, p.n_A, p.n_B, 3, 3), dtype=torch.complex128, device=cuda)
dev.preprocess_D_device(d, dc, nmap.idx)
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    dev.preprocess_D_device(d, dc, nmap.idx)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
res["preprocess_D"] = {"ms": ms, "GB/s": (d.numel() + dc.numel()) * 16 / ms / 1e6,
                       "note": "algorithmic bytes: read D once + write Dc (the 4-term gather re-reads D rows from L2)"}
peaks = {}
try:
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as fh:
        peaks = json.load(fh)
except Exception:
    pass
hbm = float(peaks.get("hbm_gbs", 6542.4))
res["hbm_peak_gbs"] = hbm
res["hbm_peak_source"] = "MEASURED_PEAKS.json" if peaks else "B200_PROFILING.md fallback"
for k in ("to_atom_major", "to_grid_major", "preprocess_D"):
    res[k]["frac"] = res[k]["GB/s"] / hbm
print(json.dumps(res))
