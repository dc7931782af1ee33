"""SSE Sigma^{<>} benchmark on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config paper]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...

One step = one Sigma^{<>} evaluation of a Born iteration (both polarities;
sse.py:533) on the paper-scale FinFET workload (BASELINE.json configs[2]:
NA=4864, NB=4, No=12, NE=706, Nw=70, Nkz=Nqz=3), strong-scaled over N GPUs
by atom sharding (one process per GPU, NCCL halo exchange of G inside the
step).  `value` = device time per step (CUDA events, inputs resident in HBM,
max over ranks); `e2e` = the same step through the host C-ABI call
(sse_sigma_c128_slab) from pinned host buffers with H2D/D2H inside.
`--impl reference` times the reference's CPU algorithm (the oracle's
BATCHED_FUSED restatement, the fastest reference arrangement) on a bounded
sample of (atom, neighbour) pairs and extrapolates per pair.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "SSE time per Born iteration (s) and achieved FP64 TFLOP/s at 1/2/4/8 B200 vs CPU ref"
FP64_PEAK_TFLOPS = 36.85  # measured DMMA.8x8x4 sustained, profiles/r01_fp64_peak.json
FP64_PEAK_SOURCE = "measured DMMA m8n8k4 sustained on this pool's B200 (profiles/r01_fp64_peak.json); MEASURED_PEAKS.json has no FP64 entry"


def k3_kernel_name() -> str:
    """The K3 variant libsse launches for the bench workload (SSE_SIGMA_KERNEL, default 3)."""
    return {
        "0": "sigma_dmma_kernel<12> (K3 simple)",
        "1": "sigma_dmma_pipe_kernel<12> (K3 register-pipelined)",
    }.get(os.environ.get("SSE_SIGMA_KERNEL", "3"),
          "sigma_dmma_slide_kernel<12,12,3> (K3 TMA sliding window, 12 warps x 3 row tiles)")


def k6_kernel_name() -> str:
    """The K6 variant libsse launches for the bench workload (SSE_PI_KERNEL, default 3)."""
    return {
        "0": "pi_dmma_direct_kernel (K6 direct)",
        "1": "pi_dmma_kernel (K6 v1, 2 momenta per CTA)",
        "2": "pi_dmma2_kernel (K6 v2, half stages)",
        "3": "pi_dmma3_kernel (K6 v3: one m-tile x 9 n-tiles per warp, TMA ring of V, 3 CTAs/SM)",
    }.get(os.environ.get("SSE_PI_KERNEL", "4"),
          "pi_dmma4_kernel<12,4,4,3,4,true> (K6 v4: 2 lag tiles x 9 n-tiles per warp, 4-warp CTAs for lag "
          "tiles 0-7 + tail CTAs for the 9th tile of every q in the same launch, TMA ring of V)")


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload_name(p) -> str:
    return (f"NA={p.n_A} NB={p.n_B} No={p.n_orb} NE={p.n_E} Nw={p.n_w} Nkz={p.n_kz} Nqz={p.n_qz} "
            "(Sigma lesser+greater)")


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus: str):
        self.gpus = gpus
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", self.gpus],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        return False

    def summary(self) -> dict:
        sm, mx, reasons, power = [], [], set(), []
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": float(max(power))}


# ---------------------------------------------------------------------------
# CPU reference (oracle BATCHED_FUSED port) on a bounded pair sample
# ---------------------------------------------------------------------------
def cpu_sample(p, grid, idx, n_pairs: int, seed: int = 0, first_atom: int | None = None) -> dict:
    """Time the reference's BATCHED_FUSED algorithm (oracle port) on n_pairs (atom, slot) pairs.

    The per-pair work of BATCHED_FUSED is independent of NA (sse.py:279-301),
    so seconds per Born iteration = per-pair time x NA x NB.
    """
    from oracle import sse_oracle as orc
    from paper_1912_08810_b200 import inputs

    a0 = p.n_A // 2 if first_atom is None else first_atom
    pairs_g = [(a0 + i // p.n_B, i % p.n_B) for i in range(n_pairs)]
    out_atoms = sorted({a for a, _ in pairs_g})
    others = sorted({int(idx[a, s]) for a in out_atoms for s in range(p.n_B)} - set(out_atoms))
    order = out_atoms + others  # sub-problem atoms: sampled outputs first, then their neighbours
    pos = {a: i for i, a in enumerate(order)}
    sub_idx = np.zeros((len(order), p.n_B), dtype=np.int64)
    for a in out_atoms:
        sub_idx[pos[a]] = [pos[int(idx[a, s])] for s in range(p.n_B)]
    g_l = inputs.atom_keyed_electron(seed, inputs.G_LESSER, p, order)
    g_g = inputs.atom_keyed_electron(seed, inputs.G_GREATER, p, order)
    rng = np.random.default_rng(seed)
    shape = (p.n_qz, p.n_w, len(order), p.n_B, 3, 3)
    dc_l = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    dc_g = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    dh = inputs.atom_keyed_dh(seed, p, order)
    off, wt = np.array(grid.offsets), np.array(grid.weights)
    pairs = [(pos[a], s) for a, s in pairs_g]
    t0 = time.perf_counter()
    orc.sigma_batched_fused(g_l, g_g, dc_l, dc_g, dh, sub_idx, off, wt, pairs=pairs)
    dt = time.perf_counter() - t0
    per_pair = dt / n_pairs
    return {"seconds": dt, "per_pair_s": per_pair, "pairs": n_pairs,
            "extrapolated_s": per_pair * p.n_A * p.n_B}


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info

        return max((i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"), default=1)
    except Exception:
        return 1


def run_reference(args, p, grid, idx) -> None:
    rank, world, _ = env_rank()
    if rank != 0:
        return
    n_pairs = args.ref_pairs
    for _ in range(args.warmup):
        cpu_sample(p, grid, idx, n_pairs)
    samples = [cpu_sample(p, grid, idx, n_pairs) for _ in range(args.steps)]
    per_pair = float(np.mean([s["per_pair_s"] for s in samples]))
    value = per_pair * p.n_A * p.n_B
    from paper_1912_08810_b200.sse import alg_flops

    flops = alg_flops(p.n_kz, p.n_qz, p.n_E, p.n_A, p.n_B, p.n_orb, grid.offsets)
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64)",
        "data": "synthetic (atom-keyed generator)",
        "config": {"workload": workload_name(p), "name": args.config, "parallelism": "cpu"},
        "tflops": flops / value / 1e12,
        "cpu_baseline": {
            "value": value, "unit": "s", "cores": blas_threads(), "kind": "port",
            "sample": (f"{n_pairs} (atom, neighbour) pairs per step of the reference BATCHED_FUSED algorithm "
                       f"(oracle/sse_oracle.py:sigma_batched_fused, sse.py:265-302) at the real per-pair "
                       f"shapes, x NA*NB={p.n_A * p.n_B}; numpy/OpenBLAS with {blas_threads()} threads "
                       f"of {os.cpu_count()} host cores (the path is ~1 busy core)"),
        },
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def e2e_phase(args, p, grid, idx, rank, world, local_rank) -> dict:
    """Per-rank host-memory drop-in call (pinned buffers, H2D/D2H inside)."""
    import torch

    from paper_1912_08810_b200 import inputs
    from paper_1912_08810_b200 import sse as dev
    from paper_1912_08810_b200.problem import chunk

    lo, hi = chunk(p.n_A, world, rank)
    rows = idx[lo:hi]
    glo, ghi = int(min(lo, rows.min())), int(max(hi, rows.max() + 1))
    gA, oA = ghi - glo, hi - lo
    no2 = p.n_orb * p.n_orb
    cuda = torch.device("cuda", local_rank)
    pin = dict(dtype=torch.complex128, pin_memory=True)
    g_host = [torch.empty((p.n_kz, p.n_E, gA, p.n_orb, p.n_orb), **pin) for _ in range(2)]
    s_host = [torch.empty((p.n_kz, p.n_E, oA, p.n_orb, p.n_orb), **pin) for _ in range(2)]
    dc_host = [torch.empty((p.n_qz, p.n_w, oA, p.n_B, 3, 3), **pin) for _ in range(2)]
    dh_host = torch.empty((oA, p.n_B, 3, p.n_orb, p.n_orb), **pin)
    # inputs generated on the device (same atom-keyed values as the resident run), copied once
    for pol, tid in ((0, inputs.G_LESSER), (1, inputs.G_GREATER)):
        tmp = torch.empty(g_host[pol].shape, dtype=torch.complex128, device=cuda)
        dev.fill_synthetic(tmp, 0, tid, glo, gA, p.n_kz * p.n_E, no2, no2, gA * no2)
        g_host[pol].copy_(tmp)
        del tmp
    slots = (p.n_B + 1) * 9
    for pol, tid in ((0, inputs.D_LESSER), (1, inputs.D_GREATER)):
        d = torch.empty((p.n_qz, p.n_w, gA, p.n_B + 1, 3, 3), dtype=torch.complex128, device=cuda)
        dev.fill_synthetic(d, 0, tid, glo, gA, p.n_qz * p.n_w, slots, slots, gA * slots)
        dc = torch.empty(dc_host[pol].shape, dtype=torch.complex128, device=cuda)
        dev.preprocess_D_device(d, dc, idx, d_atom0=glo, out_atom0=lo)
        dc_host[pol].copy_(dc)
        del d, dc
    dht = torch.empty(dh_host.shape, dtype=torch.complex128, device=cuda)
    inner = p.n_B * 3 * no2
    dev.fill_synthetic(dht, 0, inputs.DH, lo, oA, 1, inner, inner, 0, scale=inputs.DH_SCALE)
    dh_host.copy_(dht)
    del dht
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    offs, wts = np.array(grid.offsets), np.array(grid.weights)

    def call():
        return dev.sigma_host_slab(g_host[0], g_host[1], dc_host[0], dc_host[1], dh_host, rows, offs, wts,
                                   s_host[0], s_host[1], n_a=p.n_A, g_atom0=glo, out_atom0=lo,
                                   device=local_rank)

    for _ in range(args.e2e_warmup):
        call()
    times, tim = [], None
    for _ in range(args.e2e_steps):
        barrier(world)
        tim = call()
        times.append(tim["total_ms"])
    t = allreduce_max(float(np.mean(times)), world)
    h2d = allreduce_sum(float(tim["h2d_bytes"]), world)
    d2h = allreduce_sum(float(tim["d2h_bytes"]), world)
    out = {"value": t / 1e3, "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
           "steps": args.e2e_steps, "warmup": args.e2e_warmup,
           "path": "sse_sigma_c128_slab (C ABI) from pinned host memory, 3-stream H2D/compute/D2H pipeline"}
    del g_host, s_host, dc_host, dh_host
    return out


def phase_e2e(args, p, grid, idx, local_rank) -> dict:
    """the whole SSE phase of a Born iteration (preprocess_D + Sigma + Pi) through
    sse_phase (C ABI sse_phase_c128) from pinned host memory, N = 1."""
    import torch

    from paper_1912_08810_b200 import inputs
    from paper_1912_08810_b200 import sse as dev
    from paper_1912_08810_b200.sse import Profile
    from paper_1912_08810_b200.types import GreensTensor, NeighborMap

    no2 = p.n_orb * p.n_orb
    cuda = torch.device("cuda", local_rank)
    pin = dict(dtype=torch.complex128, pin_memory=True)
    e_shape = (p.n_kz, p.n_E, p.n_A, p.n_orb, p.n_orb)
    ph_shape = (p.n_qz, p.n_w, p.n_A, p.n_B + 1, 3, 3)
    g_host = [torch.empty(e_shape, **pin) for _ in range(2)]
    d_host = [torch.empty(ph_shape, **pin) for _ in range(2)]
    out = [torch.empty(e_shape, **pin) for _ in range(2)] + [torch.empty(ph_shape, **pin) for _ in range(2)]
    dh_host = torch.empty((p.n_A, p.n_B, 3, p.n_orb, p.n_orb), **pin)
    for pol, tid in ((0, inputs.G_LESSER), (1, inputs.G_GREATER)):
        tmp = torch.empty(e_shape, dtype=torch.complex128, device=cuda)
        dev.fill_synthetic(tmp, 0, tid, 0, p.n_A, p.n_kz * p.n_E, no2, no2, p.n_A * no2)
        g_host[pol].copy_(tmp)
        del tmp
    slots = (p.n_B + 1) * 9
    for pol, tid in ((0, inputs.D_LESSER), (1, inputs.D_GREATER)):
        d = torch.empty(ph_shape, dtype=torch.complex128, device=cuda)
        dev.fill_synthetic(d, 0, tid, 0, p.n_A, p.n_qz * p.n_w, slots, slots, p.n_A * slots)
        d_host[pol].copy_(d)
        del d
    dht = torch.empty(dh_host.shape, dtype=torch.complex128, device=cuda)
    inner = p.n_B * 3 * no2
    dev.fill_synthetic(dht, 0, inputs.DH, 0, p.n_A, 1, inner, inner, 0, scale=inputs.DH_SCALE)
    dh_host.copy_(dht)
    del dht
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    g = GreensTensor(g_host[0].numpy(), g_host[1].numpy())
    gph = GreensTensor(d_host[0].numpy(), d_host[1].numpy())
    outs = tuple(o.numpy() for o in out)
    nmap = NeighborMap(idx)

    def call(tim):
        dev.sse_phase(g, gph, dh_host.numpy(), nmap, grid, p.n_qz, device=local_rank, out=outs, timing=tim)

    call({})
    times = []
    with Profile(device=local_rank) as prof:
        for _ in range(args.phase_steps):
            tim = {}
            call(tim)
            times.append(tim["total_ms"])
    res = {"value": float(np.mean(times)) / 1e3, "unit": "s", "steps": args.phase_steps, "warmup": 1,
           "h2d_bytes_per_step": int(tim["h2d_bytes"]), "d2h_bytes_per_step": int(tim["d2h_bytes"]),
           "kernel_ms_per_step": {k: v["ms"] / args.phase_steps for k, v in prof.result.items() if v["launches"]},
           "path": "sse_phase (C ABI sse_phase_c128): G<> + raw D<> + dH in once, device preprocess_D, "
                   "pipelined Sigma (K2+K3), Pi (K5-K7) on the resident G, Sigma + Pi out"}
    del g, gph, outs, g_host, d_host, out, dh_host
    return res


def load_traffic():
    path = os.path.join(REPO, "profiles", "sigma_kernel_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except Exception:
        return None


def pi_phase(args, p, grid, idx, prob, world, local_rank, step_ms, start, end, stream):
    """Pi (the other half of the SSE phase, sse.py:534) on the same resident G."""
    import torch

    from paper_1912_08810_b200.sse import Profile

    if args.pi_steps <= 0:
        return None
    prob.pi()
    torch.cuda.synchronize()
    barrier(world)
    with Profile(device=local_rank) as pprof:
        start.record(stream)
        for _ in range(args.pi_steps):
            prob.pi()
        end.record(stream)
        torch.cuda.synchronize()
    pi_ms = allreduce_max(start.elapsed_time(end) / args.pi_steps, world)
    k6 = pprof.result["pi"]
    k6_tflops = allreduce_sum(k6["flops"] / (k6["ms"] * 1e-3) / 1e12 if k6["ms"] > 0 else 0.0, world) / world
    terms = sum(max(0, p.n_E - int(o)) for o in grid.offsets)
    pi_flops = 16 * p.n_A * p.n_B * p.n_qz * p.n_kz * 9 * p.n_orb**2 * terms
    pi_info = {
        "s_per_eval": pi_ms / 1e3, "steps": args.pi_steps, "tflops": pi_flops / (pi_ms * 1e-3) / 1e12,
        "flops_alg": pi_flops,
        "roofline": {"bound": "tensor", "kernel": k6_kernel_name(),
                     "achieved": k6_tflops, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": k6_tflops / FP64_PEAK_TFLOPS},
        "kernels": {k: pprof.result[k] for k in ("pi_build", "pi", "pi_assemble")},
        "note": "phonon self-energy Pi (sse_pi) per Born iteration, V form: chain = w_E sum <G1(E+off)^T, "
                "dH_j G2 dH_i>; not part of `value` (north_star's path is Sigma)",
    }
    return pi_info


def gf_layout_phase(args, p, grid, idx, prob, world, local_rank, step_ms, start, end, stream):
    """the step as it follows a distributed GF phase: G from the (k, E)-point layout and raw D
    from the (q, w) points by NCCL all-to-all into the atom slabs (halos included), Sigma back to the point
    owners by a second all-to-all."""
    import torch

    from paper_1912_08810_b200 import dist as sdist

    if args.gf_layout_steps <= 0 or world <= 1:
        return None
    # the GF phase's layout of the same G: rank r holds every atom of its (k, E) points;
    # built from the owned atoms with the return collective itself
    g_pts = [sdist.atom_slab_to_points(prob.g[pol][prob.lo - prob.glo:prob.hi - prob.glo], idx, p.n_kz, p.n_E)
             for pol in range(2)]
    # raw D from the phonon GF phase's (q, w) points
    d_own = slice(prob.lo - prob.glo, prob.hi - prob.glo)
    d_pts = [sdist.columns_to_points(prob.d[pol][:, :, d_own].reshape(p.n_qz * p.n_w, prob.n_owned, -1),
                                     sdist.owned_ranges(p.n_A, world), p.n_qz * p.n_w, p.n_A, False)
             .view(-1, p.n_A, p.n_B + 1, 3, 3) for pol in range(2)]

    def digest(ts):  # bit-pattern checksum (int64 wrap-around sum): equal inputs <=> equal digests
        return [int(torch.view_as_real(t).view(torch.int64).sum()) for t in ts]

    want = digest(prob.g) + digest(prob.d)

    def gf_step():
        for pol in range(2):
            prob.g[pol].copy_(sdist.points_to_atom_slab(g_pts[pol], idx, p.n_kz, p.n_E))
            prob.d[pol].copy_(sdist.phonon_points_to_slab(d_pts[pol], idx, p.n_qz, p.n_w))
        prob.preprocess()
        prob.sigma()
        return [sdist.atom_slab_to_points(prob.sig[pol], idx, p.n_kz, p.n_E) for pol in range(2)]

    gf_step()
    torch.cuda.synchronize()
    same = float(digest(prob.g) + digest(prob.d) == want)
    same = -allreduce_max(-same, world)  # min over ranks
    barrier(world)
    start.record(stream)
    for _ in range(args.gf_layout_steps):
        gf_step()
    end.record(stream)
    torch.cuda.synchronize()
    gf_ms = allreduce_max(start.elapsed_time(end) / args.gf_layout_steps, world)
    blk = p.n_orb * p.n_orb * 16
    pts_r = p.n_kz * p.n_E / world
    gf_info = {"s_per_step": gf_ms / 1e3, "steps": args.gf_layout_steps,
               "vs_halo_step": gf_ms / step_ms,
               "slab_digest_equal_to_halo_exchange": bool(same == 1.0),
               "a2a_bytes_per_rank_approx": int(2 * pts_r * (prob.n_slab + p.n_A) * blk),
               "note": "G from the GF (k,E)-point layout and raw D from the phonon (q,w)-point layout -> "
                       "atom slabs (NCCL all_to_all_single, halos included) + preprocess_D + K2 + K3 + Sigma "
                       "back to points (all_to_all_single)"}
    del g_pts, d_pts
    torch.cuda.empty_cache()
    return gf_info


def gf_fused_phase(args, p, grid, idx, prob, world, local_rank, step_ms, start, end, stream):
    """SURVEY 8f-3 fused: G read from the GF point owners and Sigma written back to them inside the Sigma
    kernel (NVLink peer memory via CUDA IPC): no slab assembly, halo or return collective; one device-side
    all-reduce per step orders the peers' stores."""
    import torch
    import torch.distributed as dist

    from paper_1912_08810_b200 import dist as sdist

    if args.gf_fused_steps <= 0 or world <= 1:
        return None

    own = slice(prob.lo - prob.glo, prob.hi - prob.glo)
    peer_g = sdist.PeerPointBuffers(p.n_kz, p.n_E, p.n_A, p.n_orb, device=local_rank)
    for pol in range(2):
        peer_g.tensors[pol].copy_(sdist.atom_slab_to_points(prob.g[pol][own].contiguous(), idx, p.n_kz, p.n_E))
    peer_s = sdist.PeerPointBuffers(p.n_kz, p.n_E, p.n_A, p.n_orb, device=local_rank)
    token = torch.zeros(1, device=prob.device)
    # raw D still comes from the phonon (q, w) points through the (small) NCCL all-to-all
    d_pts = [sdist.columns_to_points(prob.d[pol][:, :, own].reshape(p.n_qz * p.n_w, prob.n_owned, -1),
                                     sdist.owned_ranges(p.n_A, world), p.n_qz * p.n_w, p.n_A, False)
             .view(-1, p.n_A, p.n_B + 1, 3, 3) for pol in range(2)]

    def fused_step():
        for pol in range(2):
            prob.d[pol].copy_(sdist.phonon_points_to_slab(d_pts[pol], idx, p.n_qz, p.n_w))
        prob.preprocess()
        prob.sigma_peer(peer_g, peer_s)
        dist.all_reduce(token)  # every rank's peer stores done before anyone reads its points

    fused_step()
    ref_pts = [sdist.atom_slab_to_points(prob.sig[pol], idx, p.n_kz, p.n_E) for pol in range(2)]
    torch.cuda.synchronize()
    same = float(all(torch.equal(peer_s.tensors[pol], ref_pts[pol]) for pol in range(2)))
    same = -allreduce_max(-same, world)
    del ref_pts
    barrier(world)
    start.record(stream)
    for _ in range(args.gf_fused_steps):
        fused_step()
    end.record(stream)
    torch.cuda.synchronize()
    fused_ms = allreduce_max(start.elapsed_time(end) / args.gf_fused_steps, world)
    fused_info = {"s_per_step": fused_ms / 1e3, "steps": args.gf_fused_steps, "vs_halo_step": fused_ms / step_ms,
                  "sigma_points_bitwise_equal_to_all_to_all": bool(same == 1.0),
                  "note": "G read from the GF (k,E)-point owners by TMA over NVLink and Sigma stored to them "
                          "from the K3 epilogue (CUDA IPC peer memory); raw D from the (q,w) points by NCCL "
                          "all-to-all; preprocess_D + K2 + K3 + one device-side all-reduce per step"}
    # pull variant: the G slab (owned + halo) pulled from the point owners by one kernel per polarity
    # (NVLink loads), then the slab kernels; Sigma still stored to the owners from the K3 epilogue
    def g_digest():  # bit-pattern digest (no second copy of the slab in HBM)
        return [int(torch.view_as_real(t).view(torch.int64).sum()) for t in prob.g]

    g_keep = g_digest()

    def pull_step():
        for pol in range(2):
            prob.d[pol].copy_(sdist.phonon_points_to_slab(d_pts[pol], idx, p.n_qz, p.n_w))
        prob.pull_g(peer_g)
        prob.preprocess()
        prob.sigma_scatter(peer_s)
        dist.all_reduce(token)

    for t in prob.g:
        t.fill_(float("nan"))
    pull_step()
    torch.cuda.synchronize()
    same_g = float(g_digest() == g_keep)
    same_g = -allreduce_max(-same_g, world)
    del g_keep
    barrier(world)
    start.record(stream)
    for _ in range(args.gf_fused_steps):
        prob.pull_g(peer_g)
    end.record(stream)
    torch.cuda.synchronize()
    pull_ms = allreduce_max(start.elapsed_time(end) / args.gf_fused_steps, world)
    barrier(world)
    start.record(stream)
    for _ in range(args.gf_fused_steps):
        pull_step()
    end.record(stream)
    torch.cuda.synchronize()
    pull_step_ms = allreduce_max(start.elapsed_time(end) / args.gf_fused_steps, world)
    slab_bytes = 2 * prob.n_slab * p.n_kz * p.n_E * p.n_orb ** 2 * 16
    fused_info["pull"] = {
        "s_per_step": pull_step_ms / 1e3, "vs_halo_step": pull_step_ms / step_ms,
        "pull_ms": pull_ms, "pull_GB_per_s": slab_bytes / (pull_ms * 1e-3) / 1e9,
        "slab_bitwise_equal": bool(same_g == 1.0),
        "note": "G slab (owned + halo atoms, both polarities) pulled from the point owners by sse_slab_from_points "
                "(NVLink loads), then preprocess_D + K2 + K3 with Sigma stored to the owners from the epilogue",
    }
    if args.pi_steps > 0:
        # Pi from the point layout too (K5 / K6 read G over NVLink), returned to the (q, w) owners
        def fused_pi():
            prob.pi_peer(peer_g)
            return [sdist.pi_to_points(prob.pi_out[pol], p.n_A, p.n_qz, p.n_w) for pol in range(2)]

        fused_pi()
        torch.cuda.synchronize()
        barrier(world)
        start.record(stream)
        for _ in range(args.pi_steps):
            fused_pi()
        end.record(stream)
        torch.cuda.synchronize()
        fused_info["pi_s_per_eval"] = allreduce_max(start.elapsed_time(end) / args.pi_steps, world) / 1e3
        fused_info["pi_note"] = ("Pi with G read from the point owners (K5 G2, K6 G1 rows over NVLink) + "
                                 "Pi to the (q,w) point owners (NCCL all-to-all)")

        def pull_pi():  # the slab is already pulled by pull_step
            prob.pi()
            return [sdist.pi_to_points(prob.pi_out[pol], p.n_A, p.n_qz, p.n_w) for pol in range(2)]

        pull_pi()
        torch.cuda.synchronize()
        barrier(world)
        start.record(stream)
        for _ in range(args.pi_steps):
            pull_pi()
        end.record(stream)
        torch.cuda.synchronize()
        fused_info["pull"]["pi_s_per_eval"] = allreduce_max(start.elapsed_time(end) / args.pi_steps, world) / 1e3
    barrier(world)
    del d_pts
    peer_g.close()
    peer_s.close()
    return fused_info


def cpu_baseline_leg(args, p, grid, idx, prob):
    """The bench's CPU leg: parity of a few Sigma blocks of this run against the oracle
    (pointwise, host regeneration of the atom-keyed inputs) and the reference algorithm
    (oracle port of BATCHED_FUSED) timed on a bounded sample."""
    check = None
    if args.check:
        sys.path.insert(0, os.path.join(REPO, "tests"))
        from tests.scale_helpers import host_point

        worst = 0.0
        for a in (prob.lo, prob.lo + 1, prob.hi - 1):
            for (k, e) in ((0, p.n_E - 1), (p.n_kz - 1, p.n_E // 2)):
                for pol in (0, 1):
                    got = prob.sigma_block(pol, k, e, a)
                    ref = host_point(prob, pol, k, e, a)
                    worst = max(worst, float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300)))
        check = worst
    cpu = None
    if args.cpu_pairs > 0:
        s = cpu_sample(p, grid, idx, args.cpu_pairs)
        cpu = {"value": s["extrapolated_s"], "unit": "s", "cores": blas_threads(), "kind": "port",
               "sample": (f"{s['pairs']} (atom, neighbour) pairs of the reference BATCHED_FUSED algorithm "
                          f"(oracle port of sse.py:265-302) at the real per-pair shapes in {s['seconds']:.1f} s, "
                          f"x NA*NB={p.n_A * p.n_B}; {os.cpu_count()} host cores, ~1 busy")}
    return check, cpu


def run_gpu(args, p, grid, idx) -> None:
    import torch

    rank, world, local_rank = env_rank()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_1912_08810_b200 import dist as sdist
    from paper_1912_08810_b200.problem import ShardProblem
    from paper_1912_08810_b200.sse import Profile, alg_flops

    prob = ShardProblem(p, rank=rank, world=world, device=local_rank, seed=0, grid=grid, idx=idx)
    prob.allocate()
    prob.fill(owned_g_only=world > 1)
    exchange = None
    plan = None
    if world > 1:
        plan = sdist.halo_plan(idx, world, rank)
        exchange = lambda pr: sdist.exchange_halos(pr.g, plan)  # noqa: E731
    for _ in range(args.warmup):
        prob.step(exchange)
    torch.cuda.synchronize()
    barrier(world)

    stream = torch.cuda.current_stream()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(",".join(str(i) for i in range(world)) if rank == 0 else "0") as clocks:
        with Profile(device=local_rank) as prof:
            torch.cuda.synchronize()
            barrier(world)
            start.record(stream)
            for _ in range(args.steps):
                prob.step(exchange)
            end.record(stream)
            torch.cuda.synchronize()
        barrier(world)
    step_ms = start.elapsed_time(end) / args.steps
    step_ms = allreduce_max(step_ms, world)
    total_flops = alg_flops(p.n_kz, p.n_qz, p.n_E, p.n_A, p.n_B, p.n_orb, grid.offsets)
    sig = prof.result["sigma"]
    k3_ms_per_launch = sig["ms"] / max(sig["launches"], 1)
    k3_flops_per_launch = sig["flops"] / max(sig["launches"], 1)
    k3_tflops = k3_flops_per_launch / (k3_ms_per_launch * 1e-3) / 1e12 if sig["ms"] > 0 else 0.0
    k3_tflops = allreduce_sum(k3_tflops, world) / world  # mean over ranks (per-GPU kernel rate)
    launches = sum(v["launches"] for v in prof.result.values())
    if world > 1:
        launches += 0  # NCCL kernels are the library's, not counted as ours
    k3_share = sig["ms"] / (step_ms * args.steps) if step_ms > 0 else None
    clk = clocks.summary() if rank == 0 else {}

    # cpu_baseline leg (rank 0, N = 1): the reference algorithm timed on the host cores, and the
    # oracle as the checker of a few output blocks of this run (the only oracle use in the bench)
    check, cpu = None, None
    if rank == 0 and world == 1:
        check, cpu = cpu_baseline_leg(args, p, grid, idx, prob)

    common = (args, p, grid, idx, prob, world, local_rank, step_ms, start, end, stream)
    pi_info = pi_phase(*common)
    gf_info = gf_layout_phase(*common)
    fused_info = gf_fused_phase(*common)

    prob.free()
    del prob
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    barrier(world)

    e2e = None
    if args.e2e:
        e2e = e2e_phase(args, p, grid, idx, rank, world, local_rank)

    phase = None
    if args.phase_steps > 0 and world == 1:
        phase = phase_e2e(args, p, grid, idx, local_rank)


    if rank == 0:
        traffic = load_traffic()
        line = {
            "metric": METRIC, "value": step_ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic (atom-keyed counter-based generator, filled on device)",
            "config": {
                "workload": workload_name(p), "name": args.config,
                "parallelism": f"atom-shard x{world}" + (" + NCCL G halo exchange" if world > 1 else ""),
                "l2": "no flush: inputs (G 47.5 GB) >> 126 MB L2",
                "step": "preprocess_D + operator build (K2) + fused DMMA Sigma (K3), both polarities"
                        + (" + G halo exchange" if world > 1 else ""),
            },
            "tflops": total_flops / (step_ms * 1e-3) / 1e12,
            "tflops_per_gpu": total_flops / (step_ms * 1e-3) / 1e12 / world,
            "roofline": {
                "bound": "tensor", "kernel": k3_kernel_name(),
                "achieved": k3_tflops, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": k3_tflops / FP64_PEAK_TFLOPS, "peak_source": FP64_PEAK_SOURCE,
                "traffic": (traffic or {}).get("dram_bytes_per_launch"),
                "k3_ms_per_launch": k3_ms_per_launch, "k3_launches_per_step": sig["launches"] / args.steps,
                "k3_share_of_step": k3_share,
            },
            "gpu_launches": launches,
            "kernels": prof.result,
            "clocks": clk,
        }
        if plan is not None:
            line["halo"] = {"atoms_received": plan.halo_atoms(),
                            "bytes_per_step": sdist.halo_bytes(plan, p.n_kz * p.n_E * p.n_orb**2 * 16)}
        if check is not None:
            line["parity_check_max_rel_dev"] = check
        if pi_info is not None:
            line["pi"] = pi_info
            # the whole SSE phase of a Born iteration (sse.py:532-534): Sigma (`value`, SURVEY 8d's
            # unit of work) + Pi, both device-resident
            line["sse_phase_device_s"] = step_ms / 1e3 + pi_info["s_per_eval"]
        if gf_info is not None:
            line["gf_layout"] = gf_info
        if fused_info is not None:
            line["gf_layout_fused"] = fused_info
        if e2e is not None:
            line["e2e"] = e2e
        if phase is not None:
            line["sse_phase_e2e"] = phase
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--config", default="paper", choices=("tiny", "small", "paper", "kheavy", "large"))
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-warmup", type=int, default=1)
    ap.add_argument("--cpu-pairs", type=int, default=2, help="pairs timed for cpu_baseline (0 = skip)")
    ap.add_argument("--ref-pairs", type=int, default=1, help="pairs per step of --impl reference")
    ap.add_argument("--no-check", dest="check", action="store_false")
    ap.add_argument("--pi-steps", type=int, default=1, help="timed Pi evaluations after Sigma (0 = skip)")
    ap.add_argument("--phase-steps", type=int, default=0,
                    help="N=1: timed SSE phases (preprocess_D + Sigma + Pi) through sse_phase from pinned host memory")
    ap.add_argument("--gf-fused-steps", type=int, default=0,
                    help="N>1: timed steps reading G from / writing Sigma to the GF point owners over NVLink")
    ap.add_argument("--gf-layout-steps", type=int, default=0,
                    help="N>1: timed steps starting from the GF (k,E)-point layout (two all-to-alls)")
    args = ap.parse_args()

    from paper_1912_08810_b200.inputs import config

    p, grid, nmap = config(args.config)
    if args.impl == "reference":
        run_reference(args, p, grid, nmap.idx)
    else:
        run_gpu(args, p, grid, nmap.idx)


if __name__ == "__main__":
    main()
