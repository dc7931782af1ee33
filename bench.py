"""SSE Sigma^{<>} benchmark on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config paper]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...

One step = one Sigma^{<>} evaluation of a Born iteration (both polarities;
sse.py:533) on the paper-scale FinFET workload (BASELINE.json configs[2]:
NA=4864, NB=4, No=12, NE=706, Nw=70, Nkz=Nqz=3), strong-scaled over N GPUs
by atom sharding (one process per GPU, NCCL halo exchange of G inside the
step).  `value` = device time per step (CUDA events, inputs resident in HBM,
max over ranks).  `e2e` = the same step through the public drop-in
`paper_1912_08810_b200.sse_sigma(...)` on pageable numpy arrays (N=1; per rank
`sigma_host_slab` on numpy slabs for N>1), wall clock around the call, H2D/D2H
inside; `e2e.pinned` = the same C-ABI pipeline from pinned buffers.
`cpu_baseline` / `--impl reference` time the UNMODIFIED reference
(negflow.sse.sse_sigma(BATCHED_FUSED), bytecode staged in oracle/_ref by
oracle/make_ref.py) on single (atom, neighbour) pairs, x NA*NB.
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
FP64_PEAK_SOURCE = ("measured DMMA m8n8k4 sustained on this pool's B200 (profiles/r01_fp64_peak.json); MEASURED_PEAKS.json "
                    "has no FP64 entry; a DMMA-only loop later reached 37.15 TF/s (profiles/r02_dmma_k6_pattern.log), "
                    "the nominal rate is 148 SM x 64 FMA/clk x the SM clock: `frac_vs_nominal`")


def nominal_fp64_tflops(sm_mhz) -> float | None:
    """148 SMs x 128 flop/clk (64 DMMA FMA per SM per clock) x the SM clock measured during the run."""
    return 148 * 128 * sm_mhz / 1e6 if sm_mhz else None


def launched_kernel(kind: str) -> str:
    """Name (with template arguments) of the kernel of `kind` libsse actually launched last."""
    from paper_1912_08810_b200 import _lib

    return _lib.kernel_name(kind)


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
# CPU reference: the UNMODIFIED reference negflow (oracle/_ref) on single (atom, slot) pairs
# ---------------------------------------------------------------------------
def sample_pairs(p) -> list[tuple[int, int]]:
    """The (atom, neighbour slot) pairs the reference arm cycles through: both chain ends
    (duplicate neighbour slots, device.py:123-127) and interior atoms, every slot."""
    na, nb = p.n_A, p.n_B
    atoms = [0, na - 1, 1, na - 2, na // 2, na // 4, 3 * na // 4, na // 2 + 1]
    return [(a, i % nb) for i, a in enumerate(atoms)]


def negflow_pair(nf, p, idx, a: int, s: int, seed: int = 0) -> dict:
    """Sigma contribution of ONE (atom a, slot s) pair through the reference's own entry point
    negflow.sse.sse_sigma(BATCHED_FUSED) (sse.py:265-329), timed.

    The pair is a one-atom sub-problem with the self-map idx = [[0]] (sse_sigma checks neither
    f(a,s) != a nor reverse closure, sse.py:315-318): G column = G[:, :, f(a,s)], Dc row =
    Dc[:, :, a, s], dH row = dH[a, s], the full config's frequency map.  BATCHED_FUSED's per-pair
    work is independent of NA (sse.py:279-301), so NA * NB of these are one Sigma evaluation, and
    the NB pairs of an atom sum to Sigma[:, :, a].
    """
    from oracle import sse_oracle as orc
    from paper_1912_08810_b200 import inputs

    b = int(idx[a, s])
    g_l = inputs.atom_keyed_electron(seed, inputs.G_LESSER, p, [b])
    g_g = inputs.atom_keyed_electron(seed, inputs.G_GREATER, p, [b])
    atoms = sorted({a, *(int(x) for x in idx[a])})
    dcs = []
    for tid in (inputs.D_LESSER, inputs.D_GREATER):
        raw = inputs.atom_keyed_values(seed, tid, atoms, p.n_qz * p.n_w, (p.n_B + 1) * 9)
        d = {x: raw[i].reshape(p.n_qz, p.n_w, p.n_B + 1, 3, 3) for i, x in enumerate(atoms)}
        dcs.append(orc.preprocess_D_atom(lambda x: d[x], idx, a)[:, :, s].reshape(p.n_qz, p.n_w, 1, 1, 3, 3))
    dh = inputs.atom_keyed_dh(seed, p, [a])[:, s:s + 1].copy()
    ref_p = nf.params.SimParams(n_kz=p.n_kz, n_qz=p.n_qz, n_E=p.n_E, n_w=p.n_w, n_A=p.n_A, n_B=p.n_B,
                                n_orb=p.n_orb)
    grid = nf.params.default_grid(ref_p)
    g = nf.gf.GreensTensor(g_l, g_g)
    dc = nf.sse.CombinedD(dcs[0], dcs[1])
    nmap = nf.device.NeighborMap(np.zeros((1, 1), dtype=np.int64))
    t0 = time.perf_counter()
    out = nf.sse.sse_sigma(nf.sse.SseVariant.BATCHED_FUSED, g, dc, dh, nmap, grid)
    dt = time.perf_counter() - t0
    return {"seconds": dt, "atom": a, "slot": s, "sigma_l": out.lesser[:, :, 0], "sigma_g": out.greater[:, :, 0]}


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info

        return max((i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"), default=1)
    except Exception:
        return 1


def ref_provenance() -> str:
    from oracle.ref import ref_path

    path = ref_path()
    return f"{os.path.relpath(path, REPO) if path.startswith(REPO) else path}/negflow (unmodified reference)"


def bench_config(args, p) -> dict:
    """The workload both arms measure (identical dicts, so the driver can match the arms)."""
    return {"workload": workload_name(p), "name": args.config,
            "l2": "no flush: inputs (G 47.5 GB at paper) >> 126 MB L2"}


def run_reference(args, p, grid, idx) -> None:
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from oracle.ref import import_negflow

    # all host cores for the reference's BLAS, also under torchrun (which sets OMP_NUM_THREADS=1)
    try:
        from threadpoolctl import threadpool_limits

        _blas_limit = threadpool_limits(limits=os.cpu_count(), user_api="blas")  # noqa: F841 (kept alive)
    except Exception:
        pass
    nf = import_negflow()
    pairs = sample_pairs(p)
    for i in range(args.warmup):
        negflow_pair(nf, p, idx, *pairs[i % len(pairs)])
    times = []
    for i in range(args.steps):
        a, s = pairs[i % len(pairs)]
        times.append((a, s, negflow_pair(nf, p, idx, a, s)["seconds"]))
    per_pair = float(np.mean([t for _, _, t in times]))
    value = per_pair * p.n_A * p.n_B
    from paper_1912_08810_b200.sse import alg_flops

    flops = alg_flops(p.n_kz, p.n_qz, p.n_E, p.n_A, p.n_B, p.n_orb, grid.offsets)
    sample = (f"{args.steps} steps, one (atom, neighbour) pair each, cycling {len(pairs)} pairs (chain ends "
              f"and interior atoms, every slot) through negflow.sse.sse_sigma(BATCHED_FUSED) "
              f"(sse.py:265-329, the fastest reference arrangement) at the real per-pair shapes; "
              f"value = mean s/pair x NA*NB={p.n_A * p.n_B}; numpy/OpenBLAS {blas_threads()} threads of "
              f"{os.cpu_count()} host cores (the path is ~1 busy core)")
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64)",
        "data": "synthetic (atom-keyed generator)", "parallelism": "cpu (reference)",
        "config": bench_config(args, p),
        "tflops": flops / value / 1e12,
        "per_pair_s": {"mean": per_pair, "min": min(t for *_, t in times), "max": max(t for *_, t in times),
                       "pairs": [{"atom": a, "slot": s, "s": t} for a, s, t in times]},
        "cpu_baseline": {"value": value, "unit": "s", "cores": blas_threads(), "kind": "reference",
                         "sample": sample, "reference": ref_provenance()},
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


def _host_inputs(p, idx, glo, gA, lo, oA, local_rank, pinned: bool):
    """The step's inputs in host memory (same atom-keyed values as the resident run, generated on
    the device and copied out once): G slab [Nkz, NE, gA, No, No], Dc / dH of the owned atoms.
    pinned=False gives pageable numpy arrays (what a reference caller hands over)."""
    import torch

    from paper_1912_08810_b200 import inputs
    from paper_1912_08810_b200 import sse as dev

    no2 = p.n_orb * p.n_orb
    cuda = torch.device("cuda", local_rank)

    def host(t):
        if pinned:
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t)
            return h
        return t.cpu().numpy()

    g = []
    for tid in (inputs.G_LESSER, inputs.G_GREATER):
        tmp = torch.empty((p.n_kz, p.n_E, gA, p.n_orb, p.n_orb), dtype=torch.complex128, device=cuda)
        dev.fill_synthetic(tmp, 0, tid, glo, gA, p.n_kz * p.n_E, no2, no2, gA * no2)
        g.append(host(tmp))
        del tmp
    slots = (p.n_B + 1) * 9
    dc = []
    for tid in (inputs.D_LESSER, inputs.D_GREATER):
        d = torch.empty((p.n_qz, p.n_w, gA, p.n_B + 1, 3, 3), dtype=torch.complex128, device=cuda)
        dev.fill_synthetic(d, 0, tid, glo, gA, p.n_qz * p.n_w, slots, slots, gA * slots)
        out = torch.empty((p.n_qz, p.n_w, oA, p.n_B, 3, 3), dtype=torch.complex128, device=cuda)
        dev.preprocess_D_device(d, out, idx, d_atom0=glo, out_atom0=lo)
        dc.append(host(out))
        del d, out
    dht = torch.empty((oA, p.n_B, 3, p.n_orb, p.n_orb), dtype=torch.complex128, device=cuda)
    inner = p.n_B * 3 * no2
    dev.fill_synthetic(dht, 0, inputs.DH, lo, oA, 1, inner, inner, 0, scale=inputs.DH_SCALE)
    dh = host(dht)
    del dht
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return g, dc, dh


def _digest(arrays) -> int:
    """Layout-independent bit checksum (wrap-around int64 sum of the raw doubles)."""
    tot = 0
    for a in arrays:
        v = a if isinstance(a, np.ndarray) else a.numpy()
        tot += int(v.view(np.int64).sum(dtype=np.int64))
    return tot & ((1 << 64) - 1)


def e2e_phase(args, p, grid, idx, rank, world, local_rank, want_digest) -> dict:
    """End to end through the public API, host memory in and out, H2D/D2H inside the timed region.

    N = 1: `paper_1912_08810_b200.sse_sigma(BATCHED_FUSED, GreensTensor, CombinedD, dH, NeighborMap,
    EnergyGrid)` -- the drop-in for negflow.sse.sse_sigma (sse.py:305-329) -- on pageable numpy
    arrays, output allocated by the call as the reference does, wall clock (perf_counter) around
    the call.  N > 1: each rank's share through sigma_host_slab (sse_sigma_c128_slab) on pageable
    numpy slabs.  Also timed from pinned buffers (e2e.pinned), the same C-ABI pipeline without the
    staging ring.  The outputs are checked bit-for-bit against the device-resident run (digest).
    """
    from paper_1912_08810_b200 import sse as dev
    from paper_1912_08810_b200.problem import chunk
    from paper_1912_08810_b200.types import CombinedD, GreensTensor, NeighborMap, SseVariant

    lo, hi = chunk(p.n_A, world, rank)
    rows = idx[lo:hi]
    glo, ghi = int(min(lo, rows.min())), int(max(hi, rows.max() + 1))
    gA, oA = ghi - glo, hi - lo
    offs, wts = np.array(grid.offsets), np.array(grid.weights)
    res = {}
    for pinned in (False, True):
        g, dc, dh = _host_inputs(p, idx, glo, gA, lo, oA, local_rank, pinned)
        if world == 1 and not pinned:
            g_t, dc_t, nmap = GreensTensor(g[0], g[1]), CombinedD(dc[0], dc[1]), NeighborMap(idx)

            def call(tim):
                out = dev.sse_sigma(SseVariant.BATCHED_FUSED, g_t, dc_t, dh, nmap, grid, timing=tim)
                return out.lesser, out.greater
        else:
            import torch

            shape = (p.n_kz, p.n_E, oA, p.n_orb, p.n_orb)
            outs = ([torch.empty(shape, dtype=torch.complex128, pin_memory=True) for _ in range(2)] if pinned
                    else None)

            def call(tim):
                o = outs if pinned else [dev.alloc_host(shape) for _ in range(2)]
                tim.update(dev.sigma_host_slab(g[0], g[1], dc[0], dc[1], dh, rows, offs, wts, o[0], o[1],
                                               n_a=p.n_A, g_atom0=glo, out_atom0=lo, device=local_rank))
                return o[0], o[1]
        for _ in range(args.e2e_warmup):
            call({})
        times, tim, out = [], {}, None
        for _ in range(args.e2e_steps):
            barrier(world)
            tim = {}
            out = None
            t0 = time.perf_counter()
            out = call(tim)
            times.append(time.perf_counter() - t0)
        same = float(_digest(out) == want_digest)
        same = -allreduce_max(-same, world)
        t = allreduce_max(float(np.mean(times)), world)
        h2d = allreduce_sum(float(tim["h2d_bytes"]), world)
        d2h = allreduce_sum(float(tim["d2h_bytes"]), world)
        entry = {"value": t, "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                 "steps": args.e2e_steps, "warmup": args.e2e_warmup, "step_s": times,
                 "bitwise_equal_to_device_run": bool(same == 1.0),
                 "host_pack_ms": tim.get("h2d_ms"), "host_unpack_ms": tim.get("d2h_ms"),
                 "library_gpu_span_s": (tim.get("total_ms") or 0) / 1e3,
                 "staged": tim.get("staged"), "host_threads": tim.get("host_threads")}
        if pinned:
            entry["path"] = ("sigma_host_slab -> sse_sigma_c128_slab (C ABI) from pinned torch buffers: direct DMA "
                             "in the 3-stream H2D / compute / D2H pipeline")
            res["pinned"] = entry
        else:
            entry["path"] = (("paper_1912_08810_b200.sse_sigma (the drop-in, public API) on pageable numpy arrays, "
                              "output allocated by the call; " if world == 1 else
                              "sigma_host_slab (sse_sigma_c128_slab, C ABI) on pageable numpy slabs per rank; ")
                             + "libsse stages through its pinned ring (host worker pool) under the compute; "
                               "wall clock around the call")
            res.update(entry)
        del g, dc, dh, out, call
    return res


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
        "roofline": {"bound": "tensor", "kernel": launched_kernel("pi"), "build_kernel": launched_kernel("pi_build"),
                     "achieved": k6_tflops, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": k6_tflops / FP64_PEAK_TFLOPS},
        "kernels": {k: pprof.result[k] for k in ("pi_build", "pi", "pi_assemble")},
        "note": "phonon self-energy Pi (sse_pi) per Born iteration, V form: chain = w_E sum <G1(E+off)^T, "
                "dH_j G2 dH_i>; not part of `value` (north_star's path is Sigma)",
    }
    return pi_info


def device_phase(args, p, grid, idx, prob, world, local_rank, step_ms, start, end, stream):
    """the whole SSE phase (preprocess_D + Sigma + Pi) as ONE device call on the
    resident slabs (sse_phase_device; no host copies), CUDA events, max over ranks."""
    import torch

    from paper_1912_08810_b200.sse import Profile

    if args.phase_device_steps <= 0:
        return None
    prob.phase()
    torch.cuda.synchronize()
    barrier(world)
    with Profile(device=local_rank) as prof:
        start.record(stream)
        for _ in range(args.phase_device_steps):
            prob.phase()
        end.record(stream)
        torch.cuda.synchronize()
    ms = allreduce_max(start.elapsed_time(end) / args.phase_device_steps, world)
    return {"s_per_phase": ms / 1e3, "steps": args.phase_device_steps,
            "kernel_ms_per_phase": {k: v["ms"] / args.phase_device_steps for k, v in prof.result.items()
                                    if v["launches"]},
            "path": "sse_phase_device (C ABI): preprocess_D -> K2/K3 Sigma -> K5-K7 Pi on the resident G / raw D "
                    "slabs, outputs left in HBM (the loop's device-resident SSE phase, "
                    "loop.self_consistent_loop_device)"}


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
    """The bench's CPU leg (rank 0, N = 1).

    * check: a few Sigma blocks of this run against the pointwise oracle (oracle.sigma_point,
      pinned to the reference by tests/test_oracle.py);
    * cpu_baseline: the UNMODIFIED reference (negflow from oracle/_ref) on the NB pairs of one
      chain-end atom, timed; their sum is the reference's Sigma[:, :, a] over every (k, E) and is
      compared with this run's GPU Sigma of that atom (reference_atom_parity).
    """
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
    cpu, atom_parity = None, None
    if args.cpu_atoms > 0:
        from oracle.ref import import_negflow

        nf = import_negflow()
        a = p.n_A - 1
        runs = [negflow_pair(nf, p, idx, a, s) for s in range(p.n_B)]
        secs = [r["seconds"] for r in runs]
        ref_l = sum(r["sigma_l"] for r in runs)
        ref_g = sum(r["sigma_g"] for r in runs)
        got_l = prob.sig[0][a - prob.lo].cpu().numpy()
        got_g = prob.sig[1][a - prob.lo].cpu().numpy()
        scale = max(np.max(np.abs(ref_l)), np.max(np.abs(ref_g)))
        dev = max(np.max(np.abs(got_l - ref_l)), np.max(np.abs(got_g - ref_g))) / scale
        atom_parity = {"atom": a, "blocks": int(2 * p.n_kz * p.n_E), "max_rel_dev": float(dev),
                       "metric": "max|gpu - ref| / max(max|ref<|, max|ref>|) over Sigma[:, :, a] (test_acceptance.py:163-171)"}
        per_pair = float(np.mean(secs))
        cpu = {"value": per_pair * p.n_A * p.n_B, "unit": "s", "cores": blas_threads(), "kind": "reference",
               "sample": (f"the {p.n_B} (atom, neighbour) pairs of chain-end atom {a} through "
                          f"negflow.sse.sse_sigma(BATCHED_FUSED) (unmodified reference, sse.py:265-329) in "
                          f"{sum(secs):.1f} s ({min(secs):.2f}-{max(secs):.2f} s per pair), x NA*NB="
                          f"{p.n_A * p.n_B} / {p.n_B}; {os.cpu_count()} host cores, ~1 busy"),
               "reference": ref_provenance()}
    return check, cpu, atom_parity


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
    k3_name = launched_kernel("sigma")
    # layout-independent bit checksum of this rank's Sigma (checked against the e2e outputs)
    sig_digest = sum(int(torch.view_as_real(t).view(torch.int64).sum()) for t in prob.sig) & ((1 << 64) - 1)
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
    check, cpu, atom_parity = None, None, None
    if rank == 0 and world == 1:
        check, cpu, atom_parity = cpu_baseline_leg(args, p, grid, idx, prob)

    common = (args, p, grid, idx, prob, world, local_rank, step_ms, start, end, stream)
    pi_info = pi_phase(*common)
    phase_dev = device_phase(*common)
    gf_info = gf_layout_phase(*common)
    fused_info = gf_fused_phase(*common)

    prob.free()
    del prob
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    from paper_1912_08810_b200 import _lib as sse_lib

    sse_lib.context(device=local_rank).trim()  # the device legs' cached scratch (Pi operands: up to 48 GiB)
    barrier(world)

    e2e = None
    if args.e2e:
        e2e = e2e_phase(args, p, grid, idx, rank, world, local_rank, sig_digest)

    phase = None
    if args.phase_steps > 0 and world == 1:
        phase = phase_e2e(args, p, grid, idx, local_rank)


    if rank == 0:
        traffic = load_traffic()
        if traffic and traffic.get("launch_name") and traffic["launch_name"] not in k3_name:
            traffic = None  # the committed capture describes another K3 build: no traffic claim
        line = {
            "metric": METRIC, "value": step_ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic (atom-keyed counter-based generator, filled on device)",
            "config": bench_config(args, p),
            "parallelism": f"atom-shard x{world}" + (" + NCCL G halo exchange" if world > 1 else ""),
            "step": "preprocess_D + operator build (K2) + fused DMMA Sigma (K3), both polarities"
                    + (" + G halo exchange" if world > 1 else ""),
            "tflops": total_flops / (step_ms * 1e-3) / 1e12,
            "tflops_per_gpu": total_flops / (step_ms * 1e-3) / 1e12 / world,
            "roofline": {
                "bound": "tensor", "kernel": k3_name,
                "achieved": k3_tflops, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": k3_tflops / FP64_PEAK_TFLOPS, "peak_source": FP64_PEAK_SOURCE,
                "frac_vs_nominal": (k3_tflops / nominal_fp64_tflops(clk.get("sm_mhz"))
                                    if nominal_fp64_tflops(clk.get("sm_mhz")) else None),
                "traffic": (traffic or {}).get("dram_bytes_per_launch"),
                "traffic_source": (traffic or {}).get("capture"),
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
        if atom_parity is not None:
            line["reference_atom_parity"] = atom_parity
        if pi_info is not None:
            line["pi"] = pi_info
            # the whole SSE phase of a Born iteration (sse.py:532-534): Sigma (`value`, SURVEY 8d's
            # unit of work) + Pi, both device-resident
            line["sigma_plus_pi_device_s"] = step_ms / 1e3 + pi_info["s_per_eval"]
        if phase_dev is not None:
            line["sse_phase_device"] = phase_dev
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
    ap.add_argument("--cpu-atoms", type=int, default=1,
                    help="cpu_baseline: time the reference on the NB pairs of one atom and compare (0 = skip)")
    ap.add_argument("--no-check", dest="check", action="store_false")
    ap.add_argument("--pi-steps", type=int, default=1, help="timed Pi evaluations after Sigma (0 = skip)")
    ap.add_argument("--phase-device-steps", type=int, default=1,
                    help="timed SSE phases (preprocess_D + Sigma + Pi) as one device call (0 = skip)")
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
