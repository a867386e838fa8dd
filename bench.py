#!/usr/bin/env python3
"""Benchmark of the universal-split-preconditioner hot path on B200.

Metric (BASELINE.json): voxel-iterations/s (device-timed) and % of HBM
roofline.  Workload at N=1: BASELINE.json configs[4] "C5" -- 3-D Helmholtz
1024^3 complex64, 100 iterations of Algorithm 1 (the config the north star's
roofline target is quoted on; it fits one GPU).

One step = the whole hot path over one synthetic input:
canonical form + V/B setup (a0), source setup (s, Delta_0, n0), and 100
iterations (a1..a10), inputs resident in HBM.  Inputs (8 GiB each) are far
larger than L2 (126 MB), so no explicit flush is needed.

--impl reference runs the CPU oracle (oracle/, complex128, plain C + OpenMP)
on a bounded sample of the same workload on the host cores (this tier has no
installable reference implementation; the oracle is the reference arm).

Multi-GPU (torchrun, one process per GPU, N>1): C5 is split into N z-slabs
(libusp's slab decomposition: the two transposes around the z pass fused
into the K_B / K_C stores over NVLink -- an NCCL window, else CUDA IPC; NCCL
all-to-all if neither maps -- with an LSA-barrier, rank-ordered residual
all-gather; config.transposes says which ran) -- strong scaling, the total
work fixed.
Before timing, a closed-form check (constant V, 128^3) runs through the same
communicator; if it fails, the run falls back to N independent replicas
("scaling": "weak") and says so.  --replicas forces the replica mode.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "voxel-iterations/s (device-timed) and % of HBM roofline at 1/2/4/8 B200"
UNIT = "voxel-iterations/s"

# Algorithmic HBM bytes per voxel and iteration of each kernel class
# (complex64 = 8 B, float32 = 4 B
# per value), by the algebraic form the x pass ran (reading R-30 / R-31):
#   x_sparse  Algorithm 1 literally, source on <= 64 x-lines (s not read)
#   x_dense   Algorithm 1 literally, s read densely
#   delta     the Delta-form recurrence
# x pass (K_A): read work + x + B (+ s | + Delta), write x + work (+ Delta).
# Each strided pass (K_B, K_C, K_D) reads and writes work once (16 B).
# The plane-chained pass (kernels_plane.cu, NEXT-4) runs K_D, K_A and K_B
# with work L2-resident in between: HBM sees K_D's read and K_B's write of
# work (16 B) plus the x pass's operands.
XPASS_BYTES = {"x_sparse": 40, "x_dense": 48, "delta": 56}
PLANE_BYTES = {"x_sparse": 40, "x_dense": 48, "delta": 56}
STRIDED_BYTES = 16
# real path (C4 diffusion, float32 fields, half spectra; the 16 padding
# columns per spectrum row are overhead, not work)
XPASS_BYTES_REAL = {"x_sparse": 24, "x_dense": 24, "delta": 28}
STRIDED_BYTES_REAL = 8


def bytes_model(schedule, real):
    """(kernel -> {form -> B/voxel}, iteration {form -> B/voxel})."""
    if real:
        k = {"xpass": XPASS_BYTES_REAL, "y_fwd": STRIDED_BYTES_REAL, "z_fwd_mul_inv": STRIDED_BYTES_REAL,
             "y_inv": STRIDED_BYTES_REAL}
    elif schedule == "plane":
        k = {"plane_dab": PLANE_BYTES, "z_fwd_mul_inv": STRIDED_BYTES}
    else:
        k = {"xpass": XPASS_BYTES, "y_fwd": STRIDED_BYTES, "z_fwd_mul_inv": STRIDED_BYTES, "y_inv": STRIDED_BYTES}
    forms = ("x_sparse", "x_dense", "delta")
    it = {f: sum(v[f] if isinstance(v, dict) else v for v in k.values()) for f in forms}
    return k, it


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl" if args.impl == "usp" else "gloo")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(world, v: float) -> float:
    if world <= 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def ncu_traffic(workload):
    """Per-launch DRAM bytes of the kernels from the committed ncu --set full
    capture summary (profiles/ncu_traffic.json) when it was taken on this
    workload, else {}."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("bytes_per_launch", {}) if d.get("workload") == workload else {}
    except Exception:
        return {}


# ----------------------------------------------------------------- oracle --
def cpu_oracle_sample(shape=(256, 256, 256), iters=100):
    """The oracle as it stands (x-form Alg. 1, c128) on a bounded sample of the
    C5 recipe; returns (vox-it/s, seconds, threads, description)."""
    from oracle import oracle as O
    from synth import make

    O.build()
    p = make("C5", shape)
    med = p.medium.astype("complex64").astype("complex128")
    sp = O.canonical(p.kind, med)
    w = O.medium_to_w(p.kind, med)
    t0 = time.perf_counter()
    res = O.fixed_point(w, p.source, p.h, sp.D, sp.sigma, sp.c, 0.75, 0.0, iters)
    dt = time.perf_counter() - t0
    nvox = p.n_vox
    return nvox * res.n_done / dt, dt, O.num_threads(), (
        f"oracle x-form Alg. 1 (complex128) on the C5 recipe at {shape[0]}^3 "
        f"(lambda=8, GRF ell=4, seed 3), {iters} iterations incl. its setup FFT round trip")


REF_SAMPLE_ITERS = 10   # iterations of Alg. 1 per reference-arm step (256^3 sample)


def c5_workload(n_iter=100, shape=(1024, 1024, 1024)):
    """The usp arm's config.workload string for the default (C5, complex64) bench."""
    return (f"C5 3-D Helmholtz {shape[2]}x{shape[1]}x{shape[0]} complex64, "
            f"{n_iter} iterations of Alg. 1 per step (setup + iterations), alpha=0.75")


def run_reference(args, world, rank):
    """The reference arm: the CPU oracle as it stands on the box's host cores,
    on the usp arm's config / metric / unit; each step is a bounded sample of
    that workload (the C5 recipe at 256^3, setup + REF_SAMPLE_ITERS iterations
    of Alg. 1), stated in config.sample and cpu_baseline.sample."""
    if rank != 0:
        return 0
    from oracle import oracle as O
    from synth import make

    n_it = REF_SAMPLE_ITERS
    sample = (f"each step: the C5 recipe at 256^3 (lambda=8, GRF ell=4, seed 3), setup (n0 FFT round trip) + "
              f"{n_it} iterations of Alg. 1 (x-form, complex128) on the host cores")
    cfg = {"workload": c5_workload(), "grid": [1024, 1024, 1024], "iterations_per_step": 100,
           "sample": sample, "sample_grid": [256, 256, 256], "sample_iterations_per_step": n_it}
    O.build()
    p = make("C5", (256, 256, 256))
    med = p.medium.astype("complex64").astype("complex128")
    sp = O.canonical(p.kind, med)
    w = O.medium_to_w(p.kind, med)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        O.fixed_point(w, p.source, p.h, sp.D, sp.sigma, sp.c, 0.75, 0.0, n_it)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    tot = sum(times)
    # like the usp arm: voxel-iterations advanced / time of setup + iterations
    value = p.n_vox * n_it * args.steps / tot
    model, nproc = host_cpu()
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": O.num_threads(), "kind": "oracle",
                             "sample": sample, "seconds": round(tot, 2), "cpu_model": model, "nproc": nproc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------------- GPU --
def solver_comparison(dev, name="C3", tol=1e-6):
    """Time to tolerance of the two solvers on one config (Table 1b analogue
    on B200): the fixed-point iteration (Alg. 1, alpha = 0.75) and BiCGSTAB
    on the same preconditioned system (NEXT-2), device-timed."""
    import torch
    from paper_2207_14222_b200 import Plan
    from synth import make

    p = make(name, None, device=str(dev))
    med, src = p.medium.to(torch.complex64), p.source.to(torch.complex64)
    stream = torch.cuda.Stream(device=dev)
    out = {"config": name, "grid": list(p.shape), "tol": tol}
    with torch.cuda.stream(stream):
        plan = Plan(p.shape, kind=p.kind, h=p.h, D=p.D, stream=stream, device=dev)
        for solver in ("fixed_point", "bicgstab", "gmres20", "fixed_point", "bicgstab", "gmres20"):   # 2nd round timed
            plan.set_potential(med, 0.95)
            plan.set_source(src)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            if solver == "fixed_point":
                n, term = plan.iterate(20000, p.alpha, tol)
            elif solver == "bicgstab":
                n, term = plan.bicgstab(5000, tol)
            else:
                n, term = plan.gmres(20, 20000, tol)
            b.record(stream)
            torch.cuda.synchronize()
            unit = {"fixed_point": "iterations", "bicgstab": "passes (2 x (L+1)^-1)",
                    "gmres20": "Arnoldi steps (1 x (L+1)^-1)"}[solver]
            out[solver] = {"count": n, "term": term, "ms": round(a.elapsed_time(b), 3), "count_unit": unit}
        plan.close()
    return out


def slab_selfcheck(comm, world, rank, dev, separate, n_iter=8, shape=(128, 128, 128)):
    """Constant V through the decomposed path: x^_k = x^*(1 - q^k) per
    Fourier mode (the closed form of tests/test_gpu_parity.py).  Returns the
    relative L2 error (all ranks)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2207_14222_b200 import Plan

    k2 = (2 * math.pi / 8 * (1.0 + 0.05j)) ** 2
    sigma, c, alpha = -k2.real, -1j * abs(k2.imag) / 0.95, 0.75
    S = np.zeros(shape, dtype=np.complex64)
    S[tuple(s // 3 for s in shape)] = 1.0
    S[tuple(s // 5 for s in shape)] = 0.5 - 0.25j
    plan = Plan(shape, sigma=sigma, c=c, comm=comm, device=dev, separate_transposes=separate)
    z0, nzl = plan.z0, plan.local_shape[0]
    plan.set_potential(torch.full(plan.local_shape, k2, dtype=torch.complex64, device=dev), -1.0)
    plan.set_source(torch.from_numpy(np.ascontiguousarray(S[z0:z0 + nzl])).to(dev))
    plan.iterate(n_iter, alpha, 0.0)
    x = plan.get_field()
    parts = [torch.empty_like(x) for _ in range(world)]
    dist.all_gather(parts, x)
    plan.close()
    err = torch.zeros(1, dtype=torch.float64, device=dev)
    if rank == 0:
        xg = torch.cat(parts).cpu().numpy().astype(np.complex128)
        w = -complex(np.complex64(k2))
        b = 1.0 - (w - sigma) / c
        p2 = sum(np.meshgrid(*[(2 * np.pi * np.fft.fftfreq(n)) ** 2 for n in shape], indexing="ij"))
        g = c / (p2 + sigma + c)
        q = 1.0 - alpha * b * (1.0 - b * g)
        ref = np.fft.ifftn(g * np.fft.fftn(S.astype(np.complex128) / c) / (1.0 - b * g) * (1.0 - q ** n_iter))
        err[0] = float(np.linalg.norm(xg - ref) / np.linalg.norm(ref))
    dist.broadcast(err, src=0)
    return float(err.item())


def host_cpu():
    """CPU model and core count of the host (lscpu), for the cpu_baseline."""
    model, cores = None, os.cpu_count()
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return model, cores


def timed_iterations(plan, stream, n, alpha=0.75, warm=3):
    """Device time per iteration of n iterations (after `warm`), kernel-class
    profile, and the form summary of the plan."""
    import torch

    plan.iterate(warm, alpha, 0.0)
    plan.profile(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    nd, _ = plan.iterate(n, alpha, 0.0)
    b.record(stream)
    torch.cuda.synchronize()
    prof = plan.profile_read()
    plan.profile(False)
    return a.elapsed_time(b) / nd, prof


def variant_rooflines(dev, stream, med, src, p, hbm, n=20):
    """The same C5 problem on other plan options, each timed over n
    iterations: the general case (Delta-form, s read densely: what a dense
    source or a converging solve runs), and the plane-chained pass (NEXT-4)
    next to the default 4-pass schedule."""
    import torch
    from paper_2207_14222_b200 import Plan

    nloc = med.numel()
    out = {}
    for key, opts, form, desc in (
            ("general_delta_dense", {"delta_form": True, "dense_source": True}, "delta",
             "Delta-form (P:L613), s read densely"),
            ("plane_xform_sparse", {"plane_chain": True}, "x_sparse",
             "x-form, sparse source, plane-chained pass (K_C + one K_D/K_A/K_B kernel)"),
            ("plane_general", {"plane_chain": True, "delta_form": True, "dense_source": True}, "delta",
             "Delta-form, s read densely, plane-chained pass")):
        with torch.cuda.stream(stream):
            plan = Plan(p.shape, kind=p.kind, h=p.h, D=p.D, stream=stream, device=dev, **opts)
            plan.set_potential(med, 0.95)
            plan.set_source(src)
            ms, prof = timed_iterations(plan, stream, n)
            plan.close()
            del plan
            torch.cuda.empty_cache()
        sched = "plane" if "plane_dab" in prof else "4-pass"
        kmodel, itmodel = bytes_model(sched, False)
        bpv = itmodel[form]
        kern = {k: round(v[0] / v[1], 4) for k, v in prof.items() if k in kmodel}
        dk = max(kern, key=lambda k: kern[k] * prof[k][1])
        kb = kmodel[dk] if not isinstance(kmodel[dk], dict) else kmodel[dk][form]
        out[key] = {"form": desc, "schedule": sched, "bytes_per_voxel": bpv, "iter_ms": ms,
                    "achieved_gbs": bpv * nloc / (ms / 1e3) / 1e9, "frac": bpv * nloc / (ms / 1e3) / 1e9 / hbm,
                    "value": nloc / (ms / 1e3), "kernel_ms_per_launch": kern,
                    "dominant": {"kernel": dk, "bytes_per_voxel": kb, "ms": kern[dk],
                                 "frac": kb * nloc / (kern[dk] / 1e3) / 1e9 / hbm}}
    return out


def c4_line(dev, hbm, n_iter=200):
    """BASELINE.json C4 (512^3 float32 diffusion, the real half-spectrum
    path), one step of 200 iterations after a warm-up step, device-timed."""
    import torch
    from paper_2207_14222_b200 import Plan
    from synth import make

    p = make("C4", None, device=str(dev))
    med, src = p.medium.to(torch.float32), p.source.to(torch.float32)
    p.medium = p.source = None
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        plan = Plan(p.shape, kind=p.kind, h=p.h, D=p.D, dtype="r32", stream=stream, device=dev)
        for rep in range(2):
            plan.set_potential(med, 0.95)
            plan.set_source(src)
            if rep == 1:
                plan.profile(True)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            nd, _ = plan.iterate(n_iter, p.alpha, 0.0)
            b.record(stream)
            torch.cuda.synchronize()
        prof = plan.profile_read()
        h = plan.history()
        xf_plan, _, r_sw = plan.iteration_form()
        plan.close()
    ms = a.elapsed_time(b)
    nvox = med.numel()
    below = [k for k, r in enumerate(h[:n_iter]) if r < r_sw]
    n_x = (min(n_iter, below[0] + 1) if below else n_iter) if xf_plan else 0
    fx = n_x / n_iter
    kmodel, itmodel = bytes_model("4-pass", True)
    bpv = fx * itmodel["x_dense"] + (1 - fx) * itmodel["delta"]
    it_ms = ms / n_iter
    kx = fx * kmodel["xpass"]["x_dense"] + (1 - fx) * kmodel["xpass"]["delta"]
    xms = prof["xpass"][0] / n_iter
    return {"workload": "C4 3-D diffusion 512x512x512 float32 (half-spectrum real path), 200 iterations",
            "value": nvox * n_iter / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
            "iteration_form": f"x-form for {n_x} of {n_iter} iterations, then Delta-form",
            "iteration_roofline": {"bytes_per_voxel": bpv, "iter_ms": it_ms,
                                   "achieved_gbs": bpv * nvox / (it_ms / 1e3) / 1e9,
                                   "frac": bpv * nvox / (it_ms / 1e3) / 1e9 / hbm},
            "xpass_roofline": {"bytes_per_voxel": kx, "ms": xms, "frac": kx * nvox / (xms / 1e3) / 1e9 / hbm},
            "kernel_ms_per_launch": {k: round(v[0] / v[1], 4) for k, v in prof.items()}}


def run_usp(args, world, rank, local):
    import numpy as np
    import torch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2207_14222_b200 import Plan
    from synth import make

    name = args.config
    # multi-GPU: z-slabs over the ranks (strong scaling) unless the check fails
    comm, slab_check, mode = None, None, ("1 GPU" if world == 1 else "replicas")
    transposes = None
    separate = args.separate_transposes
    if world > 1 and not args.replicas:
        from paper_2207_14222_b200 import comm_init

        comm = comm_init()
        # fused peer-store transposes first; if their closed-form check fails,
        # the NCCL all-to-all transposes; if that fails too, replicas
        for sep in ((True,) if separate else (False, True)):
            slab_check = slab_selfcheck(comm, world, rank, dev, sep)
            if slab_check <= 1e-4:
                mode = "slabs"
                separate = sep
                transposes = "NCCL all-to-all" if sep else "fused peer-memory stores"
                break
        if mode != "slabs":
            comm.close()
            comm = None
    p = make(name, None if args.size is None else (args.size,) * 3, device=str(dev))
    shape = p.shape
    n_iter = args.iters if args.iters else p.n_iter
    stream = torch.cuda.Stream(device=dev)
    if args.virtual_ranks > 1 and world == 1:
        mode = "virtual"
    real = p.kind == "diffusion"          # C4: float32 data, the real (half-spectrum) path
    fdt = torch.float32 if real else torch.complex64
    esz = 4 if real else 8
    with torch.cuda.stream(stream):
        plan = Plan(shape, kind=p.kind, h=p.h, D=p.D, stream=stream, device=dev, comm=comm,
                    dtype="r32" if real else "c64", virtual_ranks=args.virtual_ranks if mode == "virtual" else 0,
                    separate_transposes=separate)
    z0, nzl = plan.z0, plan.local_shape[0]
    if real:
        med = p.medium[z0:z0 + nzl].real.to(fdt).contiguous()
        src = p.source[z0:z0 + nzl].real.to(fdt).contiguous()
    else:
        med = p.medium[z0:z0 + nzl].to(fdt).contiguous()
        src = p.source[z0:z0 + nzl].to(fdt).contiguous()
    del p.medium, p.source
    torch.cuda.empty_cache()
    nvox = int(np.prod(shape))              # global voxels
    nloc = int(np.prod(plan.local_shape))   # voxels this rank holds
    units = nvox if mode == "slabs" else nvox * world   # voxels all ranks advance per iteration

    it_events = []

    def step(m, s, where_host=False, out=None, timed=False):
        plan.set_potential(m, 0.95)
        plan.set_source(s)
        if timed:
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ea.record(stream)
        n, term = plan.iterate(n_iter, p.alpha, 0.0)
        if timed:
            eb.record(stream)
            it_events.append((ea, eb))
        assert n == n_iter, (n, term)
        if out is not None:
            plan.get_field(out)

    torch.cuda.synchronize()
    for _ in range(args.warmup):
        step(med, src)
    # ------------------------------------------------ timed region (device)
    sampler = ClockSampler(local)
    plan.profile(True)
    l0 = plan.launch_count()
    barrier(world)
    torch.cuda.synchronize()
    sampler.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step(med, src, timed=True)
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    barrier(world)
    ms = e0.elapsed_time(e1)
    launches = plan.launch_count() - l0
    prof = plan.profile_read()
    plan.profile(False)
    ms_max = max_over_ranks(world, ms)
    value = units * n_iter * args.steps / (ms_max / 1e3)

    # dominant kernel roofline: its algorithmic HBM bytes per iteration over
    # its device time per iteration
    hbm, peak_kind = peaks()
    n_it_total = n_iter * args.steps
    schedule = "plane" if "plane_dab" in prof else "4-pass"
    kmodel, itmodel = bytes_model(schedule, real)
    # which algebraic form ran: every timed step starts from set_source (x-form
    # on x-form plans) and ends still in the x-form unless r fell below r_switch
    xform_plan, xform_now, r_switch = plan.iteration_form()
    xform_all = xform_plan and xform_now
    n_x = 0                                         # x-form iterations per step
    if xform_all:
        n_x = n_iter
    elif xform_plan:
        # iteration k runs the x-form while r_{k-1} >= r_switch (R-30)
        h = plan.history()
        below = [k for k, r in enumerate(h[:n_iter]) if r < r_switch]
        n_x = min(n_iter, below[0] + 1) if below else n_iter
    fx = n_x / n_iter
    sparse_lines = plan.source_lines()
    xf = "x_sparse" if sparse_lines else "x_dense"

    def mix(v):
        return v if not isinstance(v, dict) else fx * v[xf] + (1 - fx) * v["delta"]

    kbytes = {k: mix(v) for k, v in kmodel.items()}
    form_desc = ("x-form (Algorithm 1 literally) throughout" +
                 (f", source on {sparse_lines} x-line(s) (s not streamed)" if sparse_lines else "") if xform_all else
                 (f"x-form for {n_x} of {n_iter} iterations, then Delta-form below r_switch = {r_switch:g}"
                  if xform_plan else "Delta-form"))
    dname = max((k for k in prof if k in kbytes), key=lambda k: prof[k][0])
    dms, dcount = prof[dname]
    d_ms_per_iter = dms / n_it_total
    dbytes = int(kbytes[dname] * nloc)              # per iteration (= per launch)
    # algorithmic bytes of the iterations over the kernel's total time (x-form
    # plans add one launch per iterate call that skips itself: time only)
    achieved = dbytes / (d_ms_per_iter / 1e3) / 1e9
    traffic = ncu_traffic(name).get(dname) if args.size is None and mode != "virtual" else None
    # iteration time: device time of the iterate() calls / iterations
    iter_ms = sum(a.elapsed_time(b) for a, b in it_events) / n_it_total
    kernel_share = {k: round(v[0] / sum(x[0] for x in prof.values()), 4) for k, v in prof.items()}

    variants = None
    if world == 1 and not args.no_variants and name == "C5" and mode == "1 GPU" and args.size is None:
        variants = variant_rooflines(dev, stream, med, src, p, hbm)

    # ------------------------------------------------ e2e (host buffers)
    e2e = None
    if not args.no_e2e:
        h_med = torch.empty(plan.local_shape, dtype=fdt, pin_memory=True)
        h_src = torch.empty(plan.local_shape, dtype=fdt, pin_memory=True)
        h_out = torch.empty(plan.local_shape, dtype=fdt, pin_memory=True)
        h_med.copy_(med)
        h_src.copy_(src)
        del med, src
        torch.cuda.empty_cache()
        # a sequence of --e2e-steps solves whatever --steps is (the default
        # --steps 3 would leave the unoverlapped first H2D / last D2H at ~9 %)
        e2e_steps = max(1, args.e2e_steps)
        step(h_med, h_src, out=h_out)   # warm the host path
        barrier(world)
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        n_serial = min(3, e2e_steps)       # the un-pipelined reference number
        for _ in range(n_serial):
            step(h_med, h_src, out=h_out)
        f1.record(stream)
        torch.cuda.synchronize()
        ems = max_over_ranks(world, f0.elapsed_time(f1))
        serial = units * n_iter * n_serial / (ems / 1e3)
        # pipelined through usp_stage_inputs: the next problem's medium and
        # source are copied on the plan's copy stream while this one iterates
        # (every step still copies its inputs in and its field out inside
        # the timed region)
        # results read back asynchronously (usp_get_field_async): step k's
        # field goes to the host while step k+1 runs; the last one is waited
        # for inside the timed region
        h_outs = [h_out, torch.empty_like(h_out).pin_memory()]

        def step_staged(i, last):
            plan.set_potential("staged", 0.95)
            plan.set_source("staged")
            if not last:
                plan.stage_inputs(h_med, h_src)
            n, term = plan.iterate(n_iter, p.alpha, 0.0)
            assert n == n_iter, (n, term)
            plan.get_field_async(h_outs[i % 2])

        plan.stage_inputs(h_med, h_src)   # warm the staged path
        step_staged(0, True)
        plan.wait_field()
        barrier(world)
        torch.cuda.synchronize()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        plan.stage_inputs(h_med, h_src)
        for i in range(e2e_steps):
            step_staged(i, i == e2e_steps - 1)
        plan.wait_field()                  # the last field is on the host
        g1.record(stream)
        torch.cuda.synchronize()
        gms = max_over_ranks(world, g0.elapsed_time(g1))
        e2e = {"value": units * n_iter * e2e_steps / (gms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": 2 * nloc * esz * world, "d2h_bytes_per_step": nloc * esz * world,
               "steps": e2e_steps, "input_copies": "pipelined (usp_stage_inputs: next problem's H2D during "
                                                   "this one's iterations; usp_get_field_async: the field's D2H "
                                                   "during the next one's)",
               "serial_value": serial}

    z_pass_buffer, transport = plan.work_layout(), plan.transport()
    # every rank destroys the plan here, in the same order: with the NCCL
    # window transport the destruction is collective (window deregistration,
    # device communicator)
    plan.close()   # the remaining measurements allocate their own plans
    del plan
    if rank != 0:
        return 0
    torch.cuda.empty_cache()
    solvers = None
    if world == 1 and not args.no_solvers and name == "C5":
        solvers = solver_comparison(dev)
    c4 = None
    if world == 1 and not args.no_variants and name == "C5" and args.size is None:
        c4 = c4_line(dev, hbm)
    cpu = None
    if world == 1 and not args.no_cpu:
        v, dt, thr, desc = cpu_oracle_sample()
        model, ncpu = host_cpu()
        cpu = {"value": v, "unit": UNIT, "cores": thr, "kind": "oracle", "sample": desc, "seconds": round(dt, 2),
               "cpu_model": model, "nproc": ncpu}
    # separate transposes (NCCL all-to-all / device copies) add their staging
    # reads and writes; the fused (peer-store) transposes add nothing to HBM
    iter_bpv = mix(itmodel) + ((16 if real else 32) if "all_to_all" in prof else 0)
    it_bytes = iter_bpv * nloc
    parallelism = {"1 GPU": "1 GPU", "replicas": f"{world} independent replicas",
                   "slabs": f"{world} z-slabs, transposes: {transposes} (self-check first)",
                   "virtual": f"1 GPU, {args.virtual_ranks} virtual z-slabs ("
                              + ("separate transposes" if separate else
                                 "transposes fused into the K_B / K_C stores") + ")"}[mode]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if mode == "slabs" else "weak", "vs_baseline": None, "dtype": "f32" if real else "c64",
        "data": "synthetic",
        "config": {"workload": f"{name} 3-D {'diffusion' if real else 'Helmholtz'} {shape[2]}x{shape[1]}x{shape[0]} "
                               f"{'float32 (half-spectrum path)' if real else 'complex64'}, "
                               f"{n_iter} iterations of Alg. 1 per step (setup + iterations), alpha=0.75",
                   "grid": list(shape), "iterations_per_step": n_iter, "iteration_form": form_desc,
                   "parallelism": parallelism, "slab_check_rel_l2": slab_check,
                   "z_pass_buffer": z_pass_buffer, "transposes": transport,
                   "l2": "inputs (8 GiB fields) larger than L2; no flush"},
        "roofline": {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic, "peak_kind": peak_kind,
                     "algorithmic_bytes_per_iteration": dbytes, "ms_per_iteration": d_ms_per_iter,
                     "launches_per_iteration": dcount // n_it_total, "launches_per_step": dcount / args.steps,
                     "schedule": schedule},
        "iteration_roofline": {"bytes_per_voxel": iter_bpv, "iter_ms": iter_ms,
                               "achieved_gbs": it_bytes / (iter_ms / 1e3) / 1e9,
                               "frac": it_bytes / (iter_ms / 1e3) / 1e9 / hbm},
        "kernel_share": kernel_share,
        "kernel_ms_per_launch": {k: round(v[0] / v[1], 4) for k, v in prof.items()},
        "gpu_launches": launches,
        "clocks": clocks,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "solvers_to_tol": solvers,
        "variants": variants,
        "c4_real_path": c4,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="usp", choices=["usp", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--size", type=int, default=None, help="override cubic grid edge (debug)")
    ap.add_argument("--iters", type=int, default=None)
    # a pipelined sequence: the first problem's H2D (16 GiB at C5) is not
    # overlapped by anything, so the number is over a sequence of 10 solves
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent replicas instead of slabs")
    ap.add_argument("--no-solvers", action="store_true", help="skip the C3 fixed-point vs BiCGSTAB comparison")
    ap.add_argument("--no-variants", action="store_true",
                    help="skip the general-case / 4-pass rooflines and the C4 line")
    ap.add_argument("--separate-transposes", action="store_true",
                    help="slab decomposition: NCCL all-to-all transposes instead of the fused peer stores")
    ap.add_argument("--virtual-ranks", type=int, default=0,
                    help="N=1: run the slab-decomposed path with this many virtual slabs (measurement)")
    args = ap.parse_args()
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        rc = run_reference(args, world, rank)
    else:
        rc = run_usp(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
