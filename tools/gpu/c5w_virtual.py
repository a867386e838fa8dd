"""C5w (BASELINE.json configs[4], weak scaling: 2048 x 1024 x 1024 complex64)
as 8 virtual z-slabs on one B200: every kernel, layout and peer-pointer
index of the 8-GPU slab decomposition (fused peer-store transposes), one GPU.

  1. closed form: constant V, a source of grid plane waves; every voxel of
     x_k has a closed form (tests/test_gpu_parity.py), compared in z-chunks;
  2. timing: the C5w recipe (C5's GRF medium at 2048 x 1024^2, point source),
     100 iterations of Algorithm 1, device-timed, per-kernel times.

Writes one JSON object (stdout and --out).
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def closed_form(P, shape, K=3):
    import numpy as np
    import torch
    from paper_2207_14222_b200 import Plan

    nz, ny, nx = shape
    dev = "cuda"
    k0, nidx = 2 * math.pi / 8, 1.0 + 0.05j
    k2 = (k0 * nidx) ** 2
    sigma, c = -k2.real, -1j * abs(k2.imag) / 0.95
    alpha = 0.75
    rng = np.random.default_rng(11)
    modes = [(int(rng.integers(-nz // 2, nz // 2)), int(rng.integers(-ny // 2, ny // 2)),
              int(rng.integers(-nx // 2, nx // 2))) for _ in range(4)] + [(0, 0, 0), (nz // 2, 5, -9)]
    amps = rng.standard_normal(len(modes)) + 1j * rng.standard_normal(len(modes))
    az, ay, ax = (torch.arange(n, device=dev, dtype=torch.float64) for n in shape)

    def field_chunk(coefs, z0, z1):
        out = torch.zeros((z1 - z0, ny, nx), dtype=torch.complex128, device=dev)
        for (mz, my, mx), a in zip(modes, coefs):
            ez = torch.exp(1j * 2 * math.pi * mz * az[z0:z1] / nz)
            ey = torch.exp(1j * 2 * math.pi * my * ay / ny)
            ex = torch.exp(1j * 2 * math.pi * mx * ax / nx)
            out += complex(a) * ez[:, None, None] * ey[None, :, None] * ex[None, None, :]
        return out

    plan = Plan(shape, sigma=sigma, c=c, virtual_ranks=P)
    S = torch.empty(shape, dtype=torch.complex64, device=dev)
    for z0 in range(0, nz, 128):
        S[z0:z0 + 128] = field_chunk(amps, z0, z0 + 128).to(torch.complex64)
    plan.set_potential(torch.full(shape, k2, dtype=torch.complex64, device=dev), -1.0)
    plan.set_source(S)
    del S
    torch.cuda.empty_cache()
    plan.iterate(K, alpha, 0.0)
    x = plan.get_field()
    w = -complex(np.complex64(k2))
    b = 1.0 - (w - sigma) / c
    coefs = []
    for (mz, my, mx), a in zip(modes, amps):
        p2 = sum((2 * math.pi * ((m + n // 2) % n - n // 2) / n) ** 2 for m, n in zip((mz, my, mx), shape))
        g = c / (p2 + sigma + c)
        q = 1.0 - alpha * b * (1.0 - b * g)
        coefs.append(a / c * g / (1.0 - b * g) * (1.0 - q ** K))
    num = den = 0.0
    for z0 in range(0, nz, 128):
        ref = field_chunk(coefs, z0, z0 + 128)
        d = x[z0:z0 + 128].to(torch.complex128) - ref
        num += float(torch.vdot(d.flatten(), d.flatten()).real)
        den += float(torch.vdot(ref.flatten(), ref.flatten()).real)
    plan.close()
    del x
    torch.cuda.empty_cache()
    return math.sqrt(num / den)


def timing(P, n_iter=100, steps=2):
    import torch
    from paper_2207_14222_b200 import Plan
    from synth import make

    dev = torch.device("cuda", 0)
    p = make("C5w", None, device="cuda")
    med, src = p.medium.to(torch.complex64), p.source.to(torch.complex64)
    p.medium = p.source = None
    torch.cuda.empty_cache()
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        plan = Plan(p.shape, stream=stream, device=dev, virtual_ranks=P)
        plan.set_potential(med, 0.95)
        plan.set_source(src)
        plan.iterate(3, p.alpha, 0.0)          # warm-up
        ms = []
        for s in range(steps):
            plan.set_potential(med, 0.95)
            plan.set_source(src)
            plan.profile(s == steps - 1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            nd, _ = plan.iterate(n_iter, p.alpha, 0.0)
            b.record(stream)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        prof = plan.profile_read()
        form = plan.iteration_form()
        lines = plan.source_lines()
        plan.close()
    nvox = med.numel()
    it_ms = min(ms) / n_iter
    return {"grid": list(p.shape), "iterations": n_iter, "iter_ms": it_ms, "value": nvox / (it_ms / 1e3),
            "iterate_ms": ms, "form": {"xform_plan": form[0], "xform_now": form[1], "source_lines": lines},
            "kernel_ms_per_launch": {k: round(v[0] / v[1], 4) for k, v in prof.items()}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    torch.cuda.set_device(0)
    t0 = time.time()
    err = closed_form(args.P, (2048, 1024, 1024))
    rec = {"workload": "C5w 2048x1024x1024 complex64 as 8 virtual z-slabs on one B200 "
                       "(fused peer-store transposes through the slab layouts)",
           "virtual_ranks": args.P, "closed_form_rel_l2_3_iterations": err}
    rec.update(timing(args.P))
    rec["wall_s"] = round(time.time() - t0, 1)
    rec["pass"] = err <= 2e-5
    print(json.dumps(rec), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main()
