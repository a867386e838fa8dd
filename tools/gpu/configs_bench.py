"""Throughput of every BASELINE.json config at its full size on one B200
(device-timed with CUDA events around usp_iterate / usp_bicgstab, after a
warm-up solve).  Prints one JSON line per config."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2207_14222_b200 import Plan
from synth import make

dev = torch.device("cuda", 0)
only = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]
for name in only:
    p = make(name, None, device=str(dev) if name in ("C3", "C4", "C5") else None)
    real = p.kind == "diffusion"
    if isinstance(p.medium, np.ndarray):
        med = torch.from_numpy(np.asarray(p.medium).real.astype(np.float32) if real else np.asarray(p.medium).astype(np.complex64)).to(dev)
        src = torch.from_numpy(np.asarray(p.source).real.astype(np.float32) if real else np.asarray(p.source).astype(np.complex64)).to(dev)
    else:
        med = p.medium.real.float() if real else p.medium.to(torch.complex64)
        src = p.source.real.float() if real else p.source.to(torch.complex64)
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        plan = Plan(p.shape, kind=p.kind, h=p.h, D=p.D, dtype="r32" if real else "c64", stream=stream, device=dev)
        res = {}
        for solver in ("fixed_point", "fixed_point", "bicgstab", "bicgstab", "gmres20", "gmres20"):
            if solver != "fixed_point" and (real or len(p.shape) == 1):
                continue
            plan.set_potential(med, 0.95)
            plan.set_source(src)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(stream)
            if solver == "fixed_point":
                n, term = plan.iterate(p.n_iter, p.alpha, p.tol)
            elif solver == "bicgstab":
                n, term = plan.bicgstab(20000, p.tol if p.tol > 0 else 1e-6)
            else:
                if getattr(plan, "kworkspace", None) is not None:   # BiCGSTAB's 5 fields are not needed any more
                    plan.kworkspace = None
                    torch.cuda.empty_cache()
                m = 20 if int(np.prod(p.shape)) <= 256 ** 3 else 5     # basis memory: (m + 2) fields
                n, term = plan.gmres(m, 40000, p.tol if p.tol > 0 else 1e-6)
            b.record(stream)
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            nvox = int(np.prod(p.shape))
            res[solver] = {"count": n, "term": term, "ms": round(ms, 3), "ms_per_count": round(ms / max(n, 1), 5),
                           "vox_it_per_s": nvox * n / (ms / 1e3), "residual": plan.residual()[0]}
        print(json.dumps({"config": name, "shape": list(p.shape), "dtype": "f32 (real path)" if real else "c64",
                          "tol": p.tol, "n_iter": p.n_iter, **res}), flush=True)
        plan.close()
    del med, src, p
    torch.cuda.empty_cache()
