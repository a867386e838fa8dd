"""Full-length parity runs at the BASELINE.json sizes (test infrastructure; run
on a GPU box, not collected by pytest):

    python tests/parity_fullsize.py [--configs C1,C2,C3,C4,C5] [--out profiles/parity_fullsize_r02.json]

Per config, the CUDA path (C-ABI, the bench's launch configuration) and the
CPU oracle (complex128, Algorithm 1 literally) run the same
seeded inputs for the config's own iteration count / tolerance:

* C1 (256, 1-D) and C2 (512^2): to 1e-6 -- counts (north_star: +-1) and the
  field at the GPU's count;
* C3 (256^3): exactly 500 iterations, and to 1e-6 (count +-1);
* C4 (512^3 float32, real path): exactly 200 iterations;
* C5 (1024^3): exactly 100 iterations (~50 min of oracle time on 16 cores,
  ~130 GiB of host RAM).

Writes one JSON object per config (relative L2 of the field, max relative
deviation of the residual history, counts, wall times) into --out.
"""
from __future__ import annotations

import argparse
import gc
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def inputs(name):
    import torch
    from synth import make

    p = make(name, device="cuda")
    if p.kind == "helmholtz":
        med, src, dtype = p.medium.to(torch.complex64), p.source.to(torch.complex64), "c64"
    else:
        med, src, dtype = p.medium.to(torch.float32), p.source.to(torch.float32), "r32"
    p.medium = p.source = None
    torch.cuda.empty_cache()
    return p, med, src, dtype


def gpu_run(p, med, src, dtype, n, tol):
    import torch
    from paper_2207_14222_b200 import Plan

    plan = Plan(p.shape, kind=p.kind, h=p.h, D=p.D, dtype=dtype)
    plan.set_potential(med, 0.95)
    plan.set_source(src)
    torch.cuda.synchronize()
    t0 = time.time()
    nd, term = plan.iterate(n, p.alpha, tol)
    torch.cuda.synchronize()
    t = time.time() - t0
    x = plan.get_field().cpu().numpy()
    h = plan.history()
    plan.close()
    torch.cuda.empty_cache()
    return x, nd, term, h, t


def oracle_run(O, p, med_np, src_np, n, tol):
    t0 = time.time()
    sp = O.canonical(p.kind, med_np, 0.95, D=p.D)
    gc.collect()
    w = np.empty(med_np.shape, dtype=np.complex128)
    if p.kind == "helmholtz":
        np.negative(med_np, out=w)
    else:
        w[...] = med_np
    S = np.zeros(src_np.shape, dtype=np.complex128)
    nz = np.flatnonzero(src_np)
    S.flat[nz] = src_np.flat[nz]
    res = O.fixed_point(w, S, p.h, sp.D, sp.sigma, sp.c, p.alpha, tol, n)
    del w, S
    gc.collect()
    return res, time.time() - t0


def rel_l2_chunked(xg, xr):
    num = den = 0.0
    for z0 in range(0, xr.shape[0], 64):
        a = xg[z0:z0 + 64].astype(np.complex128)
        b = xr[z0:z0 + 64]
        d = a - b
        num += float(np.vdot(d, d).real)
        den += float(np.vdot(b, b).real)
    return math.sqrt(num / den)


def one(O, name, n, tol, tag):
    p, med, src, dtype = inputs(name)
    xg, ng, term, h, tg = gpu_run(p, med, src, dtype, n, tol)
    med_np, src_np = med.cpu().numpy(), src.cpu().numpy()
    del med, src
    res, to = oracle_run(O, p, med_np, src_np, n, tol)
    rec = dict(config=name, run=tag, grid=list(p.shape), dtype=dtype, alpha=p.alpha, tol=tol, n_max=n,
               gpu_count=int(ng), gpu_term=term, oracle_count=int(res.n_done), gpu_s=round(tg, 4),
               oracle_s=round(to, 1), oracle_threads=O.num_threads())
    if tol > 0 and res.n_done != ng:
        res, to2 = oracle_run(O, p, med_np, src_np, ng, 0.0)
        rec["oracle_s"] = round(to + to2, 1)
    m = min(ng, res.n_done)
    rec["rel_l2_field"] = rel_l2_chunked(xg, res.x)
    rec["hist_max_rel_dev"] = float(np.max(np.abs(h[:m] - res.hist[:m]) / res.hist[:m]))
    rec["r_last_gpu"] = float(h[ng - 1])
    rec["r_last_oracle"] = float(res.hist[m - 1])
    hh = h[: ng + 1]
    rec["monotone_gpu"] = bool(np.all(np.diff(hh) <= 1e-5 * hh[:-1]))
    rec["pass"] = bool(rec["rel_l2_field"] <= 1e-4 and (tol <= 0 or abs(ng - rec["oracle_count"]) <= 1))
    del xg, res
    gc.collect()
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "parity_fullsize_r02.json"))
    args = ap.parse_args()
    from oracle import oracle as O

    O.build()
    out = []
    if os.path.exists(args.out):
        with open(args.out) as f:
            out = json.load(f)
    plan = {"C1": [(2000, 1e-6, "to 1e-6")], "C2": [(20000, 1e-6, "to 1e-6")],
            "C3": [(500, 1e-6, "to 1e-6"), (500, 0.0, "500 iterations")],
            "C4": [(200, 0.0, "200 iterations")], "C5": [(100, 0.0, "100 iterations")]}
    for name in args.configs.split(","):
        for n, tol, tag in plan[name]:
            rec = one(O, name, n, tol, tag)
            print(json.dumps(rec), flush=True)
            out = [r for r in out if not (r["config"] == name and r["run"] == tag)] + [rec]
            with open(args.out, "w") as f:
                json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
