"""Small cases of every kernel family for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck):

    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py all

CASE in: c3_xform (3-D x-form, sparse source, switch to the Delta-form, to
tol), c5_delta (Delta-form, ragged 3-D), c2_persistent (2-D persistent
cooperative solver, grid barrier), c1 (1-D on-chip solve), slabs_fused
(virtual slabs P = 2, transposes fused into the stores), slabs_separate,
real (half-spectrum path), z1024 (k_stile<1024> with the two-round FLIP
exchange and tensor-map stores), plane (the plane-chained pass), krylov
(BiCGSTAB + GMRES), anti, tdiff, staging (asynchronous staging and
read-back), or "all" (every case in one process: the pool allows one
compute-sanitizer run per gpurun call).  Prints "CASE ok" per case.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def inputs(name, shape):
    from synth import make

    p = make(name, shape)
    if p.kind == "helmholtz":
        return p, np.asarray(p.medium).astype(np.complex64), np.asarray(p.source).astype(np.complex64), "c64"
    return p, np.asarray(p.medium).real.astype(np.float32), np.asarray(p.source).real.astype(np.float32), "r32"


def solve(name, shape, n, tol=0.0, **opts):
    import torch
    from paper_2207_14222_b200 import Plan

    p, med, src, dtype = inputs(name, shape)
    plan = Plan(p.shape, kind=p.kind, h=p.h, D=p.D, dtype=dtype, **opts)
    plan.set_potential(torch.from_numpy(med).cuda(), 0.95)
    plan.set_source(torch.from_numpy(src).cuda())
    nd, term = plan.iterate(n, p.alpha, tol)
    plan.residual()
    x = plan.get_field()
    torch.cuda.synchronize()
    assert torch.isfinite(x).all()
    return plan, nd, term


def main(case):
    import torch

    torch.cuda.set_device(0)
    if case == "c3_xform":
        plan, nd, term = solve("C3", (32, 32, 32), 400, tol=1e-6)
        assert term == "converged" and plan.source_lines() == 1
    elif case == "c5_delta":
        solve("C5", (32, 64, 128), 6, delta_form=True)
    elif case == "c2_persistent":
        solve("C2", (64, 64), 40)
    elif case == "c1":
        solve("C1", None, 50)
    elif case == "slabs_fused":
        solve("C5", (64, 64, 32), 4, virtual_ranks=2)
    elif case == "slabs_separate":
        solve("C5", (64, 64, 32), 4, virtual_ranks=2, separate_transposes=True)
    elif case == "real":
        solve("C4", (64, 64, 64), 4)
    elif case == "z1024":
        solve("C5", (1024, 64, 16), 3)
    elif case == "plane":   # plane-chained pass (nx = ny = 1024), x-form then Delta-form
        solve("C5", (64, 1024, 1024), 3, r_switch=0.9, plane_chain=True)
        solve("C5", (64, 1024, 1024), 2, delta_form=True, plane_chain=True)
    elif case == "krylov":
        from paper_2207_14222_b200 import Plan

        p, med, src, dtype = inputs("C5", (32, 32, 64))
        plan = Plan(p.shape)
        plan.set_potential(torch.from_numpy(med).cuda(), 0.95)
        plan.set_source(torch.from_numpy(src).cuda())
        plan.bicgstab(3, 0.0)
        plan.set_source(torch.from_numpy(src).cuda())
        plan.gmres(4, 6, 0.0)
        torch.cuda.synchronize()
    elif case == "anti":
        solve("C5", (64, 64, 64), 3, antisymmetric=True)
    elif case == "tdiff":
        from paper_2207_14222_b200 import Plan

        shape = (64, 64)
        rng = np.random.default_rng(1)
        mu = (0.01 + 0.02 * rng.random(shape)).astype(np.float32)
        D = np.zeros(shape + (2, 2), dtype=np.float32)
        D[..., 0, 0], D[..., 1, 1], D[..., 0, 1], D[..., 1, 0] = 1.0, 1.5, 0.2, 0.2
        S = np.zeros(shape, dtype=np.float32)
        S[32, 32] = 1.0
        plan = Plan(shape, kind="diffusion", tensor_diffusion=True)
        plan.set_tensor_medium(torch.from_numpy(mu).cuda(), torch.from_numpy(D).cuda(), 0.95)
        plan.set_source(torch.from_numpy(S).cuda())
        plan.iterate(3, 0.75, 0.0)
        plan.get_field()
        torch.cuda.synchronize()
    elif case == "staging":
        from paper_2207_14222_b200 import Plan

        p, med, src, dtype = inputs("C5", (32, 32, 64))
        plan = Plan(p.shape)
        hm, hs = torch.from_numpy(med).pin_memory(), torch.from_numpy(src).pin_memory()
        out = torch.empty(p.shape, dtype=torch.complex64).pin_memory()
        plan.stage_inputs(hm, hs)
        for i in range(2):
            plan.set_potential("staged")
            plan.set_source("staged")
            if i == 0:
                plan.stage_inputs(hm, hs)
            plan.iterate(3, 0.75, 0.0)
            plan.get_field_async(out)
        plan.wait_field()
    else:
        raise SystemExit(f"unknown case {case}")
    print(f"{case} ok", flush=True)


ALL = ["c3_xform", "c5_delta", "c2_persistent", "c1", "slabs_fused", "slabs_separate", "real", "z1024", "plane",
       "krylov", "anti", "tdiff", "staging"]

if __name__ == "__main__":
    # one process for every case: the pool allows one compute-sanitizer run per gpurun call
    for c in (ALL if sys.argv[1] == "all" else sys.argv[1:]):
        main(c)
