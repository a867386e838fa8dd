"""Helpers for the -m gpu parity tests: run the CUDA path (through the C-ABI
binding) and the CPU oracle on the *same* seeded inputs.

Both sides receive the complex64-rounded medium and source (the GPU path's
input precision), so the comparison isolates the arithmetic of the path.
"""
import numpy as np

TOL_FIELD = 1e-4      # north_star: relative L2 of the field after the same count
TOL_COUNT = 1         # north_star: iteration counts to 1e-6 within +-1


def rounded_inputs(p):
    if p.kind == "helmholtz":
        med = np.asarray(p.medium).astype(np.complex64)
        src = np.asarray(p.source).astype(np.complex64)
        return med, src, "c64"
    med = np.asarray(p.medium).real.astype(np.float32)
    src = np.asarray(p.source).real.astype(np.float32)
    return med, src, "r32"


def run_gpu(p, n_iter=None, tol=None, alpha=None, med=None, src=None, dtype=None, plan=None, profile=False):
    import torch
    from paper_2207_14222_b200 import Plan

    if med is None:
        med, src, dtype = rounded_inputs(p)
    if plan is None:
        plan = Plan(p.shape, kind=p.kind, h=p.h, D=p.D, dtype=dtype)
    plan.set_potential(torch.from_numpy(med).cuda(), 0.95)
    plan.set_source(torch.from_numpy(src).cuda())
    if profile:
        plan.profile(True)
    n, term = plan.iterate(p.n_iter if n_iter is None else n_iter, p.alpha if alpha is None else alpha,
                           p.tol if tol is None else tol)
    x = plan.get_field().cpu().numpy().astype(np.complex128)
    return x, n, term, plan


def run_oracle(orc, p, n_iter=None, tol=None, alpha=None):
    med, src, _ = rounded_inputs(p)
    med64 = med.astype(np.complex128)
    sp = orc.canonical(p.kind, med64, 0.95, D=p.D)
    w = orc.medium_to_w(p.kind, med64)
    res = orc.fixed_point(w, src.astype(np.complex128), p.h, sp.D, sp.sigma, sp.c,
                          p.alpha if alpha is None else alpha, p.tol if tol is None else tol,
                          p.n_iter if n_iter is None else n_iter)
    return res, sp


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def monotone(h, rel=1e-5):
    """Cor. 1: r_{k+1} <= r_k, up to fp32 rounding."""
    h = np.asarray(h)
    return bool(np.all(np.diff(h) <= rel * h[:-1]))
