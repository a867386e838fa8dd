"""GPU parity at the BASELINE.json sizes: the CUDA path (C-ABI, the bench's
launch configuration) against the CPU oracle on the same seeded inputs,
element by element, at the full grid of C3, C4 and C5.

Bars (BASELINE.json north_star): relative L2 of the field <= 1e-4 after the
same iteration count; iteration counts to 1e-6 identical within +-1.
Algorithm 1 is PAPER.md L80-89; the oracle runs it literally in complex128.

The file is named so it runs last: these tests take minutes (the oracle on
the host cores: ~7e7 voxel-iterations/s at 256^3 on 16 cores, C5's four
1024^3 FFT round trips ~2-3 min) and C5 needs ~130 GiB of host RAM, which is
checked first -- the test fails loudly if the host is short, it never skips.
The full-length runs (C3 500, C4 200, C5 100 iterations) are in
tests/parity_fullsize.py, results in profiles/parity_fullsize_r02.json.
"""
import gc
import math
import os

import numpy as np
import pytest

from gpu_helpers import TOL_COUNT, TOL_FIELD, monotone, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")


def _host_free_gib():
    with open("/proc/meminfo") as f:
        for line in f:
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) / 2**20
    return 0.0


def _inputs_on_device(name, shape=None):
    """Seeded synthetic inputs generated on the GPU (synth's torch back end:
    the same counter-based numbers as the numpy one), rounded to the GPU
    path's input precision; the oracle gets exactly these values."""
    import torch
    from synth import make

    p = make(name, shape, device="cuda")
    if p.kind == "helmholtz":
        med, src, dtype = p.medium.to(torch.complex64), p.source.to(torch.complex64), "c64"
    else:
        med, src, dtype = p.medium.to(torch.float32), p.source.to(torch.float32), "r32"
    p.medium = p.source = None
    torch.cuda.empty_cache()
    return p, med, src, dtype


def _gpu(p, med, src, dtype, n, tol):
    from paper_2207_14222_b200 import Plan

    plan = Plan(p.shape, kind=p.kind, h=p.h, D=p.D, dtype=dtype)
    plan.set_potential(med, 0.95)
    plan.set_source(src)
    nd, term = plan.iterate(n, p.alpha, tol)
    x = plan.get_field().cpu().numpy()
    h = plan.history()
    xform = plan.iteration_form()[0]
    plan.close()
    return x, nd, term, h, xform


def _oracle(orc, p, med_np, src_np, n, tol):
    med = med_np.astype(np.complex128)
    sp = orc.canonical(p.kind, med, 0.95, D=p.D)
    w = orc.medium_to_w(p.kind, med)
    del med
    res = orc.fixed_point(w, src_np.astype(np.complex128), p.h, sp.D, sp.sigma, sp.c, p.alpha, tol, n)
    return res


def test_fullsize_C3_to_tolerance(orc):
    """C3 (256^3) to 1e-6: counts within +-1, field <= 1e-4 at the GPU's count,
    residual histories agree, monotone (Cor. 1)."""
    p, med, src, dtype = _inputs_on_device("C3")
    tol = 1e-6
    xg, ng, term, h, xform = _gpu(p, med, src, dtype, 500, tol)
    assert term == "converged" and xform
    med_np, src_np = med.cpu().numpy(), src.cpu().numpy()
    res = _oracle(orc, p, med_np, src_np, 500, tol)
    assert res.hist[-1] < tol
    assert abs(ng - res.n_done) <= TOL_COUNT, (ng, res.n_done)
    if res.n_done != ng:
        res = _oracle(orc, p, med_np, src_np, ng, 0.0)
    assert rel_l2(xg.astype(np.complex128), res.x) <= TOL_FIELD
    m = min(ng, res.n_done)
    assert np.allclose(h[:m], res.hist[:m], rtol=1e-3, atol=0.0)
    assert h.size == ng and monotone(h)   # r_0 .. r_{ng-1} (R-5)


def test_fullsize_C4_real_path(orc):
    """C4 (512^3 float32 diffusion, the real half-spectrum path with its
    k_stile<512> y/z passes on 272-column rows) for 25 iterations: the x-form
    passes, the switch to the Delta-form (r < 1e-2 near iteration 22) and
    Delta-form passes after it, against the oracle."""
    p, med, src, dtype = _inputs_on_device("C4")
    n = 25
    xg, ng, term, h, xform = _gpu(p, med, src, dtype, n, 0.0)
    assert ng == n and xform
    assert h[n - 1] < 1e-2 < h[0], "the run must cross r_switch"
    res = _oracle(orc, p, med.cpu().numpy(), src.cpu().numpy(), n, 0.0)
    assert np.abs(res.x.imag).max() <= 1e-12 * np.abs(res.x.real).max()
    assert rel_l2(xg.astype(np.float64), res.x.real) <= TOL_FIELD
    assert np.allclose(h[:n], res.hist[:n], rtol=1e-3, atol=0.0)


def test_fullsize_C4_closed_form_constant_mu():
    """512^3 real path with constant mu_a and a source of real grid plane
    waves (cosines): every voxel of x_k has a closed form (per Fourier mode
    x^_k = x^*(1 - q^k), tests/test_oracle_iteration derives it)."""
    import torch
    from paper_2207_14222_b200 import Plan

    n, K, alpha = 512, 5, 0.75
    shape = (n, n, n)
    mu, sigma, c = 0.05, 0.03, 0.04                     # V = (mu - sigma)/c = 0.5
    rng = np.random.default_rng(7)
    modes = [tuple(int(m) for m in rng.integers(-n // 2, n // 2, 3)) for _ in range(4)] + [(0, 0, 0), (n // 2, 3, -7)]
    amps = rng.standard_normal(len(modes))
    ar = torch.arange(n, device="cuda", dtype=torch.float64)

    def field(coefs):
        out = torch.zeros(shape, dtype=torch.float64, device="cuda")
        for (mz, my, mx), a in zip(modes, coefs):
            ph = 2 * math.pi * (mz * ar[:, None, None] + my * ar[None, :, None] + mx * ar[None, None, :]) / n
            out += float(a) * torch.cos(ph)
        return out

    S = field(amps).to(torch.float32)
    plan = Plan(shape, kind="diffusion", dtype="r32", sigma=sigma, c=c)
    plan.set_potential(torch.full(shape, mu, dtype=torch.float32, device="cuda"), -1.0)
    plan.set_source(S)
    del S
    nd, _ = plan.iterate(K, alpha, 0.0)
    assert nd == K
    x = plan.get_field().to(torch.float64)
    plan.close()
    b = 1.0 - (float(np.float32(mu)) - sigma) / c
    coefs = []
    for (mz, my, mx), a in zip(modes, amps):
        p2 = sum((2 * math.pi * ((m + n // 2) % n - n // 2) / n) ** 2 for m in (mz, my, mx))
        g = c / (p2 + sigma + c)
        q = 1.0 - alpha * b * (1.0 - b * g)
        coefs.append(a / c * g / (1.0 - b * g) * (1.0 - q ** K))
    ref = field(coefs)
    err = float(torch.linalg.vector_norm(x - ref) / torch.linalg.vector_norm(ref))
    assert err <= 2e-5, err


def test_fullsize_C5_against_oracle(orc):
    """C5 at its full size (1024^3 complex64, the heterogeneous GRF medium,
    the point source: the bench's workload and launch configuration -- x-form
    with the sparse-source x pass, R-30/R-31) for 3 iterations against the
    oracle, element by element over all 2^30 voxels."""
    import torch

    need = 140.0
    have = _host_free_gib()
    assert have >= need, f"C5 oracle parity needs ~{need:.0f} GiB of host RAM, {have:.0f} GiB available"
    p, med, src, dtype = _inputs_on_device("C5")
    n = 3
    xg, ng, term, h, xform = _gpu(p, med, src, dtype, n, 0.0)
    assert ng == n and xform
    med_np = med.cpu().numpy()
    src_np = src.cpu().numpy()
    del med, src
    torch.cuda.empty_cache()
    nz = np.flatnonzero(src_np)
    assert nz.size == 1                                   # the point source (R-16)
    sp = orc.canonical(p.kind, med_np, 0.95, D=p.D)       # smallest circle of the 2^30 values
    gc.collect()
    w = np.empty(med_np.shape, dtype=np.complex128)
    np.negative(med_np, out=w)                            # w = -k^2 (R-1), exactly the c64 values
    del med_np
    S = np.zeros(src_np.shape, dtype=np.complex128)
    S.flat[nz] = src_np.flat[nz]
    del src_np
    gc.collect()
    res = orc.fixed_point(w, S, p.h, sp.D, sp.sigma, sp.c, p.alpha, 0.0, n)
    del w, S
    gc.collect()
    num = 0.0
    den = 0.0
    xr = res.x
    for z0 in range(0, xr.shape[0], 64):                 # chunked: no 16 GiB temporaries
        d = xg[z0:z0 + 64].astype(np.complex128) - xr[z0:z0 + 64]
        num += float(np.vdot(d, d).real)
        den += float(np.vdot(xr[z0:z0 + 64], xr[z0:z0 + 64]).real)
    err = math.sqrt(num / den)
    assert err <= TOL_FIELD, err
    assert np.allclose(h[:n], res.hist[:n], rtol=1e-3, atol=0.0)
