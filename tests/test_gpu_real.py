"""GPU tests of the real path (kernels_real.cu): steady-state diffusion with
float32 data (BASELINE.json config C4, §3.2) runs on half spectra
(R2C / C2R x pass, 16-column strided passes over rows of nx/2 + 16), 52
instead of 104 B per voxel and iteration.

* vs the oracle (complex128) after the same count: relative L2 <= 1e-4;
* vs the complex path on the same input (desc.complex_path): same iterate to fp32
  rounding;
* closed form for constant mu_a (every Fourier mode decouples);
* the slab decomposition of the real path (virtual slabs) is bit-identical
  to one slab.
"""
import numpy as np
import pytest

from gpu_helpers import TOL_FIELD, rel_l2, rounded_inputs, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")


def _run(p, n, virtual_ranks=0, tol=0.0, **opts):
    import torch
    from paper_2207_14222_b200 import Plan

    med, src, dtype = rounded_inputs(p)
    assert dtype == "r32"
    plan = Plan(p.shape, kind=p.kind, h=p.h, D=p.D, dtype=dtype, virtual_ranks=virtual_ranks, **opts)
    plan.set_potential(torch.from_numpy(med).cuda(), 0.95)
    plan.set_source(torch.from_numpy(src).cuda())
    nd, term = plan.iterate(n, p.alpha, tol)
    return plan.get_field().cpu().numpy(), nd, term, plan


def _ws_bytes(plan):
    return plan.workspace.numel()


@pytest.mark.parametrize("shape,n", [((64, 64, 64), 150), ((128, 64, 256), 60), ((64, 256, 64), 40),
                                     ((256, 64, 32), 40), ((64, 64, 1024), 20), ((64, 64, 2048), 10)])
def test_real_path_matches_oracle(orc, shape, n):
    from synth import make

    p = make("C4", shape)
    x, nd, term, plan = _run(p, n)
    assert nd == n and term == "max_iter" and x.dtype == np.float32
    # the real path's workspace: 3 float32 fields (+ s for the x-form, R-30) + the half
    # spectrum (twice with the z pass's plane-pair buffer)
    nz, ny, nx = shape
    spectra = 2 if plan.work_layout() == "z-pair" else 1
    assert _ws_bytes(plan) < 4 * 4 * nz * ny * nx + spectra * 8 * nz * ny * (nx // 2 + 16) + 4096
    res, _ = run_oracle(orc, p, n_iter=n)
    assert np.abs(res.x.imag).max() <= 1e-12 * np.abs(res.x).max()
    err = rel_l2(x.astype(np.complex128), res.x)
    assert err <= TOL_FIELD, err
    assert np.allclose(plan.history()[:n], res.hist[:n], rtol=1e-3, atol=0.0)


def test_real_path_equals_complex_path():
    from synth import make

    p = make("C4", (64, 128, 64))
    # the same (Delta-form) arithmetic on both paths
    xr, _, _, pr = _run(p, 50, delta_form=True)
    xc, _, _, pc = _run(p, 50, delta_form=True, complex_path=True)
    assert _ws_bytes(pr) < 0.7 * _ws_bytes(pc)
    assert rel_l2(xr.astype(np.float64), xc.astype(np.float64)) <= 2e-6
    assert np.allclose(pr.history(), pc.history(), rtol=1e-5, atol=0.0)


def test_real_path_converges_like_oracle(orc):
    from synth import make

    p = make("C4", (64, 64, 64))
    x, nd, term, plan = _run(p, 2000, tol=1e-6)
    res, _ = run_oracle(orc, p, n_iter=2000, tol=1e-6)
    assert term == "converged" and abs(nd - res.n_done) <= 1, (nd, res.n_done)


@pytest.mark.parametrize("shape", [(64, 64, 64), (128, 64, 512)])
def test_real_path_closed_form(shape):
    """Constant mu_a = m0 with explicit (sigma, c): V = (m0 - sigma)/c is a
    real constant v0 and every Fourier mode evolves as x^_k = x^*(1 - q^k),
    q = 1 - alpha b (1 - b g), b = 1 - v0, x^* = g s^ / (1 - b g)."""
    import torch
    from paper_2207_14222_b200 import Plan

    D, m0, sigma, c, alpha = 1.0, 0.02, 0.05, 0.04, 0.75
    S = np.zeros(shape, dtype=np.float32)
    S[tuple(s // 2 for s in shape)] = 1.0
    S[tuple(s // 5 for s in shape)] = -0.5
    plan = Plan(shape, kind="diffusion", D=D, sigma=sigma, c=c, dtype="r32")
    plan.set_potential(torch.full(shape, m0, dtype=torch.float32, device="cuda"), -1.0)
    plan.set_source(torch.from_numpy(S).cuda())
    v0 = (float(np.float32(m0)) - sigma) / c
    b = 1.0 - v0
    p2 = sum(np.meshgrid(*[(2 * np.pi * np.fft.fftfreq(n)) ** 2 for n in shape], indexing="ij"))
    g = c / (D * p2 + sigma + c)
    q = 1.0 - alpha * b * (1.0 - b * g)
    xstar = g * np.fft.fftn(S.astype(np.float64) / c) / (1.0 - b * g)
    done = 0
    for k in (1, 8, 40):
        plan.iterate(k - done, alpha, 0.0)
        done = k
        x = plan.get_field().cpu().numpy().astype(np.float64)
        ref = np.fft.ifftn(xstar * (1.0 - q ** k)).real
        assert rel_l2(x, ref) <= 2e-5, (k, rel_l2(x, ref))


@pytest.mark.parametrize("shape,P", [((64, 64, 64), 2), ((128, 64, 128), 4)])
def test_real_path_virtual_slabs_bit_identical(shape, P):
    from synth import make

    p = make("C4", shape)
    x1, _, _, pl1 = _run(p, 30)
    xp, _, _, plp = _run(p, 30, virtual_ranks=P)
    assert np.array_equal(x1.view(np.uint8), xp.view(np.uint8))
    assert np.array_equal(pl1.history(), plp.history())
