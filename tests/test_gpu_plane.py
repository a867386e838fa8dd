"""GPU tests of the plane-chained pass (kernels_plane.cu, SURVEY.md §8(f)
NEXT-4): on grids with nx = ny = 1024 an iteration is the z pass plus one
persistent kernel running the y-inverse, x and y-forward passes plane by
plane.  Per element it computes what the 4-pass schedule computes (same line
FFTs, same update), so fields agree to fp32 rounding; the residual is summed
in another (fixed) order.  Also against the oracle (the closed form at 1024^3
runs through this pass in tests/test_gpu_parity.py).
"""
import numpy as np
import pytest

from gpu_helpers import TOL_COUNT, TOL_FIELD, rel_l2, rounded_inputs, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

SHAPE = (64, 1024, 1024)          # (nz, ny, nx): the plane-chained pass applies


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")


def _plan(p, **opts):
    from paper_2207_14222_b200 import Plan

    _, _, dtype = rounded_inputs(p)
    return Plan(p.shape, kind=p.kind, h=p.h, D=p.D, dtype=dtype, **opts)


def _launches(plan):
    return {k: v[1] for k, v in plan.profile_read().items()}


@pytest.mark.parametrize("form", ["xform_sparse", "xform_dense", "delta"])
def test_plane_equals_four_pass(form):
    from synth import make

    p = make("C5", SHAPE)
    med, src, dtype = rounded_inputs(p)
    if form == "xform_dense":
        rng = np.random.default_rng(3)
        src = src + (1e-3 * (rng.standard_normal(src.shape) + 1j * rng.standard_normal(src.shape))).astype(np.complex64)
    opts = {"delta_form": form == "delta"}
    pa = _plan(p, plane_chain=True, **opts)
    pa.profile(True)
    xa, na, _, _ = run_gpu(p, n_iter=12, tol=0.0, plan=pa, med=med, src=src, dtype=dtype)
    la = _launches(pa)
    # the setup runs the 4-pass chain once (its y-inverse and one y-forward
    # more); every iteration is K_C + the plane-chained kernel
    assert la.get("plane_dab", 0) >= 12 and "xpass" not in la and la.get("y_inv", 0) == 1
    pb = _plan(p, **opts)
    xb, nb, _, _ = run_gpu(p, n_iter=12, tol=0.0, plan=pb, med=med, src=src, dtype=dtype)
    assert na == nb == 12
    assert pa.source_lines() == (1 if form == "xform_sparse" else 0)
    assert rel_l2(xa, xb) <= 2e-6, rel_l2(xa, xb)
    assert np.allclose(pa.history(), pb.history(), rtol=1e-5, atol=0.0)


def test_plane_to_tolerance_matches_oracle(orc):
    """x-form, the switch to the Delta-form (r_switch raised so it happens
    early) and the stop test through the plane-chained pass: counts within
    +-1 of the oracle (x-form throughout), field <= 1e-4."""
    from synth import make

    p = make("C5", (64, 1024, 1024))
    pa = _plan(p, plane_chain=True, r_switch=0.3)
    xg, ng, term, _ = run_gpu(p, n_iter=400, tol=0.1, plan=pa)
    assert term == "converged" and not pa.iteration_form()[1]
    res, _ = run_oracle(orc, p, n_iter=400, tol=0.1)
    assert abs(ng - res.n_done) <= TOL_COUNT, (ng, res.n_done)
    if res.n_done != ng:
        res, _ = run_oracle(orc, p, n_iter=ng, tol=0.0)
    assert rel_l2(xg, res.x) <= TOL_FIELD
    h = pa.history()
    m = min(ng, res.n_done)
    assert np.allclose(h[:m], res.hist[:m], rtol=1e-3, atol=0.0)


def test_plane_resume_probe_and_stop():
    """Resumed calls, the residual probe after x-form iterations and the
    final x-only update give the 4-pass schedule's results."""
    from synth import make

    p = make("C5", SHAPE)
    med, src, dtype = rounded_inputs(p)
    res = []
    for chain in (True, False):
        pl = _plan(p, plane_chain=chain, r_switch=0.3)
        run_gpu(p, n_iter=3, tol=0.0, plan=pl, med=med, src=src, dtype=dtype)
        r3 = pl.residual()
        pl.iterate(5, p.alpha, 0.0)
        r8 = pl.residual()
        n, term = pl.iterate(500, p.alpha, 0.1)
        x = pl.get_field().cpu().numpy().astype(np.complex128)
        res.append((r3, r8, n, term, x, pl.history()))
    (a3, a8, an, at, ax, ah), (b3, b8, bn, bt, bx, bh) = res
    assert a3[2] == b3[2] == 3 and a8[2] == b8[2] == 8
    assert abs(a3[0] - b3[0]) <= 1e-5 * b3[0] and abs(a8[0] - b8[0]) <= 1e-5 * b8[0]
    assert at == bt == "converged" and an == bn
    assert rel_l2(ax, bx) <= 2e-6
    assert np.allclose(ah, bh, rtol=1e-5, atol=0.0)
