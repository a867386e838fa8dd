"""x-form vs Delta-form of the GPU iteration (reading R-30).

Algorithm 1 literally (x-form: Delta_k = B[(L+1)^-1(B x_k + s)
- x_k], x_{k+1} = x_k + alpha Delta_k) and the Neumann recurrence of L613
(Delta-form) are the same iteration in exact arithmetic.  The GPU runs the
x-form (8 fewer HBM bytes per voxel) while r >= r_switch and the Delta-form
below it.  These tests pin the two against each other and the hybrid
against the oracle: same fields and counts, residual histories equal up to
the x-form's fp32 cancellation (relative error ~ eps |x| / |Delta_k|).
"""
import numpy as np
import pytest

from gpu_helpers import TOL_COUNT, TOL_FIELD, rel_l2, rounded_inputs, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def orc():
    from oracle import oracle as O

    O.build()
    return O


def _plan(p, monkeypatch, xform, **opts):
    from paper_2207_14222_b200 import Plan

    _, _, dtype = rounded_inputs(p)
    return Plan(p.shape, kind=p.kind, h=p.h, D=p.D, dtype=dtype, delta_form=not xform, **opts)


@pytest.mark.parametrize("shape,n", [((32, 32, 32), 40), ((64, 32, 128), 25)])
def test_xform_equals_delta_form_fixed_count(monkeypatch, shape, n):
    from synth import make

    p = make("C5", shape)
    px = _plan(p, monkeypatch, True)
    pd = _plan(p, monkeypatch, False)
    assert px.iteration_form()[0] and not pd.iteration_form()[0]
    xx, nx_, _, _ = run_gpu(p, n_iter=n, tol=0.0, plan=px)
    xd, nd_, _, _ = run_gpu(p, n_iter=n, tol=0.0, plan=pd)
    assert nx_ == nd_ == n
    assert rel_l2(xx, xd) <= 1e-5
    hx, hd = px.history(), pd.history()
    assert len(hx) == len(hd) == n + 1            # r_0 .. r_n in both forms
    assert np.allclose(hx, hd, rtol=1e-4, atol=0.0)
    rx, rd = px.residual(), pd.residual()
    assert rx[2] == rd[2] == n and abs(rx[0] - rd[0]) <= 1e-4 * rd[0]


def test_xform_switch_converges_like_delta_form_and_oracle(monkeypatch, orc):
    """C3 recipe to 1e-6: x-form, switch below r_switch, Delta-form to the end."""
    from synth import make

    p = make("C3", (32, 32, 32))
    px = _plan(p, monkeypatch, True)
    pd = _plan(p, monkeypatch, False)
    xx, nx_, tx, _ = run_gpu(p, n_iter=2000, tol=1e-6, plan=px)
    xd, nd_, td, _ = run_gpu(p, n_iter=2000, tol=1e-6, plan=pd)
    assert tx == td == "converged"
    assert abs(nx_ - nd_) <= TOL_COUNT
    assert not px.iteration_form()[1]             # switched to the Delta-form
    res, _ = run_oracle(orc, p, n_iter=2000, tol=1e-6)
    assert abs(nx_ - res.n_done) <= TOL_COUNT
    ref, _ = run_oracle(orc, p, n_iter=nx_, tol=0.0)
    assert rel_l2(xx, ref.x) <= TOL_FIELD
    h = px.history()[:nx_]
    assert np.all(h[1:] <= h[:-1] * (1 + 1e-3))   # monotone (Cor. 1), up to fp32 noise


def test_xform_form_reporting(monkeypatch):
    from synth import make

    p = make("C5", (32, 32, 32))
    px = _plan(p, monkeypatch, True)
    run_gpu(p, n_iter=3, tol=0.0, plan=px)
    xf, now, rsw = px.iteration_form()
    assert xf and now and rsw == 1e-2 and px.residual()[0] > rsw
    px.iterate(400, 0.75, 0.0)
    assert not px.iteration_form()[1] and px.residual()[0] < rsw


def test_xform_resume_and_stop_semantics(monkeypatch):
    """Split calls equal one call (the end-of-call probe leaves x and the
    x-form chain input unchanged); a resumed call with tol above the current
    residual applies exactly one update (reading R-5)."""
    from synth import make

    p = make("C5", (32, 32, 32))
    pa = _plan(p, monkeypatch, True)
    xa, _, _, _ = run_gpu(p, n_iter=9, tol=0.0, plan=pa)
    pb = _plan(p, monkeypatch, True)
    run_gpu(p, n_iter=4, tol=0.0, plan=pb)
    n, _ = pb.iterate(5, 0.75, 0.0)
    assert n == 5 and np.array_equal(pb.get_field().cpu().numpy().astype(np.complex128), xa)
    assert np.array_equal(pa.history(), pb.history())
    r9 = pa.residual()[0]
    n, term = pa.iterate(100, 0.75, r9 * 1.01)
    assert n == 1 and term == "converged"


def test_xform_sweep_bytes_lower(monkeypatch):
    """The x-form plan keeps s in one extra field of the workspace."""
    from synth import make

    p = make("C5", (32, 32, 32))
    px = _plan(p, monkeypatch, True)
    pd = _plan(p, monkeypatch, False)
    fx, fd = px.workspace.numel(), pd.workspace.numel()
    assert fx == fd + 8 * 32 * 32 * 32 or fx == fd + 256 * ((8 * 32 ** 3 + 255) // 256)


@pytest.mark.parametrize("shape,n", [((64, 64, 64), 30), ((32, 64, 128), 20)])
def test_xform_real_path_equals_delta_form(monkeypatch, shape, n):
    """The real (half-spectrum) path's x-form against its Delta-form."""
    from synth import make

    p = make("C4", shape)
    px = _plan(p, monkeypatch, True)
    pd = _plan(p, monkeypatch, False)
    assert px.iteration_form()[0] and not pd.iteration_form()[0]
    xx, _, _, _ = run_gpu(p, n_iter=n, tol=0.0, plan=px)
    xd, _, _, _ = run_gpu(p, n_iter=n, tol=0.0, plan=pd)
    assert rel_l2(xx, xd) <= 1e-5
    assert np.allclose(px.history(), pd.history(), rtol=1e-3, atol=0.0)
    xt, nt, tt, _ = run_gpu(p, n_iter=2000, tol=1e-6, plan=px)
    xu, nu, tu, _ = run_gpu(p, n_iter=2000, tol=1e-6, plan=pd)
    assert tt == tu == "converged" and abs(nt - nu) <= TOL_COUNT and rel_l2(xt, xu) <= 1e-4


def test_sparse_source_xform(monkeypatch):
    """Reading R-31: a point source lives on one x-line; the x-form passes then
    never read s (its x-transform is added after each x pass).  Same iterate
    as the dense-s x-form and the Delta-form; a dense source keeps dense s."""
    from synth import make

    p = make("C5", (32, 32, 64))
    pa = _plan(p, monkeypatch, True)
    xa, na, _, _ = run_gpu(p, n_iter=30, tol=0.0, plan=pa)
    assert pa.source_lines() == 1
    pb = _plan(p, monkeypatch, True, dense_source=True)
    xb, nb, _, _ = run_gpu(p, n_iter=30, tol=0.0, plan=pb)
    assert pb.source_lines() == 0
    pd = _plan(p, monkeypatch, False)
    xd, _, _, _ = run_gpu(p, n_iter=30, tol=0.0, plan=pd)
    assert rel_l2(xa, xb) <= 1e-6 and rel_l2(xa, xd) <= 1e-5
    assert np.allclose(pa.history(), pd.history(), rtol=1e-4, atol=0.0)
    # to tolerance (x-form with the added source lines, switch, Delta-form)
    xt, nt, tt, _ = run_gpu(p, n_iter=3000, tol=1e-6, plan=pa)
    xu, nu, tu, _ = run_gpu(p, n_iter=3000, tol=1e-6, plan=pd)
    assert tt == tu == "converged" and abs(nt - nu) <= TOL_COUNT and rel_l2(xt, xu) <= 1e-4
    # a source on many lines stays dense
    rng = np.random.default_rng(5)
    med, src, _ = rounded_inputs(p)
    src = (rng.standard_normal(src.shape) + 1j * rng.standard_normal(src.shape)).astype(np.complex64)
    pc = _plan(p, monkeypatch, True)
    run_gpu(p, n_iter=3, tol=0.0, plan=pc, med=med, src=src, dtype="c64")
    assert pc.source_lines() == 0
