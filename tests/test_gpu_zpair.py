"""GPU tests of the z-pair layout of the FFT chain buffer (usp_internal.h
WLayout): planes 2zp and 2zp+1 interleaved in 128-byte x
blocks so the z pass moves 256-byte rows.  Only addresses change -- every
line FFT, the multiplier (Eq. 12) and the update of Alg. 1
(L80-89) are the same -- so fields must be BIT-identical to the plain [z][y][x] layout (the default)
in every form of the x pass and through the Krylov solvers; the residual
partials are summed in another fixed order (the x pass deals its lines to
the CTAs by plane pairs), so histories agree to fp64 rounding; and the
default (z-pair) path must match the oracle.
"""
import numpy as np
import pytest

from gpu_helpers import TOL_FIELD, rel_l2, rounded_inputs, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")


def _plan(p, dtype, **opts):
    from paper_2207_14222_b200 import Plan

    return Plan(p.shape, kind=p.kind, h=p.h, D=p.D, dtype=dtype, **opts)


def _dense(src):
    rng = np.random.default_rng(11)
    return src + (1e-3 * (rng.standard_normal(src.shape) + 1j * rng.standard_normal(src.shape))).astype(np.complex64)


# (nz, ny, nx): every x extent the layout takes (U = 2 / 1 lines per x unit,
# N1 = 16 / 32 lanes per line), y / z tiles of 64 .. 1024 rows, the HALFX
# two-round exchange (nz >= 512) and the full one (nz <= 256)
SHAPES = [(64, 64, 256), (128, 64, 512), (64, 128, 1024), (512, 64, 256), (1024, 64, 256), (64, 64, 2048),
          (256, 256, 256)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("form", ["xform_sparse", "xform_dense", "delta"])
def test_zpair_bit_identical_to_flat(shape, form):
    from synth import make

    p = make("C3", shape)
    med, src, dtype = rounded_inputs(p)
    if form == "xform_dense":
        src = _dense(src)
    opts = {"delta_form": form == "delta", "r_switch": 0.3}
    out = {}
    for flat in (False, True):
        pl = _plan(p, dtype, zpair_work=not flat, **opts)
        assert pl.work_layout() == ("flat" if flat else "z-pair")
        x, n, term, _ = run_gpu(p, n_iter=14, tol=0.0, plan=pl, med=med, src=src, dtype=dtype)
        assert n == 14
        out[flat] = (x, pl.history(), pl.source_lines(), pl.iteration_form()[1])
    (xa, ha, sa, fa), (xb, hb, sb, fb) = out[False], out[True]
    assert sa == sb == (1 if form == "xform_sparse" else 0)
    assert fa == fb
    assert np.array_equal(xa, xb), rel_l2(xa, xb)
    assert np.allclose(ha, hb, rtol=1e-12, atol=0.0)


def test_zpair_stop_resume_identical():
    """Resumed calls, the x-form residual probe, the converged stop and its
    final x-only update: identical on both layouts."""
    from synth import make

    p = make("C3", (128, 64, 512))
    med, src, dtype = rounded_inputs(p)
    res = []
    for flat in (False, True):
        pl = _plan(p, dtype, zpair_work=not flat, r_switch=0.3)
        run_gpu(p, n_iter=3, tol=0.0, plan=pl, med=med, src=src, dtype=dtype)
        r3 = pl.residual()
        pl.iterate(5, p.alpha, 0.0)
        r8 = pl.residual()
        n, term = pl.iterate(500, p.alpha, 1e-3)
        x = pl.get_field().cpu().numpy()
        res.append((r3, r8, n, term, x, pl.history()))
    (a3, a8, an, at, ax, ah), (b3, b8, bn, bt, bx, bh) = res
    assert a3[2] == b3[2] == 3 and a8[2] == b8[2] == 8 and an == bn and at == bt == "converged"
    assert abs(a3[0] - b3[0]) <= 1e-12 * b3[0] and abs(a8[0] - b8[0]) <= 1e-12 * b8[0]
    assert np.array_equal(ax, bx) and np.allclose(ah, bh, rtol=1e-12, atol=0.0)


@pytest.mark.parametrize("solver", ["bicgstab", "gmres"])
def test_zpair_krylov_identical(solver):
    """BiCGSTAB / GMRES(8) use the chain through their own x passes (k_xop):
    identical pass counts, fields and residuals on both layouts."""
    import torch

    from synth import make

    p = make("C3", (64, 64, 256))
    med, src, dtype = rounded_inputs(p)
    res = []
    for flat in (False, True):
        pl = _plan(p, dtype, zpair_work=not flat)
        pl.set_potential(torch.from_numpy(med).cuda(), 0.95)
        pl.set_source(torch.from_numpy(src).cuda())
        n, term = pl.bicgstab(12, 0.0) if solver == "bicgstab" else pl.gmres(8, 20, 0.0)
        res.append((n, term, pl.get_field().cpu().numpy(), pl.residual()[0]))
    (an, at, ax, ar), (bn, bt, bx, br) = res
    assert an == bn and at == bt and abs(ar - br) <= 1e-12 * br
    assert np.array_equal(ax, bx)


def test_zpair_matches_oracle(orc):
    """The z-pair path against the oracle: x-form with the sparse source,
    switch to the Delta-form, field <= 1e-4 after the same count."""
    from synth import make

    p = make("C3", (64, 64, 256))
    pl = _plan(p, rounded_inputs(p)[2], r_switch=0.3, zpair_work=True)
    assert pl.work_layout() == "z-pair"
    xg, ng, _, _ = run_gpu(p, n_iter=40, tol=0.0, plan=pl)
    res, _ = run_oracle(orc, p, n_iter=40, tol=0.0)
    assert ng == res.n_done == 40
    assert rel_l2(xg, res.x) <= TOL_FIELD, rel_l2(xg, res.x)
    assert np.allclose(pl.history()[:40], res.hist[:40], rtol=1e-3, atol=0.0)


def test_zpair_where_it_applies():
    """z-pair only on request (desc.zpair_work) and where every pass that
    touches the chain buffer supports it."""
    from paper_2207_14222_b200 import Plan

    z = {"zpair_work": True}
    assert Plan((64, 64, 256), **z).work_layout() == "z-pair"
    assert Plan((64, 64, 256)).work_layout() == "flat"            # the default
    assert Plan((64, 64, 128), **z).work_layout() == "flat"       # x lines < 256 points
    assert Plan((32, 64, 256), **z).work_layout() == "flat"       # z lines of 32: register-staged pass
    assert Plan((2048, 64, 256), **z).work_layout() == "flat"     # z tiles of 8 columns
    assert Plan((64, 256), **z).work_layout() == "flat"           # 2-D
    assert Plan((64, 64, 256), virtual_ranks=2, **z).work_layout() == "flat"
    assert Plan((64, 64, 256), kind="diffusion", dtype="r32", **z).work_layout() == "flat"   # real path
    assert Plan((64, 64, 256), antisymmetric=True, **z).work_layout() == "flat"
