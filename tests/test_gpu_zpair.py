"""GPU tests of the z-pair chain buffer (usp_internal.h): the
y-forward pass writes a second buffer in which planes 2zp and 2zp+1 are
interleaved in 128-byte x blocks, the z pass moves 256-byte rows on it and
the y-inverse pass reads it back.  Only addresses change -- every line FFT,
the multiplier (Eq. 12) and the update of Alg. 1
(L80-89) are the same -- so fields and residual histories must be
BIT-identical to the in-place z pass (desc.flat_work) in every form of the
x pass and through the Krylov solvers, and the default path must match the
oracle.
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


# (nz, ny, nx): x extents 32 .. 2048, y / z tiles of 64 .. 1024 rows, the
# HALFX two-round exchange (nz >= 512) and the full one (nz <= 256)
SHAPES = [(64, 64, 256), (128, 64, 512), (64, 128, 1024), (512, 64, 256), (1024, 64, 256), (64, 64, 2048),
          (256, 256, 256), (64, 64, 32), (128, 1024, 64)]


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
        pl = _plan(p, dtype, flat_work=flat, **opts)
        assert pl.work_layout() == ("flat" if flat else "z-pair")
        x, n, term, _ = run_gpu(p, n_iter=14, tol=0.0, plan=pl, med=med, src=src, dtype=dtype)
        assert n == 14
        out[flat] = (x, pl.history(), pl.source_lines(), pl.iteration_form()[1])
    (xa, ha, sa, fa), (xb, hb, sb, fb) = out[False], out[True]
    assert sa == sb == (1 if form == "xform_sparse" else 0)
    assert fa == fb
    assert np.array_equal(xa, xb), rel_l2(xa, xb)
    assert np.array_equal(ha, hb)


def test_zpair_stop_resume_identical():
    """Resumed calls, the x-form residual probe, the converged stop and its
    final x-only update: identical on both layouts."""
    from synth import make

    p = make("C3", (128, 64, 512))
    med, src, dtype = rounded_inputs(p)
    res = []
    for flat in (False, True):
        pl = _plan(p, dtype, flat_work=flat, r_switch=0.3)
        run_gpu(p, n_iter=3, tol=0.0, plan=pl, med=med, src=src, dtype=dtype)
        r3 = pl.residual()
        pl.iterate(5, p.alpha, 0.0)
        r8 = pl.residual()
        n, term = pl.iterate(500, p.alpha, 1e-3)
        x = pl.get_field().cpu().numpy()
        res.append((r3, r8, n, term, x, pl.history()))
    (a3, a8, an, at, ax, ah), (b3, b8, bn, bt, bx, bh) = res
    assert a3[2] == b3[2] == 3 and a8[2] == b8[2] == 8 and an == bn and at == bt == "converged"
    assert a3 == b3 and a8 == b8
    assert np.array_equal(ax, bx) and np.array_equal(ah, bh)


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
        pl = _plan(p, dtype, flat_work=flat)
        pl.set_potential(torch.from_numpy(med).cuda(), 0.95)
        pl.set_source(torch.from_numpy(src).cuda())
        n, term = pl.bicgstab(12, 0.0) if solver == "bicgstab" else pl.gmres(8, 20, 0.0)
        res.append((n, term, pl.get_field().cpu().numpy(), pl.residual()[0]))
    (an, at, ax, ar), (bn, bt, bx, br) = res
    assert an == bn and at == bt and ar == br
    assert np.array_equal(ax, bx)


def test_zpair_matches_oracle(orc):
    """The default (z-pair) path against the oracle: x-form with the sparse
    source, switch to the Delta-form, field <= 1e-4 after the same count."""
    from synth import make

    p = make("C3", (64, 64, 256))
    pl = _plan(p, rounded_inputs(p)[2], r_switch=0.3)
    assert pl.work_layout() == "z-pair"
    xg, ng, _, _ = run_gpu(p, n_iter=40, tol=0.0, plan=pl)
    res, _ = run_oracle(orc, p, n_iter=40, tol=0.0)
    assert ng == res.n_done == 40
    assert rel_l2(xg, res.x) <= TOL_FIELD, rel_l2(xg, res.x)
    assert np.allclose(pl.history()[:40], res.hist[:40], rtol=1e-3, atol=0.0)


def test_zpair_where_it_applies():
    """The z-pair buffer by default where the passes around the z pass support
    it; desc.flat_work keeps the z pass in place."""
    from paper_2207_14222_b200 import Plan

    assert Plan((64, 64, 256)).work_layout() == "z-pair"
    assert Plan((64, 64, 256), flat_work=True).work_layout() == "flat"
    assert Plan((64, 64, 16)).work_layout() == "z-pair"           # any x extent
    assert Plan((64, 64, 256), kind="diffusion", dtype="r32").work_layout() == "z-pair"   # real path
    assert Plan((32, 64, 256)).work_layout() == "flat"            # z lines of 32: register-staged pass
    assert Plan((2048, 64, 256)).work_layout() == "flat"          # z tiles of 8 columns
    assert Plan((64, 2048, 256)).work_layout() == "flat"          # y tiles of 8 columns
    assert Plan((64, 256)).work_layout() == "flat"                # 2-D
    assert Plan((64, 64, 256), virtual_ranks=2).work_layout() == "flat"
    assert Plan((64, 64, 256), antisymmetric=True).work_layout() == "flat"


@pytest.mark.parametrize("shape", [(64, 64, 128), (128, 64, 512), (512, 64, 64)])
def test_zpair_real_path_identical(shape):
    """The half-spectrum real path (rows of nx/2 + 16 columns) on the z-pair
    buffer: bit-identical to the in-place z pass (C4 recipe)."""
    from synth import make

    p = make("C4", shape)
    med, src, dtype = rounded_inputs(p)
    assert dtype == "r32"
    out = []
    for flat in (False, True):
        pl = _plan(p, dtype, flat_work=flat, r_switch=0.3)
        assert pl.work_layout() == ("flat" if flat else "z-pair")
        x, n, _, _ = run_gpu(p, n_iter=12, tol=0.0, plan=pl, med=med, src=src, dtype=dtype)
        out.append((x, pl.history()))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
