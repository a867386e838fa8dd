"""Pins of the oracle's BiCGSTAB (oracle/usp_oracle.c orc_bicgstab) -- the
preconditioned system of Eq. 5 solved with BiCGSTAB, the
"BiCGSTAB" column of Table 1b (L305-311).

Pinned against things other than itself:
* scipy.sparse.linalg.bicgstab (an independent implementation of the same
  van der Vorst recurrence) on the DENSE preconditioned operator
  M = B[1 - (L+1)^-1 B] built from tests/dense_ref.py (no FFT): same iterate
  after 1, 4 and 15 passes;
* converged iterate = dense LU solution of A x = s;
* the reported residual = ||b - M x|| / ||b|| recomputed densely;
* a single Fourier mode with constant V is an eigenvector of M, so BiCGSTAB
  stops after the first half step (s = 0) at the closed-form x = g s / (1 - b g).
"""
import math

import numpy as np
import pytest

from dense_ref import dense_A, dense_L1


def _problem(shape, seed):
    rng = np.random.default_rng(seed)
    k0 = 2 * math.pi / 6
    nr = 1.0 + 0.5 * rng.random(shape)
    ni = 0.3 * rng.random(shape)
    k2 = (k0 * (nr + 1j * ni)) ** 2
    S = np.zeros(shape, dtype=complex)
    S[tuple(s // 2 for s in shape)] = 1.0
    S += 0.1 * (rng.standard_normal(shape) + 1j * rng.standard_normal(shape))
    return k2, S


def _dense_M_b(orc, shape, k2, S):
    sp = orc.canonical("helmholtz", k2)
    w = orc.medium_to_w("helmholtz", k2)
    V = ((w - sp.sigma) / sp.c).ravel()
    Bd = np.diag(1.0 - V)
    G = np.linalg.inv(dense_L1(shape, sp.sigma, sp.D, sp.c))
    M = Bd @ (np.eye(len(V)) - G @ Bd)
    b = Bd @ G @ (S.ravel() / sp.c)
    return sp, w, M, b


@pytest.mark.parametrize("shape,seed", [((64,), 1), ((16, 16), 2), ((8, 8, 8), 3)])
def test_iterates_equal_scipy_bicgstab(orc, shape, seed):
    from scipy.sparse.linalg import LinearOperator, bicgstab

    k2, S = _problem(shape, seed)
    sp, w, M, b = _dense_M_b(orc, shape, k2, S)
    n = M.shape[0]
    op = LinearOperator((n, n), matvec=lambda u: M @ u, dtype=complex)
    for k in (1, 4, 15):
        ref, _ = bicgstab(op, b, rtol=0.0, atol=0.0, maxiter=k)
        res = orc.bicgstab(w, S, [1.0] * len(shape), sp.D, sp.sigma, sp.c, 0.0, k)
        assert res.n_done == k and not res.half and res.rc == 0
        assert np.linalg.norm(res.x.ravel() - ref) <= 1e-10 * np.linalg.norm(ref), k


@pytest.mark.parametrize("shape,seed", [((32,), 4), ((64,), 5), ((16, 16), 6), ((8, 8, 8), 7)])
def test_converged_equals_dense_LU_and_residual(orc, shape, seed):
    k2, S = _problem(shape, seed)
    sp, w, M, b = _dense_M_b(orc, shape, k2, S)
    res = orc.bicgstab(w, S, [1.0] * len(shape), sp.D, sp.sigma, sp.c, 1e-12, 5000)
    assert res.rc == 0 and res.hist[-1] < 1e-12
    A = dense_A(shape, w, sp.D, sp.c)
    xref = np.linalg.solve(A, (S / sp.c).ravel())
    assert np.linalg.norm(res.x.ravel() - xref) <= 1e-9 * np.linalg.norm(xref)
    # the reported (recursive) residual is the true preconditioned residual of
    # the returned x, to rounding (checked where rounding is far below it)
    res6 = orc.bicgstab(w, S, [1.0] * len(shape), sp.D, sp.sigma, sp.c, 1e-6, 5000)
    true_r = np.linalg.norm(b - M @ res6.x.ravel()) / np.linalg.norm(b)
    assert res6.hist[-1] < 1e-6 and abs(true_r - res6.hist[-1]) <= 1e-4 * res6.hist[-1]
    assert abs(res.nb - np.linalg.norm(b)) <= 1e-12 * np.linalg.norm(b)


@pytest.mark.parametrize("shape", [(64,), (16, 32), (8, 16, 8)])
def test_single_mode_stops_after_half_step(orc, shape):
    """Constant V and a single-Fourier-mode source: M p = lambda p, so s = 0
    after the first half step and x = g s^/(1 - b g) (mode by mode)."""
    k0, nn = 2 * math.pi / 8, 1.0 + 0.05j
    k2 = (k0 * nn) ** 2
    sigma, c, D = -k2.real, -1j * abs(k2.imag) / 0.95, 1.0
    grids = np.meshgrid(*[np.arange(s) for s in shape], indexing="ij")
    m = [1 + a for a in range(len(shape))]
    phase = sum(2 * np.pi * mi * gi / s for mi, gi, s in zip(m, grids, shape))
    S = np.exp(1j * phase)
    w = -k2 * np.ones(shape)
    res = orc.bicgstab(w, S, [1.0] * len(shape), D, sigma, c, 1e-10, 10)
    assert res.rc == 0 and res.n_done == 1 and res.half
    b = 1.0 - (-k2 - sigma) / c
    p2 = sum((2 * np.pi * mi / s) ** 2 for mi, s in zip(m, shape))
    g = c / (D * p2 + sigma + c)
    xstar = g * (S / c) / (1.0 - b * g)
    assert np.linalg.norm(res.x - xstar) <= 1e-12 * np.linalg.norm(xstar)


def test_fewer_operator_applications_than_fixed_point_on_C1(orc):
    """Table 1b (L307) reports BiCGSTAB among the fastest preconditioned
    methods; on the C1 stand-in it needs fewer applications of (L+1)^-1 than
    the fixed-point iteration at alpha = 0.75 (reading, qualitative: the
    paper's grid is unstated)."""
    from synth import make

    p = make("C1")
    med = np.asarray(p.medium)
    sp = orc.canonical(p.kind, med)
    w = orc.medium_to_w(p.kind, med)
    kr = orc.bicgstab(w, p.source, p.h, sp.D, sp.sigma, sp.c, 1e-6, 2000)
    fp = orc.fixed_point(w, p.source, p.h, sp.D, sp.sigma, sp.c, 0.75, 1e-6, 2000)
    assert kr.rc == 0 and kr.hist[-1] < 1e-6
    assert 2 * kr.n_done < fp.n_done
    assert np.linalg.norm(kr.x - fp.x) <= 1e-4 * np.linalg.norm(fp.x)


# ------------------------------------------------------------- GMRES(m) --
@pytest.mark.parametrize("shape,seed,m", [((64,), 1, 5), ((16, 16), 2, 20), ((8, 8, 8), 3, 5)])
def test_gmres_cycles_equal_scipy_gmres(orc, shape, seed, m):
    """After k full restart cycles, orc_gmres = scipy's GMRES(m) (an
    independent implementation; the iterate of a cycle is unique: it
    minimises the residual over the Krylov space) on the dense operator."""
    from scipy.sparse.linalg import LinearOperator, gmres

    k2, S = _problem(shape, seed)
    sp, w, M, b = _dense_M_b(orc, shape, k2, S)
    n = M.shape[0]
    op = LinearOperator((n, n), matvec=lambda u: M @ u, dtype=complex)
    for cycles in (1, 3):
        ref, _ = gmres(op, b, rtol=0.0, atol=0.0, restart=m, maxiter=cycles)
        res = orc.gmres(w, S, [1.0] * len(shape), sp.D, sp.sigma, sp.c, m, 0.0, cycles * m)
        assert res.n_done == cycles * m and res.rc == 0
        assert np.linalg.norm(res.x.ravel() - ref) <= 1e-9 * np.linalg.norm(ref), cycles
        true_r = np.linalg.norm(b - M @ res.x.ravel()) / np.linalg.norm(b)
        assert abs(true_r - res.hist[-1]) <= 1e-6 * true_r + 1e-13   # estimate = true residual


@pytest.mark.parametrize("shape,seed,m", [((32,), 4, 5), ((16, 16), 6, 20), ((8, 8, 8), 7, 10)])
def test_gmres_converged_equals_dense_LU(orc, shape, seed, m):
    k2, S = _problem(shape, seed)
    sp, w, M, b = _dense_M_b(orc, shape, k2, S)
    res = orc.gmres(w, S, [1.0] * len(shape), sp.D, sp.sigma, sp.c, m, 1e-11, 20000)
    assert res.rc == 0 and res.hist[-1] < 1e-11
    A = dense_A(shape, w, sp.D, sp.c)
    xref = np.linalg.solve(A, (S / sp.c).ravel())
    assert np.linalg.norm(res.x.ravel() - xref) <= 1e-8 * np.linalg.norm(xref)
    # GMRES minimises the residual: non-increasing within a cycle
    for c0 in range(0, len(res.hist), m):
        seg = res.hist[c0:c0 + m]
        assert np.all(np.diff(seg) <= 1e-12 * seg[:-1])
