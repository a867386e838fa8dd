"""Pins of the oracle's first-order tensor-diffusion system (§3.2
Eqs. 16-18; oracle orc_fixed_point_tdiff + canonical_tdiff),
against things other than itself:

* isotropic D = d I: the (u, F) system's u equals the SECOND-order solution
  of -d lap u + mu u = S (the oracle's scalar path, itself pinned to dense
  LU), in 2-D and 3-D;
* anisotropic, heterogeneous D: dense LU of A_raw [u; F] = [S; 0] built from
  numpy-DFT gradient matrices (not the oracle's FFT): u and F match;
* monotone residual (Cor. 1) and ||V|| < 1 from the canonical form.
"""
import numpy as np
import pytest


def _grad_mats(shape, h):
    """Dense spectral d/dx_k (symbol i p_k, p = 2 pi fftfreq) on a C-ordered grid."""
    mats = []
    for a, n in enumerate(shape):
        W = np.fft.fft(np.eye(n), axis=0)
        Winv = np.fft.ifft(np.eye(n), axis=0)
        p = 2 * np.pi * np.fft.fftfreq(n, h[a])
        G1 = Winv @ np.diag(1j * p) @ W
        ops = [np.eye(s) for s in shape]
        ops[a] = G1
        M = ops[0]
        for o in ops[1:]:
            M = np.kron(M, o)
        mats.append(M)
    return mats[::-1]          # order: x (last axis) first, then y, z


def _aniso(shape, seed):
    rng = np.random.default_rng(seed)
    d = len(shape)
    mu = 0.02 + 0.08 * rng.random(shape)
    A = rng.standard_normal(shape + (d, d)) * 0.3
    D = np.einsum("...ij,...kj->...ik", A, A) + np.eye(d) * (0.5 + rng.random(shape)[..., None, None])
    S = np.zeros(shape)
    S[tuple(s // 2 for s in shape)] = 1.0
    S += 0.1 * rng.random(shape)
    return mu, D, S


@pytest.mark.parametrize("shape", [(32, 32), (16, 16, 16)])
def test_isotropic_equals_second_order(orc, shape):
    rng = np.random.default_rng(1)
    mu = 0.05 + 0.05 * rng.random(shape)
    dcoef = 1.7
    D = np.zeros(shape + (len(shape), len(shape)))
    for k in range(len(shape)):
        D[..., k, k] = dcoef
    S = np.zeros(shape)
    S[tuple(s // 2 for s in shape)] = 1.0
    sp = orc.canonical_tdiff(mu, D)
    r = orc.fixed_point_tdiff(mu, D, S, [1.0] * len(shape), sp, 0.75, 1e-11, 50000)
    assert r.rc == 0 and r.hist[-1] < 1e-11
    u = r.x[0] / np.sqrt(sp.s_u)
    spd = orc.canonical("diffusion", mu.astype(complex), D=dcoef)
    f = orc.fixed_point(mu.astype(complex), S.astype(complex), [1.0] * len(shape), dcoef, spd.sigma, spd.c, 0.75,
                        1e-12, 50000)
    assert np.linalg.norm(u - f.x) <= 1e-8 * np.linalg.norm(f.x)
    assert np.all(np.diff(r.hist) <= 1e-12 * r.hist[:-1])


@pytest.mark.parametrize("shape,seed", [((8, 16), 2), ((16, 8), 3), ((4, 8, 8), 4)])
def test_anisotropic_equals_dense_first_order_LU(orc, shape, seed):
    mu, D, S = _aniso(shape, seed)
    d = len(shape)
    n = int(np.prod(shape))
    G = _grad_mats(shape, [1.0] * d)
    Dinv = np.linalg.inv(D).reshape(n, d, d)
    A = np.zeros(((d + 1) * n, (d + 1) * n), dtype=complex)
    A[:n, :n] = np.diag(mu.ravel())
    for k in range(d):
        A[:n, (k + 1) * n:(k + 2) * n] = G[k]          # div F
        A[(k + 1) * n:(k + 2) * n, :n] = G[k]          # grad u
        for m in range(d):
            A[(k + 1) * n:(k + 2) * n, (m + 1) * n:(m + 2) * n] = np.diag(Dinv[:, k, m])
    rhs = np.zeros((d + 1) * n, dtype=complex)
    rhs[:n] = S.ravel()
    ref = np.linalg.solve(A, rhs)
    sp = orc.canonical_tdiff(mu, D)
    r = orc.fixed_point_tdiff(mu, D, S, [1.0] * d, sp, 0.75, 1e-12, 400000)
    assert r.rc == 0 and r.hist[-1] < 1e-12
    u = r.x[0].ravel() / np.sqrt(sp.s_u)
    F = np.concatenate([r.x[k + 1].ravel() / np.sqrt(sp.s_F) for k in range(d)])
    assert np.linalg.norm(u - ref[:n]) <= 1e-8 * np.linalg.norm(ref[:n])
    assert np.linalg.norm(F - ref[n:]) <= 1e-8 * np.linalg.norm(ref[n:])
    assert np.all(np.diff(r.hist) <= 1e-12 * r.hist[:-1])


def test_canonical_tdiff_norm_below_one(orc):
    mu, D, S = _aniso((8, 8, 8), 5)
    sp = orc.canonical_tdiff(mu, D, 0.95)
    dpk = orc.dinv_field(D)
    d = 3
    Vf = np.zeros((512, d, d))
    for q, (i, j) in enumerate([(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]):
        Vf[:, i, j] = Vf[:, j, i] = ((dpk[..., q] - sp.dbar[q]) / (sp.c * sp.s_F)).ravel()
    spec = np.abs(np.linalg.eigvalsh(Vf)).max()
    vu = np.abs((mu - sp.mubar) / (sp.c * sp.s_u)).max()
    assert max(spec, vu) <= 0.95 * (1 + 1e-12) and max(spec, vu) > 0.5
