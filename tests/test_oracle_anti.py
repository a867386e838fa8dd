"""Pins of the oracle's antisymmetrised system (Eq. 9-10, PAPER.md
L100-128; oracle/usp_oracle.c orc_fixed_point_anti), against things other
than itself:

* dense LU of the ORIGINAL system A_raw x = S (tests/dense_ref.py, no FFT):
  the converged first component is its solution and the second -> 0
  (s' = 0), also for a NON-accretive problem (a gain medium, Im k^2 < 0),
  where the standard canonical form of §2.2 does not apply;
* the dense 2N x 2N antisymmetrised operator is skew-Hermitian (so accretive:
  Re[A] = 0) for any A_raw, with ||V|| = 0.95 for c = r/0.95;
* monotone residual (Corollary 1, L478-491) since A is accretive and
  ||V|| < 1.
"""
import math

import numpy as np
import pytest

from dense_ref import dense_A, re_part


def _gain_problem(shape, seed, gain):
    rng = np.random.default_rng(seed)
    k0 = 2 * math.pi / 6
    n = 1.0 + 0.3 * rng.random(shape) + 1j * (0.2 * rng.random(shape) - gain)   # Im n < 0 somewhere: gain
    k2 = (k0 * n) ** 2
    S = np.zeros(shape, dtype=complex)
    S[tuple(s // 3 for s in shape)] = 1.0
    S += 0.05 * (rng.standard_normal(shape) + 1j * rng.standard_normal(shape))
    return k2, S


@pytest.mark.parametrize("shape,seed,gain", [((16,), 1, 0.0), ((32,), 2, 0.15), ((8, 8), 3, 0.15),
                                             ((4, 4, 8), 4, 0.1)])
def test_anti_converges_to_dense_solution(orc, shape, seed, gain):
    k2, S = _gain_problem(shape, seed, gain)
    w = orc.medium_to_w("helmholtz", k2)
    sp = orc.canonical_anti("helmholtz", k2)
    A_raw = dense_A(shape, w, sp.D, 1.0)          # -D lap + diag(w)
    if gain > 0:
        # not accretive for any complex scale: the numerical range of A_raw
        # straddles the origin (Re[e^{i phi} A_raw] < 0 for every phi tried)
        assert all(re_part(np.exp(1j * ph) * A_raw) < 0 for ph in np.linspace(0, 2 * np.pi, 72))
    xref = np.linalg.solve(A_raw, S.ravel()).reshape(shape)
    res = orc.fixed_point_anti(w, S, [1.0] * len(shape), sp.D, sp.sigma, sp.c.real, 0.9, 1e-11, 400000)
    assert res.rc == 0 and res.hist[-1] < 1e-11
    assert np.linalg.norm(res.x[0] - xref) <= 1e-7 * np.linalg.norm(xref)
    assert np.linalg.norm(res.x[1]) <= 1e-7 * np.linalg.norm(xref)
    assert np.all(np.diff(res.hist) <= 1e-12 * res.hist[:-1])     # Cor. 1: monotone


@pytest.mark.parametrize("shape", [(16,), (4, 8)])
def test_anti_operator_is_skew_hermitian_with_norm_V(orc, shape):
    k2, S = _gain_problem(shape, 7, 0.2)
    w = orc.medium_to_w("helmholtz", k2)
    sp = orc.canonical_anti("helmholtz", k2)
    c = sp.c.real
    A_raw = dense_A(shape, w, sp.D, 1.0)
    Z = np.zeros_like(A_raw)
    A = np.block([[Z, -A_raw.conj().T], [A_raw, Z]]) / c
    assert np.abs(A + A.conj().T).max() <= 1e-12 * np.abs(A).max()   # skew-Hermitian -> accretive
    Vraw = (w - sp.sigma).ravel()
    V = np.block([[Z, -np.diag(Vraw.conj())], [np.diag(Vraw), Z]]) / c
    assert abs(np.linalg.norm(V, 2) - 0.95) <= 1e-12
