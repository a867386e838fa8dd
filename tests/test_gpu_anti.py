"""GPU parity of the antisymmetrised system (Eq. 9-10;
desc.antisymmetric, kernels_anti.cu) against the oracle's
orc_fixed_point_anti, including a NON-accretive gain medium that the
standard form rejects."""
import math

import numpy as np
import pytest

from gpu_helpers import TOL_FIELD, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")


def _medium(shape, seed, gain):
    rng = np.random.default_rng(seed)
    k0 = 2 * math.pi / 8
    n = 1.0 + 0.3 * rng.random(shape) + 1j * (0.1 * rng.random(shape) - gain)
    k2 = ((k0 * n) ** 2).astype(np.complex64)
    S = np.zeros(shape, dtype=np.complex64)
    S[tuple(s // 3 for s in shape)] = 1.0
    return k2, S


def _gpu(shape, k2, S, n, tol=0.0):
    import torch
    from paper_2207_14222_b200 import Plan

    plan = Plan(shape, antisymmetric=True)
    plan.set_potential(torch.from_numpy(k2).cuda(), 0.95)
    plan.set_source(torch.from_numpy(S).cuda())
    nd, term = plan.iterate(n, 0.75, tol)
    return plan.get_field().cpu().numpy().astype(np.complex128), nd, term, plan


# every x extent of the TMA-pipelined x pass (k_anti_pipe<64 .. 1024>)
@pytest.mark.parametrize("shape,gain,n", [((64, 64), 0.0, 200), ((64, 128), 0.05, 150), ((64, 64, 64), 0.05, 60),
                                          ((128, 64, 64), 0.0, 40), ((64, 256), 0.05, 80), ((64, 512), 0.0, 60),
                                          ((64, 1024), 0.05, 40), ((64, 64, 256), 0.05, 20),
                                          ((128, 128, 256), 0.05, 8)])
def test_anti_matches_oracle(orc, shape, gain, n):
    k2, S = _medium(shape, 5, gain)
    x, nd, term, plan = _gpu(shape, k2, S, n)
    assert nd == n and term == "max_iter"
    k2d = k2.astype(np.complex128)
    w = orc.medium_to_w("helmholtz", k2d)
    sp = orc.canonical_anti("helmholtz", k2d)
    res = orc.fixed_point_anti(w, S.astype(np.complex128), [1.0] * len(shape), sp.D, sp.sigma, sp.c.real,
                               0.75, 0.0, n)
    s = plan.split
    assert abs(s.c.real - sp.c.real) <= 1e-12 * sp.c.real and s.c.imag == 0.0
    assert abs(s.sigma - sp.sigma) <= 1e-12 * abs(sp.sigma)
    assert rel_l2(x, res.x[0]) <= TOL_FIELD, rel_l2(x, res.x[0])
    h = plan.history()
    assert np.allclose(h[:n], res.hist[:n], rtol=1e-3, atol=0.0)          # r_0 .. r_{n-1}
    assert np.all(np.diff(h[: n + 1]) <= 1e-5 * h[:n])       # Cor. 1: monotone


@pytest.mark.parametrize("shape", [(64, 1024), (64, 64, 128)])
def test_anti_split_iterate_equals_one_call(shape):
    """iterate(a) + iterate(b) == iterate(a + b) bit for bit (the state the
    pipelined x pass leaves between calls is complete)."""
    k2, S = _medium(shape, 7, 0.05)
    x1, _, _, p1 = _gpu(shape, k2, S, 25)
    x2, n2, _, p2 = _gpu(shape, k2, S, 10)
    n3, _ = p2.iterate(15, 0.75, 0.0)
    x2 = p2.get_field().cpu().numpy().astype(np.complex128)
    assert n2 + n3 == 25 and np.array_equal(x1, x2)
    assert np.array_equal(p1.history()[:26], p2.history()[:26])


def test_gain_medium_rejected_by_standard_form_solved_by_anti():
    import torch
    from paper_2207_14222_b200 import Plan, USPError

    shape = (64, 64)
    k2, S = _medium(shape, 6, 0.2)
    plan = Plan(shape)
    with pytest.raises(USPError, match="NOT_ACCRETIVE"):
        plan.set_potential(torch.from_numpy(k2).cuda(), 0.95)
    x, nd, term, pa = _gpu(shape, k2, S, 300)
    h = pa.history()
    assert np.isfinite(x).all() and h[300] < h[1] and np.all(np.diff(h[:301]) <= 1e-5 * h[:300])
