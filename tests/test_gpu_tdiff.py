"""GPU parity of the first-order tensor-diffusion system (§3.2
Eqs. 16-18; desc.tensor_diffusion, kernels_tdiff.cu) against the oracle's
orc_fixed_point_tdiff on the same float32-rounded mu_a, D and S."""
import numpy as np
import pytest

from gpu_helpers import TOL_FIELD, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")


def _medium(shape, seed, aniso=True):
    rng = np.random.default_rng(seed)
    d = len(shape)
    mu = (0.02 + 0.08 * rng.random(shape)).astype(np.float32)
    if aniso:
        A = rng.standard_normal(shape + (d, d)) * 0.3
        D = np.einsum("...ij,...kj->...ik", A, A) + np.eye(d) * (0.5 + rng.random(shape)[..., None, None])
    else:
        D = np.broadcast_to(np.eye(d) * 1.3, shape + (d, d)).copy()
        D[tuple(s // 4 for s in shape)] *= 2.0
    D = D.astype(np.float32)
    S = np.zeros(shape, dtype=np.float32)
    S[tuple(s // 2 for s in shape)] = 1.0
    return mu, D, S


def _gpu(shape, mu, D, S, n, tol=0.0):
    import torch
    from paper_2207_14222_b200 import Plan

    plan = Plan(shape, kind="diffusion", tensor_diffusion=True)
    plan.set_tensor_medium(torch.from_numpy(mu).cuda(), torch.from_numpy(D).cuda(), 0.95)
    plan.set_source(torch.from_numpy(S).cuda())
    nd, term = plan.iterate(n, 0.75, tol)
    return plan.get_field().cpu().numpy().astype(np.float64), nd, term, plan


def _orc(orc, shape, mu, D, S, n, tol=0.0):
    sp = orc.canonical_tdiff(mu.astype(np.float64), D.astype(np.float64))
    r = orc.fixed_point_tdiff(mu.astype(np.float64), D.astype(np.float64), S.astype(np.float64),
                              [1.0] * len(shape), sp, 0.75, tol, n)
    return r, sp


# x extents 64-256 (and 2-D 512) run the fused TMA-pipelined x pass
# (k_tdiff_pipe); 3-D with x extent 512 the k_xfft + k_tdiff_upd sequence
@pytest.mark.parametrize("shape,aniso,n", [((64, 64), True, 150), ((64, 128), False, 100), ((64, 64, 64), True, 60),
                                           ((128, 64, 64), True, 30), ((64, 256), True, 80), ((64, 512), True, 60),
                                           ((64, 1024), True, 40), ((64, 64, 256), True, 20),
                                           ((64, 64, 512), True, 10), ((64, 128, 256), True, 6)])
def test_tdiff_matches_oracle(orc, shape, aniso, n):
    mu, D, S = _medium(shape, 3, aniso)
    u, nd, term, plan = _gpu(shape, mu, D, S, n)
    assert nd == n and term == "max_iter"
    r, sp = _orc(orc, shape, mu, D, S, n)
    ref = (r.x[0] / np.sqrt(sp.s_u)).real
    s = plan.split
    assert abs(s.c.real - sp.c) <= 1e-5 * sp.c and abs(s.centre.real - sp.s_u) <= 1e-5 * sp.s_u
    assert rel_l2(u, ref) <= TOL_FIELD, rel_l2(u, ref)
    h = plan.history()
    k = r.hist[:n] > 1e-10        # above the oracle's x-form floor (the GPU Delta-form has none, R-17)
    assert np.allclose(h[:n][k], r.hist[:n][k], rtol=1e-3, atol=0.0)
    assert np.all(np.diff(h[: n + 1]) <= 1e-5 * h[:n])          # Cor. 1: monotone


@pytest.mark.parametrize("shape", [(64, 256), (64, 64, 128)])
def test_tdiff_split_iterate_equals_one_call(shape):
    """iterate(a) + iterate(b) == iterate(a + b) bit for bit: the state the
    fused x pass leaves between calls (x-transformed work) is complete."""
    mu, D, S = _medium(shape, 6, True)
    u1, _, _, p1 = _gpu(shape, mu, D, S, 25)
    mu2, D2, S2 = _medium(shape, 6, True)
    u2, n2, _, p2 = _gpu(shape, mu2, D2, S2, 10)
    n3, _ = p2.iterate(15, 0.75, 0.0)
    u2 = p2.get_field().cpu().numpy().astype(np.float64)
    assert n2 + n3 == 25 and np.array_equal(u1, u2)
    assert np.array_equal(p1.history()[:26], p2.history()[:26])


def test_tdiff_converges_like_oracle(orc):
    shape = (64, 64)
    mu, D, S = _medium(shape, 4, True)
    u, nd, term, plan = _gpu(shape, mu, D, S, 20000, 1e-5)
    r, sp = _orc(orc, shape, mu, D, S, 20000, 1e-5)
    assert term == "converged" and abs(nd - r.n_done) <= 1, (nd, r.n_done)
    assert rel_l2(u, (r.x[0] / np.sqrt(sp.s_u)).real) <= TOL_FIELD


def test_tdiff_isotropic_equals_scalar_path():
    """Isotropic constant D = d I: u of the (u, F) system = the scalar
    second-order solution (the standard plan), both converged."""
    import torch
    from paper_2207_14222_b200 import Plan

    shape = (64, 64)
    rng = np.random.default_rng(9)
    mu = (0.03 + 0.05 * rng.random(shape)).astype(np.float32)
    D = np.broadcast_to(np.eye(2, dtype=np.float32) * 1.5, shape + (2, 2)).copy()
    S = np.zeros(shape, dtype=np.float32)
    S[32, 32] = 1.0
    u, nd, term, _ = _gpu(shape, mu, D, S, 40000, 1e-7)
    ps = Plan(shape, kind="diffusion", D=1.5, dtype="r32")
    ps.set_potential(torch.from_numpy(mu).cuda(), 0.95)
    ps.set_source(torch.from_numpy(S).cuda())
    ps.iterate(40000, 0.75, 1e-7)
    us = ps.get_field().cpu().numpy().astype(np.float64)
    assert term == "converged" and rel_l2(u, us) <= 2e-5, rel_l2(u, us)
