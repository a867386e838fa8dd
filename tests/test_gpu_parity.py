"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the
same seeded inputs, and against closed forms at full size.

Bars (BASELINE.json north_star): relative L2 of the field <= 1e-4 after the
same iteration count; iteration counts to 1e-6 identical within +-1.
"""
import math

import numpy as np
import pytest

from gpu_helpers import TOL_COUNT, TOL_FIELD, monotone, rel_l2, rounded_inputs, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")


# ------------------------------------------------------------ canonical --
@pytest.mark.parametrize("name,shape", [("C1", None), ("C2", (128, 128)), ("C3", (32, 32, 32)), ("C4", (32, 32, 32))])
def test_split_matches_oracle(orc, name, shape):
    """Device smallest-circle + scale == oracle's Welzl."""
    from synth import make

    p = make(name, shape)
    med, src, dtype = rounded_inputs(p)
    _, _, _, plan = run_gpu(p, n_iter=1)
    sp = orc.canonical(p.kind, med.astype(np.complex128), 0.95)
    s = plan.split
    assert abs(s.radius - sp.radius) <= 1e-12 * sp.radius
    assert abs(s.centre - sp.bias) <= 1e-12 * abs(sp.bias)
    assert abs(s.c - sp.c) <= 1e-12 * abs(sp.c) and abs(s.sigma - sp.sigma) <= 1e-12 * abs(sp.sigma)
    assert abs(s.max_abs_V - 0.95) <= 1e-6


# --------------------------------------------------------- closed form --
def _homog(shape, k0=2 * math.pi / 8, n=1.0 + 0.05j):
    k2 = (k0 * n) ** 2
    sigma, c = -k2.real, -1j * abs(k2.imag) / 0.95
    return k2, sigma, c


SHAPES = [(16,), (64,), (256,), (1024,), (2048,), (16, 16), (32, 512), (512, 64), (1024, 16), (16, 2048),
          (2048, 16), (16, 32, 64), (64, 16, 128), (32, 256, 16), (16, 16, 1024), (128, 128, 128),
          (2048, 16, 16), (16, 2048, 16), (16, 16, 2048), (32, 64, 32), (64, 32, 64), (512, 512, 64),
          (512, 64, 512)]


@pytest.mark.parametrize("shape", SHAPES)
def test_closed_form_constant_V(shape):
    """Constant V: x^_k = x^*(1 - q^k) per Fourier mode (tests/test_oracle_iteration
    derives it); covers every pass kernel, every supported line length and
    ragged (non-cubic) grids."""
    import torch
    from paper_2207_14222_b200 import Plan

    k2, sigma, c = _homog(shape)
    alpha, D = 0.75, 1.0
    S = np.zeros(shape, dtype=np.complex64)
    S[tuple(s // 3 for s in shape)] = 1.0
    S[tuple(s // 5 for s in shape)] = 0.5 - 0.25j
    plan = Plan(shape, sigma=sigma, c=c)
    plan.set_potential(torch.full(shape, k2, dtype=torch.complex64, device="cuda"), -1.0)
    plan.set_source(torch.from_numpy(S).cuda())
    w = -complex(np.complex64(k2))
    v0 = (w - sigma) / c
    b = 1.0 - v0
    p2 = sum(np.meshgrid(*[(2 * np.pi * np.fft.fftfreq(n)) ** 2 for n in shape], indexing="ij"))
    ghat = c / (D * p2 + sigma + c)
    q = 1.0 - alpha * b * (1.0 - b * ghat)
    shat = np.fft.fftn(S.astype(np.complex128) / c)
    xstar = ghat * shat / (1.0 - b * ghat)
    done = 0
    for k in (1, 7, 30):
        n, term = plan.iterate(k - done, alpha, 0.0)
        assert n == k - done and term == "max_iter"
        done = k
        x = plan.get_field().cpu().numpy().astype(np.complex128)
        ref = np.fft.ifftn(xstar * (1.0 - q ** k))
        err = rel_l2(x, ref)
        assert err <= 2e-5, (shape, k, err)
    hist = plan.history()
    d0 = b * ghat * shat
    r_ref = np.array([np.linalg.norm(q ** j * d0) / np.linalg.norm(d0) for j in range(31)])
    assert np.allclose(hist[:31], r_ref, rtol=1e-4, atol=1e-7)


# --------------------------------------------------------- config parity --
def _parity_tol(orc, p):
    xg, ng, term, plan = run_gpu(p)
    res, _ = run_oracle(orc, p)
    assert term == "converged" and res.hist[-1] < p.tol
    assert abs(ng - res.n_done) <= TOL_COUNT, (ng, res.n_done)
    ref, _ = run_oracle(orc, p, n_iter=ng, tol=0.0)
    err = rel_l2(xg, ref.x)
    assert err <= TOL_FIELD, err
    h = plan.history()
    assert h.size == ng                # converged: r_0 .. r_{ng-1} (R-5: x_ng's own residual is not computed)
    assert monotone(h)                                            # Cor. 1: monotone
    return ng, res.n_done, err


def test_parity_C1(orc):
    from synth import make

    ng, no, err = _parity_tol(orc, make("C1"))
    assert no == 228                                              # DESIGN.md expected count


@pytest.mark.parametrize("shape", [(128, 128), (512, 512)])
def test_parity_C2(orc, shape):
    from synth import make

    _parity_tol(orc, make("C2", shape))


@pytest.mark.parametrize("name,shape,n", [("C3", (64, 64, 64), 200), ("C4", (64, 64, 64), 200),
                                          ("C5", (64, 64, 64), 100), ("C3", (32, 64, 128), 120),
                                          ("C5", (16, 128, 32), 60), ("C4", (32, 16, 64), 80)])
def test_parity_fixed_count(orc, name, shape, n):
    from synth import make

    p = make(name, shape)
    xg, ng, term, plan = run_gpu(p, n_iter=n)
    assert ng == n and term == "max_iter"
    res, _ = run_oracle(orc, p, n_iter=n)
    err = rel_l2(xg, res.x)
    assert err <= TOL_FIELD, err
    h = plan.history()
    assert np.allclose(h[:n], res.hist[:n], rtol=1e-3, atol=0.0)   # r_k, k = 0..n-1
    assert monotone(h[: n + 1])


def test_full_size_C3_first_iterations(orc):
    """BASELINE.json C3 at its full size (256^3) in the bench's launch
    configuration: the first iterations match the oracle element by element."""
    from synth import make

    p = make("C3")
    xg, ng, term, _ = run_gpu(p, n_iter=4)
    res, _ = run_oracle(orc, p, n_iter=4)
    assert rel_l2(xg, res.x) <= TOL_FIELD


def test_resume_equals_single_call(orc):
    """usp_iterate is resumable: 3 + 4 iterations == 7 iterations."""
    from synth import make

    p = make("C5", (32, 32, 32))
    x7, _, _, _ = run_gpu(p, n_iter=7)
    _, _, _, plan = run_gpu(p, n_iter=3)
    n, _ = plan.iterate(4, 0.75, 0.0)
    x34 = plan.get_field().cpu().numpy()
    assert n == 4 and np.array_equal(x34.astype(np.complex128), x7)


def test_validation_errors():
    """Theorem 1's hypotheses are checked: ||V|| < 1 and accretive A."""
    import torch
    from paper_2207_14222_b200 import Plan, USPError

    shape = (16, 16)
    k2 = torch.full(shape, (2 * math.pi / 8) ** 2 + 0.0j, dtype=torch.complex64, device="cuda")
    plan = Plan(shape, sigma=-0.5, c=-0.1j)
    with pytest.raises(USPError) as e:
        plan.set_potential(k2, -1.0)                   # |V| = |0.117/0.1| > 1
    assert e.value.name == "USP_ERR_NOT_CONTRACTIVE"
    gain = k2.clone()
    gain[3, 3] = gain[3, 3] - 0.01j                    # Im k^2 < 0: gain, not accretive
    plan2 = Plan(shape)
    with pytest.raises(USPError) as e:
        plan2.set_potential(gain, 0.95)
    assert e.value.name == "USP_ERR_NOT_ACCRETIVE"
    plan3 = Plan(shape)
    with pytest.raises(USPError) as e:
        plan3.set_potential(torch.full(shape, 1.0 + 0.1j, dtype=torch.complex64, device="cuda"), 0.95)
    assert e.value.name == "USP_ERR_ARG"               # homogeneous: radius 0
    with pytest.raises(USPError):
        plan3.iterate(1, 0.75, 0.0)                    # no source yet -> state error


def test_zero_source_and_tol_one():
    import torch
    from paper_2207_14222_b200 import Plan
    from synth import make

    p = make("C5", (16, 16, 16))
    med, src, _ = rounded_inputs(p)
    plan = Plan(p.shape)
    plan.set_potential(torch.from_numpy(med).cuda(), 0.95)
    plan.set_source(torch.zeros(p.shape, dtype=torch.complex64, device="cuda"))
    n, term = plan.iterate(10, 0.75, 1e-6)
    assert n == 0 and term == "converged" and float(plan.get_field().abs().max()) == 0.0
    plan.set_source(torch.from_numpy(src).cuda())
    n, term = plan.iterate(10, 0.75, 2.0)              # r_0 = 1 < tol: one iteration (R-5)
    assert n == 1 and term == "converged"


def test_full_size_C5_plane_waves():
    """1024^3 (BASELINE.json C5 grid) with constant V and a source made of a few
    grid plane waves: every voxel of x_k has a closed form."""
    import torch
    from paper_2207_14222_b200 import Plan

    n = 1024
    shape = (n, n, n)
    k2, sigma, c = _homog(shape)
    alpha, K = 0.75, 3
    rng = np.random.default_rng(5)
    modes = [tuple(int(m) for m in rng.integers(-n // 2, n // 2, 3)) for _ in range(4)] + [(0, 0, 0), (n // 2, 1, -3)]
    amps = rng.standard_normal(len(modes)) + 1j * rng.standard_normal(len(modes))
    dev = "cuda"
    ar = torch.arange(n, device=dev, dtype=torch.float64)

    def field(coefs):
        out = torch.zeros(shape, dtype=torch.complex64, device=dev)
        for (mz, my, mx), a in zip(modes, coefs):
            ez = torch.exp(1j * 2 * math.pi * mz * ar / n)
            ey = torch.exp(1j * 2 * math.pi * my * ar / n)
            ex = torch.exp(1j * 2 * math.pi * mx * ar / n)
            out += (complex(a) * ez[:, None, None] * ey[None, :, None] * ex[None, None, :]).to(torch.complex64)
        return out

    S = field(amps)
    plan = Plan(shape, sigma=sigma, c=c)
    plan.set_potential(torch.full(shape, k2, dtype=torch.complex64, device=dev), -1.0)
    plan.set_source(S)
    del S
    nd, _ = plan.iterate(K, alpha, 0.0)
    assert nd == K
    x = plan.get_field()
    w = -complex(np.complex64(k2))
    b = 1.0 - (w - sigma) / c
    coefs = []
    for (mz, my, mx), a in zip(modes, amps):
        p2 = sum((2 * math.pi * ((m + n // 2) % n - n // 2) / n) ** 2 for m in (mz, my, mx))
        g = c / (p2 + sigma + c)
        q = 1.0 - alpha * b * (1.0 - b * g)
        coefs.append(a / c * g / (1.0 - b * g) * (1.0 - q ** K))
    ref = field(coefs)
    err = float(torch.linalg.vector_norm(x - ref) / torch.linalg.vector_norm(ref))
    assert err <= 2e-5, err


def test_full_size_C5_linear_in_source():
    """BASELINE.json C5 at its full size (1024^3, the heterogeneous GRF medium,
    the bench's launch configuration), where the oracle cannot run: with
    x_0 = 0 and a fixed count, Alg. 1 is a fixed linear map of the
    source, so x_k(s1 + 2 s2) = x_k(s1) + 2 x_k(s2) voxel by voxel (up to fp32
    rounding), and the residual is monotone (Cor. 1)."""
    import torch
    from paper_2207_14222_b200 import Plan
    from synth import make

    p = make("C5", device="cuda")
    shape, K = p.shape, 5
    med = p.medium.to(torch.complex64)
    s1 = p.source.to(torch.complex64)
    del p
    s2 = torch.zeros_like(s1)
    s2[300, 700, 123] = 1.0 - 0.5j
    s2[900, 64, 1000] = 0.25
    plan = Plan(shape)
    plan.set_potential(med, 0.95)
    del med
    xs = []
    for s in (s1, s2, s1 + 2 * s2):
        plan.set_source(s)
        nd, term = plan.iterate(K, 0.75, 0.0)
        assert nd == K and term == "max_iter"
        h = plan.history()[: K + 1]
        assert np.all(np.diff(h) <= 1e-5 * h[:-1]), h
        xs.append(plan.get_field())
    x1, x2, x12 = xs
    err = float(torch.linalg.vector_norm(x12 - x1 - 2 * x2) / torch.linalg.vector_norm(x12))
    assert err <= 1e-5, err
    assert float(torch.linalg.vector_norm(x2)) > 0.1 * float(torch.linalg.vector_norm(x1))
