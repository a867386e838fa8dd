"""Pins of the oracle's operator pieces: (L+1)^-1 (Eq. 12), the canonical
form (§2.2, §3.1: smallest circle, scale), and V/B/s assembly."""
import os

import numpy as np
import pytest

from dense_ref import dense_A, dense_L1, neg_laplacian, re_part

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _read_golden(name):
    vals = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if line:
                k, v = line.split("=", 1)
                vals[k.strip()] = v.strip()
    return vals


@pytest.mark.parametrize("shape,h", [((32,), (1.0,)), ((8, 16), (0.5, 1.0)), ((4, 8, 8), (1.0, 1.0, 2.0))])
def test_Linv_equals_dense_inverse(orc, shape, h):
    """(L+1)^-1 from the FFT path == inverse of the dense (L+1) built from the
    closed-form spectral second-derivative matrix (tests/dense_ref.py)."""
    rng = np.random.default_rng(1)
    D, sigma, c = 1.3, -0.9 - 0.2j, -0.4j
    u = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    got = orc.apply_Linv(u, h, D, sigma, c)
    M = dense_L1(shape, sigma, D, c, list(h))
    ref = np.linalg.solve(M, u.ravel()).reshape(shape)
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_Linv_plane_wave_eigenfunction(orc):
    """(L+1) e^{ip.r} = ((D|p|^2 + sigma)/c + 1) e^{ip.r}  (-lap of a plane wave
    is |p|^2 times it), so (L+1)^-1 must divide by that factor."""
    shape, h = (16, 32), (1.0, 0.25)
    D, sigma, c = 1.0, -2.1 - 0.3j, -0.37j
    y, x = np.meshgrid(np.arange(16) * h[0], np.arange(32) * h[1], indexing="ij")
    for (my, mx) in [(0, 0), (3, -5), (-8, 16), (7, 1)]:
        py, px = 2 * np.pi * my / (16 * h[0]), 2 * np.pi * mx / (32 * h[1])
        u = np.exp(1j * (px * x + py * y))
        got = orc.apply_Linv(u, h, D, sigma, c)
        lam = (D * (px * px + py * py) + sigma) / c + 1.0
        assert np.abs(got * lam - u).max() <= 1e-12


def test_setup_V_B_s(orc):
    rng = np.random.default_rng(5)
    w = rng.standard_normal(64) + 1j * rng.standard_normal(64)
    S = rng.standard_normal(64) + 0j
    sigma, c = 0.3 - 0.1j, 2.0 - 1.0j
    V, B, s = orc.setup(w, S, sigma, c)
    assert np.allclose(c * V + sigma, w, rtol=0, atol=1e-14)    # V := A - L = (w - sigma)/c
    assert np.allclose(B + V, 1.0, rtol=0, atol=1e-15)           # B := 1 - V
    assert np.allclose(c * s, S, rtol=0, atol=1e-15)             # s := S / c


def _brute_mec(pts):
    """Exhaustive smallest enclosing circle: over all pairs (diameter) and
    triples (circumcircle), the smallest circle that contains every point."""
    pts = np.asarray(pts)
    best = (None, np.inf)
    n = len(pts)
    cands = [(p, 0.0) for p in pts]
    for i in range(n):
        for j in range(i + 1, n):
            cands.append(((pts[i] + pts[j]) / 2, abs(pts[i] - pts[j]) / 2))
            for k in range(j + 1, n):
                a, b, c = pts[i], pts[j], pts[k]
                d = 2 * (a.real * (b.imag - c.imag) + b.real * (c.imag - a.imag) + c.real * (a.imag - b.imag))
                if abs(d) < 1e-14:
                    continue
                ux = (abs(a) ** 2 * (b.imag - c.imag) + abs(b) ** 2 * (c.imag - a.imag) + abs(c) ** 2 * (a.imag - b.imag)) / d
                uy = (abs(a) ** 2 * (c.real - b.real) + abs(b) ** 2 * (a.real - c.real) + abs(c) ** 2 * (b.real - a.real)) / d
                o = complex(ux, uy)
                cands.append((o, abs(a - o)))
    for o, r in cands:
        if r < best[1] and np.all(np.abs(pts - o) <= r * (1 + 1e-12) + 1e-15):
            best = (o, r)
    return best


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_mec_matches_brute_force(orc, seed):
    rng = np.random.default_rng(seed)
    pts = rng.standard_normal(30) + 1j * rng.standard_normal(30)
    c, r = orc.mec(pts)
    cb, rb = _brute_mec(pts)
    assert abs(r - rb) <= 1e-12 * rb and abs(c - cb) <= 1e-10


def test_mec_special_cases(orc):
    assert orc.mec([3 + 4j]) == (3 + 4j, 0.0)                     # S:L119 single point
    c, r = orc.mec([-1.0, 1.0])
    assert abs(c) < 1e-15 and abs(r - 1.0) < 1e-15                 # S:L120 two points
    c, r = orc.mec(np.array([0.3, 0.1, 0.9, 0.5, 0.7]) + 0j)        # real points -> mid-range
    assert abs(c - 0.5) < 1e-15 and abs(r - 0.4) < 1e-15


def test_paper_worked_scale_value(orc):
    """c = -(1/(0.95 i)) ||k^2 - kbar^2||; with radius 1 this is
    1/0.95 i = 1.05263i (golden fixture)."""
    g = _read_golden("helmholtz_scale.txt")
    k2 = np.array([0.0, 2.0, 1.0 + 0.5j]) + 0j          # MEC: centre 1, radius 1
    sp = orc.canonical("helmholtz", k2, target_norm=float(g["target_norm"]))
    c_paper = -sp.c                                      # unified form stores -c_paper (R-1)
    assert abs(c_paper - complex(g["c_paper"])) <= 1e-12
    assert abs(sp.bias - 1.0) < 1e-15 and abs(sp.radius - 1.0) < 1e-15


@pytest.mark.parametrize("name,shape", [("C1", None), ("C2", (64, 64)), ("C3", (16, 16, 16)), ("C4", (16, 16, 16))])
def test_canonical_gives_norm_095_and_accretive(orc, name, shape):
    """After scaling, max |V| = 0.95 exactly and A is
    accretive (Eq. 1), checked on a dense A for the small instances."""
    from synth import make

    p = make(name, shape)
    sp = orc.canonical(p.kind, p.medium)
    w = orc.medium_to_w(p.kind, p.medium)
    V, B, s = orc.setup(w, p.source, sp.sigma, sp.c)
    assert abs(np.abs(V).max() - 0.95) <= 1e-12
    if p.n_vox <= 4096:
        A = dense_A(p.shape, w, sp.D, sp.c, list(p.h))
        assert re_part(A) >= -1e-10
