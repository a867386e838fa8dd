"""Pins of the oracle's DFT (oracle/usp_oracle.c orc_fft1d / orc_fftn) against
the definition (brute-force sums), Parseval, special cases and a library FFT."""
import numpy as np
import pytest


def brute_dft(x, inverse=False):
    """X[k] = sum_n x[n] exp(-+ 2 pi i k n / N) written out term by term."""
    n = len(x)
    sgn = 1.0 if inverse else -1.0
    out = np.zeros(n, dtype=np.complex128)
    for k in range(n):
        acc = 0j
        for j in range(n):
            acc += x[j] * np.exp(sgn * 2j * np.pi * k * j / n)
        out[k] = acc / (n if inverse else 1)
    return out


@pytest.mark.parametrize("n", [1, 2, 4, 8, 16, 32, 64])
def test_fft1d_matches_definition(orc, n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    for inv in (False, True):
        got = orc.fft1d(x, inverse=inv)
        ref = brute_dft(x, inverse=inv)
        assert np.abs(got - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max()) * n


@pytest.mark.parametrize("shape", [(8, 4), (4, 8, 2), (2, 16)])
def test_fftn_is_separable_definition(orc, shape):
    rng = np.random.default_rng(7)
    x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    ref = x.copy()
    for ax in range(len(shape)):
        ref = np.apply_along_axis(brute_dft, ax, ref)
    got = orc.fftn(x)
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_parseval_roundtrip_impulse(orc):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((16, 8, 32)) + 1j * rng.standard_normal((16, 8, 32))
    X = orc.fftn(x)
    assert abs(np.vdot(X, X).real - x.size * np.vdot(x, x).real) <= 1e-11 * x.size * np.vdot(x, x).real
    assert np.abs(orc.ifftn(X) - x).max() <= 1e-13 * np.abs(x).max() * 10
    d = np.zeros((8, 8), dtype=complex)
    d[0, 0] = 1.0
    assert np.abs(orc.fftn(d) - 1.0).max() == 0.0


def test_fftn_matches_library(orc):
    rng = np.random.default_rng(11)
    x = rng.standard_normal((32, 16, 64)) + 1j * rng.standard_normal((32, 16, 64))
    assert np.abs(orc.fftn(x) - np.fft.fftn(x)).max() <= 1e-12 * np.abs(x).sum() ** 0.5 * 10
    assert np.abs(orc.ifftn(x) - np.fft.ifftn(x)).max() <= 1e-14 * 10 * np.abs(x).max()


def test_non_power_of_two_rejected(orc):
    with pytest.raises(ValueError):
        orc.fftn(np.zeros(12, dtype=complex))
