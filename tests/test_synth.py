"""The seeded input generator: deterministic, back-end independent, and
matching the recipes of DESIGN.md (readings R-9 .. R-16)."""
import numpy as np
import pytest

from synth import make
from synth.inputs import absorber_ramp, white_noise


def test_white_noise_same_bits_numpy_and_torch():
    torch = pytest.importorskip("torch")
    a = white_noise((4, 8, 16), seed=3)
    b = white_noise((4, 8, 16), seed=3, device="cpu").numpy()
    assert np.abs(a - b).max() <= 1e-15
    assert abs(a.mean()) < 0.2 and abs(a.std() - 1) < 0.1
    c = white_noise((4, 8, 16), seed=4)
    assert np.abs(a - c).max() > 0.1


def test_absorber_ramp_R9():
    r = absorber_ramp((16,), 4)
    assert np.allclose(r[:4], [1.0, 0.75, 0.5, 0.25]) and np.allclose(r[-4:], [0.25, 0.5, 0.75, 1.0])
    assert np.all(r[4:12] == 0)


def test_configs_shapes_and_ranges():
    p1 = make("C1")
    assert p1.shape == (256,) and p1.tol == 1e-6 and p1.n_iter == 2000
    assert p1.source[64] == 1 and np.count_nonzero(p1.source) == 1
    assert np.all(p1.medium.imag >= 0)                 # gain-free
    p2 = make("C2")
    assert abs(p2.meta["fill"] - 0.2247) < 1e-3 and p2.meta["n_disks"] == 200
    p3 = make("C3", (32, 32, 32))
    nre = np.sqrt(p3.medium).real / (2 * np.pi / 6)
    assert nre.min() >= 1.33 - 1e-9 and nre.max() <= 1.45 + 1e-9
    p4 = make("C4", (32, 32, 32))
    assert p4.kind == "diffusion" and np.all(p4.medium > 0)
    assert abs(np.median(p4.medium) - 0.01) < 0.002


def test_deterministic():
    a = make("C5", (16, 16, 16))
    b = make("C5", (16, 16, 16))
    assert np.array_equal(a.medium, b.medium)
