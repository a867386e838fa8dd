"""Seeded generators for the five BASELINE.json configs (C1..C5, C5w).

Everything here is *input synthesis*: refractive-index / absorption maps and
sources of the physical problems the paper solves (§3.1 Eq. 8 for
Helmholtz, §3.2 for diffusion).  The method itself (bias, scale, V, B,
(L+1)^-1, Algorithm 1) lives in ``oracle/`` (CPU, test infrastructure) and in
``paper_2207_14222_b200`` (CUDA product) -- never here.

The paper states no geometry for these configs (they are BASELINE.json's
synthetic stand-ins, PAPER.md:L178 / L367 geometries are figure-defined), so
the recipes follow SURVEY.md §8(c) readings R-9 .. R-16, restated in DESIGN.md:

* R-9  absorbing layer: ``Im n += 0.2 * ramp``, ramp linear from 0.2/W at the
  first absorbing cell to 1 at the outermost cell, per axis, max over axes.
* R-10 C1 slab ``x in [3N/8, 5N/8)`` with ``n = 1.5+0.01i``, unit source at
  ``x = N/4``.
* R-12 C2: 200 disks, centre/radius/index drawn from numpy PCG64(seed) in the
  order cx, cy, r, n; later disks overwrite earlier ones.
* R-13 C2 source: row ``y = 48``: ``exp(-((x-256)/40)^2)``.
* R-14 Gaussian random field: white N(0,1) from a counter-based hash (so the
  numpy and torch back ends draw the same numbers at any size), periodic
  separable Gaussian smoothing with kernel std ``ell`` voxels truncated at
  ``ceil(4 ell)``, then standardised to mean 0 / std 1.
* R-15 C4: ``mu_a = 0.01 exp(0.5 G)``, Gaussian source (std 3 voxels) at the
  centre.
* R-16 point sources at voxel ``(N/2, N/2, N/2)``.

Arrays are C-ordered ``[z][y][x]`` (x fastest).  ``make`` returns float64 /
complex128 arrays -- numpy on the host, or torch tensors on ``device`` for
sizes that are impractical to synthesise on the host (1024^3).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Any, Dict, Optional, Tuple

import numpy as np

M32 = 0xFFFFFFFF


# --------------------------------------------------------------------------
# array back ends (numpy on host, torch on a device) -- plumbing only
# --------------------------------------------------------------------------
class _Numpy:
    name = "numpy"

    def arange(self, n):
        return np.arange(n, dtype=np.int64)

    def asf(self, a):
        return np.asarray(a, dtype=np.float64)

    def zeros(self, shape, complex_=False):
        return np.zeros(shape, dtype=np.complex128 if complex_ else np.float64)

    def roll(self, a, shift, axis):
        return np.roll(a, shift, axis=axis)

    def exp(self, a):
        return np.exp(a)

    def log(self, a):
        return np.log(a)

    def cos(self, a):
        return np.cos(a)

    def sqrt(self, a):
        return np.sqrt(a)

    def clip(self, a, lo, hi):
        return np.clip(a, lo, hi)

    def maximum(self, a, b):
        return np.maximum(a, b)

    def mean(self, a):
        return float(a.mean())

    def std(self, a):
        return float(a.std())

    def reshape(self, a, shape):
        return a.reshape(shape)

    def to_float(self, a):
        return a.astype(np.float64)

    def complex(self, re, im):
        return re + 1j * im


class _Torch:
    name = "torch"

    def __init__(self, device):
        import torch

        self.t = torch
        self.device = torch.device(device)

    def arange(self, n):
        return self.t.arange(n, dtype=self.t.int64, device=self.device)

    def asf(self, a):
        return self.t.as_tensor(a, dtype=self.t.float64, device=self.device)

    def zeros(self, shape, complex_=False):
        dt = self.t.complex128 if complex_ else self.t.float64
        return self.t.zeros(shape, dtype=dt, device=self.device)

    def roll(self, a, shift, axis):
        return self.t.roll(a, shifts=shift, dims=axis)

    def exp(self, a):
        return self.t.exp(a)

    def log(self, a):
        return self.t.log(a)

    def cos(self, a):
        return self.t.cos(a)

    def sqrt(self, a):
        return self.t.sqrt(a)

    def clip(self, a, lo, hi):
        return self.t.clamp(a, lo, hi)

    def maximum(self, a, b):
        return self.t.maximum(a, b)

    def mean(self, a):
        return float(a.mean())

    def std(self, a):
        return float(a.std(unbiased=False))

    def reshape(self, a, shape):
        return a.reshape(shape)

    def to_float(self, a):
        return a.to(self.t.float64)

    def complex(self, re, im):
        return self.t.complex(re, im)


def _backend(device: Optional[str]):
    if device is None or device == "cpu-numpy" or device == "numpy":
        return _Numpy()
    return _Torch(device)


# --------------------------------------------------------------------------
# counter-based random numbers (identical bits on every back end)
# --------------------------------------------------------------------------
def _mul32(x, m: int):
    """(x * m) mod 2^32 for 0 <= x < 2^32 without int64 overflow."""
    lo, hi = m & 0xFFFF, m >> 16
    return (x * lo + ((x * hi) & 0xFFFF) * 65536) & M32


def _hash32(x):
    """'lowbias32' integer hash (C. Wellons) on int64 arrays holding u32."""
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def _uniform(xp, n: int, seed: int, stream: int):
    """n uniforms in (0,1) for counter i = 0..n-1, keyed by (seed, stream)."""
    idx = xp.arange(n)
    key = int(_hash32(np.int64((seed * 2654435761 + stream * 40503 + 12345) & M32)))
    lo = idx & M32
    hi = idx >> 32
    h = _hash32(lo ^ key)
    h = _hash32(h ^ ((hi * 0x9E37 + 0x79B9) & M32) ^ ((key * 7 + 1) & M32))
    return (xp.to_float(h) + 0.5) * (1.0 / 4294967296.0)


def white_noise(shape: Tuple[int, ...], seed: int, device: Optional[str] = None):
    """Standard normal samples (Box-Muller on two hashed uniform streams)."""
    xp = _backend(device)
    n = int(np.prod(shape))
    u1 = _uniform(xp, n, seed, 0)
    u2 = _uniform(xp, n, seed, 1)
    g = xp.sqrt(-2.0 * xp.log(u1)) * xp.cos((2.0 * math.pi) * u2)
    return xp.reshape(g, shape)


def gaussian_random_field(shape, ell: float, seed: int, device=None):
    """R-14: periodic Gaussian-smoothed white noise, standardised."""
    xp = _backend(device)
    g = white_noise(shape, seed, device)
    rad = int(math.ceil(4.0 * ell))
    taps = np.array([math.exp(-0.5 * (d / ell) ** 2) for d in range(-rad, rad + 1)])
    taps /= taps.sum()
    for axis in range(len(shape)):
        acc = None
        for i, d in enumerate(range(-rad, rad + 1)):
            term = float(taps[i]) * xp.roll(g, d, axis)
            acc = term if acc is None else acc + term
        g = acc
    mu = xp.mean(g)
    sd = xp.std(g)
    return (g - mu) * (1.0 / sd)


# --------------------------------------------------------------------------
# geometry helpers
# --------------------------------------------------------------------------
def absorber_ramp(shape, width: int, device=None):
    """R-9: per-axis linear ramp, max over axes; 0 in the interior."""
    xp = _backend(device)
    nd = len(shape)
    out = None
    for axis, n in enumerate(shape):
        i = np.arange(n, dtype=np.float64)
        r = np.zeros(n)
        if width > 0:
            lo = i < width
            hi = i >= n - width
            r[lo] = (width - i[lo]) / width
            r[hi] = (i[hi] - (n - width) + 1) / width
        view = [1] * nd
        view[axis] = n
        rr = xp.reshape(xp.asf(r), tuple(view))
        out = rr if out is None else xp.maximum(out, rr)
    # broadcast to full shape
    return out + xp.zeros(shape)


def _k2_from_index(xp, n_re, n_im, k0: float):
    """k^2 = (k0 n)^2 for complex n = n_re + i n_im (Eq. 8's k(r))."""
    re = (k0 * k0) * (n_re * n_re - n_im * n_im)
    im = (k0 * k0) * (2.0 * n_re * n_im)
    return xp.complex(re, im)


# --------------------------------------------------------------------------
# configs
# --------------------------------------------------------------------------
@dataclass
class Problem:
    """A physical problem in the unified form of DESIGN.md (reading R-1):

    Helmholtz (Eq. 8):  lap psi + k^2 psi = -S    -> medium = k^2
    Diffusion (§3.2, stationary, scalar D):
                                 -D lap u + mu_a u = S    -> medium = mu_a
    """

    name: str
    kind: str                      # "helmholtz" | "diffusion"
    shape: Tuple[int, ...]         # C order, x last
    medium: Any                    # k^2 (complex128) or mu_a (float64)
    source: Any                    # S (complex128 for helmholtz, float64 for diffusion)
    D: float = 1.0
    h: Tuple[float, ...] = ()
    alpha: float = 0.75
    tol: float = 0.0               # 0 -> run exactly n_iter
    n_iter: int = 100              # max iterations (tol>0) or exact count (tol=0)
    meta: Dict[str, Any] = field(default_factory=dict)

    @property
    def n_vox(self) -> int:
        return int(np.prod(self.shape))


CONFIGS = {
    # name: (BASELINE.json configs index, default shape)
    "C1": (0, (256,)),
    "C2": (1, (512, 512)),
    "C3": (2, (256, 256, 256)),
    "C4": (3, (512, 512, 512)),
    "C5": (4, (1024, 1024, 1024)),
    "C5w": (4, (2048, 1024, 1024)),
}


def config_names():
    return list(CONFIGS)


def _c1(shape, device):
    xp = _backend(device)
    (n,) = shape
    lam, width = 8.0, max(1, round(32 * n / 256))
    k0 = 2.0 * math.pi / lam
    n_re = np.ones(n)
    n_im = np.zeros(n)
    s0, s1 = (3 * n) // 8, (5 * n) // 8
    n_re[s0:s1] = 1.5
    n_im[s0:s1] = 0.01
    n_im = n_im + 0.2 * np.asarray(_to_np(absorber_ramp(shape, width)))
    k2 = _k2_from_index(xp, xp.asf(n_re), xp.asf(n_im), k0)
    src = xp.zeros(shape, complex_=True)
    src[n // 4] = 1.0
    return Problem("C1", "helmholtz", shape, k2, src, alpha=0.75, tol=1e-6, n_iter=2000,
                   meta=dict(wavelength=lam, absorber=width, slab=(s0, s1), src=n // 4))


def _c2(shape, device, seed=2):
    xp = _backend(device)
    ny, nx = shape
    s = nx / 512.0
    lam, width = 8.0, max(1, round(32 * s))
    k0 = 2.0 * math.pi / lam
    rng = np.random.Generator(np.random.PCG64(seed))
    n_re = np.ones(shape)
    jj, ii = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    n_disks = max(1, round(200 * s * s))
    disks = []
    for _ in range(n_disks):
        cx = rng.uniform(width, nx - width)
        cy = rng.uniform(width, ny - width)
        r = rng.uniform(4.0 * s, 16.0 * s)
        nd = rng.uniform(1.0, 1.5)
        inside = (ii - cx) ** 2 + (jj - cy) ** 2 <= r * r
        n_re[inside] = nd
        disks.append((cx, cy, r, nd))
    n_im = 0.2 * np.asarray(_to_np(absorber_ramp(shape, width)))
    k2 = _k2_from_index(xp, xp.asf(n_re), xp.asf(n_im), k0)
    src_np = np.zeros(shape, dtype=np.complex128)
    y0 = int(round(48 * s))
    x = np.arange(nx, dtype=np.float64)
    src_np[y0, :] = np.exp(-(((x - nx / 2) / (40.0 * s)) ** 2))
    if xp.name == "numpy":
        src = src_np
    else:
        src = xp.complex(xp.asf(src_np.real), xp.asf(src_np.imag))
    return Problem("C2", "helmholtz", shape, k2, src, alpha=0.75, tol=1e-6, n_iter=20000,
                   meta=dict(wavelength=lam, absorber=width, n_disks=n_disks, src_row=y0,
                             fill=float((n_re > 1.0).mean())))


def _helmholtz_grf(name, shape, device, lam, width, ell, seed, n_iter):
    xp = _backend(device)
    k0 = 2.0 * math.pi / lam
    g = gaussian_random_field(shape, ell, seed, device)
    n_re = 1.33 + 0.12 * xp.clip(g, 0.0, 1.0)
    del g
    n_im = 0.2 * absorber_ramp(shape, width, device)
    k2 = _k2_from_index(xp, n_re, n_im, k0)
    del n_re, n_im
    src = xp.zeros(shape, complex_=True)
    c = tuple(n // 2 for n in shape)
    src[c] = 1.0
    return Problem(name, "helmholtz", tuple(shape), k2, src, alpha=0.75, tol=0.0, n_iter=n_iter,
                   meta=dict(wavelength=lam, absorber=width, ell=ell, seed=seed, src=c))


def _c4(shape, device, seed=4):
    xp = _backend(device)
    g = gaussian_random_field(shape, 8.0, seed, device)
    mu = 0.01 * xp.exp(0.5 * g)
    del g
    nd = len(shape)
    out = None
    for axis, n in enumerate(shape):
        r = (np.arange(n, dtype=np.float64) - n // 2) ** 2
        view = [1] * nd
        view[axis] = n
        rr = xp.reshape(xp.asf(r), tuple(view))
        out = rr if out is None else out + rr
    src = xp.exp(out * (-1.0 / (2.0 * 9.0))) + xp.zeros(shape)
    return Problem("C4", "diffusion", tuple(shape), mu, src, D=1.0, alpha=0.75, tol=0.0,
                   n_iter=200, meta=dict(ell=8.0, seed=seed, src_sigma=3.0))


def _to_np(a):
    if isinstance(a, np.ndarray):
        return a
    return a.detach().cpu().numpy()


def make(name: str, shape: Optional[Tuple[int, ...]] = None, device: Optional[str] = None,
         **over) -> Problem:
    """Build config ``name`` (C1..C5, C5w) at ``shape`` (default: BASELINE size).

    Smaller shapes keep the wavelength and correlation length (in voxels) and
    scale the absorber width / geometry with the grid, so a "mini" instance is
    the same recipe on a smaller box (a parity-test case, not a bench line).
    ``device=None`` -> numpy on the host; ``device='cuda'`` -> torch tensors.
    """
    if name not in CONFIGS:
        raise KeyError(f"unknown config {name!r}; have {config_names()}")
    shape = tuple(shape) if shape is not None else CONFIGS[name][1]
    if name == "C1":
        p = _c1(shape, device)
    elif name == "C2":
        p = _c2(shape, device)
    elif name == "C3":
        w = max(1, round(16 * shape[-1] / 256))
        p = _helmholtz_grf("C3", shape, device, 6.0, w, 4.0, 3, 500)
    elif name in ("C5", "C5w"):
        w = max(1, round(32 * shape[-1] / 1024))
        p = _helmholtz_grf(name, shape, device, 8.0, w, 4.0, 3, 100)
    elif name == "C4":
        p = _c4(shape, device)
    else:  # pragma: no cover
        raise KeyError(name)
    p.h = tuple(1.0 for _ in shape)
    for k, v in over.items():
        setattr(p, k, v)
    return p


def homogeneous(shape, k0: float = 2 * math.pi / 8, n: complex = 1.0 + 0.05j, device=None,
                src_at=None) -> Problem:
    """Homogeneous medium (constant k^2) with a unit point source: the input of
    the closed-form pin (constant V) of DESIGN.md §Oracle pins."""
    xp = _backend(device)
    k2c = (k0 * n) ** 2
    k2 = xp.zeros(shape, complex_=True) + complex(k2c)
    src = xp.zeros(shape, complex_=True)
    c = tuple(s // 2 for s in shape) if src_at is None else src_at
    src[c] = 1.0
    return Problem("homog", "helmholtz", tuple(shape), k2, src, alpha=0.75, tol=0.0, n_iter=50,
                   h=tuple(1.0 for _ in shape), meta=dict(k0=k0, n=n, src=c))
