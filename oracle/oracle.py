"""Python face of the CPU oracle (``usp_oracle.c``).

TEST INFRASTRUCTURE ONLY -- only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this.
It imports nothing from the CUDA product (``paper_2207_14222_b200``) and the
product imports nothing from here.

What it computes (PAPER.md = /root/reference/PAPER.md):

* ``fftn`` / ``ifftn``             -- the DFT the method's F denotes (L171).
* ``apply_Linv``                   -- (L+1)^-1 via Eq. 12 (L168-172).
* ``canonical``                    -- §2.2 / §3.1 canonical form: smallest
  enclosing circle of the medium values (L167) -> bias; scale c so that
  max|V| = target_norm (L99, L167).
* ``fixed_point``                  -- Algorithm 1 (L80-89), x-form, or the
  Delta-form recurrence (L613) for the R-17 cross-check.
* ``canonical_anti``, ``fixed_point_anti`` -- the antisymmetrised system of
  Eq. 9-10 (L100-128) for problems that are not accretive.
* ``canonical_tdiff``, ``fixed_point_tdiff`` -- the first-order (u, F)
  form of tensor-D steady diffusion, §3.2 Eqs. 16-18 (L199-227).
* ``gmres``                        -- restarted GMRES(m) on the same system
  (Table 1b's GMRES5 / GMRES20 columns).
* ``bicgstab``                     -- BiCGSTAB on the preconditioned system
  Gamma^-1 A x = Gamma^-1 s, Eq. 5 (L73-76) -- Table 1b's BiCGSTAB column.

Pins: see tests/test_oracle_*.py.  Parity status per function is listed in
DESIGN.md ("Oracle and its pins"); every function here is pinned.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "usp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C11 + OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", _SRC, "-o", _LIB, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        lp = ctypes.POINTER(ctypes.c_long)
        L.orc_fft1d.argtypes = [dp, ctypes.c_long, ctypes.c_int]
        L.orc_fftn.argtypes = [dp, ctypes.c_int, lp, ctypes.c_int]
        L.orc_apply_Linv.argtypes = [dp, ctypes.c_int, lp, dp, ctypes.c_double] + [ctypes.c_double] * 4
        L.orc_setup.argtypes = [dp, dp, ctypes.c_long] + [ctypes.c_double] * 4 + [dp, dp, dp]
        L.orc_fixed_point.argtypes = ([dp, dp, ctypes.c_int, lp, dp, ctypes.c_double]
                                      + [ctypes.c_double] * 4
                                      + [ctypes.c_double, ctypes.c_double, ctypes.c_long, ctypes.c_int,
                                         dp, dp, lp, dp])
        L.orc_mec.argtypes = [dp, dp, ctypes.c_long, dp, dp, dp]
        L.orc_fixed_point_anti.argtypes = ([dp, dp, ctypes.c_int, lp, dp, ctypes.c_double] + [ctypes.c_double] * 3
                                           + [ctypes.c_double, ctypes.c_double, ctypes.c_long, dp, dp, lp, dp])
        L.orc_fixed_point_tdiff.argtypes = ([dp, dp, dp, ctypes.c_int, lp, dp, ctypes.c_double, dp]
                                            + [ctypes.c_double] * 5 + [ctypes.c_long, dp, dp, lp, dp])
        L.orc_gmres.argtypes = ([dp, dp, ctypes.c_int, lp, dp, ctypes.c_double] + [ctypes.c_double] * 4
                                + [ctypes.c_int, ctypes.c_double, ctypes.c_long, dp, dp, lp, dp])
        L.orc_bicgstab.argtypes = ([dp, dp, ctypes.c_int, lp, dp, ctypes.c_double] + [ctypes.c_double] * 4
                                   + [ctypes.c_double, ctypes.c_long, dp, dp, lp, dp,
                                      ctypes.POINTER(ctypes.c_int)])
        L.orc_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _dims(shape: Sequence[int]):
    arr = (ctypes.c_long * len(shape))(*shape)
    return arr


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.complex128)


def num_threads() -> int:
    return int(lib().orc_num_threads())


# ------------------------------------------------------------------- DFT --
def fft1d(a, inverse: bool = False) -> np.ndarray:
    x = _c128(a).copy()
    rc = lib().orc_fft1d(_dp(x.view(np.float64)), x.size, int(inverse))
    if rc:
        raise ValueError(f"orc_fft1d rc={rc}")
    return x


def fftn(a, inverse: bool = False) -> np.ndarray:
    x = _c128(a).copy()
    rc = lib().orc_fftn(_dp(x.view(np.float64)), x.ndim, _dims(x.shape), int(inverse))
    if rc:
        raise ValueError(f"orc_fftn rc={rc}")
    return x


def ifftn(a) -> np.ndarray:
    return fftn(a, inverse=True)


# ------------------------------------------------------------- operators --
@dataclass
class Split:
    """Canonical-form parameters in the unified reading R-1."""

    D: float
    sigma: complex
    c: complex
    bias: complex          # centre of the smallest enclosing circle of the medium
    radius: float


def apply_Linv(u, h: Sequence[float], D: float, sigma: complex, c: complex) -> np.ndarray:
    x = _c128(u).copy()
    hh = np.ascontiguousarray(h, dtype=np.float64)
    rc = lib().orc_apply_Linv(_dp(x.view(np.float64)), x.ndim, _dims(x.shape), _dp(hh), float(D),
                              float(np.real(sigma)), float(np.imag(sigma)), float(np.real(c)),
                              float(np.imag(c)))
    if rc:
        raise ValueError(f"orc_apply_Linv rc={rc}")
    return x


def setup(w, S, sigma: complex, c: complex):
    """V, B, s of the canonical system."""
    wc, Sc = _c128(w), _c128(S)
    V = np.empty_like(wc)
    B = np.empty_like(wc)
    s = np.empty_like(wc)
    lib().orc_setup(_dp(wc.view(np.float64)), _dp(Sc.view(np.float64)), wc.size,
                    float(np.real(sigma)), float(np.imag(sigma)), float(np.real(c)), float(np.imag(c)),
                    _dp(V.view(np.float64)), _dp(B.view(np.float64)), _dp(s.view(np.float64)))
    return V, B, s


def mec(points) -> Tuple[complex, float]:
    """Smallest enclosing circle of complex points."""
    p = np.asarray(points).ravel()
    re = np.ascontiguousarray(np.real(p), dtype=np.float64)
    im = np.ascontiguousarray(np.imag(p), dtype=np.float64)
    cr, ci, r = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    rc = lib().orc_mec(_dp(re), _dp(im), re.size, ctypes.byref(cr), ctypes.byref(ci), ctypes.byref(r))
    if rc:
        raise ValueError(f"orc_mec rc={rc}")
    return complex(cr.value, ci.value), float(r.value)


def medium_to_w(kind: str, medium) -> np.ndarray:
    """w(r) of the unified form: Helmholtz w = -k^2 (Eq. 8 times -1), diffusion w = mu_a."""
    m = _c128(medium)
    return -m if kind == "helmholtz" else m


def real_bias_circle(points) -> Tuple[float, float]:
    """Smallest circle CENTRED ON THE REAL AXIS enclosing the points: the
    real bias of the earlier convergent-Born-series work the paper compares
    against (Table 1b's "R bias" rows).  f(t) = max_i
    |z_i - t| is convex in t; golden-section search to machine precision."""
    z = _c128(points).ravel()
    f = lambda t: float(np.max(np.abs(z - t)))
    lo, hi = float(z.real.min()), float(z.real.max())
    g = (math.sqrt(5.0) - 1.0) / 2.0
    a, b = lo, hi
    for _ in range(200):
        c1, c2 = b - g * (b - a), a + g * (b - a)
        if f(c1) <= f(c2):
            b = c2
        else:
            a = c1
    t = 0.5 * (a + b)
    return t, f(t)


def canonical(kind: str, medium, target_norm: float = 0.95, D: float = 1.0, real_bias: bool = False) -> Split:
    """Canonical form of §2.2 / §3.1.

    Helmholtz: kbar^2 = centre of the smallest circle enclosing the k^2 values,
    c_paper = -(1/(0.95 i)) r = i r / 0.95 (L167); in the unified form
    sigma = -kbar^2, c = -c_paper.  Diffusion (§3.2 scalar, reading R-15):
    mu0 = centre (mid-range) of mu_a, c = r / 0.95 (real, so A stays accretive).
    real_bias: the centre is restricted to the real axis (the prior real-bias
    choice the paper improves on, L174, L396).
    """
    if real_bias:
        t, r = real_bias_circle(_c128(medium))
        centre = complex(t)
    else:
        centre, r = mec(_c128(medium))
    if r == 0.0:
        raise ValueError("homogeneous medium: smallest circle has radius 0; pass sigma, c explicitly")
    if kind == "helmholtz":
        c_paper = -(1.0 / (target_norm * 1j)) * r
        return Split(D=D, sigma=-centre, c=-c_paper, bias=centre, radius=r)
    if kind == "diffusion":
        return Split(D=D, sigma=centre, c=complex(r / target_norm), bias=centre, radius=r)
    raise ValueError(kind)


@dataclass
class Result:
    x: np.ndarray
    n_done: int
    hist: np.ndarray
    n0: float
    rc: int


def fixed_point(w, S, h: Sequence[float], D: float, sigma: complex, c: complex, alpha: float,
                tol: float, n_max: int, form: str = "x") -> Result:
    """Algorithm 1; ``form='delta'`` runs the Neumann
    recurrence of L613 instead (same iterates in exact arithmetic)."""
    wc, Sc = _c128(w), _c128(S)
    if wc.shape != Sc.shape:
        raise ValueError("w and S shapes differ")
    x = np.zeros_like(wc)
    hist = np.zeros(n_max, dtype=np.float64)
    hh = np.ascontiguousarray(h, dtype=np.float64)
    nd = ctypes.c_long(0)
    n0 = ctypes.c_double(0.0)
    rc = lib().orc_fixed_point(_dp(wc.view(np.float64)), _dp(Sc.view(np.float64)), wc.ndim,
                               _dims(wc.shape), _dp(hh), float(D), float(np.real(sigma)),
                               float(np.imag(sigma)), float(np.real(c)), float(np.imag(c)),
                               float(alpha), float(tol), int(n_max), 0 if form == "x" else 1,
                               _dp(x.view(np.float64)), _dp(hist), ctypes.byref(nd), ctypes.byref(n0))
    if rc < 0:
        raise ValueError(f"orc_fixed_point rc={rc}")
    return Result(x=x, n_done=int(nd.value), hist=hist[: nd.value].copy(), n0=float(n0.value), rc=rc)


def canonical_anti(kind: str, medium, target_norm: float = 0.95, D: float = 1.0) -> Split:
    """Canonical form of the antisymmetrised system (Eq. 9-10, PAPER.md
    L100-128): bias = smallest-circle centre of w (as the standard form),
    REAL scale c = r / target_norm so that ||V|| = max|V_raw| / c = target_norm."""
    w = medium_to_w(kind, medium)
    centre, r = mec(w)
    if r == 0.0:
        raise ValueError("homogeneous medium: smallest circle has radius 0")
    return Split(D=D, sigma=centre, c=complex(r / target_norm), bias=centre, radius=r)


def fixed_point_anti(w, S, h: Sequence[float], D: float, sigma: complex, c: float, alpha: float, tol: float,
                     n_max: int) -> Result:
    """Algorithm 1 on the antisymmetrised system (usp_oracle.c); x has shape
    (2, *S.shape): [x, x'] (x solves A_raw x = S; x' -> 0 for s' = 0)."""
    wc, Sc = _c128(w), _c128(S)
    x = np.zeros((2,) + wc.shape, dtype=np.complex128)
    hist = np.zeros(n_max, dtype=np.float64)
    hh = np.ascontiguousarray(h, dtype=np.float64)
    nd, n0 = ctypes.c_long(0), ctypes.c_double(0.0)
    rc = lib().orc_fixed_point_anti(_dp(wc.view(np.float64)), _dp(Sc.view(np.float64)), wc.ndim, _dims(wc.shape),
                                    _dp(hh), float(D), float(np.real(sigma)), float(np.imag(sigma)),
                                    float(np.real(c)), float(alpha), float(tol), int(n_max),
                                    _dp(x.view(np.float64)), _dp(hist), ctypes.byref(nd), ctypes.byref(n0))
    if rc < 0:
        raise ValueError(f"orc_fixed_point_anti rc={rc}")
    return Result(x=x, n_done=int(nd.value), hist=hist[: nd.value].copy(), n0=float(n0.value), rc=rc)


@dataclass
class TdiffSplit:
    """Canonical form of the first-order tensor-diffusion system (reading R-29)."""

    mubar: float
    dbar: np.ndarray      # packed symmetric Dbar^-1 (2-D: xx, xy, yy; 3-D: xx, xy, xz, yy, yz, zz)
    s_u: float
    s_F: float
    c: float


def _sym_pack_index(d):
    return [(0, 0), (0, 1), (1, 1)] if d == 2 else [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]


def dinv_field(D):
    """Per-voxel inverse of the symmetric tensor field D[..., d, d], packed."""
    Dinv = np.linalg.inv(np.asarray(D, dtype=np.float64))
    d = Dinv.shape[-1]
    return np.stack([Dinv[..., i, j] for i, j in _sym_pack_index(d)], axis=-1)


def canonical_tdiff(mu, D, target_norm: float = 0.95) -> TdiffSplit:
    """§3.2 (L222-225): the centre of the smallest circle of every element of
    V_raw goes into L (for real values: the mid-range) -> mubar, Dbar^-1;
    the radii are equilibrated by S = diag(s_u, s_F, ..) with s_u = radius of
    mu and s_F = the largest radius of the D^-1 elements (reading R-29 of the
    paper's [duff2001] equilibration); finally c = max_r ||V(r)||_F-bound /
    target_norm, using max(|mu - mubar|/s_u, ||D^-1 - Dbar^-1||_F / s_F)."""
    mu = np.asarray(mu, dtype=np.float64)
    dpk = dinv_field(D)
    d = np.asarray(D).shape[-1]
    mubar = 0.5 * (mu.max() + mu.min())
    r_mu = 0.5 * (mu.max() - mu.min())
    lo, hi = dpk.reshape(-1, dpk.shape[-1]).min(axis=0), dpk.reshape(-1, dpk.shape[-1]).max(axis=0)
    dbar = 0.5 * (hi + lo)
    r_d = 0.5 * (hi - lo)
    s_u = r_mu if r_mu > 0 else 1.0
    s_F = r_d.max() if r_d.max() > 0 else 1.0
    diff = (dpk - dbar) / s_F
    w = np.ones(dpk.shape[-1])
    for k, (i, j) in enumerate(_sym_pack_index(d)):
        w[k] = 1.0 if i == j else 2.0          # off-diagonal elements appear twice in ||.||_F
    fro = np.sqrt(np.sum(w * diff ** 2, axis=-1))
    vmax = max(np.abs(mu - mubar).max() / s_u, fro.max())
    return TdiffSplit(mubar=float(mubar), dbar=dbar.astype(np.float64), s_u=float(s_u), s_F=float(s_F),
                      c=float(vmax / target_norm))


def fixed_point_tdiff(mu, D, S, h: Sequence[float], split: TdiffSplit, alpha: float, tol: float,
                      n_max: int) -> Result:
    """Algorithm 1 on the first-order (u, F) system of §3.2 (Eqs. 16-18).
    Returns Result with x = E [(d+1), *shape] (E[0] = sqrt(s_u) u)."""
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    dpk = np.ascontiguousarray(dinv_field(D), dtype=np.float64)
    Sr = np.ascontiguousarray(np.real(S), dtype=np.float64)
    d = mu.ndim
    E = np.zeros((d + 1,) + mu.shape, dtype=np.complex128)
    hist = np.zeros(n_max, dtype=np.float64)
    hh = np.ascontiguousarray(h, dtype=np.float64)
    nd, n0 = ctypes.c_long(0), ctypes.c_double(0.0)
    db = np.ascontiguousarray(split.dbar, dtype=np.float64)
    rc = lib().orc_fixed_point_tdiff(_dp(mu), _dp(dpk), _dp(Sr), d, _dims(mu.shape), _dp(hh), split.mubar, _dp(db),
                                     split.s_u, split.s_F, split.c, float(alpha), float(tol), int(n_max),
                                     _dp(E.view(np.float64)), _dp(hist), ctypes.byref(nd), ctypes.byref(n0))
    if rc < 0:
        raise ValueError(f"orc_fixed_point_tdiff rc={rc}")
    return Result(x=E, n_done=int(nd.value), hist=hist[: nd.value].copy(), n0=float(n0.value), rc=rc)


@dataclass
class KrylovResult:
    x: np.ndarray
    n_done: int          # BiCGSTAB loop passes (two applications of M each)
    half: bool           # stopped after the half step (||s|| < tol)
    hist: np.ndarray     # [||s_0||, ||r_1||, ||s_1||, ...] / ||b||
    nb: float            # ||b|| = ||B (L+1)^-1 s||
    rc: int


def bicgstab(w, S, h: Sequence[float], D: float, sigma: complex, c: complex, tol: float,
             n_max: int) -> KrylovResult:
    """BiCGSTAB on M x = b with M = B[1 - (L+1)^-1 B] (Eq. 5 with alpha = 1,
    reading R-25), b = B (L+1)^-1 s, x_0 = 0 (see usp_oracle.c)."""
    wc, Sc = _c128(w), _c128(S)
    x = np.zeros_like(wc)
    hist = np.zeros(2 * n_max, dtype=np.float64)
    hh = np.ascontiguousarray(h, dtype=np.float64)
    nd, nb, half = ctypes.c_long(0), ctypes.c_double(0.0), ctypes.c_int(0)
    rc = lib().orc_bicgstab(_dp(wc.view(np.float64)), _dp(Sc.view(np.float64)), wc.ndim, _dims(wc.shape),
                            _dp(hh), float(D), float(np.real(sigma)), float(np.imag(sigma)),
                            float(np.real(c)), float(np.imag(c)), float(tol), int(n_max),
                            _dp(x.view(np.float64)), _dp(hist), ctypes.byref(nd), ctypes.byref(nb),
                            ctypes.byref(half))
    if rc < 0:
        raise ValueError(f"orc_bicgstab rc={rc}")
    k = int(nd.value)
    nh = 2 * k - 1 if half.value else 2 * k
    return KrylovResult(x=x, n_done=k, half=bool(half.value), hist=hist[:nh].copy(), nb=float(nb.value), rc=rc)


def gmres(w, S, h: Sequence[float], D: float, sigma: complex, c: complex, m: int, tol: float,
          n_max: int) -> KrylovResult:
    """Restarted GMRES(m) on M x = b (same system as bicgstab; reading R-28).
    n_done counts Arnoldi steps; hist[k-1] = residual estimate after step k."""
    wc, Sc = _c128(w), _c128(S)
    x = np.zeros_like(wc)
    hist = np.zeros(n_max, dtype=np.float64)
    hh = np.ascontiguousarray(h, dtype=np.float64)
    nd, nb = ctypes.c_long(0), ctypes.c_double(0.0)
    rc = lib().orc_gmres(_dp(wc.view(np.float64)), _dp(Sc.view(np.float64)), wc.ndim, _dims(wc.shape), _dp(hh),
                         float(D), float(np.real(sigma)), float(np.imag(sigma)), float(np.real(c)),
                         float(np.imag(c)), int(m), float(tol), int(n_max), _dp(x.view(np.float64)), _dp(hist),
                         ctypes.byref(nd), ctypes.byref(nb))
    if rc < 0:
        raise ValueError(f"orc_gmres rc={rc}")
    k = int(nd.value)
    return KrylovResult(x=x, n_done=k, half=False, hist=hist[:k].copy(), nb=float(nb.value), rc=rc)


def solve_problem(p, target_norm: float = 0.95, form: str = "x", n_iter: Optional[int] = None,
                  tol: Optional[float] = None, alpha: Optional[float] = None, split: Optional[Split] = None,
                  medium=None):
    """Convenience: canonical form + Algorithm 1 for a ``synth`` Problem.
    ``medium`` may override p.medium (e.g. the complex64-rounded values the
    GPU receives, so both sides see identical inputs)."""
    med = p.medium if medium is None else medium
    med = np.asarray(med)
    sp = split if split is not None else canonical(p.kind, med, target_norm, D=p.D)
    w = medium_to_w(p.kind, med)
    res = fixed_point(w, np.asarray(p.source), p.h, sp.D, sp.sigma, sp.c,
                      p.alpha if alpha is None else alpha,
                      p.tol if tol is None else tol,
                      p.n_iter if n_iter is None else n_iter, form=form)
    return sp, res
