"""Dense reference operators for tiny grids (test-side pins of the oracle).

Independent of the oracle's FFT: the periodic spectral second-derivative
matrix is written from its closed form (Trefethen, *Spectral Methods in
MATLAB*, SIAM 2000, ch. 3, Eq. 3.12 for the 2 pi-periodic grid with N even):

    S''(0)    = -pi^2 / (3 h^2) - 1/6
    S''(x_j)  = -(-1)^j / (2 sin^2(j h / 2)),   j != 0,   h = 2 pi / N

rescaled to a grid of spacing ``dx`` (period N dx).  Its symbol is -m^2 for
|m| < N/2 and -(N/2)^2 at the Nyquist mode, which is the reading R-7 of
DESIGN.md (|p|^2 with p = 2 pi m / (N dx)).
"""
import numpy as np


def d2_periodic(n: int, dx: float = 1.0) -> np.ndarray:
    """Dense periodic spectral second-derivative matrix (N even or N = 1, 2)."""
    if n == 1:
        return np.zeros((1, 1))
    h = 2 * np.pi / n
    col = np.empty(n)
    col[0] = -np.pi ** 2 / (3 * h ** 2) - 1.0 / 6.0
    j = np.arange(1, n)
    col[1:] = -((-1.0) ** j) / (2 * np.sin(j * h / 2) ** 2)
    idx = (np.arange(n)[:, None] - np.arange(n)[None, :]) % n
    D2 = col[idx]
    # rescale from period 2 pi to period n * dx
    return D2 * (2 * np.pi / (n * dx)) ** 2


def neg_laplacian(shape, h=None) -> np.ndarray:
    """Dense -lap on a C-ordered grid (x = last axis) as a Kronecker sum."""
    nd = len(shape)
    h = h or [1.0] * nd
    N = int(np.prod(shape))
    K = np.zeros((N, N))
    for a in range(nd):
        mats = [np.eye(s) for s in shape]
        mats[a] = -d2_periodic(shape[a], h[a])
        M = mats[0]
        for m in mats[1:]:
            M = np.kron(M, m)
        K += M
    return K


def dense_A(shape, w, D, c, h=None) -> np.ndarray:
    """A = (1/c)(-D lap + diag(w))   (unified reading R-1)."""
    K = neg_laplacian(shape, h)
    return (D * K + np.diag(np.asarray(w).ravel())) / c


def dense_L1(shape, sigma, D, c, h=None) -> np.ndarray:
    """L + 1 = (1/c)(-D lap + sigma) + 1."""
    K = neg_laplacian(shape, h)
    N = K.shape[0]
    return (D * K + sigma * np.eye(N)) / c + np.eye(N)


def re_part(X: np.ndarray) -> float:
    """Re[X] of PAPER.md Eq. 1: inf over x of Re<x,Xx>/<x,x> = min eig of the
    Hermitian part."""
    H = 0.5 * (X + X.conj().T)
    return float(np.linalg.eigvalsh(H).min())
