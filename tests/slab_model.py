"""CPU model of the slab decomposition's data movement (test infrastructure).

It runs the Delta-form iteration of Algorithm 1 in
float64 on P torch.distributed ranks (gloo), with exactly the layouts and
exchanges include/usp.h documents for the multi-GPU path:

  rank r holds z-slab r ([nz/P][ny][nx]) of x, Delta, B;
  x FFT, y FFT on the slab; rows y of plane z go to block q = y // (ny/P) of
  the SEND layout [q][z_loc][y_loc][x]; all-to-all -> RECEIVE layout
  [q][z_loc][y_loc][x] == [z][y_loc][x] (the y-slab r); z FFT, multiplier with
  GLOBAL y = r*ny/P + y_loc, inverse z FFT; all-to-all back; inverse y FFT
  reading the send layout; inverse x FFT; update; residual = all-gather of
  the P local sums, summed in rank order.

The per-axis transforms are numpy FFTs (this checks the decomposition, not
the kernels: the kernels' parity is the GPU suite's job).
"""
from __future__ import annotations

import numpy as np


def to_send_layout(a_slab, P):
    """[z_loc][y][x] -> [q][z_loc][y_loc][x] (block q = y rows q*ny/P ...)."""
    nzl, ny, nx = a_slab.shape
    return np.ascontiguousarray(a_slab.reshape(nzl, P, ny // P, nx).transpose(1, 0, 2, 3))


def from_send_layout(buf, P):
    """inverse of to_send_layout"""
    _, nzl, nyl, nx = buf.shape
    return np.ascontiguousarray(buf.transpose(1, 0, 2, 3).reshape(nzl, P * nyl, nx))


def alltoall(buf, P):
    """buf [q][...]: block q goes to rank q; returns the blocks received,
    indexed by source rank."""
    import torch
    import torch.distributed as dist

    src = torch.from_numpy(np.ascontiguousarray(buf)).view(torch.float64)
    dst = torch.empty_like(src)
    dist.all_to_all_single(dst, src)
    return dst.view(torch.complex128).numpy().reshape(buf.shape)


def allgather_sum(v, P):
    import torch
    import torch.distributed as dist

    out = [torch.zeros(1, dtype=torch.float64) for _ in range(P)]
    dist.all_gather(out, torch.tensor([v], dtype=torch.float64))
    total = 0.0
    for t in out:              # rank order
        total += float(t[0])
    return total


def apply_Linv_slab(u_slab, P, r, shape, h, D, sigma, c):
    """(L+1)^-1 u (Eq. 12) on the rank's z-slab, through the two transposes."""
    nz, ny, nx = shape
    nyl = ny // P
    a = np.fft.fft(np.fft.fft(u_slab, axis=2), axis=1)
    recv = alltoall(to_send_layout(a, P), P)            # [q][z_loc][y_loc][x]
    ys = recv.reshape(nz, nyl, nx)                       # y-slab r: [z][y_loc][x]
    ys = np.fft.fft(ys, axis=0)
    pz = 2 * np.pi * np.fft.fftfreq(nz, h[0])
    py = 2 * np.pi * np.fft.fftfreq(ny, h[1])[r * nyl:(r + 1) * nyl]
    px = 2 * np.pi * np.fft.fftfreq(nx, h[2])
    p2 = pz[:, None, None] ** 2 + py[None, :, None] ** 2 + px[None, None, :] ** 2
    ys = np.fft.ifft(ys * (c / (D * p2 + sigma + c)), axis=0)
    back = alltoall(ys.reshape(P, nz // P, nyl, nx), P)  # [q][z_loc][y_loc][x] of slab r
    b = from_send_layout(back, P)
    return np.fft.ifft(np.fft.ifft(b, axis=1), axis=2)


def delta_form_slab(w_slab, S_slab, P, r, shape, h, D, sigma, c, alpha, n_iter):
    """n_iter Delta-form iterations (L613) on the rank's slab; returns
    (x_slab, residual history r_0..r_n)."""
    V = (w_slab - sigma) / c
    B = 1.0 - V
    s = S_slab / c
    d = B * apply_Linv_slab(s, P, r, shape, h, D, sigma, c)
    n0 = np.sqrt(allgather_sum(float(np.sum(np.abs(d) ** 2)), P))
    x = np.zeros_like(d)
    hist = [1.0]
    for _ in range(n_iter):
        y = apply_Linv_slab(B * d, P, r, shape, h, D, sigma, c)
        x = x + alpha * d
        d = d + alpha * B * (y - d)
        hist.append(np.sqrt(allgather_sum(float(np.sum(np.abs(d) ** 2)), P)) / n0)
    return x, np.array(hist)
