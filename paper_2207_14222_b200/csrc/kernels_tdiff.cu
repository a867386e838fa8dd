// kernels_tdiff.cu -- first-order tensor-diffusion system (SURVEY.md §8(f)
// NEXT-3; §3.2 Eqs. 16-18; reading R-29):
//
//     mu u + div F = S,   D^-1 F + grad u = 0   ->   A_raw [u; F] = [S; 0]
//     E = S^1/2 [u; F],  s = c^-1 S^-1/2 [S; 0],  S = diag(s_u, s_F, .., s_F)
//     V = c^-1 S^-1/2 [[mu - mubar, 0], [0, D^-1 - Dbar^-1]] S^-1/2   (per voxel, block-diagonal)
//     (L+1)^-1 per mode: [[a, i q^T], [i q, Dm]]^-1 by its Schur complement
//         w = Dm^-1 q,  sig = a + q^T w,  out_u = (u - i w.F)/sig,  out_F = Dm^-1 F - i w out_u
//
// d + 1 complex components, stored component-major; the y / z FFTs are the
// k_stile passes over (d + 1) x the planes, the x FFT a plain line kernel,
// and the coupling lives in three elementwise kernels:
//   k_tdiff_pot  D -> D^-1 per voxel, min/max reductions for the canonical
//                form, then (second mode) v_u, V_F per voxel and max |V|
//   k_tdiff_mul  the per-mode Schur-complement symbol (with 1/N_vox)
//   k_tdiff_upd  Delta <- Delta + alpha B (y - Delta), x <- x + alpha Delta,
//                residual, work <- B Delta (the next chain's input)
// Capability path (register-staged, no TMA): the (d + 1)-fold fields make it
// ~4x the bytes of the scalar path per voxel.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fft_core.cuh"
#include "kcommon.cuh"
#include "usp_internal.h"

namespace usp {

// ------------------------------------------------------- plain x FFT pass --
template <int N, bool INV>
__global__ void __launch_bounds__(128) k_xfft(float2 *data, const float2 *__restrict__ tw, long long nlines) {
    using G = LineGeo<N>;
    extern __shared__ float2 smem_x[];
    constexpr int LPC = 128 / G::N1;
    const int tid = threadIdx.x, lq = tid / G::N1, j = tid % G::N1;
    const LayRow<N> lay{smem_x + lq * LayRow<N>::kFloat2PerLine};
    const long long ng = (nlines + LPC - 1) / LPC;
    for (long long g = blockIdx.x; g < ng; g += gridDim.x) {
        const long long line = g * LPC + lq;
        const bool valid = line < nlines;
        const long long base = line * N + j;
        float2 v[G::N2];
#pragma unroll
        for (int m = 0; m < G::N2; ++m) {
            const float2 a = valid ? data[base + G::N1 * m] : make_float2(0.f, 0.f);
            v[m] = INV ? cconj(a) : a;
        }
        fft_line<N, false, LayRow<N>>(v, lay, j, tw);
        if (valid)
#pragma unroll
            for (int m = 0; m < G::N2; ++m) data[base + G::N1 * m] = INV ? cconj(v[m]) : v[m];
    }
}

// ------------------------------------------------------------ helpers --
__device__ __forceinline__ void sym_get(const float *pk, int d, float M[3][3]) {
    if (d == 2) {
        M[0][0] = pk[0]; M[0][1] = M[1][0] = pk[1]; M[1][1] = pk[2];
    } else {
        M[0][0] = pk[0]; M[0][1] = M[1][0] = pk[1]; M[0][2] = M[2][0] = pk[2];
        M[1][1] = pk[3]; M[1][2] = M[2][1] = pk[4]; M[2][2] = pk[5];
    }
}

// ---------------------------------------------------------- setup ------
// mode 0: per voxel D^-1 (fp64 cofactors, stored packed in dinv) and
//         per-CTA min/max of mu and of every packed D^-1 element
// mode 1: the per-CTA max of max(|v_u|, ||V_F||_F) (the bound the canonical
//         form scales to target_norm); mode 2: the same, and V per voxel
//         written (vu over the staged mu, vf packed)
__global__ void __launch_bounds__(256) k_tdiff_pot(TDParams p, int mode) {
    const int d = p.d, np = d * (d + 1) / 2;
    float lo[7], hi[7], vmax = 0.f;
    for (int q = 0; q < 7; ++q) { lo[q] = 3.4e38f; hi[q] = -3.4e38f; }
    unsigned nbad = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < p.n; i += (long long)gridDim.x * blockDim.x) {
        if (mode == 0) {
            double M[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
            const float *dp = p.Dpk + i * np;
            if (d == 2) {
                M[0][0] = dp[0]; M[0][1] = M[1][0] = dp[1]; M[1][1] = dp[2];
                const double det = M[0][0] * M[1][1] - M[0][1] * M[1][0];
                const double r[3] = {M[1][1] / det, -M[0][1] / det, M[0][0] / det};
                for (int q = 0; q < 3; ++q) p.dinv[i * np + q] = (float)r[q];
                if (!(det > 0.0) || !isfinite(det)) ++nbad;
            } else {
                M[0][0] = dp[0]; M[0][1] = M[1][0] = dp[1]; M[0][2] = M[2][0] = dp[2];
                M[1][1] = dp[3]; M[1][2] = M[2][1] = dp[4]; M[2][2] = dp[5];
                const double c00 = M[1][1] * M[2][2] - M[1][2] * M[2][1];
                const double c01 = M[1][2] * M[2][0] - M[1][0] * M[2][2];
                const double c02 = M[1][0] * M[2][1] - M[1][1] * M[2][0];
                const double det = M[0][0] * c00 + M[0][1] * c01 + M[0][2] * c02;
                const double r[6] = {c00 / det, c01 / det, c02 / det,
                                     (M[0][0] * M[2][2] - M[0][2] * M[2][0]) / det,
                                     (M[0][2] * M[1][0] - M[0][0] * M[1][2]) / det,
                                     (M[0][0] * M[1][1] - M[0][1] * M[1][0]) / det};
                for (int q = 0; q < 6; ++q) p.dinv[i * np + q] = (float)r[q];
                if (!(det > 0.0) || !isfinite(det)) ++nbad;
            }
            const float mu = p.mu[i];
            if (!isfinite(mu)) ++nbad;
            lo[0] = fminf(lo[0], mu);
            hi[0] = fmaxf(hi[0], mu);
            for (int q = 0; q < np; ++q) {
                const float e = p.dinv[i * np + q];
                lo[q + 1] = fminf(lo[q + 1], e);
                hi[q + 1] = fmaxf(hi[q + 1], e);
            }
        } else {
            const float vu = (p.mu[i] - p.mubar) * p.inv_cu;
            if (mode == 2) p.vu[i] = vu;
            float fro = 0.f;
            for (int q = 0; q < np; ++q) {
                const float e = (p.dinv[i * np + q] - p.dbar[q]) * p.inv_cf;
                if (mode == 2) p.vf[i * np + q] = e;
                const bool diag = (d == 2) ? (q != 1) : (q == 0 || q == 3 || q == 5);
                fro = fmaf(diag ? 1.f : 2.f, e * e, fro);
            }
            vmax = fmaxf(vmax, fmaxf(fabsf(vu), sqrtf(fro)));
        }
    }
    // CTA reductions (min/max are exact in any order)
    __shared__ float s_lo[8][7], s_hi[8][7], s_v[8];
    __shared__ unsigned s_bad[8];
    for (int o = 16; o > 0; o >>= 1) {
        for (int q = 0; q < 7; ++q) {
            lo[q] = fminf(lo[q], __shfl_xor_sync(0xffffffffu, lo[q], o));
            hi[q] = fmaxf(hi[q], __shfl_xor_sync(0xffffffffu, hi[q], o));
        }
        vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
        nbad += __shfl_xor_sync(0xffffffffu, nbad, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        for (int q = 0; q < 7; ++q) { s_lo[w][q] = lo[q]; s_hi[w][q] = hi[q]; }
        s_v[w] = vmax;
        s_bad[w] = nbad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int x = 1; x < 8; ++x) {
            for (int q = 0; q < 7; ++q) {
                s_lo[0][q] = fminf(s_lo[0][q], s_lo[x][q]);
                s_hi[0][q] = fmaxf(s_hi[0][q], s_hi[x][q]);
            }
            s_v[0] = fmaxf(s_v[0], s_v[x]);
            s_bad[0] += s_bad[x];
        }
        float *out = p.red + blockIdx.x * 16;
        for (int q = 0; q < 7; ++q) { out[q] = s_lo[0][q]; out[7 + q] = s_hi[0][q]; }
        out[14] = s_v[0];
        out[15] = (float)s_bad[0];
    }
}

// ------------------------------------------------------ per-mode symbol --
__global__ void __launch_bounds__(256) k_tdiff_mul(TDParams p, int check_state) {
    if (check_state && (p.st->status != ST_RUNNING || p.st->k >= p.st->kmax)) return;
    const int d = p.d;
    const long long n = p.n;
    const MulParams &mp = p.mp;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int ix = (int)(i % mp.nx);
        const long long r = i / mp.nx;
        const int iy = (int)(r % mp.ny), iz = (int)(r / mp.ny);
        float q[3] = {mp.kx * freq_m(ix, mp.nx) * p.qs, mp.ky * freq_m(iy, mp.ny) * p.qs,
                      d == 3 ? mp.kz * freq_m(iz, mp.nz) * p.qs : 0.f};
        float w[3];
        float sig = p.a;
        for (int k = 0; k < d; ++k) {
            w[k] = 0.f;
            for (int m = 0; m < d; ++m) w[k] = fmaf(p.dm_inv[k * 3 + m], q[m], w[k]);
            sig = fmaf(q[k], w[k], sig);
        }
        const float is = p.inv_n / sig;
        const float2 u = p.work[i];
        float2 F[3], wF = make_float2(0.f, 0.f);
        for (int k = 0; k < d; ++k) {
            F[k] = p.work[(k + 1) * n + i];
            wF = make_float2(fmaf(w[k], F[k].x, wF.x), fmaf(w[k], F[k].y, wF.y));
        }
        // out_u = (u - i wF) / sig ;  out_F = Dm^-1 F - i w out_u  (1/N_vox folded in)
        const float2 ou = make_float2((u.x + wF.y) * is, (u.y - wF.x) * is);
        p.work[i] = ou;
        for (int k = 0; k < d; ++k) {
            float2 acc = make_float2(0.f, 0.f);
            for (int m = 0; m < d; ++m)
                acc = make_float2(fmaf(p.dm_inv[k * 3 + m], F[m].x, acc.x), fmaf(p.dm_inv[k * 3 + m], F[m].y, acc.y));
            acc = cscale(acc, p.inv_n);
            p.work[(k + 1) * n + i] = make_float2(acc.x + w[k] * ou.y, acc.y - w[k] * ou.x);
        }
    }
}

// ----------------------------------------------- update + residual ------
// mode X_SRC_FWD: work = s = [S / (c sqrt s_u); 0]        (no reduction)
// mode X_SRC_EPI: Delta_0 = B y, x_0 = 0, n0, work = B Delta_0
// mode X_ITER:    Delta <- Delta + alpha B (y - Delta), x <- x + alpha Delta, work = B Delta
__device__ __forceinline__ void tdiff_B(const TDParams &p, long long i, const float2 *in, float2 *out) {
    const int d = p.d, np = d * (d + 1) / 2;
    float Vf[3][3];
    sym_get(p.vf + i * np, d, Vf);
    const float bu = 1.f - p.vu[i];
    out[0] = cscale(in[0], bu);
    for (int k = 0; k < d; ++k) {
        float2 acc = in[k + 1];
        for (int m = 0; m < d; ++m) acc = make_float2(fmaf(-Vf[k][m], in[m + 1].x, acc.x), fmaf(-Vf[k][m], in[m + 1].y, acc.y));
        out[k + 1] = acc;
    }
}

template <int MODE>
__global__ void __launch_bounds__(256) k_tdiff_upd(TDParams p) {
    __shared__ double sh_red[8];
    const int d = p.d;
    const long long n = p.n;
    bool xonly = false;
    float alpha = 0.f;
    if (MODE == X_ITER) {
        const int status = p.st->status;
        if (p.st->k >= p.st->kmax || (status != ST_RUNNING && status != ST_STOP_PENDING)) return;
        xonly = status == ST_STOP_PENDING;
        alpha = (float)p.st->alpha;
    }
    double acc = 0.0;
    float la = 0.f;
    int cnt = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        if (MODE == X_SRC_FWD) {
            p.work[i] = make_float2(p.Sraw[i] * p.s_scale, 0.f);
            for (int k = 1; k <= d; ++k) p.work[k * n + i] = make_float2(0.f, 0.f);
            continue;
        }
        float2 y[4], dl[4], t[4];
        if (MODE == X_ITER && xonly) {
            for (int k = 0; k <= d; ++k) {
                const float2 dd = p.delta[k * n + i], xx = p.x[k * n + i];
                p.x[k * n + i] = make_float2(fmaf(alpha, dd.x, xx.x), fmaf(alpha, dd.y, xx.y));
            }
            continue;
        }
        for (int k = 0; k <= d; ++k) y[k] = p.work[k * n + i];
        if (MODE == X_SRC_EPI) {
            tdiff_B(p, i, y, dl);
            for (int k = 0; k <= d; ++k) p.x[k * n + i] = make_float2(0.f, 0.f);
        } else {
            float2 od[4];
            for (int k = 0; k <= d; ++k) {
                od[k] = p.delta[k * n + i];
                t[k] = csub(y[k], od[k]);
            }
            tdiff_B(p, i, t, dl);
            for (int k = 0; k <= d; ++k) {
                const float2 xx = p.x[k * n + i];
                p.x[k * n + i] = make_float2(fmaf(alpha, od[k].x, xx.x), fmaf(alpha, od[k].y, xx.y));
                dl[k] = make_float2(fmaf(alpha, dl[k].x, od[k].x), fmaf(alpha, dl[k].y, od[k].y));
            }
        }
        for (int k = 0; k <= d; ++k) {
            p.delta[k * n + i] = dl[k];
            la += cabs2(dl[k]);
        }
        tdiff_B(p, i, dl, t);                      // next chain input: u = B Delta
        for (int k = 0; k <= d; ++k) p.work[k * n + i] = t[k];
        if (++cnt == 64) { acc += (double)la; la = 0.f; cnt = 0; }
    }
    if (MODE == X_SRC_FWD) return;
    acc += (double)la;
    double total;
    const double mine = block_sum_d<256>(acc, sh_red);
    if (!last_block_total<256>(mine, p.st, p.red_d.partials, sh_red, &total)) return;
    if (threadIdx.x != 0) return;
    finish_xpass(MODE == X_SRC_EPI, xonly, total, p.st, p.red_d);
}

// u = E_0 / sqrt(s_u) as float32 (the solution of A_raw, reading R-29)
__global__ void k_tdiff_out(const float2 *E0, float *out, float scale, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = E0[i].x * scale;
}

// ========================================================= launchers ====
template <int N, bool INV>
static cudaError_t xfft_t(float2 *data, const float2 *tw, long long nlines, int grid, cudaStream_t s) {
    constexpr int LPC = 128 / LineGeo<N>::N1;
    k_xfft<N, INV><<<grid, 128, LPC * LayRow<N>::kFloat2PerLine * 8, s>>>(data, tw, nlines);
    return cudaGetLastError();
}

cudaError_t launch_xfft(int N, bool inv, float2 *data, const float2 *tw, long long nlines, int grid, cudaStream_t s) {
#define XF_CASE(n) \
    case n: return inv ? xfft_t<n, true>(data, tw, nlines, grid, s) : xfft_t<n, false>(data, tw, nlines, grid, s);
    switch (N) { XF_CASE(64) XF_CASE(128) XF_CASE(256) XF_CASE(512) XF_CASE(1024)
    default: return cudaErrorInvalidValue; }
#undef XF_CASE
}

cudaError_t launch_tdiff_pot(const TDParams &p, int mode, int grid, cudaStream_t s) {
    k_tdiff_pot<<<grid, 256, 0, s>>>(p, mode);
    return cudaGetLastError();
}
cudaError_t launch_tdiff_mul(const TDParams &p, int check_state, int grid, cudaStream_t s) {
    k_tdiff_mul<<<grid, 256, 0, s>>>(p, check_state);
    return cudaGetLastError();
}
cudaError_t launch_tdiff_upd(XMode mode, const TDParams &p, int grid, cudaStream_t s) {
    if (mode == X_SRC_FWD) k_tdiff_upd<X_SRC_FWD><<<grid, 256, 0, s>>>(p);
    else if (mode == X_SRC_EPI) k_tdiff_upd<X_SRC_EPI><<<grid, 256, 0, s>>>(p);
    else k_tdiff_upd<X_ITER><<<grid, 256, 0, s>>>(p);
    return cudaGetLastError();
}
cudaError_t launch_tdiff_out(const float2 *E0, float *out, float scale, long long n, int grid, cudaStream_t s) {
    k_tdiff_out<<<grid, 256, 0, s>>>(E0, out, scale, n);
    return cudaGetLastError();
}

}  // namespace usp
