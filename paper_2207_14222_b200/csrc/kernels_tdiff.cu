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
#include "tma.cuh"
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
// (templated on d so every component loop unrolls into registers)
template <int d>
__global__ void __launch_bounds__(256) k_tdiff_mul(TDParams p, int check_state) {
    if (check_state && (p.st->status != ST_RUNNING || p.st->k >= p.st->kmax)) return;
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
#pragma unroll
        for (int k = 0; k < d; ++k) {
            w[k] = 0.f;
#pragma unroll
            for (int m = 0; m < d; ++m) w[k] = fmaf(p.dm_inv[k * 3 + m], q[m], w[k]);
            sig = fmaf(q[k], w[k], sig);
        }
        const float is = p.inv_n / sig;
        const float2 u = p.work[i];
        float2 F[3], wF = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < d; ++k) {
            F[k] = p.work[(k + 1) * n + i];
            wF = make_float2(fmaf(w[k], F[k].x, wF.x), fmaf(w[k], F[k].y, wF.y));
        }
        // out_u = (u - i wF) / sig ;  out_F = Dm^-1 F - i w out_u  (1/N_vox folded in)
        const float2 ou = make_float2((u.x + wF.y) * is, (u.y - wF.x) * is);
        p.work[i] = ou;
#pragma unroll
        for (int k = 0; k < d; ++k) {
            float2 acc = make_float2(0.f, 0.f);
#pragma unroll
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
template <int d>
__device__ __forceinline__ void tdiff_B(const float (&Vf)[3][3], float bu, const float2 *in, float2 *out) {
    out[0] = cscale(in[0], bu);
#pragma unroll
    for (int k = 0; k < d; ++k) {
        float2 acc = in[k + 1];
#pragma unroll
        for (int m = 0; m < d; ++m) acc = make_float2(fmaf(-Vf[k][m], in[m + 1].x, acc.x), fmaf(-Vf[k][m], in[m + 1].y, acc.y));
        out[k + 1] = acc;
    }
}

template <int d, int MODE>
__global__ void __launch_bounds__(256) k_tdiff_upd(TDParams p) {
    __shared__ double sh_red[8];
    constexpr int np = d * (d + 1) / 2;
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
#pragma unroll
            for (int k = 1; k <= d; ++k) p.work[k * n + i] = make_float2(0.f, 0.f);
            continue;
        }
        float2 y[4], dl[4], t[4];
        if (MODE == X_ITER && xonly) {
#pragma unroll
            for (int k = 0; k <= d; ++k) {
                const float2 dd = p.delta[k * n + i], xx = p.x[k * n + i];
                p.x[k * n + i] = make_float2(fmaf(alpha, dd.x, xx.x), fmaf(alpha, dd.y, xx.y));
            }
            continue;
        }
        float Vf[3][3];
        sym_get(p.vf + i * np, d, Vf);
        const float bu = 1.f - p.vu[i];
#pragma unroll
        for (int k = 0; k <= d; ++k) y[k] = p.work[k * n + i];
        if (MODE == X_SRC_EPI) {
            tdiff_B<d>(Vf, bu, y, dl);
#pragma unroll
            for (int k = 0; k <= d; ++k) p.x[k * n + i] = make_float2(0.f, 0.f);
        } else {
            float2 od[4];
#pragma unroll
            for (int k = 0; k <= d; ++k) {
                od[k] = p.delta[k * n + i];
                t[k] = csub(y[k], od[k]);
            }
            tdiff_B<d>(Vf, bu, t, dl);
#pragma unroll
            for (int k = 0; k <= d; ++k) {
                const float2 xx = p.x[k * n + i];
                p.x[k * n + i] = make_float2(fmaf(alpha, od[k].x, xx.x), fmaf(alpha, od[k].y, xx.y));
                dl[k] = make_float2(fmaf(alpha, dl[k].x, od[k].x), fmaf(alpha, dl[k].y, od[k].y));
            }
        }
#pragma unroll
        for (int k = 0; k <= d; ++k) {
            p.delta[k * n + i] = dl[k];
            la += cabs2(dl[k]);
        }
        tdiff_B<d>(Vf, bu, dl, t);                 // next chain input: u = B Delta
#pragma unroll
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

// ------------------------------------- fused x pass (TMA-pipelined) ------
// The iteration's x inverse FFT -> k_tdiff_upd's update -> x forward FFT in
// one pass (k_anti_pipe's structure): a producer warp bulk-copies a unit's
// work, Delta and x of every component plus v_u and V_F into the consumer
// warp's stage; the consumer transforms the components one at a time (each
// y_c parked back in its own slot), runs the update element by element (x,
// Delta stored, u = B Delta parked in the work slots) and forward-transforms
// u.  Saves the two k_xfft passes (2 x 16 (d + 1) B/voxel).  The stage is
// (3 (d + 1) + 1 + d (d + 1) / 2) x 8 B per element of the unit; where fewer
// than two stages fit (x extent >= 512) the three-kernel sequence runs.
constexpr int kTdSmemBudget = 232448 - 2048;

template <int N, int d>
struct TPipe {
    using G = LineGeo<N>;
    static constexpr int C = d + 1, NP = d * (d + 1) / 2;
    static constexpr int U = 32 / G::N1;
    static constexpr int UE = 32 * G::N2;
    static constexpr int VU = 3 * C * UE;                // float2 offset of v_u (UE floats)
    static constexpr int VF = VU + UE / 2;               // float2 offset of V_F (NP UE floats)
    static constexpr int STAGE = VF + NP * UE / 2;
    static constexpr int XBUF = U * LayRow<N>::kFloat2PerLine;
    static constexpr int XC0 = (kTdSmemBudget - N * 8) / ((STAGE + XBUF) * 8);
    static constexpr int XC = XC0 > 6 ? 6 : XC0;
    static constexpr bool FITS = XC >= 2;
    static constexpr int S = XC;
    static constexpr int NT = 32 * (XC + 1);
    static constexpr int SMEM = (S * STAGE + XC * XBUF + N) * 8 + 2 * S * 8;
};

template <int N, int d>
__global__ void __launch_bounds__(TPipe<N, d>::NT, 1) k_tdiff_pipe(TDParams p) {
    using G = LineGeo<N>;
    using T = TPipe<N, d>;
    constexpr int C = T::C;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float2 *stages = reinterpret_cast<float2 *>(smem_raw);
    float2 *xbufs = stages + T::S * T::STAGE;
    float2 *sm_tw = xbufs + T::XC * T::XBUF;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm_tw + N);
    uint64_t *empty = full + T::S;
    __shared__ double sh_red[T::NT / 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int status = p.st->status;
    if (p.st->k >= p.st->kmax || (status != ST_RUNNING && status != ST_STOP_PENDING)) return;
    const bool xonly = status == ST_STOP_PENDING;
    const float alpha = (float)p.st->alpha;
    const long long n = p.n;
    double acc = 0.0;
    if (xonly) {   // the final x += alpha Delta after the stop test (R-5)
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < C * n;
             i += (long long)gridDim.x * blockDim.x) {
            const float2 dd = p.delta[i], xx = p.x[i];
            p.x[i] = make_float2(fmaf(alpha, dd.x, xx.x), fmaf(alpha, dd.y, xx.y));
        }
    } else {
        if (threadIdx.x == 0) {
            for (int s = 0; s < T::S; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&empty[s], 1);
            }
            fence_mbar_init();
        }
        load_twiddles<N>(sm_tw, p.twx);
        __syncthreads();
        const long long nunits = n / T::UE;
        const int nloc = (int)((nunits - blockIdx.x + gridDim.x - 1) / gridDim.x);
        const uint32_t ub = T::UE * 8u;
        if (warp == T::XC) {
            if (lane == 0) {   // producer
                for (int i = 0; i < nloc; ++i) {
                    const int s = i % T::S;
                    if (i >= T::S && !mbar_wait(&empty[s], ((i / T::S) - 1) & 1)) {
                        if (atomicCAS(&p.st->err, 0, 33) == 0) p.st->err_info = i;
                        break;
                    }
                    const long long off = (blockIdx.x + (long long)i * gridDim.x) * T::UE;
                    float2 *st = stages + s * T::STAGE;
                    mbar_arrive_expect_tx(&full[s], 3 * C * ub + T::UE * 4u * (1 + T::NP));
#pragma unroll
                    for (int c = 0; c < C; ++c) {
                        bulk_g2s(st + c * T::UE, p.work + c * n + off, ub, &full[s]);
                        bulk_g2s(st + (C + c) * T::UE, p.delta + c * n + off, ub, &full[s]);
                        bulk_g2s(st + (2 * C + c) * T::UE, p.x + c * n + off, ub, &full[s]);
                    }
                    bulk_g2s(st + T::VU, p.vu + off, T::UE * 4u, &full[s]);
                    bulk_g2s(st + T::VF, p.vf + off * T::NP, T::UE * 4u * T::NP, &full[s]);
                }
            }
            __syncwarp();
        } else {
            const int lq = lane / G::N1, j = lane % G::N1;
            const LayRow<N> lay{xbufs + warp * T::XBUF + lq * LayRow<N>::kFloat2PerLine};
            for (int i = warp; i < nloc; i += T::XC) {
                const int s = i % T::S;
                if (!mbar_wait(&full[s], (i / T::S) & 1)) {
                    if (lane == 0 && atomicCAS(&p.st->err, 0, 34) == 0) p.st->err_info = i;
                    break;
                }
                float2 *st = stages + s * T::STAGE;
                const float *svu = reinterpret_cast<const float *>(st + T::VU);
                const float *svf = reinterpret_cast<const float *>(st + T::VF);
                const long long gb = (blockIdx.x + (long long)i * gridDim.x) * T::UE + lq * N + j;
                const int sb = lq * N + j;
                float2 v[G::N2];
#pragma unroll 1
                for (int c = 0; c < C; ++c) {   // x inverse (conj trick); y_c parked in its slot
                    float2 *w = st + c * T::UE + sb;
#pragma unroll
                    for (int m = 0; m < G::N2; ++m) v[m] = cconj(w[G::N1 * m]);
                    fft_line<N, false, LayRow<N>, true>(v, lay, j, sm_tw);
#pragma unroll
                    for (int m = 0; m < G::N2; ++m) w[G::N1 * m] = cconj(v[m]);
                }
                float lacc = 0.f;
#pragma unroll 2
                for (int m = 0; m < G::N2; ++m) {
                    const int e = sb + G::N1 * m;
                    const long long gi = gb + G::N1 * m;
                    float Vf[3][3];
                    sym_get(svf + e * T::NP, d, Vf);
                    const float bu = 1.f - svu[e];
                    float2 od[C], t[C], dl[C];
#pragma unroll
                    for (int c = 0; c < C; ++c) {
                        od[c] = st[(C + c) * T::UE + e];
                        t[c] = csub(st[c * T::UE + e], od[c]);
                    }
                    tdiff_B<d>(Vf, bu, t, dl);
#pragma unroll
                    for (int c = 0; c < C; ++c) {
                        const float2 xx = st[(2 * C + c) * T::UE + e];
                        p.x[c * n + gi] = make_float2(fmaf(alpha, od[c].x, xx.x), fmaf(alpha, od[c].y, xx.y));
                        dl[c] = make_float2(fmaf(alpha, dl[c].x, od[c].x), fmaf(alpha, dl[c].y, od[c].y));
                        p.delta[c * n + gi] = dl[c];
                        lacc += cabs2(dl[c]);
                    }
                    tdiff_B<d>(Vf, bu, dl, t);   // next chain input: u = B Delta
#pragma unroll
                    for (int c = 0; c < C; ++c) st[c * T::UE + e] = t[c];
                }
                acc += (double)lacc;
                __syncwarp();
#pragma unroll 1
                for (int c = 0; c < C; ++c) {   // x forward of u
#pragma unroll
                    for (int m = 0; m < G::N2; ++m) v[m] = st[c * T::UE + sb + G::N1 * m];
                    if (c == C - 1) {            // the stage is consumed: let it refill
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty[s]);
                    }
                    fft_line<N, false, LayRow<N>, true>(v, lay, j, sm_tw);
#pragma unroll
                    for (int m = 0; m < G::N2; ++m) p.work[c * n + gb + G::N1 * m] = v[m];
                }
            }
        }
    }
    double total;
    const double mine = block_sum_d<T::NT>(acc, sh_red);
    if (!last_block_total<T::NT>(mine, p.st, p.red_d.partials, sh_red, &total)) return;
    if (threadIdx.x != 0) return;
    finish_xpass(false, xonly, total, p.st, p.red_d);
}

template <int N, int d>
static cudaError_t tdiff_pipe_t(const TDParams &p, int grid, cudaStream_t s) {
    if constexpr (!TPipe<N, d>::FITS) {
        return cudaErrorInvalidValue;
    } else {
        static bool attr = false;
        if (!attr) {
            cudaError_t e = cudaFuncSetAttribute(k_tdiff_pipe<N, d>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 TPipe<N, d>::SMEM);
            if (e != cudaSuccess) return e;
            attr = true;
        }
        k_tdiff_pipe<N, d><<<grid, TPipe<N, d>::NT, TPipe<N, d>::SMEM, s>>>(p);
        return cudaGetLastError();
    }
}

cudaError_t launch_tdiff_pipe(int N, const TDParams &p, int grid, cudaStream_t s) {
#define TP_CASE(n) \
    case n: return p.d == 2 ? tdiff_pipe_t<n, 2>(p, grid, s) : tdiff_pipe_t<n, 3>(p, grid, s);
    switch (N) { TP_CASE(64) TP_CASE(128) TP_CASE(256) TP_CASE(512) TP_CASE(1024)
    default: return cudaErrorInvalidValue; }
#undef TP_CASE
}

int tdiff_pipe_units(int N, int d) {   // lines per warp unit; 0: the stage does not fit
#define TU_CASE(n) \
    case n: return (d == 2 ? TPipe<n, 2>::FITS : TPipe<n, 3>::FITS) ? TPipe<n, 2>::U : 0;
    switch (N) { TU_CASE(64) TU_CASE(128) TU_CASE(256) TU_CASE(512) TU_CASE(1024)
    default: return 0; }
#undef TU_CASE
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
    if (p.d == 2) k_tdiff_mul<2><<<resident_grid<k_tdiff_mul<2>>(grid, 256), 256, 0, s>>>(p, check_state);
    else k_tdiff_mul<3><<<resident_grid<k_tdiff_mul<3>>(grid, 256), 256, 0, s>>>(p, check_state);
    return cudaGetLastError();
}
template <int d>
static void tdiff_upd_t(XMode mode, const TDParams &p, int grid, cudaStream_t s) {
    if (mode == X_SRC_FWD) k_tdiff_upd<d, X_SRC_FWD><<<resident_grid<k_tdiff_upd<d, X_SRC_FWD>>(grid, 256), 256, 0, s>>>(p);
    else if (mode == X_SRC_EPI) k_tdiff_upd<d, X_SRC_EPI><<<resident_grid<k_tdiff_upd<d, X_SRC_EPI>>(grid, 256), 256, 0, s>>>(p);
    else k_tdiff_upd<d, X_ITER><<<resident_grid<k_tdiff_upd<d, X_ITER>>(grid, 256), 256, 0, s>>>(p);
}
cudaError_t launch_tdiff_upd(XMode mode, const TDParams &p, int grid, cudaStream_t s) {
    if (p.d == 2) tdiff_upd_t<2>(mode, p, grid, s);
    else tdiff_upd_t<3>(mode, p, grid, s);
    return cudaGetLastError();
}
cudaError_t launch_tdiff_out(const float2 *E0, float *out, float scale, long long n, int grid, cudaStream_t s) {
    k_tdiff_out<<<grid, 256, 0, s>>>(E0, out, scale, n);
    return cudaGetLastError();
}

}  // namespace usp
