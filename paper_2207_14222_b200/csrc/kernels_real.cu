// kernels_real.cu -- x pass of the REAL path (steady-state diffusion with real
// data; §3.2, Eq. 12 with real D, sigma, c).
//
// For real mu_a, sigma, c the whole iteration stays real: V, B, s, x, Delta
// are float32 and the symbol g(p) = c / (D|p|^2 + sigma + c) of (L+1)^-1 is
// real and even, so (L+1)^-1 maps real fields to real fields.  The spectrum
// of a real x-line of N points is Hermitian: X[0..N/2] (N/2 + 1 values)
// determine it.  Fields and bytes therefore halve (52 instead of 104 B per
// voxel and iteration, SURVEY.md §8 geometry table).
//
// Layout: x, Delta, B: float32 [z][y][x].  The chain buffer `work` holds the
// half spectrum, rows of RP = N/2 + 16 complex64 (X[0..N/2] then zero
// padding, so the strided passes keep 16-column tiles): [z][y][RP].
//
// A real line x[0..N) is processed as the complex line z[n] = x[2n] + i
// x[2n+1] of M = N/2 points (its float2 view: no repacking) with the
// four-step FFT of fft_core.cuh, plus the standard split/merge steps
// (Z = DFT_M z, W = exp(-2 pi i/N)):
//   forward : X[k] = (Z[k] + conj Z[M-k])/2 + W^k (Z[k] - conj Z[M-k])/(2i),
//             k = 0..M (Z[M] = Z[0])
//   inverse : Z[k] = (X[k] + conj X[M-k]) + i W^-k (X[k] - conj X[M-k]),
//             z = IDFT_M Z  = N (x[2n] + i x[2n+1])  (unnormalised, as the
//             complex path: the 1/N_vox lives in g)
// The forward step needs Z[M-k], held by another lane: one extra pass
// through the line's shared-memory buffer.  The inverse reads X[M-k] from
// the staged row directly.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fft_core.cuh"
#include "kcommon.cuh"
#include "tma.cuh"
#include "usp_internal.h"

namespace usp {

constexpr int kSmemBudgetR = 232448 - 2048;

template <int N>   // N = real line length
struct XReal {
    static constexpr int M = N / 2;
    using G = LineGeo<M>;
    static constexpr int RP = M + 16;                       // spectrum row pitch (complex64)
    static constexpr int U = 32 / G::N1;                    // lines per warp unit
    static constexpr int XC = 5;                            // consumer warps
    static constexpr int NT = 32 * (XC + 1);
    static constexpr int XBUF = U * LayRow<M>::kFloat2PerLine;
    static constexpr int W0 = 0, D0 = U * RP, X0 = D0 + U * M, B0 = X0 + U * M;
    static constexpr int STAGE = B0 + U * M;                // float2 per stage
    static constexpr int SPW0 = (kSmemBudgetR - XC * XBUF * 8 - 2 * M * 8) / (XC * STAGE * 8);
    static constexpr int SPW = SPW0 > 2 ? 2 : SPW0;
    static constexpr int S = XC * SPW;
    static_assert(SPW >= 1, "real x pipeline needs >= 1 stage per consumer warp");
    static_assert(LayRow<M>::kFloat2PerLine >= M, "partner buffer");
    static constexpr int SMEM = (S * STAGE + XC * XBUF + 2 * M) * 8 + 2 * S * 8;
};

template <int N, int MODE>
__global__ void __launch_bounds__(XReal<N>::NT, 1) k_xpass_real(XParams p) {
    using T = XReal<N>;
    constexpr int M = T::M;
    using G = typename T::G;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float2 *stages = reinterpret_cast<float2 *>(smem_raw);
    float2 *xbufs = stages + T::S * T::STAGE;
    float2 *sm_tw = xbufs + T::XC * T::XBUF;     // four-step table of the M-point FFT
    float2 *sm_twr = sm_tw + M;                  // W_N^k, k < M (split/merge)
    uint64_t *full = reinterpret_cast<uint64_t *>(sm_twr + M);
    uint64_t *empty = full + T::S;
    __shared__ double sh_red[T::NT / 32];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float *xr = reinterpret_cast<float *>(p.x);
    float *dr = reinterpret_cast<float *>(p.delta);

    bool xonly = false;
    float alpha = 0.f;
    int act = ACT_DELTA;   // X_ITER: Delta-form, x-form, probe or x-form -> Delta-form (kcommon.cuh, R-30)
    if (MODE == X_ITER) {
        const int status = p.st->status;
        const long long k = p.st->k, kmax = p.st->kmax;
        const bool probe = p.st->form == FORM_PROBE && status == ST_RUNNING;
        if (!probe && (k >= kmax || (status != ST_RUNNING && status != ST_STOP_PENDING))) return;
        xonly = (status == ST_STOP_PENDING);
        alpha = (float)p.st->alpha;
        act = xform_act(p.st);
    }
    const bool dform = act == ACT_DELTA;
    const float c1 = dform ? alpha : 1.f;
    const float e1 = (act == ACT_X || act == ACT_PROBE) ? 1.f : 0.f;
    const bool store_x = act == ACT_DELTA || act == ACT_X, store_d = act != ACT_X;
    const bool u_from_d = act == ACT_DELTA || act == ACT_TO_DELTA;
    // stage slot D0: Delta (Delta-form) or s (x-form passes; source setup of x-form plans)
    const float2 *slot_d = (MODE == X_ITER && act != ACT_DELTA) || (MODE == X_SRC_EPI && p.s) ? p.s : p.delta;
    double acc = 0.0;
    const long long nvox = p.nlines * (long long)N;

    if (MODE == X_ITER && xonly) {
        // final x_{k+1} = x_k + alpha Delta_k after the stop test (reading R-5)
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvox;
             i += (long long)gridDim.x * blockDim.x)
            xr[i] = fmaf(alpha, dr[i], xr[i]);
    } else {
        if (threadIdx.x == 0) {
            for (int s = 0; s < T::S; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&empty[s], 1);
            }
            fence_mbar_init();
        }
        load_twiddles<M>(sm_tw, p.tw);
        for (int i = threadIdx.x; i < M; i += blockDim.x) sm_twr[i] = __ldg(&p.twr[i]);
        __syncthreads();
        const long long nunits = p.nlines / T::U;
        const int nloc = (int)((nunits - blockIdx.x + gridDim.x - 1) / gridDim.x);
        const uint32_t wb = T::U * T::RP * 8u, fb = T::U * M * 8u;   // bytes: spectrum rows, one real field
        if (warp == T::XC) {
            // ------------------------------------------------ producer warp
            if (lane == 0) {
                for (int i = 0; i < nloc; ++i) {
                    const int s = i % T::S;
                    if (i >= T::S && !mbar_wait(&empty[s], ((i / T::S) - 1) & 1)) {
                        if (atomicCAS(&p.st->err, 0, 6) == 0) p.st->err_info = i;
                        break;
                    }
                    const long long u = blockIdx.x + (long long)i * gridDim.x;
                    const long long offw = u * T::U * T::RP, offf = u * T::U * M;
                    float2 *st = stages + s * T::STAGE;
                    if (MODE == X_SRC_FWD) {            // raw real source staged in x
                        mbar_arrive_expect_tx(&full[s], fb);
                        bulk_g2s(st + T::D0, p.x + offf, fb, &full[s]);
                    } else if (MODE == X_SRC_EPI) {
                        mbar_arrive_expect_tx(&full[s], wb + (p.s ? 2 : 1) * fb);
                        bulk_g2s(st + T::W0, p.work + offw, wb, &full[s]);
                        if (p.s) bulk_g2s(st + T::D0, slot_d + offf, fb, &full[s]);
                        bulk_g2s(st + T::B0, p.B + offf, fb, &full[s]);
                    } else {
                        mbar_arrive_expect_tx(&full[s], wb + 3 * fb);
                        bulk_g2s(st + T::W0, p.work + offw, wb, &full[s]);
                        bulk_g2s(st + T::D0, slot_d + offf, fb, &full[s]);
                        bulk_g2s(st + T::X0, p.x + offf, fb, &full[s]);
                        bulk_g2s(st + T::B0, p.B + offf, fb, &full[s]);
                    }
                }
            }
            __syncwarp();
        } else {
            // ------------------------------------------------ consumer warps
            const int lq = lane / G::N1, j = lane % G::N1;
            const LayRow<M> lay{xbufs + warp * T::XBUF + lq * LayRow<M>::kFloat2PerLine};
            float2 *zb = lay.base;   // partner buffer (the exchange buffer is free between FFTs)
            const float cr = p.inv_c.x;   // 1/c, real on this path
            for (int i = warp; i < nloc; i += T::XC) {
                const int s = i % T::S;
                if (!mbar_wait(&full[s], (i / T::S) & 1)) {
                    if (lane == 0 && atomicCAS(&p.st->err, 0, 7) == 0) p.st->err_info = i;
                    break;
                }
                const float2 *st = stages + s * T::STAGE;
                const long long u = blockIdx.x + (long long)i * gridDim.x;
                const long long gf = u * T::U * M + lq * M + j;        // float2 index of (x[2n], x[2n+1])
                const long long gw = u * T::U * T::RP + lq * T::RP;   // this line's spectrum row
                const float2 *row = st + T::W0 + lq * T::RP;
                const int fbase = lq * M + j;
                float2 v[G::N2];
                if (MODE == X_SRC_FWD) {
#pragma unroll
                    for (int m = 0; m < G::N2; ++m) {
                        v[m] = cscale(st[T::D0 + fbase + G::N1 * m], cr);   // s = S/c
                        if (p.s) p.s[gf + G::N1 * m] = v[m];                // x-form plans keep s
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[s]);
                } else {
                    // inverse merge: Z[k] = (X[k] + conj X[M-k]) + i W^-k (X[k] - conj X[M-k])
#pragma unroll
                    for (int m = 0; m < G::N2; ++m) {
                        const int k = j + G::N1 * m;
                        const float2 a = row[k], b = cconj(row[M - k]);
                        const float2 e = cadd(a, b);
                        const float2 o = cmulc(csub(a, b), sm_twr[k]);
                        v[m] = cconj(make_float2(e.x - o.y, e.y + o.x));   // conj: inverse via forward DFT
                    }
                }
#pragma unroll 1
                for (int pass = (MODE == X_SRC_FWD) ? 1 : 0; pass < 2; ++pass) {
                    fft_line<M, false, LayRow<M>, true>(v, lay, j, sm_tw);
                    if (pass == 0) {
                        float lacc = 0.f;
#pragma unroll
                        for (int m = 0; m < G::N2; ++m) {
                            const int e = fbase + G::N1 * m;
                            const long long gi = gf + G::N1 * m;
                            const float2 y = cconj(v[m]);             // (L+1)^-1 u at x[2n], x[2n+1]
                            const float2 b = st[T::B0 + e];
                            float2 dn;
                            if (MODE == X_SRC_EPI) {
                                dn = make_float2(b.x * y.x, b.y * y.y);          // Delta_0 = B (L+1)^-1 s
                                p.x[gi] = make_float2(0.f, 0.f);                 // x_0 = 0 (L83)
                                p.delta[gi] = dn;
                                lacc = fmaf(dn.x, dn.x, fmaf(dn.y, dn.y, lacc));
                                // u = B Delta (x-form plans: u_0 = s)
                                v[m] = p.s ? st[T::D0 + e] : make_float2(b.x * dn.x, b.y * dn.y);
                                continue;
                            }
                            // every action in one body (see kernels_pipe.cu; real, elementwise):
                            // Delta-form  dn = d + alpha B (y - d), x += alpha d, u = B dn
                            // x-form      dn = B (y - x), x += alpha dn, u = B x + s
                            // probe       dn = B (y - x) stored, u = B x + s;  to-Delta: u = B dn
                            const float2 a1 = st[T::D0 + e], xx = st[T::X0 + e];
                            const float2 z = dform ? a1 : xx;
                            const float2 t = make_float2(b.x * (y.x - z.x), b.y * (y.y - z.y));
                            const float2 d0 = dform ? a1 : make_float2(0.f, 0.f);
                            dn = make_float2(fmaf(c1, t.x, d0.x), fmaf(c1, t.y, d0.y));
                            const float2 xi = dform ? a1 : t;
                            const float2 xn = make_float2(fmaf(alpha, xi.x, xx.x), fmaf(alpha, xi.y, xx.y));
                            if (store_x) p.x[gi] = xn;
                            if (store_d) p.delta[gi] = dn;
                            lacc = fmaf(dn.x, dn.x, fmaf(dn.y, dn.y, lacc));
                            const float2 w = u_from_d ? dn : (act == ACT_X ? xn : xx);
                            v[m] = make_float2(fmaf(e1, a1.x, b.x * w.x), fmaf(e1, a1.y, b.y * w.y));
                        }
                        acc += (double)lacc;
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty[s]);
                    }
                }
                // forward split: X[k] = (Z[k] + conj Z[M-k])/2 - i W^k (Z[k] - conj Z[M-k])/2
#pragma unroll
                for (int m = 0; m < G::N2; ++m) zb[j + G::N1 * m] = v[m];
                __syncwarp();
                float2 zp[G::N2];
#pragma unroll
                for (int m = 0; m < G::N2; ++m) zp[m] = cconj(zb[(M - (j + G::N1 * m)) & (M - 1)]);
                __syncwarp();
#pragma unroll
                for (int m = 0; m < G::N2; ++m) {
                    const int k = j + G::N1 * m;
                    const float2 e = cscale(cadd(v[m], zp[m]), 0.5f);
                    const float2 d = csub(v[m], zp[m]);
                    const float2 o = make_float2(0.5f * d.y, -0.5f * d.x);   // (Z - conj Zp)/(2i)
                    const float2 X = cadd(e, cmul(o, sm_twr[k]));
                    p.work[gw + k] = X;
                    if (k == 0) p.work[gw + M] = make_float2(e.x - o.x, 0.f);   // X[M] = E[0] - O[0]
                }
            }
        }
    }

    if (MODE == X_SRC_FWD) return;
    double total;
    const double mine = block_sum_d<T::NT>(acc, sh_red);
    if (!last_block_total<T::NT>(mine, p.st, p.red.partials, sh_red, &total)) return;
    if (threadIdx.x != 0) return;
    if (p.red.local_sum) {   // slab-decomposed: k_finish sums the ranks' totals after the all-gather
        *p.red.local_sum = total;
        return;
    }
    finish_xpass(MODE == X_SRC_EPI, xonly, total, p.st, p.red, act);
}

// ========================================================= launchers ====
template <int N, int MODE>
static cudaError_t xreal_t(const XParams &p, int grid, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_xpass_real<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             XReal<N>::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    k_xpass_real<N, MODE><<<grid, XReal<N>::NT, XReal<N>::SMEM, s>>>(p);
    return cudaGetLastError();
}

bool xreal_supported(long long n) { return n >= 32 && n <= 2048 && (n & (n - 1)) == 0; }
int xreal_row_pitch(int N) { return N / 2 + 16; }
int xreal_lines_per_unit(int N) { return 32 / (1 << (ilog2(N / 2) / 2)); }

cudaError_t launch_xpass_real(int N, XMode mode, const XParams &p, int grid, cudaStream_t s) {
#define XR_CASE(n)                                                           \
    case n:                                                                  \
        if (mode == X_SRC_FWD) return xreal_t<n, X_SRC_FWD>(p, grid, s);     \
        if (mode == X_SRC_EPI) return xreal_t<n, X_SRC_EPI>(p, grid, s);     \
        return xreal_t<n, X_ITER>(p, grid, s);
    switch (N) { XR_CASE(32) XR_CASE(64) XR_CASE(128) XR_CASE(256) XR_CASE(512) XR_CASE(1024) XR_CASE(2048)
    default: return cudaErrorInvalidValue; }
#undef XR_CASE
}

}  // namespace usp
