// kernels_anti.cu -- the antisymmetrised system (
// PAPER.md Eq. 9-10) for problems whose numerical range is not
// confined to a half plane (e.g. gain media), where the standard canonical
// form does not apply:
//
//     E = [x; x'],   A = c^-1 [[0, -A_raw^*], [A_raw, 0]]   (c REAL: A skew-Hermitian),
//     s = c^-1 [0; S]  (no adjoint problem: s' = 0),  v = (w - sigma)/c pointwise,
//     B = 1 - V = [[1, conj v], [-v, 1]]                                (pointwise 2x2)
//     (L+1)^-1 = F^-1 [[1, conj a], [-a, 1]] / (1 + |a|^2) F,  a = (D|p|^2 + sigma)/c   (per mode 2x2)
//
// Algorithm 1 in the Delta-form (L613, reading R-17) on the two-component
// field.  The components are stored component-major ([comp][z][y][x]), so the
// y / z FFT passes are the k_stile kernels run over 2 x the planes; the
// component coupling lives in
//   k_anti_pipe (per x-line pair, TMA-pipelined) x inverse FFT of both
//               components -> update Delta, x (2x2 B) + residual -> u = B Delta
//               -> x forward FFT
//   k_anti_x    the same line structure, register-staged, for the source setup
//               (s -> F_x s; Delta_0 = B (L+1)^-1 s)
//   k_anti_mul  (per Fourier mode) the 2x2 symbol of (L+1)^-1 with 1/N_vox
// A capability path, not the bench path.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fft_core.cuh"
#include "kcommon.cuh"
#include "tma.cuh"
#include "usp_internal.h"

namespace usp {

template <int N>
struct AX {
    using G = LineGeo<N>;
    static constexpr int NT = 128;
    static constexpr int LPC = NT / G::N1;   // line pairs per CTA step
    static constexpr int SMEM = LPC * LayRow<N>::kFloat2PerLine * 8;
};

template <int N, int MODE>
__global__ void __launch_bounds__(AX<N>::NT) k_anti_x(AParams p) {
    using G = LineGeo<N>;
    using T = AX<N>;
    extern __shared__ float2 smem_a[];
    __shared__ double sh_red[T::NT / 32];
    const int tid = threadIdx.x, lq = tid / G::N1, j = tid % G::N1;
    const LayRow<N> lay{smem_a + lq * LayRow<N>::kFloat2PerLine};
    const long long n = p.nlines * (long long)N;    // voxels per component
    double acc = 0.0;
    const long long ng = (p.nlines + T::LPC - 1) / T::LPC;
    for (long long g = blockIdx.x; g < ng; g += gridDim.x) {
        const long long line = g * T::LPC + lq;
        const bool valid = line < p.nlines;
        const long long base = line * N + j;
        float2 a[G::N2], b[G::N2];
        if (MODE == X_SRC_FWD) {
            // s = [0; S/c], the raw source staged in the first component of x
#pragma unroll
            for (int m = 0; m < G::N2; ++m) {
                const long long i = base + G::N1 * m;
                a[m] = make_float2(0.f, 0.f);
                b[m] = valid ? cscale(p.x[i], p.inv_c) : make_float2(0.f, 0.f);
            }
        } else {
#pragma unroll
            for (int m = 0; m < G::N2; ++m) {
                const long long i = base + G::N1 * m;
                a[m] = valid ? cconj(p.work[i]) : make_float2(0.f, 0.f);
                b[m] = valid ? cconj(p.work[n + i]) : make_float2(0.f, 0.f);
            }
            fft_line<N, false, LayRow<N>>(a, lay, j, p.tw);   // x inverse (conj trick), component 1
            fft_line<N, false, LayRow<N>>(b, lay, j, p.tw);   // component 2
            float lacc = 0.f;
#pragma unroll
            for (int m = 0; m < G::N2; ++m) {
                const long long i = base + G::N1 * m;
                const float2 y1 = cconj(a[m]), y2 = cconj(b[m]);
                const float2 v = valid ? p.v[i] : make_float2(0.f, 0.f);
                // Delta_0 = B (L+1)^-1 s, x_0 = 0
                const float2 d1 = cadd(y1, cmulc(y2, v));    // y1 + conj(v) y2
                const float2 d2 = csub(y2, cmul(v, y1));     // -v y1 + y2
                if (valid) {
                    p.x[i] = make_float2(0.f, 0.f);
                    p.x[n + i] = make_float2(0.f, 0.f);
                    p.delta[i] = d1;
                    p.delta[n + i] = d2;
                }
                lacc += cabs2(d1) + cabs2(d2);
                a[m] = cadd(d1, cmulc(d2, v));               // u = B Delta
                b[m] = csub(d2, cmul(v, d1));
            }
            acc += (double)lacc;
        }
        fft_line<N, false, LayRow<N>>(a, lay, j, p.tw);       // x forward
        fft_line<N, false, LayRow<N>>(b, lay, j, p.tw);
        if (valid)
#pragma unroll
            for (int m = 0; m < G::N2; ++m) {
                const long long i = base + G::N1 * m;
                p.work[i] = a[m];
                p.work[n + i] = b[m];
            }
    }
    if (MODE == X_SRC_FWD) return;
    double total;
    const double mine = block_sum_d<T::NT>(acc, sh_red);
    if (!last_block_total<T::NT>(mine, p.st, p.red.partials, sh_red, &total)) return;
    if (threadIdx.x != 0) return;
    finish_xpass(true, false, total, p.st, p.red);
}

// The iteration's x pass, TMA-pipelined (k_xpass_pipe's structure): one
// producer warp bulk-copies a unit's seven line slots -- work, Delta, x of
// both components and v -- into the consumer warp's stage; the consumer runs
// the two components through the line FFT one at a time (y_1 parked in its
// own stage slot, so only one component is live in registers), the 2x2
// update (the same arithmetic as k_anti_x), u = B Delta (u_1 parked in the
// stage again) and the two forward FFTs.  Measured on B200 (256^3): the
// register-staged k_anti_x ran at 33 % of the copy bandwidth.
constexpr int kAntiSmemBudget = 232448 - 2048;

template <int N>
struct APipe {
    using G = LineGeo<N>;
    static constexpr int U = 32 / G::N1;                 // lines per warp unit
    static constexpr int UE = 32 * G::N2;                // elements per unit
    static constexpr int NSLOT = 7;                      // W1 W2 D1 D2 X1 X2 V
    static constexpr int STAGE = NSLOT * UE;
    static constexpr int XBUF = U * LayRow<N>::kFloat2PerLine;
    static constexpr int XC0 = (kAntiSmemBudget - N * 8) / ((STAGE + XBUF) * 8);
    static constexpr int XC = XC0 > 6 ? 6 : XC0;         // consumer warps, one stage each
    static_assert(XC >= 2, "antisymmetrised x pipeline needs >= 2 consumer warps");
    static constexpr int S = XC;
    static constexpr int NT = 32 * (XC + 1);
    static constexpr int SMEM = (S * STAGE + XC * XBUF + N) * 8 + 2 * S * 8;
};

template <int N>
__global__ void __launch_bounds__(APipe<N>::NT, 1) k_anti_pipe(AParams p) {
    using G = LineGeo<N>;
    using T = APipe<N>;
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
    const long long n = p.nlines * (long long)N;          // voxels per component
    double acc = 0.0;
    if (xonly) {   // the final x += alpha Delta after the stop test (R-5)
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < 2 * n;
             i += (long long)gridDim.x * blockDim.x) {
            const float2 d = p.delta[i], xx = p.x[i];
            p.x[i] = make_float2(fmaf(alpha, d.x, xx.x), fmaf(alpha, d.y, xx.y));
        }
    } else {
        if (threadIdx.x == 0) {
            for (int s = 0; s < T::S; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&empty[s], 1);
            }
            fence_mbar_init();
        }
        load_twiddles<N>(sm_tw, p.tw);
        __syncthreads();
        const long long nunits = p.nlines / T::U;
        const int nloc = (int)((nunits - blockIdx.x + gridDim.x - 1) / gridDim.x);
        const uint32_t ub = T::UE * 8u;
        if (warp == T::XC) {
            if (lane == 0) {   // producer
                for (int i = 0; i < nloc; ++i) {
                    const int s = i % T::S;
                    if (i >= T::S && !mbar_wait(&empty[s], ((i / T::S) - 1) & 1)) {
                        if (atomicCAS(&p.st->err, 0, 31) == 0) p.st->err_info = i;
                        break;
                    }
                    const long long off = (blockIdx.x + (long long)i * gridDim.x) * T::UE;
                    float2 *st = stages + s * T::STAGE;
                    mbar_arrive_expect_tx(&full[s], T::NSLOT * ub);
                    bulk_g2s(st, p.work + off, ub, &full[s]);
                    bulk_g2s(st + T::UE, p.work + n + off, ub, &full[s]);
                    bulk_g2s(st + 2 * T::UE, p.delta + off, ub, &full[s]);
                    bulk_g2s(st + 3 * T::UE, p.delta + n + off, ub, &full[s]);
                    bulk_g2s(st + 4 * T::UE, p.x + off, ub, &full[s]);
                    bulk_g2s(st + 5 * T::UE, p.x + n + off, ub, &full[s]);
                    bulk_g2s(st + 6 * T::UE, p.v + off, ub, &full[s]);
                }
            }
            __syncwarp();
        } else {
            const int lq = lane / G::N1, j = lane % G::N1;
            const LayRow<N> lay{xbufs + warp * T::XBUF + lq * LayRow<N>::kFloat2PerLine};
            for (int i = warp; i < nloc; i += T::XC) {
                const int s = i % T::S;
                if (!mbar_wait(&full[s], (i / T::S) & 1)) {
                    if (lane == 0 && atomicCAS(&p.st->err, 0, 32) == 0) p.st->err_info = i;
                    break;
                }
                float2 *st = stages + s * T::STAGE;
                const long long gb = (blockIdx.x + (long long)i * gridDim.x) * T::UE + lq * N + j;
                const int sb = lq * N + j;
                float2 v[G::N2];
                // component 1: x inverse (conj trick); y_1 parked in its own slot
#pragma unroll
                for (int m = 0; m < G::N2; ++m) v[m] = cconj(st[sb + G::N1 * m]);
                fft_line<N, false, LayRow<N>, true>(v, lay, j, sm_tw);
#pragma unroll
                for (int m = 0; m < G::N2; ++m) st[sb + G::N1 * m] = cconj(v[m]);
                // component 2
#pragma unroll
                for (int m = 0; m < G::N2; ++m) v[m] = cconj(st[T::UE + sb + G::N1 * m]);
                fft_line<N, false, LayRow<N>, true>(v, lay, j, sm_tw);
                float lacc = 0.f;
#pragma unroll
                for (int m = 0; m < G::N2; ++m) {
                    const int e = sb + G::N1 * m;
                    const long long gi = gb + G::N1 * m;
                    const float2 y1 = st[e], y2 = cconj(v[m]);
                    const float2 o1 = st[2 * T::UE + e], o2 = st[3 * T::UE + e];
                    const float2 x1 = st[4 * T::UE + e], x2 = st[5 * T::UE + e], vv = st[6 * T::UE + e];
                    const float2 e1 = csub(y1, o1), e2 = csub(y2, o2);
                    const float2 g1 = cadd(e1, cmulc(e2, vv)), g2 = csub(e2, cmul(vv, e1));   // B (y - Delta)
                    const float2 d1 = make_float2(fmaf(alpha, g1.x, o1.x), fmaf(alpha, g1.y, o1.y));
                    const float2 d2 = make_float2(fmaf(alpha, g2.x, o2.x), fmaf(alpha, g2.y, o2.y));
                    p.x[gi] = make_float2(fmaf(alpha, o1.x, x1.x), fmaf(alpha, o1.y, x1.y));
                    p.x[n + gi] = make_float2(fmaf(alpha, o2.x, x2.x), fmaf(alpha, o2.y, x2.y));
                    p.delta[gi] = d1;
                    p.delta[n + gi] = d2;
                    lacc += cabs2(d1) + cabs2(d2);
                    st[e] = cadd(d1, cmulc(d2, vv));                  // u_1 = (B Delta)_1, parked
                    v[m] = csub(d2, cmul(vv, d1));                    // u_2
                }
                acc += (double)lacc;
                __syncwarp();
                fft_line<N, false, LayRow<N>, true>(v, lay, j, sm_tw);   // x forward, component 2
#pragma unroll
                for (int m = 0; m < G::N2; ++m) p.work[n + gb + G::N1 * m] = v[m];
#pragma unroll
                for (int m = 0; m < G::N2; ++m) v[m] = st[sb + G::N1 * m];
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);           // the stage can refill now
                fft_line<N, false, LayRow<N>, true>(v, lay, j, sm_tw);   // component 1
#pragma unroll
                for (int m = 0; m < G::N2; ++m) p.work[gb + G::N1 * m] = v[m];
            }
        }
    }
    double total;
    const double mine = block_sum_d<T::NT>(acc, sh_red);
    if (!last_block_total<T::NT>(mine, p.st, p.red.partials, sh_red, &total)) return;
    if (threadIdx.x != 0) return;
    finish_xpass(false, xonly, total, p.st, p.red);
}

template <int N>
static cudaError_t anti_pipe_t(const AParams &p, int grid, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_anti_pipe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, APipe<N>::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    k_anti_pipe<N><<<grid, APipe<N>::NT, APipe<N>::SMEM, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_anti_pipe(int N, const AParams &p, int grid, cudaStream_t s) {
    switch (N) {
    case 64: return anti_pipe_t<64>(p, grid, s);
    case 128: return anti_pipe_t<128>(p, grid, s);
    case 256: return anti_pipe_t<256>(p, grid, s);
    case 512: return anti_pipe_t<512>(p, grid, s);
    case 1024: return anti_pipe_t<1024>(p, grid, s);
    default: return cudaErrorInvalidValue;
    }
}

int anti_pipe_units(int N) { return 32 / (1 << (ilog2(N) / 2)); }

// Per Fourier mode: [u1; u2] <- [[1, conj a], [-a, 1]] [u1; u2] / ((1 + |a|^2) N_vox),
// a = (D |p|^2 + sigma) / c.  One warp per x row (|p_y|^2 + |p_z|^2 once per
// row), two modes per lane per 16-byte access.  Skips itself after a stop
// (check_state).
__global__ void __launch_bounds__(256) k_anti_mul(AParams p, int check_state) {
    if (check_state && (p.st->status != ST_RUNNING || p.st->k >= p.st->kmax)) return;
    const long long n = p.nvox;
    const MulParams &mp = p.mp;
    const long long rows = n / mp.nx;
    const int lane = threadIdx.x & 31;
    const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    float4 *u1p = reinterpret_cast<float4 *>(p.work), *u2p = reinterpret_cast<float4 *>(p.work + n);
    for (long long r = w0; r < rows; r += nw) {
        const int iy = (int)(r % mp.ny), iz = (int)(r / mp.ny);
        const float py = mp.ky * freq_m(iy, mp.ny);
        const float pz = mp.nz > 1 ? mp.kz * freq_m(iz, mp.nz) : 0.f;   // 2-D: no z
        const float pyz = fmaf(py, py, pz * pz);
        for (int e = 2 * lane; e < mp.nx; e += 64) {
            const long long q = (r * mp.nx + e) >> 1;
            const float4 A = u1p[q], Bv = u2p[q];
            float2 u1[2] = {make_float2(A.x, A.y), make_float2(A.z, A.w)};
            float2 u2[2] = {make_float2(Bv.x, Bv.y), make_float2(Bv.z, Bv.w)};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float px = mp.kx * freq_m(e + h, mp.nx);
                const float p2 = fmaf(px, px, pyz);
                // a = (D p^2 + sigma) / c  (c real: p.inv_c = 1/c); det = 1 + |a|^2; folded 1/N_vox
                const float2 a = make_float2((mp.D * p2 + p.sigma.x) * p.inv_c, p.sigma.y * p.inv_c);
                const float s = p.inv_n / (1.f + cabs2(a));
                const float2 v1 = cscale(cadd(u1[h], cmulc(u2[h], a)), s);   // u1 + conj(a) u2
                const float2 v2 = cscale(csub(u2[h], cmul(a, u1[h])), s);    // u2 - a u1
                u1[h] = v1;
                u2[h] = v2;
            }
            u1p[q] = make_float4(u1[0].x, u1[0].y, u1[1].x, u1[1].y);
            u2p[q] = make_float4(u2[0].x, u2[0].y, u2[1].x, u2[1].y);
        }
    }
}

// ========================================================= launchers ====
template <int N, int MODE>
static cudaError_t anti_x_t(const AParams &p, int grid, cudaStream_t s) {
    k_anti_x<N, MODE><<<grid, AX<N>::NT, AX<N>::SMEM, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_anti_x(int N, XMode mode, const AParams &p, int grid, cudaStream_t s) {
#define AX_CASE(n)                                                        \
    case n:                                                               \
        if (mode == X_SRC_FWD) return anti_x_t<n, X_SRC_FWD>(p, grid, s); \
        if (mode == X_SRC_EPI) return anti_x_t<n, X_SRC_EPI>(p, grid, s); \
        return cudaErrorInvalidValue;   /* X_ITER: k_anti_pipe */
    switch (N) { AX_CASE(64) AX_CASE(128) AX_CASE(256) AX_CASE(512) AX_CASE(1024)
    default: return cudaErrorInvalidValue; }
#undef AX_CASE
}

cudaError_t launch_anti_mul(const AParams &p, int check_state, int grid, cudaStream_t s) {
    k_anti_mul<<<resident_grid<k_anti_mul>(grid, 256), 256, 0, s>>>(p, check_state);
    return cudaGetLastError();
}

int anti_lines_per_cta(int N) { return 128 / (1 << (ilog2(N) / 2)); }

}  // namespace usp
