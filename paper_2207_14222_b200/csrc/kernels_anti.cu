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
//   k_anti_x   (per x-line pair) x inverse FFT of both components -> update
//              Delta, x (2x2 B) + residual -> u = B Delta -> x forward FFT
//   k_anti_mul (per Fourier mode) the 2x2 symbol of (L+1)^-1 with 1/N_vox
// Register-staged (the component pair doubles the fields a line needs, which
// leaves no room for TMA stages of useful depth); this is a capability path,
// not the bench path.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fft_core.cuh"
#include "kcommon.cuh"
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
    bool xonly = false;
    float alpha = 0.f;
    if (MODE == X_ITER) {
        const int status = p.st->status;
        if (p.st->k >= p.st->kmax || (status != ST_RUNNING && status != ST_STOP_PENDING)) return;
        xonly = status == ST_STOP_PENDING;
        alpha = (float)p.st->alpha;
    }
    const long long n = p.nlines * (long long)N;    // voxels per component
    double acc = 0.0;
    const long long ng = (p.nlines + T::LPC - 1) / T::LPC;
    for (long long g = blockIdx.x; g < ng; g += gridDim.x) {
        const long long line = g * T::LPC + lq;
        const bool valid = line < p.nlines;
        const long long base = line * N + j;
        float2 a[G::N2], b[G::N2];
        if (MODE == X_ITER && xonly) {
            if (valid)
#pragma unroll
                for (int m = 0; m < G::N2; ++m) {
                    const long long i = base + G::N1 * m;
                    for (int q = 0; q < 2; ++q) {
                        const float2 d = p.delta[q * n + i], xx = p.x[q * n + i];
                        p.x[q * n + i] = make_float2(fmaf(alpha, d.x, xx.x), fmaf(alpha, d.y, xx.y));
                    }
                }
            continue;
        }
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
                float2 d1, d2;
                if (MODE == X_SRC_EPI) {   // Delta_0 = B (L+1)^-1 s, x_0 = 0
                    d1 = cadd(y1, cmulc(y2, v));             // y1 + conj(v) y2
                    d2 = csub(y2, cmul(v, y1));              // -v y1 + y2
                    if (valid) {
                        p.x[i] = make_float2(0.f, 0.f);
                        p.x[n + i] = make_float2(0.f, 0.f);
                    }
                } else {
                    const float2 o1 = valid ? p.delta[i] : make_float2(0.f, 0.f);
                    const float2 o2 = valid ? p.delta[n + i] : make_float2(0.f, 0.f);
                    const float2 e1 = csub(y1, o1), e2 = csub(y2, o2);
                    const float2 g1 = cadd(e1, cmulc(e2, v)), g2 = csub(e2, cmul(v, e1));   // B (y - Delta)
                    d1 = make_float2(fmaf(alpha, g1.x, o1.x), fmaf(alpha, g1.y, o1.y));
                    d2 = make_float2(fmaf(alpha, g2.x, o2.x), fmaf(alpha, g2.y, o2.y));
                    if (valid) {
                        const float2 x1 = p.x[i], x2 = p.x[n + i];
                        p.x[i] = make_float2(fmaf(alpha, o1.x, x1.x), fmaf(alpha, o1.y, x1.y));
                        p.x[n + i] = make_float2(fmaf(alpha, o2.x, x2.x), fmaf(alpha, o2.y, x2.y));
                    }
                }
                if (valid) {
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
    finish_xpass(MODE == X_SRC_EPI, xonly, total, p.st, p.red);
}

// Per Fourier mode: [u1; u2] <- [[1, conj a], [-a, 1]] [u1; u2] / ((1 + |a|^2) N_vox),
// a = (D |p|^2 + sigma) / c.  Skips itself after a stop (check_state).
__global__ void __launch_bounds__(256) k_anti_mul(AParams p, int check_state) {
    if (check_state && (p.st->status != ST_RUNNING || p.st->k >= p.st->kmax)) return;
    const long long n = p.nvox;
    const MulParams &mp = p.mp;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int ix = (int)(i % mp.nx);
        const long long r = i / mp.nx;
        const int iy = (int)(r % mp.ny), iz = (int)(r / mp.ny);
        const float px = mp.kx * freq_m(ix, mp.nx), py = mp.ky * freq_m(iy, mp.ny);
        const float pz = mp.nz > 1 ? mp.kz * freq_m(iz, mp.nz) : 0.f;   // 2-D: no z
        const float p2 = fmaf(px, px, fmaf(py, py, pz * pz));
        // a = (D p^2 + sigma) / c  (c real: p.inv_c = 1/c); det = 1 + |a|^2; folded 1/N_vox
        const float2 a = make_float2((mp.D * p2 + p.sigma.x) * p.inv_c, p.sigma.y * p.inv_c);
        const float s = p.inv_n / (1.f + cabs2(a));
        const float2 u1 = p.work[i], u2 = p.work[n + i];
        p.work[i] = cscale(cadd(u1, cmulc(u2, a)), s);          // u1 + conj(a) u2
        p.work[n + i] = cscale(csub(u2, cmul(a, u1)), s);       // u2 - a u1
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
        return anti_x_t<n, X_ITER>(p, grid, s);
    switch (N) { AX_CASE(64) AX_CASE(128) AX_CASE(256) AX_CASE(512) AX_CASE(1024)
    default: return cudaErrorInvalidValue; }
#undef AX_CASE
}

cudaError_t launch_anti_mul(const AParams &p, int check_state, int grid, cudaStream_t s) {
    k_anti_mul<<<grid, 256, 0, s>>>(p, check_state);
    return cudaGetLastError();
}

int anti_lines_per_cta(int N) { return 128 / (1 << (ilog2(N) / 2)); }

}  // namespace usp
