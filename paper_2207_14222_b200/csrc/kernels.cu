// kernels.cu -- sm_100a kernels of the universal-split-preconditioner hot path
// that are not pass pipelines: the register-staged strided pass for short
// lines (N = 16, 32), the on-chip 1-D solve, the setup kernels (potential,
// farthest point of the smallest-circle search), the rank-ordered residual
// finish, and small state / copy kernels.
//
// One iteration of Algorithm 1 is a chain of FFT passes:
//
//   3-D:  K_B  y forward                               (k_stile<S_FWD>, kernels_stile.cu)
//         K_C  z forward, x g(p), z inverse  (Eq. 12)  (k_stile<S_FWD_MUL_INV>)
//         K_D  y inverse                               (k_stile<S_INV>)
//         K_A  x inverse -> update -> prologue -> x forward   (k_xpass_pipe, kernels_pipe.cu)
//   2-D:  one persistent cooperative kernel (kernels_small.cu), or K_Y (y forward,
//         x g, y inverse) and K_A per pass
//   1-D:  one CTA runs the whole solve (k_solve1d, here).
//
// K_A's update is Algorithm 1 lines 3-4 (x-form while r_k >= r_switch) or the
// Delta-form of L613 (readings R-17, R-30):
//     y = (L+1)^-1 u                      (the chain that just completed)
//     x-form:  Delta_k = B (y - x_k),  x_{k+1} = x_k + alpha Delta_k,  u = B x_{k+1} + s
//     Delta-form: x_{k+1} = x_k + alpha Delta_k,
//              Delta_{k+1} = Delta_k + alpha B (y - Delta_k),  u = B Delta_{k+1}
//     r = ||Delta|| / n0                  (line 5, reading R-4)
// The residual is reduced per CTA (fp32 per line -> fp64), and the last CTA
// to finish sums the CTA partials in a fixed order (deterministic) and
// updates the device-side IterState (stop flag, counter, history).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "fft_core.cuh"
#include "kcommon.cuh"
#include "usp_internal.h"

namespace usp {

// ========================================================== strided pass ==
// Strided axes (y: stride nx, z: stride nx*ny).  A CTA transforms tiles of
// COLS adjacent columns x N rows; thread (c, j) owns column c and rows
// j + N1*m.  A warp load/store touches 32/COLS rows of COLS*8 contiguous
// bytes.  COLS = 8 with N1 = 32 gives 256-thread CTAs, two per SM, so one
// CTA's loads overlap the other's FFT arithmetic.  The inverse transform is
// computed as conj(DFT(conj(.))) so a single FFT body is compiled and the
// kernel stays inside the instruction cache; twiddles are read from smem.
template <int N, int COLS>
struct SGeo {
    using G = LineGeo<N>;
    static constexpr int NT = COLS * G::N1;
    static constexpr int PAD = (COLS == 16 || COLS == 32) ? 0 : 8;
    static constexpr int PITCH = G::N2 * COLS + PAD;                    // float2 per n1 row
    static constexpr int SMEM = (G::N1 * PITCH + N) * (int)sizeof(float2);   // exchange + twiddles
    static constexpr int MINB = (NT <= 256) ? 2 : 1;
};

template <int N, int MODE, int COLS>
__global__ void __launch_bounds__(SGeo<N, COLS>::NT, SGeo<N, COLS>::MINB) k_strided(SParams p) {
    using G = LineGeo<N>;
    using SG = SGeo<N, COLS>;
    extern __shared__ float2 smem[];
    float2 *sm_tw = smem + G::N1 * SG::PITCH;
    const int tid = threadIdx.x;
    const int c = tid % COLS, j = tid / COLS;
    if (p.check_state && !iter_running(p.st)) return;
    load_twiddles<N>(sm_tw, p.tw);
    __syncthreads();
    const LayCol<N, COLS, SG::PAD, 0> lay{smem, c};
    const long long tpo = p.ncols / COLS;
    const long long ntiles = tpo * p.nouter;
    constexpr int NPASS = (MODE == S_FWD_MUL_INV) ? 2 : 1;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long o = tile / tpo;
        const long long col = (tile - o * tpo) * COLS + c;
        const float2 *lb = p.data + (o * p.ostride + col) + (long long)j * p.stride;
        const long long lstep = (long long)G::N1 * p.stride;
        float2 v[G::N2];
#pragma unroll
        for (int m = 0; m < G::N2; ++m) {
            const float2 t = lb[m * lstep];
            v[m] = (MODE == S_INV) ? cconj(t) : t;
        }
#pragma unroll 1
        for (int pass = 0; pass < NPASS; ++pass) {
            fft_line<N, false, LayCol<N, COLS, SG::PAD, 0>, true>(v, lay, j, sm_tw);
            if (MODE == S_FWD_MUL_INV && pass == 0) {
                // (L+1)^-1 multiplier, Eq. 12: |p|^2 = px^2 + py^2 + p_line^2; then
                // conjugate so the second forward DFT computes the inverse.
                float pt2;
                if (p.line_axis == 2) {
                    const int ix = (int)(col % p.mp.nx), iy = (int)(col / p.mp.nx);
                    const float px = p.mp.kx * freq_m(ix, p.mp.nx), py = p.mp.ky * freq_m(iy, p.mp.ny);
                    pt2 = fmaf(px, px, py * py);
                } else {
                    const float px = p.mp.kx * freq_m((int)col, p.mp.nx);
                    pt2 = px * px;
                }
                const float kl = (p.line_axis == 2) ? p.mp.kz : p.mp.ky;
#pragma unroll
                for (int m = 0; m < G::N2; ++m) {
                    const float pl = kl * freq_m(j + G::N1 * m, N);
                    v[m] = cconj(cmul(v[m], multiplier(p.mp, fmaf(pl, pl, pt2))));
                }
            }
        }
        // recompute the store addresses (an opaque stride keeps the compiler from
        // holding 32 load addresses live across the FFT, which would spill)
        long long stride = p.stride;
        asm volatile("" : "+l"(stride));
        float2 *sb = p.data + (o * p.ostride + col) + (long long)j * stride;
        const long long step = (long long)G::N1 * stride;
#pragma unroll
        for (int m = 0; m < G::N2; ++m) {
            sb[0] = (MODE == S_FWD) ? v[m] : cconj(v[m]);
            sb += step;
        }
    }
}

// =================================================================== 1-D ==
// The whole 1-D solve in one CTA (one line; latency bound):
// O_SETUP computes Delta_0 = B (L+1)^-1 (S/c), n0, x_0 = 0; O_ITER loops the
// iteration on-chip until the stop test or kmax, then writes the state back.
template <int N>
__device__ __forceinline__ void mul_line(float2 (&v)[LineGeo<N>::N2], const MulParams &mp, int j) {
    using G = LineGeo<N>;
#pragma unroll
    for (int m = 0; m < G::N2; ++m) {
        const float pl = mp.kx * freq_m(j + G::N1 * m, N);
        v[m] = cmul(v[m], multiplier(mp, pl * pl));
    }
}

template <int N, int MODE>
__global__ void __launch_bounds__(LineGeo<N>::N1) k_solve1d(OneParams p) {
    using G = LineGeo<N>;
    __shared__ float2 smem[LayRow<N>::kFloat2PerLine];
    const int j = threadIdx.x;
    const LayRow<N> lay{smem};
    float2 b[G::N2], d[G::N2], xx[G::N2], v[G::N2];
#pragma unroll
    for (int m = 0; m < G::N2; ++m) b[m] = p.B[j + G::N1 * m];
    IterState *st = p.st;

    if constexpr (MODE == O_SETUP) {
#pragma unroll
        for (int m = 0; m < G::N2; ++m) {
            const int i = j + G::N1 * m;
            const float2 sv = p.src_real ? make_float2(reinterpret_cast<const float *>(p.x)[i], 0.f) : p.x[i];
            v[m] = cmul(sv, p.inv_c);
        }
        fft_line<N, false>(v, lay, j, p.tw);
        mul_line<N>(v, p.mp, j);
        fft_line<N, true>(v, lay, j, p.tw);
        float lacc = 0.f;
#pragma unroll
        for (int m = 0; m < G::N2; ++m) {
            d[m] = cmul(b[m], v[m]);
            lacc += cabs2(d[m]);
            p.delta[j + G::N1 * m] = d[m];
            p.x[j + G::N1 * m] = make_float2(0.f, 0.f);
        }
        const double n0 = sqrt(warp_sum_d((double)lacc));
        if (j == 0) {
            st->n0 = n0;
            st->r = n0 > 0.0 ? 1.0 : 0.0;
            st->k = 0;
            st->status = n0 > 0.0 ? ST_RUNNING : ST_DONE_CONV;
            if (n0 > 0.0 && st->tol > 0.0 && 1.0 < st->tol) st->status = ST_STOP_PENDING;
            p.red.hist[0] = st->r;
        }
        return;
    } else {

#pragma unroll
    for (int m = 0; m < G::N2; ++m) {
        d[m] = p.delta[j + G::N1 * m];
        xx[m] = p.x[j + G::N1 * m];
    }
    const float alpha = (float)st->alpha;
    const double tol = st->tol, n0 = st->n0;
    long long k = st->k;
    const long long kmax = st->kmax;
    int status = st->status;
    double r = st->r;
    while (k < kmax && status == ST_RUNNING) {
#pragma unroll
        for (int m = 0; m < G::N2; ++m) v[m] = cmul(b[m], d[m]);
        fft_line<N, false>(v, lay, j, p.tw);
        mul_line<N>(v, p.mp, j);
        fft_line<N, true>(v, lay, j, p.tw);
        float lacc = 0.f;
#pragma unroll
        for (int m = 0; m < G::N2; ++m) {
            xx[m] = make_float2(fmaf(alpha, d[m].x, xx[m].x), fmaf(alpha, d[m].y, xx[m].y));
            const float2 t = cmul(b[m], csub(v[m], d[m]));
            d[m] = make_float2(fmaf(alpha, t.x, d[m].x), fmaf(alpha, t.y, d[m].y));
            lacc += cabs2(d[m]);
        }
        r = sqrt(warp_sum_d((double)lacc)) / n0;
        ++k;
        if (j == 0) p.red.hist[k % p.red.hist_cap] = r;
        if (!(r <= 1e6)) status = ST_DIVERGED;
        else if (tol > 0.0 && r < tol) status = ST_STOP_PENDING;
    }
    if (status == ST_STOP_PENDING && k < kmax) {
#pragma unroll
        for (int m = 0; m < G::N2; ++m) xx[m] = make_float2(fmaf(alpha, d[m].x, xx[m].x), fmaf(alpha, d[m].y, xx[m].y));
        ++k;
        status = ST_DONE_CONV;
    }
#pragma unroll
    for (int m = 0; m < G::N2; ++m) {
        p.delta[j + G::N1 * m] = d[m];
        p.x[j + G::N1 * m] = xx[m];
    }
    if (j == 0) {
        st->k = k;
        st->r = r;
        st->status = status;
    }
    }
}

// ================================================================= setup ==
// V = (w - sigma)/c, B = 1 - V, with the Theorem 1
// hypotheses checked pointwise: |V| < 1 and Re(w/c) >= 0 (accretive A for
// D Re(c) >= 0, Eq. 1).
__global__ void __launch_bounds__(256) k_potential(PotParams p) {
    double v2max = 0.0;   // max |V|^2 (one sqrt per thread at the end: sqrt is monotonic)
    unsigned nacc = 0, nnf = 0;
    const double cr = p.c_re, ci = p.c_im, inv_c2 = 1.0 / (cr * cr + ci * ci);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < p.n;
         i += (long long)gridDim.x * blockDim.x) {
        double mr, mi;
        if (p.medium_real) {
            mr = reinterpret_cast<const float *>(p.medium)[i];
            mi = 0.0;
        } else {
            const float2 m = reinterpret_cast<const float2 *>(p.medium)[i];
            mr = m.x;
            mi = m.y;
        }
        const double wr = p.medium_is_k2 ? -mr : mr, wi = p.medium_is_k2 ? -mi : mi;
        const double ar = wr - p.sig_re, ai = wi - p.sig_im;
        // V = (w - sigma)/c = (w - sigma) conj(c) / |c|^2
        const double vr = (ar * cr + ai * ci) * inv_c2, vi = (ai * cr - ar * ci) * inv_c2;
        const double av2 = vr * vr + vi * vi;
        if (!isfinite(vr) || !isfinite(vi)) ++nnf;
        v2max = fmax(v2max, av2);
        // Re(w/c) < -1e-6 |w/c|, without the square root
        const double wcr = (wr * cr + wi * ci) * inv_c2, wci = (wi * cr - wr * ci) * inv_c2;
        if (!p.store_v && wcr < 0.0 && wcr * wcr > 1e-12 * (wcr * wcr + wci * wci)) ++nacc;
        if (p.store_v) p.B[i] = make_float2((float)vr, (float)vi);
        else if (p.b_real) reinterpret_cast<float *>(p.B)[i] = (float)(1.0 - vr);
        else p.B[i] = make_float2((float)(1.0 - vr), (float)(-vi));
    }
    float vmax = (float)sqrt(v2max);
    if (v2max >= 1.0) vmax = fmaxf(vmax, 1.0f);
    // CTA reduce then one atomic each
    __shared__ float smax[8];
    __shared__ unsigned sacc[8], snf[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
        nacc += __shfl_xor_sync(0xffffffffu, nacc, o);
        nnf += __shfl_xor_sync(0xffffffffu, nnf, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        smax[w] = vmax;
        sacc[w] = nacc;
        snf[w] = nnf;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            smax[0] = fmaxf(smax[0], smax[i]);
            sacc[0] += sacc[i];
            snf[0] += snf[i];
        }
        atomicMax(p.max_absV_bits, __float_as_uint(smax[0]));
        if (sacc[0]) atomicAdd(p.n_nonaccretive, sacc[0]);
        if (snf[0]) atomicAdd(p.n_nonfinite, snf[0]);
    }
}

// Farthest medium value from (cre, cim) -- one pass of the smallest-circle
// driver (usp_api.cu).  Exact double distances of the complex64 values.
__global__ void __launch_bounds__(256) k_farthest(FarParams p) {
    double best = -1.0;
    long long bi = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < p.n;
         i += (long long)gridDim.x * blockDim.x) {
        double mr, mi;
        if (p.medium_real) {
            mr = reinterpret_cast<const float *>(p.medium)[i];
            mi = 0.0;
        } else {
            const float2 m = reinterpret_cast<const float2 *>(p.medium)[i];
            mr = m.x;
            mi = m.y;
        }
        const double dx = mr - p.cre, dy = mi - p.cim, d2 = dx * dx + dy * dy;
        if (d2 > best) {
            best = d2;
            bi = i;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
        }
    }
    __shared__ double sb[8];
    __shared__ long long si[8];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        sb[w] = best;
        si[w] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i)
            if (sb[i] > sb[0] || (sb[i] == sb[0] && si[i] < si[0])) {
                sb[0] = sb[i];
                si[0] = si[i];
            }
        p.best_d2[blockIdx.x] = sb[0];
        p.best_idx[blockIdx.x] = si[0];
    }
}

// Slab-decomposed runs: after the all-gather of the ranks' x-pass totals,
// every rank sums them in rank order (deterministic, identical on all ranks)
// and takes the same stop decision (reading R-4).
__global__ void k_finish(IterState *st, const double *sums, int P, int src_epi, Red red) {
    bool xonly = false;
    int act = ACT_DELTA;
    if (!src_epi) {
        const int status = st->status;
        const bool probe = st->form == FORM_PROBE && status == ST_RUNNING;
        if (!probe && (st->k >= st->kmax || (status != ST_RUNNING && status != ST_STOP_PENDING))) return;
        xonly = (status == ST_STOP_PENDING);
        act = xform_act(st);   // unchanged since the x pass read it (it did not finish)
    }
    double total = 0.0;
    for (int q = 0; q < P; ++q) total += sums[q];
    finish_xpass(src_epi != 0, xonly, total, st, red, act);
}

__global__ void k_set_form(IterState *st, int form) { st->form = form; }

// Byte copy by the SMs (16-byte vectors when both ends allow): device-to-device
// and device-to-mapped-host copies that must not queue behind bulk transfers
// on the copy engines (asynchronous staging / read-back, usp_stage_inputs).
__global__ void k_copy_bytes(char *dst, const char *src, size_t n) {
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
        const size_t n16 = n / 16;
        for (size_t i = tid; i < n16; i += nt)
            reinterpret_cast<uint4 *>(dst)[i] = reinterpret_cast<const uint4 *>(src)[i];
        for (size_t i = n16 * 16 + tid; i < n; i += nt) dst[i] = src[i];
    } else {
        for (size_t i = tid; i < n; i += nt) dst[i] = src[i];
    }
}

__global__ void k_set_state(IterState *st, double alpha, double tol, long long kmax) {
    st->alpha = alpha;
    st->tol = tol;
    st->kmax = kmax;
    st->counter = 0u;
    const bool below = tol > 0.0 && st->r < tol;
    // x-form state (reading R-30): st->r may be r_{k-1}; the next x-form pass
    // computes r_k and stops itself after its update (the same count)
    if (st->form == FORM_X) return;
    if (st->status == ST_RUNNING && below) st->status = ST_STOP_PENDING;
    if (st->status == ST_STOP_PENDING && !below) st->status = ST_RUNNING;
}

// ============================================================= launchers ==
#define USP_FOR_EACH_N(X) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048)

bool supported_n(long long n) { return n >= 16 && n <= 2048 && (n & (n - 1)) == 0; }

template <int N, int MODE, int COLS>
static cudaError_t strided_t(const SParams &p, int grid, cudaStream_t s) {
    constexpr int SM = SGeo<N, COLS>::SMEM;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_strided<N, MODE, COLS>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    k_strided<N, MODE, COLS><<<grid, SGeo<N, COLS>::NT, SM, s>>>(p);
    return cudaGetLastError();
}

template <int N, int COLS>
static cudaError_t strided_mode(SMode mode, const SParams &p, int grid, cudaStream_t s) {
    if (mode == S_FWD) return strided_t<N, S_FWD, COLS>(p, grid, s);
    if (mode == S_INV) return strided_t<N, S_INV, COLS>(p, grid, s);
    return strided_t<N, S_FWD_MUL_INV, COLS>(p, grid, s);
}

// Register-staged passes for the short strided lines k_stile does not take
// (N = 16, 32): 16-column tiles.
cudaError_t launch_strided(int N, SMode mode, const SParams &p, int grid, cudaStream_t s) {
    switch (N) {
    case 16: return strided_mode<16, 16>(mode, p, grid, s);
    case 32: return strided_mode<32, 16>(mode, p, grid, s);
    default: return cudaErrorInvalidValue;
    }
}


cudaError_t launch_solve1d(int N, OneMode mode, const OneParams &p, cudaStream_t s) {
#define O_CASE(n)                                                                   \
    case n:                                                                         \
        if (mode == O_SETUP) k_solve1d<n, O_SETUP><<<1, LineGeo<n>::N1, 0, s>>>(p); \
        else k_solve1d<n, O_ITER><<<1, LineGeo<n>::N1, 0, s>>>(p);                  \
        return cudaGetLastError();
    switch (N) { USP_FOR_EACH_N(O_CASE) default: return cudaErrorInvalidValue; }
#undef O_CASE
}

cudaError_t launch_potential(const PotParams &p, int grid, cudaStream_t s) {
    k_potential<<<resident_grid<k_potential>(grid, 256), 256, 0, s>>>(p);
    return cudaGetLastError();
}

int farthest_grid(int grid) { return resident_grid<k_farthest>(grid, 256); }

cudaError_t launch_farthest(const FarParams &p, int grid, cudaStream_t s) {
    k_farthest<<<grid, 256, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_finish(IterState *st, const double *sums, int P, int src_epi, const Red &red, cudaStream_t s) {
    k_finish<<<1, 1, 0, s>>>(st, sums, P, src_epi, red);
    return cudaGetLastError();
}

cudaError_t launch_copy_bytes(void *dst, const void *src, size_t n, int grid, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const size_t need = (n + 16 * 256 - 1) / (16 * 256);
    const int g = (int)(need < (size_t)grid ? (need ? need : 1) : grid);
    k_copy_bytes<<<g, 256, 0, s>>>(static_cast<char *>(dst), static_cast<const char *>(src), n);
    return cudaGetLastError();
}

cudaError_t launch_set_form(IterState *st, int form, cudaStream_t s) {
    k_set_form<<<1, 1, 0, s>>>(st, form);
    return cudaGetLastError();
}

__global__ void k_put_blob(unsigned char *dst, Blob v, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = v.b[i];
}

cudaError_t launch_put_bytes(void *dst, const void *src, size_t n, cudaStream_t s) {
    if (n > sizeof(Blob)) return cudaErrorInvalidValue;
    Blob b;
    memcpy(b.b, src, n);
    k_put_blob<<<1, 128, 0, s>>>(static_cast<unsigned char *>(dst), b, (int)n);
    return cudaGetLastError();
}

cudaError_t launch_put_state(IterState *st, const IterState &h, cudaStream_t s) {
    return launch_put_bytes(st, &h, sizeof h, s);
}

cudaError_t launch_set_state(IterState *st, double alpha, double tol, long long kmax, cudaStream_t s) {
    k_set_state<<<1, 1, 0, s>>>(st, alpha, tol, kmax);
    return cudaGetLastError();
}


}  // namespace usp
