// kernels_pipe.cu -- TMA-pipelined pass kernels (the default path on sm_100a).
//
// Same arithmetic as kernels.cu (four-step line FFTs, fused update), but the
// global loads are issued by one producer warp as asynchronous bulk copies
// into a ring of shared-memory stages, completing on mbarriers:
//
//   k_xpass_pipe  : each stage holds one "unit" (32/N1 consecutive x-lines,
//                   i.e. one warp's lines) of up to four fields -- work,
//                   Delta, x, B -- fetched with cp.async.bulk (1-D, 8 KiB per
//                   field for N = 1024).  Consumer warps each own a unit.
//   k_strided_pipe: each stage holds a COLS x N tile of a strided axis
//                   (y: stride nx; z: stride nx*ny), fetched with tensor-map
//                   TMA boxes (cp.async.bulk.tensor, <= 256 rows per box).
//                   All consumer warps transform one tile together.
//
// Loads therefore cost no registers and keep up to S stages in flight per SM
// (Little's law needs ~35 KB/SM at 6.5 TB/s; a stage is 32-64 KB), while the
// consumers' FFT arithmetic overlaps the next stages' transfers.  Results are
// stored straight from registers (coalesced 128/256-byte rows).
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fft_core.cuh"
#include "kcommon.cuh"
#include "tma.cuh"
#include "usp_internal.h"

namespace usp {

constexpr int kSmemBudget = 232448 - 2048;   // max dynamic smem per CTA on sm_100 minus slack

// ============================================================ x pass ====
template <int N>
struct XPipe {
    using G = LineGeo<N>;
    static constexpr int U = 32 / G::N1;                    // lines per warp unit
    static constexpr int UE = 32 * G::N2;                   // elements per unit (= U * N)
    static constexpr int XC = (N >= 2048) ? 2 : 5;          // consumer warps
    static constexpr int NT = 32 * (XC + 1);
    static constexpr int XBUF = U * LayRow<N>::kFloat2PerLine;   // float2 per consumer warp
    static constexpr int STAGE = 4 * UE;                    // float2 per stage (4 slots)
    // Bulk copies complete out of order, so a stage may only be reused by the
    // warp that consumed it: S = XC * SPW and unit i -> stage i % S, warp
    // i % XC.  A consumer at unit i has itself finished unit i - S, so the
    // mbarrier it tests is never one phase behind (no parity ABA).
    static constexpr int SPW0 = (kSmemBudget - XC * XBUF * 8 - N * 8) / (XC * STAGE * 8);
    static constexpr int SPW = SPW0 > 2 ? 2 : SPW0;
    static constexpr int S = XC * SPW;
    static_assert(SPW >= 1, "x pipeline needs >= 1 stage per consumer warp");
    static constexpr int SMEM = (S * STAGE + XC * XBUF + N) * 8 + 2 * S * 8;   // stages, exchange, twiddles, barriers
};

template <int N, int MODE>
__global__ void __launch_bounds__(XPipe<N>::NT, 1) k_xpass_pipe(XParams p) {
    using G = LineGeo<N>;
    using T = XPipe<N>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float2 *stages = reinterpret_cast<float2 *>(smem_raw);
    float2 *xbufs = stages + T::S * T::STAGE;
    float2 *sm_tw = xbufs + T::XC * T::XBUF;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm_tw + N);
    uint64_t *empty = full + T::S;
    __shared__ double sh_red[T::NT / 32];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    bool xonly = false;
    float alpha = 0.f;
    if (MODE == X_ITER) {
        const int status = p.st->status;
        const long long k = p.st->k, kmax = p.st->kmax;
        if (k >= kmax || (status != ST_RUNNING && status != ST_STOP_PENDING)) return;
        xonly = (status == ST_STOP_PENDING);
        alpha = (float)p.st->alpha;
    }
    double acc = 0.0;
    const long long nvox = p.nlines * (long long)N;

    if (MODE == X_ITER && xonly) {
        // final x_{k+1} = x_k + alpha Delta_k after the stop test (reading R-5)
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvox;
             i += (long long)gridDim.x * blockDim.x) {
            const float2 d = p.delta[i];
            float2 xx = p.x[i];
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
        const uint32_t ub = T::UE * 8u;                       // bytes per complex slot
        if (warp == T::XC) {
            // ------------------------------------------------ producer warp
            if (lane == 0) {
                for (int i = 0; i < nloc; ++i) {
                    const int s = i % T::S;
                    if (i >= T::S && !mbar_wait(&empty[s], ((i / T::S) - 1) & 1)) {
                        if (atomicCAS(&p.st->err, 0, 1) == 0) p.st->err_info = i;
                        break;
                    }
                    const long long off = (blockIdx.x + (long long)i * gridDim.x) * T::UE;
                    float2 *st = stages + s * T::STAGE;
                    if (MODE == X_SRC_FWD) {
                        const uint32_t sb = p.src_real ? ub / 2 : ub;
                        mbar_arrive_expect_tx(&full[s], sb);
                        const char *src = reinterpret_cast<const char *>(p.x) + off * (p.src_real ? 4 : 8);
                        bulk_g2s(st, src, sb, &full[s]);
                    } else if (MODE == X_SRC_EPI) {
                        mbar_arrive_expect_tx(&full[s], 2 * ub);
                        bulk_g2s(st, p.work + off, ub, &full[s]);
                        bulk_g2s(st + 3 * T::UE, p.B + off, ub, &full[s]);
                    } else {
                        mbar_arrive_expect_tx(&full[s], 4 * ub);
                        bulk_g2s(st, p.work + off, ub, &full[s]);
                        bulk_g2s(st + 1 * T::UE, p.delta + off, ub, &full[s]);
                        bulk_g2s(st + 2 * T::UE, p.x + off, ub, &full[s]);
                        bulk_g2s(st + 3 * T::UE, p.B + off, ub, &full[s]);
                    }
                }
            }
            __syncwarp();
        } else {
            // ------------------------------------------------ consumer warps
            const int lq = lane / G::N1, j = lane % G::N1;
            const LayRow<N> lay{xbufs + warp * T::XBUF + lq * LayRow<N>::kFloat2PerLine};
            for (int i = warp; i < nloc; i += T::XC) {
                const int s = i % T::S;
                if (!mbar_wait(&full[s], (i / T::S) & 1)) {
                    if (lane == 0 && atomicCAS(&p.st->err, 0, 2) == 0) p.st->err_info = i;
                    break;
                }
                const float2 *st = stages + s * T::STAGE;
                const long long gb = (blockIdx.x + (long long)i * gridDim.x) * T::UE + lq * N + j;
                const int sbase = lq * N + j;
                float2 v[G::N2];
                if (MODE == X_SRC_FWD) {
#pragma unroll
                    for (int m = 0; m < G::N2; ++m) {
                        const int e = sbase + G::N1 * m;
                        const float2 sv = p.src_real ? make_float2(reinterpret_cast<const float *>(st)[e], 0.f)
                                                     : st[e];
                        v[m] = cmul(sv, p.inv_c);               // s = S / c
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[s]);   // the warp's stage can refill now
                } else {
#pragma unroll
                    for (int m = 0; m < G::N2; ++m) v[m] = cconj(st[sbase + G::N1 * m]);
                }
                // pass 0: x inverse as conj(DFT(conj(u))) + update; pass 1: x forward.
                // One FFT body in the binary keeps the kernel inside the I-cache.
#pragma unroll 1
                for (int pass = (MODE == X_SRC_FWD) ? 1 : 0; pass < 2; ++pass) {
                    fft_line<N, false, LayRow<N>, true>(v, lay, j, sm_tw);
                    if (pass == 0) {
                        float lacc = 0.f;
#pragma unroll
                        for (int m = 0; m < G::N2; ++m) {
                            const int e = sbase + G::N1 * m;
                            const long long gi = gb + G::N1 * m;
                            const float2 y = cconj(v[m]);           // (L+1)^-1 u, chain complete
                            const float2 b = st[3 * T::UE + e];
                            float2 dn;
                            if (MODE == X_SRC_EPI) {
                                dn = cmul(b, y);                    // Delta_0 = B (L+1)^-1 s
                                p.x[gi] = make_float2(0.f, 0.f);    // x_0 = 0 (L83)
                            } else {
                                const float2 d = st[1 * T::UE + e];
                                const float2 xx = st[2 * T::UE + e];
                                const float2 t = cmul(b, csub(y, d));
                                dn = make_float2(fmaf(alpha, t.x, d.x), fmaf(alpha, t.y, d.y));
                                p.x[gi] = make_float2(fmaf(alpha, d.x, xx.x), fmaf(alpha, d.y, xx.y));
                            }
                            p.delta[gi] = dn;
                            lacc += cabs2(dn);
                            v[m] = cmul(b, dn);                     // next chain: u = B Delta
                        }
                        acc += (double)lacc;
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty[s]);
                    }
                }
#pragma unroll
                for (int m = 0; m < G::N2; ++m) p.work[gb + G::N1 * m] = v[m];
            }
        }
    }

    if (MODE == X_SRC_FWD) return;
    double total;
    const double mine = block_sum_d<T::NT>(acc, sh_red);
    if (!last_block_total<T::NT>(mine, p.st, p.red.partials, sh_red, &total)) return;
    if (threadIdx.x != 0) return;
    finish_xpass(MODE == X_SRC_EPI, xonly, total, p.st, p.red);
}

// ====================================================== strided pass ====
template <int N>
struct SPipe {
    using G = LineGeo<N>;
    static constexpr int COLS = (G::N1 >= 32) ? 8 : 16;     // columns per tile (64 / 128-byte rows)
    static constexpr int PAD = (COLS == 8) ? 8 : 0;
    static constexpr int CT = COLS * G::N1;                 // consumer threads
    static constexpr int CW = CT / 32;
    static constexpr int NT = CT + 32;
    static constexpr int TILE = COLS * N;                   // float2 per stage
    static constexpr int XB = LayCol<N, COLS, PAD, CT>::kFloat2;
    static constexpr int BOXN = N < 256 ? N : 256;
    static constexpr int S0 = (kSmemBudget - XB * 8) / (TILE * 8);
    static constexpr int S = S0 > 4 ? 4 : S0;
    static_assert(S >= 2, "strided pipeline needs >= 2 stages");
    static constexpr int SMEM = (S * TILE + XB) * 8 + 2 * S * 8;
};

template <int N, int MODE, int RANK>
__global__ void __launch_bounds__(SPipe<N>::NT, 1) k_strided_pipe(const __grid_constant__ CUtensorMap tmap,
                                                                  SParams p) {
    using G = LineGeo<N>;
    using T = SPipe<N>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float2 *stages = reinterpret_cast<float2 *>(smem_raw);
    float2 *xbuf = stages + T::S * T::TILE;
    uint64_t *full = reinterpret_cast<uint64_t *>(xbuf + T::XB);
    uint64_t *empty = full + T::S;
    if (p.check_state) {
        if (p.st->status != ST_RUNNING || p.st->k >= p.st->kmax) return;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < T::S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], T::CW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const long long tpo = p.ncols / T::COLS;
    const long long ntiles = tpo * p.nouter;
    const int nloc = (int)((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);
    if (warp == T::CW) {
        // ---------------------------------------------------- producer warp
        if (lane == 0) {
            prefetch_tmap(&tmap);
            for (int i = 0; i < nloc; ++i) {
                const int s = i % T::S;
                if (i >= T::S && !mbar_wait(&empty[s], ((i / T::S) - 1) & 1)) {
                    if (atomicCAS(&p.st->err, 0, 3) == 0) p.st->err_info = i;
                    break;
                }
                const long long t = blockIdx.x + (long long)i * gridDim.x;
                const long long o = t / tpo;
                const int c0 = (int)((t - o * tpo) * T::COLS);
                float2 *st = stages + s * T::TILE;
                mbar_arrive_expect_tx(&full[s], T::TILE * 8);
#pragma unroll
                for (int b = 0; b < N / T::BOXN; ++b) {
                    if (RANK == 3) tma_load_3d(st + b * T::BOXN * T::COLS, &tmap, c0, b * T::BOXN, (int)o, &full[s]);
                    else tma_load_2d(st + b * T::BOXN * T::COLS, &tmap, c0, b * T::BOXN, &full[s]);
                }
            }
        }
        return;   // the producer takes no part in the consumers' named barriers
    }
    // -------------------------------------------------------- consumers
    const int c = threadIdx.x % T::COLS, j = threadIdx.x / T::COLS;
    const LayCol<N, T::COLS, T::PAD, T::CT> lay{xbuf, c};
    for (int i = 0; i < nloc; ++i) {
        const int s = i % T::S;
        if (!mbar_wait(&full[s], (i / T::S) & 1)) {
            if (threadIdx.x == 0 && atomicCAS(&p.st->err, 0, 4) == 0) p.st->err_info = i;
            return;
        }
        const long long t = blockIdx.x + (long long)i * gridDim.x;
        const long long o = t / tpo;
        const long long col = (t - o * tpo) * T::COLS + c;
        const float2 *st = stages + s * T::TILE;
        float2 v[G::N2];
#pragma unroll
        for (int m = 0; m < G::N2; ++m) v[m] = st[(j + G::N1 * m) * T::COLS + c];
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        fft_line<N, MODE == S_INV>(v, lay, j, p.tw);
        if (MODE == S_FWD_MUL_INV) {
            // (L+1)^-1 multiplier, Eq. 12: |p|^2 = p_x^2 + p_y^2 + p_line^2
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
                v[m] = cmul(v[m], multiplier(p.mp, fmaf(pl, pl, pt2)));
            }
            fft_line<N, true>(v, lay, j, p.tw);
        }
        float2 *dst = p.data + (o * p.ostride + col);
#pragma unroll
        for (int m = 0; m < G::N2; ++m) dst[(long long)(j + G::N1 * m) * p.stride] = v[m];
    }
}

// ========================================================= launchers ====
#define USP_PIPE_X_N(X) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048)
#define USP_PIPE_S_N(X) X(16) X(32) X(64) X(128) X(256) X(512) X(1024)

template <int N, int MODE>
static cudaError_t xpipe_t(const XParams &p, int grid, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_xpass_pipe<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             XPipe<N>::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    k_xpass_pipe<N, MODE><<<grid, XPipe<N>::NT, XPipe<N>::SMEM, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_xpass_pipe(int N, XMode mode, const XParams &p, int grid, cudaStream_t s) {
#define XP_CASE(n)                                                           \
    case n:                                                                  \
        if (mode == X_SRC_FWD) return xpipe_t<n, X_SRC_FWD>(p, grid, s);     \
        if (mode == X_SRC_EPI) return xpipe_t<n, X_SRC_EPI>(p, grid, s);     \
        return xpipe_t<n, X_ITER>(p, grid, s);
    switch (N) { USP_PIPE_X_N(XP_CASE) default: return cudaErrorInvalidValue; }
#undef XP_CASE
}

template <int N, int MODE, int RANK>
static cudaError_t spipe_t(const CUtensorMap &map, const SParams &p, int grid, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_strided_pipe<N, MODE, RANK>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, SPipe<N>::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    k_strided_pipe<N, MODE, RANK><<<grid, SPipe<N>::NT, SPipe<N>::SMEM, s>>>(map, p);
    return cudaGetLastError();
}

template <int N>
static cudaError_t spipe_mode(SMode mode, int rank, const CUtensorMap &map, const SParams &p, int grid,
                              cudaStream_t s) {
    if (rank == 3) {
        if (mode == S_FWD) return spipe_t<N, S_FWD, 3>(map, p, grid, s);
        if (mode == S_INV) return spipe_t<N, S_INV, 3>(map, p, grid, s);
        return spipe_t<N, S_FWD_MUL_INV, 3>(map, p, grid, s);
    }
    if (mode == S_FWD) return spipe_t<N, S_FWD, 2>(map, p, grid, s);
    if (mode == S_INV) return spipe_t<N, S_INV, 2>(map, p, grid, s);
    return spipe_t<N, S_FWD_MUL_INV, 2>(map, p, grid, s);
}

bool strided_pipe_supported(long long n) { return n >= 16 && n <= 1024; }
int strided_pipe_cols(int N) { return (1 << (ilog2(N) / 2)) >= 32 ? 8 : 16; }
int strided_pipe_box(int N) { return N < 256 ? N : 256; }

cudaError_t launch_strided_pipe(int N, SMode mode, int rank, const CUtensorMap &map, const SParams &p, int grid,
                                cudaStream_t s) {
#define SP_CASE(n) \
    case n: return spipe_mode<n>(mode, rank, map, p, grid, s);
    switch (N) { USP_PIPE_S_N(SP_CASE) default: return cudaErrorInvalidValue; }
#undef SP_CASE
}

}  // namespace usp
