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
// (The strided y/z passes are in kernels_stile.cu.)
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
// LEAN (reading R-31): the x-form passes of a sparse-source plan need only
// work, x, B -> 3-slot stages, and the smem saved buys a sixth consumer warp.
// (A Delta-form pass landing on a LEAN launch reads Delta from global memory.)
template <int N, bool LEAN = false>
struct XPipe {
    using G = LineGeo<N>;
    static constexpr int U = 32 / G::N1;                    // lines per warp unit
    static constexpr int UE = 32 * G::N2;                   // elements per unit (= U * N)
    static constexpr int XC = (N >= 2048) ? 2 : (LEAN ? 6 : 5);   // consumer warps
    static constexpr int NT = 32 * (XC + 1);
    static constexpr int XBUF = U * LayRow<N>::kFloat2PerLine;   // float2 per consumer warp
    static constexpr int NSLOT = LEAN ? 3 : 4;
    static constexpr int STAGE = NSLOT * UE;                // float2 per stage
    // slot offsets (float2): work, Delta-or-s (not LEAN), x, B
    static constexpr int SD = UE, SX = (LEAN ? 1 : 2) * UE, SB = (LEAN ? 2 : 3) * UE;
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

// DSPEC: the Delta-form update has its own loop body (launched when the host
// expects the Delta-form).  Extra bodies that a launch does not execute still
// cost: the dense x-form measured 8.3 ms with the general body alone and
// 10.3 ms next to a Delta-form body, the Delta-form 13.4 vs 9.7 ms the other
// way round -- so each expected form gets its own instantiation.
template <int N, int MODE, bool LEAN, bool DSPEC, bool XSPEC = false>
__global__ void __launch_bounds__(XPipe<N, LEAN>::NT, 1) k_xpass_pipe(XParams p) {
    using G = LineGeo<N>;
    using T = XPipe<N, LEAN>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float2 *stages = reinterpret_cast<float2 *>(smem_raw);
    float2 *xbufs = stages + T::S * T::STAGE;
    float2 *sm_tw = xbufs + T::XC * T::XBUF;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm_tw + N);
    uint64_t *empty = full + T::S;
    __shared__ double sh_red[T::NT / 32];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    pdl_trigger();
    pdl_wait();
    bool xonly = false;
    float alpha = 0.f;
    int act = ACT_DELTA;   // X_ITER: Delta-form, x-form, probe or x-form -> Delta-form (kcommon.cuh)
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
    const float c1 = dform ? alpha : 1.f;                       // Delta_new = d0 + c1 t
    const float e1 = (act == ACT_X || act == ACT_PROBE) ? 1.f : 0.f;   // u = B w + e1 s
    const bool store_x = act == ACT_DELTA || act == ACT_X, store_d = act != ACT_X;
    const bool u_from_d = act == ACT_DELTA || act == ACT_TO_DELTA;
    // stage slot 1: Delta (Delta-form) or s (x-form passes; source setup of x-form plans).
    // Sparse source (R-31): the x-form passes form u = B x without s (k_sadd
    // adds the transformed source lines), so slot 1 is not loaded at all.
    const float2 *slot1 = (MODE == X_ITER && act != ACT_DELTA) || (MODE == X_SRC_EPI && p.s) ? p.s : p.delta;
    const bool need1 = !(MODE == X_ITER && p.s_sparse && act != ACT_DELTA);
    const bool stage1 = need1 && !LEAN;   // slot 1 streamed through the stage
    const float e1s = need1 ? e1 : 0.f;
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
                        mbar_arrive_expect_tx(&full[s], (p.s ? 3 : 2) * ub);
                        bulk_g2s(st, p.work + off, ub, &full[s]);
                        if (p.s) bulk_g2s(st + T::SD, slot1 + off, ub, &full[s]);
                        bulk_g2s(st + T::SB, p.B + off, ub, &full[s]);
                    } else {
                        mbar_arrive_expect_tx(&full[s], (stage1 ? 4 : 3) * ub);
                        bulk_g2s(st, p.work + off, ub, &full[s]);
                        if (stage1) bulk_g2s(st + T::SD, slot1 + off, ub, &full[s]);
                        bulk_g2s(st + T::SX, p.x + off, ub, &full[s]);
                        bulk_g2s(st + T::SB, p.B + off, ub, &full[s]);
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
                        if (p.s) p.s[gb + G::N1 * m] = v[m];   // x-form plans keep s
                    }
                    if (p.s_flag) {   // does this x-line carry any source? (R-31)
                        bool nz = false;
#pragma unroll
                        for (int m = 0; m < G::N2; ++m) nz |= (v[m].x != 0.f) || (v[m].y != 0.f);
                        const unsigned bal = __ballot_sync(0xffffffffu, nz);
                        const unsigned lmask = (G::N1 >= 32) ? 0xffffffffu : (((1u << G::N1) - 1u) << (lq * G::N1));
                        if (j == 0) p.s_flag[(blockIdx.x + (long long)i * gridDim.x) * T::U + lq] = (bal & lmask) != 0u;
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
                        if (LEAN && MODE == X_ITER && act == ACT_X && !need1) {
                            // the lean pass's common case, without the selects of the
                            // general body: Delta_k = B (y - x_k), x_{k+1}, u = B x_{k+1}
#pragma unroll
                            for (int m = 0; m < G::N2; ++m) {
                                const int e = sbase + G::N1 * m;
                                const float2 y = cconj(v[m]), b = st[T::SB + e], xx = st[T::SX + e];
                                const float2 dk = cmul(b, csub(y, xx));
                                const float2 xn = make_float2(fmaf(alpha, dk.x, xx.x), fmaf(alpha, dk.y, xx.y));
                                p.x[gb + G::N1 * m] = xn;
                                lacc += cabs2(dk);
                                v[m] = cmul(b, xn);
                            }
                        } else if (XSPEC && !LEAN && MODE == X_ITER && act == ACT_X && need1) {
                            // the dense-source x-form's dedicated body: u = B x_{k+1} + s
#pragma unroll
                            for (int m = 0; m < G::N2; ++m) {
                                const int e = sbase + G::N1 * m;
                                const float2 y = cconj(v[m]), b = st[T::SB + e];
                                const float2 sv = st[T::SD + e], xx = st[T::SX + e];
                                const float2 dk = cmul(b, csub(y, xx));
                                const float2 xn = make_float2(fmaf(alpha, dk.x, xx.x), fmaf(alpha, dk.y, xx.y));
                                p.x[gb + G::N1 * m] = xn;
                                lacc += cabs2(dk);
                                const float2 bx = cmul(b, xn);
                                v[m] = make_float2(bx.x + sv.x, bx.y + sv.y);
                            }
                        } else if (DSPEC && !LEAN && MODE == X_ITER && act == ACT_DELTA) {
                            // the Delta-form's dedicated body
#pragma unroll
                            for (int m = 0; m < G::N2; ++m) {
                                const int e = sbase + G::N1 * m;
                                const long long gi = gb + G::N1 * m;
                                const float2 y = cconj(v[m]), b = st[T::SB + e];
                                const float2 d = st[T::SD + e], xx = st[T::SX + e];
                                const float2 t = cmul(b, csub(y, d));
                                const float2 dn = make_float2(fmaf(alpha, t.x, d.x), fmaf(alpha, t.y, d.y));
                                p.x[gi] = make_float2(fmaf(alpha, d.x, xx.x), fmaf(alpha, d.y, xx.y));
                                p.delta[gi] = dn;
                                lacc += cabs2(dn);
                                v[m] = cmul(b, dn);
                            }
                        } else
#pragma unroll
                        for (int m = 0; m < G::N2; ++m) {
                            const int e = sbase + G::N1 * m;
                            const long long gi = gb + G::N1 * m;
                            const float2 y = cconj(v[m]);           // (L+1)^-1 u, chain complete
                            const float2 b = st[T::SB + e];
                            float2 dn;
                            if (MODE == X_SRC_EPI) {
                                dn = cmul(b, y);                    // Delta_0 = B (L+1)^-1 s
                                p.x[gi] = make_float2(0.f, 0.f);    // x_0 = 0 (L83)
                                p.delta[gi] = dn;
                                lacc += cabs2(dn);
                                // next chain: u = B Delta (x-form plans: u_0 = s)
                                v[m] = p.s ? st[T::SD + e] : cmul(b, dn);
                                continue;
                            }
                            // One body for every action (uniform selects, no duplicated code):
                            //   Delta-form: t = B (y - Delta_k), Delta_{k+1} = Delta_k + alpha t,
                            //                        x_{k+1} = x_k + alpha Delta_k, u = B Delta_{k+1}
                            //   x-form (Alg. 1 lines 3-4): Delta_k = B (y - x_k),
                            //                        x_{k+1} = x_k + alpha Delta_k, u = B x_{k+1} + s
                            //   probe: Delta_k = B (y - x_k) stored, x kept, u = B x_k + s
                            //   x-form -> Delta-form: Delta_k stored, x kept, u = B Delta_k
                            // Delta_k or s (LEAN: a Delta-form pass reads Delta from global memory)
                            const float2 a1 = !need1 ? make_float2(0.f, 0.f) : (LEAN ? slot1[gi] : st[T::SD + e]);
                            const float2 xx = st[T::SX + e];
                            const float2 t = cmul(b, csub(y, dform ? a1 : xx));
                            const float2 d0 = dform ? a1 : make_float2(0.f, 0.f);
                            dn = make_float2(fmaf(c1, t.x, d0.x), fmaf(c1, t.y, d0.y));
                            const float2 xi = dform ? a1 : t;
                            const float2 xn = make_float2(fmaf(alpha, xi.x, xx.x), fmaf(alpha, xi.y, xx.y));
                            if (store_x) p.x[gi] = xn;
                            if (store_d) p.delta[gi] = dn;
                            lacc += cabs2(dn);
                            const float2 w = u_from_d ? dn : (act == ACT_X ? xn : xx);
                            const float2 bw = cmul(b, w);
                            v[m] = make_float2(fmaf(e1s, a1.x, bw.x), fmaf(e1s, a1.y, bw.y));
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
    if (p.red.local_sum) {   // slab-decomposed: k_finish sums the ranks' totals after the all-gather
        *p.red.local_sum = total;
        return;
    }
    finish_xpass(MODE == X_SRC_EPI, xonly, total, p.st, p.red, act);
}

// ================================================ sparse source (R-31) ==
// Source lines: count the flagged x-lines, gather their x-transformed source
// (work after the x-form setup holds FFT_x(s)) into a compact buffer, and
// after each x-form pass add them to the forward x-transform of B x
// (FFT_x(B x + s) = FFT_x(B x) + FFT_x(s): the x pass then never reads s).
__global__ void k_sparse_count(const unsigned char *flag, long long nlines, unsigned *count) {
    unsigned c = 0;
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < nlines;
         l += (long long)gridDim.x * blockDim.x)
        c += flag[l] ? 1u : 0u;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

__global__ void k_sparse_gather(const unsigned char *flag, long long nlines, const float2 *work, int n, int *list,
                                float2 *comp, unsigned *count) {
    for (long long l = blockIdx.x; l < nlines; l += gridDim.x) {
        if (!flag[l]) continue;   // uniform per CTA
        __shared__ unsigned idx;
        if (threadIdx.x == 0) {
            idx = atomicAdd(count, 1u);
            list[idx] = (int)l;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) comp[(long long)idx * n + i] = work[l * n + i];
        __syncthreads();
    }
}

__global__ void k_sparse_add(SAddParams p) {
    pdl_wait();
    if (!p.st->add_s) return;
    for (int q = blockIdx.x; q < p.count; q += gridDim.x) {
        float2 *w = p.work + (long long)p.list[q] * p.n;
        const float2 *c = p.comp + (long long)q * p.n;
        for (int i = threadIdx.x; i < p.n; i += blockDim.x) {
            const float2 a = w[i], b = c[i];
            w[i] = make_float2(a.x + b.x, a.y + b.y);
        }
    }
}

__global__ void k_sparse_clear(IterState *st) { st->add_s = 0; }

cudaError_t launch_sparse_count(const unsigned char *flag, long long nlines, unsigned *count, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(count, 0, sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    k_sparse_count<<<296, 256, 0, s>>>(flag, nlines, count);
    return cudaGetLastError();
}

cudaError_t launch_sparse_gather(const unsigned char *flag, long long nlines, const float2 *work, int n, int *list,
                                 float2 *comp, unsigned *count, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(count, 0, sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    k_sparse_gather<<<592, 256, 0, s>>>(flag, nlines, work, n, list, comp, count);
    return cudaGetLastError();
}

cudaError_t launch_sparse_add(const SAddParams &p, cudaStream_t s) {
    const int grid = p.count < 148 ? p.count : 148;
    if (grid > 0) {
        cudaError_t e = launch_pdl(k_sparse_add, grid, 256, 0, s, p);
        if (e != cudaSuccess) return e;
    }
    k_sparse_clear<<<1, 1, 0, s>>>(p.st);
    return cudaGetLastError();
}

// ========================================================= launchers ====
#define USP_PIPE_X_N(X) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048)

template <int N, int MODE, bool LEAN, bool DSPEC, bool XSPEC = false>
static cudaError_t xpipe_t(const XParams &p, int grid, cudaStream_t s) {
    using T = XPipe<N, LEAN>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_xpass_pipe<N, MODE, LEAN, DSPEC, XSPEC>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    return launch_pdl(k_xpass_pipe<N, MODE, LEAN, DSPEC, XSPEC>, grid, T::NT, T::SMEM, s, p);
}


// X_ITER variants by the form the host expects: lean (sparse-source x-form:
// 3-slot stages, one more consumer warp; N <= 1024), x-form (general body),
// Delta-form (dedicated body)
cudaError_t launch_xpass_pipe(int N, XMode mode, const XParams &p, int grid, cudaStream_t s, bool lean,
                              bool expect_x) {
#define XP_CASE(n)                                                                    \
    case n:                                                                           \
        if (mode == X_SRC_FWD) return xpipe_t<n, X_SRC_FWD, false, false>(p, grid, s); \
        if (mode == X_SRC_EPI) return xpipe_t<n, X_SRC_EPI, false, false>(p, grid, s); \
        if (lean && n <= 1024) return xpipe_t<n, X_ITER, true, false>(p, grid, s);    \
        if (expect_x) return xpipe_t<n, X_ITER, false, false, true>(p, grid, s);  \
        return xpipe_t<n, X_ITER, false, true>(p, grid, s);
    switch (N) { USP_PIPE_X_N(XP_CASE) default: return cudaErrorInvalidValue; }
#undef XP_CASE
}

}  // namespace usp
