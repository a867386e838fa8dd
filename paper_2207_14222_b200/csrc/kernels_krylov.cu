// kernels_krylov.cu -- BiCGSTAB on the preconditioned system (SURVEY.md §8(f)
// NEXT-2; Eq. 5, Table 1b).
//
//     M u = B [u - (L+1)^-1 (B u)]        (Gamma^-1 A with alpha = 1, R-25)
//     M x = b,  b = B (L+1)^-1 s  (= Delta_0 of the fixed-point iteration)
//
// One BiCGSTAB pass (two applications of M) is five launches plus two FFT
// chains (the strided passes of the fixed-point path, unchanged):
//   K_PFWD  p = r + beta (p - omega v);  u = B p  -> x forward FFT   (work)
//   chain   y forward, z forward * g(p)/N * z inverse, y inverse
//   K_VINV  x inverse FFT -> y;  v = B (p - y);  (rhat, v) -> alpha = rho / (rhat, v)
//   K_SFWD  s = r - alpha v;  ||s||;  u = B s  -> x forward FFT      (half-step stop test)
//   chain
//   K_TINV  x inverse FFT -> y;  t = B (s - y);  (t, s), (t, t) -> omega
//   k_kupd  x += alpha p + omega s;  r = s - omega t;  (rhat, r), ||r||
//           -> rho', beta = (rho'/rho)(alpha/omega); full-step stop test
// The x-FFT kernels use the TMA bulk-copy pipeline of k_xpass_pipe
// (producer warp, per-warp stages).  The inner products are reduced in a
// fixed order (fp32 per line -> fp64 per thread -> CTA -> last CTA sums the
// CTA partials in order), so runs are deterministic; the scalar recurrences
// run in fp64 on the device (KState) and the stop decisions update the
// shared IterState, so the strided passes skip themselves after a stop.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fft_core.cuh"
#include "kcommon.cuh"
#include "tma.cuh"
#include "usp_internal.h"

namespace usp {

constexpr int kSmemBudgetK = 232448 - 2048;

__device__ __forceinline__ double2 dmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 ddiv(double2 a, double2 b) {
    const double m = b.x * b.x + b.y * b.y;
    return make_double2((a.x * b.x + a.y * b.y) / m, (a.y * b.x - a.x * b.y) / m);
}
__device__ __forceinline__ float2 tof(double2 a) { return make_float2((float)a.x, (float)a.y); }

// Fixed-order reduction of NV doubles per thread over the grid; returns true
// in thread 0 of the last CTA with tot[] = the grid totals.
template <int NT, int NV>
__device__ __forceinline__ bool grid_sums(const double (&mine)[NV], IterState *st, double *partials,
                                          double (&tot)[NV]) {
    __shared__ double sh[NT / 32][NV];
    __shared__ int am_last;
    double v[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = warp_sum_d(mine[q]);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0)
#pragma unroll
        for (int q = 0; q < NV; ++q) sh[w][q] = v[q];
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            double s = 0.0;
            for (int i = 0; i < NT / 32; ++i) s += sh[i][q];
            partials[(size_t)blockIdx.x * NV + q] = s;
        }
        __threadfence();
        am_last = (atomicAdd(&st->counter, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (!am_last || threadIdx.x != 0) return false;
    __threadfence();
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        double s = 0.0;
        for (unsigned i = 0; i < gridDim.x; ++i) s += __ldcg(&partials[(size_t)i * NV + q]);
        tot[q] = s;
    }
    st->counter = 0u;
    return true;
}

template <int N>
struct XOp {
    using G = LineGeo<N>;
    static constexpr int U = 32 / G::N1;
    static constexpr int UE = 32 * G::N2;
    static constexpr int XC = (N >= 2048) ? 2 : 5;
    static constexpr int NT = 32 * (XC + 1);
    static constexpr int XBUF = U * LayRow<N>::kFloat2PerLine;
    static constexpr int STAGE = 4 * UE;
    static constexpr int SPW0 = (kSmemBudgetK - XC * XBUF * 8 - N * 8) / (XC * STAGE * 8);
    static constexpr int SPW = SPW0 > 2 ? 2 : SPW0;
    static constexpr int S = XC * SPW;
    static_assert(SPW >= 1, "krylov x pipeline needs >= 1 stage per consumer warp");
    static constexpr int SMEM = (S * STAGE + XC * XBUF + N) * 8 + 2 * S * 8;
};

// Stage slots per mode (each slot = one unit of one field):
//   K_PFWD: r, p, v, B     K_VINV: work, p, B, rhat
//   K_SFWD: r, v, B        K_TINV: work, s, B
//   K_OFWD: p, B           K_OINV: work, p, B      (plain M p -> v, for GMRES)
template <int N, int MODE>
__global__ void __launch_bounds__(XOp<N>::NT, 1) k_xop(KParams p) {
    using G = LineGeo<N>;
    using T = XOp<N>;
    constexpr int NSLOT = (MODE == K_OFWD) ? 2 : ((MODE == K_SFWD || MODE == K_TINV || MODE == K_OINV) ? 3 : 4);
    constexpr bool INV = (MODE == K_VINV || MODE == K_TINV || MODE == K_OINV);
    constexpr bool PLAIN = (MODE == K_OFWD || MODE == K_OINV);   // GMRES: host-driven, no device state
    constexpr int NV = (MODE == K_TINV) ? 3 : (MODE == K_VINV ? 2 : (MODE == K_SFWD ? 1 : 0));
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float2 *stages = reinterpret_cast<float2 *>(smem_raw);
    float2 *xbufs = stages + T::S * T::STAGE;
    float2 *sm_tw = xbufs + T::XC * T::XBUF;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm_tw + N);
    uint64_t *empty = full + T::S;

    if (!PLAIN) {
        const int status = p.st->status;
        if (p.st->k >= p.st->kmax || status != ST_RUNNING) return;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const KState ks = PLAIN ? KState{} : *p.ks;
    const float2 beta = tof(ks.beta), omega = tof(ks.omega), alpha = tof(ks.alpha);
    double acc[NV > 0 ? NV : 1];
#pragma unroll
    for (int q = 0; q < (NV > 0 ? NV : 1); ++q) acc[q] = 0.0;

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
    const float2 *src[4];
    if (MODE == K_PFWD) { src[0] = p.r; src[1] = p.p; src[2] = p.v; src[3] = p.B; }
    if (MODE == K_VINV) { src[0] = p.work; src[1] = p.p; src[2] = p.B; src[3] = p.rh; }
    if (MODE == K_SFWD) { src[0] = p.r; src[1] = p.v; src[2] = p.B; src[3] = nullptr; }
    if (MODE == K_TINV) { src[0] = p.work; src[1] = p.s; src[2] = p.B; src[3] = nullptr; }
    if (MODE == K_OFWD) { src[0] = p.p; src[1] = p.B; src[2] = nullptr; src[3] = nullptr; }
    if (MODE == K_OINV) { src[0] = p.work; src[1] = p.p; src[2] = p.B; src[3] = nullptr; }

    if (warp == T::XC) {
        if (lane == 0) {
            for (int i = 0; i < nloc; ++i) {
                const int s = i % T::S;
                if (i >= T::S && !mbar_wait(&empty[s], ((i / T::S) - 1) & 1)) {
                    if (atomicCAS(&p.st->err, 0, 8) == 0) p.st->err_info = i;
                    break;
                }
                const long long off = (blockIdx.x + (long long)i * gridDim.x) * T::UE;
                float2 *st = stages + s * T::STAGE;
                mbar_arrive_expect_tx(&full[s], NSLOT * ub);
#pragma unroll
                for (int q = 0; q < NSLOT; ++q) bulk_g2s(st + q * T::UE, src[q] + off, ub, &full[s]);
            }
        }
        __syncwarp();
    } else {
        const int lq = lane / G::N1, j = lane % G::N1;
        const LayRow<N> lay{xbufs + warp * T::XBUF + lq * LayRow<N>::kFloat2PerLine};
        for (int i = warp; i < nloc; i += T::XC) {
            const int s = i % T::S;
            if (!mbar_wait(&full[s], (i / T::S) & 1)) {
                if (lane == 0 && atomicCAS(&p.st->err, 0, 9) == 0) p.st->err_info = i;
                break;
            }
            const float2 *st = stages + s * T::STAGE;
            const long long gb = (blockIdx.x + (long long)i * gridDim.x) * T::UE + lq * N + j;
            const int sb = lq * N + j;
            float2 v[G::N2];
            float la[4] = {0.f, 0.f, 0.f, 0.f};
            if constexpr (!INV) {
                // prologue: the new direction (p or s), stored, then u = B * it
#pragma unroll
                for (int m = 0; m < G::N2; ++m) {
                    const int e = sb + G::N1 * m;
                    const long long gi = gb + G::N1 * m;
                    float2 d;
                    if (MODE == K_OFWD) {   // plain: u = B p
                        d = st[e];
                    } else if (MODE == K_PFWD) {   // p = r + beta (p - omega v)
                        const float2 t = csub(st[T::UE + e], cmul(omega, st[2 * T::UE + e]));
                        d = cadd(st[e], cmul(beta, t));
                        p.p[gi] = d;
                    } else {                // s = r - alpha v
                        d = csub(st[e], cmul(alpha, st[T::UE + e]));
                        p.s[gi] = d;
                        la[0] += cabs2(d);
                    }
                    v[m] = cmul(st[(MODE == K_PFWD ? 3 : (MODE == K_OFWD ? 1 : 2)) * T::UE + e], d);
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                fft_line<N, false, LayRow<N>, true>(v, lay, j, sm_tw);
#pragma unroll
                for (int m = 0; m < G::N2; ++m) p.work[gb + G::N1 * m] = v[m];
            } else {
                // x inverse (conj trick) -> y = (L+1)^-1 B u; out = B (u - y) + inner products
#pragma unroll
                for (int m = 0; m < G::N2; ++m) v[m] = cconj(st[sb + G::N1 * m]);
                fft_line<N, false, LayRow<N>, true>(v, lay, j, sm_tw);
#pragma unroll
                for (int m = 0; m < G::N2; ++m) {
                    const int e = sb + G::N1 * m;
                    const long long gi = gb + G::N1 * m;
                    const float2 u = st[T::UE + e], b = st[2 * T::UE + e];
                    const float2 o = cmul(b, csub(u, cconj(v[m])));
                    if (MODE == K_OINV) {                 // plain: v = M p
                        p.v[gi] = o;
                    } else if (MODE == K_VINV) {          // v; (rhat, v)
                        p.v[gi] = o;
                        const float2 rh = st[3 * T::UE + e];
                        la[0] += rh.x * o.x + rh.y * o.y;
                        la[1] += rh.x * o.y - rh.y * o.x;
                    } else {                              // t; (t, s), (t, t)
                        p.t[gi] = o;
                        la[0] += o.x * u.x + o.y * u.y;
                        la[1] += o.x * u.y - o.y * u.x;
                        la[2] += cabs2(o);
                    }
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
#pragma unroll
            for (int q = 0; q < (NV > 0 ? NV : 1); ++q) acc[q] += (double)la[q];
        }
    }
    if constexpr (NV > 0) {
        double tot[NV];
        if (!grid_sums<T::NT, NV>(acc, p.st, p.partials, tot)) return;
        KState *k = p.ks;
        if (MODE == K_VINV) {
            const double2 rv = make_double2(tot[0], tot[1]);
            if (rv.x == 0.0 && rv.y == 0.0) { p.st->status = ST_DIVERGED; k->breakdown = 1; return; }
            k->alpha = ddiv(k->rho, rv);
        } else if (MODE == K_SFWD) {
            const double rs = sqrt(tot[0]) / k->nb;
            k->res_s = rs;
            if (!(rs <= 1e6)) p.st->status = ST_DIVERGED;
            else if (p.st->tol > 0.0 && rs < p.st->tol) p.st->status = ST_STOP_PENDING;   // half-step stop
        } else {
            if (tot[2] == 0.0) { p.st->status = ST_DIVERGED; k->breakdown = 1; return; }
            k->omega = make_double2(tot[0] / tot[2], tot[1] / tot[2]);
        }
    }
}

// x += alpha p + omega s; r = s - omega t; (rhat, r), ||r||  (or, after the
// half-step stop, x += alpha p only).  Grid-stride over all voxels.
__global__ void __launch_bounds__(256) k_kupd(KParams p) {
    const int status = p.st->status;
    if (p.st->k >= p.st->kmax || (status != ST_RUNNING && status != ST_STOP_PENDING)) return;
    const bool half = status == ST_STOP_PENDING;
    const KState ks = *p.ks;
    const float2 alpha = tof(ks.alpha), omega = tof(ks.omega);
    float la[3] = {0.f, 0.f, 0.f};
    double acc[3] = {0.0, 0.0, 0.0};
    // 128-bit accesses (two complex values) and 2 pairs per thread and step,
    // so each thread keeps ~10 independent loads in flight (the kernel is
    // HBM-bound; one complex per step left it latency-bound, ncu)
    const long long n2 = p.nvox / 2;                // nvox is even (power-of-two extents)
    const float4 *P = reinterpret_cast<const float4 *>(p.p), *Sv = reinterpret_cast<const float4 *>(p.s);
    const float4 *Tv = reinterpret_cast<const float4 *>(p.t), *RH = reinterpret_cast<const float4 *>(p.rh);
    float4 *X = reinterpret_cast<float4 *>(p.x), *R = reinterpret_cast<float4 *>(p.r);
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < n2; i0 += 2 * stride) {
        float4 pp[2], xx[2], ss[2], tt[2], rh[2];
        bool ok[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const long long i = i0 + u * stride;
            ok[u] = i < n2;
            if (ok[u]) {
                pp[u] = P[i];
                xx[u] = X[i];
                if (!half) {
                    ss[u] = Sv[i];
                    tt[u] = Tv[i];
                    rh[u] = RH[i];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (!ok[u]) continue;
            const long long i = i0 + u * stride;
            float2 x0 = cadd(make_float2(xx[u].x, xx[u].y), cmul(alpha, make_float2(pp[u].x, pp[u].y)));
            float2 x1 = cadd(make_float2(xx[u].z, xx[u].w), cmul(alpha, make_float2(pp[u].z, pp[u].w)));
            if (half) {
                X[i] = make_float4(x0.x, x0.y, x1.x, x1.y);
                continue;
            }
            const float2 s0 = make_float2(ss[u].x, ss[u].y), s1 = make_float2(ss[u].z, ss[u].w);
            x0 = cadd(x0, cmul(omega, s0));
            x1 = cadd(x1, cmul(omega, s1));
            X[i] = make_float4(x0.x, x0.y, x1.x, x1.y);
            const float2 r0 = csub(s0, cmul(omega, make_float2(tt[u].x, tt[u].y)));
            const float2 r1 = csub(s1, cmul(omega, make_float2(tt[u].z, tt[u].w)));
            R[i] = make_float4(r0.x, r0.y, r1.x, r1.y);
            const float2 h0 = make_float2(rh[u].x, rh[u].y), h1 = make_float2(rh[u].z, rh[u].w);
            la[0] += h0.x * r0.x + h0.y * r0.y + h1.x * r1.x + h1.y * r1.y;
            la[1] += h0.x * r0.y - h0.y * r0.x + h1.x * r1.y - h1.y * r1.x;
            la[2] += cabs2(r0) + cabs2(r1);
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) { acc[q] += (double)la[q]; la[q] = 0.f; }   // fp64 across steps
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) acc[q] += (double)la[q];
    double tot[3];
    if (!grid_sums<256, 3>(acc, p.st, p.partials, tot)) return;
    KState *k = p.ks;
    IterState *st = p.st;
    const long long k1 = st->k + 1;
    st->k = k1;
    if (half) {   // converged at the half step: r = s, reported residual ||s|| / ||b||
        st->r = k->res_s;
        p.hist[k1 % p.hist_cap] = k->res_s;
        st->status = ST_DONE_CONV;
        return;
    }
    const double rr = sqrt(tot[2]) / k->nb;
    st->r = rr;
    p.hist[k1 % p.hist_cap] = rr;
    const double2 rho1 = make_double2(tot[0], tot[1]);
    if (!(rr <= 1e6)) { st->status = ST_DIVERGED; return; }
    if (st->tol > 0.0 && rr < st->tol) { st->status = ST_DONE_CONV; return; }
    if ((rho1.x == 0.0 && rho1.y == 0.0) || (k->omega.x == 0.0 && k->omega.y == 0.0)) {
        st->status = ST_DIVERGED;
        k->breakdown = 1;
        return;
    }
    k->beta = dmul(ddiv(rho1, k->rho), ddiv(k->alpha, k->omega));
    k->rho = rho1;
}

// GMRES(m) Gram-Schmidt blocks (NB <= 8 basis vectors per launch):
//   GS_DOT:  partials of (U_j, z), j < NB (and ||z||^2 when want_norm)
//   GS_AXPY: z <- scale (z - sum_j c_j U_j)  (and ||z||^2 of the result)
// Per-thread fp32 over chunks of 64 steps, fp64 across chunks, fixed-order
// CTA sums -> one row of partials per CTA (the host sums them in order).
// The axpy moves two complex values per thread and access (128-bit; n is
// even: power-of-two extents).
// Launched with kGsCtasPerSm = 3 CTAs per SM and a grid of 3 x SMs, so every
// CTA is resident at once (the grid-stride loop gives all CTAs equal work;
// before, a 4 x SMs grid of an 80-register kernel ran its last quarter as a
// second wave: the dot at 62 % of the copy peak), and the register budget
// (85) lets ptxas keep the NB + 1 loads back to back.
template <int NB, int MODE>
__global__ void __launch_bounds__(256, kGsCtasPerSm) k_gs(GSParams p) {
    constexpr int K = (MODE == GS_DOT) ? 2 * NB + 1 : 1;
    // the fp64 accumulators live in shared memory (the dot's 2 NB + 1 of them
    // would take 34 registers)
    __shared__ double acc_sh[K][256];
    float la[K];
#pragma unroll
    for (int q = 0; q < K; ++q) { acc_sh[q][threadIdx.x] = 0.0; la[q] = 0.f; }
    const long long stride = (long long)gridDim.x * blockDim.x;
    int cnt = 0;
    if (MODE == GS_DOT) {
        // one complex per thread and step (2 NB + 1 fp32 partials and NB + 1
        // 64-bit loads in flight)
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < p.n; i += stride) {
            const float2 z = p.z[i];
            float2 u[NB];
#pragma unroll
            for (int b = 0; b < NB; ++b) u[b] = p.U[b][i];
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                la[2 * b] += u[b].x * z.x + u[b].y * z.y;
                la[2 * b + 1] += u[b].x * z.y - u[b].y * z.x;
            }
            la[2 * NB] += cabs2(z);
            if (++cnt == 64) {
#pragma unroll
                for (int q = 0; q < K; ++q) { acc_sh[q][threadIdx.x] += (double)la[q]; la[q] = 0.f; }
                cnt = 0;
            }
        }
    } else {
        // two complex values per thread and step (128-bit accesses)
        const long long n2 = p.n / 2;
        float4 *Z = reinterpret_cast<float4 *>(p.z);
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += stride) {
            const float4 z4 = Z[i];
            float4 u4[NB];
#pragma unroll
            for (int b = 0; b < NB; ++b) u4[b] = reinterpret_cast<const float4 *>(p.U[b])[i];
            float2 z[2] = {make_float2(z4.x, z4.y), make_float2(z4.z, z4.w)};
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                z[0] = csub(z[0], cmul(p.c[b], make_float2(u4[b].x, u4[b].y)));
                z[1] = csub(z[1], cmul(p.c[b], make_float2(u4[b].z, u4[b].w)));
            }
            z[0] = cmul(p.scale, z[0]);
            z[1] = cmul(p.scale, z[1]);
            Z[i] = make_float4(z[0].x, z[0].y, z[1].x, z[1].y);
            la[0] += cabs2(z[0]) + cabs2(z[1]);
            if (++cnt == 64) {
                acc_sh[0][threadIdx.x] += (double)la[0];
                la[0] = 0.f;
                cnt = 0;
            }
        }
    }
    __shared__ double sh[8][K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
        double v = warp_sum_d(acc_sh[q][threadIdx.x] + (double)la[q]);
        if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5][q] = v;
    }
    __syncthreads();
    if (threadIdx.x < K) {
        double s = 0.0;
        for (int w = 0; w < 8; ++w) s += sh[w][threadIdx.x];
        p.partials[(size_t)blockIdx.x * K + threadIdx.x] = s;
    }
}

// ========================================================= launchers ====
template <int N, int MODE>
static cudaError_t xop_t(const KParams &p, int grid, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_xop<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, XOp<N>::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    k_xop<N, MODE><<<grid, XOp<N>::NT, XOp<N>::SMEM, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_xop(int N, KMode mode, const KParams &p, int grid, cudaStream_t s) {
#define XO_CASE(n)                                                   \
    case n:                                                          \
        if (mode == K_PFWD) return xop_t<n, K_PFWD>(p, grid, s);     \
        if (mode == K_VINV) return xop_t<n, K_VINV>(p, grid, s);     \
        if (mode == K_SFWD) return xop_t<n, K_SFWD>(p, grid, s);     \
        if (mode == K_OFWD) return xop_t<n, K_OFWD>(p, grid, s);     \
        if (mode == K_OINV) return xop_t<n, K_OINV>(p, grid, s);     \
        return xop_t<n, K_TINV>(p, grid, s);
    switch (N) { XO_CASE(16) XO_CASE(32) XO_CASE(64) XO_CASE(128) XO_CASE(256) XO_CASE(512) XO_CASE(1024)
                 XO_CASE(2048) default: return cudaErrorInvalidValue; }
#undef XO_CASE
}

template <int MODE>
static cudaError_t gs_mode(int nb, const GSParams &p, int grid, cudaStream_t s) {
    switch (nb) {
#define GS_CASE(b) \
    case b: k_gs<b, MODE><<<grid, 256, 0, s>>>(p); break;
        GS_CASE(1) GS_CASE(2) GS_CASE(3) GS_CASE(4) GS_CASE(5) GS_CASE(6) GS_CASE(7) GS_CASE(8)
#undef GS_CASE
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_gs(int mode, int nb, const GSParams &p, int grid, cudaStream_t s) {
    return mode == GS_DOT ? gs_mode<GS_DOT>(nb, p, grid, s) : gs_mode<GS_AXPY>(nb, p, grid, s);
}

cudaError_t launch_kupd(const KParams &p, int grid, cudaStream_t s) {
    k_kupd<<<resident_grid<k_kupd>(grid, 256), 256, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace usp
