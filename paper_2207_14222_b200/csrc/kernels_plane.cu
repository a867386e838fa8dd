// kernels_plane.cu -- the plane-chained pass.
//
// One iteration of Algorithm 1 on the 4-pass schedule is
// K_B (y forward) -> K_C (z forward, g(p), z inverse; Eq. 12) -> K_D (y
// inverse) -> K_A (x inverse, update, x forward), each a full sweep of the
// 8 GiB `work` array through HBM.  Here the iteration is K_C followed by ONE
// persistent kernel that runs K_D, K_A and K_B of the next iteration plane
// by plane: a z-plane's `work` (8 MiB at 1024^2) is written by its y-inverse
// units, read and rewritten by its x units and read again by its y-forward
// units while it sits in L2, so HBM sees only K_C's sweep (16 B/voxel), the
// y-inverse's read and the y-forward's write of `work` (8 + 8) and the x
// pass's operands (x read + write, B read; + s or Delta by form): 56 instead
// of 88 B/voxel per iteration for the C5 workload (x-form, sparse source).
// The invariant between iterations becomes "work = FFT_y FFT_x (u)" (the
// setup runs one K_B after its x pass).
//
// CTA roles (one cooperative launch, 1 CTA per SM, 512 threads; all CTAs
// co-resident, so roles can wait on each other):
//   y CTAs (blockIdx < ny_ctas) claim y units from a global counter:
//     D(z, t)  y inverse of columns [16 t, 16 t + 16) of plane z: TMA tile load
//              of K_C's output, the 16-column four-step FFT of kernels_stile.cu,
//              register stores into `work` (L2); d_done[z] += 1
//     B(z, t)  y forward of the same tile once a_done[z] = 1024: TMA load from
//              L2, FFT, stores to `work` (HBM, for the next K_C)
//     in "stages" s = [D(s, *), B(s - 3, *)], the next tile's load issued as
//     soon as the current one is in registers (as k_stile);
//   x CTAs (the rest) run the x pass of kernels_pipe.cu's k_xpass_pipe on the
//     lines l = rank + i * n_x (plane order): one producer warp issues bulk
//     copies of work (L2), x, B (+ s | Delta) into one stage per consumer
//     warp once d_done[z] = 64; consumer warps run the x inverse FFT, the
//     update of the form the state selects (x-form, Delta-form, probe,
//     switch; kcommon.cuh xform_act), the next chain's u, the x forward FFT
//     and the sparse source lines (R-31), store x and work, and publish the
//     line (a_done[z] += 1) with its residual partial.
// Every wait is for work claimed or assigned before it in plane order, so
// the schedule cannot deadlock.  Cross-CTA data moves through L2: generic
// stores are published with fence.proxy.async.global + a gpu-scope release
// and read by TMA / bulk copies after the matching acquire.  The residual:
// one fixed-order fp64 partial per line (lanes -> warp shuffle tree), summed
// by the last CTA in line order -- deterministic whatever the timing.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fft_core.cuh"
#include "kcommon.cuh"
#include "stile_core.cuh"
#include "tma.cuh"
#include "usp_internal.h"

namespace usp {

struct PlaneGeo {
    static constexpr int N = kPlaneN;          // nx = ny
    using G = LineGeo<N>;                      // N1 = N2 = 32
    using T = STile<N>;                        // 16 columns x N rows, 512 threads, two-round exchange
    static_assert(G::N1 == 32 && G::N2 == 32 && T::COLS == 16 && T::FLIP, "plane pass geometry");
    static constexpr int NT = T::NT;           // 512
    static constexpr int TPP = N / T::COLS;    // 64 tiles (D or B units) per plane
    static constexpr int LAG = 3;              // B(z) sits LAG y-stages after D(z)
    static constexpr int YPS = 2 * TPP;        // y units per stage
    static constexpr int H = G::N2 / 2;
    static constexpr int XWP = H + 1;          // x exchange: row pitch (float2), odd
    static constexpr int XW = G::N1 * XWP;     // float2 per consumer warp (two-round exchange)
    static constexpr int YSMEM = (T::TILE + T::XB + N) * 8 + 64;
};

// x role geometry per instance: LEAN = x-form passes of a sparse-source plan
// (stages hold work, x, B); otherwise work, (s | Delta), x, B
template <bool LEAN>
struct XRole {
    using PG = PlaneGeo;
    static constexpr int N = PG::N;
    static constexpr int XC = LEAN ? 7 : 6;    // consumer warps (+ one producer warp)
    static constexpr int NSLOT = LEAN ? 3 : 4;
    static constexpr int S = XC;               // one stage per consumer warp (bulk copies complete out of order)
    static constexpr int SD = N, SX = (LEAN ? 1 : 2) * N, SB = (LEAN ? 2 : 3) * N;   // slot offsets (float2)
    static constexpr int STAGE = NSLOT * N;
    static constexpr int SMEM = (S * STAGE + XC * PG::XW + N) * 8 + 2 * S * 8 + 64;
    static_assert(SMEM <= 232448, "x role shared memory");
};

template <bool LEAN>
constexpr int plane_smem() {
    return PlaneGeo::YSMEM > XRole<LEAN>::SMEM ? PlaneGeo::YSMEM : XRole<LEAN>::SMEM;
}

enum : int { U_D = 0, U_B = 2, U_NONE = 3 };

struct YUnit {
    int type;
    int idx;        // tile t
    long long z;
};

__device__ __forceinline__ YUnit ydecode(unsigned long long u, long long nz) {
    using PG = PlaneGeo;
    YUnit r{U_NONE, 0, 0};
    const long long s = (long long)(u / PG::YPS);
    const int q = (int)(u - (unsigned long long)s * PG::YPS);
    if (q < PG::TPP) {
        if (s < nz) r = YUnit{U_D, q, s};
    } else if (s >= PG::LAG && s - PG::LAG < nz) {
        r = YUnit{U_B, q - PG::TPP, s - PG::LAG};
    }
    return r;
}

// Build-time tracing (tools only): -DUSP_PLANE_TRACE=1 accumulates per-role
// wait times (globaltimer ns, summed over threads that wait) and the last CTA
// prints them.
#ifndef USP_PLANE_TRACE
#define USP_PLANE_TRACE 0
#endif
enum { TR_Y_ROLE = 0, TR_Y_MBAR, TR_Y_DEP, TR_X_ROLE, TR_X_FULL, TR_X_EMPTY, TR_X_DEP, TR_Y_UNITS, TR_X_LINES, TR_N };
__device__ unsigned long long g_trace[TR_N + 1];   // [TR_N]: discarded
struct TraceT {
    int k;
    uint64_t t0;
    __device__ explicit TraceT(int key) : k(key), t0(USP_PLANE_TRACE ? globaltimer_ns() : 0) {}
    __device__ ~TraceT() {
        if (USP_PLANE_TRACE) atomicAdd(&g_trace[k], (unsigned long long)(globaltimer_ns() - t0));
    }
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// generic-proxy global writes <-> async-proxy (TMA / bulk copy) accesses
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// wait until *cnt >= want (acquire); false after 4 s (watchdog)
__device__ __forceinline__ bool wait_count(const unsigned *cnt, unsigned want) {
    if (ld_acquire(cnt) >= want) return true;
    const uint64_t t0 = globaltimer_ns();
    unsigned n = 0;
    while (ld_acquire(cnt) < want) {
        __nanosleep(32);
        if ((++n & 255u) == 0 && globaltimer_ns() - t0 > 4000000000ull) return false;
    }
    return true;
}

// Four-step DFT of one line held by one warp (lane j: x[j + 32 n2]); the
// exchange runs in two rounds through a half-size per-warp buffer with the
// shift flips of stile_fft (kernels_stile.cu header), the flip bit being the
// lane's top row bit (b = j >> 4; the caller negates odd inputs / outputs
// for b = 1).
__device__ __forceinline__ void xline_fft(float2 (&v)[32], float2 *xw, const float2 *sm_tw, int j) {
    using PG = PlaneGeo;
    constexpr int H = PG::H, N1 = 32, P = PG::XWP;
    dft<32, false>(v);
    const int b = (j >> 4) & 1;
    const float2 *tw0 = sm_tw + (H * b) * N1 + j;
    const float2 *tw1 = sm_tw + (H * (1 - b)) * N1 + j;
#pragma unroll
    for (int s = 0; s < 32; ++s) {
        const float2 w = (s < H) ? tw0[s * N1] : tw1[(s - H) * N1];
        v[s] = cmul(v[s], w);
    }
    float2 *wb = xw + j * P;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
#pragma unroll
        for (int q = 0; q < H; ++q) wb[q] = v[r * H + q];
        __syncwarp();
        const float2 *rb = xw + (H * (r ^ b)) * P + (j & (H - 1));
#pragma unroll
        for (int q = 0; q < H; ++q) v[r * H + q] = rb[q * P];
        __syncwarp();
    }
    dft<32, false>(v);
}

__device__ __forceinline__ void flip_odd(float2 (&v)[32], float sg) {
#pragma unroll
    for (int m = 1; m < 32; m += 2) v[m] = cscale(v[m], sg);
}

// ---------------------------------------------------------------- y role --
__device__ __noinline__ void y_role(const CUtensorMap &mapy, const PParams &p, unsigned char *smem_raw, int act) {
    using PG = PlaneGeo;
    using T = PG::T;
    constexpr int N = PG::N;
    float2 *stage = reinterpret_cast<float2 *>(smem_raw);
    float2 *xb = stage + T::TILE;
    float2 *sm_tw = xb + T::XB;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm_tw + N);
    __shared__ unsigned long long sh_u;
    __shared__ int sh_ok;
    const int tid = threadIdx.x;
    const long long nz = p.nz;
    const long long plane = (long long)N * N;
    const unsigned long long nunits = (unsigned long long)PG::YPS * (unsigned long long)(nz + PG::LAG);
    const int c = tid % T::COLS, j = tid / T::COLS;
    const float sg = ((j >> 4) & 1) ? -1.f : 1.f;   // warp-uniform (shift flips)
    // sparse source (R-31): the x role formed FFT_x(B x); FFT_x(s) of the
    // source lines is added to the tile before its y forward FFT (linearity)
    const bool add_lines = p.s_sparse && (act == ACT_X || act == ACT_PROBE);

    // thread 0: units are claimed one ahead (the atomic's latency hides
    // behind a tile's FFT); a claimed index past the empty slots of the first
    // and last stages is replaced by the next one
    auto valid = [&](unsigned long long u) -> unsigned long long {
        while (u < nunits && ydecode(u, nz).type == U_NONE) u = atomicAdd(p.ctr, 1ull);
        return u;
    };
    // thread 0: issue the tile load of unit u (a B tile once its plane's x lines are in)
    auto issue = [&](unsigned long long uu) -> bool {
        const YUnit y = ydecode(uu, nz);
        if (y.type == U_B) {
            bool okw;
            {
                TraceT tr(TR_Y_DEP);
                okw = wait_count(p.a_done + y.z, N);
            }
            if (!okw) {
                if (atomicCAS(&p.st->err, 0, 23) == 0) p.st->err_info = (int)y.z;
                return false;
            }
            fence_proxy_async_global();   // the x lines' generic stores -> this TMA read
        }
        mbar_arrive_expect_tx(full, T::TILE * 8);
#pragma unroll
        for (int bx = 0; bx < N / T::BOXN; ++bx)
            tma_load_3d(stage + bx * T::BOXN * T::COLS, &mapy, y.idx * T::COLS, bx * T::BOXN, (int)y.z, full);
        return true;
    };

    unsigned long long ahead = 0;   // thread 0: the claim after the next
    if (tid == 0) {
        mbar_init(full, 1);
        fence_mbar_init();
        unsigned long long u0 = valid(atomicAdd(p.ctr, 1ull));
        if (u0 < nunits && !issue(u0)) u0 = ~0ull;
        sh_u = u0;
        ahead = atomicAdd(p.ctr, 1ull);
    }
    load_twiddles<N>(sm_tw, p.tw);
    __syncthreads();
    unsigned long long cur = sh_u;
    int it = 0;
    long long pend_z = -1;          // a finished D tile not yet published (d_done)
    while (cur < nunits) {
        const YUnit u = ydecode(cur, nz);
        sh_ok = 1;
        bool okm;
        {
            if (USP_PLANE_TRACE && tid == 0) {
                TraceT tr(TR_Y_MBAR);
                okm = mbar_wait(full, it & 1);
                atomicAdd(&g_trace[TR_Y_UNITS], 1ull);
            } else {
                okm = mbar_wait(full, it & 1);
            }
        }
        if (!okm) {
            if (tid == 0 && atomicCAS(&p.st->err, 0, 21) == 0) p.st->err_info = (int)u.z;
            sh_ok = 0;
        }
        ++it;
        if (add_lines && u.type == U_B) {
            // rows y of this plane that carry source lines (a handful at most)
            for (int q = 0; q < p.s_count; ++q) {
                const int l = p.s_list[q];
                if ((long long)(l / N) != u.z) continue;
                if (tid < T::COLS) {
                    const float2 a = p.s_comp[(long long)q * N + u.idx * T::COLS + tid];
                    float2 &w = stage[(l % N) * T::COLS + tid];
                    w = make_float2(w.x + a.x, w.y + a.y);
                }
            }
            __syncthreads();
        }
        float2 v[32];
#pragma unroll
        for (int m = 0; m < 32; ++m) {
            const float2 a = stage[(j + 32 * m) * T::COLS + c];
            v[m] = (u.type == U_D) ? cconj(a) : a;
        }
        fence_proxy_async_smem();
        if (pend_z >= 0) {                      // the previous D tile's stores are long done:
            fence_proxy_async_global();         //   generic stores -> the x role's bulk reads
            __threadfence();                    //   release at gpu scope (with the barrier below)
        }
        __syncthreads();                        // stage consumed: load the next tile
        if (tid == 0) {
            if (pend_z >= 0) atomicAdd(p.d_done + pend_z, 1u);
            unsigned long long nx = valid(ahead);
            if (nx < nunits) {
                if (!issue(nx)) nx = ~0ull;
                ahead = atomicAdd(p.ctr, 1ull);
            }
            sh_u = nx;
        }
        pend_z = -1;
        if (!sh_ok) break;
        flip_odd(v, sg);
        stile_fft<N>(v, xb, sm_tw, c, j, 1);   // (its barriers also publish sh_u)
        flip_odd(v, sg);
        float2 *tb = p.work + u.z * plane + u.idx * T::COLS + c;
        if (u.type == U_D) {
            store_slots<N, S_INV, 0, 32>(v, tb, N, j, c);
            pend_z = u.z;
        } else {
            store_slots<N, S_FWD, 0, 32>(v, tb, N, j, c);
        }
        __syncthreads();
        cur = sh_u;
    }
    if (pend_z >= 0) {
        fence_proxy_async_global();
        __threadfence();
        __syncthreads();
        if (tid == 0) atomicAdd(p.d_done + pend_z, 1u);
    }
}

// ---------------------------------------------------------------- x role --
template <bool LEAN, bool DSPEC>
__device__ __noinline__ void x_role(const PParams &p, unsigned char *smem_raw, float alpha, int act) {
    using PG = PlaneGeo;
    using X = XRole<LEAN>;
    constexpr int N = PG::N;
    float2 *stages = reinterpret_cast<float2 *>(smem_raw);
    float2 *xws = stages + X::S * X::STAGE;
    float2 *sm_tw = xws + X::XC * PG::XW;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm_tw + N);
    uint64_t *empty = full + X::S;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long long nz = p.nz;
    const long long rank = blockIdx.x - p.ny_ctas, nxc = gridDim.x - p.ny_ctas;
    const long long nlines = nz * N;
    const int nloc = (int)((nlines - rank + nxc - 1) / nxc);

    const bool dform = act == ACT_DELTA;
    const float c1 = dform ? alpha : 1.f;
    const bool store_x = act == ACT_DELTA || act == ACT_X, store_d = act != ACT_X;
    const bool u_from_d = act == ACT_DELTA || act == ACT_TO_DELTA;
    // slot 1: Delta (Delta-form) or s (x-form passes); the sparse source is
    // added as transformed lines instead (R-31)
    const float2 *a1p = (act != ACT_DELTA) ? p.s : p.delta;
    const bool need1 = !(p.s_sparse && act != ACT_DELTA);
    const bool stage1 = need1 && !LEAN;
    const float e1 = ((act == ACT_X || act == ACT_PROBE) && need1) ? 1.f : 0.f;

    if (tid == 0) {
        for (int s = 0; s < X::S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_mbar_init();
    }
    load_twiddles<N>(sm_tw, p.tw);
    __syncthreads();

    if (warp == X::XC) {
        // ---------------------------------------------------- producer warp
        if (lane == 0) {
            const uint32_t ub = N * 8u;
            long long zready = -1;
            for (int i = 0; i < nloc; ++i) {
                const int s = i % X::S;
                bool oke = true;
                if (i >= X::S) {
                    TraceT tr(TR_X_EMPTY);
                    oke = mbar_wait(&empty[s], ((i / X::S) - 1) & 1);
                }
                if (!oke) {
                    if (atomicCAS(&p.st->err, 0, 24) == 0) p.st->err_info = i;
                    break;
                }
                const long long line = rank + (long long)i * nxc;
                const long long z = line / N;
                if (z > zready) {   // plane z's y-inverse tiles are in `work`
                    bool okd;
                    {
                        TraceT tr(TR_X_DEP);
                        okd = wait_count(p.d_done + z, PG::TPP);
                    }
                    if (!okd) {
                        if (atomicCAS(&p.st->err, 0, 22) == 0) p.st->err_info = (int)z;
                        break;
                    }
                    fence_proxy_async_global();
                    zready = z;
                }
                const long long off = line * N;
                float2 *st = stages + s * X::STAGE;
                mbar_arrive_expect_tx(&full[s], (stage1 ? 4 : 3) * ub);
                bulk_g2s(st, p.work + off, ub, &full[s]);
                if (stage1) bulk_g2s(st + X::SD, a1p + off, ub, &full[s]);
                bulk_g2s(st + X::SX, p.x + off, ub, &full[s]);
                bulk_g2s(st + X::SB, p.B + off, ub, &full[s]);
            }
        }
        __syncwarp();
    } else if (warp < X::XC) {
        // ---------------------------------------------------- consumer warps
        const int j = lane;
        const float sg = ((j >> 4) & 1) ? -1.f : 1.f;   // per lane
        float2 *xw = xws + warp * PG::XW;
        long long pend_z = -1;   // the previous line's plane, published one line late
        auto publish = [&]() {   // the previous line's work stores -> a_done (release)
            fence_proxy_async_global();   // generic stores -> the y role's TMA reads
            __threadfence();
            __syncwarp();
            if (lane == 0) atomicAdd(p.a_done + pend_z, 1u);
            pend_z = -1;
        };
        for (int i = warp; i < nloc; i += X::XC) {
            const int s = i % X::S;
            // never wait for the producer with a line unpublished (the producer
            // may be waiting for y tiles that wait for this plane's lines)
            if (pend_z >= 0 && !mbar_try_wait(&full[s], (i / X::S) & 1)) publish();
            bool okf;
            if (USP_PLANE_TRACE && lane == 0) {
                TraceT tr(TR_X_FULL);
                okf = mbar_wait(&full[s], (i / X::S) & 1);
                atomicAdd(&g_trace[TR_X_LINES], 1ull);
            } else {
                okf = mbar_wait(&full[s], (i / X::S) & 1);
            }
            if (!okf) {
                if (lane == 0 && atomicCAS(&p.st->err, 0, 25) == 0) p.st->err_info = i;
                break;
            }
            const float2 *st = stages + s * X::STAGE;
            const long long line = rank + (long long)i * nxc;
            const long long gb = line * N + j;
            float2 v[32];
#pragma unroll
            for (int m = 0; m < 32; ++m) v[m] = cconj(st[j + 32 * m]);
            float lacc = 0.f;
#pragma unroll 1
            for (int pass = 0; pass < 2; ++pass) {
                flip_odd(v, sg);
                xline_fft(v, xw, sm_tw, j);
                flip_odd(v, sg);
                if (pass == 1) break;
                // publish the previous line here: its stores were issued before
                // this line's inverse FFT and none since, so the fence is cheap
                if (pend_z >= 0) publish();
                // y = conj(v) = (L+1)^-1 u at positions j + 32 m (the chain is complete)
                if (LEAN && act == ACT_X && !need1) {
#pragma unroll
                    for (int m = 0; m < 32; ++m) {
                        const int e = j + 32 * m;
                        const float2 y = cconj(v[m]), b = st[X::SB + e], xx = st[X::SX + e];
                        const float2 dk = cmul(b, csub(y, xx));
                        const float2 xn = make_float2(fmaf(alpha, dk.x, xx.x), fmaf(alpha, dk.y, xx.y));
                        p.x[gb + 32 * m] = xn;
                        lacc += cabs2(dk);
                        v[m] = cmul(b, xn);
                    }
                } else if (DSPEC && !LEAN && act == ACT_DELTA) {
#pragma unroll
                    for (int m = 0; m < 32; ++m) {
                        const int e = j + 32 * m;
                        const long long gi = gb + 32 * m;
                        const float2 y = cconj(v[m]), b = st[X::SB + e];
                        const float2 d = st[X::SD + e], xx = st[X::SX + e];
                        const float2 t = cmul(b, csub(y, d));
                        const float2 dn = make_float2(fmaf(alpha, t.x, d.x), fmaf(alpha, t.y, d.y));
                        p.x[gi] = make_float2(fmaf(alpha, d.x, xx.x), fmaf(alpha, d.y, xx.y));
                        p.delta[gi] = dn;
                        lacc += cabs2(dn);
                        v[m] = cmul(b, dn);
                    }
                } else {
#pragma unroll
                    for (int m = 0; m < 32; ++m) {
                        // one body for every action (kernels_pipe.cu k_xpass_pipe); a
                        // Delta-form pass on a LEAN launch reads Delta from global memory
                        const int e = j + 32 * m;
                        const long long gi = gb + 32 * m;
                        const float2 y = cconj(v[m]), b = st[X::SB + e];
                        const float2 a1 = !need1 ? make_float2(0.f, 0.f) : (LEAN ? a1p[gi] : st[X::SD + e]);
                        const float2 xx = st[X::SX + e];
                        const float2 t = cmul(b, csub(y, dform ? a1 : xx));
                        const float2 d0 = dform ? a1 : make_float2(0.f, 0.f);
                        const float2 dn = make_float2(fmaf(c1, t.x, d0.x), fmaf(c1, t.y, d0.y));
                        const float2 xi = dform ? a1 : t;
                        const float2 xn = make_float2(fmaf(alpha, xi.x, xx.x), fmaf(alpha, xi.y, xx.y));
                        if (store_x) p.x[gi] = xn;
                        if (store_d) p.delta[gi] = dn;
                        lacc += cabs2(dn);
                        const float2 w = u_from_d ? dn : (act == ACT_X ? xn : xx);
                        const float2 bw = cmul(b, w);
                        v[m] = make_float2(fmaf(e1, a1.x, bw.x), fmaf(e1, a1.y, bw.y));
                    }
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);   // the warp's stage can refill now
            }
#pragma unroll
            for (int m = 0; m < 32; ++m) p.work[gb + 32 * m] = v[m];
            // the line's residual partial (lanes in fp64, fixed shuffle tree)
            const double wsum = warp_sum_d((double)lacc);
            if (lane == 0) p.upart[line] = wsum;
            pend_z = line / N;
        }
        if (pend_z >= 0) publish();
    }
}

template <bool LEAN, bool DSPEC>
__global__ void __launch_bounds__(PlaneGeo::NT, 1) k_plane(const __grid_constant__ CUtensorMap mapy, const __grid_constant__ PParams p) {
    using PG = PlaneGeo;
    constexpr int N = PG::N;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ double sh_red[PG::NT / 32];
    __shared__ int am_last;
    const int tid = threadIdx.x;
    pdl_trigger();
    if (tid == 0) prefetch_tmap(&mapy);
    pdl_wait();

    // the launch's action, read by every CTA before the last CTA's finish
    const int status = p.st->status;
    const long long k = p.st->k, kmax = p.st->kmax;
    const bool probe = p.st->form == FORM_PROBE && status == ST_RUNNING;
    if (!probe && (k >= kmax || (status != ST_RUNNING && status != ST_STOP_PENDING))) return;
    const bool xonly = status == ST_STOP_PENDING;
    const float alpha = (float)p.st->alpha;
    const int act = xform_act(p.st);
    const long long nlines = p.nz * N;

    if (xonly) {
        // final x_{k+1} = x_k + alpha Delta_k after the stop test (reading R-5)
        const long long nv = nlines * N;
        for (long long i = blockIdx.x * (long long)blockDim.x + tid; i < nv; i += (long long)gridDim.x * blockDim.x) {
            const float2 d = p.delta[i];
            const float2 xx = p.x[i];
            p.x[i] = make_float2(fmaf(alpha, d.x, xx.x), fmaf(alpha, d.y, xx.y));
        }
    } else if ((int)blockIdx.x < p.ny_ctas) {
        TraceT tr(TR_Y_ROLE);
        y_role(mapy, p, smem_raw, act);
        if (USP_PLANE_TRACE && tid != 0) tr.k = TR_N;   // one thread per CTA counts the role time
    } else {
        TraceT tr(TR_X_ROLE);
        x_role<LEAN, DSPEC>(p, smem_raw, alpha, act);
        if (USP_PLANE_TRACE && tid != 0) tr.k = TR_N;
    }

    // last CTA: the residual over every line in a fixed order, the finish,
    // and the counters reset for the next launch
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        am_last = atomicAdd(&p.st->counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    double s = 0.0;
    if (!xonly)
        for (long long i = tid; i < nlines; i += PG::NT) s += __ldcg(p.upart + i);
    const double total = block_sum_d<PG::NT>(s, sh_red);
    for (long long i = tid; i < p.nz; i += PG::NT) {
        p.d_done[i] = 0u;
        p.a_done[i] = 0u;
    }
    if (tid == 0) {
        *p.ctr = 0ull;
        p.st->counter = 0u;
        if (p.st->err == 0) finish_xpass(false, xonly, total, p.st, p.red, act);
        if (USP_PLANE_TRACE) {
            printf("plane trace: y_ctas %d  y_role %.3f ms/CTA  y_mbar %.3f  y_dep %.3f  y_units %llu | x_role %.3f "
                   "ms/CTA  x_full %.3f ms/warp  x_empty %.3f  x_dep %.3f  lines %llu\n",
                   p.ny_ctas, g_trace[TR_Y_ROLE] * 1e-6 / p.ny_ctas, g_trace[TR_Y_MBAR] * 1e-6 / p.ny_ctas,
                   g_trace[TR_Y_DEP] * 1e-6 / p.ny_ctas, g_trace[TR_Y_UNITS],
                   g_trace[TR_X_ROLE] * 1e-6 / (gridDim.x - p.ny_ctas),
                   g_trace[TR_X_FULL] * 1e-6 / ((gridDim.x - p.ny_ctas) * XRole<LEAN>::XC),
                   g_trace[TR_X_EMPTY] * 1e-6 / (gridDim.x - p.ny_ctas), g_trace[TR_X_DEP] * 1e-6 / (gridDim.x - p.ny_ctas),
                   g_trace[TR_X_LINES]);
            for (int q = 0; q < TR_N; ++q) g_trace[q] = 0ull;
        }
    }
}

template <bool LEAN, bool DSPEC>
static cudaError_t plane_t(const CUtensorMap &mapy, const PParams &p, int grid, cudaStream_t s) {
    constexpr int SM = plane_smem<LEAN>();
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(k_plane<LEAN, DSPEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    // cooperative: every CTA is resident (the roles wait on each other);
    // programmatic serialization lets the launch overlap K_C's tail
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(PlaneGeo::NT);
    cfg.dynamicSmemBytes = SM;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, k_plane<LEAN, DSPEC>, mapy, p);
}

// instance by the form the host expects (as launch_xpass_pipe): lean
// (sparse-source x-form), dense x-form, Delta-form
cudaError_t launch_plane(const CUtensorMap &mapy, const PParams &p, int grid, cudaStream_t s, bool lean, bool expect_x) {
    if (lean) return plane_t<true, false>(mapy, p, grid, s);
    if (expect_x) return plane_t<false, false>(mapy, p, grid, s);   // the general body (a dedicated
                                                                     // dense x-form body spills at 128 registers)
    return plane_t<false, true>(mapy, p, grid, s);
}

}  // namespace usp
