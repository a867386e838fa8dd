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
// Work units (every CTA of the persistent grid claims them in order from a
// global counter; 1 CTA per SM, 512 threads):
//   D(z, t)  y inverse of columns [16 t, 16 t + 16) of plane z: TMA tile load
//            (prefetched while the CTA's previous unit runs), the 16-column
//            four-step FFT of kernels_stile.cu, register stores into `work`
//   A(z, g)  x pass of lines [16 g, 16 g + 16) of plane z, one line per warp:
//            x inverse FFT, the update of the form the state selects (x-form,
//            Delta-form, probe, switch; kcommon.cuh xform_act), the next
//            chain's u, x forward FFT, sparse source lines (R-31); the
//            line's x / B / (s | Delta) are L2-prefetched one unit ahead
//   B(z, t)  y forward of columns [16 t, 16 t + 16) of plane z, loaded from L2
// in the order of "stages": stage s = [D(s, *), A(s-1, *), B(s-2, *)], so a
// unit's inputs were claimed ~200 claims earlier (148 CTAs in flight) and are
// almost always complete; an A unit waits for d_done[z] = 64, a B unit for
// a_done[z] = 64 (release / acquire at gpu scope, 4-second watchdog).  Units
// only ever wait for units claimed before them, so the schedule cannot
// deadlock whatever the CTA residency.
//
// Cross-unit data moves through L2 with generic-proxy stores and .cg loads
// (the only TMA loads read K_C's output, written by the previous kernel).
// The residual: each A unit writes the fixed-order fp64 sum of its 16 lines;
// the last CTA sums the nz * 64 unit partials in a fixed order (deterministic
// for any assignment of units to CTAs) and runs the x pass's finish.
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
    static constexpr int LPU = NT / 32;        // 16 lines per A unit, one per warp
    static constexpr int APP = N / LPU;        // 64 A units per plane
    static constexpr int UPS = TPP + APP + TPP;   // units per stage
    static constexpr int H = G::N2 / 2;
    static constexpr int XWP = H + 1;          // x exchange: row pitch (float2), odd
    static constexpr int XW = G::N1 * XWP;     // float2 per warp
    static constexpr int XREG = (T::XB > LPU * XW) ? T::XB : LPU * XW;
    static constexpr int SMEM = (T::TILE + XREG + N) * 8 + 64;
};

enum : int { U_D = 0, U_A = 1, U_B = 2, U_NONE = 3 };

struct Unit {
    int type;
    int idx;        // tile t or A group g
    long long z;
};

__device__ __forceinline__ Unit decode(unsigned long long u, long long nz) {
    using PG = PlaneGeo;
    Unit r{U_NONE, 0, 0};
    const long long s = (long long)(u / PG::UPS);
    const int q = (int)(u - (unsigned long long)s * PG::UPS);
    if (q < PG::TPP) {
        if (s < nz) r = Unit{U_D, q, s};
    } else if (q < PG::TPP + PG::APP) {
        if (s >= 1 && s - 1 < nz) r = Unit{U_A, q - PG::TPP, s - 1};
    } else {
        if (s >= 2 && s - 2 < nz) r = Unit{U_B, q - PG::TPP - PG::APP, s - 2};
    }
    return r;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// thread 0: wait until *cnt >= want (acquire); false after 4 s (watchdog)
__device__ __forceinline__ bool wait_count(const unsigned *cnt, unsigned want) {
    if (ld_acquire(cnt) >= want) return true;
    const uint64_t t0 = globaltimer_ns();
    unsigned n = 0;
    while (ld_acquire(cnt) < want) {
        __nanosleep(64);
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

template <bool LEAN, bool DSPEC, bool XSPEC>
__global__ void __launch_bounds__(PlaneGeo::NT, 1) k_plane(const __grid_constant__ CUtensorMap mapy, PParams p) {
    using PG = PlaneGeo;
    using T = PG::T;
    constexpr int N = PG::N;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float2 *stage = reinterpret_cast<float2 *>(smem_raw);
    float2 *xreg = stage + T::TILE;
    float2 *sm_tw = xreg + PG::XREG;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm_tw + N);
    __shared__ unsigned long long sh_next;
    __shared__ double sh_part[PG::LPU];
    __shared__ int sh_ok;
    __shared__ double sh_red[PG::NT / 32];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
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
    const long long nz = p.nz;
    const long long plane = (long long)N * N;

    if (xonly) {
        // final x_{k+1} = x_k + alpha Delta_k after the stop test (reading R-5)
        for (long long i = blockIdx.x * (long long)blockDim.x + tid; i < nz * plane; i += (long long)gridDim.x * blockDim.x) {
            const float2 d = p.delta[i];
            const float2 xx = p.x[i];
            p.x[i] = make_float2(fmaf(alpha, d.x, xx.x), fmaf(alpha, d.y, xx.y));
        }
    } else {
        const bool dform = act == ACT_DELTA;
        const float c1 = dform ? alpha : 1.f;
        const bool store_x = act == ACT_DELTA || act == ACT_X, store_d = act != ACT_X;
        const bool u_from_d = act == ACT_DELTA || act == ACT_TO_DELTA;
        // slot 1: Delta (Delta-form) or s (x-form passes); the sparse source is
        // added as transformed lines instead (R-31)
        const float2 *a1p = (act != ACT_DELTA) ? p.s : p.delta;
        const bool need1 = !(p.s_sparse && act != ACT_DELTA);
        const float e1 = ((act == ACT_X || act == ACT_PROBE) && need1) ? 1.f : 0.f;
        const bool add_lines = p.s_sparse && (act == ACT_X || act == ACT_PROBE);
        const unsigned long long nunits = (unsigned long long)PG::UPS * (unsigned long long)(nz + 2);

        if (tid == 0) {
            mbar_init(full, 1);
            fence_mbar_init();
        }
        load_twiddles<N>(sm_tw, p.tw);
        int lphase = 0;   // completed TMA stage loads of this CTA (mbarrier parity)

        // thread 0: start the next unit's inputs moving (never blocks)
        auto prepare = [&](const Unit &u) {
            if (u.type == U_D) {
                mbar_arrive_expect_tx(full, T::TILE * 8);
#pragma unroll
                for (int bx = 0; bx < N / T::BOXN; ++bx)
                    tma_load_3d(stage + bx * T::BOXN * T::COLS, &mapy, u.idx * T::COLS, bx * T::BOXN, (int)u.z, full);
            } else if (u.type == U_A) {
                const long long off = u.z * plane + (long long)u.idx * PG::LPU * N;
                const uint32_t bytes = PG::LPU * N * 8;
                prefetch_l2(p.x + off, bytes);
                prefetch_l2(p.B + off, bytes);
                if (need1) prefetch_l2(a1p + off, bytes);
            }
        };

        unsigned long long cur = 0;
        if (tid == 0) {
            cur = atomicAdd(p.ctr, 1ull);
            sh_next = cur;
            if (cur < nunits) prepare(decode(cur, nz));
        }
        __syncthreads();
        cur = sh_next;

        while (cur < nunits) {
            const Unit u = decode(cur, nz);
            __syncthreads();   // everyone has read sh_next / finished the previous unit's smem use
            if (tid == 0) {
                sh_next = atomicAdd(p.ctr, 1ull);
                sh_ok = 1;
            }
            __syncthreads();
            const unsigned long long nxt = sh_next;
            const Unit un = (nxt < nunits) ? decode(nxt, nz) : Unit{U_NONE, 0, 0};

            if (u.type == U_NONE) {   // an empty slot of the first / last stages
                if (tid == 0) prepare(un);
            } else if (u.type == U_D || u.type == U_B) {
                // ------------------------------------------------ y pass of a tile
                const int c = tid % T::COLS, j = tid / T::COLS;
                const float sg = ((j >> 4) & 1) ? -1.f : 1.f;   // warp-uniform (shift flips)
                float2 v[32];
                float2 *tb = p.work + u.z * plane + u.idx * T::COLS;   // column 0 of the tile, row 0
                if (u.type == U_D) {
                    if (!mbar_wait(full, lphase & 1)) {
                        if (tid == 0 && atomicCAS(&p.st->err, 0, 21) == 0) p.st->err_info = (int)u.z;
                        sh_ok = 0;
                    }
                    ++lphase;
#pragma unroll
                    for (int m = 0; m < 32; ++m) v[m] = cconj(stage[(j + 32 * m) * T::COLS + c]);
                    fence_proxy_async_smem();
                    __syncthreads();              // stage consumed
                    if (tid == 0) prepare(un);
                } else {
                    if (tid == 0) {
                        prepare(un);
                        if (!wait_count(p.a_done + u.z, PG::APP)) {
                            if (atomicCAS(&p.st->err, 0, 23) == 0) p.st->err_info = (int)u.z;
                            sh_ok = 0;
                        }
                    }
                    __syncthreads();
#pragma unroll
                    for (int m = 0; m < 32; ++m) v[m] = __ldcg(tb + (long long)(j + 32 * m) * N + c);
                }
                if (!sh_ok) break;
                flip_odd(v, sg);
                stile_fft<N>(v, xreg, sm_tw, c, j, 1);
                flip_odd(v, sg);
                if (u.type == U_D) store_slots<N, S_INV, 0, 32>(v, tb + c, N, j, c);
                else store_slots<N, S_FWD, 0, 32>(v, tb + c, N, j, c);
                if (u.type == U_D) {   // publish the tile (release at gpu scope)
                    __threadfence();
                    __syncthreads();
                    if (tid == 0) atomicAdd(p.d_done + u.z, 1u);
                }
            } else {
                // ------------------------------------------------ x pass of 16 lines
                if (tid == 0) {
                    prepare(un);
                    if (!wait_count(p.d_done + u.z, PG::TPP)) {
                        if (atomicCAS(&p.st->err, 0, 22) == 0) p.st->err_info = (int)u.z;
                        sh_ok = 0;
                    }
                }
                __syncthreads();
                if (!sh_ok) break;
                const int j = lane;
                const float sg = ((j >> 4) & 1) ? -1.f : 1.f;   // per lane
                const long long line = u.z * N + (long long)u.idx * PG::LPU + warp;
                const long long gb = line * N + j;
                float2 *xw = xreg + warp * PG::XW;
                float2 v[32];
#pragma unroll
                for (int m = 0; m < 32; ++m) v[m] = cconj(__ldcg(p.work + gb + 32 * m));
                float lacc = 0.f;
#pragma unroll 1
                for (int pass = 0; pass < 2; ++pass) {
                    flip_odd(v, sg);
                    xline_fft(v, xw, sm_tw, j);
                    flip_odd(v, sg);
                    if (pass == 1) break;
                    // y = conj(v) = (L+1)^-1 u at positions j + 32 m (the chain is complete)
                    if (LEAN && act == ACT_X && !need1) {
#pragma unroll
                        for (int m = 0; m < 32; ++m) {
                            const long long gi = gb + 32 * m;
                            const float2 y = cconj(v[m]), b = __ldcg(p.B + gi), xx = __ldcg(p.x + gi);
                            const float2 dk = cmul(b, csub(y, xx));
                            const float2 xn = make_float2(fmaf(alpha, dk.x, xx.x), fmaf(alpha, dk.y, xx.y));
                            p.x[gi] = xn;
                            lacc += cabs2(dk);
                            v[m] = cmul(b, xn);
                        }
                    } else if (XSPEC && act == ACT_X && need1) {
#pragma unroll
                        for (int m = 0; m < 32; ++m) {
                            const long long gi = gb + 32 * m;
                            const float2 y = cconj(v[m]), b = __ldcg(p.B + gi);
                            const float2 sv = __ldcg(p.s + gi), xx = __ldcg(p.x + gi);
                            const float2 dk = cmul(b, csub(y, xx));
                            const float2 xn = make_float2(fmaf(alpha, dk.x, xx.x), fmaf(alpha, dk.y, xx.y));
                            p.x[gi] = xn;
                            lacc += cabs2(dk);
                            const float2 bx = cmul(b, xn);
                            v[m] = make_float2(bx.x + sv.x, bx.y + sv.y);
                        }
                    } else if (DSPEC && act == ACT_DELTA) {
#pragma unroll
                        for (int m = 0; m < 32; ++m) {
                            const long long gi = gb + 32 * m;
                            const float2 y = cconj(v[m]), b = __ldcg(p.B + gi);
                            const float2 d = __ldcg(p.delta + gi), xx = __ldcg(p.x + gi);
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
                            // one body for every action (kernels_pipe.cu k_xpass_pipe)
                            const long long gi = gb + 32 * m;
                            const float2 y = cconj(v[m]), b = __ldcg(p.B + gi);
                            const float2 a1 = need1 ? __ldcg(a1p + gi) : make_float2(0.f, 0.f);
                            const float2 xx = __ldcg(p.x + gi);
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
                }
                if (add_lines) {   // sparse source (R-31): FFT_x(B x + s) = FFT_x(B x) + FFT_x(s)
                    for (int q = 0; q < p.s_count; ++q) {
                        if (p.s_list[q] != (int)line) continue;
                        const float2 *cl = p.s_comp + (long long)q * N + j;
#pragma unroll
                        for (int m = 0; m < 32; ++m) {
                            const float2 a = cl[32 * m];
                            v[m] = make_float2(v[m].x + a.x, v[m].y + a.y);
                        }
                    }
                }
#pragma unroll
                for (int m = 0; m < 32; ++m) p.work[gb + 32 * m] = v[m];
                // this unit's residual partial: lanes in fp64, fixed shuffle tree, warps in order
                const double wsum = warp_sum_d((double)lacc);
                if (lane == 0) sh_part[warp] = wsum;
                __threadfence();   // the lines are published with the unit (release at gpu scope)
                __syncthreads();
                if (tid == 0) {
                    double s = 0.0;
#pragma unroll
                    for (int w = 0; w < PG::LPU; ++w) s += sh_part[w];
                    p.upart[u.z * PG::APP + u.idx] = s;
                    atomicAdd(p.a_done + u.z, 1u);
                }
            }
            cur = nxt;
        }
    }

    // last CTA: the residual over every A unit in a fixed order, the finish,
    // and the counters reset for the next launch
    __syncthreads();
    __shared__ int am_last;
    if (tid == 0) {
        __threadfence();
        am_last = atomicAdd(&p.st->counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    double s = 0.0;
    if (!xonly)
        for (long long i = tid; i < nz * PlaneGeo::APP; i += PlaneGeo::NT) s += __ldcg(p.upart + i);
    const double total = block_sum_d<PlaneGeo::NT>(s, sh_red);
    for (long long i = tid; i < nz; i += PlaneGeo::NT) {
        p.d_done[i] = 0u;
        p.a_done[i] = 0u;
    }
    if (tid == 0) {
        *p.ctr = 0ull;
        p.st->counter = 0u;
        if (p.st->err == 0) finish_xpass(false, xonly, total, p.st, p.red, act);
    }
}

template <bool LEAN, bool DSPEC, bool XSPEC>
static cudaError_t plane_t(const CUtensorMap &mapy, const PParams &p, int grid, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_plane<LEAN, DSPEC, XSPEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             PlaneGeo::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    return launch_pdl(k_plane<LEAN, DSPEC, XSPEC>, grid, PlaneGeo::NT, PlaneGeo::SMEM, s, mapy, p);
}

// instance by the form the host expects (as launch_xpass_pipe): lean
// (sparse-source x-form), dense x-form, Delta-form
cudaError_t launch_plane(const CUtensorMap &mapy, const PParams &p, int grid, cudaStream_t s, bool lean, bool expect_x) {
    if (lean) return plane_t<true, false, false>(mapy, p, grid, s);
    if (expect_x) return plane_t<false, false, true>(mapy, p, grid, s);
    return plane_t<false, true, false>(mapy, p, grid, s);
}

}  // namespace usp
