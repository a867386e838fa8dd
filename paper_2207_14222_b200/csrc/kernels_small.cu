// kernels_small.cu -- persistent 2-D solver for grids whose fields stay in L2
// (BASELINE.json config C2, 512^2: 2 MiB per field; SURVEY.md §7 hard part 8
// "latency-bound small configs ... use a persistent kernel").
//
// The 4-pass schedule launches 2 kernels per iteration; at 512^2 each is
// ~10 us of mostly launch/ramp latency for ~2 us of work.  k_solve2d runs
// the whole iteration loop of Algorithm 1 (Delta-form, reading R-17) inside
// one cooperative launch (all CTAs co-resident) with two grid barriers per
// iteration:
//   Y phase  y forward FFT, x g(p)/N (Eq. 12), y inverse, 16/32-column tiles
//   -- barrier --
//   X phase  x inverse FFT -> update x, Delta (L613) -> residual partial ->
//            u = B Delta -> x forward FFT
//   -- barrier --  every CTA sums the CTA partials in the same fixed order,
//            so all take the same stop decision (R-4, R-5) without a host
//            round trip; CTA 0 publishes the state and the residual history.
// The arithmetic per line is the same four-step FFT of fft_core.cuh as the
// pass kernels (register loads from L2 instead of TMA stages: the data is
// resident and the phases are short).
#include <cuda_runtime.h>
#include <cstdlib>
#include <math.h>
#include <stdint.h>

#include "fft_core.cuh"
#include "kcommon.cuh"
#include "tma.cuh"
#include "usp_internal.h"

namespace usp {

// Sense-reversing grid barrier over co-resident CTAs (cooperative launch).
// A 4-second watchdog turns a scheduling failure into an error code.
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acqrel_gpu(unsigned *p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// Sense-reversing grid barrier over co-resident CTAs (cooperative launch).
// Scoped acquire/release at gpu scope instead of full fences: the CTA
// barrier orders the CTA's writes before thread 0's release (cumulativity).
// A 4-second watchdog turns a scheduling failure into an error code.
__device__ __forceinline__ bool grid_barrier(unsigned *count, volatile unsigned *gen, IterState *st) {
    __syncthreads();
    __shared__ int ok;
    if (threadIdx.x == 0) {
        ok = 1;
        unsigned *genp = const_cast<unsigned *>(gen);
        const unsigned g = ld_acquire_gpu(genp);
        if (atom_add_acqrel_gpu(count, 1u) == gridDim.x - 1) {
            *count = 0u;   // ordered before the release below
            st_release_gpu(genp, g + 1u);
        } else {
            const uint64_t t0 = globaltimer_ns();
            unsigned n = 0;
            while (ld_acquire_gpu(genp) == g) {
                if ((++n & 255u) == 0 && globaltimer_ns() - t0 > 4000000000ull) {
                    if (atomicCAS(&st->err, 0, 10) == 0) st->err_info = blockIdx.x;
                    ok = 0;
                    break;
                }
            }
        }
    }
    __syncthreads();
    return ok != 0;
}

template <int NX, int NY, int NT_ = 256>
struct S2 {
    using GX = LineGeo<NX>;
    using GY = LineGeo<NY>;
    static constexpr int NT = NT_;
    // work is dealt per CTA: an x unit = LPC lines, a y unit = COLS columns.
    // (Dealing 32/N1-line warp units over every warp of 148 CTAs measured
    // slower at 512^2: 26 vs 22 us per iteration -- more CTAs at each grid
    // barrier, 16-byte column accesses.)
    static constexpr int LPC = NT / GX::N1;                  // x lines per CTA step
    static constexpr int XS = LPC * LayRow<NX>::kFloat2PerLine;
    static constexpr int COLS = NT / GY::N1;                 // y tile columns (16 or 32): all threads work
    // writer rows of the y exchange: pitch = 8 or 4 (mod 16) float2 keeps the
    // 16 lanes of a 64-bit phase on distinct banks for 8 / 4 columns
    static constexpr int YPAD = (COLS == 16 || COLS == 32) ? 0 : (COLS == 8 ? 8 : 4);
    static constexpr int YS = GY::N1 * (GY::N2 * COLS + YPAD);
    static constexpr int BUF = XS > YS ? XS : YS;
    // X phase: B, Delta, x of the CTA's lines prefetched into shared memory
    // (cp.async) before the inverse FFT, so the update does not wait on L2
    static constexpr int PFE = LPC * NX;                      // float2 per field
    static constexpr bool PF = (BUF + NX + NY + 3 * PFE) * 8 <= 200 * 1024;
    static constexpr int SMEM = (BUF + NX + NY + (PF ? 3 * PFE : 0)) * 8;
};

template <int NX, int NY, int NT>
__global__ void __launch_bounds__(NT, 1) k_solve2d(S2Params p) {
    using T = S2<NX, NY, NT>;
    using GX = typename T::GX;
    using GY = typename T::GY;
    extern __shared__ __align__(16) float2 smem2[];
    float2 *buf = smem2;
    float2 *twx = buf + T::BUF;
    float2 *twy = twx + NX;
    float2 *pf = twy + NY;   // PF: [B | Delta | x][lq][line element]
    __shared__ double sh_red[8];
    __shared__ int s_status;
    __shared__ long long s_k;
    IterState *st = p.st;

    for (int i = threadIdx.x; i < NX; i += blockDim.x) twx[i] = __ldg(&p.twx[i]);
    for (int i = threadIdx.x; i < NY; i += blockDim.x) twy[i] = __ldg(&p.twy[i]);
    __syncthreads();

    const float alpha = (float)st->alpha;
    const double tol = st->tol, n0 = st->n0;
    const long long kmax = st->kmax;
    long long k = st->k;
    int status = st->status;
    double r = st->r;
    int parity = 0;
    const int tid = threadIdx.x;

    while (k < kmax && (status == ST_RUNNING || status == ST_STOP_PENDING)) {
        const bool xonly = status == ST_STOP_PENDING;
        if (!xonly) {
            // ---------------------------------------------------- Y phase
            {
                const int c = tid % T::COLS, j = tid / T::COLS;
                const LayCol<NY, T::COLS, T::YPAD, 0> lay{buf, c};
                const int ntile = NX / T::COLS;
                for (int tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
                    const int col = tile * T::COLS + c;
                    float2 v[GY::N2];
#pragma unroll
                    for (int m = 0; m < GY::N2; ++m) v[m] = __ldcg(&p.work[(long long)(j + GY::N1 * m) * NX + col]);
                    const float px = p.mp.kx * freq_m(col, NX), pt2 = px * px;
#pragma unroll 1
                    for (int pass = 0; pass < 2; ++pass) {
                        fft_line<NY, false, LayCol<NY, T::COLS, T::YPAD, 0>, true>(v, lay, j, twy);
                        if (pass == 0) {
#pragma unroll
                            for (int m = 0; m < GY::N2; ++m) {
                                const float pl = p.mp.ky * freq_m(j + GY::N1 * m, NY);
                                v[m] = cconj(cmul(v[m], multiplier(p.mp, fmaf(pl, pl, pt2))));
                            }
                        }
                    }
#pragma unroll
                    for (int m = 0; m < GY::N2; ++m) p.work[(long long)(j + GY::N1 * m) * NX + col] = cconj(v[m]);
                }
            }
            if (!grid_barrier(p.bar_count, p.bar_gen, st)) return;
        }
        // -------------------------------------------------------- X phase
        double acc = 0.0;
        {
            const int lq = tid / GX::N1, j = tid % GX::N1;
            const LayRow<NX> lay{buf + lq * LayRow<NX>::kFloat2PerLine};
            const int ngroups = NY / T::LPC;
            for (int g = blockIdx.x; g < ngroups; g += gridDim.x) {
                const long long base = (long long)(g * T::LPC + lq) * NX + j;
                float2 v[GX::N2];
                if (xonly) {
#pragma unroll
                    for (int m = 0; m < GX::N2; ++m) {
                        const long long i = base + GX::N1 * m;
                        const float2 d = p.delta[i], xx = p.x[i];
                        p.x[i] = make_float2(fmaf(alpha, d.x, xx.x), fmaf(alpha, d.y, xx.y));
                    }
                    continue;
                }
                const int eb = lq * NX + j;   // this thread's elements in the PF block: eb + N1 m
                if constexpr (T::PF) {
#pragma unroll
                    for (int m = 0; m < GX::N2; ++m) {
                        const long long i = base + GX::N1 * m;
                        cp_async8(pf + eb + GX::N1 * m, p.B + i);
                        cp_async8(pf + T::PFE + eb + GX::N1 * m, p.delta + i);
                        cp_async8(pf + 2 * T::PFE + eb + GX::N1 * m, p.x + i);
                    }
                    cp_async_commit();
                }
#pragma unroll
                for (int m = 0; m < GX::N2; ++m) v[m] = cconj(__ldcg(&p.work[base + GX::N1 * m]));
                fft_line<NX, false, LayRow<NX>, true>(v, lay, j, twx);   // inverse via conj
                if constexpr (T::PF) cp_async_wait0();
                float lacc = 0.f;
#pragma unroll
                for (int m = 0; m < GX::N2; ++m) {
                    const long long i = base + GX::N1 * m;
                    float2 b, d, xx;
                    if constexpr (T::PF) {
                        b = pf[eb + GX::N1 * m];
                        d = pf[T::PFE + eb + GX::N1 * m];
                        xx = pf[2 * T::PFE + eb + GX::N1 * m];
                    } else {
                        b = p.B[i];
                        d = p.delta[i];
                        xx = p.x[i];
                    }
                    const float2 y = cconj(v[m]);
                    const float2 t = cmul(b, csub(y, d));
                    const float2 dn = make_float2(fmaf(alpha, t.x, d.x), fmaf(alpha, t.y, d.y));
                    p.x[i] = make_float2(fmaf(alpha, d.x, xx.x), fmaf(alpha, d.y, xx.y));
                    p.delta[i] = dn;
                    lacc += cabs2(dn);
                    v[m] = cmul(b, dn);
                }
                acc += (double)lacc;
                fft_line<NX, false, LayRow<NX>, true>(v, lay, j, twx);   // forward
#pragma unroll
                for (int m = 0; m < GX::N2; ++m) p.work[base + GX::N1 * m] = v[m];
            }
        }
        // residual: CTA partial -> barrier -> every CTA sums all partials in order
        const double mine = block_sum_d<NT>(acc, sh_red);
        double *part = p.partials + parity * gridDim.x;
        if (tid == 0) part[blockIdx.x] = mine;
        if (!grid_barrier(p.bar_count, p.bar_gen, st)) return;
        if (tid < 32) {
            // warp 0 sums the CTA partials: lane l takes partials l, l+32, ...
            // (loads in flight together), then a fixed shuffle tree -- the
            // same order in every CTA, so every CTA takes the same decision
            double total = 0.0;
            for (unsigned b = tid; b < gridDim.x; b += 32) total += __ldcg(&part[b]);
            total = warp_sum_d(total);
            if (tid == 0) {
            const long long k1 = k + 1;
            int stt = status;
            double rr = r;
            if (xonly) {
                stt = ST_DONE_CONV;
            } else {
                rr = sqrt(total) / n0;
                if (!(rr <= 1e6)) stt = ST_DIVERGED;
                else if (tol > 0.0 && rr < tol) stt = ST_STOP_PENDING;
                if (blockIdx.x == 0) p.red.hist[k1 % p.red.hist_cap] = rr;
            }
            s_status = stt;
            s_k = k1;
            sh_red[0] = rr;
            }
        }
        __syncthreads();
        status = s_status;
        k = s_k;
        r = sh_red[0];
        __syncthreads();
        parity ^= 1;
    }
    if (blockIdx.x == 0 && tid == 0) {
        st->k = k;
        st->r = r;
        st->status = status;
    }
}

// ========================================================= launchers ====
template <int NX, int NY, int NT>
static cudaError_t solve2d_t(const S2Params &p, int nsm, cudaStream_t s, int *grid_out) {
    using T = S2<NX, NY, NT>;
    static int grid = 0;
    if (!grid) {
        cudaError_t e = cudaFuncSetAttribute(k_solve2d<NX, NY, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             T::SMEM);
        if (e != cudaSuccess) return e;
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve2d<NX, NY, NT>, NT, T::SMEM);
        if (e != cudaSuccess) return e;
        if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
        // enough CTAs for the larger phase, at most one wave of co-resident CTAs
        const int work = (NY / T::LPC) > (NX / T::COLS) ? (NY / T::LPC) : (NX / T::COLS);
        grid = work < nsm * per_sm ? work : nsm * per_sm;
    }
    if (grid_out) *grid_out = grid;
    S2Params pp = p;
    void *args[] = {&pp};
    return cudaLaunchCooperativeKernel((const void *)k_solve2d<NX, NY, NT>, dim3(grid), dim3(NT), args, T::SMEM,
                                       s);
}

// CTA size 128: twice the CTAs of the 256-thread version, and the X phase's
// B, Delta, x fit the shared-memory prefetch.  C2 (512^2, 1680 iterations to
// 1e-6): 256 threads 35.9 ms, 128 threads 25.5 ms (15.2 us per iteration),
// 64 threads 25.6 ms.
template <int NX, int NY>
static cudaError_t solve2d_nt(const S2Params &p, int nsm, cudaStream_t s) {
    return solve2d_t<NX, NY, 128>(p, nsm, s, nullptr);
}

bool solve2d_supported(long long nx, long long ny) {
    auto ok = [](long long n) { return n >= 64 && n <= 512 && (n & (n - 1)) == 0; };
    return ok(nx) && ok(ny);
}

cudaError_t launch_solve2d(int nx, int ny, const S2Params &p, int nsm, cudaStream_t s) {
#define S2_Y(X, Y) \
    case Y: return solve2d_nt<X, Y>(p, nsm, s);
#define S2_X(X)                                                                  \
    case X:                                                                      \
        switch (ny) { S2_Y(X, 64) S2_Y(X, 128) S2_Y(X, 256) S2_Y(X, 512) default: return cudaErrorInvalidValue; }
    switch (nx) { S2_X(64) S2_X(128) S2_X(256) S2_X(512) default: return cudaErrorInvalidValue; }
#undef S2_X
#undef S2_Y
}

}  // namespace usp
