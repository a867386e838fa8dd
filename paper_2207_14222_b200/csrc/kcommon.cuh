// kcommon.cuh -- device helpers shared by the pass kernels: deterministic
// reductions, the last-CTA-done residual reduction, and the Fourier
// multiplier of (L+1)^-1 (Eq. 12).
#pragma once
#include <cuda_runtime.h>


#include "fft_core.cuh"
#include "usp_internal.h"

namespace usp {

// Launch with programmatic stream serialization (PDL, see tma.cuh
// pdl_trigger/pdl_wait): the next kernel's launch overlaps the tail of this
// one instead of following its completion.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), int grid, int block, int smem, cudaStream_t s,
                              const Args &...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// ------------------------------------------------------------ helpers --
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Fixed-order CTA reduction of one double per thread; result valid in tid 0.
template <int NT>
__device__ __forceinline__ double block_sum_d(double v, double *sh) {
    v = warp_sum_d(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NT / 32; ++i) s += sh[i];
    }
    __syncthreads();
    return s;
}

// Last-CTA-done reduction: every CTA contributes `mine` (valid in tid 0);
// returns true in the last CTA, where *total holds the fixed-order sum.
template <int NT>
__device__ __forceinline__ bool last_block_total(double mine, IterState *st, double *partials, double *sh,
                                 double *total) {
    __shared__ int am_last;
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = mine;
        __threadfence();
        const unsigned t = atomicAdd(&st->counter, 1u);
        am_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!am_last) return false;
    __threadfence();
    double s = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += NT) s += __ldcg(&partials[i]);
    s = block_sum_d<NT>(s, sh);
    if (threadIdx.x == 0) {
        *total = s;
        st->counter = 0u;
    }
    return true;
}

// Fourier multiplier g(p)/N_vox of (L+1)^-1 (Eq. 12, unified form R-1):
//   g = c / (D |p|^2 + sigma + c)
__device__ __forceinline__ float2 multiplier(const MulParams &mp, float p2) {
    const float dr = fmaf(mp.D, p2, mp.sc.x), di = mp.sc.y;
    const float inv = 1.0f / fmaf(dr, dr, di * di);
    return make_float2((mp.cn.x * dr + mp.cn.y * di) * inv, (mp.cn.y * dr - mp.cn.x * di) * inv);
}

__device__ __forceinline__ float freq_m(int k, int n) { return (float)(k < (n >> 1) ? k : k - n); }

// The x pass's action for this launch (read by every CTA before the last
// CTA's finish changes the state): the x-form state turns into the
// Delta-form once the last residual is below r_sw (reading R-30).
__device__ __forceinline__ int xform_act(const IterState *st) {
    const int f = st->form;
    if (f == FORM_X) return (st->r < st->r_sw) ? ACT_TO_DELTA : ACT_X;
    return f == FORM_PROBE ? ACT_PROBE : ACT_DELTA;
}

// Does an iteration launch run?  (RUNNING below kmax, or the end-of-call probe.)
__device__ __forceinline__ bool iter_running(const IterState *st) {
    return (st->status == ST_RUNNING && st->k < st->kmax) || (st->form == FORM_PROBE && st->status == ST_RUNNING);
}

// Thread 0 of the last CTA of an x pass: publish n0 (source setup) or
// the residual and the stop decision (iteration), see kernels.cu header.
//   ACT_DELTA     Delta-form: x_{k+1} done, r_{k+1} of Delta_{k+1}; below tol
//                 -> STOP_PENDING (the next pass applies x += alpha Delta_{k+1})
//   ACT_X         x-form: x_{k+1} done, r_k of the Delta_k it used; below tol
//                 -> converged (reading R-5)
//   ACT_TO_DELTA  Delta_k stored, x not updated, r_k; k unchanged; below tol
//                 -> STOP_PENDING, as the Delta-form
//   ACT_PROBE     as ACT_TO_DELTA but the state stays in the x-form and the
//                 status is left alone (an on-demand query of r_k)
__device__ __forceinline__ void finish_xpass(bool src_epi, bool xonly, double total, IterState *st,
                                             const Red &red, int act = ACT_DELTA) {
    if (src_epi) {
        const double n0 = sqrt(total);
        st->n0 = n0;
        st->r = (n0 > 0.0) ? 1.0 : 0.0;
        st->k = 0;
        st->status = (n0 > 0.0) ? ST_RUNNING : ST_DONE_CONV;
        st->form = st->xform ? FORM_X : FORM_DELTA;
        red.hist[0] = st->r;
        return;
    }
    const long long k = st->k;
    if (xonly) {                       // the final update x_{k+1} = x_k + alpha Delta_k
        st->k = k + 1;
        st->status = ST_DONE_CONV;
        return;
    }
    const double r = sqrt(total) / st->n0;
    st->r = r;
    long long hi = k;                  // index of the Delta whose norm this is
    if (act == ACT_DELTA || act == ACT_X) st->k = k + 1;
    if (act == ACT_DELTA) hi = k + 1;
    if (act == ACT_TO_DELTA) st->form = FORM_DELTA;
    if (act == ACT_PROBE) st->form = FORM_X;
    st->add_s = (act == ACT_X || act == ACT_PROBE) ? 1 : 0;   // sparse source: k_sadd adds s
    red.hist[hi % red.hist_cap] = r;
    if (!(r <= 1e6)) st->status = ST_DIVERGED;            // NaN, Inf or r > 1e6
    // (a probe only reports r_k: the x-form pass that follows decides the stop)
    else if (st->tol > 0.0 && r < st->tol && act != ACT_PROBE)
        st->status = (act == ACT_X) ? ST_DONE_CONV : ST_STOP_PENDING;
}

// Grid of a grid-stride kernel clamped to the CTAs resident at once: every
// CTA of a grid-stride loop gets the same work, so CTAs beyond one wave run
// as a second, partly empty wave (measured: the GMRES dot at 62 % of the copy
// peak with 3 of its 4 CTAs per SM resident).  K is the kernel itself, so the
// cached occupancy is per kernel instance.
template <auto K>
inline int resident_grid(int grid, int nt, size_t smem = 0) {
    static int cap = -1;
    if (cap < 0) {
        int dev = 0, nsm = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, K, nt, smem);
        cap = nsm * (per > 0 ? per : 1);
    }
    return grid < cap ? grid : cap;
}

}  // namespace usp
