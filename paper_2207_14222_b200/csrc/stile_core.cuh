// stile_core.cuh -- the strided-axis tile FFT shared by the strided passes
// (kernels_stile.cu) and the plane-chained pass (kernels_plane.cu): tile
// geometry, the four-step FFT of a 16-column tile (two-round exchange with
// DFT shift flips for N >= 512) and the register stores of a tile.
// See kernels_stile.cu for the layout and the flip identities.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fft_core.cuh"
#include "usp_internal.h"

namespace usp {

template <int N>
struct STile {
    using G = LineGeo<N>;
    // GROUPS independent thread groups per CTA, each with its own stage,
    // exchange buffer, mbarrier and named barrier.  Two groups of 8 columns at
    // N = 1024 (one computes while the other waits) measured 1.6x SLOWER than
    // one group of 16 columns (y 5.0 vs 3.1 ms, z 7.4 vs 4.6 ms: 64-byte TMA
    // rows), so one group of 16 columns (128-byte rows) is used.
    static constexpr int GROUPS = 1;
    // N = 2048 (N2 = 64 values per thread): 8 columns, so 256 threads keep
    // their 64 complex values in registers (64-byte rows; used for the
    // 2048-plane z pass of C5w and its slab decomposition)
    static constexpr int COLS = (GROUPS == 2 || N == 2048) ? 8 : 16;
    static constexpr int NTG = COLS * G::N1;                    // threads per group
    static constexpr int NT = GROUPS * NTG;
    static constexpr int TILE = COLS * N;                       // float2 per stage
    // two-round exchange only where a full buffer would not fit next to the stage
    static constexpr bool HALFX = (N >= 512);
    static constexpr bool FLIP = HALFX && G::R == 1;   // N1 == N2: halves chosen by shift flips
    static constexpr int XPAD = (COLS == 8) ? 8 : 0;   // 8-column rows: offset writer rows by 64 B (banks)
    static constexpr int XPITCH = (HALFX ? (G::N2 / 2) * COLS : G::N2 * COLS) + XPAD;   // float2 per writer row
    static constexpr int XB = G::N1 * XPITCH;
    static constexpr int GSM = TILE + XB;                       // float2 per group
    static constexpr int BOXN = N < 256 ? N : 256;
    static constexpr int SMEM = (GROUPS * GSM + N) * 8 + 16 * GROUPS;
    static constexpr int FIT_SMEM = 232448 / (SMEM + 1024);
    static constexpr int FIT_REGS = 65536 / (NT * 96);            // keep >= 96 registers per thread
    static constexpr int FIT_THR = 2048 / NT;
    static constexpr int MINB0 = FIT_SMEM < FIT_REGS ? FIT_SMEM : FIT_REGS;
    static constexpr int MINB1 = MINB0 < FIT_THR ? MINB0 : FIT_THR;
    static constexpr int MINB = MINB1 < 1 ? 1 : MINB1;
};

__device__ __forceinline__ int ilog2c(int n) { return 31 - __clz(n); }   // n a power of two

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// One forward four-step DFT of the thread's line (the shared body).
// v[n2] = x[j + N1 n2] on entry; v[m] = X[j + N1 m] on exit (up to the
// shift flips of HALFX, which the caller applies).
template <int N>
__device__ __forceinline__ void gsync(int bar) {   // the calling thread group (named barrier)
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(STile<N>::NTG) : "memory");
}

template <int N>
__device__ __forceinline__ void stile_fft(float2 (&v)[LineGeo<N>::N2], float2 *xb, const float2 *sm_tw, int c,
                                          int j, int bar) {
    using G = LineGeo<N>;
    using T = STile<N>;
    dft<G::N2, false>(v);
    if constexpr (T::FLIP) {
        constexpr int H = G::N2 / 2;
        const int b = (j >> (ilog2(G::N1) - 1)) & 1;
        // slot s holds k2 = s ^ (H b): twiddle W_N^(j k2)
        const float2 *tw0 = sm_tw + (H * b) * G::N1 + j;
        const float2 *tw1 = sm_tw + (H * (1 - b)) * G::N1 + j;
#pragma unroll
        for (int s = 0; s < G::N2; ++s) {
            const float2 w = (s < H) ? tw0[s * G::N1] : tw1[(s - H) * G::N1];
            v[s] = cmul(v[s], w);
        }
        float2 *wb = xb + j * T::XPITCH + c;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
#pragma unroll
            for (int q = 0; q < H; ++q) wb[q * T::COLS] = v[r * H + q];
            gsync<N>(bar);
            const float2 *rb = xb + (H * (r ^ b)) * T::XPITCH + (j & (H - 1)) * T::COLS + c;
#pragma unroll
            for (int q = 0; q < H; ++q) v[r * H + q] = rb[q * T::XPITCH];
            gsync<N>(bar);
        }
        dft<G::N1, false>(v);
    } else if constexpr (T::HALFX) {
        // N2 = 2 N1: round t moves the k2-half t; thread j reads k2 = j + N1 t
#pragma unroll
        for (int k2 = 1; k2 < G::N2; ++k2) v[k2] = cmul(v[k2], sm_tw[k2 * G::N1 + j]);
        float2 *wb = xb + j * T::XPITCH + c;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
#pragma unroll
            for (int q = 0; q < G::N1; ++q) wb[q * T::COLS] = v[t * G::N1 + q];
            gsync<N>(bar);
#pragma unroll
            for (int n1 = 0; n1 < G::N1; ++n1) v[t * G::N1 + n1] = xb[n1 * T::XPITCH + j * T::COLS + c];
            gsync<N>(bar);
        }
#pragma unroll
        for (int t = 0; t < 2; ++t) dft<G::N1, false>(v + t * G::N1);
        float2 o[G::N2];
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int k1 = 0; k1 < G::N1; ++k1) o[t + 2 * k1] = v[t * G::N1 + k1];
#pragma unroll
        for (int m = 0; m < G::N2; ++m) v[m] = o[m];
    } else {
#pragma unroll
        for (int k2 = 1; k2 < G::N2; ++k2) v[k2] = cmul(v[k2], sm_tw[k2 * G::N1 + j]);
        float2 *wb = xb + j * T::XPITCH + c;
#pragma unroll
        for (int k2 = 0; k2 < G::N2; ++k2) wb[k2 * T::COLS] = v[k2];
        gsync<N>(bar);
#pragma unroll
        for (int t = 0; t < G::R; ++t)
#pragma unroll
            for (int n1 = 0; n1 < G::N1; ++n1)
                v[t * G::N1 + n1] = xb[n1 * T::XPITCH + (j + G::N1 * t) * T::COLS + c];
        gsync<N>(bar);
#pragma unroll
        for (int t = 0; t < G::R; ++t) dft<G::N1, false>(v + t * G::N1);
        if constexpr (G::R > 1) {
            float2 o[G::N2];
#pragma unroll
            for (int t = 0; t < G::R; ++t)
#pragma unroll
                for (int k1 = 0; k1 < G::N1; ++k1) o[t + G::R * k1] = v[t * G::N1 + k1];
#pragma unroll
            for (int m = 0; m < G::N2; ++m) v[m] = o[m];
        }
    }
}

// Stores from registers: 64-bit stores, except the inverse y pass (K_D),
// where adjacent-column lanes pair up into 128-bit stores.  Measured at
// 1024^3 (medians of 5, one process): K_D 3.30 -> 2.77 ms with paired
// stores, while K_B (2.67 -> 2.82) and K_C (4.45 -> 4.51) are faster with
// 64-bit stores.
// Store register slots m in [M0, M1) (rows j + N1 m of column c) of a tile.
// Paired stores: adjacent-column lane pairs swap one value per slot pair with
// a shuffle so each lane writes two columns of one row with one 128-bit store
// (half the store instructions).  base = &dst[row 0][column c].
template <int N, int MODE, int M0, int M1>
__device__ __forceinline__ void store_slots(const float2 (&v)[LineGeo<N>::N2], float2 *base, long long stride,
                                            int j, int c) {
    using G = LineGeo<N>;
    auto val = [&](int m) { return (MODE == S_FWD) ? v[m] : cconj(v[m]); };
    constexpr bool paired = MODE == S_INV;
    if constexpr (paired && STile<N>::COLS == 16 && ((M1 - M0) % 2) == 0) {
        const bool odd = c & 1;
        float2 *b = base - (odd ? 1 : 0) + (long long)(j + (odd ? G::N1 : 0)) * stride;
        const long long step = 2LL * G::N1 * stride;
#pragma unroll
        for (int m = M0; m < M1; m += 2) {
            const float2 a0 = val(m), a1 = val(m + 1);
            const float2 send = odd ? a0 : a1, keep = odd ? a1 : a0;
            const float2 recv = make_float2(__shfl_xor_sync(0xffffffffu, send.x, 1),
                                            __shfl_xor_sync(0xffffffffu, send.y, 1));
            const float4 o4 = odd ? make_float4(recv.x, recv.y, keep.x, keep.y)
                                  : make_float4(keep.x, keep.y, recv.x, recv.y);
            *reinterpret_cast<float4 *>(b + (long long)((m - M0) / 2) * step + (long long)M0 * G::N1 * stride) = o4;
        }
    } else {
        float2 *sb = base + (long long)(j + G::N1 * M0) * stride;
        const long long step = (long long)G::N1 * stride;
#pragma unroll
        for (int m = M0; m < M1; ++m) {
            sb[0] = val(m);
            sb += step;
        }
    }
}

}  // namespace usp
