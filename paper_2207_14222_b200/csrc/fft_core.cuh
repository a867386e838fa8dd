// fft_core.cuh -- register/shared-memory FFT building blocks for sm_100a.
//
// The method's F ("the Fourier transform over all spatial
// dimensions") is applied one axis at a time.  A line of length N = N1*N2 is
// held by N1 threads, N2 complex64 values each, and transformed with the
// four-step (Bailey / "six-step") factorisation:
//
//   thread j holds x[j + N1*n2], n2 = 0..N2-1
//   1. DFT_N2 over n2 in registers                -> Y[j][k2]
//   2. twiddle   Y[j][k2] *= W_N^(j*k2)           (fp64-built, fp32-rounded table)
//   3. one shared-memory exchange (transpose)     -> thread j gets k2 = j + N1*t
//   4. DFT_N1 over n1 in registers                -> X[k2 + N2*k1]
//
// so the thread ends up holding X at positions j + N1*m (m = t + R*k1): the
// same "lane j, stride N1" pattern it started from.  Loads and stores of a
// warp therefore touch contiguous runs (x axis) or full 128-byte rows of a
// 16-column tile (strided axes), and epilogues/prologues fuse in registers.
// Exactly one smem round trip per 1-D transform.
//
// Twiddles: in-register DFT constants come from tw64.h (float64 -> float32
// correctly rounded); the inter-step table is built on the host in float64.
// No fast-math (hard part 2: ~1e-6-accurate twiddles push the
// 512^2 parity error to 2.4e-4 > 1e-4).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "tw64.h"

namespace usp {

__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n >> 1); }

__host__ __device__ __forceinline__ constexpr int bitrev(int i, int bits) {
    int r = 0;
    for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
    return r;
}

template <int N>
struct LineGeo {
    static constexpr int LOG = ilog2(N);
    static constexpr int N1 = 1 << (LOG / 2);  // threads per line
    static constexpr int N2 = N / N1;          // values per thread (N2 >= N1)
    static constexpr int R = N2 / N1;          // 1 or 2
    static_assert(N1 * N2 == N && (N & (N - 1)) == 0, "power of two");
};

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
// a * b
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float cabs2(float2 a) { return fmaf(a.x, a.x, a.y * a.y); }

// a * W_64^E (forward, W = exp(-2 pi i/64)) or a * conj(W_64^E) (inverse);
// E is a template constant so quarter turns cost nothing and the constants
// become immediates.
template <bool INV, int E>
__device__ __forceinline__ float2 mul_w64(float2 a) {
    constexpr int e = E & 63;
    if constexpr (e == 0) {
        return a;
    } else if constexpr (e == 16) {
        return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
    } else if constexpr (e == 32) {
        return make_float2(-a.x, -a.y);
    } else if constexpr (e == 48) {
        return INV ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x);
    } else {
        constexpr float wr = kW64re[e];
        constexpr float wi = INV ? -kW64im[e] : kW64im[e];
        return make_float2(fmaf(a.x, wr, -a.y * wi), fmaf(a.x, wi, a.y * wr));
    }
}

template <int I, int BITS>
struct BitRev {
    static constexpr int value = bitrev(I, BITS);
};

template <bool INV, int LEN, int I, int J>
__device__ __forceinline__ void butterfly(float2 *t) {
    constexpr int H = LEN / 2;
    constexpr int e = (J * (64 / LEN)) & 63;
    const float2 a = t[I];
    if constexpr (e == 0 || e == 16 || e == 32 || e == 48) {
        const float2 b = mul_w64<INV, e>(t[I + H]);   // free: quarter turns
        t[I] = cadd(a, b);
        t[I + H] = csub(a, b);
    } else {
        // a + b w with two FMA chains, then a - b w = 2a - (a + b w):
        // 6 instructions instead of 8 (cmul + 4 adds)
        constexpr float wr = kW64re[e];
        constexpr float wi = INV ? -kW64im[e] : kW64im[e];
        const float2 b = t[I + H];
        const float2 s = make_float2(fmaf(b.x, wr, fmaf(-b.y, wi, a.x)), fmaf(b.x, wi, fmaf(b.y, wr, a.y)));
        t[I] = s;
        t[I + H] = make_float2(fmaf(2.f, a.x, -s.x), fmaf(2.f, a.y, -s.y));
    }
}

template <bool INV, int LEN, int... B>
__device__ __forceinline__ void dft_stage(float2 *t, std::integer_sequence<int, B...>) {
    (butterfly<INV, LEN, (B / (LEN / 2)) * LEN + (B % (LEN / 2)), B % (LEN / 2)>(t), ...);
}

template <int N, bool INV, int LEN>
__device__ __forceinline__ void dft_stages(float2 *t) {
    if constexpr (LEN <= N) {
        dft_stage<INV, LEN>(t, std::make_integer_sequence<int, N / 2>{});
        dft_stages<N, INV, LEN * 2>(t);
    }
}

template <int N, int... I>
__device__ __forceinline__ void load_bitrev(float2 *t, const float2 *v, std::integer_sequence<int, I...>) {
    ((t[I] = v[BitRev<I, ilog2(N)>::value]), ...);
}

// In-register DFT of length N <= 64 (radix-2 decimation in time, fully
// expanded at compile time; the bit reversal is a register renaming).
// Natural order in and out.
template <int N, bool INV>
__device__ __forceinline__ void dft(float2 *v) {
    if constexpr (N > 1) {
        static_assert(N <= 64, "register DFT up to 64 points");
        float2 t[N];
        load_bitrev<N>(t, v, std::make_integer_sequence<int, N>{});
        dft_stages<N, INV, 2>(t);
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] = t[i];
    }
}

__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }

// Copy the N-entry four-step twiddle table into shared memory (all threads).
template <int N>
__device__ __forceinline__ void load_twiddles(float2 *sm_tw, const float2 *__restrict__ tw) {
    for (int i = threadIdx.x; i < N; i += blockDim.x) sm_tw[i] = __ldg(&tw[i]);
}

// Shared-memory layouts for the exchange step.  A layout maps (n1, k2) of
// the calling thread's line to a float2 offset and knows which threads share
// the line (sync()).
// Contiguous lines (x axis): one buffer per line, rows n1 padded to N2+1
// float2 (odd stride: conflict-free 64-bit phases of 16 lanes); the line
// lives inside one warp, so __syncwarp orders the exchange.
template <int N>
struct LayRow {
    float2 *base;  // this line's buffer: N1*(N2+1) float2
    __device__ __forceinline__ int off(int n1, int k2) const { return n1 * (LineGeo<N>::N2 + 1) + k2; }
    __device__ __forceinline__ void sync() const { __syncwarp(); }
    static constexpr int kFloat2PerLine = LineGeo<N>::N1 * (LineGeo<N>::N2 + 1);
};
// Strided lines (y, z axes): COLS columns interleaved innermost, so the 16
// lanes of a 64-bit phase hit consecutive float2; PAD float2 per n1 row keep
// two rows of an 8-column tile on different banks.  BAR = 0: the whole CTA
// shares the tile (__syncthreads); BAR = NT > 0: named barrier 1 over NT
// consumer threads.
template <int N, int COLS, int PAD, int BAR>
struct LayCol {
    float2 *base;
    int c;
    __device__ __forceinline__ int off(int n1, int k2) const {
        return n1 * (LineGeo<N>::N2 * COLS + PAD) + k2 * COLS + c;
    }
    __device__ __forceinline__ void sync() const {
        if constexpr (BAR == 0) __syncthreads();
        else asm volatile("bar.sync 1, %0;" ::"n"(BAR) : "memory");
    }
    static constexpr int kFloat2 = LineGeo<N>::N1 * (LineGeo<N>::N2 * COLS + PAD);
};

// Four-step FFT of one line.  On entry v[n2] = x[j + N1*n2]; on exit
// v[m] = X[j + N1*m] (unnormalised DFT, sign - for forward, + for INV).
// tw[k2*N1 + j] = W_N^(j*k2) (forward); the inverse uses its conjugate.
// TWS: the twiddle table lives in shared memory (plain loads) instead of
// global memory (read-only path).
template <int N, bool INV, class Lay, bool TWS = false>
__device__ __forceinline__ void fft_line(float2 (&v)[LineGeo<N>::N2], const Lay &lay, int j,
                                         const float2 *__restrict__ tw) {
    using G = LineGeo<N>;
    dft<G::N2, INV>(v);
#pragma unroll
    for (int k2 = 1; k2 < G::N2; ++k2) {
        const float2 w = TWS ? tw[k2 * G::N1 + j] : __ldg(&tw[k2 * G::N1 + j]);
        v[k2] = INV ? cmulc(v[k2], w) : cmul(v[k2], w);
    }
#pragma unroll
    for (int k2 = 0; k2 < G::N2; ++k2) lay.base[lay.off(j, k2)] = v[k2];
    lay.sync();
#pragma unroll
    for (int t = 0; t < G::R; ++t)
#pragma unroll
        for (int n1 = 0; n1 < G::N1; ++n1) v[t * G::N1 + n1] = lay.base[lay.off(n1, j + G::N1 * t)];
    lay.sync();
#pragma unroll
    for (int t = 0; t < G::R; ++t) dft<G::N1, INV>(v + t * G::N1);
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

}  // namespace usp
