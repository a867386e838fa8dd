// zwrite.cu -- does the z pass's write side gain from wider rows?
// Out-of-place tile copies a -> b of a 1024^3 complex64 array (rows = planes,
// 8 MB apart).  Every CTA reads a tile of RW columns x 16384/RW rows and
// writes 128 KB back as WW columns x 16384/WW rows (the written tile is a
// different region of b when RW != WW -- the data is not a transpose, only
// the access pattern matters).  Plain 64-bit loads/stores, 512 threads, the
// k_stile thread layout (a warp covers 32/W rows of W columns).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zwrite zwrite.cu && ./zwrite
#include <cstdio>
#include <cuda_runtime.h>

constexpr long long NN = 1024, S = NN * NN;   // row pitch (elements)

template <int RW, int WW>
__global__ void __launch_bounds__(512, 1) k_copy(const float2 *__restrict__ a, float2 *__restrict__ b) {
    constexpr int RR = 16384 / RW, WR = 16384 / WW;      // rows per tile
    const long long ntiles = S / 16;                     // 128 KB tiles
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        // read tile: columns [RW * (t / (1024/RR))...] -- tile t covers RW columns x RR rows
        const long long rt_c = (t / (NN / RR)) * RW, rt_r = (t % (NN / RR)) * RR;
        const long long wt_c = (t / (NN / WR)) * WW, wt_r = (t % (NN / WR)) * WR;
        float2 v[32];
        {
            const int c = threadIdx.x % RW, j = threadIdx.x / RW;
            constexpr int step = 512 / RW;
            const float2 *p = a + rt_c + c + (rt_r + j) * S;
#pragma unroll
            for (int m = 0; m < 32; ++m) v[m] = __ldcs(p + (long long)m * step * S);
        }
        {
            const int c = threadIdx.x % WW, j = threadIdx.x / WW;
            constexpr int step = 512 / WW;
            float2 *p = b + wt_c + c + (wt_r + j) * S;
#pragma unroll
            for (int m = 0; m < 32; ++m) __stcs(p + (long long)m * step * S, v[m]);
        }
    }
}

template <int RW, int WW>
void run(const float2 *a, float2 *b, int nsm) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_copy<RW, WW><<<nsm, 512>>>(a, b);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    const double gb = 2.0 * S * NN * 8 / 1e9;
    printf("read %3d-col rows (%4d B), write %3d-col rows (%4d B): %.3f ms  %.0f GB/s  (%s)\n", RW, RW * 8, WW,
           WW * 8, best, gb / best * 1e3, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const size_t bytes = (size_t)S * NN * sizeof(float2);
    float2 *a, *b;
    if (cudaMalloc(&a, bytes) != cudaSuccess || cudaMalloc(&b, bytes) != cudaSuccess) {
        printf("malloc failed\n");
        return 1;
    }
    cudaMemset(a, 0, bytes);
    cudaMemset(b, 0, bytes);
    for (int rep = 0; rep < 2; ++rep) {
        run<16, 16>(a, b, nsm);
        run<16, 32>(a, b, nsm);
        run<16, 64>(a, b, nsm);
        run<32, 16>(a, b, nsm);
        run<32, 32>(a, b, nsm);
        run<64, 64>(a, b, nsm);
    }
    return 0;
}
