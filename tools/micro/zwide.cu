// zwide.cu -- is the z pass limited by the number of distinct rows (pages)
// a tile touches?  Same bytes per tile (128 KB), different shapes on the
// z-stride pattern (rows 8 MB apart): W columns x (16384/W) rows, W = 16,
// 32, 64, 128.  In-place read + write with plain 64-bit loads/stores,
// 512 threads x 32 values.  GB/s = 2 x 8 GiB / time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zwide zwide.cu && ./zwide
#include <cstdio>
#include <cuda_runtime.h>

template <int W>
__global__ void __launch_bounds__(512, 1) k_tiles(float2 *a, long long n) {
    constexpr int J = 512 / W;          // row groups per tile pass
    constexpr int H = 32 * J;           // rows per tile
    const int c = threadIdx.x % W, j = threadIdx.x / W;
    const long long S = n * n;          // row stride (plane pitch)
    const long long cblocks = S / W, rblocks = n / H;
    const long long ntiles = cblocks * rblocks;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const long long cb = t / rblocks, rb = t - cb * rblocks;
        float2 *p = a + cb * W + c + (rb * H + j) * S;
        float2 v[32];
#pragma unroll
        for (int m = 0; m < 32; ++m) v[m] = __ldcg(p + (long long)m * J * S);
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 32; ++m) p[(long long)m * J * S] = make_float2(v[m].x * 1.0001f, v[m].y);
    }
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const long long n = 1024;
    const size_t bytes = (size_t)n * n * n * sizeof(float2);
    float2 *a;
    if (cudaMalloc(&a, bytes) != cudaSuccess) { printf("malloc failed\n"); return 1; }
    cudaMemset(a, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep)
        for (int w = 16; w <= 128; w *= 2) {
            float best = 1e9f;
            for (int r = 0; r < 5; ++r) {
                cudaEventRecord(e0);
                if (w == 16) k_tiles<16><<<nsm, 512>>>(a, n);
                if (w == 32) k_tiles<32><<<nsm, 512>>>(a, n);
                if (w == 64) k_tiles<64><<<nsm, 512>>>(a, n);
                if (w == 128) k_tiles<128><<<nsm, 512>>>(a, n);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (r > 0 && ms < best) best = ms;
            }
            const double gb = 2.0 * n * n * n * 8 / 1e9;
            printf("W=%3d cols x %4d rows  %.3f ms  %.0f GB/s  (%s)\n", w, 16384 / w, best, gb / best * 1e3,
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
