// zstride.cu -- DRAM efficiency of the strided-pass tile pattern vs the row stride.
// Each CTA walks tiles of 16 complex64 columns x 1024 rows (128-byte rows,
// stride S elements between rows), loads a tile into registers (plain
// 64-bit loads, 512 threads x 32 values, the k_stile thread layout) and
// writes it back in place.  Reports GB/s (read + write) for several S.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zstride zstride.cu && ./zstride
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) k_tiles(float2 *a, long long S, long long ncols, long long nouter,
                                                   long long ostride) {
    const int c = threadIdx.x % 16, j = threadIdx.x / 16;
    const long long tpo = ncols / 16, ntiles = tpo * nouter;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const long long o = t / tpo, col = (t - o * tpo) * 16 + c;
        float2 *p = a + o * ostride + col + (long long)j * S;
        float2 v[32];
#pragma unroll
        for (int m = 0; m < 32; ++m) v[m] = __ldcg(p + (long long)m * 32 * S);
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 32; ++m) p[(long long)m * 32 * S] = make_float2(v[m].x * 1.0001f, v[m].y);
    }
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const long long n = 1024;
    struct Case { const char *name; long long S, ncols, nouter, ostride, pad; };
    // z pass: rows = planes (stride = plane pitch), columns = the plane's n*n elements
    // y pass: rows = y (stride = n), columns = x, outer = planes
    Case cases[] = {
        {"z  S=n^2        ", n * n, n * n, 1, 0, 0},
        {"z  S=n^2+16     ", n * n + 16, n * n, 1, 0, 16},
        {"z  S=n^2+64     ", n * n + 64, n * n, 1, 0, 64},
        {"z  S=n^2+512    ", n * n + 512, n * n, 1, 0, 512},
        {"z  S=n^2+4096   ", n * n + 4096, n * n, 1, 0, 4096},
        {"z' S=16K, 64 x [1024][16K] (128 KB rows pitch)", 16384, 16384, 64, 1024 * 16384, 0},
        {"z' S=128K, 8 x [1024][128K] (1 MB pitch)", 131072, 131072, 8, 1024 * 131072, 0},
        {"y  S=n          ", n, n, n, n * n, 0},
        {"y  S=n, planes+512", n, n, n, n * n + 512, 512},
    };
    const size_t bytes = (size_t)(n * n + 4096) * n * sizeof(float2) + 4096 * 8;
    float2 *a;
    if (cudaMalloc(&a, bytes) != cudaSuccess) { printf("malloc failed\n"); return 1; }
    cudaMemset(a, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (const Case &cs : cases) {
        float best = 1e9f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            k_tiles<<<nsm, 512>>>(a, cs.S, cs.ncols, cs.nouter, cs.ostride);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r > 0 && ms < best) best = ms;
        }
        const double gb = 2.0 * n * n * n * 8 / 1e9;
        printf("%s  %.3f ms  %.0f GB/s  (%s)\n", cs.name, best, gb / best * 1e3, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
