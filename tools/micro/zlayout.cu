// zlayout.cu -- does the z pass pay for 8 MB-strided LOADS or STORES?
// Tiles of 16 complex64 columns x 1024 rows move from src to dst (out of
// place).  Row stride and tile offset are chosen per side, so each case
// names where the 8 MB (plane-pitch) stride sits:
//   nat->nat : z pass on the natural [z][y][x] layout (loads and stores 8 MB apart)
//   T->T     : both sides in [y][z][x] (rows 8 KB apart, the y-pass pattern)
//   nat->T   : loads 8 MB apart, stores 8 KB apart
//   T->nat   : loads 8 KB apart, stores 8 MB apart
// Plain 64-bit loads/stores, 512 threads x 32 values (the k_stile layout).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zlayout zlayout.cu && ./zlayout
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) k_move(const float2 *__restrict__ src, float2 *__restrict__ dst,
                                                  long long ls, long long lo, long long ss, long long so,
                                                  long long n) {
    const int c = threadIdx.x % 16, j = threadIdx.x / 16;
    const long long tpo = n / 16, ntiles = tpo * n;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const long long o = t / tpo, col = (t - o * tpo) * 16 + c;
        const float2 *p = src + o * lo + col + (long long)j * ls;
        float2 v[32];
#pragma unroll
        for (int m = 0; m < 32; ++m) v[m] = __ldcg(p + (long long)m * 32 * ls);
        float2 *q = dst + o * so + col + (long long)j * ss;
#pragma unroll
        for (int m = 0; m < 32; ++m) q[(long long)m * 32 * ss] = make_float2(v[m].x * 1.0001f, v[m].y);
    }
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const long long n = 1024, n2 = n * n;
    struct Case { const char *name; long long ls, lo, ss, so; };
    Case cases[] = {
        {"nat->nat (z in, z out)   ", n2, n, n2, n},
        {"T->T     (8KB in, 8KB out)", n, n2, n, n2},
        {"nat->T   (z in, 8KB out) ", n2, n, n, n2},
        {"T->nat   (8KB in, z out) ", n, n2, n2, n},
    };
    const size_t bytes = (size_t)n2 * n * sizeof(float2);
    float2 *a, *b;
    if (cudaMalloc(&a, bytes) != cudaSuccess || cudaMalloc(&b, bytes) != cudaSuccess) {
        printf("malloc failed\n");
        return 1;
    }
    cudaMemset(a, 0, bytes);
    cudaMemset(b, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep)
        for (const Case &cs : cases) {
            float best = 1e9f;
            for (int r = 0; r < 5; ++r) {
                cudaEventRecord(e0);
                k_move<<<nsm, 512>>>(a, b, cs.ls, cs.lo, cs.ss, cs.so, n);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (r > 0 && ms < best) best = ms;
            }
            const double gb = 2.0 * n * n * n * 8 / 1e9;
            printf("%s  %.3f ms  %.0f GB/s  (%s)\n", cs.name, best, gb / best * 1e3,
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
