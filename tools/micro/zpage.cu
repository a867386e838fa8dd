// zpage.cu -- is the z pass's strided-tile loss address translation?
// Same tile walk as zstride.cu (16 complex64 columns x 1024 rows, rows one
// 8 MB plane apart, plain 64-bit loads and in-place stores, 512 threads x 32
// values per tile), on memory obtained four ways:
//   cudaMalloc                     (what torch's caching allocator returns)
//   cuMemCreate, one 8 GiB chunk   (VMM, single physical allocation)
//   cuMemCreate, 2 MiB chunks      (VMM, one physical allocation per 2 MiB:
//                                   the driver cannot back it with pages > 2 MiB)
//   cudaMallocAsync from a pool    (stream-ordered allocator)
// plus the y pattern (rows 8 KB apart) on the first as the reference.  If the
// one-chunk VMM mapping is faster than the 2 MiB-chunk mapping on the z
// pattern, page size (TLB reach) is what costs; if all four agree, it is not.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zpage zpage.cu -lcuda && ./zpage
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <vector>

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

static const long long n = 1024;
static int nsm = 0;

static void run(const char *name, float2 *a, bool zpat) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int r = 0; r < 6; ++r) {
        cudaEventRecord(e0);
        if (zpat) k_tiles<<<nsm, 512>>>(a, n * n, n * n, 1, 0);
        else k_tiles<<<nsm, 512>>>(a, n, n, n, n * n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    const double gb = 2.0 * n * n * n * 8 / 1e9;
    printf("%-44s %s  %.3f ms  %.0f GB/s  (%s)\n", name, zpat ? "z" : "y", best, gb / best * 1e3,
           cudaGetErrorString(cudaGetLastError()));
}

#define CK(x)                                                                          \
    do {                                                                               \
        CUresult rr = (x);                                                             \
        if (rr != CUDA_SUCCESS) { printf("%s failed: %d\n", #x, (int)rr); return 1; } \
    } while (0)

int main() {
    cudaFree(0);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const size_t bytes = (size_t)n * n * n * sizeof(float2);   // 8 GiB

    {   // cudaMalloc
        float2 *a;
        if (cudaMalloc(&a, bytes) != cudaSuccess) { printf("cudaMalloc failed\n"); return 1; }
        cudaMemset(a, 0, bytes);
        run("cudaMalloc", a, false);
        run("cudaMalloc", a, true);
        cudaFree(a);
    }
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = 0;
    size_t gmin = 0, grec = 0;
    CK(cuMemGetAllocationGranularity(&gmin, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
    CK(cuMemGetAllocationGranularity(&grec, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    printf("VMM granularity: minimum %zu, recommended %zu\n", gmin, grec);
    CUmemAccessDesc acc = {};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    for (size_t chunk : {bytes, (size_t)(512u << 20), (size_t)(2u << 20)}) {
        CUdeviceptr va;
        const size_t align = chunk < (size_t)(1u << 30) ? chunk : (size_t)(1u << 30);
        CK(cuMemAddressReserve(&va, bytes, align, 0, 0));
        std::vector<CUmemGenericAllocationHandle> hs;
        for (size_t off = 0; off < bytes; off += chunk) {
            CUmemGenericAllocationHandle h;
            CK(cuMemCreate(&h, chunk, &prop, 0));
            CK(cuMemMap(va + off, chunk, 0, h, 0));
            hs.push_back(h);
        }
        CK(cuMemSetAccess(va, bytes, &acc, 1));
        cudaMemset((void *)va, 0, bytes);
        char name[96];
        snprintf(name, sizeof name, "cuMemCreate, %zu MiB chunks", chunk >> 20);
        run(name, (float2 *)va, false);
        run(name, (float2 *)va, true);
        CK(cuMemUnmap(va, bytes));
        for (auto h : hs) CK(cuMemRelease(h));
        CK(cuMemAddressFree(va, bytes));
    }
    {   // stream-ordered pool
        float2 *a;
        if (cudaMallocAsync((void **)&a, bytes, 0) != cudaSuccess) { printf("cudaMallocAsync failed\n"); return 1; }
        cudaMemsetAsync(a, 0, bytes, 0);
        cudaDeviceSynchronize();
        run("cudaMallocAsync", a, true);
        cudaFreeAsync(a, 0);
        cudaDeviceSynchronize();
    }
    return 0;
}
