// zgroups.cu -- K_C's structure (16-column x 1024-row z tiles, rows 8 MB
// apart, TMA {16, 256} boxes into one 128 KB stage, next tile prefetched once
// the stage is copied to registers) with K_C-sized synthetic arithmetic:
// per tile two "FFTs" = FMA block, two-round shared-memory exchange, FMA
// block, and a multiplier block between them (~1900 FMAs per thread).
//   A  one group of 16 warps (thread (c, j) = tid % 16, tid / 16): every
//      exchange round syncs the whole CTA (K_C today)
//   B  two groups of 8 warps on 8 columns each (shared 16-column stage), each
//      exchange syncs only its group (named barrier), the stage is released
//      by whichever group copies it last -- groups drift apart, so one
//      group's FMA blocks can overlap the other's exchanges
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zgroups zgroups.cu -lcuda && ./zgroups
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t par) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok)
                     : "r"(smem_u32(b)), "r"(par)
                     : "memory");
}
__device__ __forceinline__ void tma2d(void *dst, const CUtensorMap *m, int c0, int c1, uint64_t *b) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(smem_u32(b))
        : "memory");
}
__device__ __forceinline__ void tma2d_store(const CUtensorMap *m, int c0, int c1, const void *src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"((uint64_t)m),
                 "r"(c0), "r"(c1), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa(const void *p, uint32_t rank) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
    return a;
}
__device__ __forceinline__ float2 ld_dsmem(uint32_t a) {
    float2 v;
    asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void st_dsmem(uint32_t a, float2 v) {
    asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}


constexpr long long NN = 1024;
constexpr int NT = 512;

__device__ __forceinline__ void nbar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int R>
__device__ __forceinline__ void fma_block(float2 (&v)[32], float f) {
    for (int r = 0; r < R; ++r) {
#pragma unroll
        for (int m = 0; m < 32; ++m) v[m] = make_float2(fmaf(v[m].x, f, v[m ^ 1].y), fmaf(v[m].y, f, -v[m ^ 2].x));
    }
}

// GROUPS = 1: cols per group 16, 512 threads per group; GROUPS = 2: 8 columns, 256 threads
template <int GROUPS, int R>
__global__ void __launch_bounds__(NT, 1) k_g(const __grid_constant__ CUtensorMap map, float2 *data, float f) {
    constexpr int GC = 16 / GROUPS;            // columns per group
    constexpr int GT = NT / GROUPS;            // threads per group
    constexpr int XP = 16 * GC + (GC == 8 ? 8 : 0);   // exchange row pitch (float2)
    constexpr int XBG = 32 * XP;               // exchange floats per group (half exchange: 16 slots x 32 rows)
    extern __shared__ __align__(128) unsigned char sm[];
    float2 *stage = (float2 *)sm;
    float2 *xb = stage + 16 * NN + (threadIdx.x / GT) * XBG;
    uint64_t *full = (uint64_t *)(stage + 16 * NN + GROUPS * XBG);
    unsigned *taken = (unsigned *)(full + 1);
    const int g = threadIdx.x / GT, tl = threadIdx.x % GT;
    const int cl = tl % GC, j = tl / GC, c = g * GC + cl;
    const int bar = 1 + g;
    const long long ntiles = NN * NN / 16;
    const long long t0 = blockIdx.x, tstep = gridDim.x;
    const int nloc = (int)((ntiles - t0 + tstep - 1) / tstep);
    auto issue = [&](int i) {
        const long long t = t0 + (long long)i * tstep;
        mbar_expect(full, 16 * NN * 8);
        for (int b = 0; b < 4; ++b) tma2d(stage + b * 256 * 16, &map, (int)(t * 16), b * 256, full);
    };
    if (threadIdx.x == 0) {
        mbar_init(full, 1);
        *taken = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (nloc > 0) issue(0);
    }
    __syncthreads();
    for (int i = 0; i < nloc; ++i) {
        mbar_wait(full, i & 1);
        float2 v[32];
#pragma unroll
        for (int m = 0; m < 32; ++m) v[m] = stage[(j + 32 * m) * 16 + c];
        fence_async();
        nbar(bar, GT);
        if (tl == 0) {   // the group that copies last releases the stage
            if (GROUPS == 1 || atomicAdd(taken, 1u) % GROUPS == GROUPS - 1)
                if (i + 1 < nloc) issue(i + 1);
        }
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
            fma_block<R>(v, f);
#pragma unroll
            for (int r = 0; r < 2; ++r) {   // two-round exchange (half buffer)
                float2 *wb = xb + j * XP + cl;
#pragma unroll
                for (int q = 0; q < 16; ++q) wb[q * GC] = v[r * 16 + q];
                nbar(bar, GT);
                const float2 *rb = xb + (16 * r) * XP + (j & 15) * GC + cl;
#pragma unroll
                for (int q = 0; q < 16; ++q) v[r * 16 + q] = rb[q * XP];
                nbar(bar, GT);
            }
            fma_block<R>(v, f);
            if (pass == 0) fma_block<R>(v, f);   // multiplier
        }
        const long long t = t0 + (long long)i * tstep;
        float2 *p = data + t * 16 + c + (long long)j * NN * NN;
#pragma unroll
        for (int m = 0; m < 32; ++m) p[(long long)m * 32 * NN * NN] = v[m];
    }
}

typedef CUresult (*EncFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                          const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int GROUPS, int R>
float run(const CUtensorMap &m, float2 *a, int nsm) {
    constexpr int GC = 16 / GROUPS;
    constexpr int XP = 16 * GC + (GC == 8 ? 8 : 0);
    const int smem = 16 * NN * 8 + GROUPS * 32 * XP * 8 + 64;
    cudaFuncSetAttribute(k_g<GROUPS, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int r = 0; r < 4; ++r) {
        cudaEventRecord(e0);
        k_g<GROUPS, R><<<nsm, NT, smem>>>(m, a, 1.0000001f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    return best;
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const size_t bytes = (size_t)NN * NN * NN * sizeof(float2);
    float2 *a;
    if (cudaMalloc(&a, bytes) != cudaSuccess) { printf("malloc failed\n"); return 1; }
    cudaMemset(a, 0, bytes);
    void *fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncFn enc = (EncFn)fp;
    CUtensorMap m16;
    const cuuint64_t dims[2] = {(cuuint64_t)(NN * NN), (cuuint64_t)NN};
    const cuuint64_t str[1] = {(cuuint64_t)(NN * NN * 8)};
    const cuuint32_t b16[2] = {16, 256}, es[2] = {1, 1};
    enc(&m16, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, a, dims, str, b16, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int rep = 0; rep < 2; ++rep) {
        printf("R=0: A %.3f ms  B %.3f ms\n", run<1, 0>(m16, a, nsm), run<2, 0>(m16, a, nsm));
        printf("R=3: A %.3f ms  B %.3f ms\n", run<1, 3>(m16, a, nsm), run<2, 3>(m16, a, nsm));
        printf("R=6: A %.3f ms  B %.3f ms\n", run<1, 6>(m16, a, nsm), run<2, 6>(m16, a, nsm));
        printf("R=9: A %.3f ms  B %.3f ms\n", run<1, 9>(m16, a, nsm), run<2, 9>(m16, a, nsm));
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
