// zpair.cu -- data movement of the z pass (K_C) with TMA tiles, 1024^3
// complex64, in place: can pairs of CTAs get the 256-byte-row efficiency of
// 32-column tiles (tools/micro/zwide.cu: 16 columns 4.2 TB/s, 32 columns
// 5.8 TB/s) while each CTA still holds only 16 columns x 1024 rows?
//
//   A  one CTA per tile (16 columns x 1024 rows; 4 TMA boxes {16, 256}),
//      single stage, next tile prefetched after the copy to registers,
//      stores from registers -- the k_stile data path
//   B  2-CTA clusters on adjacent 16-column tiles, a cluster barrier per tile
//      so both CTAs issue their boxes together (same rows, adjacent 128 B)
//   C  2-CTA clusters on a 32-column tile: CTA r loads rows [512 r, 512 r + 512)
//      of all 32 columns ({32, 256} boxes, 256-byte rows) and each CTA reads
//      its 16 columns of the partner's rows through distributed shared memory
//   D  as C, and stores go back through shared memory as {32, 256} TMA boxes
//      (each CTA writes its 16 columns of all 1024 rows into the two CTAs'
//      stages, then CTA r stores rows [512 r, 512 r + 512))
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zpair zpair.cu -lcuda && ./zpair
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

// zoverlap: K_C's data path (16-column tiles x 1024 rows, rows 8 MB apart,
// TMA {16,256} boxes into one stage, next tile prefetched right after the
// stage is copied to registers, register stores) with W rounds of synthetic
// register arithmetic per tile between the copy and the stores.  Does the
// arithmetic hide under the in-flight load (time = max) or add (time = sum)?
template <int W>
__global__ void __launch_bounds__(NT, 1) k_o(const __grid_constant__ CUtensorMap map, float2 *data, float f) {
    extern __shared__ __align__(128) unsigned char sm[];
    float2 *stage = (float2 *)sm;
    uint64_t *full = (uint64_t *)(stage + 16 * NN);
    const int c = threadIdx.x % 16, j = threadIdx.x / 16;
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
        __syncthreads();
        if (threadIdx.x == 0 && i + 1 < nloc) issue(i + 1);
        for (int w = 0; w < W; ++w) {
#pragma unroll
            for (int m = 0; m < 32; ++m) v[m] = make_float2(fmaf(v[m].x, f, v[(m + 1) & 31].y), fmaf(v[m].y, f, -v[m].x));
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

template <int W>
float run(const CUtensorMap &m, float2 *a, int nsm, int smA) {
    cudaFuncSetAttribute(k_o<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, smA);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int r = 0; r < 4; ++r) {
        cudaEventRecord(e0);
        k_o<W><<<nsm, NT, smA>>>(m, a, 1.0000001f);
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
    const int smA = 16 * NN * 8 + 64;
    const double gb = 2.0 * NN * NN * NN * 8 / 1e9;
    for (int rep = 0; rep < 2; ++rep) {
        float t;
        t = run<0>(m16, a, nsm, smA);  printf("W=0   %.3f ms  %.0f GB/s\n", t, gb / t * 1e3);
        t = run<4>(m16, a, nsm, smA);  printf("W=4   %.3f ms\n", t);
        t = run<8>(m16, a, nsm, smA);  printf("W=8   %.3f ms\n", t);
        t = run<16>(m16, a, nsm, smA); printf("W=16  %.3f ms\n", t);
        t = run<32>(m16, a, nsm, smA); printf("W=32  %.3f ms\n", t);
        t = run<64>(m16, a, nsm, smA); printf("W=64  %.3f ms\n", t);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
