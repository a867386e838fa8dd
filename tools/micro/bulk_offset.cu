// micro-test: cp.async.bulk from offsets beyond 2^31 / 2^32 bytes
#include <cstdio>
#include <cuda_runtime.h>
#include "tma.cuh"
using namespace usp;
__global__ void k(const float2* base, long long off_elems, float* out, int bytes) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, bytes);
    bulk_g2s(sm, base + off_elems, bytes, &bar);
  }
  bool ok = mbar_wait(&bar, 0);
  float2 v = reinterpret_cast<float2*>(sm)[threadIdx.x];
  out[threadIdx.x] = ok ? v.x : -1.f;
}
int main() {
  size_t n = (size_t)5 << 27;   // 5 * 128M float2 = 5 GiB
  float2* d; cudaMalloc(&d, n * sizeof(float2));
  float* o; cudaMalloc(&o, 32 * sizeof(float));
  long long offs[] = {0, (1LL << 28) - 1024, (1LL << 28) + 1024, (1LL << 29) + 4096, (1LL<<29) + (1LL<<28)};
  for (long long off : offs) {
    float2 h[32]; for (int i = 0; i < 32; ++i) h[i] = make_float2((float)(off % 1000) + i, 0.f);
    cudaMemcpy(d + off, h, sizeof h, cudaMemcpyHostToDevice);
    k<<<1, 32, 8192>>>(d, off, o, 8192);
    cudaError_t e = cudaDeviceSynchronize();
    float r[32]; cudaMemcpy(r, o, sizeof r, cudaMemcpyDeviceToHost);
    printf("off elems %lld bytes %.3f GiB: %s r0=%g r31=%g expect %g\n", off, off * 8.0 / (1 << 30), cudaGetErrorString(e), r[0], r[31], (double)(off % 1000) + 31);
    if (e) break;
  }
}
