// Read-only HBM bandwidth probe (context for the decode roofline, whose
// denominator is the driver's read+write copy): streams a 4 GiB buffer with
// 16-byte non-coherent loads (and, second, with 32 KB cp.async.bulk copies
// into shared memory), grid = k x 148 CTAs, best of 10 by CUDA events.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void read_ldg(const uint4* __restrict__ p, size_t n, unsigned* sink) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}
__global__ void read_bulk(const uint8_t* p, size_t chunks, unsigned* sink) {
  extern __shared__ __align__(128) uint8_t buf[];
  __shared__ __align__(8) uint64_t bar[4];
  constexpr uint32_t kChunk = 32768;
  const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(bar);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0 + 8 * s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int k = 0;
  for (size_t c = blockIdx.x; c < chunks; c += gridDim.x, ++k) {
    const int s = k & 3;
    const uint32_t bar_s = b0 + 8 * s;
    if (k >= 4) {
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q; }"
                     : "=r"(done) : "r"(bar_s), "r"(((k >> 2) - 1) & 1) : "memory");
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_s), "r"(kChunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"((uint32_t)__cvta_generic_to_shared(buf + s * kChunk)), "l"(p + c * kChunk), "r"(kChunk), "r"(bar_s) : "memory");
  }
  for (int s = 0; s < 4 && s < k; ++s) {
    const int kk = k - 1 - s;  // drain the last four
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q; }"
                   : "=r"(done) : "r"(b0 + 8 * (kk & 3)), "r"((kk >> 2) & 1) : "memory");
  }
  if (buf[0] == 0x5a && buf[1] == 0xa5) sink[0] = 1;
}
int main() {
  const size_t bytes = size_t(4) << 30;
  uint8_t* p; unsigned* sink;
  cudaMalloc(&p, bytes); cudaMalloc(&sink, 4); cudaMemset(p, 1, bytes);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaFuncSetAttribute(read_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
  for (int mode = 0; mode < 2; ++mode)
    for (int k : {1, 2, 4, 8}) {
      float best = 1e9;
      for (int rep = 0; rep < 10; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) read_ldg<<<148 * k, 512>>>((const uint4*)p, bytes / 16, sink);
        else read_bulk<<<148 * k, 32, 4 * 32768>>>(p, bytes / 32768, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
      }
      printf("{\"probe\": \"%s\", \"ctas_per_sm\": %d, \"read_gbs\": %.1f}\n", mode ? "cp.async.bulk 32KB x4" : "ldg.nc.v4",
             k, bytes / (best * 1e-3) / 1e9);
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
