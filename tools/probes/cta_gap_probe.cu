// CTA turnover probe: 1024 CTAs of 384 threads with K3's 197 KB of dynamic
// shared memory (one CTA per SM), each spinning ~20 us; per-CTA globaltimer
// start / end and SM id -> idle gap between consecutive CTAs on an SM.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
__global__ void spin(unsigned long long* rec, unsigned long long ns, int tmem, float4* out, int stores) {
  extern __shared__ char sm[];
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  __shared__ unsigned slot;
  if (tmem && (threadIdx.x >> 5) == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  __syncthreads();
  unsigned long long t = t0;
  while (t - t0 < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0) sm[0] = 1;
  // the K3 epilogue: 2 x 128 rows x 128 fp32 outputs per CTA, from 256 threads
  if (stores == 1 && threadIdx.x >= 128)
    for (int e = 0; e < 32; ++e)
      out[(size_t(blockIdx.x) * 256 + (threadIdx.x - 128)) * 32 + e] = make_float4(1.f, 2.f, 3.f, float(e));
  if (stores == 2) {  // stage in shared memory, one thread issues bulk async stores
    if (threadIdx.x >= 128)
      for (int e = 0; e < 32; ++e)
        reinterpret_cast<float4*>(sm)[(threadIdx.x - 128) * 32 + e] = make_float4(1.f, 2.f, 3.f, float(e));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int c = 0; c < 64; ++c)  // 64 x 2 KB
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 2048;" ::"l"(
                         reinterpret_cast<char*>(out) + (size_t(blockIdx.x) * 64 + c) * 2048),
                     "r"((unsigned)__cvta_generic_to_shared(sm + c * 2048)) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
  }
  unsigned long long t_end;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
  t = t_end;
  __syncthreads();
  if (tmem && (threadIdx.x >> 5) == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(slot) : "memory");
  }
  if (threadIdx.x == 0) {
    unsigned smid; asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    rec[blockIdx.x * 3] = t0; rec[blockIdx.x * 3 + 1] = t; rec[blockIdx.x * 3 + 2] = smid;
  }
}
int main() {
  const int n = 1024, smem = 197 * 1024;
  unsigned long long* rec; cudaMalloc(&rec, n * 3 * 8);
  cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  float4* out; cudaMalloc(&out, size_t(n) * 256 * 32 * 16);
  for (int tmem = 0; tmem < 6; tmem += 1) {
    if (tmem & 1) continue;
    for (int rep = 0; rep < 2; ++rep) spin<<<n, 384, smem>>>(rec, 20000, tmem & 1, out, tmem >> 1);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h(n * 3);
    cudaMemcpy(h.data(), rec, n * 3 * 8, cudaMemcpyDeviceToHost);
    std::vector<double> gaps;
    for (int s = 0; s < 148; ++s) {
      std::vector<std::pair<unsigned long long, unsigned long long>> v;
      for (int i = 0; i < n; ++i) if ((int)h[i * 3 + 2] == s) v.push_back({h[i * 3], h[i * 3 + 1]});
      std::sort(v.begin(), v.end());
      for (size_t i = 1; i < v.size(); ++i) gaps.push_back((double)(v[i].first - v[i - 1].second) / 1e3);
    }
    std::sort(gaps.begin(), gaps.end());
    printf("tmem %d stores %d: %zu gaps, median %.2f us, p90 %.2f us\n", tmem & 1, tmem >> 1, gaps.size(), gaps[gaps.size() / 2], gaps[gaps.size() * 9 / 10]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
