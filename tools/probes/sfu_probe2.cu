// Packed-exp2 throughput on the SFU: ex2.approx.f32 vs ex2.approx.f16x2 vs
// ex2.approx.ftz.bf16x2 (elements / clk / SM, one CTA per SM)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__global__ void probe(uint32_t* out, long long* clk, int iters) {
  uint32_t a[16];
  for (int i = 0; i < 16; ++i) a[i] = 0xbc00bc00u ^ (threadIdx.x + i);  // small negative halves / bf16s
  float f[16];
  for (int i = 0; i < 16; ++i) f[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
      if (MODE == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
      if (MODE == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
      if (MODE == 3) {  // f32 pair -> packed bf16x2 (F2FP), fed back through a float add
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(f[i]), "f"(f[(i + 1) & 15]));
        f[i] = __uint_as_float(r) + 1.0f;
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < 16; ++i) s ^= a[i] ^ __float_as_uint(f[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
int main() {
  uint32_t* out; long long* clk; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 148 * 8);
  const int iters = 2048;
  const char* names[4] = {"ex2.f32", "ex2.f16x2", "ex2.bf16x2", "cvt.bf16x2"};
  for (int mode = 0; mode < 4; ++mode)
    for (int warps : {4, 16}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) probe<0><<<148, warps * 32>>>(out, clk, iters);
        if (mode == 1) probe<1><<<148, warps * 32>>>(out, clk, iters);
        if (mode == 2) probe<2><<<148, warps * 32>>>(out, clk, iters);
        if (mode == 3) probe<3><<<148, warps * 32>>>(out, clk, iters);
      }
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      double elems = double(iters) * 16 * warps * 32 * (mode == 1 || mode == 2 ? 2 : 1);
      printf("%-10s warps %2d: %.2f ops/clk/SM (per packed pair for cvt)\n", names[mode], warps, elems / c);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
