// Throughput probe: MUFU.EX2 vs FMA-pipe exp2 emulation vs FFMA2 on one SM
// (clock64 per CTA, 1 CTA per SM, W warps).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm volatile("{\n .reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " mov.b64 rc, {%6, %7};\n fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0, %1}, rd;\n}\n"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
template <int MODE>
__global__ void probe(float* out, long long* clk, int iters) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (MODE == 0) { a[i] = ex2(a[i]) - 1.0f; a[i + 1] = ex2(a[i + 1]) - 1.0f; }
      else if (MODE == 1) {
        float2 x = make_float2(a[i], a[i + 1]);
        x = ffma2(x, make_float2(0.999f, 0.999f), make_float2(-0.001f, -0.001f));
        a[i] = x.x; a[i + 1] = x.y;
      } else {
        float2 x = make_float2(fmaxf(a[i], -125.f), fmaxf(a[i + 1], -125.f));
        float2 j = ffma2(x, make_float2(1.f, 1.f), make_float2(12582912.f, 12582912.f));
        float2 ii = ffma2(j, make_float2(1.f, 1.f), make_float2(-12582912.f, -12582912.f));
        float2 f = ffma2(ii, make_float2(-1.f, -1.f), x);
        float2 p = ffma2(f, make_float2(0.055f, 0.055f), make_float2(0.242f, 0.242f));
        p = ffma2(p, f, make_float2(0.693f, 0.693f));
        p = ffma2(p, f, make_float2(1.f, 1.f));
        a[i] = __int_as_float(__float_as_int(p.x) + (__float_as_int(j.x) << 23)) - 1.0f;
        a[i + 1] = __int_as_float(__float_as_int(p.y) + (__float_as_int(j.y) << 23)) - 1.0f;
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* clk; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 148 * 8);
  const int iters = 4096;
  const char* names[3] = {"MUFU.EX2", "FFMA2", "emu exp2"};
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {4, 8, 16, 32}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) probe<0><<<148, warps * 32>>>(out, clk, iters);
        if (mode == 1) probe<1><<<148, warps * 32>>>(out, clk, iters);
        if (mode == 2) probe<2><<<148, warps * 32>>>(out, clk, iters);
      }
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      double elems = double(iters) * 16 * warps * 32;  // per SM
      printf("%-9s warps %2d: %.2f elements/clk/SM\n", names[mode], warps, elems / c);
    }
  return 0;
}
