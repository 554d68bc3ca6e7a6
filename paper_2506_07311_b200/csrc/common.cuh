// Device helpers shared by the sm_100a kernels (cp.async, mma.sync, dtype
// conversion, byte copies).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "pkv200.h"
#include "status.h"

namespace pkv {

#define PKV_CHECK_LAUNCH()                                                                \
  do {                                                                                    \
    cudaError_t _e = cudaGetLastError();                                                  \
    if (_e != cudaSuccess)                                                                \
      return pkv::fail(PKV_CUDA_ERROR, "%s: %s", __func__, cudaGetErrorString(_e));       \
  } while (0)

inline int elem_bytes(int dt) { return dt == PKV_F32 ? 4 : 2; }

// Message of a failed runtime call; also clears the (non-sticky) last error
// so a later launch check does not report this failure again.
inline const char* cuda_err_str(cudaError_t e) {
  cudaGetLastError();
  return cudaGetErrorString(e);
}

// Launch on the stream's device: entry points may be called while another
// device is current (a store on cuda:1 driven from a thread whose current
// device is cuda:0).  The legacy null stream has no device of its own and
// keeps the current one.  Restores the caller's device on exit.
// Load every kernel of the library on the current device once (CUDA's lazy
// module loading would otherwise load a kernel at its first launch — ~10 ms
// in the middle of a serving loop the first time a step needs, say, the
// cluster-mode decode variant).  Cheap after the first call: one flag test.
void preload_kernels();

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(cudaStream_t s) {
    if (s) {
      int dev = 0, cur = 0;
      if (cudaStreamGetDevice(s, &dev) != cudaSuccess || cudaGetDevice(&cur) != cudaSuccess) {
        cudaGetLastError();
      } else if (dev != cur && cudaSetDevice(dev) == cudaSuccess) {
        prev = cur;
      }
    }
    preload_kernels();
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// ---------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int VEC>
__device__ __forceinline__ void cp_async(uint32_t dst, const void* src, int src_bytes) {
  if constexpr (VEC == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
                 "r"(src_bytes));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(dst), "l"(src),
                 "n"(VEC), "r"(src_bytes));
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// element type traits: convert 16-byte chunks to fp32
template <typename T>
struct Elem;
template <>
struct Elem<float> {
  static constexpr int kBytes = 4;
  static constexpr int kPerChunk = 4;
  __device__ __forceinline__ static void unpack(const uint4& c, float* f) {
    f[0] = __uint_as_float(c.x);
    f[1] = __uint_as_float(c.y);
    f[2] = __uint_as_float(c.z);
    f[3] = __uint_as_float(c.w);
  }
};
template <>
struct Elem<__nv_bfloat16> {
  static constexpr int kBytes = 2;
  static constexpr int kPerChunk = 8;
  __device__ __forceinline__ static void unpack(const uint4& c, float* f) {
    const uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
};
template <>
struct Elem<__half> {
  static constexpr int kBytes = 2;
  static constexpr int kPerChunk = 8;
  __device__ __forceinline__ static void unpack(const uint4& c, float* f) {
    const uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 h = *reinterpret_cast<const __half2*>(&w[i]);
      float2 v = __half22float2(h);
      f[2 * i] = v.x;
      f[2 * i + 1] = v.y;
    }
  }
};

__device__ __forceinline__ float load_as_float(const void* base, int64_t idx, int dtype) {
  if (dtype == PKV_F32) return static_cast<const float*>(base)[idx];
  if (dtype == PKV_BF16) return __bfloat162float(static_cast<const __nv_bfloat16*>(base)[idx]);
  return __half2float(static_cast<const __half*>(base)[idx]);
}
__device__ __forceinline__ void store_from_float(void* base, int64_t idx, int dtype, float v) {
  if (dtype == PKV_F32)
    static_cast<float*>(base)[idx] = v;
  else if (dtype == PKV_BF16)
    static_cast<__nv_bfloat16*>(base)[idx] = __float2bfloat16_rn(v);
  else
    static_cast<__half*>(base)[idx] = __float2half_rn(v);
}

// four consecutive outputs (idx a multiple of 4) with one vector store: one
// dtype switch instead of four (the merge tails run once per launch from a
// cold instruction cache, so their code size is their latency)
__device__ __forceinline__ void store4_from_float(void* base, int64_t idx, int dtype, float4 v) {
  if (dtype == PKV_F32) {
    *reinterpret_cast<float4*>(static_cast<float*>(base) + idx) = v;
  } else if (dtype == PKV_BF16) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 w;
    w.x = *reinterpret_cast<uint32_t*>(&a);
    w.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(base) + idx) = w;
  } else {
    __half2 a = __floats2half2_rn(v.x, v.y), b = __floats2half2_rn(v.z, v.w);
    uint2 w;
    w.x = *reinterpret_cast<uint32_t*>(&a);
    w.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(static_cast<__half*>(base) + idx) = w;
  }
}
// two consecutive outputs (idx even)
__device__ __forceinline__ void store2_from_float(void* base, int64_t idx, int dtype, float a, float b) {
  if (dtype == PKV_F32) {
    *reinterpret_cast<float2*>(static_cast<float*>(base) + idx) = make_float2(a, b);
  } else if (dtype == PKV_BF16) {
    *reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(base) + idx) = __floats2bfloat162_rn(a, b);
  } else {
    *reinterpret_cast<__half2*>(static_cast<__half*>(base) + idx) = __floats2half2_rn(a, b);
  }
}

// byte copy with the widest vector the alignment allows
__device__ __forceinline__ void copy_bytes(char* dst, const char* src, int64_t n, int64_t tid,
                                           int64_t nthreads) {
  if ((n & 15) == 0) {
    for (int64_t i = tid; i < (n >> 4); i += nthreads)
      reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
  } else if ((n & 3) == 0) {
    for (int64_t i = tid; i < (n >> 2); i += nthreads)
      reinterpret_cast<uint32_t*>(dst)[i] = reinterpret_cast<const uint32_t*>(src)[i];
  } else {
    for (int64_t i = tid; i < (n >> 1); i += nthreads)
      reinterpret_cast<uint16_t*>(dst)[i] = reinterpret_cast<const uint16_t*>(src)[i];
  }
}
__device__ __forceinline__ void zero_bytes(char* dst, int64_t n, int64_t tid, int64_t nthreads) {
  if ((n & 15) == 0) {
    for (int64_t i = tid; i < (n >> 4); i += nthreads)
      reinterpret_cast<uint4*>(dst)[i] = make_uint4(0, 0, 0, 0);
  } else if ((n & 3) == 0) {
    for (int64_t i = tid; i < (n >> 2); i += nthreads) reinterpret_cast<uint32_t*>(dst)[i] = 0;
  } else {
    for (int64_t i = tid; i < (n >> 1); i += nthreads) reinterpret_cast<uint16_t*>(dst)[i] = 0;
  }
}


// bulk prefetch of `bytes` (multiple of 16, 16-B aligned) into L2
__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                            uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1,
                                                  uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// D(16x8, f32) += A(16x16) * B(16x8), bf16 or fp16 inputs
template <typename T>
__device__ __forceinline__ void mma_16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1);
template <>
__device__ __forceinline__ void mma_16816<__nv_bfloat16>(float* d, const uint32_t* a, uint32_t b0,
                                                        uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <>
__device__ __forceinline__ void mma_16816<__half>(float* d, const uint32_t* a, uint32_t b0,
                                                 uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// pack two floats into a bf16x2 / f16x2 register (round to nearest even)
template <typename T>
__device__ __forceinline__ uint32_t pack2(float lo, float hi);
template <>
__device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
template <>
__device__ __forceinline__ uint32_t pack2<__half>(float lo, float hi) {
  __half2 v = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// sum of the two 16-bit lanes of a packed register, as fp32
template <typename T>
__device__ __forceinline__ float unpack_sum(uint32_t v);
template <>
__device__ __forceinline__ float unpack_sum<__nv_bfloat16>(uint32_t v) {
  return __uint_as_float(v << 16) + __uint_as_float(v & 0xffff0000u);
}
template <>
__device__ __forceinline__ float unpack_sum<__half>(uint32_t v) {
  const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&v));
  return f.x + f.y;
}

// 2^x on the SFU, flushing denormal results to zero (exp2f adds a
// range-reduction fix-up of ~3 instructions per call for denormals, which
// softmax never needs: p < 2^-126 is zero for every purpose here)
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// packed fp32 FMA / add (sm_100 FFMA2 / FADD2): two lanes per instruction
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n .reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " mov.b64 rc, {%6, %7};\n fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0, %1}, rd;\n}\n"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " add.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;\n}\n"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

// wrapping increment with acquire-release semantics at GPU scope
__device__ __forceinline__ unsigned atom_inc_acq_rel(unsigned* addr, unsigned wrap) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.inc.u32 %0, [%1], %2;\n" : "=r"(old) : "l"(addr), "r"(wrap) : "memory");
  return old;
}

template <typename T>
__device__ __forceinline__ float round_to(float x);
template <>
__device__ __forceinline__ float round_to<__nv_bfloat16>(float x) {
  return __bfloat162float(__float2bfloat16_rn(x));
}
template <>
__device__ __forceinline__ float round_to<__half>(float x) {
  return __half2float(__float2half_rn(x));
}

}  // namespace pkv
