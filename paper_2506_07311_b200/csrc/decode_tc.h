// Internal interface between the attention dispatcher (kernels.cu) and the
// tensor-core decode kernel (decode_tc.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace pkv {

constexpr int kSmemPlanMax = 2048;        // queries planned in shared memory
constexpr int kMaxExtraSplitsTc = 8192;   // same bound as the CUDA-core path

struct TcParams {
  const void* q;
  int q_dtype;
  int nq;
  const int32_t* q_seq;
  const int32_t* q_nkeys;
  const char* k;
  const char* v;
  char* kw;  // same caches, written by the fused append
  char* vw;
  const char* k_new;  // optional [nq, hkv, D] new-token rows (fused append)
  const char* v_new;
  const int32_t* bt;
  int64_t bt_stride;
  const int32_t* seq_row;
  const int64_t* seq_start;
  int log2ps;
  int hq, hkv, group, qgroups, head_items;
  int64_t row_stride;  // Hkv * D * 2 bytes
  float qscale;        // scale * log2(e)
  void* out;
  int out_dtype;
  const int32_t* plan_global;  // non-null when nq > kSmemPlanMax
  int64_t target_items;
  float* ws_ml;
  float* ws_o;
  unsigned* counters;  // [nq * head_items], zero-initialised, self-resetting
  int ring_offset;
};

using TcFn = void (*)(TcParams);

bool decode_tc_supported(int kv_dtype, int head_dim);
int decode_tc_smem_bytes(int head_dim, int64_t nq);
int launch_decode_tc(TcParams p, int kv_dtype, int head_dim, int num_sms, cudaStream_t stream);
int decode_tc_warps();

}  // namespace pkv
