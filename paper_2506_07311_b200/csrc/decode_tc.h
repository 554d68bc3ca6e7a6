// Internal interface between the attention dispatcher (kernels.cu) and the
// tensor-core decode kernel (decode_tc.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace pkv {

constexpr int kSmemPlanMax = 512;         // queries planned in shared memory
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
  const int32_t* plan_global;  // global plan buffer, used when nq > kSmemPlanMax
  void* plan_scratch;          // int64 sort scratch for the global plan
  int64_t target_items;
  float* ws_ml;
  float* ws_o;
  // [0] work cursor, [1] finished warps, [2 + q*head_items + hi] split merge;
  // zero-initialised and left zeroed by every launch
  unsigned* counters;
  int ring_offset;
  int merge_offset;
  int kv_dtype;
};

using TcFn = void (*)(TcParams);

bool decode_tc_supported(int kv_dtype, int head_dim);
int64_t decode_tc_plan_bytes(int64_t nq);  // global plan + sort scratch
int launch_decode_tc(TcParams p, int kv_dtype, int head_dim, int num_sms, cudaStream_t stream);
int decode_tc_warps();
int debug_trace(int enable, uint64_t* out, int64_t n);

}  // namespace pkv
