// Internal interface between the attention dispatcher (kernels.cu) and the
// tensor-core decode kernel + host planner (decode_tc.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace pkv {

constexpr int kSmemPlanMax = 512;  // queries whose plan is staged in shared memory

struct TcParams {
  const void* q;
  int q_dtype;
  int nq;
  const char* k;
  const char* v;
  char* kw;  // same caches, written by the fused append
  char* vw;
  const char* k_new;  // optional [nq, hkv, D] new-token rows (fused append)
  const char* v_new;
  const int32_t* bt;  // NULL: gathered (contiguous) source
  int64_t bt_stride;
  int log2ps;
  int hq, hkv, group;
  int64_t row_stride;  // Hkv * D * 2 bytes
  float qscale;        // scale * log2(e)
  void* out;
  int out_dtype;
  const int32_t* plan;  // device copy of the host plan (plan_decode)
  float* ws_ml;         // split partials (m, l)
  float* ws_o;          // split partials O
  int plan_in_smem;
  int merge_offset;
  int ring_offset;
  int kv_dtype;
};

// cluster mode with few queries: the plan rides in a second launch parameter
// of a separate kernel instantiation (no dependent plan loads before the
// first block-table read; the other instantiations keep the small TcParams)
struct ClusterInline {
  int hb, wph, qgs, qgroups, head_items, cluster;
  int32_t nkrow[2 * 64];  // nk[nq] | row[nq]
};

using TcFn = void (*)(TcParams);

bool decode_tc_supported(int kv_dtype, int head_dim);
int64_t decode_plan_ints(int64_t nq, int hq);
int plan_decode(const int32_t* nk, const int32_t* row, int64_t nq, int page_size, int hq, int hkv, int head_dim,
                int num_sms, int waves, int32_t* out, int64_t cap, int64_t* n_out);
// cudaFuncGetAttributes on every decode_tc instance (forces lazy loading)
void preload_decode_tc_kernels();
void preload_prefill_kernels();  // prefill_sm100.cu
int launch_decode_tc(TcParams p, const int32_t* plan_host, int kv_dtype, int head_dim, int num_sms,
                     cudaStream_t stream);
int decode_tc_warps();
int debug_trace(int enable, uint64_t* out, int64_t n);

}  // namespace pkv
