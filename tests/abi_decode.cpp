// Pure C-ABI client of libpkv200.so (no Python, no torch): the path a
// foreign-language binding of the reference's paged_attention would take
// (INTEGRATION.md).  Builds a scattered paged cache with the native
// allocator, appends K/V with pkv_kv_append, plans and runs one bf16 GQA
// decode step with pkv_paged_attention, and checks it against a CPU fp32
// reference computed here.  Prints "abi ok <rel err>" and exits 0 on success.
//
//   g++ -O2 -I include tests/abi_decode.cpp -L paper_2506_07311_b200 -lpkv200 \
//       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,...
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "pkv200.h"

#define CK(x)                                                                 \
  do {                                                                        \
    int _s = (x);                                                             \
    if (_s) {                                                                 \
      std::fprintf(stderr, "%s -> %d (%s)\n", #x, _s, pkv_last_error());      \
      return 1;                                                               \
    }                                                                         \
  } while (0)
#define CU(x)                                                                 \
  do {                                                                        \
    cudaError_t _e = (x);                                                     \
    if (_e != cudaSuccess) {                                                  \
      std::fprintf(stderr, "%s -> %s\n", #x, cudaGetErrorString(_e));         \
      return 1;                                                               \
    }                                                                         \
  } while (0)

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }

int main() {
  const int hq = 32, hkv = 8, d = 128, ps = 16, G = hq / hkv;
  const std::vector<int> lens = {37, 700, 1};
  const int B = static_cast<int>(lens.size());
  const uint64_t cap_pages = 256;
  pkv_pool* pool = nullptr;
  CK(pkv_pool_create(cap_pages, ps, &pool));
  // scattered tables: a throw-away reservation between the real ones
  std::vector<uint32_t> pages(64);
  int64_t got = 0;
  for (int b = 0; b < B; ++b) {
    CK(pkv_pool_reserve(pool, 1000 + b, ps * (1 + b), pages.data(), &got));
    CK(pkv_pool_reserve(pool, b, lens[b] + 1, pages.data(), &got));
  }
  for (int b = 0; b < B; ++b) CK(pkv_pool_free(pool, 1000 + b, &got));
  int64_t rows = 0, cols = 0;
  CK(pkv_pool_mirror_shape(pool, &rows, &cols));
  std::vector<int32_t> mirror(rows * cols);
  CK(pkv_pool_mirror_export(pool, mirror.data(), rows, cols));
  std::vector<int32_t> seq_row(B);
  for (int b = 0; b < B; ++b) CK(pkv_pool_mirror_row(pool, b, &seq_row[b]));

  // host data (bf16-rounded) and device buffers
  std::mt19937 rng(7);
  std::normal_distribution<float> nd;
  const size_t row_elems = size_t(hkv) * d;
  std::vector<std::vector<float>> K(B), V(B);
  for (int b = 0; b < B; ++b) {
    const int n = lens[b] + 1;  // the prompt plus the token appended by the step
    K[b].resize(n * row_elems);
    V[b].resize(n * row_elems);
    for (auto& x : K[b]) x = bf(nd(rng));
    for (auto& x : V[b]) x = bf(nd(rng));
  }
  std::vector<float> Q(size_t(B) * hq * d);
  for (auto& x : Q) x = bf(nd(rng));
  const size_t cache_rows = cap_pages * ps;
  __nv_bfloat16 *kc, *vc, *knew, *q;
  float* out;
  int32_t *dmirror, *meta;
  CU(cudaMalloc(&kc, cache_rows * row_elems * 2));
  CU(cudaMalloc(&vc, cache_rows * row_elems * 2));
  CU(cudaMemset(kc, 0, cache_rows * row_elems * 2));
  CU(cudaMemset(vc, 0, cache_rows * row_elems * 2));
  CU(cudaMalloc(&dmirror, mirror.size() * 4));
  CU(cudaMemcpy(dmirror, mirror.data(), mirror.size() * 4, cudaMemcpyHostToDevice));

  // K1: append every prompt with pkv_kv_append (one sequence per call)
  for (int b = 0; b < B; ++b) {
    const int n = lens[b];
    std::vector<__nv_bfloat16> kh(n * row_elems), vh(n * row_elems);
    for (size_t i = 0; i < kh.size(); ++i) {
      kh[i] = __float2bfloat16(K[b][i]);
      vh[i] = __float2bfloat16(V[b][i]);
    }
    std::vector<int32_t> pos(n), row(1, seq_row[b]);
    for (int i = 0; i < n; ++i) pos[i] = i;
    __nv_bfloat16 *dk, *dv;
    int32_t *dpos, *drow;
    CU(cudaMalloc(&dk, kh.size() * 2));
    CU(cudaMalloc(&dv, vh.size() * 2));
    CU(cudaMalloc(&dpos, n * 4));
    CU(cudaMalloc(&drow, 4));
    CU(cudaMemcpy(dk, kh.data(), kh.size() * 2, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(dv, vh.data(), vh.size() * 2, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(dpos, pos.data(), n * 4, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(drow, row.data(), 4, cudaMemcpyHostToDevice));
    CK(pkv_kv_append(dk, dv, n, drow, 0, dpos, dmirror, cols, ps, kc, vc, int64_t(row_elems) * 2, nullptr));
    CU(cudaDeviceSynchronize());
    cudaFree(dk);
    cudaFree(dv);
    cudaFree(dpos);
    cudaFree(drow);
  }
  // the decode step: new token (fused append) + attention over len+1 keys
  std::vector<__nv_bfloat16> qh(Q.size()), kn(size_t(B) * row_elems), vn(size_t(B) * row_elems);
  for (size_t i = 0; i < Q.size(); ++i) qh[i] = __float2bfloat16(Q[i]);
  for (int b = 0; b < B; ++b)
    for (size_t i = 0; i < row_elems; ++i) {
      kn[b * row_elems + i] = __float2bfloat16(K[b][lens[b] * row_elems + i]);
      vn[b * row_elems + i] = __float2bfloat16(V[b][lens[b] * row_elems + i]);
    }
  __nv_bfloat16* vnew;
  CU(cudaMalloc(&q, qh.size() * 2));
  CU(cudaMalloc(&knew, kn.size() * 2));
  CU(cudaMalloc(&vnew, vn.size() * 2));
  CU(cudaMalloc(&out, Q.size() * 4));
  CU(cudaMemcpy(q, qh.data(), qh.size() * 2, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(knew, kn.data(), kn.size() * 2, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(vnew, vn.data(), vn.size() * 2, cudaMemcpyHostToDevice));
  std::vector<int32_t> nk(B), qseq(B);
  for (int b = 0; b < B; ++b) {
    nk[b] = lens[b] + 1;
    qseq[b] = b;
  }
  const int64_t plan_cap = pkv_attention_plan_ints(B, hq);
  std::vector<int32_t> host(3 * B + plan_cap);
  int64_t plan_n = 0;
  CK(pkv_attention_plan(nk.data(), seq_row.data(), B, ps, hq, hkv, 0, 0, host.data() + 3 * B, plan_cap, &plan_n));
  std::memcpy(host.data(), qseq.data(), B * 4);
  std::memcpy(host.data() + B, nk.data(), B * 4);
  std::memcpy(host.data() + 2 * B, seq_row.data(), B * 4);
  CU(cudaMalloc(&meta, host.size() * 4));
  CU(cudaMemcpy(meta, host.data(), (3 * B + plan_n) * 4, cudaMemcpyHostToDevice));
  const int64_t ws_bytes = pkv_attention_workspace_bytes(B, hq, d);
  void* ws;
  CU(cudaMalloc(&ws, ws_bytes));
  pkv_attention_args a;
  std::memset(&a, 0, sizeof(a));
  a.q = q;
  a.q_dtype = PKV_BF16;
  a.n_queries = B;
  a.q_seq = meta;
  a.q_nkeys = meta + B;
  a.k_cache = kc;
  a.v_cache = vc;
  a.kv_dtype = PKV_BF16;
  a.block_table = dmirror;
  a.bt_stride = cols;
  a.seq_row = meta + 2 * B;
  a.page_size = ps;
  a.hq = hq;
  a.hkv = hkv;
  a.head_dim = d;
  a.scale = 1.0f / std::sqrt(float(d));
  a.out = out;
  a.out_dtype = PKV_F32;
  a.workspace = ws;
  a.workspace_bytes = ws_bytes;
  a.k_new = knew;
  a.v_new = vnew;
  a.plan = meta + 3 * B;
  a.plan_host = host.data() + 3 * B;
  CK(pkv_paged_attention(&a, nullptr));
  CU(cudaDeviceSynchronize());
  std::vector<float> got_out(Q.size());
  CU(cudaMemcpy(got_out.data(), out, Q.size() * 4, cudaMemcpyDeviceToHost));

  // CPU fp32 reference (reference attention.py:259-329 semantics, GQA fold)
  double max_err = 0, max_ref = 0;
  for (int b = 0; b < B; ++b) {
    const int n = lens[b] + 1;
    for (int h = 0; h < hq; ++h) {
      const int kh_ = h / G;
      std::vector<double> s(n);
      double mx = -1e300;
      for (int i = 0; i < n; ++i) {
        double acc = 0;
        for (int e = 0; e < d; ++e) acc += double(Q[(size_t(b) * hq + h) * d + e]) * K[b][i * row_elems + kh_ * d + e];
        s[i] = acc * a.scale;
        mx = std::max(mx, s[i]);
      }
      double den = 0;
      for (int i = 0; i < n; ++i) den += (s[i] = std::exp(s[i] - mx));
      for (int e = 0; e < d; ++e) {
        double o = 0;
        for (int i = 0; i < n; ++i) o += s[i] * V[b][i * row_elems + kh_ * d + e];
        o /= den;
        max_ref = std::max(max_ref, std::fabs(o));
        max_err = std::max(max_err, std::fabs(o - got_out[(size_t(b) * hq + h) * d + e]));
      }
    }
  }
  const double rel = max_err / max_ref;  // the reference metric (verify.py:40-43)
  pkv_pool_destroy(pool);
  std::printf("abi ok %.3e\n", rel);
  return rel <= 2e-2 ? 0 : 2;
}
