// sm_100a data-plane kernels of the paged-attention engine.
//
//   K0a page_zero      KvStore.clear_pages        (reference store.py:95-100)
//   K0b page_copy      KvStore.copy_rows          (reference store.py:85-93)
//   K1  kv_append      KvStore.assign scatter     (reference store.py:146-150)
//   K2  split-K decode paged_attention            (reference attention.py:259-354)
//   K2c combine        merge of split partials
//   mirror_apply       device block-table mirror update (new)
//
// Layout in HBM (one store = one layer): K and V caches are row-major
// [pages * page_size, Hkv, D] in the element type of the store — the
// reference's NHD row layout (store.py:74-76) — so one (page, kv-head) slice is
// page_size rows of D*s bytes at a stride of Hkv*D*s bytes.
//
// K2 design (memory bound): the unit of work is one *warp* on
// (query, kv-head, q-head group, key split).  Each warp streams its split
// through a private multi-stage cp.async ring in shared memory (16-byte
// copies, zero-fill past the valid keys), computes scores with the G grouped
// query heads held in registers (so each K/V byte is read from HBM once per
// group), and keeps one online-softmax state per lane group; states are merged
// with warp shuffles at the end of the split.  Splits are planned on the device
// from the per-query key counts (plan kernel), so a decode step needs no host
// round trip and the schedule depends only on logical lengths — paged and
// gathered sources therefore produce bit-identical results.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <chrono>
#include <vector>
#include <cstdint>
#include <cstring>

#include "common.cuh"
#include "pool_internal.h"
#include "decode_tc.h"
#include "step_graph.h"
#include "pkv200.h"
#include "status.h"

namespace {
using namespace pkv;

constexpr int kMaxExtraSplits = 8192;  // planner bound, see workspace_bytes
constexpr float kLog2e = 1.4426950408889634f;

// ---------------------------------------------------------------------------
// K0 / K1 / mirror
// ---------------------------------------------------------------------------
__global__ void mirror_apply_kernel(int32_t* table, const int32_t* pairs, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    table[pairs[2 * i]] = pairs[2 * i + 1];
}

__global__ void page_zero_kernel(char* k, char* v, const int32_t* pages, int64_t n,
                                 int64_t page_bytes) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    int64_t off = int64_t(pages[i]) * page_bytes;
    zero_bytes(k + off, page_bytes, threadIdx.x, blockDim.x);
    zero_bytes(v + off, page_bytes, threadIdx.x, blockDim.x);
  }
}

// triples == NULL: one copy given by (src0, dst0, rows0) (a fork's partial
// page: no metadata upload)
__global__ void page_copy_kernel(char* k, char* v, const int32_t* triples, int64_t n,
                                 int64_t row_bytes, int page_size, int64_t src0, int64_t dst0, int64_t rows0) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const int64_t src = triples ? triples[3 * i] : src0, dst = triples ? triples[3 * i + 1] : dst0;
    const int64_t rows = triples ? triples[3 * i + 2] : rows0;
    const int64_t pb = row_bytes * page_size;
    const int64_t keep = rows * row_bytes;
    // src == dst would alias; the allocator never reports that
    copy_bytes(k + dst * pb, k + src * pb, keep, threadIdx.x, blockDim.x);
    copy_bytes(v + dst * pb, v + src * pb, keep, threadIdx.x, blockDim.x);
    zero_bytes(k + dst * pb + keep, pb - keep, threadIdx.x, blockDim.x);
    zero_bytes(v + dst * pb + keep, pb - keep, threadIdx.x, blockDim.x);
  }
}

// All page work of one decode step in ONE launch, for every attached store:
// blocks [0, n_stores * (n_zero + n_copy)) each clear or copy one page of one
// store, and every block also applies a slice of the block-table mirror pairs.
// Copy destinations are removed from the zero list on the host (a copy writes
// the whole destination page), so no two blocks touch the same bytes.
__global__ void step_aux_kernel(const uint64_t* __restrict__ caches, int n_stores,
                                const int32_t* __restrict__ zero_pages, int64_t n_zero,
                                const int32_t* __restrict__ triples, int64_t n_copy,
                                int32_t* __restrict__ mirror, const int32_t* __restrict__ pairs,
                                int64_t n_pairs, int64_t row_bytes, int page_size) {
  // the decode launch behind this kernel may start its prologue now (PDL;
  // it waits for this grid's completion before touching pages or the table)
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t pb = row_bytes * page_size;
  const int64_t per_store = n_zero + n_copy;
  for (int64_t w = blockIdx.x; w < per_store * n_stores; w += gridDim.x) {
    const int64_t st = w / per_store, i = w % per_store;
    char* k = reinterpret_cast<char*>(caches[2 * st]);
    char* v = reinterpret_cast<char*>(caches[2 * st + 1]);
    if (i < n_zero) {
      const int64_t off = int64_t(zero_pages[i]) * pb;
      zero_bytes(k + off, pb, threadIdx.x, blockDim.x);
      zero_bytes(v + off, pb, threadIdx.x, blockDim.x);
    } else {
      const int32_t* t = triples + 3 * (i - n_zero);
      const int64_t src = t[0], dst = t[1], keep = int64_t(t[2]) * row_bytes;
      copy_bytes(k + dst * pb, k + src * pb, keep, threadIdx.x, blockDim.x);
      copy_bytes(v + dst * pb, v + src * pb, keep, threadIdx.x, blockDim.x);
      zero_bytes(k + dst * pb + keep, pb - keep, threadIdx.x, blockDim.x);
      zero_bytes(v + dst * pb + keep, pb - keep, threadIdx.x, blockDim.x);
    }
  }
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n_pairs;
       i += int64_t(gridDim.x) * blockDim.x)
    mirror[pairs[2 * i]] = pairs[2 * i + 1];
}

// One warp per token (grid-stride over tokens); the slot is resolved
// in-kernel from the block-table mirror (shift/mask: the page size is a power
// of two).  kVec (16-byte rows and pointers): every lane keeps four 16-byte
// K and four V loads in flight before its stores, so a 2 KB row pair moves in
// one round trip per warp.
// tok_pos == NULL: a contiguous run, token t at position pos0 + t of mirror
// row row0 (no per-token metadata at all)
template <bool kVec>
__global__ void __launch_bounds__(256) kv_append_kernel(const char* __restrict__ kn, const char* __restrict__ vn,
                                 int64_t n_tok, const int32_t* __restrict__ tok_row,
                                 int row_stride, const int32_t* __restrict__ tok_pos,
                                 const int32_t* __restrict__ bt, int64_t bt_stride, int log2ps,
                                 char* __restrict__ kc, char* __restrict__ vc, int64_t row_bytes,
                                 int32_t pos0, int32_t row0) {
  const int ps = 1 << log2ps;
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t t = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); t < n_tok; t += warps) {
    const int32_t pos = tok_pos ? tok_pos[t] : pos0 + static_cast<int32_t>(t);
    const int64_t r = tok_pos ? tok_row[t * row_stride] : row0;
    const int64_t page = bt[r * bt_stride + (pos >> log2ps)];
    const int64_t dst = (page * ps + (pos & (ps - 1))) * row_bytes;
    if (kVec) {
      const uint4* ks = reinterpret_cast<const uint4*>(kn + t * row_bytes);
      const uint4* vs = reinterpret_cast<const uint4*>(vn + t * row_bytes);
      uint4* kd = reinterpret_cast<uint4*>(kc + dst);
      uint4* vd = reinterpret_cast<uint4*>(vc + dst);
      const int64_t n16 = row_bytes >> 4;
      for (int64_t b = lane; b < n16; b += 128) {
        uint4 a[4], c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (b + 32 * u < n16) {
            a[u] = __ldg(ks + b + 32 * u);
            c[u] = __ldg(vs + b + 32 * u);
          }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (b + 32 * u < n16) {
            kd[b + 32 * u] = a[u];
            vd[b + 32 * u] = c[u];
          }
      }
    } else {
      copy_bytes(kc + dst, kn + t * row_bytes, row_bytes, lane, 32);
      copy_bytes(vc + dst, vn + t * row_bytes, row_bytes, lane, 32);
    }
  }
}

// grid of the append: one warp per token, at most 16 CTAs of 8 warps per SM
inline unsigned append_blocks(int64_t n_tok) {
  const int64_t want = (n_tok + 7) / 8;
  return static_cast<unsigned>(want < 148 * 16 ? want : 148 * 16);
}
inline bool append_vec(const void* a, const void* b, const void* c, const void* d, int64_t row_bytes) {
  const uintptr_t m = reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
                      reinterpret_cast<uintptr_t>(c) | reinterpret_cast<uintptr_t>(d);
  return (row_bytes & 15) == 0 && (m & 15) == 0;
}

// K-gather (store.py:152-161, 187-190): out[t] = cache[slot(t)] for the
// concatenated positions [0, len_s) of every view sequence s, in view order.
// One warp per row (K and V), lanes stride over the row in 16/4/2-byte
// units; the sequence of a row is found by binary search over the int32
// exclusive prefix cu[0..n_seq] (cu[n_seq] = rows).
__global__ void kv_gather_kernel(const char* __restrict__ kc, const char* __restrict__ vc,
                                 const int32_t* __restrict__ bt, int64_t bt_stride,
                                 const int32_t* __restrict__ seq_row, const int32_t* __restrict__ cu,
                                 int n_seq, int log2ps, int64_t row_bytes, char* __restrict__ ko,
                                 char* __restrict__ vo) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  const int64_t rows = cu[n_seq];
  const int ps = 1 << log2ps;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); t < rows; t += warps) {
    int lo = 0, hi = n_seq - 1;  // last s with cu[s] <= t
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (cu[mid] <= t) lo = mid; else hi = mid - 1;
    }
    const int64_t pos = t - cu[lo];
    const int64_t page = bt[int64_t(seq_row[lo]) * bt_stride + (pos >> log2ps)];
    const int64_t src = (page * ps + (pos & (ps - 1))) * row_bytes;
    copy_bytes(ko + t * row_bytes, kc + src, row_bytes, lane, 32);
    copy_bytes(vo + t * row_bytes, vc + src, row_bytes, lane, 32);
  }
}

// decode-step append for the exact path: query i appends its token at
// position q_nkeys[i]-1 of view sequence q_seq[i]
__global__ void append_decode_kernel(const char* __restrict__ kn, const char* __restrict__ vn,
                                     int64_t nq, const int32_t* __restrict__ q_seq,
                                     const int32_t* __restrict__ q_nkeys,
                                     const int32_t* __restrict__ seq_row,
                                     const int32_t* __restrict__ bt, int64_t bt_stride, int log2ps,
                                     char* __restrict__ kc, char* __restrict__ vc, int64_t row_bytes) {
  const int ps = 1 << log2ps;
  for (int64_t i = blockIdx.x; i < nq; i += gridDim.x) {
    const int32_t pos = q_nkeys[i] - 1;
    const int64_t r = seq_row[q_seq[i]];
    const int64_t page = bt[r * bt_stride + (pos >> log2ps)];
    const int64_t dst = (page * ps + (pos & (ps - 1))) * row_bytes;
    copy_bytes(kc + dst, kn + i * row_bytes, row_bytes, threadIdx.x, blockDim.x);
    copy_bytes(vc + dst, vn + i * row_bytes, row_bytes, threadIdx.x, blockDim.x);
  }
}

// ---------------------------------------------------------------------------
// split planner (device): plan[0] = split_pages, plan[1] = total splits,
// plan[4 + i] = exclusive prefix of per-query split counts (n_queries + 1)
// ---------------------------------------------------------------------------
constexpr int kPlanThreads = 1024;

__global__ void __launch_bounds__(kPlanThreads) plan_kernel(
    const int32_t* __restrict__ q_nkeys, int64_t nq, int log2ps, int head_items,
    int64_t target_items, int32_t* __restrict__ plan) {
  __shared__ long long red[kPlanThreads / 32];
  __shared__ int scan[kPlanThreads / 32];
  __shared__ long long s_total;
  __shared__ int s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ps = 1 << log2ps;
  long long pages = 0;
  for (int64_t i = tid; i < nq; i += kPlanThreads) pages += (q_nkeys[i] + ps - 1) >> log2ps;
#pragma unroll
  for (int o = 16; o; o >>= 1) pages += __shfl_xor_sync(0xffffffffu, pages, o);
  if (lane == 0) red[warp] = pages;
  __syncthreads();
  if (tid == 0) {
    long long t = 0;
    for (int w = 0; w < kPlanThreads / 32; ++w) t += red[w];
    s_total = t;
    s_carry = 0;
  }
  __syncthreads();
  const long long total_pages = s_total;
  long long sp = (total_pages * head_items + target_items - 1) / target_items;
  const long long sp_cap = (total_pages + kMaxExtraSplits - 1) / kMaxExtraSplits;
  if (sp < sp_cap) sp = sp_cap;
  if (sp < 1) sp = 1;
  for (int64_t base = 0; base < nq; base += kPlanThreads) {
    const int64_t i = base + tid;
    int cnt = 0;
    if (i < nq) {
      const long long p = (q_nkeys[i] + ps - 1) >> log2ps;
      cnt = static_cast<int>((p + sp - 1) / sp);
    }
    int x = cnt;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) scan[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int w = scan[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      scan[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int carry = s_carry;
    const int excl = carry + (warp ? scan[warp - 1] : 0) + x - cnt;
    if (i < nq) plan[4 + i] = excl;
    __syncthreads();
    if (tid == kPlanThreads - 1) s_carry = excl + cnt;
    __syncthreads();
  }
  if (tid == 0) {
    plan[0] = static_cast<int32_t>(sp);
    plan[1] = s_carry;
    plan[4 + nq] = s_carry;
  }
}

// ---------------------------------------------------------------------------
// K2: split-K paged decode
// ---------------------------------------------------------------------------
struct DecodeParams {
  const void* q;
  int q_dtype;
  int64_t nq;
  const int32_t* q_seq;
  const int32_t* q_nkeys;
  const char* k;
  const char* v;
  const int32_t* bt;
  int64_t bt_stride;
  const int32_t* seq_row;
  const int64_t* seq_start;
  int log2ps;
  int hq, hkv, d, group, head_items;
  int64_t row_stride_bytes;  // Hkv * D * s
  float qscale;              // scale * log2(e)
  void* out;
  int out_dtype;
  const int32_t* plan;
  float* ws_ml;  // [splits, hq, 2]
  float* ws_o;   // [splits, hq, D]
};

// compile-time geometry of one kernel instance
template <typename T, int DP, int R>
struct Geo {
  static constexpr int S = Elem<T>::kBytes;
  static constexpr int CE = Elem<T>::kPerChunk;      // elements per 16-B chunk
  static constexpr int ROWB = DP * S;                // padded smem row bytes
  static constexpr int EPL = (DP < 32 / S) ? DP : 32 / S;  // elements per lane
  static constexpr int NCH = EPL * S / 16;           // 16-B chunks per lane (1 or 2)
  static constexpr int LPK = DP / EPL;               // lanes per key
  static constexpr int KG = 32 / LPK;                // key groups per warp
  static constexpr int CH0 = 4096 / ROWB;
  static constexpr int CH = CH0 > 32 ? 32 : (CH0 < 4 ? 4 : CH0);  // keys per chunk
  static constexpr int KPL = CH / KG;                // keys per lane group per chunk
  static constexpr int STAGE = 2 * CH * ROWB;        // K + V bytes per stage
  static_assert(NCH == 1 || NCH == 2, "lane owns one or two 16-byte chunks");
  static_assert(LPK >= 1 && LPK <= 32 && KPL >= 1, "bad geometry");
};

constexpr int kWarps = 8;   // warps per CTA (one CTA per SM)
constexpr int kStages = 3;  // cp.async ring depth per warp

template <typename T, int DP, int R>
__global__ void __launch_bounds__(kWarps * 32, 1) decode_kernel(const __grid_constant__ DecodeParams p) {
  using G = Geo<T, DP, R>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  unsigned char* wsm = smem + warp * (kStages * G::STAGE);
  const uint32_t wsm_addr = smem_addr(wsm);
  // zero the ring once: row padding (D..DP) is never written by cp.async
  for (int i = lane; i < kStages * G::STAGE / 16; i += 32)
    reinterpret_cast<uint4*>(wsm)[i] = make_uint4(0, 0, 0, 0);
  __syncwarp();

  const int kg = lane / G::LPK;  // key group
  const int lk = lane % G::LPK;  // lane within key
  const int ps = 1 << p.log2ps;
  const int row_real = p.d * G::S;  // real bytes of one head row
  // copy granularity for the real bytes of a row
  const int vec = (row_real & 15) == 0 ? 16 : ((row_real & 7) == 0 ? 8 : 4);
  const int cpr = row_real / vec;  // copies per row
  const bool cpr_pow2 = (cpr & (cpr - 1)) == 0;
  const int cpr_sh = __ffs(cpr) - 1;

  const int split_pages = p.plan[0];
  const int64_t total_items = int64_t(p.plan[1]) * p.head_items;
  const int32_t* offsets = p.plan + 4;
  const int64_t gwarp = int64_t(blockIdx.x) * kWarps + warp;
  const int64_t nwarps = int64_t(gridDim.x) * kWarps;
  const int qgroups = p.group / R;

  for (int64_t w = gwarp; w < total_items; w += nwarps) {
    const int64_t sg = w / p.head_items;
    const int hi = static_cast<int>(w - sg * p.head_items);
    const int kvh = hi / qgroups;
    const int qh0 = kvh * p.group + (hi - kvh * qgroups) * R;
    // query owning split sg: offsets[qi] <= sg < offsets[qi+1]
    int64_t lo = 0, hi_q = p.nq;
    while (hi_q - lo > 1) {
      const int64_t mid = (lo + hi_q) >> 1;
      if (offsets[mid] <= sg) lo = mid; else hi_q = mid;
    }
    const int64_t qi = lo;
    const int split = static_cast<int>(sg - offsets[qi]);
    const int nsplit = offsets[qi + 1] - offsets[qi];
    const int nk = p.q_nkeys[qi];
    const int sv = p.q_seq[qi];
    const int kb = split * split_pages * ps;
    const int ke = min(nk, kb + split_pages * ps);
    const int n_chunks = (ke - kb + G::CH - 1) / G::CH;
    const int64_t bt_off = p.bt ? int64_t(p.seq_row[sv]) * p.bt_stride : 0;
    const int64_t gstart = p.bt ? 0 : p.seq_start[sv];
    const int npages_seq = (nk + ps - 1) >> p.log2ps;
    const char* kbase = p.k + int64_t(kvh) * row_real;
    const char* vbase = p.v + int64_t(kvh) * row_real;

    // ---- queries of the R grouped heads, pre-scaled into the log2 domain
    float qv[R][G::EPL];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t qoff = (qi * p.hq + qh0 + r) * int64_t(p.d);
#pragma unroll
      for (int n = 0; n < G::NCH; ++n)
#pragma unroll
        for (int e = 0; e < G::CE; ++e) {
          const int d = (lk + n * G::LPK) * G::CE + e;
          if (n * G::CE + e < G::EPL)
            qv[r][n * G::CE + e] = d < p.d ? load_as_float(p.q, qoff + d, p.q_dtype) * p.qscale : 0.f;
        }
    }

    // ---- block-table window: lane i holds the page of logical page win+i
    int win = -1, win_val = 0;
    auto issue = [&](int c) {
      const int stage = c % kStages;
      const int k0 = kb + c * G::CH;
      const int nvalid = min(G::CH, ke - k0);
      int row = 0;
      if (p.bt) {
        const int plo = k0 >> p.log2ps, phi = (k0 + G::CH - 1) >> p.log2ps;
        if (win < 0 || plo < win || phi - win >= 32) {  // warp-uniform
          win = plo;
          const int idx = plo + lane;
          win_val = idx < npages_seq ? p.bt[bt_off + idx] : 0;
        }
        const int key = k0 + lane;
        int src = (key >> p.log2ps) - win;
        src = src < 0 ? 0 : (src > 31 ? 31 : src);
        const int page = __shfl_sync(0xffffffffu, win_val, src);
        row = page * ps + (key & (ps - 1));
      } else {
        row = static_cast<int>(gstart + k0 + lane);
      }
      const uint32_t kdst = wsm_addr + stage * G::STAGE;
      const uint32_t vdst = kdst + G::CH * G::ROWB;
      const int total = G::CH * cpr;
      for (int base = 0; base < total; base += 32) {
        const int i = base + lane;
        const int r = cpr_pow2 ? (i >> cpr_sh) : (i / cpr);
        const int cc = i - r * cpr;
        const int rrow = __shfl_sync(0xffffffffu, row, r & 31);
        if (i < total) {
          const bool ok = r < nvalid;
          const int64_t goff = ok ? int64_t(rrow) * p.row_stride_bytes + cc * vec : 0;
          const uint32_t soff = r * G::ROWB + cc * vec;
          const int nb = ok ? vec : 0;
          if (vec == 16) {
            cp_async<16>(kdst + soff, kbase + goff, nb);
            cp_async<16>(vdst + soff, vbase + goff, nb);
          } else if (vec == 8) {
            cp_async<8>(kdst + soff, kbase + goff, nb);
            cp_async<8>(vdst + soff, vbase + goff, nb);
          } else {
            cp_async<4>(kdst + soff, kbase + goff, nb);
            cp_async<4>(vdst + soff, vbase + goff, nb);
          }
        }
      }
    };

    float m[R], l[R], acc[R][G::EPL];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      m[r] = -INFINITY;
      l[r] = 0.f;
#pragma unroll
      for (int e = 0; e < G::EPL; ++e) acc[r][e] = 0.f;
    }

#pragma unroll
    for (int c = 0; c < kStages - 1; ++c) {
      if (c < n_chunks) issue(c);
      cp_async_commit();
    }
    for (int c = 0; c < n_chunks; ++c) {
      cp_async_wait<kStages - 2>();
      __syncwarp();
      if (c + kStages - 1 < n_chunks) issue(c + kStages - 1);
      cp_async_commit();

      const unsigned char* ks = wsm + (c % kStages) * G::STAGE;
      const unsigned char* vs = ks + G::CH * G::ROWB;
      const int k0 = kb + c * G::CH;
      // scores
      float s[R][G::KPL];
#pragma unroll
      for (int j = 0; j < G::KPL; ++j) {
        const int key = kg + j * G::KG;
        float kf[G::EPL];
#pragma unroll
        for (int n = 0; n < G::NCH; ++n) {
          const uint4 ch = *reinterpret_cast<const uint4*>(ks + key * G::ROWB + (lk + n * G::LPK) * 16);
          Elem<T>::unpack(ch, kf + n * G::CE);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float a = 0.f;
#pragma unroll
          for (int e = 0; e < G::EPL; ++e) a = fmaf(qv[r][e], kf[e], a);
          s[r][j] = a;
        }
      }
#pragma unroll
      for (int o = 1; o < G::LPK; o <<= 1)
#pragma unroll
        for (int j = 0; j < G::KPL; ++j)
#pragma unroll
          for (int r = 0; r < R; ++r) s[r][j] += __shfl_xor_sync(0xffffffffu, s[r][j], o);
      // mask + online softmax (per lane group)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float mx = m[r];
#pragma unroll
        for (int j = 0; j < G::KPL; ++j) {
          if (k0 + kg + j * G::KG >= ke) s[r][j] = -INFINITY;
          mx = fmaxf(mx, s[r][j]);
        }
        if (mx == -INFINITY) {
#pragma unroll
          for (int j = 0; j < G::KPL; ++j) s[r][j] = 0.f;
          continue;
        }
        const float corr = exp2f(m[r] - mx);  // m = -inf -> 0
        float sum = 0.f;
#pragma unroll
        for (int j = 0; j < G::KPL; ++j) {
          s[r][j] = exp2f(s[r][j] - mx);
          sum += s[r][j];
        }
        l[r] = l[r] * corr + sum;
        m[r] = mx;
#pragma unroll
        for (int e = 0; e < G::EPL; ++e) acc[r][e] *= corr;
      }
      // P @ V
#pragma unroll
      for (int j = 0; j < G::KPL; ++j) {
        const int key = kg + j * G::KG;
        float vf[G::EPL];
#pragma unroll
        for (int n = 0; n < G::NCH; ++n) {
          const uint4 ch = *reinterpret_cast<const uint4*>(vs + key * G::ROWB + (lk + n * G::LPK) * 16);
          Elem<T>::unpack(ch, vf + n * G::CE);
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int e = 0; e < G::EPL; ++e) acc[r][e] = fmaf(s[r][j], vf[e], acc[r][e]);
      }
    }
    cp_async_wait<0>();
    __syncwarp();

    // ---- merge the KG lane-group states
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float mx = m[r];
#pragma unroll
      for (int o = G::LPK; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float wgt = m[r] == -INFINITY ? 0.f : exp2f(m[r] - mx);
      l[r] *= wgt;
#pragma unroll
      for (int e = 0; e < G::EPL; ++e) acc[r][e] *= wgt;
#pragma unroll
      for (int o = G::LPK; o < 32; o <<= 1) {
        l[r] += __shfl_xor_sync(0xffffffffu, l[r], o);
#pragma unroll
        for (int e = 0; e < G::EPL; ++e) acc[r][e] += __shfl_xor_sync(0xffffffffu, acc[r][e], o);
      }
      m[r] = mx;
    }
    if (kg == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int qh = qh0 + r;
        if (nsplit == 1) {
          const float inv = 1.f / l[r];
          const int64_t ooff = (qi * p.hq + qh) * int64_t(p.d);
#pragma unroll
          for (int n = 0; n < G::NCH; ++n)
#pragma unroll
            for (int e = 0; e < G::CE; ++e) {
              const int d = (lk + n * G::LPK) * G::CE + e;
              if (n * G::CE + e < G::EPL && d < p.d)
                store_from_float(p.out, ooff + d, p.out_dtype, acc[r][n * G::CE + e] * inv);
            }
        } else {
          const int64_t slot = sg * p.hq + qh;
          if (lk == 0) {
            p.ws_ml[2 * slot] = m[r];
            p.ws_ml[2 * slot + 1] = l[r];
          }
          float* o = p.ws_o + slot * p.d;
#pragma unroll
          for (int n = 0; n < G::NCH; ++n)
#pragma unroll
            for (int e = 0; e < G::CE; ++e) {
              const int d = (lk + n * G::LPK) * G::CE + e;
              if (n * G::CE + e < G::EPL && d < p.d) o[d] = acc[r][n * G::CE + e];
            }
        }
      }
    }
  }
}

// K2c: one warp per (query, q-head) with more than one split; splits merged in
// ascending order (deterministic)
__global__ void combine_kernel(const int32_t* __restrict__ plan, int64_t nq, int hq, int d,
                               const float* __restrict__ ws_ml, const float* __restrict__ ws_o,
                               void* out, int out_dtype) {
  const int lane = threadIdx.x & 31;
  const int64_t item = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (item >= nq * hq) return;
  const int64_t qi = item / hq;
  const int qh = static_cast<int>(item - qi * hq);
  const int32_t* offsets = plan + 4;
  const int s0 = offsets[qi], ns = offsets[qi + 1] - s0;
  if (ns <= 1) return;
  float mx = -INFINITY;
  for (int s = 0; s < ns; ++s) mx = fmaxf(mx, ws_ml[2 * ((int64_t(s0) + s) * hq + qh)]);
  float den = 0.f;
  for (int s = 0; s < ns; ++s) {
    const int64_t slot = (int64_t(s0) + s) * hq + qh;
    den += exp2f(ws_ml[2 * slot] - mx) * ws_ml[2 * slot + 1];
  }
  const float inv = 1.f / den;
  for (int dd = lane; dd < d; dd += 32) {
    float a = 0.f;
    for (int s = 0; s < ns; ++s) {
      const int64_t slot = (int64_t(s0) + s) * hq + qh;
      a += exp2f(ws_ml[2 * slot] - mx) * ws_o[slot * d + dd];
    }
    store_from_float(out, (qi * hq + qh) * int64_t(d) + dd, out_dtype, a * inv);
  }
}

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
using DecodeFn = void (*)(DecodeParams);

template <typename T, int R>
DecodeFn pick_d(int dp) {
  switch (dp) {
    case 4: if constexpr (Elem<T>::kBytes == 4) return decode_kernel<T, 4, R>; else return nullptr;
    case 8: return decode_kernel<T, 8, R>;
    case 16: return decode_kernel<T, 16, R>;
    case 32: return decode_kernel<T, 32, R>;
    case 64: return decode_kernel<T, 64, R>;
    case 128: return decode_kernel<T, 128, R>;
    case 256: return decode_kernel<T, 256, R>;
    default: return nullptr;
  }
}
template <typename T>
DecodeFn pick_r(int r, int dp) {
  if (r == 4) return pick_d<T, 4>(dp);
  if (r == 2) return pick_d<T, 2>(dp);
  return pick_d<T, 1>(dp);
}
template <typename T, int DP, int R>
int stage_bytes_of() { return Geo<T, DP, R>::STAGE; }

template <typename T>
void touch_k2_kernels() {
  cudaFuncAttributes fa;
  for (int r : {1, 2, 4})
    for (int dp : {4, 8, 16, 32, 64, 128, 256})
      if (DecodeFn f = pick_r<T>(r, dp)) cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(f));
}

int ring_bytes(int dtype, int dp) {
  const int s = elem_bytes(dtype);
  const int rowb = dp * s;
  int ch = 4096 / rowb;
  ch = ch > 32 ? 32 : (ch < 4 ? 4 : ch);
  return kStages * 2 * ch * rowb;
}

int g_num_sms = 0;

}  // namespace

extern "C" {

int pkv_device_sm_count(int32_t* out) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    *out = 0;
    return pkv::fail(PKV_CUDA_ERROR, "no CUDA device visible");
  }
  *out = n;
  return PKV_OK;
}

int pkv_mirror_apply(int32_t* table, const int32_t* pairs, int64_t n_pairs, void* stream) {
  if (n_pairs <= 0) return PKV_OK;
  pkv::DeviceGuard guard(static_cast<cudaStream_t>(stream));
  const int threads = 256;
  const int64_t blocks = (n_pairs + threads - 1) / threads;
  mirror_apply_kernel<<<static_cast<unsigned>(blocks < 4096 ? blocks : 4096), threads, 0,
                        static_cast<cudaStream_t>(stream)>>>(table, pairs, n_pairs);
  PKV_CHECK_LAUNCH();
  return PKV_OK;
}

int pkv_page_zero(void* k_cache, void* v_cache, const int32_t* pages, int64_t n,
                  int64_t page_bytes, void* stream) {
  if (n <= 0) return PKV_OK;
  pkv::DeviceGuard guard(static_cast<cudaStream_t>(stream));
  if (page_bytes & 1) return pkv::fail(PKV_CONFIG_ERROR, "page bytes must be even");
  page_zero_kernel<<<static_cast<unsigned>(n < 65535 ? n : 65535), 256, 0,
                     static_cast<cudaStream_t>(stream)>>>(static_cast<char*>(k_cache),
                                                          static_cast<char*>(v_cache), pages, n,
                                                          page_bytes);
  PKV_CHECK_LAUNCH();
  return PKV_OK;
}

int pkv_page_copy(void* k_cache, void* v_cache, const int32_t* triples, int64_t n,
                  int64_t row_bytes, int32_t page_size, void* stream) {
  if (n <= 0) return PKV_OK;
  pkv::DeviceGuard guard(static_cast<cudaStream_t>(stream));
  if (row_bytes & 1) return pkv::fail(PKV_CONFIG_ERROR, "row bytes must be even");
  page_copy_kernel<<<static_cast<unsigned>(n < 65535 ? n : 65535), 256, 0,
                     static_cast<cudaStream_t>(stream)>>>(static_cast<char*>(k_cache),
                                                          static_cast<char*>(v_cache), triples, n,
                                                          row_bytes, page_size, 0, 0, 0);
  PKV_CHECK_LAUNCH();
  return PKV_OK;
}

int pkv_copy_h2d_record(void* dst, const void* src, int64_t bytes, void* event, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  pkv::DeviceGuard guard(st);
  if (bytes > 0) {
    const cudaError_t e = cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return pkv::fail(PKV_CUDA_ERROR, "metadata upload: %s", pkv::cuda_err_str(e));
  }
  if (event) {
    const cudaError_t e = cudaEventRecord(static_cast<cudaEvent_t>(event), st);
    if (e != cudaSuccess) return pkv::fail(PKV_CUDA_ERROR, "metadata upload event: %s", pkv::cuda_err_str(e));
  }
  return PKV_OK;
}

int pkv_event_wait(void* event) {
  if (!event) return PKV_OK;
  cudaError_t e = cudaEventQuery(static_cast<cudaEvent_t>(event));
  if (e == cudaErrorNotReady) e = cudaEventSynchronize(static_cast<cudaEvent_t>(event));
  return e == cudaSuccess ? PKV_OK : pkv::fail(PKV_CUDA_ERROR, "event wait: %s", pkv::cuda_err_str(e));
}

int pkv_page_copy1(void* k_cache, void* v_cache, int64_t src_page, int64_t dst_page, int64_t rows,
                   int64_t row_bytes, int32_t page_size, void* stream) {
  pkv::DeviceGuard guard(static_cast<cudaStream_t>(stream));
  if (row_bytes & 1) return pkv::fail(PKV_CONFIG_ERROR, "row bytes must be even");
  if (src_page < 0 || dst_page < 0 || src_page == dst_page || rows < 0 || rows > page_size)
    return pkv::fail(PKV_VALUE_ERROR, "bad page copy (%lld -> %lld, %lld rows)", static_cast<long long>(src_page),
                     static_cast<long long>(dst_page), static_cast<long long>(rows));
  page_copy_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<char*>(k_cache), static_cast<char*>(v_cache), nullptr, 1, row_bytes, page_size, src_page, dst_page,
      rows);
  PKV_CHECK_LAUNCH();
  return PKV_OK;
}

int pkv_kv_append(const void* k_new, const void* v_new, int64_t n_tok, const int32_t* tok_row,
                  int32_t tok_row_stride, const int32_t* tok_pos, const int32_t* block_table,
                  int64_t bt_stride, int32_t page_size, void* k_cache, void* v_cache,
                  int64_t row_bytes, void* stream) {
  if (n_tok <= 0) return PKV_OK;
  pkv::DeviceGuard guard(static_cast<cudaStream_t>(stream));
  if (page_size <= 0 || (page_size & (page_size - 1)))
    return pkv::fail(PKV_VALUE_ERROR, "page_size must be a power of two");
  if (row_bytes & 1) return pkv::fail(PKV_CONFIG_ERROR, "row bytes must be even");
  auto kern = append_vec(k_new, v_new, k_cache, v_cache, row_bytes) ? kv_append_kernel<true>
                                                                      : kv_append_kernel<false>;
  kern<<<append_blocks(n_tok), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const char*>(k_new), static_cast<const char*>(v_new), n_tok, tok_row,
      tok_row_stride, tok_pos, block_table, bt_stride, __builtin_ctz(page_size),
      static_cast<char*>(k_cache), static_cast<char*>(v_cache), row_bytes, 0, 0);
  PKV_CHECK_LAUNCH();
  return PKV_OK;
}

int pkv_kv_append_range(const void* k_new, const void* v_new, int64_t n_tok, int32_t seq_row, int32_t pos0,
                        const int32_t* block_table, int64_t bt_stride, int32_t page_size, void* k_cache,
                        void* v_cache, int64_t row_bytes, void* stream) {
  if (n_tok <= 0) return PKV_OK;
  if (pos0 < 0 || int64_t(pos0) + n_tok > (int64_t(1) << 31) || seq_row < 0)
    return pkv::fail(PKV_OUT_OF_RANGE, "append range outside int32 positions");
  pkv::DeviceGuard guard(static_cast<cudaStream_t>(stream));
  if (page_size <= 0 || (page_size & (page_size - 1)))
    return pkv::fail(PKV_VALUE_ERROR, "page_size must be a power of two");
  if (row_bytes & 1) return pkv::fail(PKV_CONFIG_ERROR, "row bytes must be even");
  auto kern = append_vec(k_new, v_new, k_cache, v_cache, row_bytes) ? kv_append_kernel<true>
                                                                      : kv_append_kernel<false>;
  kern<<<append_blocks(n_tok), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const char*>(k_new), static_cast<const char*>(v_new), n_tok, nullptr, 0, nullptr, block_table,
      bt_stride, __builtin_ctz(page_size), static_cast<char*>(k_cache), static_cast<char*>(v_cache), row_bytes,
      pos0, seq_row);
  PKV_CHECK_LAUNCH();
  return PKV_OK;
}

int pkv_kv_assign(pkv_pool* pool, int64_t seq, const int64_t* positions, int64_t n, int64_t* info_out,
                  int64_t* copies_out, int64_t copies_cap, int64_t* n_copies_out, const void* k_new,
                  const void* v_new, const int32_t* block_table, int64_t bt_stride, int32_t page_size,
                  void* k_cache, void* v_cache, int64_t row_bytes, void* stream, int32_t* launched_out) {
  if (!launched_out) return pkv::fail(PKV_VALUE_ERROR, "bad assign inputs");
  *launched_out = 0;
  int st = pkv_pool_assign_prepare(pool, seq, positions, n, info_out, copies_out, copies_cap, n_copies_out);
  if (st || n <= 0 || !block_table) return st;
  const int64_t want = PKV_ASSIGN_INCREASING | PKV_ASSIGN_CONTIGUOUS;
  if (info_out[2] != want || *n_copies_out != 0) return PKV_OK;
  int64_t pending = 0;
  int32_t full = 0;
  st = pkv_pool_mirror_pending(pool, &pending, &full);
  if (st || pending || full) return st;  // the caller brings the mirror up to date first
  if (info_out[0] >= (int64_t(1) << 31)) return PKV_OK;
  st = pkv_kv_append_range(k_new, v_new, n, static_cast<int32_t>(info_out[4]), static_cast<int32_t>(info_out[0]),
                           block_table, bt_stride, page_size, k_cache, v_cache, row_bytes,
                           stream);
  if (st) return st;
  *launched_out = 1;
  int64_t len = 0;
  st = pkv_pool_get_logical_len(pool, seq, &len);
  if (st) return st;
  if (info_out[1] + 1 > len) st = pkv_pool_set_logical_len(pool, seq, info_out[1] + 1);
  return st;
}

int pkv_kv_gather(const void* k_cache, const void* v_cache, const int32_t* block_table, int64_t bt_stride,
                  const int32_t* seq_row, const int32_t* cu_rows, int64_t n_seq, int64_t n_rows,
                  int32_t page_size, int64_t row_bytes, void* k_out, void* v_out, void* stream) {
  if (n_seq <= 0 || n_rows <= 0) return PKV_OK;
  if (page_size <= 0 || (page_size & (page_size - 1)))
    return pkv::fail(PKV_VALUE_ERROR, "page_size must be a power of two");
  if (row_bytes & 1) return pkv::fail(PKV_CONFIG_ERROR, "row bytes must be even");
  if (n_seq >= (int64_t(1) << 31) || n_rows >= (int64_t(1) << 31))
    return pkv::fail(PKV_CONFIG_ERROR, "gather of more than 2^31 rows");
  pkv::DeviceGuard guard(static_cast<cudaStream_t>(stream));
  const int threads = 256;
  const int64_t want = (n_rows + 7) / 8;
  const int64_t blocks = want < 148 * 16 ? want : 148 * 16;
  kv_gather_kernel<<<static_cast<unsigned>(blocks), threads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const char*>(k_cache), static_cast<const char*>(v_cache), block_table, bt_stride, seq_row,
      cu_rows, static_cast<int>(n_seq), __builtin_ctz(page_size), row_bytes, static_cast<char*>(k_out),
      static_cast<char*>(v_out));
  PKV_CHECK_LAUNCH();
  return PKV_OK;
}

int64_t pkv_attention_workspace_bytes(int64_t n_queries, int32_t hq, int32_t head_dim) {
  const int64_t splits = n_queries + kMaxExtraSplits;
  auto up = [](int64_t x) { return (x + 255) / 256 * 256; };
  const int64_t plan = 4 * (4 + n_queries + 1);
  return up(plan) + up(4 * splits * hq * 2) + up(4 * splits * hq * head_dim);
}

}  // extern "C"

// The allocator half of a decode step plus its metadata; on success *undo
// holds the allocator's undo record (the caller commits or rolls it back),
// on failure the allocator is unchanged.
static int decode_step_prepare(pkv_pool* pool, const int64_t* seqs, int64_t n, int32_t page_size,
                               int32_t hq, int32_t hkv, int32_t head_dim, int32_t* meta, int64_t meta_cap,
                               int64_t* meta_used, uint32_t* pages_out, int64_t pages_cap,
                               int64_t* n_pages_out, int64_t* copies_out, pkv_append_undo** undo) {
  *undo = nullptr;
  if (n <= 0) return pkv::fail(PKV_VALUE_ERROR, "no sequences");
  if (meta_cap < 3 * n + pkv_attention_plan_ints(n, hq))
    return pkv::fail(PKV_VALUE_ERROR, "metadata buffer too small");
  int32_t* q_seq = meta;
  int32_t* nkeys = meta + n;
  int32_t* rows = meta + 2 * n;
  // positions land in nkeys[] and become key counts (the appended token is attended)
  int st = pkv_pool_prepare_append_undo(pool, seqs, n, nkeys, rows, pages_out, pages_cap, n_pages_out,
                                        copies_out, undo);
  if (st) return st;
  for (int64_t i = 0; i < n; ++i) {
    q_seq[i] = static_cast<int32_t>(i);
    nkeys[i] += 1;
  }
  int64_t used = 0;
  st = pkv_attention_plan_d(nkeys, rows, n, page_size, hq, hkv, head_dim, 0, 0, meta + 3 * n,
                          meta_cap - 3 * n, &used);
  if (st) {
    pkv_pool_rollback_append(pool, *undo);
    *undo = nullptr;
    return st;
  }
  *meta_used = 3 * n + used;
  return PKV_OK;
}

extern "C" int pkv_decode_step_prepare(pkv_pool* pool, const int64_t* seqs, int64_t n, int32_t page_size,
                                       int32_t hq, int32_t hkv, int32_t* meta, int64_t meta_cap,
                                       int64_t* meta_used, uint32_t* pages_out, int64_t pages_cap,
                                       int64_t* n_pages_out, int64_t* copies_out) {
  pkv_append_undo* undo = nullptr;
  const int st = decode_step_prepare(pool, seqs, n, page_size, hq, hkv, 128, meta, meta_cap, meta_used, pages_out,
                                     pages_cap, n_pages_out, copies_out, &undo);
  pkv_pool_release_undo(undo);
  return st;
}

// host-side phase stamps of the last pkv_decode_step on this thread
// (pkv_debug_step_times): steady-clock ns since the call's entry
namespace {
thread_local int64_t t_stamp[12];
thread_local std::chrono::steady_clock::time_point t_stamp0;
inline void stamp(int i) {
  t_stamp[i] = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t_stamp0).count();
}
}  // namespace

extern "C" int pkv_debug_step_times(int64_t* out, int32_t n) {
  t_stamp[11] = std::chrono::duration_cast<std::chrono::nanoseconds>(t_stamp0.time_since_epoch()).count();
  for (int i = 0; i < n && i < 12; ++i) out[i] = t_stamp[i];
  return PKV_OK;
}

// side blocks behind the plan: granted pages, copy triples, mirror pairs, the
// zero list and the per-store cache pointer table (up to kMaxStageStores)
constexpr int64_t kMaxStageStores = 256;
static int64_t stage_extra(int64_t n) { return 24 * n + 4 * kMaxStageStores + 64; }

extern "C" int64_t pkv_decode_step_stage_ints(int64_t n, int32_t hq) {
  return 3 * n + pkv_attention_plan_ints(n, hq) + stage_extra(n);
}

static int decode_step_stage(pkv_step_stage_args* a, cudaStream_t stream, pkv_append_undo** undo);

extern "C" int pkv_decode_step_stage(pkv_step_stage_args* a, void* stream_) {
  pkv::DeviceGuard guard(static_cast<cudaStream_t>(stream_));
  pkv_append_undo* undo = nullptr;
  const int st = decode_step_stage(a, static_cast<cudaStream_t>(stream_), &undo);
  pkv_pool_release_undo(undo);
  return st;
}

// On failure the allocator is rolled back (the reference's all-or-nothing
// contract: pool.py:143-148, 165-169); on success *undo is the caller's.
static int decode_step_stage(pkv_step_stage_args* a, cudaStream_t stream, pkv_append_undo** undo) {
  *undo = nullptr;
  if (!a || !a->pool) return pkv::fail(PKV_VALUE_ERROR, "null args");
  a->meta_used = 0;
  a->needs_resync = 0;
  a->launches = 0;
  if (a->slot_event) {  // the slot's previous upload has landed (a query first: it almost always has)
    cudaError_t e = cudaEventQuery(static_cast<cudaEvent_t>(a->slot_event));
    if (e == cudaErrorNotReady) e = cudaEventSynchronize(static_cast<cudaEvent_t>(a->slot_event));
    if (e != cudaSuccess) return pkv::fail(PKV_CUDA_ERROR, "slot event: %s", pkv::cuda_err_str(e));
  }
  stamp(2);
  const int64_t n = a->n;
  const int64_t extra = stage_extra(n);
  if (a->n_stores > kMaxStageStores)
    return pkv::fail(PKV_CONFIG_ERROR, "more than %d stores on one pool", static_cast<int>(kMaxStageStores));
  if (a->meta_cap < 3 * n + pkv_attention_plan_ints(n, a->hq) + extra)
    return pkv::fail(PKV_VALUE_ERROR, "metadata slot too small");
  // 1) allocator + attention metadata + plan
  std::vector<uint32_t> pages(2 * n + 1);
  std::vector<int64_t> copies(2 * n);
  int64_t n_pages = 0, used = 0;
  // head dim for the planner's byte costs: 16-bit rows of hkv heads (the
  // tensor-core path the plan feeds), 128 when no store is attached
  const int32_t head_dim = a->row_bytes > 0 ? static_cast<int32_t>(a->row_bytes / (2 * a->hkv)) : 128;
  int st = decode_step_prepare(a->pool, a->seqs, n, a->page_size, a->hq, a->hkv, head_dim, a->meta_host,
                               a->meta_cap - extra, &used, pages.data(), static_cast<int64_t>(pages.size()),
                               &n_pages, copies.data(), undo);
  if (st) return st;
  stamp(3);
  // from here on a failure restores the allocator before returning
  auto fail_back = [&](int code) {
    pkv_pool_rollback_append(a->pool, *undo);
    *undo = nullptr;
    return code;
  };
  // 2) side blocks behind it: granted pages | copy triples | mirror pairs |
  //    zero list (granted minus copy destinations) | cache pointers
  int32_t* side = a->meta_host + used;
  int64_t off = 0;
  const int64_t pages_off = used + off;
  for (int64_t i = 0; i < n_pages; ++i) side[off++] = static_cast<int32_t>(pages[i]);
  const int64_t trip_off = used + off;
  int64_t n_copies = 0;
  for (int64_t i = 0; i < n; ++i)
    if (copies[2 * i + 1] >= 0) {
      side[off++] = static_cast<int32_t>(copies[2 * i]);
      side[off++] = static_cast<int32_t>(copies[2 * i + 1]);
      side[off++] = a->page_size;
      ++n_copies;
    }
  int64_t rows = 0, cols = 0, pending = 0, n_pairs = 0;
  int32_t full = 0;
  pkv_pool_mirror_shape(a->pool, &rows, &cols);
  pkv_pool_mirror_pending(a->pool, &pending, &full);
  const int64_t aux_ints = n_pages + 4 * int64_t(a->n_stores) + 1;  // zero list + pointer table + alignment
  const int64_t room = (a->meta_cap - used - off - aux_ints) / 2;
  const bool mirror_ok = a->mirror_dev && !full && rows == a->mirror_rows && cols == a->mirror_cols && pending <= room;
  const int64_t pairs_off = used + off;
  if (mirror_ok && pending) {
    pkv_pool_mirror_drain(a->pool, side + off, room, &n_pairs, &full);
    off += 2 * n_pairs;
  }
  a->needs_resync = mirror_ok ? 0 : 1;
  const bool page_work = a->n_stores > 0 && (n_pages || n_copies);
  int64_t zero_off = 0, n_zero = 0, ptr_off = 0;
  if (page_work) {
    zero_off = used + off;
    for (int64_t i = 0; i < n_pages; ++i) {
      bool is_dst = false;
      for (int64_t c = 0; c < n_copies && !is_dst; ++c) is_dst = side[trip_off - used + 3 * c + 1] == side[i];
      if (!is_dst) side[off++] = side[i];
    }
    n_zero = used + off - zero_off;
    if ((used + off) & 1) side[off++] = 0;  // 8-byte alignment of the pointer table
    ptr_off = used + off;
    for (int32_t st2 = 0; st2 < a->n_stores; ++st2) {
      const uint64_t kp = reinterpret_cast<uint64_t>(a->k_caches[st2]);
      const uint64_t vp = reinterpret_cast<uint64_t>(a->v_caches[st2]);
      std::memcpy(side + off, &kp, 8);
      std::memcpy(side + off + 2, &vp, 8);
      off += 4;
    }
  }
  // 3) one upload of everything, then ONE page / mirror kernel
  stamp(4);
  const int64_t total = used + off;
  if (total > a->meta_cap) return fail_back(pkv::fail(PKV_VALUE_ERROR, "metadata slot too small"));
  if (page_work && (a->row_bytes & 1)) return fail_back(pkv::fail(PKV_CONFIG_ERROR, "row bytes must be even"));
  if (pkv_debug_should_fail(PKV_FAIL_STEP_UPLOAD))
    return fail_back(pkv::fail(PKV_CUDA_ERROR, "step metadata upload: injected failure"));
  const bool recording = pkv::launch_recorder() != nullptr;  // CUDA-graph mode: record, do not issue
  if (recording && pkv::graph_copies()) {
    pkv::record_copy(a->meta_dev, a->meta_host, static_cast<size_t>(total) * 4);
    if (a->slot_event) pkv::record_event(static_cast<cudaEvent_t>(a->slot_event));
  } else {
    cudaError_t e = cudaMemcpyAsync(a->meta_dev, a->meta_host, static_cast<size_t>(total) * 4,
                                    cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess)
      return fail_back(pkv::fail(PKV_CUDA_ERROR, "step metadata upload: %s", pkv::cuda_err_str(e)));
    if (a->slot_event) cudaEventRecord(static_cast<cudaEvent_t>(a->slot_event), stream);
  }
  stamp(5);
  if (page_work || n_pairs) {
    const int n_st = page_work ? a->n_stores : 0;
    const int64_t blocks = std::max<int64_t>(n_st * (n_zero + n_copies), (n_pairs + 255) / 256);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(std::max<int64_t>(blocks, 1), 65535));
    const uint64_t* caches = reinterpret_cast<const uint64_t*>(a->meta_dev + ptr_off);
    const int32_t* zero_p = a->meta_dev + zero_off;
    const int32_t* trip_p = a->meta_dev + trip_off;
    const int32_t* pairs_p = a->meta_dev + pairs_off;
    const int ps = a->page_size;
    if (recording)
      pkv::record_kernel(step_aux_kernel, dim3(grid), dim3(256), 0u, 1u, caches, n_st, zero_p, n_zero, trip_p,
                         n_copies, a->mirror_dev, pairs_p, n_pairs, a->row_bytes, ps);
    else
      step_aux_kernel<<<grid, 256, 0, stream>>>(caches, n_st, zero_p, n_zero, trip_p, n_copies, a->mirror_dev,
                                                pairs_p, n_pairs, a->row_bytes, ps);
    const cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) return fail_back(pkv::fail(PKV_CUDA_ERROR, "step aux kernel: %s", pkv::cuda_err_str(le)));
    ++a->launches;
  }
  stamp(6);
  a->meta_used = used;
  a->n_granted = n_pages;
  a->granted_off = pages_off;
  a->n_copies = n_copies;
  a->copies_off = trip_off;
  return PKV_OK;
}

extern "C" {

int pkv_paged_attention(const pkv_attention_args* a, void* stream_) {
  if (!a) return pkv::fail(PKV_VALUE_ERROR, "null args");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  pkv::DeviceGuard guard(stream);
  if (a->meta_host && a->meta_bytes > 0) {  // stage the packed metadata (pinned host -> device)
    if (!a->meta_dev) return pkv::fail(PKV_VALUE_ERROR, "meta_host without meta_dev");
    cudaError_t e = cudaMemcpyAsync(a->meta_dev, a->meta_host, static_cast<size_t>(a->meta_bytes),
                                    cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return pkv::fail(PKV_CUDA_ERROR, "metadata upload: %s", pkv::cuda_err_str(e));
  }
  if (a->n_queries <= 0) return PKV_OK;
  if (a->hq <= 0 || a->hkv <= 0 || a->hq % a->hkv)
    return pkv::fail(PKV_SHAPE_MISMATCH, "query heads (%d) must be a multiple of kv heads (%d)",
                     a->hq, a->hkv);
  if (a->page_size <= 0 || (a->page_size & (a->page_size - 1)))
    return pkv::fail(PKV_VALUE_ERROR, "page_size must be a power of two");
  if (a->n_queries > (int64_t(1) << 30)) return pkv::fail(PKV_CONFIG_ERROR, "too many queries");
  if (a->k_new && !a->block_table)
    return pkv::fail(PKV_VALUE_ERROR, "fused append needs the paged (block-table) source");
  const int s = elem_bytes(a->kv_dtype);
  if (a->head_dim <= 0 || a->head_dim > 256 || (a->head_dim * s) % 4)
    return pkv::fail(PKV_CONFIG_ERROR,
                     "head_dim %d unsupported (need 1..256 with head_dim*elem_size %% 4 == 0)",
                     a->head_dim);
  if (a->workspace_bytes < pkv_attention_workspace_bytes(a->n_queries, a->hq, a->head_dim))
    return pkv::fail(PKV_VALUE_ERROR, "workspace too small");
  if (!g_num_sms) {
    int32_t n = 0;
    pkv_device_sm_count(&n);
    g_num_sms = n > 0 ? n : 148;
  }
  const int num_sms = a->num_sms > 0 ? a->num_sms : g_num_sms;
  const int waves = a->target_waves > 0 ? a->target_waves : 4;
  const int group = a->hq / a->hkv;
  const int log2ps = __builtin_ctz(a->page_size);

  auto up = [](int64_t x) { return (x + 255) / 256 * 256; };
  char* ws = static_cast<char*>(a->workspace);
  int32_t* plan = reinterpret_cast<int32_t*>(ws);
  const int64_t splits = a->n_queries + kMaxExtraSplits;
  const int64_t plan_bytes = 4 * (4 + a->n_queries + 1);
  float* ws_ml = reinterpret_cast<float*>(reinterpret_cast<char*>(plan) + up(plan_bytes));
  float* ws_o = reinterpret_cast<float*>(reinterpret_cast<char*>(ws_ml) + up(4 * splits * a->hq * 2));

  const bool tc_ok = decode_tc_supported(a->kv_dtype, a->head_dim);
  bool use_tc = a->mode == 2 || (a->mode == 0 && a->kv_dtype == PKV_BF16);
  if (use_tc && !tc_ok) {
    if (a->mode == 2)
      return pkv::fail(PKV_CONFIG_ERROR, "tensor-core decode needs a 16-bit cache and head_dim 64/128");
    use_tc = false;
  }

  if (use_tc) {
    if (!a->plan || !a->plan_host)
      return pkv::fail(PKV_VALUE_ERROR, "tensor-core decode needs the pkv_attention_plan() plan");
    if (a->plan_host[7] != a->n_queries)
      return pkv::fail(PKV_VALUE_ERROR, "plan was built for %d queries, call has %lld", a->plan_host[7],
                       static_cast<long long>(a->n_queries));
    if (reinterpret_cast<uintptr_t>(a->out) % 16)
      return pkv::fail(PKV_VALUE_ERROR, "attention output must be 16-byte aligned (vector stores)");
    TcParams t;
    t.q = a->q;
    t.q_dtype = a->q_dtype;
    t.nq = static_cast<int>(a->n_queries);
    t.k = static_cast<const char*>(a->k_cache);
    t.v = static_cast<const char*>(a->v_cache);
    t.kw = static_cast<char*>(const_cast<void*>(a->k_cache));
    t.vw = static_cast<char*>(const_cast<void*>(a->v_cache));
    t.k_new = static_cast<const char*>(a->k_new);
    t.v_new = static_cast<const char*>(a->v_new);
    t.bt = a->block_table;
    t.bt_stride = a->bt_stride;
    t.log2ps = log2ps;
    t.hq = a->hq;
    t.hkv = a->hkv;
    t.group = group;
    t.row_stride = int64_t(a->hkv) * a->head_dim * 2;
    t.qscale = a->scale * kLog2e;
    t.out = a->out;
    t.out_dtype = a->out_dtype;
    t.plan = a->plan;
    t.ws_ml = ws_ml;
    t.ws_o = ws_o;
    if (a->prof_start) cudaEventRecord(static_cast<cudaEvent_t>(a->prof_start), stream);
    const int st = launch_decode_tc(t, a->plan_host, a->kv_dtype, a->head_dim, num_sms, stream);
    if (st != PKV_OK) return st;
    if (a->prof_stop) cudaEventRecord(static_cast<cudaEvent_t>(a->prof_stop), stream);
    return PKV_OK;
  }

  // ---- fp32 CUDA-core path (exact; the reference's 1e-5 contract) ----------
  int dp = 4;
  while (dp < a->head_dim) dp *= 2;
  if (dp * s < 16) dp = 16 / s;
  const int r = group % 4 == 0 ? 4 : (group % 2 == 0 ? 2 : 1);
  DecodeFn fn = a->kv_dtype == PKV_F32    ? pick_r<float>(r, dp)
                : a->kv_dtype == PKV_BF16 ? pick_r<__nv_bfloat16>(r, dp)
                                          : pick_r<__half>(r, dp);
  if (!fn) return pkv::fail(PKV_CONFIG_ERROR, "no decode kernel for dtype %d head_dim %d",
                            a->kv_dtype, a->head_dim);
  if (a->k_new) {
    // unfused append of the decode tokens (positions q_nkeys-1)
    const int64_t row_bytes = int64_t(a->hkv) * a->head_dim * s;
    int threads = static_cast<int>(row_bytes / 16);
    threads = threads < 32 ? 32 : (threads > 256 ? 256 : ((threads + 31) / 32) * 32);
    append_decode_kernel<<<static_cast<unsigned>(a->n_queries < 65535 ? a->n_queries : 65535), threads, 0,
                           stream>>>(static_cast<const char*>(a->k_new), static_cast<const char*>(a->v_new),
                                     a->n_queries, a->q_seq, a->q_nkeys, a->seq_row, a->block_table,
                                     a->bt_stride, log2ps, static_cast<char*>(const_cast<void*>(a->k_cache)),
                                     static_cast<char*>(const_cast<void*>(a->v_cache)), row_bytes);
    PKV_CHECK_LAUNCH();
  }
  const int head_items = a->hkv * (group / r);
  plan_kernel<<<1, kPlanThreads, 0, stream>>>(a->q_nkeys, a->n_queries, log2ps, head_items,
                                              int64_t(num_sms) * kWarps * waves, plan);
  PKV_CHECK_LAUNCH();

  DecodeParams p;
  p.q = a->q;
  p.q_dtype = a->q_dtype;
  p.nq = a->n_queries;
  p.q_seq = a->q_seq;
  p.q_nkeys = a->q_nkeys;
  p.k = static_cast<const char*>(a->k_cache);
  p.v = static_cast<const char*>(a->v_cache);
  p.bt = a->block_table;
  p.bt_stride = a->bt_stride;
  p.seq_row = a->seq_row;
  p.seq_start = a->seq_start;
  p.log2ps = log2ps;
  p.hq = a->hq;
  p.hkv = a->hkv;
  p.d = a->head_dim;
  p.group = group;
  p.head_items = head_items;
  p.row_stride_bytes = int64_t(a->hkv) * a->head_dim * s;
  p.qscale = a->scale * kLog2e;
  p.out = a->out;
  p.out_dtype = a->out_dtype;
  p.plan = plan;
  p.ws_ml = ws_ml;
  p.ws_o = ws_o;
  const int smem = kWarps * ring_bytes(a->kv_dtype, dp);
  static bool attr_set[3][9][3] = {};
  int di = __builtin_ctz(dp), ri = r == 4 ? 2 : (r == 2 ? 1 : 0);
  if (!attr_set[a->kv_dtype][di][ri]) {
    cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_set[a->kv_dtype][di][ri] = true;
  }
  if (a->prof_start) cudaEventRecord(static_cast<cudaEvent_t>(a->prof_start), stream);
  fn<<<num_sms, kWarps * 32, smem, stream>>>(p);
  PKV_CHECK_LAUNCH();
  if (a->prof_stop) cudaEventRecord(static_cast<cudaEvent_t>(a->prof_stop), stream);
  const int64_t items = a->n_queries * a->hq;
  const int per_block = 8;
  combine_kernel<<<static_cast<unsigned>((items + per_block - 1) / per_block), per_block * 32, 0,
                   stream>>>(plan, a->n_queries, a->hq, a->head_dim, ws_ml, ws_o, a->out,
                             a->out_dtype);
  PKV_CHECK_LAUNCH();
  return PKV_OK;
}

static void plan_speculate(const int32_t* nk, const int32_t* row, int64_t n, int32_t ps, int32_t hq, int32_t hkv,
                           int32_t head_dim);

int pkv_decode_step(pkv_step_stage_args* stage, pkv_attention_args* attn, pkv_decode_io* io, void* stream_) {
  if (!stage || !attn) return pkv::fail(PKV_VALUE_ERROR, "null args");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  t_stamp0 = std::chrono::steady_clock::now();
  pkv::DeviceGuard guard(stream);
  stamp(0);
  if (io) io->launched = io->launches = 0;
  // the input copies go first so they overlap the host-side allocator / plan
  auto h2d = [&](const void* src, const void* dst, int64_t bytes, const char* what) -> int {
    if (!src) return PKV_OK;
    if (!dst || bytes <= 0) return pkv::fail(PKV_VALUE_ERROR, "%s: host source without device buffer", what);
    if (pkv::launch_recorder() && pkv::graph_copies()) {
      pkv::record_copy(const_cast<void*>(dst), src, static_cast<size_t>(bytes));
      return PKV_OK;
    }
    cudaError_t e = cudaMemcpyAsync(const_cast<void*>(dst), src, static_cast<size_t>(bytes),
                                    cudaMemcpyHostToDevice, stream);
    return e == cudaSuccess ? PKV_OK : pkv::fail(PKV_CUDA_ERROR, "%s upload: %s", what, pkv::cuda_err_str(e));
  };
  if (io) {
    int st = h2d(io->q_host, attn->q, io->q_bytes, "q");
    if (!st) st = h2d(io->k_host, attn->k_new, io->kv_bytes, "k_new");
    if (!st) st = h2d(io->v_host, attn->v_new, io->kv_bytes, "v_new");
    if (st) return st;
  }
  stamp(1);
  pkv_append_undo* undo = nullptr;
  int st = decode_step_stage(stage, stream, &undo);
  if (st) return st;
  // a failure past the stage puts the allocator back (all-or-nothing step)
  auto fail_back = [&](int code) {
    pkv_pool_rollback_append(stage->pool, undo);
    return code;
  };
  if (stage->n_stores == 0 && (stage->n_granted || stage->n_copies))
    return fail_back(pkv::fail(PKV_VALUE_ERROR, "decode step needs the stores attached for page clears / copies"));
  if (io) io->launches = stage->launches;
  const int64_t n = stage->n;
  int32_t* md = stage->meta_dev;
  attn->n_queries = n;
  attn->q_seq = md;
  attn->q_nkeys = md + n;
  attn->seq_row = md + 2 * n;
  attn->plan = md + 3 * n;
  attn->plan_host = stage->meta_host + 3 * n;
  attn->meta_host = nullptr;
  attn->meta_bytes = 0;
  // block-table shape changed: the caller re-exports the mirror, points
  // attn->block_table at it and launches pkv_paged_attention(attn) itself
  if (stage->needs_resync) {
    pkv_pool_release_undo(undo);
    return PKV_OK;
  }
  if (pkv_debug_should_fail(PKV_FAIL_STEP_LAUNCH))
    return fail_back(pkv::fail(PKV_CUDA_ERROR, "decode launch: injected failure"));
  stamp(7);
  st = pkv_paged_attention(attn, stream_);
  if (st) return fail_back(st);
  stamp(8);
  pkv_pool_release_undo(undo);
  const bool tensor = attn->mode == 2 || (attn->mode == 0 && attn->kv_dtype == PKV_BF16);
  if (io) {
    io->launches += tensor ? 1 : 4;
    if (io->out_host) {
      if (io->out_bytes <= 0) return pkv::fail(PKV_VALUE_ERROR, "out_host without out_bytes");
      cudaError_t e = cudaMemcpyAsync(io->out_host, attn->out, static_cast<size_t>(io->out_bytes),
                                      cudaMemcpyDeviceToHost, stream);
      if (e != cudaSuccess) return pkv::fail(PKV_CUDA_ERROR, "output download: %s", pkv::cuda_err_str(e));
    }
    io->launched = 1;
  }
  // the next step's plan, computed while the GPU runs this one
  stamp(9);
  if (tensor)
    plan_speculate(stage->meta_host + n, stage->meta_host + 2 * n, n, attn->page_size, attn->hq, attn->hkv,
                   attn->head_dim);
  stamp(10);
  return PKV_OK;
}

}  // extern "C"

extern "C" int64_t pkv_attention_plan_ints(int64_t n_queries, int32_t hq) {
  return pkv::decode_plan_ints(n_queries, hq);
}

// Plan memo (host, per thread): the decode plan is a pure function of its
// inputs, and a serving loop asks for the plan of (key counts + 1) right after
// launching the current step.  pkv_decode_step computes that next plan while
// the GPU runs the current one (plan_speculate); the next prepare finds it here
// and copies it instead of recomputing, taking the planner off the critical path.
namespace {
struct PlanMemo {
  std::vector<int32_t> key, plan;
};
thread_local PlanMemo t_memo;
thread_local std::vector<int32_t> t_key;

void plan_key(std::vector<int32_t>& k, const int32_t* nk, const int32_t* row, int64_t n, int32_t ps,
              int32_t hq, int32_t hkv, int32_t d, int32_t sms, int32_t waves, int32_t bump) {
  k.resize(static_cast<size_t>(2 * n + 7));
  k[0] = static_cast<int32_t>(n);
  k[1] = ps;
  k[2] = hq;
  k[3] = hkv;
  k[4] = sms;
  k[5] = waves;
  k[6] = d;
  for (int64_t i = 0; i < n; ++i) {
    k[7 + i] = nk[i] + bump;
    k[7 + n + i] = row[i];
  }
}
}  // namespace

static int resolve_sms(int32_t num_sms) {
  if (num_sms > 0) return num_sms;
  if (!g_num_sms) {
    int32_t n = 0;
    pkv_device_sm_count(&n);
    g_num_sms = n > 0 ? n : 148;
  }
  return g_num_sms;
}

// compute and memoise the plan of the next decode step (every key count + 1)
static void plan_speculate(const int32_t* nk, const int32_t* row, int64_t n, int32_t ps, int32_t hq,
                           int32_t hkv, int32_t head_dim) {
  const int sms = resolve_sms(0);
  PlanMemo& m = t_memo;
  plan_key(m.key, nk, row, n, ps, hq, hkv, head_dim, sms, 0, 1);
  m.plan.resize(static_cast<size_t>(pkv::decode_plan_ints(n, hq)));
  std::vector<int32_t> nk1(m.key.begin() + 7, m.key.begin() + 7 + n);
  int64_t used = 0;
  if (pkv::plan_decode(nk1.data(), row, n, ps, hq, hkv, head_dim, sms, 0, m.plan.data(),
                       static_cast<int64_t>(m.plan.size()), &used) != PKV_OK) {
    m.key.clear();
    return;
  }
  m.plan.resize(static_cast<size_t>(used));
}

extern "C" void pkv_plan_memo_reset(void) {
  t_memo.key.clear();
  t_memo.plan.clear();
}

extern "C" int pkv_attention_plan_d(const int32_t* q_nkeys, const int32_t* q_row, int64_t n_queries,
                                    int32_t page_size, int32_t hq, int32_t hkv, int32_t head_dim, int32_t num_sms,
                                    int32_t target_waves, int32_t* plan_out, int64_t cap, int64_t* n_out) {
  if (n_queries > 0 && hq > 0 && hkv > 0 && !t_memo.key.empty()) {
    plan_key(t_key, q_nkeys, q_row, n_queries, page_size, hq, hkv, head_dim, resolve_sms(num_sms), target_waves,
             0);
    if (t_key == t_memo.key && cap >= static_cast<int64_t>(t_memo.plan.size())) {
      std::copy(t_memo.plan.begin(), t_memo.plan.end(), plan_out);
      if (n_out) *n_out = static_cast<int64_t>(t_memo.plan.size());
      return PKV_OK;
    }
  }
  if (n_queries <= 0) return pkv::fail(PKV_VALUE_ERROR, "no queries");
  if (hq <= 0 || hkv <= 0 || hq % hkv) return pkv::fail(PKV_SHAPE_MISMATCH, "bad head counts");
  if (page_size <= 0 || (page_size & (page_size - 1)))
    return pkv::fail(PKV_VALUE_ERROR, "page_size must be a power of two");
  if (num_sms <= 0) {
    if (!g_num_sms) {
      int32_t n = 0;
      pkv_device_sm_count(&n);
      g_num_sms = n > 0 ? n : 148;
    }
    num_sms = g_num_sms;
  }
  return pkv::plan_decode(q_nkeys, q_row, n_queries, page_size, hq, hkv, head_dim, num_sms,
                          target_waves, plan_out, cap, n_out);
}

extern "C" int pkv_attention_plan(const int32_t* q_nkeys, const int32_t* q_row, int64_t n_queries,
                                  int32_t page_size, int32_t hq, int32_t hkv, int32_t num_sms,
                                  int32_t target_waves, int32_t* plan_out, int64_t cap, int64_t* n_out) {
  return pkv_attention_plan_d(q_nkeys, q_row, n_queries, page_size, hq, hkv, 128, num_sms, target_waves,
                              plan_out, cap, n_out);
}

extern "C" int pkv_debug_trace(int32_t enable, uint64_t* out, int64_t n) {
  return pkv::debug_trace(enable, out, n);
}

namespace pkv {
void preload_kernels() {
  static std::atomic<uint64_t> done{0};  // one bit per device ordinal (< 64)
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    cudaGetLastError();
    return;
  }
  const uint64_t bit = uint64_t(1) << dev;
  if (done.load(std::memory_order_acquire) & bit) return;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (done.load(std::memory_order_relaxed) & bit) return;
  cudaFuncAttributes fa;
  auto touch = [&](const void* f) { cudaFuncGetAttributes(&fa, f); };
  touch(reinterpret_cast<const void*>(mirror_apply_kernel));
  touch(reinterpret_cast<const void*>(page_zero_kernel));
  touch(reinterpret_cast<const void*>(page_copy_kernel));
  touch(reinterpret_cast<const void*>(step_aux_kernel));
  touch(reinterpret_cast<const void*>(kv_append_kernel<true>));
  touch(reinterpret_cast<const void*>(kv_append_kernel<false>));
  touch(reinterpret_cast<const void*>(kv_gather_kernel));
  touch(reinterpret_cast<const void*>(append_decode_kernel));
  touch(reinterpret_cast<const void*>(plan_kernel));
  touch(reinterpret_cast<const void*>(combine_kernel));
  touch_k2_kernels<float>();
  touch_k2_kernels<__nv_bfloat16>();
  touch_k2_kernels<__half>();
  preload_decode_tc_kernels();
  preload_prefill_kernels();
  cudaGetLastError();  // a query failure only means that kernel loads lazily
  done.fetch_or(bit, std::memory_order_release);
}
}  // namespace pkv
