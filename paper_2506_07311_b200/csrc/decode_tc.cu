// K2-TC: split-K paged decode on the tensor cores (mma.sync m16n8k16, bf16 /
// fp16 operands, fp32 accumulation) for 16-bit KV caches.
//
// Replaces the reference streaming kernel (attention.py:259-329) for bf16
// stores.  Decode is HBM bound (GQA-4 bf16: 4 flop/B, far below the ridge), so
// the tensor cores are used to cut *issue* cost, not for FLOPs: the CUDA-core
// kernel spends ~1200 instructions per 8 KiB chunk on unpacking, FMA chains
// and shuffles; here a 16-key chunk costs 16 HMMA + 16 LDSM + the softmax.
// tcgen05 is not used: M = G <= 16 query rows is not a dense contraction and
// the TMEM round trip would cost more than it saves.
//
// Work decomposition.  A work item is (query, kv head, group of <= 16 query
// heads, key split) and is processed by a whole CTA (8 warps, one CTA per SM):
// warp w takes the item's 16-key chunks w, w+8, w+16, ...  and the 8 partial
// softmax states are merged through shared memory at the end of the item, so
// the number of *global* splits per query is 8x smaller than with warp items
// and small batches do not drown in split merges.  The item list is planned
// on the device from the per-query key counts (even page ranges per split,
// at least kMinSplitChunks chunks per split), sorted by item size and dealt
// to CTAs in snake order (LPT-style balance), so each CTA knows its whole item
// sequence up front.  That lets every warp run a *producer* that streams its
// chunks through a private 3-stage cp.async ring (16-byte XOR swizzle ->
// conflict-free LDSM; zero-fill past the valid keys) straight across item
// boundaries: the next item's pages are in flight while the current one
// merges.  The G grouped query heads are the M rows of the MMA, so every K/V
// byte is read from HBM once per group.
//
// Numerics: scores accumulate unscaled in fp32 and the softmax scale (times
// log2 e) is folded into the exp2 argument; P is rounded to the operand type
// for the P@V MMA and the denominator sums the *rounded* P.  fp32 queries are
// split hi+lo into two MMAs (fp32-accurate scores).
//
// Splits of one query are merged by the last CTA to finish (acq_rel atomic
// counters that self-reset), in ascending split order: deterministic, and no
// combine launch.  Optional fused append: with k_new/v_new the last split of
// each query reads the new token from the input and writes it into its page
// (reshape-and-cache folded into the decode launch).
#include "common.cuh"
#include "decode_tc.h"

namespace pkv {
namespace {

constexpr int kWarpsTc = 8;
constexpr int kThreadsTc = kWarpsTc * 32;
constexpr int kStagesTc = 3;
constexpr int kCh = 16;              // keys per chunk
constexpr int kMinSplitChunks = 16;  // >= 2 chunks per warp per item
constexpr int kMergeRows = 4;        // rows per CTA-merge pass
constexpr int kMaxPending = 128;     // queued split merges per CTA

struct Item {
  int qi, hi, kvh, qh0, rows, split, nsplit, kb, ke, nchunks, nk, row, slot;
  bool valid;
};

// Debug timeline (pkv_debug_trace): per CTA, globaltimer stamps of
// [start, plan done, item k consumer start..., item k merged..., end].
constexpr int kTraceSlots = 64;
}  // namespace
// external linkage + volatile reads: the flag is only ever written by the host
__device__ unsigned long long g_trace[1024 * 64];
__device__ volatile int g_trace_on;
namespace {

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace(int slot) {
  if (g_trace_on && threadIdx.x == 0 && slot < kTraceSlots && blockIdx.x < 1024)
    g_trace[blockIdx.x * kTraceSlots + slot] = gtimer();
}

// Plan arrays (shared memory, or global for large query counts).
struct PlanView {
  const int32_t* nk;      // [nq] key counts
  const int32_t* row;     // [nq] mirror row (paged) / first row (gathered)
  const int32_t* order;   // [nq] queries sorted by split size (desc)
  const int32_t* nsplit;  // [nq]
  const int32_t* ioff;    // [nq + 1] item offsets over the sorted queries
  const int32_t* soff;    // [nq + 1] split-slot offsets by query index
  int64_t total_items;
};

// ---------------------------------------------------------------------------
// Block-wide planner (used in-CTA for small query counts and by the plan
// kernel otherwise).  `keys` is scratch for the sort: 2 * nq_pow2 int64.
// ---------------------------------------------------------------------------
__device__ void plan_block(const TcParams& p, int32_t* nk, int32_t* row, int32_t* order,
                           int32_t* nsplit, int32_t* ioff, int32_t* soff, long long* keys,
                           int nq_pow2, long long* red, int* hdr) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int ps = 1 << p.log2ps;
  long long pages = 0;
  for (int i = tid; i < p.nq; i += nt) {
    const int n = p.q_nkeys[i];
    const int sv = p.q_seq[i];
    nk[i] = n;
    row[i] = p.bt ? p.seq_row[sv] : static_cast<int>(p.seq_start[sv]);
    pages += (n + ps - 1) >> p.log2ps;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) pages += __shfl_xor_sync(0xffffffffu, pages, o);
  if (lane == 0) red[warp] = pages;
  __syncthreads();
  if (tid == 0) {
    long long tot = 0;
    for (int w = 0; w < nw; ++w) tot += red[w];
    long long sp = (tot * p.head_items + p.target_items - 1) / p.target_items;
    const long long min_sp = (int64_t(kMinSplitChunks) * kCh + ps - 1) / ps;
    const long long cap = (tot + kMaxExtraSplitsTc - 1) / kMaxExtraSplitsTc;
    sp = sp < min_sp ? min_sp : sp;
    sp = sp < cap ? cap : sp;
    red[0] = sp;
  }
  __syncthreads();
  const long long sp = red[0];
  // sort key: (split size desc, query asc); padding sorts last
  for (int i = tid; i < nq_pow2; i += nt) {
    long long key = 0x7fffffffffffffffLL;
    if (i < p.nq) {
      const long long pg = (nk[i] + ps - 1) >> p.log2ps;
      const long long ns = (pg + sp - 1) / sp;
      nsplit[i] = static_cast<int32_t>(ns);
      const long long size = (pg + ns - 1) / ns;
      key = ((0x7fffffffLL - size) << 32) | i;
    }
    keys[i] = key;
  }
  __syncthreads();
  if (nq_pow2 <= 32) {
    // small batches: bitonic sort inside warp 0 with shuffles (no barriers)
    if (warp == 0) {
      long long x = lane < nq_pow2 ? keys[lane] : 0x7fffffffffffffffLL;
      for (int k = 2; k <= 32; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
          const long long y = __shfl_xor_sync(0xffffffffu, x, j);
          const bool up = (lane & k) == 0;
          const bool lower = (lane & j) == 0;
          x = (lower == up) ? (x < y ? x : y) : (x < y ? y : x);
        }
      }
      if (lane < nq_pow2) keys[lane] = x;
    }
    __syncthreads();
  }
  for (int k = 2; nq_pow2 > 32 && k <= nq_pow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < nq_pow2; i += nt) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const long long a = keys[i], b = keys[ixj];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            keys[i] = b;
            keys[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = tid; i < p.nq; i += nt) order[i] = static_cast<int32_t>(keys[i] & 0xffffffff);
  __syncthreads();
  // two exclusive scans: items over the sorted order, split slots by index
  int carry_i = 0, carry_s = 0;
  int* scan = reinterpret_cast<int*>(red);  // 2 * nw ints
  for (int base = 0; base < p.nq; base += nt) {
    const int i = base + tid;
    int ci = 0, cs = 0;
    if (i < p.nq) {
      ci = nsplit[order[i]] * p.head_items;
      cs = nsplit[i];
    }
    int xi = ci, xs = cs;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int yi = __shfl_up_sync(0xffffffffu, xi, o);
      const int ys = __shfl_up_sync(0xffffffffu, xs, o);
      if (lane >= o) {
        xi += yi;
        xs += ys;
      }
    }
    if (lane == 31) {
      scan[warp] = xi;
      scan[nw + warp] = xs;
    }
    __syncthreads();
    int bi = 0, bs = 0, ai = 0, as = 0;
    for (int w = 0; w < nw; ++w) {
      const int vi = scan[w], vs = scan[nw + w];
      if (w < warp) {
        bi += vi;
        bs += vs;
      }
      ai += vi;
      as += vs;
    }
    if (i < p.nq) {
      ioff[i] = carry_i + bi + xi - ci;
      soff[i] = carry_s + bs + xs - cs;
    }
    carry_i += ai;
    carry_s += as;
    __syncthreads();
  }
  if (tid == 0) {
    ioff[p.nq] = carry_i;
    soff[p.nq] = carry_s;
    hdr[0] = carry_i;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(1024) plan_tc_kernel(const __grid_constant__ TcParams p, int32_t* g,
                                                        long long* keys, int nq_pow2) {
  __shared__ long long red[32];
  __shared__ int hdr[1];
  const int nq = p.nq;
  plan_block(p, g + 4, g + 4 + nq, g + 4 + 2 * nq, g + 4 + 3 * nq, g + 4 + 4 * nq,
             g + 4 + 5 * nq + 1, keys, nq_pow2, red, hdr);
  if (threadIdx.x == 0) g[0] = hdr[0];
}

__device__ __forceinline__ Item make_item(int64_t gidx, const PlanView& pv, const TcParams& p) {
  Item it;
  it.valid = gidx < pv.total_items;
  if (!it.valid) return it;
  const int gi = static_cast<int>(gidx);
  int lo = 0, hi = p.nq;  // sorted position j with ioff[j] <= gi < ioff[j+1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pv.ioff[mid] <= gi) lo = mid; else hi = mid;
  }
  const int q = pv.order[lo];
  const int rem = gi - pv.ioff[lo];
  it.qi = q;
  it.split = rem / p.head_items;
  it.hi = rem - it.split * p.head_items;
  it.kvh = it.hi / p.qgroups;
  const int qg = it.hi - it.kvh * p.qgroups;
  it.qh0 = it.kvh * p.group + qg * 16;
  it.rows = min(16, p.group - qg * 16);
  it.nsplit = pv.nsplit[q];
  it.nk = pv.nk[q];
  it.row = pv.row[q];
  it.slot = pv.soff[q] + it.split;
  const int ps = 1 << p.log2ps;
  const int pages = (it.nk + ps - 1) >> p.log2ps;
  int p0, p1;
  if (it.nsplit == 1) {
    p0 = 0;
    p1 = pages;
  } else if (pages < 65536) {  // 32-bit division (64-bit is emulated)
    p0 = static_cast<int>((static_cast<unsigned>(it.split) * pages) / static_cast<unsigned>(it.nsplit));
    p1 = static_cast<int>((static_cast<unsigned>(it.split + 1) * pages) / static_cast<unsigned>(it.nsplit));
  } else {
    p0 = static_cast<int>((int64_t(it.split) * pages) / it.nsplit);
    p1 = static_cast<int>((int64_t(it.split + 1) * pages) / it.nsplit);
  }
  it.kb = p0 * ps;
  it.ke = min(it.nk, p1 * ps);
  it.nchunks = (it.ke - it.kb + kCh - 1) / kCh;
  return it;
}

// Merge the nsplit partials (m, l, unnormalised O) of one (query, head group)
// by the whole CTA, in ascending split order.  Split weights are computed once
// into shared memory (`scratch`, >= 2*rows*nsplit + rows floats when it fits;
// otherwise recomputed per element), then every thread accumulates float4
// slices of O with 8 independent loads in flight.
template <int D>
__device__ void merge_global(const TcParams& p, const Item& C, int64_t out_base, float* scratch) {
  const int ns = C.nsplit, rows = C.rows, s0 = C.slot - C.split;
  const float2* ml = reinterpret_cast<const float2*>(p.ws_ml);
  const bool staged = rows * ns * 2 + rows <= kWarpsTc * kMergeRows * D;
  float* s_w = scratch;                // [rows][ns] weights
  float* s_inv = scratch + rows * ns;  // [rows] 1 / denominator
  if (staged) {
    for (int e = threadIdx.x; e < rows * ns; e += kThreadsTc) {
      const int r = e / ns, s = e - r * ns;
      const float2 v = __ldcg(ml + (int64_t(s0 + s) * p.hq + C.qh0 + r));
      s_w[e] = v.x;
      s_w[rows * ns + rows + e] = v.y;
    }
    __syncthreads();
    for (int r = threadIdx.x >> 5; r < rows; r += kWarpsTc) {  // one warp per row
      const int lane = threadIdx.x & 31;
      float mx = -INFINITY;
      for (int s = lane; s < ns; s += 32) mx = fmaxf(mx, s_w[r * ns + s]);
#pragma unroll
      for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      float den = 0.f;
      for (int s = lane; s < ns; s += 32) {
        const float w = exp2f(s_w[r * ns + s] - mx);
        den += w * s_w[rows * ns + rows + r * ns + s];
        s_w[r * ns + s] = w;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
      if (lane == 0) s_inv[r] = 1.f / den;
    }
    __syncthreads();
  }
  constexpr int V = D / 4;  // float4 slices per row
  for (int e = threadIdx.x; e < rows * V; e += kThreadsTc) {
    const int r = e / V, dv = e - r * V;
    const int64_t col = C.qh0 + r;
    float mx = 0.f, inv = 0.f;
    if (!staged) {
      mx = -INFINITY;
      for (int s = 0; s < ns; ++s) mx = fmaxf(mx, __ldcg(ml + (int64_t(s0 + s) * p.hq + col)).x);
      float den = 0.f;
      for (int s = 0; s < ns; ++s) {
        const float2 v = __ldcg(ml + (int64_t(s0 + s) * p.hq + col));
        den += exp2f(v.x - mx) * v.y;
      }
      inv = 1.f / den;
    } else {
      inv = s_inv[r];
    }
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int sb = 0; sb < ns; sb += 8) {
      float4 ov[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        ov[u] = sb + u < ns ? __ldcg(reinterpret_cast<const float4*>(p.ws_o + (int64_t(s0 + sb + u) * p.hq + col) * D) + dv)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (sb + u >= ns) break;
        const float w = staged ? s_w[r * ns + sb + u]
                               : exp2f(__ldcg(ml + (int64_t(s0 + sb + u) * p.hq + col)).x - mx);
        acc.x += w * ov[u].x;
        acc.y += w * ov[u].y;
        acc.z += w * ov[u].z;
        acc.w += w * ov[u].w;
      }
    }
    const int64_t off = out_base + int64_t(r) * D + 4 * dv;
    store_from_float(p.out, off, p.out_dtype, acc.x * inv);
    store_from_float(p.out, off + 1, p.out_dtype, acc.y * inv);
    store_from_float(p.out, off + 2, p.out_dtype, acc.z * inv);
    store_from_float(p.out, off + 3, p.out_dtype, acc.w * inv);
  }
}

// One warp merges the 8 per-warp states of an item (rows <= kMergeRows) from
// shared memory, in warp order, and writes the output row (single split) or
// the item's global split partial.
template <int D>
__device__ void warp_merge_item(const TcParams& p, const Item& C, int64_t out_base, const float* s_mo,
                                const float* s_ml, int lane, int* s_sync, int k) {
  constexpr int E = D / 32;  // elements per lane per row
  float acc[kMergeRows][E];
  float rmx[kMergeRows], rden[kMergeRows];
  // 1) read all slots into registers (warp order: deterministic)
#pragma unroll
  for (int r = 0; r < kMergeRows; ++r) {
    if (r >= C.rows) break;
    float mw[kWarpsTc];
    float mx = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarpsTc; ++w) {
      mw[w] = s_ml[(w * kMergeRows + r) * 2];
      mx = fmaxf(mx, mw[w]);
    }
    float den = 0.f;
#pragma unroll
    for (int w = 0; w < kWarpsTc; ++w) {
      mw[w] = mw[w] == -INFINITY ? 0.f : exp2f(mw[w] - mx);
      den += mw[w] * s_ml[(w * kMergeRows + r) * 2 + 1];
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      float a = 0.f;
#pragma unroll
      for (int w = 0; w < kWarpsTc; ++w) a += mw[w] * s_mo[(w * kMergeRows + r) * D + lane + 32 * e];
      acc[r][e] = a;
    }
    rmx[r] = mx;
    rden[r] = den;
  }
  // 2) release the slots before touching global memory
  __syncwarp();
  if (lane == 0) {
    s_sync[0] = 0;
    *reinterpret_cast<volatile int*>(&s_sync[1]) = k + 1;
  }
  // 3) output row (single split) or the item's global split partial
#pragma unroll
  for (int r = 0; r < kMergeRows; ++r) {
    if (r >= C.rows) break;
    const int64_t slot = int64_t(C.slot) * p.hq + C.qh0 + r;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int d = lane + 32 * e;
      if (C.nsplit == 1)
        store_from_float(p.out, out_base + int64_t(r) * D + d, p.out_dtype, acc[r][e] / rden[r]);
      else
        __stcg(p.ws_o + slot * D + d, acc[r][e]);
    }
    if (C.nsplit > 1 && lane == 0) __stcg(reinterpret_cast<float2*>(p.ws_ml) + slot, make_float2(rmx[r], rden[r]));
  }
}

// Single-warp split merge (overflow fallback of the queued CTA merges).
template <int D>
__device__ void merge_global_warp(const TcParams& p, const Item& C, int64_t out_base, int lane) {
  const int s0 = C.slot - C.split;
  const float2* ml = reinterpret_cast<const float2*>(p.ws_ml);
  for (int r = 0; r < C.rows; ++r) {
    const int64_t col = C.qh0 + r;
    float mx = -INFINITY;
    for (int s = lane; s < C.nsplit; s += 32) mx = fmaxf(mx, __ldcg(ml + (int64_t(s0 + s) * p.hq + col)).x);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float den = 0.f;
    for (int s = lane; s < C.nsplit; s += 32) {
      const float2 v = __ldcg(ml + (int64_t(s0 + s) * p.hq + col));
      den += exp2f(v.x - mx) * v.y;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
    for (int d = lane; d < D; d += 32) {
      float acc = 0.f;
      for (int s = 0; s < C.nsplit; ++s) {
        const int64_t slot = int64_t(s0 + s) * p.hq + col;
        acc += exp2f(__ldcg(ml + slot).x - mx) * __ldcg(p.ws_o + slot * D + d);
      }
      store_from_float(p.out, out_base + int64_t(r) * D + d, p.out_dtype, acc / den);
    }
  }
}

// k-th item of CTA b in snake order over the size-sorted item list
__device__ __forceinline__ int64_t item_of(int b, int64_t k, int G) {
  return k * G + ((k & 1) ? (G - 1 - b) : b);
}

template <typename T, int D, bool SPLITQ, bool ROWS16>
__global__ void __launch_bounds__(kThreadsTc, 1) decode_tc_kernel(const __grid_constant__ TcParams p) {
  constexpr int ROWB = D * 2;            // smem row bytes
  constexpr int CPR = ROWB / 16;         // 16-B chunks per row (8 or 16)
  constexpr int RPI = 32 / CPR;          // rows per copy iteration
  constexpr int NIT = kCh / RPI;         // copy iterations per chunk
  constexpr int STAGE = 2 * kCh * ROWB;  // K + V
  constexpr int KS = D / 16;             // k-steps of Q K^T
  constexpr int NT = D / 8;              // n-tiles of P V
  static_assert(CPR >= 8 && CPR <= 32, "D must be 64 or 128");

  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ long long s_red[32];
  __shared__ int s_hdr[2];
  __shared__ int s_sync[3];  // arrivals of the current item, items merged, queued merges
  __shared__ long long s_pend[kMaxPending];
  if (threadIdx.x < 3) s_sync[threadIdx.x] = 0;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  trace(0);
  const int ps = 1 << p.log2ps;
  float* s_mo = reinterpret_cast<float*>(smem + p.merge_offset);             // [W][4][D]
  float* s_ml = s_mo + kWarpsTc * kMergeRows * D;                            // [W][4][2]

  // ---------------- plan -------------------------------------------------
  PlanView pv;
  if (p.plan_global) {
    const int nq = p.nq;
    const int32_t* g = p.plan_global;
    pv.nk = g + 4;
    pv.row = g + 4 + nq;
    pv.order = g + 4 + 2 * nq;
    pv.nsplit = g + 4 + 3 * nq;
    pv.ioff = g + 4 + 4 * nq;
    pv.soff = g + 4 + 5 * nq + 1;
    pv.total_items = g[0];
  } else {
    int32_t* base = reinterpret_cast<int32_t*>(smem);
    const int nq = p.nq;
    int32_t *nk = base, *row = nk + nq, *order = row + nq, *ns = order + nq, *ioff = ns + nq,
            *soff = ioff + nq + 1;
    int nq_pow2 = 1;
    while (nq_pow2 < nq) nq_pow2 <<= 1;
    // the sort scratch lives in the (not yet used) merge buffer
    plan_block(p, nk, row, order, ns, ioff, soff, reinterpret_cast<long long*>(s_mo), nq_pow2, s_red,
               s_hdr);
    pv.nk = nk;
    pv.row = row;
    pv.order = order;
    pv.nsplit = ns;
    pv.ioff = ioff;
    pv.soff = soff;
    pv.total_items = s_hdr[0];
  }
  __syncthreads();
  trace(1);
  const int G = gridDim.x;
  const int b = blockIdx.x;

  unsigned char* ring = smem + p.ring_offset + warp * (kStagesTc * STAGE);
  const uint32_t ring_addr = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  const int t4 = lane & 3, g = lane >> 2;
  unsigned* merge_cnt = p.counters + 2;

  // ======================= producer (per warp) ===========================
  const int cc = lane % CPR, r0 = lane / CPR;  // copy geometry of this lane
  Item P;
  int64_t pk = 0;  // producer item counter (within this CTA's sequence)
  int pc = 0;      // next chunk of P to issue (warp-strided)
  int win = -1, win_val = 0;
  auto start_item = [&]() {
    for (;;) {
      P = make_item(item_of(b, pk, G), pv, p);
      pc = warp;
      win = -1;
      if (!P.valid) return;
      if (warp == 0) {
        // warm L2 with the item's query rows: every warp's consumer loads them
        // at item start, after this warp's prefetched pages
        const int qe = p.q_dtype == PKV_F32 ? 4 : 2;
        const char* qrow = static_cast<const char*>(p.q) + (int64_t(P.qi) * p.hq + P.qh0) * D * qe;
        if (lane * 128 < P.rows * D * qe) asm volatile("prefetch.global.L2 [%0];" ::"l"(qrow + lane * 128));
      }
      if (warp == 0 && p.k_new != nullptr && P.split == P.nsplit - 1) {
        // fused append: write the new token's head slice into its page
        const int pos = P.nk - 1;
        const int64_t page = p.bt[int64_t(P.row) * p.bt_stride + (pos >> p.log2ps)];
        const int64_t dst = (page * ps + (pos & (ps - 1))) * p.row_stride + int64_t(P.kvh) * ROWB;
        const int64_t src = (int64_t(P.qi) * p.hkv + P.kvh) * ROWB;
        if (lane < CPR) {
          reinterpret_cast<uint4*>(p.kw + dst)[lane] = reinterpret_cast<const uint4*>(p.k_new + src)[lane];
          reinterpret_cast<uint4*>(p.vw + dst)[lane] = reinterpret_cast<const uint4*>(p.v_new + src)[lane];
        }
      }
      if (pc < P.nchunks) return;
      ++pk;  // this warp has no chunk in the item: skip it
    }
  };

  long long gissue = 0;
  auto issue_next = [&]() {
    if (P.valid) {
      const int stage = static_cast<int>(gissue % kStagesTc);
      const int k0 = P.kb + pc * kCh;
      const int nvalid = min(kCh, P.ke - k0);
      int rowidx = 0;  // cache row of key k0 + lane (lane < kCh)
      if (p.bt) {
        const int plo = k0 >> p.log2ps, phi = (k0 + kCh - 1) >> p.log2ps;
        if (win < 0 || plo < win || phi - win >= 32) {
          win = plo;
          const int idx = plo + lane;
          const int npages = (P.nk + ps - 1) >> p.log2ps;
          win_val = idx < npages ? p.bt[int64_t(P.row) * p.bt_stride + idx] : 0;
        }
        const int key = k0 + lane;
        int src = (key >> p.log2ps) - win;
        src = src < 0 ? 0 : (src > 31 ? 31 : src);
        const int page = __shfl_sync(0xffffffffu, win_val, src);
        rowidx = page * ps + (key & (ps - 1));
      } else {
        rowidx = P.row + k0 + lane;
      }
      const bool fuse = p.k_new != nullptr && P.split == P.nsplit - 1;
      const int64_t head_off = int64_t(P.kvh) * ROWB;
      const int64_t new_off = (int64_t(P.qi) * p.hkv + P.kvh) * ROWB + cc * 16;
      const uint32_t kdst = ring_addr + stage * STAGE;
      const uint32_t vdst = kdst + kCh * ROWB;
#pragma unroll
      for (int it = 0; it < NIT; ++it) {
        const int r = r0 + it * RPI;
        const int rw = __shfl_sync(0xffffffffu, rowidx, r);
        const bool ok = r < nvalid;
        const char* ks_ = p.k + int64_t(rw) * p.row_stride + head_off + cc * 16;
        const char* vs_ = p.v + int64_t(rw) * p.row_stride + head_off + cc * 16;
        if (fuse && k0 + r == P.nk - 1) {
          ks_ = p.k_new + new_off;
          vs_ = p.v_new + new_off;
        }
        const uint32_t soff = r * ROWB + ((cc ^ (r & 7)) << 4);
        cp_async<16>(kdst + soff, ok ? ks_ : p.k, ok ? 16 : 0);
        cp_async<16>(vdst + soff, ok ? vs_ : p.v, ok ? 16 : 0);
      }
      ++gissue;
      pc += kWarpsTc;
      if (pc >= P.nchunks) {
        ++pk;
        start_item();
      }
    }
    cp_async_commit();
  };

  start_item();
#pragma unroll
  for (int i = 0; i < kStagesTc - 1; ++i) issue_next();

  // ======================= consumer ======================================
  long long gcons = 0;
  const float qscale = p.qscale;
  for (int64_t k = 0;; ++k) {
    const Item C = make_item(item_of(b, k, G), pv, p);
    if (!C.valid) break;
    trace(2 + 3 * int(k));

    float o[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

    if (warp < C.nchunks) {
      // Q fragments (A operand), unscaled
      uint32_t qa[KS][4];
      uint32_t qb[SPLITQ ? KS : 1][4];
      {
        const int64_t qbase = int64_t(C.qi) * p.hq + C.qh0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int row = g + ((h & 1) ? 8 : 0);
            const int d = ks * 16 + ((h & 2) ? 8 : 0) + 2 * t4;
            const bool in = row < C.rows;
            const int64_t off = (qbase + row) * D + d;
            if constexpr (SPLITQ) {
              float2 x = in ? *reinterpret_cast<const float2*>(static_cast<const float*>(p.q) + off)
                            : make_float2(0.f, 0.f);
              qa[ks][h] = pack2<T>(x.x, x.y);
              qb[ks][h] = pack2<T>(x.x - round_to<T>(x.x), x.y - round_to<T>(x.y));
            } else {
              if (p.q_dtype == p.kv_dtype) {
                qa[ks][h] = in ? *reinterpret_cast<const uint32_t*>(static_cast<const uint16_t*>(p.q) + off) : 0u;
              } else {
                const float x0 = in ? load_as_float(p.q, off, p.q_dtype) : 0.f;
                const float x1 = in ? load_as_float(p.q, off + 1, p.q_dtype) : 0.f;
                qa[ks][h] = pack2<T>(x0, x1);
              }
            }
          }
        }
      }

      for (int c = warp; c < C.nchunks; c += kWarpsTc) {
        cp_async_wait<kStagesTc - 2>();
        __syncwarp();
        issue_next();
        const uint32_t kbase = ring_addr + static_cast<int>(gcons % kStagesTc) * STAGE;
        const uint32_t vbase = kbase + kCh * ROWB;
        ++gcons;

        // S = Q K^T for 16 keys: two n-tiles; even/odd k-steps accumulate
        // separately to halve the dependent HMMA chain
        float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
        {
          float e0[4] = {0.f, 0.f, 0.f, 0.f}, e1[4] = {0.f, 0.f, 0.f, 0.f};
          const int m = lane >> 3;
          const int key = ((m >> 1) << 3) + (lane & 7);
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            const int chunk = 2 * ks + (m & 1);
            uint32_t b00, b01, b10, b11;
            ldmatrix_x4(kbase + key * ROWB + ((chunk ^ (key & 7)) << 4), b00, b01, b10, b11);
            float* a0 = (ks & 1) ? e0 : s0;
            float* a1 = (ks & 1) ? e1 : s1;
            mma_16816<T>(a0, qa[ks], b00, b01);
            mma_16816<T>(a1, qa[ks], b10, b11);
            if constexpr (SPLITQ) {
              mma_16816<T>(a0, qb[ks], b00, b01);
              mma_16816<T>(a1, qb[ks], b10, b11);
            }
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            s0[i] += e0[i];
            s1[i] += e1[i];
          }
        }
        // mask keys beyond the split
        const int lim = C.ke - (C.kb + c * kCh + 2 * t4);  // key offsets e valid iff e < lim
        if (lim < 10) {
          if (lim <= 0) s0[0] = s0[2] = -INFINITY;
          if (lim <= 1) s0[1] = s0[3] = -INFINITY;
          if (lim <= 8) s1[0] = s1[2] = -INFINITY;
          if (lim <= 9) s1[1] = s1[3] = -INFINITY;
        }
        // online softmax in the log2 domain: p = 2^(s*qscale - m)
        float mx0 = fmaxf(fmaxf(s0[0], s0[1]), fmaxf(s1[0], s1[1]));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
        const float mn0 = fmaxf(m0, mx0 * qscale);
        const float c0 = exp2f(m0 - mn0);
        m0 = mn0;
        uint32_t pa[4];
        {
          const float p00 = exp2f(fmaf(s0[0], qscale, -mn0)), p01 = exp2f(fmaf(s0[1], qscale, -mn0));
          const float p10 = exp2f(fmaf(s1[0], qscale, -mn0)), p11 = exp2f(fmaf(s1[1], qscale, -mn0));
          pa[0] = pack2<T>(p00, p01);
          pa[2] = pack2<T>(p10, p11);
          l0 = l0 * c0 + (unpack_sum<T>(pa[0]) + unpack_sum<T>(pa[2]));
        }
        float c1 = 1.f;
        if constexpr (ROWS16) {
          float mx1 = fmaxf(fmaxf(s0[2], s0[3]), fmaxf(s1[2], s1[3]));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
          const float mn1 = fmaxf(m1, mx1 * qscale);
          c1 = exp2f(m1 - mn1);
          m1 = mn1;
          const float p02 = exp2f(fmaf(s0[2], qscale, -mn1)), p03 = exp2f(fmaf(s0[3], qscale, -mn1));
          const float p12 = exp2f(fmaf(s1[2], qscale, -mn1)), p13 = exp2f(fmaf(s1[3], qscale, -mn1));
          pa[1] = pack2<T>(p02, p03);
          pa[3] = pack2<T>(p12, p13);
          l1 = l1 * c1 + (unpack_sum<T>(pa[1]) + unpack_sum<T>(pa[3]));
        } else {
          pa[1] = pa[3] = 0u;
        }
        // rescale O only when some row's running max moved
        if (!__all_sync(0xffffffffu, c0 == 1.f && c1 == 1.f)) {
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            o[n][0] *= c0;
            o[n][1] *= c0;
            if constexpr (ROWS16) {
              o[n][2] *= c1;
              o[n][3] *= c1;
            }
          }
        }
        // O += P V
        {
          const int m = lane >> 3;
          const int key = ((m & 1) << 3) + (lane & 7);
#pragma unroll
          for (int np = 0; np < NT / 2; ++np) {
            const int chunk = 2 * np + (m >> 1);
            uint32_t b0, b1, b2, b3;
            ldmatrix_x4_trans(vbase + key * ROWB + ((chunk ^ (key & 7)) << 4), b0, b1, b2, b3);
            mma_16816<T>(o[2 * np], pa, b0, b1);
            mma_16816<T>(o[2 * np + 1], pa, b2, b3);
          }
        }
      }
      // quad-reduce the denominators (each lane summed its own keys)
      l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
      l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
      if constexpr (ROWS16) {
        l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
        l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
      }
    }

    trace(3 + 3 * int(k));
    const int64_t out_base = (int64_t(C.qi) * p.hq + C.qh0) * D;

    if (C.rows <= kMergeRows) {
      // ---- asynchronous CTA merge: each warp publishes its state into its
      // shared-memory slot and moves on to its next item; the last warp to
      // arrive merges the 8 slots in warp order (deterministic).  A warp only
      // overwrites its slot after the previous item's merge released it.
      if (k > 0) {
        if (lane == 0)
          while (*reinterpret_cast<volatile int*>(&s_sync[1]) < static_cast<int>(k)) __nanosleep(32);
        __syncwarp();
      }
      if (g < C.rows) {
        float* dst = s_mo + (warp * kMergeRows + g) * D;
#pragma unroll
        for (int n = 0; n < NT; ++n) *reinterpret_cast<float2*>(dst + n * 8 + 2 * t4) = make_float2(o[n][0], o[n][1]);
        if (t4 == 0) {
          s_ml[(warp * kMergeRows + g) * 2] = m0;
          s_ml[(warp * kMergeRows + g) * 2 + 1] = l0;
        }
      }
      // the warp barrier orders the lanes' shared stores before lane 0's
      // shared atomic; shared memory is coherent within the SM, and no
      // __threadfence_block here: MEMBAR would also wait for this warp's
      // in-flight cp.async prefetches of the next item
      __syncwarp();
      int last = 0;
      if (lane == 0) last = atomicAdd(&s_sync[0], 1) == kWarpsTc - 1;
      last = __shfl_sync(0xffffffffu, last, 0);
      trace(4 + 3 * int(k));
      if (last) {
        warp_merge_item<D>(p, C, out_base, s_mo, s_ml, lane, s_sync, static_cast<int>(k));
        if (C.nsplit > 1) {
          // publish the global partial; the last CTA of this (query, head
          // group) queues the split merge for the end of the kernel
          __syncwarp();
          int overflow = 0;
          if (lane == 0) {
            const unsigned prev =
                atom_inc_acq_rel(merge_cnt + (int64_t(C.qi) * p.head_items + C.hi), C.nsplit - 1);
            if (prev == static_cast<unsigned>(C.nsplit - 1)) {
              const int idx = atomicAdd(&s_sync[2], 1);
              if (idx < kMaxPending) s_pend[idx] = item_of(b, k, G); else overflow = 1;
            }
          }
          overflow = __shfl_sync(0xffffffffu, overflow, 0);
          if (overflow) merge_global_warp<D>(p, C, out_base, lane);
        }
      }
      continue;
    }

    // ---- synchronous CTA merge (more than kMergeRows rows), kMergeRows per pass
    for (int rb = 0; rb < C.rows; rb += kMergeRows) {
      // publish this warp's rows [rb, rb + 4)
      {
        const int rl = (rb < 8 ? g : g + 8) - rb;  // local row of this lane's fragment
        const bool mine = rl >= 0 && rl < kMergeRows;
        if (mine) {
          float* dst = s_mo + (warp * kMergeRows + rl) * D;
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            const float x0 = rb < 8 ? o[n][0] : o[n][2];
            const float x1 = rb < 8 ? o[n][1] : o[n][3];
            *reinterpret_cast<float2*>(dst + n * 8 + 2 * t4) = make_float2(x0, x1);
          }
          if (t4 == 0) {
            s_ml[(warp * kMergeRows + rl) * 2] = rb < 8 ? m0 : m1;
            s_ml[(warp * kMergeRows + rl) * 2 + 1] = rb < 8 ? l0 : l1;
          }
        }
      }
      __syncthreads();
      const int nrows = min(kMergeRows, C.rows - rb);
      for (int e = threadIdx.x; e < nrows * D; e += kThreadsTc) {
        const int rl = e / D, d = e - rl * D;
        float mx = -INFINITY;
#pragma unroll
        for (int w = 0; w < kWarpsTc; ++w) mx = fmaxf(mx, s_ml[(w * kMergeRows + rl) * 2]);
        float den = 0.f, acc = 0.f;
#pragma unroll
        for (int w = 0; w < kWarpsTc; ++w) {
          const float mw = s_ml[(w * kMergeRows + rl) * 2];
          const float wgt = mw == -INFINITY ? 0.f : exp2f(mw - mx);
          den += wgt * s_ml[(w * kMergeRows + rl) * 2 + 1];
          acc += wgt * s_mo[(w * kMergeRows + rl) * D + d];
        }
        if (C.nsplit == 1) {
          store_from_float(p.out, out_base + int64_t(rb + rl) * D + d, p.out_dtype, acc / den);
        } else {
          const int64_t slot = int64_t(C.slot) * p.hq + C.qh0 + rb + rl;
          __stcg(p.ws_o + slot * D + d, acc);
          if (d == 0) __stcg(reinterpret_cast<float2*>(p.ws_ml) + slot, make_float2(mx, den));
        }
      }
      __syncthreads();
    }
    trace(4 + 3 * int(k));
    if (C.nsplit == 1) continue;

    // ---- split partial published by every thread (ordered by the barrier
    // above); the last CTA of this (query, head group) queues the merge
    if (threadIdx.x == 0) {
      s_hdr[1] = 0;
      const unsigned prev = atom_inc_acq_rel(merge_cnt + (int64_t(C.qi) * p.head_items + C.hi), C.nsplit - 1);
      if (prev == static_cast<unsigned>(C.nsplit - 1)) {
        const int idx = s_sync[2]++;
        if (idx < kMaxPending) s_pend[idx] = item_of(b, k, G); else s_hdr[1] = 1;
      }
    }
    __syncthreads();
    if (s_hdr[1]) merge_global<D>(p, C, out_base, s_mo);  // queue overflow: merge now
    __syncthreads();
  }
  // ---- queued split merges, cooperatively by the whole CTA
  cp_async_wait<0>();
  __syncthreads();
  const int npend = s_sync[2];
  for (int i = 0; i < npend && i < kMaxPending; ++i) {
    const Item M = make_item(s_pend[i], pv, p);
    merge_global<D>(p, M, (int64_t(M.qi) * p.hq + M.qh0) * D, s_mo);
    __syncthreads();
  }
  trace(kTraceSlots - 1);
}

template <typename T, int D>
TcFn pick_rows(bool splitq, bool rows16) {
  if (splitq) return rows16 ? decode_tc_kernel<T, D, true, true> : decode_tc_kernel<T, D, true, false>;
  return rows16 ? decode_tc_kernel<T, D, false, true> : decode_tc_kernel<T, D, false, false>;
}

int pow2_at_least(int n) {
  int x = 1;
  while (x < n) x <<= 1;
  return x;
}

}  // namespace

bool decode_tc_supported(int kv_dtype, int head_dim) {
  return (kv_dtype == PKV_BF16 || kv_dtype == PKV_F16) && (head_dim == 64 || head_dim == 128);
}

int64_t decode_tc_plan_bytes(int64_t nq) {
  // int32 header + 6 arrays, then the int64 sort scratch
  const int64_t ints = 4 + 6 * nq + 2;
  const int64_t al = (ints * 4 + 255) / 256 * 256;
  return al + 8 * int64_t(pow2_at_least(static_cast<int>(nq)));
}

int launch_decode_tc(TcParams p, int kv_dtype, int head_dim, int num_sms, cudaStream_t stream) {
  const bool splitq = p.q_dtype == PKV_F32;
  const bool rows16 = p.group > 8;
  p.kv_dtype = kv_dtype;
  TcFn fn = nullptr;
  if (kv_dtype == PKV_BF16)
    fn = head_dim == 64 ? pick_rows<__nv_bfloat16, 64>(splitq, rows16) : pick_rows<__nv_bfloat16, 128>(splitq, rows16);
  else
    fn = head_dim == 64 ? pick_rows<__half, 64>(splitq, rows16) : pick_rows<__half, 128>(splitq, rows16);
  const int merge_bytes = kWarpsTc * kMergeRows * head_dim * 4 + kWarpsTc * kMergeRows * 2 * 4;
  if (p.nq <= kSmemPlanMax) {
    p.plan_global = nullptr;
    const int plan_bytes = (6 * p.nq + 2) * 4;
    p.merge_offset = (plan_bytes + 127) / 128 * 128;
    // the in-CTA sort borrows the merge buffer as scratch
    const int sort_bytes = 8 * pow2_at_least(p.nq);
    const int merge_span = merge_bytes > sort_bytes ? merge_bytes : sort_bytes;
    p.ring_offset = (p.merge_offset + merge_span + 1023) / 1024 * 1024;
  } else {
    p.merge_offset = 0;
    p.ring_offset = (merge_bytes + 1023) / 1024 * 1024;
    plan_tc_kernel<<<1, 1024, 0, stream>>>(p, const_cast<int32_t*>(p.plan_global),
                                           reinterpret_cast<long long*>(p.plan_scratch),
                                           pow2_at_least(p.nq));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(PKV_CUDA_ERROR, "decode_tc plan launch: %s", cudaGetErrorString(e));
  }
  const int smem = p.ring_offset + kWarpsTc * kStagesTc * 2 * kCh * head_dim * 2;
  static int configured[16] = {0};
  const int key = (kv_dtype == PKV_BF16) * 8 + (head_dim == 128) * 4 + splitq * 2 + rows16;
  if (configured[key] < smem) {
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess)
      return fail(PKV_CUDA_ERROR, "decode_tc smem attribute (%d B): %s", smem, cudaGetErrorString(e));
    configured[key] = smem;
  }
  fn<<<num_sms, kThreadsTc, smem, stream>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(PKV_CUDA_ERROR, "decode_tc launch: %s", cudaGetErrorString(e));
  return PKV_OK;
}

int decode_tc_warps() { return kWarpsTc; }

int debug_trace(int enable, uint64_t* out, int64_t n) {
  if (enable >= 0) {
    cudaMemcpyToSymbol(g_trace_on, &enable, sizeof(int));
    static const unsigned long long zeros[1024] = {0};
    for (int i = 0; i < kTraceSlots; ++i)
      cudaMemcpyToSymbol(g_trace, zeros, sizeof(zeros), sizeof(zeros) * i);
  }
  if (out && n > 0) {
    const int64_t m = n < 1024 * kTraceSlots ? n : 1024 * kTraceSlots;
    cudaMemcpyFromSymbol(out, g_trace, m * sizeof(unsigned long long));
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PKV_OK : fail(PKV_CUDA_ERROR, "debug trace: %s", cudaGetErrorString(e));
}

}  // namespace pkv
