// K2-TC: split-K paged decode on the tensor cores (mma.sync m16n8k16, bf16 /
// fp16 operands, fp32 accumulation) for 16-bit KV caches, with the split
// merge done inside the kernel, and its host-side planner.
//
// Replaces the reference streaming kernel (attention.py:259-329) for bf16
// stores.  Decode is HBM bound (GQA-4 bf16: 4 flop/B, far below the ridge), so
// the tensor cores are used to cut *issue* cost, not for FLOPs: a 16-key chunk
// costs 16 HMMA + 16 LDSM + the softmax instead of ~1200 CUDA-core
// instructions.  tcgen05 is not used: M = G <= 16 query rows is not a dense
// contraction and the TMEM round trip would cost more than it saves
// (SURVEY.md §2.3).
//
// Work decomposition (planned on the host, like any serving scheduler: the
// per-query key counts are host metadata).  A unit is (query, block of HB kv
// heads, group of query heads); each CTA (8 warps, one per SM) gives every kv
// head of the block WPH = 8/HB warps:
//   * large batches: HB = 8, WPH = 1 — one warp streams one kv head;
//   * small batches: HB < 8, WPH > 1 — the head's warps take its 16-key
//     chunks round-robin and merge in parallel through shared memory at a
//     named barrier.
// Schedule ("stream-K" for paged decode, plan_decode): all units are laid on
// one line (pages + a per-item overhead) and cut into one equal segment per
// SM, so every CTA streams the same bytes and runs only ~units/SMs + 1 items;
// a unit cut between CTAs is merged by the last of its pieces to finish
// (arrival counters in the per-call plan upload, self-resetting), in page
// order — deterministic.  About 128 of the 148 CTAs already saturate HBM, so
// with more units than SMs the line is cut into 128 segments, and a uniform
// batch of 70-100% as many units as SMs runs one uncut unit per CTA (no
// partials, no merges).  Small batches use cluster mode instead: each unit
// gets a thread-block cluster whose CTAs split its pages, push their partials
// into the owning peer's shared memory and merge there (DSMEM, one cluster
// barrier).  Every warp runs a producer that streams its
// chunks through a private 3-stage cp.async ring (16-byte XOR swizzle ->
// conflict-free LDSM; zero-fill past the valid keys) straight across item
// boundaries.  The G grouped query heads are the M rows of the MMA, so every
// K/V byte is read from HBM once per query-head group.
//
// Numerics: scores accumulate unscaled in fp32 and the softmax scale (times
// log2 e) is folded into the exp2 argument; P is rounded to the operand type
// for the P@V MMA and the denominator sums the *rounded* P.  fp32 queries are
// split hi+lo into two MMAs (fp32-accurate scores).  Optional fused append:
// with k_new/v_new the piece holding a query's final token reads it from the
// input and writes it into its page (reshape-and-cache folded into the
// decode launch).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "decode_tc.h"
#include "step_graph.h"

namespace pkv {

// Debug timeline (pkv_debug_trace): per CTA, globaltimer stamps of
// [start, plan loaded, item k consumer start..., chunks done, published, end].
__device__ unsigned long long g_trace[1024 * 64];
__device__ volatile int g_trace_on;
__device__ unsigned long long g_trace_sm[256];  // SM id per traced CTA (read after the timeline)

namespace {

constexpr int kWarpsTc = 8;
constexpr int kThreadsTc = kWarpsTc * 32;
constexpr int kStagesTc = 3;
constexpr int kCh = 16;        // keys per chunk
constexpr int kMergeRows = 4;  // rows per warp slot of the intra-CTA merge
constexpr int kTraceSlots = 64;

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// per warp: 32 slots [start, plan, (item start, first data, chunks done,
// stored) x 7, end]; lane 0 of every warp of CTAs < 256 records
// The switch is read once per kernel (a volatile load per stamp would add a
// global round trip to every item of production runs).
__device__ __forceinline__ void trace_at(bool on, int slot) {
  if (on && (threadIdx.x & 31) == 0 && slot < 32 && blockIdx.x < 256)
    g_trace[(blockIdx.x * 8 + (threadIdx.x >> 5)) * 32 + slot] = gtimer();
}
#define trace(slot) trace_at(trace_on, (slot))

// plan layout (int32), see plan_decode():
//   header[kHdr] | nk[nq] | row[nq] | cta_off[grid+1] | items[total][6]
//   | comb[n_comb][4] | counters[n_comb][kWarpsTc] (zeros)
// item  = {query, head item (head block x query group), first page, end page,
//          partial slot or -1 when the item covers its whole (query, head
//          item), comb record or -1}
// comb  = {query, head item, first slot, pieces}: a (query, head item) whose
//          pages were cut across CTAs; its pieces own consecutive slots.  The
//          last piece to finish (per head warp, counted in `counters`, which
//          the host uploads as zeros and the merging warp resets) merges all
//          pieces in page order — deterministic, and no combine launch.
enum {
  H_HB = 0, H_WPH, H_QGS, H_QGROUPS, H_HEAD_ITEMS, H_TOTAL_ITEMS, H_NCOMB, H_NQ,
  H_GRID, H_CTA_OFF, H_ITEMS, H_COMB, H_CTR, H_CLUSTER, kHdr = 14
};
constexpr int kItemInts = 6;
constexpr int kCombInts = 4;
constexpr int kCtaItemsSmem = 64;  // per-CTA item records staged in shared memory
__host__ __device__ constexpr int64_t o_nk(int64_t) { return kHdr; }
__host__ __device__ constexpr int64_t o_row(int64_t nq) { return kHdr + nq; }
__host__ __device__ constexpr int64_t o_cta(int64_t nq) { return kHdr + 2 * nq; }

struct PlanView {
  const int32_t *nk, *row;
  const int32_t* items;  // this CTA's first record (shared or global memory)
  int count;             // items of this CTA
  int hb, wph, qgs, qgroups, nq, ps, cluster;
};

// one warp's view of a work item
struct Item {
  int qi, kvh, sub, qh0, rows, kb, ke, nchunks, nk, row, slot, comb;
  bool valid, last;  // last: the item holds the query's final page (fused append)
};

__device__ __forceinline__ Item make_item(int k, const PlanView& pv, const TcParams& p, int warp) {
  Item it;
  it.valid = k < pv.count;
  if (!it.valid) return it;
  const int32_t* r = pv.items + k * kItemInts;
  const int q = r[0], hix = r[1], pb = r[2], pe = r[3];
  it.slot = r[4];
  it.comb = r[5];
  it.qi = q;
  const int hb = hix / pv.qgroups;
  const int qg = hix - hb * pv.qgroups;
  it.kvh = hb * pv.hb + warp / pv.wph;
  it.sub = warp % pv.wph;
  it.qh0 = it.kvh * p.group + qg * pv.qgs;
  it.rows = min(pv.qgs, p.group - qg * pv.qgs);
  it.nk = pv.nk[q];
  it.row = pv.row[q];
  it.kb = pb << p.log2ps;
  it.ke = min(it.nk, pe << p.log2ps);
  it.last = it.kb < it.nk && it.ke == it.nk;  // the piece holding the final token
  it.nchunks = (it.ke - it.kb + kCh - 1) / kCh;
  return it;
}

// Split finish: called by a whole warp after it stored the partial (m, l, O)
// rows [qh0, qh0 + rows) of its piece.  The last piece of the unit to arrive
// (per head warp slot) merges every piece in page order and writes the output.
template <int D>
__device__ __forceinline__ void finish_split(const TcParams& p, const int32_t* plan, int comb, int hslot,
                                             int qi, int qh0, int rows, int lane) {
  __threadfence();
  __syncwarp();
  int* ctr = const_cast<int32_t*>(plan) + plan[H_CTR] + comb * kWarpsTc + hslot;
  const int32_t* c = plan + plan[H_COMB] + comb * kCombInts;
  const int s0 = __ldg(c + 2), ns = __ldg(c + 3);
  int last = 0;
  if (lane == 0) last = atomicAdd(ctr, 1) == ns - 1;
  if (!__shfl_sync(0xffffffffu, last, 0)) return;
  __threadfence();
  const float2* ml = reinterpret_cast<const float2*>(p.ws_ml);
  constexpr int E = D / 32;
  for (int r = 0; r < rows; ++r) {
    const int qh = qh0 + r;
    // lanes over pieces for the row max and denominator
    float mx = -INFINITY;
    for (int s = lane; s < ns; s += 32) mx = fmaxf(mx, __ldcg(ml + int64_t(s0 + s) * p.hq + qh).x);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float den = 0.f;
    for (int s = lane; s < ns; s += 32) {
      const float2 v = __ldcg(ml + int64_t(s0 + s) * p.hq + qh);
      den += (v.x == -INFINITY ? 0.f : exp2f(v.x - mx)) * v.y;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
    // O: 8 pieces in flight per step, summed in page order
    float acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = 0.f;
    for (int sb = 0; sb < ns; sb += 8) {
      float wv[8], ov[8][E];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool in = sb + u < ns;
        const int64_t slot = int64_t(s0 + sb + (in ? u : 0)) * p.hq + qh;
        wv[u] = in ? __ldcg(ml + slot).x : -INFINITY;
#pragma unroll
        for (int e = 0; e < E; ++e) ov[u][e] = in ? __ldcg(p.ws_o + slot * D + lane + 32 * e) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float w = wv[u] == -INFINITY ? 0.f : exp2f(wv[u] - mx);
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] += w * ov[u][e];
      }
    }
    const float inv = 1.f / den;
#pragma unroll
    for (int e = 0; e < E; ++e)
      store_from_float(p.out, (int64_t(qi) * p.hq + qh) * D + lane + 32 * e, p.out_dtype, acc[e] * inv);
  }
  if (lane == 0) *ctr = 0;  // self-cleaning: the plan buffer can be replayed
}

// split-phase cluster barrier (all threads of every CTA of the cluster)
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }
// remote (DSMEM) store into CTA `rank`'s copy of `local`; fire-and-forget,
// made visible by the next barrier.cluster.arrive.release / wait.acquire
__device__ __forceinline__ void st_dsmem(float* local, uint32_t rank, float v) {
  uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(local)), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(ra), "f"(v) : "memory");
}
__device__ __forceinline__ void st_dsmem4(float* local, uint32_t rank, float4 v) {
  uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(local)), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(ra), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// a float in the shared memory of CTA `rank` of this cluster (DSMEM)
__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Split finish for a head group of `grp` threads (wph warps) that stored its
// piece's partial rows: one thread counts the arrival; if this piece is the
// unit's last, the whole group merges all pieces in page order in parallel.
template <int D>
__device__ __forceinline__ void finish_split_group(const TcParams& p, const int32_t* plan, int comb, int hslot,
                                                   int qi, int qh0, int rows, int tt, int grp, int bar_id,
                                                   int* flag) {
  // the group's partial stores happen-before the arrival: bar.sync orders
  // them at CTA scope and thread 0's gpu-scope fence is cumulative
  named_bar(bar_id, grp);
  int* ctr = const_cast<int32_t*>(plan) + plan[H_CTR] + comb * kWarpsTc + hslot;
  const int32_t* c = plan + plan[H_COMB] + comb * kCombInts;
  const int s0 = __ldg(c + 2), ns = __ldg(c + 3);
  if (tt == 0) {
    __threadfence();
    *flag = atomicAdd(ctr, 1) == ns - 1;
    __threadfence();
  }
  named_bar(bar_id, grp);
  if (!*flag) return;
  const float2* ml = reinterpret_cast<const float2*>(p.ws_ml);
  // one pass over the pieces with an online rescale, four consecutive
  // elements per thread (16-byte loads); 16 pieces' (m, l) and O loads are
  // issued together so a block of pieces costs one L2 round trip
  constexpr int D4 = D / 4;
#pragma unroll 1
  for (int e4 = tt; e4 < rows * D4; e4 += grp) {
    const int r = e4 / D4, d = (e4 - r * D4) * 4;
    const int qh = qh0 + r;
    float mx = -INFINITY, den = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int sb = 0; sb < ns; sb += 16) {
      float2 mv[16];
      float4 ov[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const bool in = sb + u < ns;
        const int64_t slot = int64_t(s0 + sb + (in ? u : 0)) * p.hq + qh;
        mv[u] = in ? __ldcg(ml + slot) : make_float2(-INFINITY, 0.f);
        ov[u] = in ? __ldcg(reinterpret_cast<const float4*>(p.ws_o + slot * D + d)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      float bm = mx;
#pragma unroll
      for (int u = 0; u < 16; ++u) bm = fmaxf(bm, mv[u].x);
      const float cr = mx == -INFINITY ? 0.f : ex2_ftz(mx - bm);
      den *= cr;
      acc.x *= cr;
      acc.y *= cr;
      acc.z *= cr;
      acc.w *= cr;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const float w = mv[u].x == -INFINITY ? 0.f : ex2_ftz(mv[u].x - bm);
        den += w * mv[u].y;
        acc.x += w * ov[u].x;
        acc.y += w * ov[u].y;
        acc.z += w * ov[u].z;
        acc.w += w * ov[u].w;
      }
      mx = bm;
    }
    const float inv = 1.f / den;
    const int64_t o = (int64_t(qi) * p.hq + qh) * D + d;
    store4_from_float(p.out, o, p.out_dtype,
                      make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv));
  }
  if (tt == 0) *ctr = 0;  // self-cleaning: the plan buffer can be replayed
}

template <typename T, int D, bool SPLITQ, bool ROWS16>
__device__ __forceinline__ void decode_tc_body(const TcParams& p, const ClusterInline* ci) {
  constexpr int ROWB = D * 2;            // smem row bytes
  constexpr int CPR = ROWB / 16;         // 16-B chunks per row (8 or 16)
  constexpr int RPI = 32 / CPR;          // rows per copy iteration
  constexpr int NIT = kCh / RPI;         // copy iterations per chunk
  constexpr int STAGE = 2 * kCh * ROWB;  // K + V
  constexpr int KS = D / 16;             // k-steps of Q K^T
  constexpr int NT = D / 8;              // n-tiles of P V
  static_assert(CPR >= 8 && CPR <= 32, "D must be 64 or 128");

  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ int s_flag[kWarpsTc];  // per head: this CTA's piece merges the split
  // cluster mode: the slices of the unit's pieces pushed here by every CTA of
  // the cluster (unnormalised O, then row max / row sum per piece)
  __shared__ __align__(16) float r_o[kMergeRows * 128 + 64];
  __shared__ float r_ml[16 * kMergeRows * 2];
  __shared__ float s_wgt[kWarpsTc * kMergeRows];       // intra-CTA merge weights per (warp, row)
  __shared__ float s_rml[kWarpsTc * kMergeRows * 2];   // per head group: row (max, sum)
  __shared__ float s_cw[16 * kMergeRows];              // cluster merge weights per (rank, row)
  __shared__ float s_cinv[kMergeRows];
  __shared__ int32_t s_cta_items[kCtaItemsSmem * kItemInts];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool trace_on = g_trace_on != 0;
  trace(0);
  if (trace_on && threadIdx.x == 0 && blockIdx.x < 256) {  // SM of this CTA
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_trace_sm[blockIdx.x] = smid;
  }
  // ---------------- plan (host-computed; staged into shared memory) ---------
  PlanView pv;
  if (ci) {
    // cluster mode, plan in the launch parameters: CTA n runs item n — its
    // cluster rank's even share of the pages of unit n / cluster
    const int nq = p.nq;
    pv.nk = ci->nkrow;
    pv.row = ci->nkrow + nq;
    pv.hb = ci->hb;
    pv.wph = ci->wph;
    pv.cluster = ci->cluster;
    pv.qgs = ci->qgs;
    pv.qgroups = ci->qgroups;
    pv.nq = nq;
    pv.count = 1;
    if (threadIdx.x == 0) {
      const int unit = static_cast<int>(blockIdx.x) / pv.cluster, c = static_cast<int>(blockIdx.x) % pv.cluster;
      const int q = unit / ci->head_items;
      const int pages = (pv.nk[q] + (1 << p.log2ps) - 1) >> p.log2ps;
      s_cta_items[0] = q;
      s_cta_items[1] = unit - q * ci->head_items;
      s_cta_items[2] = static_cast<int>(int64_t(pages) * c / pv.cluster);
      s_cta_items[3] = static_cast<int>(int64_t(pages) * (c + 1) / pv.cluster);
      s_cta_items[4] = -1;
      s_cta_items[5] = -1;
    }
    __syncthreads();
    pv.items = s_cta_items;
  } else {
    const int32_t* g = p.plan;
    const int nq = p.nq;
    const int32_t* off = g + o_cta(nq);
    const int first = __ldg(off + blockIdx.x);
    pv.count = __ldg(off + blockIdx.x + 1) - first;
    const int32_t* gitems = g + __ldg(g + H_ITEMS) + int64_t(first) * kItemInts;
    const bool items_smem = pv.count <= kCtaItemsSmem;
    for (int i = threadIdx.x; i < (items_smem ? pv.count * kItemInts : 0); i += kThreadsTc)
      s_cta_items[i] = __ldg(gitems + i);
    const int32_t* src = g;
    if (p.plan_in_smem) {
      int32_t* s = reinterpret_cast<int32_t*>(smem);
      const int n = static_cast<int>(o_cta(nq));
      for (int i = threadIdx.x; i < n; i += kThreadsTc) s[i] = __ldg(g + i);
      src = s;
    }
    __syncthreads();
    pv.items = items_smem ? s_cta_items : gitems;
    pv.nk = src + o_nk(nq);
    pv.row = src + o_row(nq);
    pv.hb = src[H_HB];
    pv.wph = src[H_WPH];
    pv.cluster = src[H_CLUSTER];
    pv.qgs = src[H_QGS];
    pv.qgroups = src[H_QGROUPS];
    pv.nq = nq;
  }
  // cluster mode: announce that this CTA runs (its shared memory may receive
  // peer stores once every CTA has arrived; waited on before the first push)
  if (pv.cluster > 1) cluster_arrive_relaxed();
  // Launched with programmatic stream serialization: everything above reads
  // only the plan / launch parameters (uploaded before the preceding kernel
  // started); the block table, the pages and the queries may still be being
  // written by that kernel (the step's page-clear / mirror aux kernel), so
  // wait for its completion here.  A no-op without a programmatic predecessor.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  trace(1);
  float* s_mo = reinterpret_cast<float*>(smem + p.merge_offset);  // [W][4][D]
  float* s_ml = s_mo + kWarpsTc * kMergeRows * D;                 // [W][4][2]
  unsigned char* ring = smem + p.ring_offset + warp * (kStagesTc * STAGE);
  const uint32_t ring_addr = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  const int t4 = lane & 3, g = lane >> 2;
  const int ps = 1 << p.log2ps;

  // ======================= producer (per warp) ===========================
  const int cc = lane % CPR, r0 = lane / CPR;  // copy geometry of this lane
  Item P;
  int64_t pk = 0;  // producer item counter (within this CTA's sequence)
  int pc = 0;      // next chunk of P to issue
  int win = -1, win_val = 0;
  auto start_item = [&]() {
    for (;;) {
      P = make_item(static_cast<int>(pk), pv, p, warp);
      pc = P.sub;
      win = -1;
      if (!P.valid) return;
      if (P.sub == 0) {
        // warm L2 with the query rows the consumer loads at item start
        const int qe = p.q_dtype == PKV_F32 ? 4 : 2;
        const char* qrow = static_cast<const char*>(p.q) + (int64_t(P.qi) * p.hq + P.qh0) * D * qe;
        if (lane * 128 < P.rows * D * qe) asm volatile("prefetch.global.L2 [%0];" ::"l"(qrow + lane * 128));
        if (p.k_new != nullptr && P.last) {
          // fused append: write the new token's head slice into its page
          const int pos = P.nk - 1;
          const int64_t page = p.bt[int64_t(P.row) * p.bt_stride + (pos >> p.log2ps)];
          const int64_t dst = (page * ps + (pos & (ps - 1))) * p.row_stride + int64_t(P.kvh) * ROWB;
          const int64_t srcb = (int64_t(P.qi) * p.hkv + P.kvh) * ROWB;
          if (lane < CPR) {
            reinterpret_cast<uint4*>(p.kw + dst)[lane] = reinterpret_cast<const uint4*>(p.k_new + srcb)[lane];
            reinterpret_cast<uint4*>(p.vw + dst)[lane] = reinterpret_cast<const uint4*>(p.v_new + srcb)[lane];
          }
        }
      }
      if (pc < P.nchunks) return;
      ++pk;  // no chunk of this item for this warp
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
      const bool fuse = p.k_new != nullptr && P.last;
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
      pc += pv.wph;
      if (pc >= P.nchunks) {
        ++pk;
        start_item();
      }
    }
    cp_async_commit();
  };

  start_item();
  trace(24);  // prologue stamps (slots 24-26 are free when a warp runs <= 5 items)
  issue_next();
  trace(25);
#pragma unroll
  for (int i = 1; i < kStagesTc - 1; ++i) issue_next();
  trace(26);

  // ======================= consumer ======================================
  long long gcons = 0;
  const float qscale = p.qscale;
  const int head_local = warp / pv.wph;
  const int cluster = pv.cluster;
  for (int64_t k = 0;; ++k) {
    const Item C = make_item(static_cast<int>(k), pv, p, warp);
    if (!C.valid) break;
    trace(2 + 4 * int(k));

    float o[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

    if (C.sub < C.nchunks) {
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

      for (int c = C.sub; c < C.nchunks; c += pv.wph) {
        cp_async_wait<kStagesTc - 2>();
        __syncwarp();
        if (c == C.sub) trace(3 + 4 * int(k));
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
        const float c0 = ex2_ftz(m0 - mn0);
        m0 = mn0;
        uint32_t pa[4];
        {
          const float p00 = ex2_ftz(fmaf(s0[0], qscale, -mn0)), p01 = ex2_ftz(fmaf(s0[1], qscale, -mn0));
          const float p10 = ex2_ftz(fmaf(s1[0], qscale, -mn0)), p11 = ex2_ftz(fmaf(s1[1], qscale, -mn0));
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
          c1 = ex2_ftz(m1 - mn1);
          m1 = mn1;
          const float p02 = ex2_ftz(fmaf(s0[2], qscale, -mn1)), p03 = ex2_ftz(fmaf(s0[3], qscale, -mn1));
          const float p12 = ex2_ftz(fmaf(s1[2], qscale, -mn1)), p13 = ex2_ftz(fmaf(s1[3], qscale, -mn1));
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
    trace(4 + 4 * int(k));
    const int64_t out_base = (int64_t(C.qi) * p.hq + C.qh0) * D;
    const int64_t pslot = int64_t(C.slot) * p.hq + C.qh0;  // split partial rows

    if (pv.wph == 1) {
      // ---- one warp owns this head: output rows or the split partial
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int d = n * 8 + 2 * t4;
        if (C.slot < 0) {
          if (g < C.rows) {
            store2_from_float(p.out, out_base + int64_t(g) * D + d, p.out_dtype, o[n][0] / l0, o[n][1] / l0);
          }
          if (ROWS16 && g + 8 < C.rows) {
            store2_from_float(p.out, out_base + int64_t(g + 8) * D + d, p.out_dtype, o[n][2] / l1, o[n][3] / l1);
          }
        } else {
          if (g < C.rows) __stcg(reinterpret_cast<float2*>(p.ws_o + (pslot + g) * D + d), make_float2(o[n][0], o[n][1]));
          if (ROWS16 && g + 8 < C.rows)
            __stcg(reinterpret_cast<float2*>(p.ws_o + (pslot + g + 8) * D + d), make_float2(o[n][2], o[n][3]));
        }
      }
      if (C.slot >= 0 && t4 == 0) {
        if (g < C.rows) __stcg(reinterpret_cast<float2*>(p.ws_ml) + pslot + g, make_float2(m0, l0));
        if (ROWS16 && g + 8 < C.rows) __stcg(reinterpret_cast<float2*>(p.ws_ml) + pslot + g + 8, make_float2(m1, l1));
      }
      if (C.slot >= 0) finish_split<D>(p, p.plan, C.comb, warp, C.qi, C.qh0, C.rows, lane);
      trace(5 + 4 * int(k));
      continue;
    }

    // ---- WPH warps share this head: the head's warps meet at a named
    // barrier and merge their partials in parallel (thread tt of the group
    // owns elements tt, tt + 32*wph, ... of the rows x D block).
    const int grp = pv.wph * 32;
    const int bar_id = 1 + head_local;
    const int tt = (warp - head_local * pv.wph) * 32 + lane;
    if (g < C.rows) {  // rows <= kMergeRows when wph > 1 (planner)
      float* dst = s_mo + (warp * kMergeRows + g) * D;
#pragma unroll
      for (int n = 0; n < NT; ++n) *reinterpret_cast<float2*>(dst + n * 8 + 2 * t4) = make_float2(o[n][0], o[n][1]);
      if (t4 == 0) {
        s_ml[(warp * kMergeRows + g) * 2] = m0;
        s_ml[(warp * kMergeRows + g) * 2 + 1] = l0;
      }
    }
    named_bar(bar_id, grp);
    trace(5 + 4 * int(k));
    const int w0 = head_local * pv.wph;
    const int E = C.rows * D;
    // slice of the rows x D block each cluster CTA merges (multiple of 4)
    const int slice = cluster > 1 ? ((E + cluster - 1) / cluster + 3) & ~3 : E;
    const uint32_t my_rank = cluster > 1 ? cluster_rank() : 0u;
    if (cluster > 1) cluster_wait();  // every peer runs: its shared memory may be written
    // per (row, warp) weights and per-row (max, sum), once per row instead
    // of once per element
    if (tt < C.rows) {
      const int r = tt;
      float mx = -INFINITY;
      for (int w = w0; w < w0 + pv.wph; ++w) mx = fmaxf(mx, s_ml[(w * kMergeRows + r) * 2]);
      float den = 0.f;
      for (int w = w0; w < w0 + pv.wph; ++w) {
        const float mw = s_ml[(w * kMergeRows + r) * 2];
        const float wgt = mw == -INFINITY ? 0.f : ex2_ftz(mw - mx);
        s_wgt[w * kMergeRows + r] = wgt;
        den += wgt * s_ml[(w * kMergeRows + r) * 2 + 1];
      }
      s_rml[(w0 * kMergeRows + r) * 2] = mx;
      s_rml[(w0 * kMergeRows + r) * 2 + 1] = den;
      if (cluster > 1)  // the row's max / sum to every peer
        for (int c = 0; c < cluster; ++c) {
          st_dsmem(&r_ml[(my_rank * kMergeRows + r) * 2], c, mx);
          st_dsmem(&r_ml[(my_rank * kMergeRows + r) * 2 + 1], c, den);
        }
    }
    named_bar(bar_id, grp);
    trace(27);
    constexpr int D4 = D / 4;
#pragma unroll 1
    for (int e4 = tt; e4 < C.rows * D4; e4 += grp) {
      const int r = e4 / D4, d = (e4 - r * D4) * 4;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int w = w0; w < w0 + pv.wph; ++w) {
        const float wgt = s_wgt[w * kMergeRows + r];
        const float4 v = *reinterpret_cast<const float4*>(s_mo + (w * kMergeRows + r) * D + d);
        acc.x += wgt * v.x;
        acc.y += wgt * v.y;
        acc.z += wgt * v.z;
        acc.w += wgt * v.w;
      }
      const int e = r * D + d;
      if (cluster > 1) {  // push the 4 elements to the CTA that merges their slice
        const int owner = e / slice;
        st_dsmem4(&r_o[my_rank * slice + (e - owner * slice)], owner, acc);
      } else if (C.slot < 0) {
        const float inv = 1.f / s_rml[(w0 * kMergeRows + r) * 2 + 1];
        store4_from_float(p.out, out_base + e, p.out_dtype,
                          make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv));
      } else {
        __stcg(reinterpret_cast<float4*>(p.ws_o + (pslot + r) * D + d), acc);
        if (d == 0)
          __stcg(reinterpret_cast<float2*>(p.ws_ml) + pslot + r,
                 make_float2(s_rml[(w0 * kMergeRows + r) * 2], s_rml[(w0 * kMergeRows + r) * 2 + 1]));
      }
    }
    trace(28);
    if (cluster > 1) {
      // Cluster mode (small batches): the unit's pieces are the CTAs of this
      // cluster.  Every CTA pushed its slice-e values into the owner's shared
      // memory above; after one cluster barrier each CTA merges its own
      // 1/cluster slice of the rows x D outputs from LOCAL shared memory, in
      // rank order.  No peer touches this CTA's memory after the barrier.
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
      if (threadIdx.x < C.rows) {  // per (rank, row) weights once
        const int r = threadIdx.x;
        float mx = -INFINITY;
        for (int c = 0; c < cluster; ++c) mx = fmaxf(mx, r_ml[(c * kMergeRows + r) * 2]);
        float den = 0.f;
        for (int c = 0; c < cluster; ++c) {
          const float mw = r_ml[(c * kMergeRows + r) * 2];
          const float w = mw == -INFINITY ? 0.f : ex2_ftz(mw - mx);
          s_cw[c * kMergeRows + r] = w;
          den += w * r_ml[(c * kMergeRows + r) * 2 + 1];
        }
        s_cinv[r] = 1.f / den;
      }
      __syncthreads();
      const int e0 = static_cast<int>(my_rank) * slice, e1 = min(E, e0 + slice);
      for (int e = e0 + 4 * static_cast<int>(threadIdx.x); e < e1; e += 4 * kThreadsTc) {
        const int r = e / D;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int c = 0; c < cluster; ++c) {
          const float w = s_cw[c * kMergeRows + r];
          const float4 v = *reinterpret_cast<const float4*>(&r_o[c * slice + (e - e0)]);
          acc.x += w * v.x;
          acc.y += w * v.y;
          acc.z += w * v.z;
          acc.w += w * v.w;
        }
        const float inv = s_cinv[r];
        store4_from_float(p.out, out_base + e, p.out_dtype,
                          make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv));
      }
      break;  // one item per CTA in cluster mode
    }
    if (C.slot >= 0) finish_split_group<D>(p, p.plan, C.comb, head_local, C.qi, C.qh0, C.rows, tt, grp, bar_id,
                                           &s_flag[head_local]);
    named_bar(bar_id, grp);  // the head's merge slots are free for its next item
    trace(30);
  }
  cp_async_wait<0>();
  trace(31);
}

template <typename T, int D, bool SPLITQ, bool ROWS16>
__global__ void __launch_bounds__(kThreadsTc, 1) decode_tc_kernel(const __grid_constant__ TcParams p) {
  decode_tc_body<T, D, SPLITQ, ROWS16>(p, nullptr);
}
template <typename T, int D, bool SPLITQ, bool ROWS16>
__global__ void __launch_bounds__(kThreadsTc, 1)
    decode_tc_cluster_kernel(const __grid_constant__ TcParams p, const __grid_constant__ ClusterInline ci) {
  decode_tc_body<T, D, SPLITQ, ROWS16>(p, &ci);
}
using TcClusterFn = void (*)(TcParams, ClusterInline);
template <typename T, int D>
TcClusterFn pick_rows_cluster(bool splitq, bool rows16) {
  if (splitq) return rows16 ? decode_tc_cluster_kernel<T, D, true, true> : decode_tc_cluster_kernel<T, D, true, false>;
  return rows16 ? decode_tc_cluster_kernel<T, D, false, true> : decode_tc_cluster_kernel<T, D, false, false>;
}

template <typename T, int D>
TcFn pick_rows(bool splitq, bool rows16) {
  if (splitq) return rows16 ? decode_tc_kernel<T, D, true, true> : decode_tc_kernel<T, D, true, false>;
  return rows16 ? decode_tc_kernel<T, D, false, true> : decode_tc_kernel<T, D, false, false>;
}

template <typename T, int D>
void touch_tc_kernels() {
  cudaFuncAttributes fa;
  for (int sq = 0; sq < 2; ++sq)
    for (int r16 = 0; r16 < 2; ++r16) {
      cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(pick_rows<T, D>(sq, r16)));
      cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(pick_rows_cluster<T, D>(sq, r16)));
    }
}

}  // namespace

bool decode_tc_supported(int kv_dtype, int head_dim) {
  return (kv_dtype == PKV_BF16 || kv_dtype == PKV_F16) && (head_dim == 64 || head_dim == 128);
}

constexpr int kMaxGrid = 1024;
int64_t decode_plan_ints(int64_t nq, int hq) {
  // header + nk/row + cta offsets + items (units + 2 cuts per CTA) + comb
  const int64_t units = nq * hq;  // head items per query <= hq
  return o_cta(nq) + (kMaxGrid + 1) + (units + 2 * kMaxGrid) * kItemInts +
         (kMaxGrid + 1) * (kCombInts + kWarpsTc);
}

// Raise (never lower) a kernel's dynamic shared-memory limit.  One record per
// kernel: the occupancy query below and the launches share it, so a query
// can no longer shrink the limit under a launch that configured more.
cudaError_t ensure_smem(const void* fn, int smem) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> limit;
  std::lock_guard<std::mutex> g(mu);
  int& cur = limit[fn];
  if (cur >= smem) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) cur = smem;
  return e;
}

// Co-resident clusters of `c` CTAs of the decode kernel (one CTA per SM):
// queried from the device once (bf16, head_dim 128 instance, full smem),
// else the measured B200 figures scaled to num_sms.
int cluster_capacity(int c, int num_sms) {
  static int cached[17] = {0};
  if (c < 2 || c > 16) return 0;
  if (!cached[c]) {
    int n = 0;
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) == cudaSuccess && dev_count > 0) {
      auto fn = decode_tc_kernel<__nv_bfloat16, 128, false, false>;
      const int smem = 214016;
      ensure_smem(reinterpret_cast<const void*>(fn), smem);
      cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(static_cast<unsigned>(c));
      cfg.blockDim = dim3(kThreadsTc);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = static_cast<unsigned>(c);
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) n = 0;
      cudaGetLastError();
    }
    if (n <= 0) {
      const int b200[17] = {0, 0, 74, 0, 33, 0, 0, 0, 15, 0, 0, 0, 0, 0, 0, 0, 7};
      n = b200[c] * num_sms / 148;
    }
    cached[c] = n;
  }
  return cached[c];
}

// Host planner ("stream-K" for paged decode).  The work of every (query,
// head item) — a head block of hb kv heads x one group of query rows — is laid
// out on one line in query order, each unit charged its pages plus a fixed
// per-item overhead; the line is cut into `grid` equal segments, one per CTA,
// so every CTA streams the same number of bytes and runs only ~units/grid + 1
// items.  A cut inside a unit splits its pages between neighbouring CTAs (the
// pieces get partial slots and a combine record); cuts that would leave a
// piece shorter than the per-item overhead snap to the unit boundary.
int plan_decode(const int32_t* nk, const int32_t* row, int64_t nq, int page_size, int hq, int hkv, int head_dim,
                int num_sms, int waves, int32_t* out, int64_t cap, int64_t* n_out) {
  if (cap < decode_plan_ints(nq, hq)) return fail(PKV_VALUE_ERROR, "plan buffer too small");
  static const int max_grid_env = [] {  // experiment knob: cap the segment grid
    const char* e = std::getenv("PKV_DECODE_MAX_GRID");
    return e ? std::atoi(e) : 0;
  }();
  if (max_grid_env > 0) num_sms = std::min(num_sms, max_grid_env);
  num_sms = std::max(1, std::min(num_sms, kMaxGrid));
  const int all_sms = num_sms;
  const int G = hq / hkv;
  const int ps = page_size;
  int64_t total_pages = 0;
  for (int64_t i = 0; i < nq; ++i) total_pages += (int64_t(nk[i]) + ps - 1) / ps;
  // head block: one warp per kv head when there are enough (query, head
  // block) units to fill the GPU, otherwise several warps per head
  int hb = 1;
  for (int cand : {8, 4, 2, 1}) {
    if (hkv % cand) continue;
    const int wph = kWarpsTc / cand;
    const int qgs = wph == 1 ? 16 : kMergeRows;
    const int64_t units = nq * (hkv / cand) * ((G + qgs - 1) / qgs);
    hb = cand;
    if (units * 2 >= num_sms) break;
  }
  static const int hb_env = [] {  // experiment knob: force the head block
    const char* e = std::getenv("PKV_DECODE_HB");
    return e ? std::atoi(e) : 0;
  }();
  if (hb_env > 0 && hkv % hb_env == 0 && kWarpsTc % hb_env == 0) hb = hb_env;
  const int wph = kWarpsTc / hb;
  const int qgs = wph == 1 ? 16 : kMergeRows;
  const int qgroups = (G + qgs - 1) / qgs;
  const int head_items = (hkv / hb) * qgroups;
  // costs in pages of one unit; the per-item overhead (pipeline refill,
  // query load, partial store) is ~4 us ~ `ovh` pages of a CTA's stream
  const int D = head_dim > 0 ? head_dim : 128;
  const int64_t page_bytes = int64_t(hb) * ps * D * 2 * 2;  // K+V of the block
  static const int64_t ovh_kb = [] {  // per-item overhead in KB of stream (tuning knob)
    const char* e = std::getenv("PKV_DECODE_ITEM_KB");
    return e ? std::max<int64_t>(1, std::atoll(e)) : int64_t(400);  // measured optimum (C2, C3, C5)
  }();
  // per-item cost charged on the line (pipeline refill, query load, partial
  // store; ~400 KB of stream, measured) and the smallest piece a cut may
  // leave; both tunable for experiments
  static const int64_t cost_kb = [] {
    const char* e = std::getenv("PKV_DECODE_COST_KB");
    // 400 KB (round 2, current kernel): C2 5.87 -> 5.99 TB/s over 3 reps
    // (350 / 450 / 500 / 600: 5.95 / 5.93 / 5.95 / 5.87); C3, C5 within noise.
    // A per-CTA timeline fit (tools/trace_decode.py, CORR=1) gives ~4.5 us
    // per item vs ~1.1 us per 64 KB page on C2.
    return e ? std::max<int64_t>(0, std::atoll(e)) : int64_t(400);
  }();
  const int64_t ovh = ((cost_kb << 10) / page_bytes) * (waves > 0 ? waves : 1);
  bool whole = false;
  int64_t min_piece = std::max<int64_t>(
      std::max<int64_t>(1, (ovh_kb << 10) / page_bytes) / 2, (2 * kCh * wph + ps - 1) / ps);
  const int64_t units = nq * head_items;
  const int64_t line = total_pages * head_items + ovh * units;
  int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(num_sms, total_pages * head_items / min_piece)));
  // Many units (more than SMs, every CTA streams several): ~128 of 148 CTAs
  // saturate HBM, and fewer, longer segments mean fewer cut pieces and
  // merges (measured: C5 7.05 -> 7.28 TB/s, 4k x 256 6.70 -> 7.10, 2k x 512
  // 6.80 -> 6.97; C2 with 128 units keeps every SM).
  if (units > all_sms && max_grid_env <= 0)
    grid = std::min(grid, std::max(1, (all_sms * 128 + 147) / 148));
  // Whole units: when there are slightly fewer (query, head item) units than
  // SMs and they are about equally long, one uncut unit per CTA beats cutting
  // them to fill the last SMs — ~120 CTAs already saturate HBM, so the extra
  // CTAs add no bandwidth while every cut adds a partial store and a merge
  // (measured: C3 2k x 64 and 4k x 32 4.9 -> 5.7 TB/s, 16k x 16 5.9 -> 6.5).
  {
    int64_t max_pages = 0;
    for (int64_t i = 0; i < nq; ++i) max_pages = std::max<int64_t>(max_pages, (int64_t(nk[i]) + ps - 1) / ps);
    static const bool whole_on = [] {
      const char* e = std::getenv("PKV_DECODE_WHOLE_UNITS");
      return !(e && e[0] == '0');
    }();
    static const int whole_min_pct = [] {  // experiment knob: lowest units / SMs ratio (%)
      const char* e = std::getenv("PKV_DECODE_WHOLE_MIN_PCT");
      return e ? std::atoi(e) : 70;
    }();
    if (whole_on && units <= num_sms && units * 100 >= int64_t(num_sms) * whole_min_pct &&
        double(max_pages) * double(nq) <= 1.15 * double(total_pages)) {
      whole = true;  // never cut a unit: a unit that does not fit opens the next CTA
      grid = static_cast<int>(units);
    }
  }
  const double seg = double(line) / grid;

  // Cluster mode (small batches, one kv head per CTA): every (query, head
  // item) unit gets a cluster of C CTAs that split its pages evenly and merge
  // through distributed shared memory — no global partials, no arrival
  // counters, no last-arriver latency.
  // Used only when every cluster is resident at once (the GPC structure caps
  // co-resident clusters below num_sms / C: 7 x 16, 15 x 8, 33 x 4, 74 x 2 on
  // a 148-SM B200) and a simple time model predicts a win over the
  // segment schedule (fewer streaming CTAs vs a much cheaper merge).
  int cluster = 1;
  if (hb == 1 && waves >= 0) {
    const int64_t units_c = nq * head_items;
    int64_t max_pages = 0;
    for (int64_t i = 0; i < nq; ++i) max_pages = std::max<int64_t>(max_pages, (int64_t(nk[i]) + ps - 1) / ps);
    // time model (us): streaming at ~45 GB/s per CTA plus the merge — a
    // DSMEM cluster merge ~1 us, the global last-arriver merge ~2 us + 0.4 us
    // per piece of a unit (measured)
    const double bytes_per_head_page = double(ps) * D * 2 * 2;
    const double stream_us = double(total_pages) * head_items * bytes_per_head_page / 45e3;
    const int64_t reg_grid = std::min<int64_t>(num_sms, std::max<int64_t>(1, total_pages * head_items / 16));
    const double reg_us = stream_us / double(reg_grid) + 2.0 + 0.4 * double((reg_grid + units_c - 1) / units_c);
    double best = reg_us;
    for (int c = 16; c >= 2; c >>= 1) {
      if (units_c > cluster_capacity(c, num_sms) || units_c * c > num_sms || max_pages < 2 * c) continue;
      const double t = stream_us / double(units_c * c) + 1.0;
      // >= 80% SM cover: measured to beat the segment schedule (B = 4-8)
      if (units_c * c * 10 >= int64_t(num_sms) * 8) {
        cluster = c;
        break;
      }
      if (t < best) {
        best = t;
        cluster = c;
      }
    }
  }
  static const int cluster_env = [] {  // experiment knob: force the cluster size (1 = segment schedule)
    const char* e = std::getenv("PKV_DECODE_CLUSTER");
    return e ? std::atoi(e) : 0;
  }();
  if (cluster_env == 1) cluster = 1;
  if (cluster_env > 1 && hb == 1 && (cluster_env & (cluster_env - 1)) == 0 && cluster_env <= 16 &&
      nq * head_items * cluster_env <= num_sms && nq * head_items <= cluster_capacity(cluster_env, num_sms))
    cluster = cluster_env;
  int32_t* o = out;
  o[H_CLUSTER] = cluster;
  o[H_HB] = hb;
  o[H_WPH] = wph;
  o[H_QGS] = qgs;
  o[H_QGROUPS] = qgroups;
  o[H_HEAD_ITEMS] = head_items;
  o[H_NQ] = static_cast<int32_t>(nq);
  for (int64_t i = 0; i < nq; ++i) {
    o[o_nk(nq) + i] = nk[i];
    o[o_row(nq) + i] = row[i];
  }
  if (cluster > 1) {
    const int64_t units_c = nq * head_items;
    const int gridc = static_cast<int>(units_c * cluster);
    int32_t* ctac = o + o_cta(nq);
    const int64_t ipos = o_cta(nq) + gridc + 1;
    if (ipos + int64_t(gridc) * kItemInts > cap) return fail(PKV_VALUE_ERROR, "plan buffer too small");
    int32_t* it = o + ipos;
    int64_t n = 0;
    for (int64_t q = 0; q < nq; ++q) {
      const int64_t pages = (int64_t(nk[q]) + ps - 1) / ps;
      for (int h = 0; h < head_items; ++h)
        for (int c = 0; c < cluster; ++c, ++n) {
          ctac[n] = static_cast<int32_t>(n);
          int32_t* r = it + n * kItemInts;
          r[0] = static_cast<int32_t>(q);
          r[1] = h;
          r[2] = static_cast<int32_t>(pages * c / cluster);
          r[3] = static_cast<int32_t>(pages * (c + 1) / cluster);
          r[4] = -1;
          r[5] = -1;
        }
    }
    ctac[gridc] = static_cast<int32_t>(n);
    o[H_TOTAL_ITEMS] = static_cast<int32_t>(n);
    o[H_NCOMB] = 0;
    o[H_GRID] = gridc;
    o[H_CTA_OFF] = static_cast<int32_t>(o_cta(nq));
    o[H_ITEMS] = static_cast<int32_t>(ipos);
    o[H_COMB] = static_cast<int32_t>(ipos + n * kItemInts);
    o[H_CTR] = o[H_COMB];
    if (n_out) *n_out = ipos + n * kItemInts;
    return PKV_OK;
  }
  int32_t* cta = o + o_cta(nq);
  const int64_t items_pos = o_cta(nq) + grid + 1;
  int32_t* items = o + items_pos;
  // items are appended in line order; the comb list is built after them
  int64_t n_items = 0, n_slots = 0;
  std::vector<int32_t> comb;
  const int64_t item_cap = (cap - items_pos) / kItemInts;
  // Fill CTAs in line order up to a capacity T (pages + one overhead per
  // piece); the smallest T that fits in `grid` CTAs is found by bisection,
  // so the heaviest CTA carries as little as the snapping rules allow and no
  // CTA is left starved at the end of the line.
  bool overflow = false;
  auto fill = [&](double T, bool emit) -> int64_t {
    int64_t c = 0;
    double used = 0.0;
    if (emit) cta[0] = 0;
    auto next = [&]() {
      ++c;
      used = 0.0;
      if (emit && c <= grid) cta[c] = static_cast<int32_t>(n_items);
    };
    for (int64_t q = 0; q < nq; ++q) {
      const int64_t pages = (int64_t(nk[q]) + ps - 1) / ps;
      for (int h = 0; h < head_items; ++h) {
        int64_t p0 = 0;
        const int64_t first_item = n_items;
        int npieces = 0;
        while (p0 < pages) {
          int64_t take = pages - p0;
          const double room = T - used - double(ovh);  // pages that still fit here
          if (whole && room < double(take) && (!emit || c < grid - 1)) {
            if (used > 0.0) take = 0;  // start the unit in the next CTA
          } else if (room < double(take) && (!emit || c < grid - 1)) {
            int64_t fit = static_cast<int64_t>(room + 0.5);
            if (fit < min_piece) fit = 0;               // too small: start in the next CTA
            if (take - fit < min_piece) fit = take;     // remainder too small: keep it here
            // a fresh CTA always takes something (else a capacity below
            // ovh + min_piece would open empty CTAs forever)
            if (fit == 0 && used == 0.0) fit = std::min<int64_t>(take, min_piece);
            if (take - fit < min_piece) fit = take;
            take = fit;
          }
          if (take > 0) {
            if (emit && n_items >= item_cap) overflow = true;
            if (emit && !overflow) {
              int32_t* r = items + n_items * kItemInts;
              r[0] = static_cast<int32_t>(q);
              r[1] = h;
              r[2] = static_cast<int32_t>(p0);
              r[3] = static_cast<int32_t>(p0 + take);
              r[4] = -1;
              r[5] = -1;
              ++n_items;
            }
            ++npieces;
            p0 += take;
            used += double(take + ovh);
          }
          if (p0 < pages) next();
        }
        if (emit && npieces > 1) {
          const int32_t comb_idx = static_cast<int32_t>(comb.size() / kCombInts);
          for (int k = 0; k < npieces; ++k) {
            items[(first_item + k) * kItemInts + 4] = static_cast<int32_t>(n_slots++);
            items[(first_item + k) * kItemInts + 5] = comb_idx;
          }
          comb.insert(comb.end(), {static_cast<int32_t>(q), h, static_cast<int32_t>(n_slots - npieces), npieces});
        }
        if (used >= T - 0.5 && (!emit || c < grid - 1)) next();  // segment filled
      }
    }
    return c + (used > 0.0 ? 1 : 0);
  };
  // the optimum sits just above the even split line/grid: start with a tight
  // bracket and widen only if it is infeasible (halves the fill passes)
  double lo = std::max(double(line) / grid, double(ovh + min_piece) - 0.5);
  double hi = lo * 1.04 + double(ovh + min_piece) * 2.0;
  for (int64_t g2 = fill(hi, false); g2 > grid; g2 = fill(hi, false)) {
    lo = hi;
    hi *= 1.5;
  }
  for (int it = 0; it < 40 && hi - lo > 0.25; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (fill(mid, false) <= grid) hi = mid; else lo = mid;
  }
  int64_t used_ctas = fill(hi, true);
  if (overflow) return fail(PKV_VALUE_ERROR, "plan buffer too small for items");
  int c = static_cast<int>(std::min<int64_t>(used_ctas, grid));
  for (int cc = c; cc <= grid; ++cc) cta[cc] = static_cast<int32_t>(n_items);
  if (n_slots > 2 * int64_t(kMaxGrid)) return fail(PKV_CONFIG_ERROR, "too many partial slots");
  const int64_t comb_pos = items_pos + n_items * kItemInts;
  const int64_t ncomb = static_cast<int64_t>(comb.size() / kCombInts);
  const int64_t ctr_pos = comb_pos + int64_t(comb.size());
  if (ctr_pos + ncomb * kWarpsTc > cap) return fail(PKV_VALUE_ERROR, "plan buffer too small for comb");
  std::copy(comb.begin(), comb.end(), o + comb_pos);
  std::fill(o + ctr_pos, o + ctr_pos + ncomb * kWarpsTc, 0);
  o[H_TOTAL_ITEMS] = static_cast<int32_t>(n_items);
  o[H_NCOMB] = static_cast<int32_t>(comb.size() / kCombInts);
  o[H_GRID] = grid;
  o[H_CTA_OFF] = static_cast<int32_t>(o_cta(nq));
  o[H_ITEMS] = static_cast<int32_t>(items_pos);
  o[H_COMB] = static_cast<int32_t>(comb_pos);
  o[H_CTR] = static_cast<int32_t>(ctr_pos);
  if (n_out) *n_out = ctr_pos + ncomb * kWarpsTc;
  return PKV_OK;
}


// Programmatic dependent launch of the decode kernel behind the step's aux
// kernel (which triggers at its start): the decode prologue (plan staging,
// launch latency) overlaps the page clears / mirror update.  PKV_DECODE_PDL=0
// turns it off (A/B switch).
static bool pdl_on() {
  static const bool on = [] {
    const char* e = std::getenv("PKV_DECODE_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

static_assert(sizeof(TcParams) + sizeof(ClusterInline) + 16 <= sizeof(RecordedOp::args),
              "graph recorder argument buffer too small");
void preload_decode_tc_kernels() {
  touch_tc_kernels<__nv_bfloat16, 64>();
  touch_tc_kernels<__nv_bfloat16, 128>();
  touch_tc_kernels<__half, 64>();
  touch_tc_kernels<__half, 128>();
}

int launch_decode_tc(TcParams p, const int32_t* plan_host, int kv_dtype, int head_dim, int num_sms,
                     cudaStream_t stream) {
  const bool splitq = p.q_dtype == PKV_F32;
  const bool rows16 = plan_host[H_QGS] > 8 && p.group > 8;
  p.kv_dtype = kv_dtype;
  TcFn fn = nullptr;
  if (kv_dtype == PKV_BF16)
    fn = head_dim == 64 ? pick_rows<__nv_bfloat16, 64>(splitq, rows16) : pick_rows<__nv_bfloat16, 128>(splitq, rows16);
  else
    fn = head_dim == 64 ? pick_rows<__half, 64>(splitq, rows16) : pick_rows<__half, 128>(splitq, rows16);
  const int merge_bytes = kWarpsTc * kMergeRows * head_dim * 4 + kWarpsTc * kMergeRows * 2 * 4;
  // cluster mode with <= 64 queries: the plan-in-parameters instantiation
  const bool inline_plan = plan_host[H_CLUSTER] > 1 && p.nq <= 64;
  ClusterInline ci{};
  TcClusterFn fnc = nullptr;
  if (inline_plan) {
    ci.hb = plan_host[H_HB];
    ci.wph = plan_host[H_WPH];
    ci.qgs = plan_host[H_QGS];
    ci.qgroups = plan_host[H_QGROUPS];
    ci.head_items = plan_host[H_HEAD_ITEMS];
    ci.cluster = plan_host[H_CLUSTER];
    for (int i = 0; i < p.nq; ++i) {
      ci.nkrow[i] = plan_host[o_nk(p.nq) + i];
      ci.nkrow[p.nq + i] = plan_host[o_row(p.nq) + i];
    }
    if (kv_dtype == PKV_BF16)
      fnc = head_dim == 64 ? pick_rows_cluster<__nv_bfloat16, 64>(splitq, rows16)
                           : pick_rows_cluster<__nv_bfloat16, 128>(splitq, rows16);
    else
      fnc = head_dim == 64 ? pick_rows_cluster<__half, 64>(splitq, rows16)
                           : pick_rows_cluster<__half, 128>(splitq, rows16);
  }
  const void* fn_any = inline_plan ? reinterpret_cast<const void*>(fnc) : reinterpret_cast<const void*>(fn);
  const int64_t plan_bytes = o_cta(p.nq) * 4;
  p.plan_in_smem = p.nq <= kSmemPlanMax;
  p.merge_offset = p.plan_in_smem ? static_cast<int>((plan_bytes + 127) / 128 * 128) : 0;
  p.ring_offset = (p.merge_offset + merge_bytes + 1023) / 1024 * 1024;
  const int smem = p.ring_offset + kWarpsTc * kStagesTc * 2 * kCh * head_dim * 2;
  const int key = (kv_dtype == PKV_BF16) * 8 + (head_dim == 128) * 4 + splitq * 2 + rows16;
  {
    const cudaError_t e = ensure_smem(fn_any, smem);
    if (e != cudaSuccess)
      return fail(PKV_CUDA_ERROR, "decode_tc smem attribute (%d B): %s", smem, pkv::cuda_err_str(e));
  }
  const int grid = plan_host[H_GRID];  // the planner's assignment is per CTA
  const int cluster = plan_host[H_CLUSTER];
  cudaError_t e;
  if (cluster > 1) {
    static bool nonportable[32] = {false};
    const int k2 = key + 16 * inline_plan;
    if (!nonportable[k2]) {
      cudaFuncSetAttribute(fn_any, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      nonportable[k2] = true;
    }
  }
  if (launch_recorder()) {  // CUDA-graph mode of the batched step
    if (inline_plan)
      record_kernel(fnc, dim3(static_cast<unsigned>(grid)), dim3(kThreadsTc), static_cast<unsigned>(smem),
                    static_cast<unsigned>(cluster), p, ci);
    else
      record_kernel(fn, dim3(static_cast<unsigned>(grid)), dim3(kThreadsTc), static_cast<unsigned>(smem),
                    static_cast<unsigned>(cluster), p);
    return PKV_OK;
  }
  if (cluster > 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(kThreadsTc);
    cfg.dynamicSmemBytes = static_cast<size_t>(smem);
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(cluster);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pdl_on() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    static const bool debug_cluster = std::getenv("PKV_DEBUG_CLUSTER") != nullptr;
    if (debug_cluster) {
      int n = -1;
      cudaError_t oe = cudaOccupancyMaxActiveClusters(&n, fn_any, &cfg);
      std::fprintf(stderr, "pkv: cluster %d grid %d smem %d -> max active clusters %d (%s)\n", cluster, grid, smem,
                   n, cudaGetErrorString(oe));
    }
    e = inline_plan ? cudaLaunchKernelEx(&cfg, fnc, p, ci) : cudaLaunchKernelEx(&cfg, fn, p);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(kThreadsTc);
    cfg.dynamicSmemBytes = static_cast<size_t>(smem);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_on() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, fn, p);
  }
  if (e != cudaSuccess)
    return fail(PKV_CUDA_ERROR, "decode_tc launch: %s (grid %d cluster %d smem %d nq %d key %d)",
                pkv::cuda_err_str(e), grid, cluster, smem, p.nq, key);
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
    if (n >= 1024 * kTraceSlots + 256)  // the SM ids follow the timeline
      cudaMemcpyFromSymbol(out + 1024 * kTraceSlots, g_trace_sm, 256 * sizeof(unsigned long long));
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PKV_OK : fail(PKV_CUDA_ERROR, "debug trace: %s", pkv::cuda_err_str(e));
}

}  // namespace pkv
