// K2-TC: split-K paged decode on the tensor cores (mma.sync m16n8k16, bf16 /
// fp16 operands, fp32 accumulation) for 16-bit KV caches.
//
// Replaces the reference streaming kernel (attention.py:259-329) for bf16
// stores.  Decode is HBM bound (GQA-4 bf16: 4 flop/B, far below the ridge), so
// the tensor cores are used to cut *issue* cost, not for FLOPs: the CUDA-core
// kernel spends ~1200 instructions per 8 KiB chunk on unpacking, FMA chains
// and shuffles; here a 16-key chunk costs 16-32 HMMA + 16 LDSM + the softmax.
// tcgen05 is not used: M = G <= 16 query rows is not a dense contraction and
// the TMEM round trip would cost more than it saves.
//
// One warp = one work item (query, kv head, group of <= 16 query heads, key
// split).  Per warp a 3-stage cp.async ring stages 16 keys x D of K and V per
// stage with a 16-byte XOR swizzle (conflict-free LDSM); zero-fill past the
// valid keys.  The G grouped query heads are the M rows of the MMA, so every
// K/V byte is read from HBM once per group (GQA reuse).  Scores live in the
// log2 domain (q pre-scaled by scale*log2 e); P is rounded to the operand type
// for the P@V MMA and the softmax denominator sums the *rounded* P, so weights
// stay normalised.  fp32 queries are split hi+lo into two bf16 MMAs so the
// scores keep fp32 accuracy.
//
// Fused scheduling: every CTA plans the key splits from the per-query key
// counts in shared memory (no plan launch for n_queries <= kSmemPlanMax), and
// the last split of a (query, head group) to finish merges all partials in
// ascending split order (atomicInc counters that self-reset), so there is no
// combine launch and the result is deterministic.  Optional fused append: with
// k_new/v_new the last split of each query reads the new token from the input
// and writes it into its page (reshape-and-cache folded into the decode).
#include "common.cuh"
#include "decode_tc.h"

namespace pkv {
namespace {

constexpr int kWarpsTc = 8;
constexpr int kStagesTc = 3;
constexpr int kCh = 16;  // keys per chunk

struct Lds {
  // per-work-item constants shared by the issue lambda
};

template <typename T, int D, bool SPLITQ, bool ROWS16>
__global__ void __launch_bounds__(kWarpsTc * 32, 1) decode_tc_kernel(const __grid_constant__ TcParams p) {
  constexpr int ROWB = D * 2;            // smem row bytes
  constexpr int CPR = ROWB / 16;         // 16-B chunks per row (8 or 16)
  constexpr int LPR = CPR;               // lanes per row in the copy
  constexpr int RPI = 32 / LPR;          // rows per copy iteration
  constexpr int NIT = kCh / RPI;         // copy iterations per chunk
  constexpr int STAGE = 2 * kCh * ROWB;  // K + V
  constexpr int KS = D / 16;             // k-steps of Q K^T
  constexpr int NT = D / 8;              // n-tiles of P V
  static_assert(CPR >= 8 && CPR <= 32, "D must be 64 or 128");

  extern __shared__ __align__(1024) unsigned char smem[];
  int32_t* s_off = reinterpret_cast<int32_t*>(smem);
  __shared__ long long s_red[kWarpsTc];
  __shared__ int s_scan[kWarpsTc];
  __shared__ int s_hdr[2];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ps = 1 << p.log2ps;

  // ---------------- split plan (in-CTA, or from the global plan) ----------
  const int32_t* offsets;
  int split_pages, total_splits;
  if (p.plan_global) {
    offsets = p.plan_global + 4;
    split_pages = p.plan_global[0];
    total_splits = p.plan_global[1];
  } else {
    long long pages = 0;
    for (int i = threadIdx.x; i < p.nq; i += blockDim.x) pages += (p.q_nkeys[i] + ps - 1) >> p.log2ps;
#pragma unroll
    for (int o = 16; o; o >>= 1) pages += __shfl_xor_sync(0xffffffffu, pages, o);
    if (lane == 0) s_red[warp] = pages;
    __syncthreads();
    long long tot = 0;
#pragma unroll
    for (int w = 0; w < kWarpsTc; ++w) tot += s_red[w];
    long long sp = (tot * p.head_items + p.target_items - 1) / p.target_items;
    const long long cap = (tot + kMaxExtraSplitsTc - 1) / kMaxExtraSplitsTc;
    sp = sp < cap ? cap : sp;
    sp = sp < 1 ? 1 : sp;
    split_pages = static_cast<int>(sp);
    int carry = 0;
    for (int base = 0; base < p.nq; base += blockDim.x) {
      const int i = base + threadIdx.x;
      int cnt = 0;
      if (i < p.nq) cnt = static_cast<int>((((p.q_nkeys[i] + ps - 1) >> p.log2ps) + sp - 1) / sp);
      int x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_scan[warp] = x;
      __syncthreads();
      int before = 0, all = 0;
#pragma unroll
      for (int w = 0; w < kWarpsTc; ++w) {
        before += w < warp ? s_scan[w] : 0;
        all += s_scan[w];
      }
      if (i < p.nq) s_off[i] = carry + before + x - cnt;
      carry += all;
      __syncthreads();
    }
    if (threadIdx.x == 0) s_off[p.nq] = carry;
    __syncthreads();
    offsets = s_off;
    total_splits = carry;
  }

  unsigned char* ring = smem + p.ring_offset + warp * (kStagesTc * STAGE);
  const uint32_t ring_addr = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  const int t4 = lane & 3, g = lane >> 2;
  const int64_t total_items = int64_t(total_splits) * p.head_items;
  const int64_t nwarps = int64_t(gridDim.x) * kWarpsTc;

  for (int64_t w = int64_t(blockIdx.x) * kWarpsTc + warp; w < total_items; w += nwarps) {
    const int sg = static_cast<int>(w / p.head_items);
    const int hi = static_cast<int>(w - int64_t(sg) * p.head_items);
    const int kvh = hi / p.qgroups;
    const int qg = hi - kvh * p.qgroups;
    const int qh0 = kvh * p.group + qg * 16;
    const int rows = min(16, p.group - qg * 16);
    int lo = 0, hq_ = p.nq;  // query owning split sg
    while (hq_ - lo > 1) {
      const int mid = (lo + hq_) >> 1;
      if (offsets[mid] <= sg) lo = mid; else hq_ = mid;
    }
    const int qi = lo;
    const int split = sg - offsets[qi];
    const int nsplit = offsets[qi + 1] - offsets[qi];
    const int nk = p.q_nkeys[qi];
    const int sv = p.q_seq[qi];
    const int kb = split * split_pages * ps;
    const int ke = min(nk, kb + split_pages * ps);
    const int n_chunks = (ke - kb + kCh - 1) / kCh;
    const int64_t bt_off = p.bt ? int64_t(p.seq_row[sv]) * p.bt_stride : 0;
    const int64_t gstart = p.bt ? 0 : p.seq_start[sv];
    const int npages_seq = (nk + ps - 1) >> p.log2ps;
    const bool fuse_new = p.k_new != nullptr && split == nsplit - 1;
    const int64_t head_off = int64_t(kvh) * ROWB;
    const char* knew = fuse_new ? p.k_new + (int64_t(qi) * p.hkv) * ROWB + head_off : nullptr;
    const char* vnew = fuse_new ? p.v_new + (int64_t(qi) * p.hkv) * ROWB + head_off : nullptr;

    // ---- fused append: write the new token's head slice into its page
    if (fuse_new) {
      const int pos = nk - 1;
      const int64_t page = p.bt[bt_off + (pos >> p.log2ps)];
      const int64_t dst = (page * ps + (pos & (ps - 1))) * p.row_stride + head_off;
      if (lane < CPR) {
        reinterpret_cast<uint4*>(p.kw + dst)[lane] = reinterpret_cast<const uint4*>(knew)[lane];
        reinterpret_cast<uint4*>(p.vw + dst)[lane] = reinterpret_cast<const uint4*>(vnew)[lane];
      }
    }

    // ---- Q fragments (A operand), pre-scaled into the log2 domain
    uint32_t qa[KS][4];
    uint32_t qb[SPLITQ ? KS : 1][4];
    {
      const int64_t qbase = int64_t(qi) * p.hq + qh0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int row = g + ((h & 1) ? 8 : 0);
          const int d = ks * 16 + ((h & 2) ? 8 : 0) + 2 * t4;
          float x0 = 0.f, x1 = 0.f;
          if (row < rows) {
            const int64_t off = (qbase + row) * D + d;
            x0 = load_as_float(p.q, off, p.q_dtype) * p.qscale;
            x1 = load_as_float(p.q, off + 1, p.q_dtype) * p.qscale;
          }
          qa[ks][h] = pack2<T>(x0, x1);
          if constexpr (SPLITQ) qb[ks][h] = pack2<T>(x0 - round_to<T>(x0), x1 - round_to<T>(x1));
        }
      }
    }

    // ---- block-table window (lane i holds logical page win + i)
    int win = -1, win_val = 0;
    // copy geometry of this lane
    const int cc = lane % LPR;
    const int r0 = lane / LPR;

    auto issue = [&](int c) {
      const int stage = c % kStagesTc;
      const int k0 = kb + c * kCh;
      const int nvalid = min(kCh, ke - k0);
      int rowidx = 0;  // cache row of key k0 + lane (lane < kCh)
      if (p.bt) {
        const int plo = k0 >> p.log2ps, phi = (k0 + kCh - 1) >> p.log2ps;
        if (win < 0 || phi - win >= 32) {
          win = plo;
          const int idx = plo + lane;
          win_val = idx < npages_seq ? p.bt[bt_off + idx] : 0;
        }
        const int key = k0 + lane;
        int src = (key >> p.log2ps) - win;
        src = src < 0 ? 0 : (src > 31 ? 31 : src);
        const int page = __shfl_sync(0xffffffffu, win_val, src);
        rowidx = page * ps + (key & (ps - 1));
      } else {
        rowidx = static_cast<int>(gstart + k0 + lane);
      }
      const uint32_t kdst = ring_addr + stage * STAGE;
      const uint32_t vdst = kdst + kCh * ROWB;
#pragma unroll
      for (int it = 0; it < NIT; ++it) {
        const int r = r0 + it * RPI;
        const int row = __shfl_sync(0xffffffffu, rowidx, r);
        const bool ok = r < nvalid;
        const char* ks_ = p.k + int64_t(row) * p.row_stride + head_off + cc * 16;
        const char* vs_ = p.v + int64_t(row) * p.row_stride + head_off + cc * 16;
        if (fuse_new && k0 + r == nk - 1) {
          ks_ = knew + cc * 16;
          vs_ = vnew + cc * 16;
        }
        const uint32_t soff = r * ROWB + ((cc ^ (r & 7)) << 4);
        cp_async<16>(kdst + soff, ok ? ks_ : p.k, ok ? 16 : 0);
        cp_async<16>(vdst + soff, ok ? vs_ : p.v, ok ? 16 : 0);
      }
    };

    float o[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

#pragma unroll
    for (int c = 0; c < kStagesTc - 1; ++c) {
      if (c < n_chunks) issue(c);
      cp_async_commit();
    }
    for (int c = 0; c < n_chunks; ++c) {
      cp_async_wait<kStagesTc - 2>();
      __syncwarp();
      if (c + kStagesTc - 1 < n_chunks) issue(c + kStagesTc - 1);
      cp_async_commit();
      const uint32_t kbase = ring_addr + (c % kStagesTc) * STAGE;
      const uint32_t vbase = kbase + kCh * ROWB;

      // S = Q K^T for 16 keys: two n-tiles (keys 0-7, 8-15)
      float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
      {
        const int m = lane >> 3;
        const int key = ((m >> 1) << 3) + (lane & 7);
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int chunk = 2 * ks + (m & 1);
          uint32_t b00, b01, b10, b11;
          ldmatrix_x4(kbase + key * ROWB + ((chunk ^ (key & 7)) << 4), b00, b01, b10, b11);
          mma_16816<T>(s0, qa[ks], b00, b01);
          mma_16816<T>(s1, qa[ks], b10, b11);
          if constexpr (SPLITQ) {
            mma_16816<T>(s0, qb[ks], b00, b01);
            mma_16816<T>(s1, qb[ks], b10, b11);
          }
        }
      }
      // mask keys beyond the split
      const int kk = kb + c * kCh + 2 * t4;
      const int lim = ke - kk;  // keys kk+e valid iff e < lim
      if (lim < 10) {
        if (lim <= 0) { s0[0] = s0[2] = -INFINITY; }
        if (lim <= 1) { s0[1] = s0[3] = -INFINITY; }
        if (lim <= 8) { s1[0] = s1[2] = -INFINITY; }
        if (lim <= 9) { s1[1] = s1[3] = -INFINITY; }
      }
      // online softmax, row g (s*[0..1]) and row g+8 (s*[2..3])
      float mx0 = fmaxf(fmaxf(s0[0], s0[1]), fmaxf(s1[0], s1[1]));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      const float mn0 = fmaxf(m0, mx0);
      const float c0 = exp2f(m0 - mn0);
      m0 = mn0;
      uint32_t pa[4];
      {
        const float p00 = exp2f(s0[0] - mn0), p01 = exp2f(s0[1] - mn0);
        const float p10 = exp2f(s1[0] - mn0), p11 = exp2f(s1[1] - mn0);
        pa[0] = pack2<T>(p00, p01);
        pa[2] = pack2<T>(p10, p11);
        l0 = l0 * c0 + (round_to<T>(p00) + round_to<T>(p01)) + (round_to<T>(p10) + round_to<T>(p11));
      }
      float c1 = 1.f;
      if constexpr (ROWS16) {
        float mx1 = fmaxf(fmaxf(s0[2], s0[3]), fmaxf(s1[2], s1[3]));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
        const float mn1 = fmaxf(m1, mx1);
        c1 = exp2f(m1 - mn1);
        m1 = mn1;
        const float p02 = exp2f(s0[2] - mn1), p03 = exp2f(s0[3] - mn1);
        const float p12 = exp2f(s1[2] - mn1), p13 = exp2f(s1[3] - mn1);
        pa[1] = pack2<T>(p02, p03);
        pa[3] = pack2<T>(p12, p13);
        l1 = l1 * c1 + (round_to<T>(p02) + round_to<T>(p03)) + (round_to<T>(p12) + round_to<T>(p13));
      } else {
        pa[1] = pa[3] = 0u;
      }
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        o[n][0] *= c0;
        o[n][1] *= c0;
        if constexpr (ROWS16) {
          o[n][2] *= c1;
          o[n][3] *= c1;
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
    cp_async_wait<0>();
    __syncwarp();

    // quad-reduce the denominators (each lane summed its own keys)
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    if constexpr (ROWS16) {
      l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
      l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    }

    if (nsplit == 1) {
      const float inv0 = 1.f / l0, inv1 = ROWS16 ? 1.f / l1 : 0.f;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int d = n * 8 + 2 * t4;
        if (g < rows) {
          const int64_t off = (int64_t(qi) * p.hq + qh0 + g) * D + d;
          store_from_float(p.out, off, p.out_dtype, o[n][0] * inv0);
          store_from_float(p.out, off + 1, p.out_dtype, o[n][1] * inv0);
        }
        if (ROWS16 && g + 8 < rows) {
          const int64_t off = (int64_t(qi) * p.hq + qh0 + g + 8) * D + d;
          store_from_float(p.out, off, p.out_dtype, o[n][2] * inv1);
          store_from_float(p.out, off + 1, p.out_dtype, o[n][3] * inv1);
        }
      }
      continue;
    }

    // ---- split partials + last-arriver merge
    {
      const int64_t slot0 = int64_t(sg) * p.hq + qh0;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int d = n * 8 + 2 * t4;
        if (g < rows) {
          float2* dst = reinterpret_cast<float2*>(p.ws_o + (slot0 + g) * D + d);
          __stcg(dst, make_float2(o[n][0], o[n][1]));
        }
        if (ROWS16 && g + 8 < rows) {
          float2* dst = reinterpret_cast<float2*>(p.ws_o + (slot0 + g + 8) * D + d);
          __stcg(dst, make_float2(o[n][2], o[n][3]));
        }
      }
      if (t4 == 0) {
        if (g < rows) __stcg(reinterpret_cast<float2*>(p.ws_ml) + slot0 + g, make_float2(m0, l0));
        if (ROWS16 && g + 8 < rows)
          __stcg(reinterpret_cast<float2*>(p.ws_ml) + slot0 + g + 8, make_float2(m1, l1));
      }
    }
    __threadfence();
    __syncwarp();
    unsigned prev = 0;
    if (lane == 0) prev = atomicInc(p.counters + (int64_t(qi) * p.head_items + hi), nsplit - 1);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev != static_cast<unsigned>(nsplit - 1)) continue;
    __threadfence();
    const int s0_ = offsets[qi];
    for (int row = 0; row < rows; ++row) {
      float mx = -INFINITY;
      for (int s = 0; s < nsplit; ++s)
        mx = fmaxf(mx, __ldcg(reinterpret_cast<const float2*>(p.ws_ml) + (int64_t(s0_ + s) * p.hq + qh0 + row)).x);
      float den = 0.f;
      float acc[D / 32];
#pragma unroll
      for (int e = 0; e < D / 32; ++e) acc[e] = 0.f;
      for (int s = 0; s < nsplit; ++s) {
        const int64_t slot = int64_t(s0_ + s) * p.hq + qh0 + row;
        const float2 ml = __ldcg(reinterpret_cast<const float2*>(p.ws_ml) + slot);
        const float wgt = exp2f(ml.x - mx);
        den += wgt * ml.y;
#pragma unroll
        for (int e = 0; e < D / 32; ++e) acc[e] += wgt * __ldcg(p.ws_o + slot * D + lane + 32 * e);
      }
      const float inv = 1.f / den;
      const int64_t off = (int64_t(qi) * p.hq + qh0 + row) * D;
#pragma unroll
      for (int e = 0; e < D / 32; ++e) store_from_float(p.out, off + lane + 32 * e, p.out_dtype, acc[e] * inv);
    }
  }
}

template <typename T, int D>
TcFn pick_rows(bool splitq, bool rows16) {
  if (splitq) return rows16 ? decode_tc_kernel<T, D, true, true> : decode_tc_kernel<T, D, true, false>;
  return rows16 ? decode_tc_kernel<T, D, false, true> : decode_tc_kernel<T, D, false, false>;
}

}  // namespace

bool decode_tc_supported(int kv_dtype, int head_dim) {
  return (kv_dtype == PKV_BF16 || kv_dtype == PKV_F16) && (head_dim == 64 || head_dim == 128);
}

int decode_tc_smem_bytes(int head_dim, int64_t nq) {
  const int plan = nq <= kSmemPlanMax ? static_cast<int>((nq + 1) * 4) : 0;
  const int plan_al = (plan + 1023) / 1024 * 1024;
  return plan_al + kWarpsTc * kStagesTc * 2 * kCh * head_dim * 2;
}

int launch_decode_tc(TcParams p, int kv_dtype, int head_dim, int num_sms, cudaStream_t stream) {
  const bool splitq = p.q_dtype == PKV_F32;
  const bool rows16 = p.group > 8;
  TcFn fn = nullptr;
  if (kv_dtype == PKV_BF16)
    fn = head_dim == 64 ? pick_rows<__nv_bfloat16, 64>(splitq, rows16) : pick_rows<__nv_bfloat16, 128>(splitq, rows16);
  else
    fn = head_dim == 64 ? pick_rows<__half, 64>(splitq, rows16) : pick_rows<__half, 128>(splitq, rows16);
  const int plan = p.plan_global ? 0 : static_cast<int>((p.nq + 1) * 4);
  p.ring_offset = (plan + 1023) / 1024 * 1024;
  const int smem = p.ring_offset + kWarpsTc * kStagesTc * 2 * kCh * head_dim * 2;
  static int configured[16] = {0};
  const int key = (kv_dtype == PKV_BF16) * 8 + (head_dim == 128) * 4 + splitq * 2 + rows16;
  if (configured[key] < smem) {
    cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    configured[key] = 227 * 1024;
  }
  fn<<<num_sms, kWarpsTc * 32, smem, stream>>>(p);
  return cudaGetLastError() == cudaSuccess ? PKV_OK : PKV_CUDA_ERROR;
}

int decode_tc_warps() { return kWarpsTc; }

}  // namespace pkv
