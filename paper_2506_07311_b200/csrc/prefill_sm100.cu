// K3: paged causal / suffix prefill attention on the 5th-generation tensor
// cores (tcgen05.mma, accumulators in TMEM, operands staged by TMA).
//
// Replaces the reference streaming kernel (attention.py:259-329) for the
// self-attention and suffix metas (attention.py:81-84, 98-110) of 16-bit
// caches: there the query tile times the key page really is a dense
// contraction.
//
// Work item (planned on the host, pkv_prefill_plan): one kv head of one tile
// of QT = 128 / G consecutive query positions of one sequence.  The item's
// 128 query rows are the M dimension of the MMAs: row r = i * G + g is query
// position q0 + i of query head kvh * G + g, so every K/V byte staged in
// shared memory serves all G grouped query heads.  Keys stream in tiles of
// 128 (N); each tile is gathered page by page from the paged cache with 3-D
// TMA boxes (64 head-dim elements x 1 head x min(ps, 128) rows, 128-byte
// swizzle) straight into the canonical K-major layout the MMA descriptors
// describe.  Pages past the end of the block table are fetched with an
// out-of-range row coordinate, which TMA fills with zeros.
//
// Warp roles (384 threads, one CTA per SM; see the kernel comment):
//   warp 0     TMA producer: Q (two query tiles) once, then 128-key K/V tiles
//              through a 2-stage ring (a tile whose pages form one contiguous
//              run is one 128-row box per chunk);
//   warps 1, 3 MMA issuers (one elected lane each), one per query tile: QK
//              of 64-key sub-tiles into double-buffered S, PV from P in TMEM;
//   warp 2     TMEM allocator (512 columns: S_A[2], S_B[2], O_A, O_B);
//   warps 4-11 two softmax + epilogue warpgroups, one per query tile: thread
//              = query row (TMEM lane), so row max / sum need no shuffles.
//              Online softmax in base 2 with a lazily updated running max:
//              O and l are rescaled only when the row max grows by more than
//              2^8 (exact — numerator and denominator share the stale max —
//              and rare after the first sub-tiles).  P is rounded to the
//              operand type and written over its S columns in TMEM.
//
// Causal masking is applied only on tiles that reach past a row's last
// allowed key; tiles entirely above the diagonal are never visited (the
// host plan sizes each item's key range).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace pkv {
namespace {

constexpr int kThreads = 384;  // 4 control warps + 2 softmax warpgroups
constexpr int kM = 128;          // query rows per item (MMA M)
constexpr int kN = 128;          // keys per tile (MMA N of QK^T, K of PV)
constexpr int kRowB = 128;       // bytes per swizzled row (64 x 16-bit)
constexpr int kChunkB = kM * kRowB;  // one 64-column chunk of a 128-row tile: 16 KB
constexpr int kItemInts = 10;
constexpr float kLog2eP = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
#ifndef PKV_K3_EMU
#define PKV_K3_EMU 1
#endif
#ifndef PKV_K3_EMU_PERIOD
#define PKV_K3_EMU_PERIOD 16
#endif
// of every kEmuPeriod packed pairs of scores, how many take the FMA-pipe
// exp2 below instead of MUFU.EX2 (16 / clk / SM, the softmax's bound once
// both query tiles' softmaxes run concurrently; period over the 32 pairs
// of a 64-key sub-tile row)
constexpr int kEmuPairs = PKV_K3_EMU;
constexpr int kEmuPeriod = PKV_K3_EMU_PERIOD;

// ---- PTX wrappers -----------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ unsigned long long gtime();
// Debug builds (-DPKV_K3_WATCHDOG): a wait that has not completed after ~4 s
// is a scheduling bug: report the barrier and trap instead of hanging the
// device.  Off by default: the extra registers in every inlined wait cost
// ~14% of K3 throughput (measured).
__device__ __noinline__ void mbar_hang(uint32_t bar, uint32_t parity) {
  printf("pkv K3: mbarrier wait timed out (smem 0x%x parity %u) block %d thread %d\n", bar, parity,
         static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));
  asm volatile("trap;");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
#ifdef PKV_K3_WATCHDOG
  uint32_t spins = 0;
  unsigned long long t0 = 0;
#endif
  for (;;) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
#ifdef PKV_K3_WATCHDOG
    if ((++spins & 0xfff) == 0) {
      const unsigned long long now = gtime();
      if (t0 == 0) t0 = now;
      else if (now - t0 > 4000000000ull) mbar_hang(bar, parity);
    }
#endif
  }
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
               : "memory");
}
// Warp-collective issue: every lane of the warp executes these with
// identical (warp-uniform) operands and one elected lane issues the
// instruction — operands then live in uniform registers instead of being
// serialised through a per-lane waterfall loop (measured ~75 cycles per MMA
// when issued from a single divergent lane).
__device__ __forceinline__ void tc_mma_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_mma_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint32_t bar) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 32 consecutive 32-bit TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
      "[%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, "
      "%32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// shared-memory matrix descriptor, 128-byte swizzle (layout type 2), sm100 version 1
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}
// instruction descriptor of kind::f16: fp32 accumulate, 16-bit A/B of
// format fmt (0 = f16, 1 = bf16), K-major A, B major b_mn, shape M x N
__host__ __device__ constexpr uint32_t instr_desc(uint32_t fmt, uint32_t b_mn, uint32_t m, uint32_t n) {
  return (1u << 4) | (fmt << 7) | (fmt << 10) | (b_mn << 16) | ((n >> 3) << 17) | ((m >> 4) << 24);
}

struct PrefillParams {
  int hq, hkv, group, qt;  // qt = query positions per item
  int log2ps, box_rows;     // keys per TMA box = min(page_size, 128)
  int64_t bt_stride;
  const int32_t* bt;
  int32_t oob_row;          // a row coordinate past the cache: zero-filled box
  float qscale;             // scale * log2(e)
  int causal;
  void* out;
  int out_dtype;
  const int32_t* items;
  int o_cols;               // > 0: full tiles leave by TMA stores of o_cols-column boxes (tm_o)
  unsigned long long* dbg;  // debug timeline of CTA 0 (nullptr = off)
};
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PDBG(slot) \
  do {             \
    if (p.dbg && blockIdx.x == 0) p.dbg[slot] = gtime(); \
  } while (0)

// 2^x on the FMA pipe for two lanes: x = i + f with i = round(x) (the
// 1.5 * 2^23 magic add leaves i in the low mantissa bits), 2^f by a degree-3
// polynomial on [-0.5, 0.5] (max relative error 1.0e-4, below the 2^-9 of
// the 16-bit P it feeds), then i is added to the exponent field.  x is
// clamped to >= -125 so the exponent stays normal (2^-125 ~ 0 next to the
// row maximum's 1; masked -inf scores land there too).
__device__ __forceinline__ float2 ex2_emu2(float2 x) {
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 j = fadd2(x, make_float2(12582912.f, 12582912.f));
  const float2 i = fadd2(j, make_float2(-12582912.f, -12582912.f));
  const float2 f = ffma2(i, make_float2(-1.f, -1.f), x);
  float2 pv = ffma2(f, make_float2(0.05500882f, 0.05500882f), make_float2(0.24221077f, 0.24221077f));
  pv = ffma2(pv, f, make_float2(0.69328291f, 0.69328291f));
  pv = ffma2(pv, f, make_float2(1.f, 1.f));
  return make_float2(__int_as_float(__float_as_int(pv.x) + (__float_as_int(j.x) << 23)),
                     __int_as_float(__float_as_int(pv.y) + (__float_as_int(j.y) << 23)));
}

template <typename T>
struct Fmt;
template <>
struct Fmt<__nv_bfloat16> {
  static constexpr uint32_t kFmt = 1;
};
template <>
struct Fmt<__half> {
  static constexpr uint32_t kFmt = 0;
};

// tcgen05.mma with the A operand (P) read from tensor memory
__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 16 consecutive 32-bit TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

// Two query tiles (A: item rows 0-127, B: rows 128-255) share every K/V
// tile; scores come in 64-key sub-tiles with S double-buffered per query
// tile, so QK of sub-tile u + 1 runs on the tensor core while the softmax
// works on sub-tile u: the per-tile chain softmax -> PV -> QK is off the
// critical path (a 128-key S per tile left the tensor core and the SFU each
// ~50% busy, profiles/r02/k3_experiments.md).  TMEM: S_A[2] | S_B[2] (64
// columns each) | O_A | O_B = 512 columns; P_t(u) (16-bit) overwrites the
// first 32 columns of S_t[u & 1].  K/V still arrive in 128-key tiles (2
// stages); sub-tile u uses half u & 1 of tile u >> 1.  Issue order of the
// MMA thread per sub-tile u and query tile t: PV_t(u) (behind P_t(u)), then
// QK_t(u + 2) into the buffer PV_t(u) has just read.  A lazy rescale of O_t
// must follow PV_t(u - 1): every sub-tile waits for the previous PV (long
// complete by then) before publishing its P.
template <typename T, int D>
__global__ void __launch_bounds__(kThreads, 1)
    prefill_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_k128,
                     const __grid_constant__ CUtensorMap tm_v128, const __grid_constant__ CUtensorMap tm_o,
                     const __grid_constant__ PrefillParams p) {
  constexpr int NCH = D / 64;
  constexpr int kQBytes = NCH * kChunkB;
  constexpr int kKVBytes = NCH * kChunkB;
  constexpr int kS = 64;  // keys per score sub-tile
  constexpr uint32_t kIdescQK = instr_desc(Fmt<T>::kFmt, 0, kM, kS);
  constexpr uint32_t kIdescPV = instr_desc(Fmt<T>::kFmt, 1, kM, D);
  constexpr uint32_t kTmemCols = 512;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sQ = smem_addr(smem);
  const uint32_t sK = sQ + 2 * kQBytes;
  const uint32_t sV = sK + 2 * kKVBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * kQBytes + 4 * kKVBytes);
  // SF / PF: [tile t][buffer b] at + 2t + b
  // OD: [tile t][parity of u] at + 2t + (u & 1): PV_t(u) complete.  Two
  // alternating barriers per tile let the softmax skip the wait when no
  // row rescales: PV_t(u + 2), the next completion on a barrier, cannot be
  // issued before the softmax publishes P_t(u + 2), so a later wait never
  // sees a barrier two phases ahead
  // KE / VE: [issuer (query tile) t][stage s] at + 2t + s: tile t's MMAs no
  // longer read that stage (each issuer releases only the K / V tiles its
  // query tile uses; the producer waits for the tiles' users)
  enum { B_Q = 0, B_KF = 1, B_VF = 3, B_KE = 5, B_VE = 9, B_SF = 13, B_PF = 17, B_OD = 21, B_N = 25 };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + B_N);
  auto bar = [&](int i) { return smem_addr(bars + i); };

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int32_t* it = p.items + static_cast<int64_t>(blockIdx.x) * kItemInts;
  const int q_row0 = it[0], qpos0 = it[3], kv_len = it[4];
  const int mrow = it[5], kvh = it[6];
  const int cnt[2] = {it[1], it[2]};
  const int nt[2] = {it[7], it[8]};
  const int n_tiles = max(nt[0], nt[1]);
  const int nu[2] = {2 * nt[0], 2 * nt[1]};
  const int n_issuers = nt[1] > 0 ? 2 : 1;  // tile A always has work

  if (p.dbg && threadIdx.x == 0) {  // per-CTA record: start, first S, end, SM
    p.dbg[512 + 4 * blockIdx.x] = gtime();
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.dbg[512 + 4 * blockIdx.x + 3] = smid;
  }
  if (threadIdx.x == 0) {
    mbar_init(bar(B_Q), 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar(B_KF + s), 1);
      mbar_init(bar(B_VF + s), 1);
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(bar(B_KE + s), 1);
      mbar_init(bar(B_VE + s), 1);
      mbar_init(bar(B_SF + s), 1);
      mbar_init(bar(B_PF + s), 128);
      mbar_init(bar(B_OD + s), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    // Q goes out right away, overlapping the TMEM allocation and the barrier
    const int ntiles_q = cnt[1] > 0 ? 2 : 1;
    mbar_expect_tx(bar(B_Q), kQBytes * ntiles_q);
    for (int t = 0; t < ntiles_q; ++t)
      for (int c = 0; c < NCH; ++c)
        tma_load_3d(sQ + t * kQBytes + c * kChunkB, &tm_q, bar(B_Q), c * 64, kvh * p.group, q_row0 + t * p.qt);
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_addr(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (128-key K/V tiles, 2 stages) ----------------
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tm_k)) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tm_v)) : "memory");
      const int ps = 1 << p.log2ps;
      const int n_pages = (kv_len + ps - 1) >> p.log2ps;
      const int boxes = kN / p.box_rows;
      const int32_t* tbl = p.bt ? p.bt + static_cast<int64_t>(mrow) * p.bt_stride : nullptr;
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j & 1;
        int rows[16];
        bool run = p.bt != nullptr && boxes > 1;
        for (int b = 0; b < boxes; ++b) {
          const int key0 = j * kN + b * p.box_rows;
          if (p.bt) {
            const int pg = key0 >> p.log2ps;
            rows[b] = pg < n_pages ? tbl[pg] * ps + (key0 & (ps - 1)) : p.oob_row;
            run = run && pg < n_pages && rows[b] == rows[0] + b * p.box_rows;
          } else {
            rows[b] = mrow + key0;
          }
        }
        const CUtensorMap* mk = run ? &tm_k128 : &tm_k;
        const CUtensorMap* mv = run ? &tm_v128 : &tm_v;
        const int nb = run ? 1 : boxes;
        // stage st last held tile j - 2: wait for the query tiles that read it
        if (j >= 2)
          for (int t = 0; t < 2; ++t)
            if (j - 2 < nt[t]) mbar_wait(bar(B_KE + 2 * t + st), ((j >> 1) - 1) & 1);
        mbar_expect_tx(bar(B_KF + st), kKVBytes);
        for (int b = 0; b < nb; ++b)
          for (int c = 0; c < NCH; ++c)
            tma_load_3d(sK + st * kKVBytes + c * kChunkB + b * p.box_rows * kRowB, mk, bar(B_KF + st), c * 64, kvh,
                        rows[b]);
        if (j >= 2)
          for (int t = 0; t < 2; ++t)
            if (j - 2 < nt[t]) mbar_wait(bar(B_VE + 2 * t + st), ((j >> 1) - 1) & 1);
        mbar_expect_tx(bar(B_VF + st), kKVBytes);
        for (int b = 0; b < nb; ++b)
          for (int c = 0; c < NCH; ++c)
            tma_load_3d(sV + st * kKVBytes + c * kChunkB + b * p.box_rows * kRowB, mv, bar(B_VF + st), c * 64, kvh,
                        rows[b]);
      }
    }
  } else if (warp == 1 || (warp == 3 && n_issuers == 2)) {
    // ---------------- MMA issuers: warp 1 for query tile A, warp 3 for B ----------------
    // one issuing warp per query tile: a tile's PV / QK never queue behind the
    // other tile's softmax; K / V stages are released by both issuers
    const int t = warp == 1 ? 0 : 1;
    const uint32_t uQ = __shfl_sync(0xffffffffu, sQ, 0), uK = __shfl_sync(0xffffffffu, sK, 0);
    const uint32_t uV = __shfl_sync(0xffffffffu, sV, 0), uT = __shfl_sync(0xffffffffu, tmem, 0);
    mbar_wait(bar(B_Q), 0);
    tc_fence_after();
    int k_waited = -1, v_waited = -1;  // last K / V tile whose full barrier was waited
    auto need_k = [&](int j) {
      if (j > k_waited) {
        mbar_wait(bar(B_KF + (j & 1)), (j >> 1) & 1);
        tc_fence_after();
        k_waited = j;
      }
    };
    auto need_v = [&](int j) {
      if (j > v_waited) {
        mbar_wait(bar(B_VF + (j & 1)), (j >> 1) & 1);
        tc_fence_after();
        v_waited = j;
      }
    };
    // S_t[u & 1] = Q_t K(u)^T over the 64 keys of sub-tile u
    auto issue_qk = [&](int t, int u) {
      const int j = u >> 1, st = j & 1, h = u & 1;
      need_k(j);
#pragma unroll
      for (int k = 0; k < D / 16; ++k) {
        const uint64_t ad = smem_desc(uQ + t * kQBytes + (k >> 2) * kChunkB + (k & 3) * 32, 16, 1024);
        const uint64_t bd =
            smem_desc(uK + st * kKVBytes + (k >> 2) * kChunkB + h * kS * kRowB + (k & 3) * 32, 16, 1024);
        tc_mma_elect(uT + t * 2 * kS + h * kS, ad, bd, kIdescQK, k > 0 ? 1u : 0u);
      }
      tc_commit_elect(bar(B_SF + 2 * t + h));
    };
    // O_t += P_t(u) V(u): P in the first 32 columns of S_t[u & 1]
    auto issue_pv = [&](int t, int u) {
      const int j = u >> 1, st = j & 1, h = u & 1;
      need_v(j);
      mbar_wait(bar(B_PF + 2 * t + h), (u >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int k = 0; k < kS / 16; ++k) {
        const uint64_t bd = smem_desc(uV + st * kKVBytes + (h * kS + k * 16) * kRowB, kChunkB, 1024);
        tc_mma_ts_elect(uT + 4 * kS + t * D, uT + t * 2 * kS + h * kS + k * 8, bd, kIdescPV,
                        (u > 0 || k > 0) ? 1u : 0u);
      }
      tc_commit_elect(bar(B_OD + 2 * t + h));
    };
    // this tile's sub-tiles: nu[t] = 2 nt[t] (even); K tile j is read by
    // QK(2j), QK(2j + 1), V tile j by PV(2j), PV(2j + 1)
    for (int u = 0; u < 2 && u < nu[t]; ++u) issue_qk(t, u);
    tc_commit_elect(bar(B_KE + 2 * t + 0));  // K tile 0 read (nt[t] >= 1)
    for (int u = 0; u < nu[t]; ++u) {
      issue_pv(t, u);
      if (u & 1) tc_commit_elect(bar(B_VE + 2 * t + ((u >> 1) & 1)));  // V tile u >> 1 read
      if (u + 2 < nu[t]) {
        issue_qk(t, u + 2);
        if (u & 1) tc_commit_elect(bar(B_KE + 2 * t + (((u + 2) >> 1) & 1)));  // K tile (u + 2) >> 1 read
      }
    }
  } else if (warp >= 4) {
    // ---------------- softmax + epilogue ----------------
    const int t = (warp - 4) >> 2;
    const int r = threadIdx.x - 128 - 128 * t;
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tO = tmem + lane_base + 4 * kS + t * D;
    const int qi = r / p.group;
    const int qpos = qpos0 + t * p.qt + qi;
    const int nk = p.causal ? min(qpos + 1, kv_len) : kv_len;
    float m_used = -INFINITY, l = 0.f;
    const float2 qs2 = make_float2(p.qscale, p.qscale);
#ifdef PKV_K3_PHASES
    long long ph[5] = {0, 0, 0, 0, 0}, pc = clock64();
#define PHASE(k)                      \
  do {                                \
    const long long now_ = clock64(); \
    ph[k] += now_ - pc;               \
    pc = now_;                        \
  } while (0)
#else
#define PHASE(k) \
  do {           \
  } while (0)
#endif
    for (int u = 0; u < nu[t]; ++u) {
      const int h = u & 1;
      const uint32_t tS = tmem + lane_base + t * 2 * kS + h * kS;
      mbar_wait(bar(B_SF + 2 * t + h), (u >> 1) & 1);
      tc_fence_after();
      PHASE(0);
      if (r == 0 && u < 64) PDBG(t * 64 + u);
      if (p.dbg && r == 0 && t == 0 && u == 0) p.dbg[512 + 4 * blockIdx.x + 1] = gtime();
      const int kbase = u * kS;
      const bool masked = __any_sync(0xffffffffu, kbase + kS > nk);
      uint32_t v[kS];
#pragma unroll
      for (int c = 0; c < kS / 32; ++c) tmem_ld32(tS + c * 32, v + 32 * c);
      tmem_wait_ld();
      PHASE(1);
      if (masked) {
        const int lim = nk - kbase;
#pragma unroll
        for (int e = 0; e < kS; ++e)
          if (e >= lim) v[e] = __float_as_uint(-INFINITY);
      }
      float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int e = 0; e < kS; ++e) mx4[e & 3] = fmaxf(mx4[e & 3], __uint_as_float(v[e]));
      const float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * p.qscale;
      float factor = 1.f;
      const bool need = mx > m_used + kRescaleThreshold;
      if (need) {
        factor = ex2_ftz(m_used - mx);  // 0 while m_used = -inf
        m_used = mx;
      }
      l *= factor;
      PHASE(2);
      const float2 negm2 = make_float2(-m_used, -m_used);
      float2 l2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
      for (int c = 0; c < kS / 32; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float2 x = make_float2(__uint_as_float(v[32 * c + e]), __uint_as_float(v[32 * c + e + 1]));
          const float2 tt = ffma2(x, qs2, negm2);
          const float2 pp =
              ((c * 16 + (e >> 1)) % kEmuPeriod) < kEmuPairs ? ex2_emu2(tt)
                                                             : make_float2(ex2_ftz(tt.x), ex2_ftz(tt.y));
          l2[(e >> 1) & 3] = fadd2(l2[(e >> 1) & 3], pp);
          pk[e >> 1] = pack2<T>(pp.x, pp.y);
        }
        tmem_st16(tS + c * 16, pk);
      }
      {
        const float2 a = fadd2(fadd2(l2[0], l2[1]), fadd2(l2[2], l2[3]));
        l += a.x + a.y;
      }
      PHASE(3);
      if (u > 0 && __any_sync(0xffffffffu, need)) {
        // rescale point: PV_t(u - 1) done, O_t holds every earlier sub-tile
        mbar_wait(bar(B_OD + 2 * t + ((u - 1) & 1)), ((u - 1) >> 1) & 1);
        tc_fence_after();
        {
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(tO + c * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * factor);
            tmem_st32(tO + c * 32, o);
          }
        }
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bar(B_PF + 2 * t + h));
      PHASE(4);
      if (r == 0 && u < 64) PDBG(128 + t * 64 + u);
    }
#ifdef PKV_K3_PHASES
    if (p.dbg && blockIdx.x == 0 && r == 0)
      for (int k = 0; k < 5; ++k) p.dbg[448 + 8 * t + k] = static_cast<unsigned long long>(ph[k]);
#endif
#undef PHASE
    if (nu[t] > 0) {
      mbar_wait(bar(B_OD + 2 * t + ((nu[t] - 1) & 1)), ((nu[t] - 1) >> 1) & 1);
      tc_fence_after();
      const bool valid = qi < cnt[t];
      const float inv = l > 0.f ? 1.f / l : 0.f;
      if (p.o_cols > 0 && cnt[t] == p.qt) {
        // full tile: stage O / l in Q_t's buffer (free: every QK of this tile
        // is done) and leave by TMA stores of o_cols-column boxes; the CTA only
        // waits for the bulk stores to READ shared memory, so it retires
        // without waiting for its 64-128 KB of output to reach memory (register
        // stores held each CTA ~6-9 us on the SM, tools/probes/cta_gap_probe.cu)
        // 128-byte staging rows (o_cols = 32 fp32 or 64 16-bit columns) in the
        // 128-byte-swizzled layout of the output map: the 16-byte units of a
        // row land at unit ^ (row & 7), so a warp's stores hit every bank
        uint8_t* my = smem + t * kQBytes + r * 128;
        const uint32_t stage_s = sQ + t * kQBytes;
        const uint32_t swz = static_cast<uint32_t>(r & 7);
        for (int c0 = 0; c0 < D; c0 += p.o_cols) {
          if (p.out_dtype == PKV_F32) {
            uint32_t o[32];
            tmem_ld32(tO + c0, o);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 8; ++k)
              *reinterpret_cast<float4*>(my + ((k ^ swz) << 4)) =
                  make_float4(__uint_as_float(o[4 * k]) * inv, __uint_as_float(o[4 * k + 1]) * inv,
                              __uint_as_float(o[4 * k + 2]) * inv, __uint_as_float(o[4 * k + 3]) * inv);
          } else {
#pragma unroll
            for (int half = 0; half < 2; ++half) {
              uint32_t o[32];
              tmem_ld32(tO + c0 + 32 * half, o);
              tmem_wait_ld();
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                uint32_t w[4];
#pragma unroll
                for (int hh = 0; hh < 4; ++hh) {
                  const float a = __uint_as_float(o[8 * k + 2 * hh]) * inv;
                  const float b = __uint_as_float(o[8 * k + 2 * hh + 1]) * inv;
                  w[hh] = p.out_dtype == PKV_BF16 ? pack2<__nv_bfloat16>(a, b) : pack2<__half>(a, b);
                }
                *reinterpret_cast<uint4*>(my + (((4 * half + k) ^ swz) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
              }
            }
          }
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          asm volatile("bar.sync %0, 128;\n" ::"r"(1 + t) : "memory");
          if (r == 0) {
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];\n" ::"l"(
                    reinterpret_cast<uint64_t>(&tm_o)),
                "r"(stage_s), "r"(c0), "r"(kvh * p.group), "r"(q_row0 + t * p.qt)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
          }
          asm volatile("bar.sync %0, 128;\n" ::"r"(1 + t) : "memory");  // staging free again
        }
      } else {
        const int64_t orow =
            (static_cast<int64_t>(q_row0) + t * p.qt + qi) * p.hq + kvh * p.group + (r - qi * p.group);
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          uint32_t o[32];
          tmem_ld32(tO + c * 32, o);
          tmem_wait_ld();
          if (valid) {
            if (p.out_dtype == PKV_F32) {
              float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.out) + orow * D + c * 32);
#pragma unroll
              for (int e = 0; e < 8; ++e)
                dst[e] = make_float4(__uint_as_float(o[4 * e]) * inv, __uint_as_float(o[4 * e + 1]) * inv,
                                     __uint_as_float(o[4 * e + 2]) * inv, __uint_as_float(o[4 * e + 3]) * inv);
            } else {
              uint4* dst = reinterpret_cast<uint4*>(static_cast<uint16_t*>(p.out) + orow * D + c * 32);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                uint32_t w[4];
#pragma unroll
                for (int hh = 0; hh < 4; ++hh) {
                  const float a = __uint_as_float(o[8 * e + 2 * hh]) * inv;
                  const float b = __uint_as_float(o[8 * e + 2 * hh + 1]) * inv;
                  w[hh] = p.out_dtype == PKV_BF16 ? pack2<__nv_bfloat16>(a, b) : pack2<__half>(a, b);
                }
                dst[e] = make_uint4(w[0], w[1], w[2], w[3]);
              }
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (p.dbg && threadIdx.x == 0) p.dbg[512 + 4 * blockIdx.x + 2] = gtime();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTmemCols)
                 : "memory");
  }
}

// ---- host side --------------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// 3-D map over [dim2][dim1][dim0] 16-bit elements, box (64, box1, box2), 128-B swizzle
int encode_map(CUtensorMap* map, const void* base, int dtype, uint64_t dim0, uint64_t dim1, uint64_t dim2,
               uint32_t box1, uint32_t box2, uint32_t box0 = 64, bool swizzle = true) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(PKV_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  const uint64_t es = dtype == PKV_F32 ? 4 : 2;
  const cuuint64_t dims[3] = {dim0, dim1, dim2};
  const cuuint64_t strides[2] = {dim0 * es, dim0 * dim1 * es};
  const cuuint32_t box[3] = {box0, box1, box2};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUtensorMapDataType ty = dtype == PKV_F32    ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : dtype == PKV_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                     : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const CUresult r = fn(map, ty, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PKV_CUDA_ERROR, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return PKV_OK;
}

// The encoded maps are cached (a cache's K / V maps are the same on every
// call; a caller that reuses its query buffer hits too): a small per-process
// table keyed by every encode argument, most recent first.
int make_map(CUtensorMap* map, const void* base, int dtype, uint64_t dim0, uint64_t dim1, uint64_t dim2,
             uint32_t box1, uint32_t box2, uint32_t box0 = 64, bool swizzle = true) {
  struct Entry {
    const void* base;
    uint64_t d0, d1, d2;
    uint32_t b0, b1, b2;
    int dtype;
    bool swz;
    CUtensorMap map;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  constexpr size_t kMaxEntries = 16;
  {
    std::lock_guard<std::mutex> g(mu);
    for (size_t i = 0; i < cache.size(); ++i) {
      const Entry& e = cache[i];
      if (e.base == base && e.d0 == dim0 && e.d1 == dim1 && e.d2 == dim2 && e.b1 == box1 && e.b2 == box2 &&
          e.dtype == dtype && e.b0 == box0 && e.swz == swizzle) {
        *map = e.map;
        if (i > 0) std::rotate(cache.begin(), cache.begin() + i, cache.begin() + i + 1);
        return PKV_OK;
      }
    }
  }
  const int st = encode_map(map, base, dtype, dim0, dim1, dim2, box1, box2, box0, swizzle);
  if (st) return st;
  std::lock_guard<std::mutex> g(mu);
  cache.insert(cache.begin(), Entry{base, dim0, dim1, dim2, box0, box1, box2, dtype, swizzle, *map});
  if (cache.size() > kMaxEntries) cache.pop_back();
  return PKV_OK;
}

template <typename T, int D>
size_t smem_bytes() {
  constexpr int NCH = D / 64;
  // at least 116 KB: one CTA per SM, so the 512-column TMEM allocation never waits
  return std::max<size_t>(1024 + NCH * kChunkB * 6 + 26 * 8 + 16, 116 * 1024);
}

template <typename T, int D>
int launch(const pkv_prefill_args* a, const PrefillParams& pp, cudaStream_t stream) {
  CUtensorMap mq, mk, mv, mk128, mv128;
  const int G = a->hq / a->hkv;
  int st = make_map(&mq, a->q, a->kv_dtype, D, a->hq, a->total_q, G, kM / G);
  if (st) return st;
  const uint32_t box_rows = static_cast<uint32_t>(pp.box_rows);
  st = make_map(&mk, a->k_cache, a->kv_dtype, D, a->hkv, a->cache_rows, 1, box_rows);
  if (st) return st;
  st = make_map(&mv, a->v_cache, a->kv_dtype, D, a->hkv, a->cache_rows, 1, box_rows);
  if (st) return st;
  // 128-row boxes for tiles whose pages form one contiguous run
  mk128 = mk;
  mv128 = mv;
  if (box_rows < static_cast<uint32_t>(kN)) {
    st = make_map(&mk128, a->k_cache, a->kv_dtype, D, a->hkv, a->cache_rows, 1, kN);
    if (st) return st;
    st = make_map(&mv128, a->v_cache, a->kv_dtype, D, a->hkv, a->cache_rows, 1, kN);
    if (st) return st;
  }
  // output map: full tiles leave by TMA stores through Q_t's buffer (no
  // swizzle; a box of o_cols columns x G heads x qt positions fills it)
  CUtensorMap mo = mq;
  PrefillParams pq = pp;
  static const bool bulk_out = [] {
    const char* e = std::getenv("PKV_K3_BULK_OUT");
    return !(e && e[0] == '0');
  }();
  const int es = a->out_dtype == PKV_F32 ? 4 : 2;
  const int o_cols = 128 / es;  // 128-byte swizzled rows: a box of kM x 128 B fills 16 KB of Q_t's buffer
  pq.o_cols = 0;
  if (bulk_out && (reinterpret_cast<uintptr_t>(a->out) & 15) == 0 && D % o_cols == 0) {
    st = make_map(&mo, a->out, a->out_dtype, D, a->hq, a->total_q, G, kM / G, static_cast<uint32_t>(o_cols), true);
    if (st) return st;
    pq.o_cols = o_cols;
  }
  const size_t smem = smem_bytes<T, D>();
  auto kern = prefill_tc_kernel<T, D>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr_set = true;
  }
  kern<<<static_cast<unsigned>(a->n_items), kThreads, smem, stream>>>(mq, mk, mv, mk128, mv128, mo, pq);
  PKV_CHECK_LAUNCH();
  return PKV_OK;
}

int query_tile(int hq, int hkv) { return kM / (hq / hkv); }

}  // namespace

void preload_prefill_kernels() {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(prefill_tc_kernel<__nv_bfloat16, 64>));
  cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(prefill_tc_kernel<__nv_bfloat16, 128>));
  cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(prefill_tc_kernel<__half, 64>));
  cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(prefill_tc_kernel<__half, 128>));
}
}  // namespace pkv

using namespace pkv;

extern "C" int pkv_prefill_supported(int32_t hq, int32_t hkv, int32_t head_dim, int32_t page_size,
                                     int32_t kv_dtype) {
  if (hq <= 0 || hkv <= 0 || hq % hkv) return 0;
  const int G = hq / hkv;
  if (G > kM || kM % G) return 0;
  if (head_dim != 64 && head_dim != 128) return 0;
  if (page_size < 8 || (page_size & (page_size - 1))) return 0;
  if (kv_dtype != PKV_BF16 && kv_dtype != PKV_F16) return 0;
  return 1;
}

extern "C" int64_t pkv_prefill_plan_ints(const int32_t* q_len, int64_t n_seqs, int32_t hq, int32_t hkv) {
  if (hq <= 0 || hkv <= 0 || hq % hkv || n_seqs < 0) return 0;
  const int qt = query_tile(hq, hkv);
  int64_t pairs = 0;
  for (int64_t s = 0; s < n_seqs; ++s) pairs += (std::max(q_len[s], 0) + 2 * qt - 1) / (2 * qt);
  return pairs * hkv * kItemInts;
}

// Work items: one kv head x two consecutive query tiles (A, B) of 128/G
// positions each; per tile the key range is the causal prefix of its last
// valid query (n_tiles of 128 keys).  Longest first.
namespace pkv {
int prefill_plan_build(const int64_t* q_start, const int32_t* q_len, const int32_t* seq_len,
                       const int32_t* seq_row, int64_t n_seqs, int32_t hq, int32_t hkv, int32_t causal,
                       int32_t* plan_out, int64_t cap, int64_t* n_items_out);
}
namespace {
// Memo of the last plan per host thread: every layer of a model runs the
// same prefill metadata, so the planner (item build + longest-first sort)
// runs once per forward instead of once per layer.
struct PrefillMemo {
  std::vector<int64_t> key;
  std::vector<int32_t> plan;
  int64_t n_items = -1;
  int64_t generation = 0;  // bumped whenever the memo is rebuilt
};
thread_local PrefillMemo t_prefill_memo;
}  // namespace

extern "C" int pkv_prefill_plan(const int64_t* q_start, const int32_t* q_len, const int32_t* seq_len,
                                const int32_t* seq_row, int64_t n_seqs, int32_t hq, int32_t hkv,
                                int32_t causal, int32_t* plan_out, int64_t cap, int64_t* n_items_out) {
  if (n_seqs < 0 || (n_seqs > 0 && (!q_start || !q_len || !seq_len || !seq_row)))
    return fail(PKV_VALUE_ERROR, "bad prefill plan inputs");
  std::vector<int64_t> key;
  key.reserve(static_cast<size_t>(4 * n_seqs + 4));
  key.push_back(n_seqs);
  key.push_back(hq);
  key.push_back(hkv);
  key.push_back(causal);
  for (int64_t s = 0; s < n_seqs; ++s) {
    key.push_back(q_start[s]);
    key.push_back(q_len[s]);
    key.push_back(seq_len[s]);
    key.push_back(seq_row[s]);
  }
  PrefillMemo& m = t_prefill_memo;
  if (m.n_items >= 0 && key == m.key) {
    const int64_t need = m.n_items * kItemInts;
    if (need > cap) return fail(PKV_VALUE_ERROR, "plan buffer too small (%lld < %lld)", static_cast<long long>(cap),
                                static_cast<long long>(need));
    if (need) std::memcpy(plan_out, m.plan.data(), need * sizeof(int32_t));
    *n_items_out = m.n_items;
    return PKV_OK;
  }
  const int st = pkv::prefill_plan_build(q_start, q_len, seq_len, seq_row, n_seqs, hq, hkv, causal, plan_out, cap,
                                         n_items_out);
  if (st) return st;
  m.key.swap(key);
  m.n_items = *n_items_out;
  m.plan.assign(plan_out, plan_out + m.n_items * kItemInts);
  ++m.generation;
  return PKV_OK;
}

// The K3 route of paged_attention / gathered_attention in one host pass:
// decide whether the query metadata is suffix-shaped (attention.py:81-84,
// 98-110: per view sequence one run of consecutive positions ending at its
// last key), report the longest run, and build (memoised) the plan.  q_seq is
// non-decreasing (MaskMeta checks it).  Not suffix-shaped: *n_items_out = -1.
// *generation_out identifies the memoised plan: equal generations on one host
// thread mean an identical plan (a caller may keep its device copy).
extern "C" int pkv_prefill_plan_meta(const int64_t* q_seq, const int64_t* q_pos, int64_t n_q,
                                     const int64_t* seq_len, const int32_t* seq_row, int64_t n_seqs, int32_t hq,
                                     int32_t hkv, int32_t causal, int32_t build, int32_t* plan_out, int64_t cap,
                                     int64_t* n_items_out, int64_t* max_run_out, int64_t* generation_out) {
  if (n_q < 0 || n_seqs < 0 || (n_q > 0 && (!q_seq || !q_pos)) || (n_seqs > 0 && (!seq_len || !seq_row)))
    return fail(PKV_VALUE_ERROR, "bad prefill metadata");
  *n_items_out = -1;
  *max_run_out = 0;
  // runs by binary search on the non-decreasing q_seq, then one vectorisable
  // pass per run checking q_seq[i] == s and q_pos[i] == len - q_len + (i - q_start)
  // (an unsorted or out-of-range q_seq fails the check: not suffix-shaped)
  std::vector<int64_t> q_start(static_cast<size_t>(n_seqs) + 1, 0);
  std::vector<int32_t> q_len(static_cast<size_t>(n_seqs), 0), sl(static_cast<size_t>(n_seqs));
  for (int64_t s = 0; s <= n_seqs; ++s) q_start[s] = std::lower_bound(q_seq, q_seq + n_q, s) - q_seq;
  if (q_start[n_seqs] != n_q) return PKV_OK;
  int64_t max_run = 0;
  uint64_t diff = static_cast<uint64_t>(q_start[0]);  // queries before sequence 0: negative q_seq
  for (int64_t s = 0; s < n_seqs; ++s) {
    if (seq_len[s] < 0 || seq_len[s] > 0x7fffffff) return fail(PKV_OUT_OF_RANGE, "sequence length beyond int32");
    sl[s] = static_cast<int32_t>(seq_len[s]);
    const int64_t a = q_start[s], len_q = q_start[s + 1] - a;
    q_len[s] = static_cast<int32_t>(len_q);
    max_run = std::max<int64_t>(max_run, len_q);
    const int64_t base = seq_len[s] - len_q - a;
    for (int64_t i = a; i < a + len_q; ++i)
      diff |= static_cast<uint64_t>(q_pos[i] ^ (base + i)) | static_cast<uint64_t>(q_seq[i] ^ s);
  }
  if (diff) return PKV_OK;
  *max_run_out = max_run;
  *n_items_out = 0;
  if (build <= 0 || max_run < build) return PKV_OK;
  const int st = pkv_prefill_plan(q_start.data(), q_len.data(), sl.data(), seq_row, n_seqs, hq, hkv, causal,
                                  plan_out, cap, n_items_out);
  if (generation_out) *generation_out = t_prefill_memo.generation;
  return st;
}

namespace pkv {
int prefill_plan_build(const int64_t* q_start, const int32_t* q_len, const int32_t* seq_len,
                       const int32_t* seq_row, int64_t n_seqs, int32_t hq, int32_t hkv, int32_t causal,
                       int32_t* plan_out, int64_t cap, int64_t* n_items_out) {
  if (hq <= 0 || hkv <= 0 || hq % hkv) return fail(PKV_SHAPE_MISMATCH, "hq must be a multiple of hkv");
  const int G = hq / hkv;
  if (G > kM || kM % G) return fail(PKV_CONFIG_ERROR, "group size %d does not divide %d", G, kM);
  const int qt = query_tile(hq, hkv);
  struct Rec {
    int32_t v[kItemInts];
  };
  std::vector<Rec> items;
  for (int64_t s = 0; s < n_seqs; ++s) {
    const int32_t ql = q_len[s], kl = seq_len[s];
    if (ql < 0 || ql > kl) return fail(PKV_OUT_OF_RANGE, "sequence %lld: %d queries over %d keys",
                                       static_cast<long long>(s), ql, kl);
    if (q_start[s] + ql > (int64_t(1) << 31)) return fail(PKV_OUT_OF_RANGE, "query rows beyond 2^31");
    for (int t0 = 0; t0 * qt < ql; t0 += 2) {
      int cnt[2], tiles[2];
      for (int u = 0; u < 2; ++u) {
        const int first = (t0 + u) * qt;
        cnt[u] = std::max(0, std::min(qt, ql - first));
        const int pos0 = kl - ql + first;
        const int nk = causal ? std::min(pos0 + cnt[u], kl) : kl;  // keys of the tile's last row
        tiles[u] = cnt[u] > 0 ? (nk + kN - 1) / kN : 0;
      }
      for (int h = 0; h < hkv; ++h) {
        Rec r;
        r.v[0] = static_cast<int32_t>(q_start[s] + int64_t(t0) * qt);
        r.v[1] = cnt[0];
        r.v[2] = cnt[1];
        r.v[3] = kl - ql + t0 * qt;
        r.v[4] = kl;
        r.v[5] = seq_row[s];
        r.v[6] = h;
        r.v[7] = tiles[0];
        r.v[8] = tiles[1];
        r.v[9] = 0;
        items.push_back(r);
      }
    }
  }
  // longest items first: the hardware block scheduler then approximates LPT
  std::stable_sort(items.begin(), items.end(), [](const Rec& x, const Rec& y) {
    return std::max(x.v[7], x.v[8]) > std::max(y.v[7], y.v[8]);
  });
  const int64_t need = static_cast<int64_t>(items.size()) * kItemInts;
  if (need > cap) return fail(PKV_VALUE_ERROR, "plan buffer too small (%lld < %lld)", static_cast<long long>(cap),
                              static_cast<long long>(need));
  if (!items.empty()) std::memcpy(plan_out, items.data(), need * sizeof(int32_t));
  *n_items_out = static_cast<int64_t>(items.size());
  return PKV_OK;
}

}  // namespace pkv

extern "C" int pkv_paged_prefill(const pkv_prefill_args* a, void* stream_) {
  if (!a) return fail(PKV_VALUE_ERROR, "null args");
  if (a->n_items <= 0) return PKV_OK;
  if (!pkv_prefill_supported(a->hq, a->hkv, a->head_dim, a->page_size, a->kv_dtype))
    return fail(PKV_CONFIG_ERROR, "tcgen05 prefill does not support hq=%d hkv=%d head_dim=%d page_size=%d dtype=%d",
                a->hq, a->hkv, a->head_dim, a->page_size, a->kv_dtype);
  if (!a->plan) return fail(PKV_VALUE_ERROR, "prefill needs the pkv_prefill_plan() items");
  if (a->cache_rows <= 0 || a->cache_rows >= (int64_t(1) << 31) - 256)
    return fail(PKV_OUT_OF_RANGE, "cache rows must be in (0, 2^31 - 256)");
  if (a->out_dtype != PKV_F32 && a->out_dtype != a->kv_dtype)
    return fail(PKV_CONFIG_ERROR, "prefill output must be fp32 or the cache dtype");
  if (a->n_items > 0x7fffffff) return fail(PKV_CONFIG_ERROR, "too many prefill items");
  PrefillParams pp;
  pp.hq = a->hq;
  pp.hkv = a->hkv;
  pp.group = a->hq / a->hkv;
  pp.qt = kM / pp.group;
  pp.log2ps = __builtin_ctz(a->page_size);
  // paged: one box per page (or per 128-key slice of a larger page);
  // gathered (block_table == NULL): one 128-row box per tile
  pp.box_rows = a->block_table ? std::min(a->page_size, kN) : kN;
  pp.bt_stride = a->bt_stride;
  pp.bt = a->block_table;
  pp.oob_row = static_cast<int32_t>(a->cache_rows);
  pp.qscale = a->scale * kLog2eP;
  pp.causal = a->causal;
  pp.out = a->out;
  pp.out_dtype = a->out_dtype;
  pp.items = a->plan;
  pp.dbg = static_cast<unsigned long long*>(a->debug);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  pkv::DeviceGuard guard(stream);
  if (a->prof_start) cudaEventRecord(static_cast<cudaEvent_t>(a->prof_start), stream);
  int st;
  if (a->kv_dtype == PKV_BF16)
    st = a->head_dim == 128 ? launch<__nv_bfloat16, 128>(a, pp, stream) : launch<__nv_bfloat16, 64>(a, pp, stream);
  else
    st = a->head_dim == 128 ? launch<__half, 128>(a, pp, stream) : launch<__half, 64>(a, pp, stream);
  if (st) return st;
  if (a->prof_stop) cudaEventRecord(static_cast<cudaEvent_t>(a->prof_stop), stream);
  return PKV_OK;
}
