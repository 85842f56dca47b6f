// nnb_gemm_tc.cuh -- tcgen05 (5th-gen tensor core) GEMM for Dense layers, 1x1
// convolutions ("rows" mode) and stride-1 KxK convolutions ("conv" mode:
// implicit GEMM over 8 x 16-pixel tiles), FP32-accurate through 3xTF32.
//
//   C[m, j] = sum_k A[m, k] * B[k, j]            A: activations  [M, K] row-major
//                                                B: weights, stored transposed
//                                                   [Npad, Kpad] (K-major)
// Every operand is split a = hi + lo (hi exactly representable in TF32, lo =
// a - hi exact in FP32); the product is a_hi*b_hi + (a_hi*b_lo + a_lo*b_hi),
// the first into a main TMEM chain and the two small ones into a correction
// chain, both restarted every CHUNK k-blocks (the tensor core truncates once
// per MMA) and summed in FP32 by the epilogue.  Weights are split at
// compile() time (B_hi, B_lo in the pool); activations by the split warps.
// Error bound and measurements: DESIGN.md section 4.
//
// Warp roles (one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer: A tile [128 x BK] (rows: 2-D box; conv: 4-D box
//               of an 8x16-pixel tile per tap, zero-filled borders = 'same'
//               padding; DWF: the depthwise input halo) and B_hi/B_lo tiles,
//               swizzled, into an NS-stage mbarrier ring
//   warp 1      TMEM allocator + single-thread MMA issuer
//               (tcgen05.mma kind::tf32, M=128, or M=256 over a CTA pair)
//   warps 2..   A-split warps: 2 (A_lo into shared memory) or 4 (A hi/lo into
//               TMEM for the "ts" MMA form, or the fused depthwise producer)
//   last 8      epilogue: warp w reads TMEM lanes 32*(w%4).. (lane-quarter
//               rule) and half of the tile's columns; bias, activation,
//               post-affine, residual, then TMA-store boxes (or staged /
//               direct stores for pooled, upsampled and KPACK tiles)
// Options per instantiation (Cfg fields): TMEM_A, PAIR (cta_group::2),
// KPACK (horizontal taps packed into N), CONCAT (second A source), POOL,
// UPF, RES, EPI_TMA, CSPLIT / CORR_WHOLE, CHUNK, ABUF, NACC, DWF, BN = 256.
#pragma once
#include "nnb_common.cuh"
#include "nnb_softmax.cuh"

// NNB_TC_DBG (diagnostics only, results are garbage): bit 0 skips the MMAs,
// bit 1 the TMA operand loads, bit 2 the A split, bit 3 the epilogue's TMEM
// reads and math.
#ifndef NNB_TC_DBG
#define NNB_TC_DBG 0
#endif
// NNB_DRAIN2: mid-tile drains of whole-K correction chains read two column
// groups per TMEM wait (dense 1024->512 at 65536 rows 0.2137 -> 0.2105 ms)
#ifndef NNB_DRAIN2
#define NNB_DRAIN2 1
#endif
// NNB_SPLIT_UNROLL: unroll of the BF16-correction split loop (8: the whole
// stage per thread in flight; 0.2110 -> 0.2096 ms)
#ifndef NNB_SPLIT_UNROLL
#define NNB_SPLIT_UNROLL 8
#endif
// The tensor core reads FP32 operands of kind::tf32 with the 13 low mantissa
// bits ignored (verified on B200 by scripts/tc_hi.py: bit-identical results
// with and without writing hi = a & 0xffffe000 back), so only lo = a - hi is
// materialised; the raw tile serves as the hi operand.
// Split rule for A in TMEM: hi = A rounded to the nearest TF32 (exactly
// representable, so the tensor core uses it as is) and lo = A - hi, exact and
// of either sign -- the tensor core's truncation of lo then errs in both
// directions instead of always toward zero.  (A read from shared memory is
// the raw FP32 tile, which the hardware truncates: there hi = trunc(A).)
#ifndef NNB_SPLIT_RN
#define NNB_SPLIT_RN 1
#endif
#ifndef NNB_HI_INPLACE
#define NNB_HI_INPLACE 0
#endif

namespace nnb {

struct __align__(64) TmaDesc { unsigned long long opaque[16]; };

__device__ __forceinline__ u32 split_hi(float a) {
  const u32 u = __float_as_uint(a);
  return ((NNB_SPLIT_RN ? u + 0x1000u : u) & 0xFFFFE000u);
}

// CORR_BF16 split of A in shared memory.  NNB_CB16_WB=1 writes the
// round-to-nearest TF32 hi back over the tile; 0 (default) leaves the raw
// tile, which the tensor core truncates, so hi = trunc(a) and lo = a - hi >= 0
// -- its bf16 rounding is unbiased either way (the tf32 truncation of lo that
// made the write-back necessary in the tf32 split does not occur).  Measured
// (cfg1 Dense 1024->512 @65536): 0.231 ms with the write-back, 0.220 without.
#ifndef NNB_CB16_WB
#define NNB_CB16_WB 0
#endif
__device__ __forceinline__ u32 cb16_hi(float a) {
  const u32 u = __float_as_uint(a);
  return ((NNB_CB16_WB ? u + 0x1000u : u) & 0xFFFFE000u);
}

__device__ __forceinline__ u32 smem_u32(const void* p) {
  return (u32)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(u64* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
#ifdef NNB_SPIN_WAIT
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "NNB_SPIN:\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra NNB_SPIN;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
  return;
#endif
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "NNB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra NNB_DONE;\n"
      "bra NNB_WAIT;\n"
      "NNB_DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const TmaDesc* map, u64* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<u64>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// L2 prefetch of a 2-D box (no shared-memory destination, no barrier)
__device__ __forceinline__ void tma_prefetch_2d(const TmaDesc* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<u64>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const TmaDesc* map, u64* bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<u64>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// TMA tensor stores (bulk-group completion, per issuing thread)
__device__ __forceinline__ void tma_store_2d(const TmaDesc* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<u64>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_store_4d(const TmaDesc* map, const void* src, int c0, int c1,
                                             int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<u64>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// K-major operand descriptor.  ROWB = bytes per row = BK*4: 128 -> 128-byte
// swizzle (layout type 2), 8-row atoms 1024 B apart; 64 -> 64-byte swizzle
// (layout type 4), atoms 512 B apart.
template <int ROWB>
__device__ __forceinline__ u64 kmajor_desc(u32 saddr) {
  constexpr u64 layout = ROWB == 128 ? 2 : 4;
  return (u64)((saddr >> 4) & 0x3FFF) | ((u64)1 << 16) | ((u64)(8 * ROWB >> 4) << 32) |
         ((u64)1 << 46) | (layout << 61);
}
__device__ __forceinline__ u64 sw128_desc(u32 saddr) { return kmajor_desc<128>(saddr); }

__device__ __forceinline__ void mma_tf32(u32 tmem_d, u64 adesc, u64 bdesc, u32 idesc, u32 acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

// A operand from tensor memory (lane = row, one tf32 per 32-bit column)
__device__ __forceinline__ void mma_tf32_ts(u32 tmem_d, u32 tmem_a, u64 bdesc, u32 idesc, u32 acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void tmem_st32(u32 taddr, const u32 (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
      "%29, %30, %31, %32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
      "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
      "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

template <int N>
__device__ __forceinline__ void tmem_st(u32 taddr, const u32 (&v)[N]) {
  if constexpr (N == 32) {
    tmem_st32(taddr, v);
  } else {
    static_assert(N == 16, "tmem_st width");
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
  }
}

// CTA-pair (cta_group::2) forms: the leader CTA issues M=256 MMAs whose rows
// 128..255 (and B columns BN/2..BN-1) live in the peer CTA's TMEM / shared
// memory at the same addresses; commits arrive on the barrier in both CTAs.
__device__ __forceinline__ void mma_tf32_ts_pair(u32 tmem_d, u32 tmem_a, u64 bdesc, u32 idesc,
                                                 u32 acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_pair(u32 tmem_d, u64 adesc, u64 bdesc, u32 idesc, u32 acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
// kind::f16 (BF16 operands, FP32 accumulator) forms: the correction products
// of the CORR_BF16 split (one K = 16 instruction per tf32 k-step)
__device__ __forceinline__ void mma_bf16(u32 tmem_d, u64 adesc, u64 bdesc, u32 idesc, u32 acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(u32 tmem_d, u64 adesc, u64 bdesc, u32 idesc, u32 acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
// two floats -> bf16x2 (round to nearest even), `lo` in the low half
__device__ __forceinline__ u32 bf16x2_rn(float lo, float hi) {
  u32 d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

__device__ __forceinline__ void mma_commit_pair(u64* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((unsigned short)3)
      : "memory");
}
__device__ __forceinline__ u32 cluster_rank() {
  u32 r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// named barrier over the two warps (64 threads) sharing a TMEM lane quarter
__device__ __forceinline__ void named_sync64(int id) {
  asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}
// named barrier over the four epilogue warps of one column group
__device__ __forceinline__ void named_sync256(int id) {
  asm volatile("bar.sync %0, 256;" ::"r"(id) : "memory");
}
__device__ __forceinline__ void named_sync128(int id) {
  asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the barrier at the same offset in the leader CTA (rank 0)
__device__ __forceinline__ void mbar_arrive_leader(u64* bar) {
  u32 r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(bar)));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
}

__device__ __forceinline__ void mma_commit(u64* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(u32 taddr, float (&v)[16]) {
  u32 r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Batched TMEM reads: several tcgen05.ld in flight, one wait.  tmem_pin
// re-defines the destination registers after the wait so no use of them
// can be scheduled above it.
__device__ __forceinline__ void tmem_ld16_async(u32 taddr, u32 (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8_async(u32 taddr, u32 (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
template <int N>
__device__ __forceinline__ void tmem_ld_async(u32 taddr, u32 (&r)[N]) {
  if constexpr (N == 16) tmem_ld16_async(taddr, r);
  else { static_assert(N == 8, "tmem_ld_async width"); tmem_ld8_async(taddr, r); }
}
template <int N>
__device__ __forceinline__ void tmem_pin_n(u32 (&r)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("" : "+r"(r[i]));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_pin(u32 (&r)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) asm volatile("" : "+r"(r[i]));
}

template <int N>
__device__ __forceinline__ void tmem_ld(u32 taddr, float (&v)[N]) {
  if constexpr (N == 16) {
    tmem_ld16(taddr, v);
  } else {
    static_assert(N == 8, "tmem_ld width");
    u32 r[8];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
  }
}

// Epilogue transpose through shared memory.  After the TMEM read every lane
// owns one output row; storing (or residual-loading) NC columns per lane
// touches 32 rows = 32 cache lines per warp instruction.  stage_rows writes
// the warp's 32 x NC block into a per-warp staging area (16-byte chunks
// XOR-swizzled so both phases are bank-conflict free); staged_chunk then
// hands lane l the chunk (l % CPR) of row p*(32/CPR) + l/CPR in pass p, so a
// warp instruction covers 32/CPR whole row segments.
template <int NC>
__device__ __forceinline__ int stage_slot(int row, int c) {
  constexpr int CPR = NC / 4, RPW = 8 / CPR;
  return row * CPR + (c ^ ((row / RPW) & (CPR - 1)));
}
template <int NC>
__device__ __forceinline__ void stage_rows(float4* st, const float* v, int lane) {
  static_assert(NC == 4 || NC == 8 || NC == 16, "staged columns");
#pragma unroll
  for (int j = 0; j < NC / 4; ++j)
    st[stage_slot<NC>(lane, j)] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  __syncwarp();
}

// C: K, N, NPAD (multiple of BN), BN (32..256, multiple of 16), NS (stages),
//    ROWS (GEMM rows per image), IN/OUT offsets, B_OFF (bias), epilogue fields.
template <class C>
struct GemmTc {
  static constexpr int BM = 128, BK = C::BK;                // 32 (SW128) or 16 (SW64)
  static constexpr int ROWB = BK * 4;
  // RS: vertical taps sharing one A box (KPACK conv tiles): the box holds the
  // TH + RS - 1 input rows of the tile (16 pixels each) and the MMAs of kernel
  // row ky read it from pixel row ky on -- a 16-row offset is a whole number
  // of swizzle atoms -- so each input pixel is loaded and split once per
  // channel block instead of once per kernel row.  A k-block then carries RS
  // B sub-tiles (W^T columns ky * CI + channel block) and RS x BK/8 k-steps.
  static constexpr int RS = C::RS;
  static constexpr int A_ROWS = BM + (RS - 1) * 16;
  static constexpr int A_BYTES = A_ROWS * BK * 4;
  static constexpr int KSTEPS = RS * (BK / 8);             // k-steps per k-block
  // PAIR: CTA pairs (cluster of 2, tcgen05 cta_group::2).  The pair computes a
  // 256 x BN tile: each CTA loads its own 128 rows of A and HALF of B (BN/2
  // rows of W^T), the leader issues M=256 MMAs that read both CTAs' operands,
  // each CTA's TMEM receives its own 128 accumulator rows.  Per SM this halves
  // the B traffic (TMA writes and tensor-core reads of shared memory), which
  // is what bounds the single-CTA kernel at BN=128.
  static constexpr bool PAIR = C::PAIR != 0;
  static constexpr int B_ROWS = PAIR ? C::BN / 2 : C::BN;   // B rows held per CTA
  static constexpr int B_BYTES = B_ROWS * BK * 4;
  static constexpr int B_SMEM = RS * B_BYTES;               // hi (or lo) B sub-tiles of a stage
  // TMEM_A: the split A operand lives in tensor memory (MMA "ts" form), so the
  // tensor core reads only B from shared memory -- for narrow N the A re-reads
  // (three products per k-step) otherwise saturate shared-memory bandwidth.
  static constexpr bool TA = C::TMEM_A != 0;
  // DWF: a depthwise conv fused as the A producer of this 1x1 conv.  A stage
  // then carries the depthwise INPUT halo of the 8 x 16 pixel tile (one 4-D
  // TMA box, zero-filled borders = 'same' padding) instead of an A tile; the
  // A-split warps compute the depthwise output (bias, taps in order, mul then
  // add, activation / post-BN) and hand it to the MMA like any A tile.
  static constexpr bool DWF = C::DWF != 0;
  static constexpr int HALO_W = DWF ? 15 * C::DW_S + C::DW_KW : 0;   // (16-1)*S + KW
  static constexpr int HALO_H = DWF ? 7 * C::DW_S + C::DW_KH : 0;    // (8-1)*S + KH
  static constexpr int HALO_TX = HALO_W * HALO_H * BK * 4;           // bytes the box delivers
  static constexpr int HALO_BYTES = (HALO_TX + 1023) / 1024 * 1024;
  static constexpr int A_SMEM = (TA ? (DWF ? 0 : A_BYTES) : 2 * A_BYTES);  // A (+ A_lo) in smem
  static constexpr int STAGE = A_SMEM + 2 * B_SMEM + HALO_BYTES;
  static constexpr int KB = (C::K + BK * RS - 1) / (BK * RS);
  static constexpr int NTN = C::NPAD / C::BN;
  // One accumulator buffer = main (a_hi*b_hi) + correction (a_hi*b_lo + a_lo*b_hi)
  // columns.  Tensor-core accumulation truncates once per MMA instruction, so the
  // error grows with the number of accumulate steps into a large running sum;
  // keeping the two small correction products out of the main sum cuts the
  // truncations on it by 3x, and the two are added in FP32 (round-to-nearest)
  // in the epilogue.
  // NACC independent (main, correction) chains per buffer: consecutive k-steps
  // rotate over them so dependent tcgen05.mma instructions overlap (for narrow
  // N a single accumulator chain is bound by MMA latency, not throughput).
  static constexpr int NACC = C::NACC;
  // CSPLIT = 0 accumulates the correction products into the main chain (half
  // the TMEM columns, so BN = 128 keeps two accumulator buffers next to a
  // TMEM-resident A); the chunk length CHUNK then bounds the truncation error.
  static constexpr bool CS = C::CSPLIT != 0;
  // epilogue activation mode: exact mode stays float64-rounded-once (the
  // interpreter's semantics, interpreter.py:102-112) here as everywhere
  static constexpr int EMODE = C::MODE;
  static constexpr int CW = (CS ? 2 : 1) * C::BN;         // columns per chain
  static constexpr int ACC_COLS = NACC * CW;              // fp32 columns per buffer
  // ABUF accumulator buffers: 2 lets the epilogue drain one while the MMA fills
  // the other; 1 frees TMEM for the A operand at BN = 128 (the MMA then waits
  // only for the short per-chunk drain).
  static constexpr int ABUF = C::ABUF;
  static constexpr int A_TCOL = ABUF * ACC_COLS;                 // first A column (TA)
  static constexpr int TMEM_NEED = TA ? ABUF * ACC_COLS + C::NS * 2 * BK : ABUF * ACC_COLS;
#ifdef NNB_TC_NDBG
  static constexpr int TMEM_COLS = 512;
#else
  static constexpr int TMEM_COLS = TMEM_NEED <= 32 ? 32 : TMEM_NEED <= 64 ? 64
                                 : TMEM_NEED <= 128 ? 128 : TMEM_NEED <= 256 ? 256 : 512;
#endif
  static_assert(TMEM_NEED <= 512, "TMEM budget");
#ifdef NNB_TC_NDBG
  // diagnostic: issue MMAs of width NNB_TC_NDBG (results meaningless)
  static constexpr u32 IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((u32)(NNB_TC_NDBG >> 3) << 17) |
                               ((u32)((PAIR ? 2 * BM : BM) >> 4) << 24);
#else
  static constexpr u32 IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((u32)(C::BN >> 3) << 17) |
                               ((u32)((PAIR ? 2 * BM : BM) >> 4) << 24);
#endif
  // CORR_BF16: the two correction products of a tf32 k-step (8 k) run as ONE
  // kind::f16 MMA of K = 16 over BF16 operands -- A_corr row = [bf16(a_hi) x 8,
  // bf16(a_lo) x 8] per k-step, B_corr = [bf16(b_lo) x 8, bf16(b_hi) x 8] (built
  // at compile() time) -- so a k-step issues 2 instruction-times of MMA instead
  // of 3 (BF16 runs at twice the TF32 rate).  A_corr replaces the A_lo tile and
  // B_corr the B_lo tile, byte for byte.  Error per product <= 2^-17 |a b|
  // (bf16 rounding of the split halves), DESIGN.md section 4.
  static constexpr bool CB16 = C::CORR_BF16 != 0;
  static constexpr u32 IDESC_B16 = (1u << 4) | (1u << 7) | (1u << 10) | ((u32)(C::BN >> 3) << 17) |
                                   ((u32)((PAIR ? 2 * BM : BM) >> 4) << 24);
  // (the N = 256 row tiles may also MERGE the correction MMA into the main
  // accumulator -- CSPLIT = 0: two 256-column buffers, so the epilogue drains
  // one chunk while the MMAs fill the next)
  static_assert(!CB16 || (!TA && !C::ALDG && !C::DWF && BK == 32 && (C::CSPLIT || C::BN == 256)),
                "bf16 correction split");
  // EARLY main products (N = 256 BF16-correction row tiles; the raw A tile is
  // never rewritten by the split there)
  static constexpr bool EARLY = CB16 && C::EARLY && !NNB_CB16_WB;
  static constexpr int SPLIT_UNROLL = NNB_SPLIT_UNROLL;
  // EPI16 (KPACK conv tiles with CO = 32): SIXTEEN epilogue warps -- four
  // per TMEM lane quarter, each draining and combining a quarter of the
  // output channels.  Those tiles are bound by the epilogue's dependent chain
  // per tile (drain, shuffles, pooled store, staged store: cfg4's 120x160x16
  // -> 32 conv runs 88 us with the mainloop ablated, 78 us with the epilogue
  // ablated); half the channels per warp was meant to shorten the chain.
  // Measured: bit-identical but SLOWER (109.5 -> 118 us; the 60x80x128 -> 32
  // conv 145.8 -> 153 us) -- 8-channel groups halve the bytes per store and
  // the extra warps add TMEM / shuffle contention.  Opt-in (tuning epi16).
  static constexpr int EPI_WARPS = C::EPI16 ? 16 : 8, EPI_THREADS = 32 * EPI_WARPS;
  static constexpr int EPI_GROUPS = EPI_WARPS / 4;               // column groups (warps per lane quarter)
  static_assert(!C::EPI16 || (C::KPACK && C::CO == 32 && C::CONV && !C::EPI_TMA && !C::EDW && !C::HEAD &&
                              !C::SETREG), "sixteen epilogue warps: KPACK conv tiles with 32 outputs");
  // ALDG: the A operand is gathered by the four loader/converter warps with
  // cp.async (16-byte LDGSTS, zero-fill for padding) straight into the swizzled
  // layout, instead of per-row TMA requests (which cap A at ~16-28 B/cycle/SM).
  static constexpr bool AL = C::ALDG != 0;
  static_assert(!(AL && TA), "A via LDGSTS lives in shared memory");
  static_assert(!PAIR || (!AL && C::BN % 16 == 0 && (C::BN / 2) % 8 == 0), "CTA-pair tile shape");
  // A splitters: 4 for A in TMEM / cp.async / depthwise producers and for
  // the bf16 correction split of narrow tiles (C::CONV_W4), else 2
  // SETREG (N = 256 BF16-correction row tiles): SIX split warps and 512
  // threads -- the launch gives every thread 128 registers, then the two
  // producer / split warpgroups hand registers back (setmaxnreg.dec 88) and
  // the two epilogue warpgroups, which hold 128 running sums per thread, take
  // them (setmaxnreg.inc 168): 256 x 88 + 256 x 168 = the whole register file.
  // Without the reallocation 168 registers x 384 threads left room for two
  // split warps only, and the split sat on every stage's critical path.
  static constexpr bool SETREG = C::SETREG != 0;
  static constexpr int CONV_WARPS = SETREG ? 6 : (TA || AL || DWF || C::CONV_W4) ? 4 : 2;
  static_assert(!SETREG || (CB16 && !TA && !AL && !DWF), "register reallocation: BF16-correction tiles");
  static constexpr int EPI_W0 = 2 + CONV_WARPS;                   // first epilogue warp
  static constexpr int THREADS = 32 * EPI_W0 + EPI_THREADS;
  static constexpr int EPI_COLS = C::BN >= 32 ? C::BN / 2 : 16;  // columns per epilogue warp
  static constexpr int CHUNK_KB = C::CHUNK;          // k-blocks per TMEM chunk
  static constexpr int NCHUNK = (KB + CHUNK_KB - 1) / CHUNK_KB;
  // WIDE: N = 256 per MMA (a tcgen05 kind::tf32 instruction costs ~100
  // cycles at N <= 128 and ~1.4x that at N = 256, scripts/mma_n256.py); the
  // epilogue keeps 128 running sums per thread (384 threads: 168 registers)
  static constexpr bool WIDE = C::BN > 128 && !C::KP9 && !C::KPACK;
  static_assert(C::BN % 16 == 0 && C::BN >= 16 && (C::BN <= 128 || C::BN == 256 ||
                                                   ((C::KP9 || C::KPACK) && C::BN <= 256)),
                "UMMA N / TMEM budget");
  static_assert(!C::CORR_WHOLE || (CS && C::NACC == 1), "whole-K correction chain");
  static_assert(!WIDE || (!TA && C::NACC == 1 && !C::CONV && !C::RES && C::UPF == 1 &&
                          C::ABUF * (C::CSPLIT ? 2 : 1) * C::BN <= 512),
                "N = 256 tiles: A in shared memory, 512 TMEM columns");
  // spatial (implicit-GEMM convolution) tiling: 8 x 16 output pixels per tile
  static constexpr int TH = 8, TW = 16;
  // KPACK: the KW horizontal taps are packed into N (N = KW*CO, K = KH*CI): a
  // tile computes per-input-column partial sums D'[pixel][kx][co] and the
  // epilogue combines out(x) = sum_kx D'(x + kx)[kx] with warp shuffles, so a
  // tile of 16 input columns yields OW = 16 - (KW - 1) output columns.
  static constexpr bool KP = C::KPACK != 0;
  // KP9: ALL KH x KW taps packed into N (N = KH*KW*CO <= 256, K = CI): one
  // A box per channel block instead of one per kernel row, i.e. every input
  // pixel is loaded and split once per tile instead of KH times.  A tile of
  // 8 x 16 input pixels yields THO = 8 - (KH - 1) rows x OW output columns;
  // the epilogue adds the KW horizontal partial sums with shuffles and the KH
  // vertical ones through shared memory (rows cross warp quarters).
  static constexpr bool K9 = C::KP9 != 0;
  static constexpr int OW = (KP || K9) ? TW - (C::KW - 1) : TW;
  static constexpr int THO = K9 ? TH - (C::KH - 1) : TH;
  static constexpr int TX = C::CONV ? (C::WO + OW - 1) / OW : 1;
  static constexpr int TPI = C::CONV ? ((C::HO + THO - 1) / THO) * TX : 1;
  static_assert(!K9 || (C::CONV && !KP && !C::POOL && !C::RES && C::UPF == 1 && !C::DPOOL &&
                        C::CO == 16 && C::KH * C::KW * C::CO == C::N && !C::CSPLIT &&
                        C::KH <= 3 && C::KW <= 3), "KP9 geometry");
  static constexpr int CB = C::CONV ? C::CI / BK : 1;       // channel blocks per tap
  static constexpr int CB0 = C::CONV ? C::C0 / BK : 1;      // ... from source 0
  static_assert(!C::CONV || C::CI % BK == 0, "conv tiles need CI % BK == 0");
  static_assert(BK == 32 || BK == 16, "K block");
  static_assert(!C::DPOOL || (C::CONV && !C::POOL && C::UPF == 1 && (KP || C::N % 16 == 0)),
                "dual pooled store: conv tiles");
  static_assert(!KP || (C::CONV && !C::POOL && !C::RES && C::CO % 16 == 0 &&
                        C::KW * C::CO == C::N), "KPACK geometry");
  static_assert(STAGE % 1024 == 0, "stage alignment");
  static_assert(RS == 1 || (KP && C::CONV && !TA && !AL && !DWF && !CB16 && RS == C::KH), "row-shared taps");
  static_assert(!DWF || (C::CONV && !KP && !AL && C::KW == 1 && C::CI % BK == 0),
                "depthwise fusion: 1x1 conv tiles");
  // EPI_TMA: the epilogue writes the tile into 64B-swizzled shared-memory
  // boxes of 32 rows x 16 columns (the layout a lane = row thread writes
  // without bank conflicts) and stores them with TMA; a residual operand is
  // prefetched into the same boxes by TMA before the accumulator is ready.
  static constexpr bool ET = C::EPI_TMA != 0;
  static constexpr int EGRP = EPI_COLS / 16;                       // 16-column groups per warp
  static constexpr int NBUF = ET ? (C::RES ? EGRP : (EGRP < 2 ? EGRP : 2)) : 1;
  static_assert(!ET || !(C::POOL || C::UPF > 1 || KP), "TMA epilogue: plain row tiles only");
  static_assert(!(C::RES && C::UPF > 1), "residual fusion excludes upsampling (planner)");
  // EDW: the DepthwiseConv2D consuming this 1x1 conv computed in the epilogue
  // (planner.fuse_pw_dw).  A 128-row tile holds 128 / (E_H * E_W) whole images
  // (cfg3's 8x8 and 4x4 maps), so the finished tile -- bias, activation,
  // post-BN applied -- is parked in shared memory as [row][BN + 4] floats
  // (lane = row float4 stores and channel-quad = lane float4 loads are both
  // conflict-free) and the eight epilogue warps run the depthwise taps over
  // it: a thread owns one output row of one image and one channel quad,
  // reads each input row of the window once into registers and slides the
  // taps over it (reference order: bias, then (ky, kx), out-of-image taps
  // skipped -- pkg/src/nnjit/interpreter.py:65-73), then stores the depthwise
  // output (512 contiguous bytes per warp and pixel).  The pointwise output
  // itself is never written.
  // Maps larger than a tile but 16 pixels wide or less (cfg3's 16x16 stage)
  // run as BANDS: a tile is EB_TR = 128 / E_W consecutive image rows starting
  // at input row tt * EB_OT * E_S - E_PT (a 2-D TMA box at that row of the
  // [pixels x K] matrix; rows above the image or of the neighbouring image
  // are loaded but never used as taps), and yields the EB_OT output rows whose
  // windows it holds -- the 1x1 conv of the overlap rows is recomputed (x1.5
  // for 3x3 taps on 16x16 maps), which costs less than a launch.
  static constexpr bool EDW = C::EDW != 0;
  static constexpr int EP = EDW ? C::E_H * C::E_W : 1;            // pixels per image
  static constexpr bool EBAND = EDW && BM % EP != 0;
  static constexpr int EB_TR = EDW ? BM / C::E_W : 1;             // image rows per band tile
  static constexpr int EB_OT = EDW ? (EB_TR - C::E_KH) / C::E_S + 1 : 1;   // output rows per band tile
  static constexpr int EB_TPI = EDW ? (C::E_HO + EB_OT - 1) / EB_OT : 1;   // band tiles per image
  static_assert(!EBAND || (BM % C::E_W == 0 && EB_TR >= C::E_KH && !PAIR && !C::E_GAP),
                "depthwise epilogue: band tiles");
  static constexpr int ETS = C::BN + 4;                           // parked tile row stride (floats)
  static constexpr int EDW_BYTES = EDW ? (BM * ETS * 4 + 1023) / 1024 * 1024 : 0;
  static_assert(!EDW || (!C::CONV && !C::RES && C::UPF == 1 && !C::HEAD && !KP && !K9 && !WIDE && !ET &&
                         !C::DPOOL && C::BN % 32 == 0 && C::N % 4 == 0 &&
                         C::ROWS == C::E_H * C::E_W && C::E_W <= 16),
                "depthwise epilogue: row tiles holding whole images or bands of one");
  static constexpr int EPI_STAGE = EDW ? EDW_BYTES : EPI_WARPS * NBUF * 2048;   // 32 x 16 fp32 per buffer
  static_assert(!K9 || 2 * (C::KH - 1) * 8 * 16 * (C::CO / 2) * 4 <= EPI_STAGE,
                "KP9 vertical exchange fits the staging area");
  // HEAD: a following Dense with HN <= 16 outputs (a classifier head, e.g.
  // cfg1's 128 -> 10 + softmax) computed in this epilogue from the finished
  // tile row: each of the two warps holding a row's column halves forms the
  // head's partial dot over its columns (weights as immediates, Cfg::hw /
  // hbias), the upper half hands its partials over through the (otherwise
  // unused) staging boxes, and the lower half adds them, applies the head's
  // activation / softmax and stores the HN outputs.  This GEMM's own output
  // is never written.  One N tile (BN >= N) so a CTA owns whole rows.
  static constexpr bool HEAD = C::HEAD != 0;
  static_assert(!HEAD || (NTN == 1 && !C::CONV && !C::RES && C::UPF == 1 && !KP && !WIDE &&
                          C::HN <= 16 && C::BN >= 32), "fused head");
  static constexpr int SMEM = C::NS * STAGE + EPI_STAGE + 1024 /*align*/ + 512 /*barriers*/;

  // the head's partial dot over this warp's columns [CB, CB + EPI_COLS)
  template <int CB>
  __device__ static __forceinline__ void head_dot(const float (&run)[EPI_COLS], float (&hp)[C::HN]) {
#pragma unroll
    for (int i = 0; i < EPI_COLS; ++i) {
      if (CB + i < C::N) {
#pragma unroll
        for (int j = 0; j < C::HN; ++j) hp[j] = fmaf(run[i], C::hw((CB + i) * C::HN + j), hp[j]);
      }
    }
  }

  // DPOOL: second store of the 2x2/2 max-pooled tile (planner.fuse_pool_dual):
  // the four pixels of a window sit in lanes w, w^1 (adjacent columns) and
  // w^16, w^17 (the next image row) of one warp; the lane of the window's top-
  // left pixel stores the NC maxima of its columns at the pooled position (and
  // its DP_UPF x DP_UPF replicas when the pooled map is upsampled).
  template <int NC>
  __device__ static __forceinline__ void dual_pool_store(float* __restrict__ arena, const float* v,
                                                         bool lead, int img, int oy, int ox,
                                                         int cofs, int n) {
    float m[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const float a = fmaxf(v[i], __shfl_xor_sync(0xffffffffu, v[i], 1));
      m[i] = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, 16));
    }
    const int py = oy >> 1, px = ox >> 1;
    if (!(lead && img < n && py < C::DP_PHO && px < C::DP_PWO)) return;
    constexpr int U = C::DP_UPF, WU = C::DP_PWO * U;
    float* d = at<float>(arena, C::DP_OFF + (long long)img * C::DP_IMG);
#pragma unroll
    for (int rep = 0; rep < U * U; ++rep) {
      float* dst = d + ((long long)(py * U + rep / U) * WU + px * U + rep % U) * C::CO + cofs;
#pragma unroll
      for (int i = 0; i < NC; i += 4)
        *reinterpret_cast<float4*>(dst + i) = make_float4(m[i], m[i + 1], m[i + 2], m[i + 3]);
    }
  }

  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena, int n,
                             const TmaDesc* tmA, const TmaDesc* tmB, const TmaDesc* tmBlo,
                             const TmaDesc* tmA1, const TmaDesc* tmO, const TmaDesc* tmR) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // The dynamic shared window starts 1024-byte aligned (no static shared
    // memory in this kernel); using the array itself keeps the compiler in the
    // shared address space (LDS/STS rather than generic LD/ST).
    // (measured: the shared-space form is 1-4% faster for the A-in-smem
    // kernels, the generic form 4-20% faster for the A-in-TMEM ones)
    unsigned char* smem = TA ? reinterpret_cast<unsigned char*>(
                                   (reinterpret_cast<u64>(smem_raw) + 1023) & ~(u64)1023)
                             : smem_raw;
    if (!TA && (smem_u32(smem_raw) & 1023u)) __trap();
    if (blockDim.x != THREADS) __trap();          // role layout needs every warp
    float4* epi_stage = reinterpret_cast<float4*>(smem + C::NS * STAGE);
    u64* bars = reinterpret_cast<u64*>(smem + C::NS * STAGE + EPI_STAGE);
    u64* full = bars;                 // [NS]  TMA landed
    u64* lo_ready = bars + C::NS;     // [NS]  A split done (64 converter arrivals)
    u64* empty = bars + 2 * C::NS;    // [NS]  MMA finished reading the stage
    u64* tfull = bars + 3 * C::NS;    // [ABUF] accumulator ready
    u64* tempty = tfull + ABUF;       // [ABUF] accumulator drained (epilogue arrivals)
    u64* rbar = tempty + ABUF;        // [EPI_WARPS] residual boxes landed (EPI_TMA)
    u64* pfull = rbar + EPI_WARPS;    // [NS]  EARLY pairs: the peer's stage landed (leader)
    u32* tmem_slot = reinterpret_cast<u32*>(pfull + C::NS);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long rows = (long long)n * C::ROWS;
    const int mtiles = C::CONV ? n * TPI : EBAND ? n * EB_TPI : (int)((rows + BM - 1) / BM);
    // pairs walk 256-row tile pairs: CTA `rank` of the pair takes 128 of them
    const int rank = PAIR ? (int)cluster_rank() : 0;
    const int tiles = (PAIR ? (mtiles + 1) / 2 : mtiles) * NTN;
    const int t0 = PAIR ? (int)blockIdx.x / 2 : (int)blockIdx.x;
    const int tstep = PAIR ? (int)gridDim.x / 2 : (int)gridDim.x;
    auto mb_of = [&](int t) { return PAIR ? (t / NTN) * 2 + rank : t / NTN; };
    // consumer-side arrivals that the (leader's) MMA warp waits for: pairs
    // count one per warp of both CTAs, single CTAs one per thread
    auto arrive_mma = [&](u64* bar) {
      if (PAIR) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive_leader(bar);
      } else {
        mbar_arrive(bar);
      }
    };

    if (threadIdx.x == 0) {
      for (int s = 0; s < C::NS; ++s) {
        mbar_init(&full[s], 1);
        // pairs: one arrival per split warp of both CTAs, on the leader's barrier
        mbar_init(&lo_ready[s], PAIR ? 2 * CONV_WARPS : 32 * CONV_WARPS);
        mbar_init(&empty[s], 1);
      }
      for (int a = 0; a < ABUF; ++a) {
        mbar_init(&tfull[a], 1);
        mbar_init(&tempty[a], PAIR ? 2 * EPI_WARPS : EPI_THREADS);
      }
      for (int w = 0; w < EPI_WARPS; ++w) mbar_init(&rbar[w], 1);
      for (int st = 0; st < C::NS; ++st) mbar_init(&pfull[st], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
      if (PAIR) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
      } else {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
      }
    }
    tc_fence_before();
    if (PAIR) cluster_sync();          // the peer's barriers exist before any remote arrive
    else __syncthreads();
    tc_fence_after();
    const u32 tmem = *tmem_slot;
    // SETREG: warpgroups 0-1 (TMA, MMA, six split warps) release registers, 2-3
    // (epilogue) take them -- issued inside each role's branch, so that ptxas
    // allocates every role within its own budget
#define NNB_SETREG_DEC() do { if constexpr (SETREG) asm volatile("setmaxnreg.dec.sync.aligned.u32 88;"); } while (0)
#define NNB_SETREG_INC() do { if constexpr (SETREG) asm volatile("setmaxnreg.inc.sync.aligned.u32 168;"); } while (0)

    if (warp == 0) {
      NNB_SETREG_DEC();
      // ---------------- TMA producer ----------------
      if (lane == 0) {
        int s = 0;
        u32 ph = 0;
        for (int t = t0; t < tiles; t += tstep) {
          const int mb = mb_of(t), nb = t % NTN;
          for (int kb = 0; kb < KB; ++kb) {
            mbar_wait(&empty[s], ph ^ 1);
            unsigned char* st = smem + s * STAGE;
            mbar_expect_tx(&full[s], (NNB_TC_DBG & 2) ? 0
                                     : (AL ? 0 : DWF ? HALO_TX : A_BYTES) + 2 * B_SMEM);
            if (NNB_TC_DBG & 2) {
              // diagnostic: no operand traffic
            } else if (AL) {
              // A is gathered by the loader warps
            } else if (DWF) {
              // depthwise input halo of the tile, channel block kb
              const int img = mb / TPI, tt = mb % TPI;
              tma_load_4d(st + A_SMEM + 2 * B_SMEM, tmA, &full[s], kb * BK,
                          (tt % TX) * TW * C::DW_S - C::DW_PL,
                          (tt / TX) * TH * C::DW_S - C::DW_PT, img);
            } else if (C::CONV) {
              // tap (ky, kx) and channel block cb of an 8x16 output-pixel tile;
              // out-of-image coordinates are zero-filled = 'same' padding
              // with CONCAT, channel blocks >= C0/32 come from the second source
              const int img = mb / TPI, tt = mb % TPI;
              const int tap = kb / CB, cb = kb % CB;     // KPACK: tap = ky only
              const bool second = C::CONCAT && cb >= CB0;
              const int kx = KP ? 0 : tap % C::KW, ky = KP ? tap : tap / C::KW;
              tma_load_4d(st, second ? tmA1 : tmA, &full[s], (second ? cb - CB0 : cb) * BK,
                          (tt % TX) * OW + kx - C::PL, (tt / TX) * THO + ky - C::PT, img);
            } else {
              // (EDW bands: the tile starts at an input row of its image, possibly
              // above it -- negative coordinates are zero-filled)
              tma_load_2d(st, tmA, &full[s], kb * BK,
                          EBAND ? (mb / EB_TPI) * EP + ((mb % EB_TPI) * EB_OT * C::E_S - C::E_PT) * C::E_W
                                : mb * BM);
              if constexpr (C::APF > 0) {
                // the A box APF k-blocks ahead into L2: its TMA load then
                // waits on L2, not HBM, latency (the ring is latency-bound)
                int pkb = kb + C::APF, pt = t;
                if (pkb >= KB) { pkb -= KB; pt += tstep; }
                if (pt < tiles) tma_prefetch_2d(tmA, pkb * BK, mb_of(pt) * BM);
              }
            }
            if (!(NNB_TC_DBG & 2)) {
              const int brow = nb * C::BN + rank * B_ROWS;         // this CTA's B rows
#pragma unroll
              for (int r = 0; r < RS; ++r) {                       // RS: kernel row r's W^T block
                tma_load_2d(st + A_SMEM + r * B_BYTES, tmB, &full[s], (r * KB + kb) * BK, brow);
                tma_load_2d(st + A_SMEM + B_SMEM + r * B_BYTES, tmBlo, &full[s], (r * KB + kb) * BK, brow);
              }
            }
            if (++s == C::NS) { s = 0; ph ^= 1; }
          }
        }
      }
    } else if (warp == 1) {
      NNB_SETREG_DEC();
      // ---------------- MMA issuer (the leader CTA of a pair) ----------------
      if (PAIR && rank != 0) {
        // the peer's MMA warp only owns the TMEM allocation
      } else {
      // K is consumed in chunks of CHUNK_KB k-blocks; every chunk starts a fresh
      // (main, correction) accumulator pair in the next TMEM buffer and is
      // reduced in FP32 by the epilogue warps (split-K inside the CTA).
      int s = 0, acc = 0;
      u32 ph = 0, aph = 0;
      for (int t = t0; t < tiles; t += tstep) {
        for (int kb = 0; kb < KB; ++kb) {
          const int kc = kb % CHUNK_KB;
          if (kc == 0) {
            mbar_wait(&tempty[acc], aph ^ 1);
            tc_fence_after();
          }
          const u32 dbuf = tmem + acc * ACC_COLS;
          if constexpr (EARLY) {
            // N = 256 BF16-correction tiles: the main product a_hi*b_hi reads
            // the raw A tile (the tensor core truncates it to TF32), so it is
            // issued once both CTAs' stage has landed (local TMA barrier + the
            // peer's pfull arrival), while the split warps build A_corr; the
            // correction MMA follows on lo_ready.  Same accumulation order per
            // chain as issuing both after lo_ready.
            mbar_wait(&full[s], ph);
            if (PAIR) mbar_wait(&pfull[s], ph);
            tc_fence_after();
            if (lane == 0) {
              const u32 base = smem_u32(smem + s * STAGE);
              const u32 b_hi = base + A_SMEM;
#pragma unroll
              for (int k = 0; k < ((NNB_TC_DBG & 1) ? 0 : BK / 8); ++k) {
                const u32 o = k * 32;
                const int ks = kc * (BK / 8) + k;
                const u32 d = dbuf + (ks % NACC) * CW;
                if (PAIR) mma_tf32_pair(d, kmajor_desc<ROWB>(base + o), kmajor_desc<ROWB>(b_hi + o), IDESC, ks >= NACC);
                else mma_tf32(d, kmajor_desc<ROWB>(base + o), kmajor_desc<ROWB>(b_hi + o), IDESC, ks >= NACC);
              }
            }
            __syncwarp();
            mbar_wait(&lo_ready[s], ph);
            tc_fence_after();
            if (lane == 0) {
              const u32 base = smem_u32(smem + s * STAGE);
              const u32 a_lo = base + A_BYTES, b_lo = base + A_SMEM + B_SMEM;
#pragma unroll
              for (int k = 0; k < ((NNB_TC_DBG & 1) ? 0 : BK / 8); ++k) {
                const u32 o = k * 32;
                const int ks = kc * (BK / 8) + k;
                const u32 dc = dbuf + (ks % NACC) * CW + (CS ? C::BN : 0);
                const u32 acc_c = !CS ? 1u   // merged: after this stage's main product into the same chain
                                  : C::CORR_WHOLE ? (u32)(kb * (BK / 8) + k > 0) : (u32)(ks >= NACC);
                if (PAIR) mma_bf16_pair(dc, kmajor_desc<ROWB>(a_lo + o), kmajor_desc<ROWB>(b_lo + o), IDESC_B16, acc_c);
                else mma_bf16(dc, kmajor_desc<ROWB>(a_lo + o), kmajor_desc<ROWB>(b_lo + o), IDESC_B16, acc_c);
              }
              if (PAIR) {
                mma_commit_pair(&empty[s]);
                if (kc == CHUNK_KB - 1 || kb == KB - 1) mma_commit_pair(&tfull[acc]);
              } else {
                mma_commit(&empty[s]);
                if (kc == CHUNK_KB - 1 || kb == KB - 1) mma_commit(&tfull[acc]);
              }
            }
            __syncwarp();
            if (++s == C::NS) { s = 0; ph ^= 1; }
            if (kc == CHUNK_KB - 1 || kb == KB - 1) {
              if (++acc == ABUF) { acc = 0; aph ^= 1; }
            }
            continue;
          }
          if (AL) mbar_wait(&full[s], ph);           // B (TMA); A comes via lo_ready
          mbar_wait(&lo_ready[s], ph);
          tc_fence_after();
          if (lane == 0) {
            const u32 base = smem_u32(smem + s * STAGE);
#pragma unroll
            for (int r = 0; r < RS; ++r) {
            const u32 a_hi = base + r * 16 * ROWB, a_lo = a_hi + A_BYTES;
            const u32 b_hi = base + A_SMEM + r * B_BYTES, b_lo = b_hi + B_SMEM;
            const u32 ta = tmem + A_TCOL + s * 2 * BK;                // TMEM A slot
#pragma unroll
            for (int k = 0; k < ((NNB_TC_DBG & 1) ? 0 : BK / 8); ++k) {
              const u32 o = k * 32;   // 8 tf32 = 32 bytes along the swizzled row
              const int ks = kc * KSTEPS + r * (BK / 8) + k;     // k-step within the chunk
#ifdef NNB_TC_NDBG
              const u32 d = tmem, dc = tmem;                     // diagnostic width test
#else
              const u32 d = dbuf + (ks % NACC) * CW;             // this step's chain
              const u32 dc = CS ? d + C::BN : d;                 // its correction columns
#endif
              const u32 accum = ks >= NACC;
              // CORR_WHOLE: the correction chain runs over the whole K (its
              // values are ~2^-11 of the main sum, so its truncations are
              // negligible); only the main chain restarts per chunk
              const u32 acc_c = CS ? (C::CORR_WHOLE ? (u32)(kb * KSTEPS + r * (BK / 8) + k > 0) : accum) : 1u;
              if (PAIR && TA) {
                mma_tf32_ts_pair(d, ta + 8 * k, kmajor_desc<ROWB>(b_hi + o), IDESC, accum);
                mma_tf32_ts_pair(dc, ta + 8 * k, kmajor_desc<ROWB>(b_lo + o), IDESC, acc_c);
                mma_tf32_ts_pair(dc, ta + BK + 8 * k, kmajor_desc<ROWB>(b_hi + o), IDESC, 1);
              } else if (PAIR && CB16) {
                mma_tf32_pair(d, kmajor_desc<ROWB>(a_hi + o), kmajor_desc<ROWB>(b_hi + o), IDESC, accum);
                mma_bf16_pair(dc, kmajor_desc<ROWB>(a_lo + o), kmajor_desc<ROWB>(b_lo + o), IDESC_B16, acc_c);
              } else if (PAIR) {
                mma_tf32_pair(d, kmajor_desc<ROWB>(a_hi + o), kmajor_desc<ROWB>(b_hi + o), IDESC, accum);
                mma_tf32_pair(dc, kmajor_desc<ROWB>(a_hi + o), kmajor_desc<ROWB>(b_lo + o), IDESC, acc_c);
                mma_tf32_pair(dc, kmajor_desc<ROWB>(a_lo + o), kmajor_desc<ROWB>(b_hi + o), IDESC, 1);
              } else if (CB16) {
                mma_tf32(d, kmajor_desc<ROWB>(a_hi + o), kmajor_desc<ROWB>(b_hi + o), IDESC, accum);
                mma_bf16(dc, kmajor_desc<ROWB>(a_lo + o), kmajor_desc<ROWB>(b_lo + o), IDESC_B16, acc_c);
              } else if (TA) {
                mma_tf32_ts(d, ta + 8 * k, kmajor_desc<ROWB>(b_hi + o), IDESC, accum);
                mma_tf32_ts(dc, ta + 8 * k, kmajor_desc<ROWB>(b_lo + o), IDESC, acc_c);
                mma_tf32_ts(dc, ta + BK + 8 * k, kmajor_desc<ROWB>(b_hi + o), IDESC, 1);
              } else {
                mma_tf32(d, kmajor_desc<ROWB>(a_hi + o), kmajor_desc<ROWB>(b_hi + o), IDESC, accum);
                mma_tf32(dc, kmajor_desc<ROWB>(a_hi + o), kmajor_desc<ROWB>(b_lo + o), IDESC, acc_c);
                mma_tf32(dc, kmajor_desc<ROWB>(a_lo + o), kmajor_desc<ROWB>(b_hi + o), IDESC, 1);
              }
            }
            }
            if (PAIR) {
              mma_commit_pair(&empty[s]);
              if (kc == CHUNK_KB - 1 || kb == KB - 1) mma_commit_pair(&tfull[acc]);
            } else {
              mma_commit(&empty[s]);
              if (kc == CHUNK_KB - 1 || kb == KB - 1) mma_commit(&tfull[acc]);
            }
          }
          __syncwarp();
          if (++s == C::NS) { s = 0; ph ^= 1; }
          if (kc == CHUNK_KB - 1 || kb == KB - 1) {
            if (++acc == ABUF) { acc = 0; aph ^= 1; }
          }
        }
      }
      }
    } else if (warp < EPI_W0) {
      NNB_SETREG_DEC();
     // (role bodies selected at compile time: only the instantiated form is
     // compiled -- NVRTC time)
     if constexpr (DWF) {
      // ---------------- depthwise producer: halo -> A tile (TMEM or smem) ----------------
      const int q = warp & 3, r = q * 32 + lane;      // tile pixel = A row = TMEM lane
      const int ty = r / TW, tx = r % TW;
      const float* dwk = at<float>(pool, C::DW_W_OFF);
      const float* dwb = at<float>(pool, C::DW_B_OFF);
      const float* dps = at<float>(pool, C::DW_PS_OFF);
      const float* dpo = at<float>(pool, C::DW_PO_OFF);
      int s = 0;
      u32 ph = 0;
      for (int t = t0; t < tiles; t += tstep) {
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[s], ph);
          const unsigned char* halo = smem + s * STAGE + A_SMEM + 2 * B_SMEM;
          unsigned char* arow = smem + s * STAGE + r * ROWB;
          const int c0 = kb * BK;
          const u32 ta = tmem + ((u32)(q * 32) << 16) + A_TCOL + s * 2 * BK;
#pragma unroll
          for (int hh = 0; hh < BK / 16; ++hh) {
            float a[16];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const int j = hh * 4 + jj;
              float4 acc = __ldg(reinterpret_cast<const float4*>(dwb + c0 + 4 * j));
#pragma unroll
              for (int ky = 0; ky < C::DW_KH; ++ky)
#pragma unroll
                for (int kx = 0; kx < C::DW_KW; ++kx) {
                  const int hp = (ty * C::DW_S + ky) * HALO_W + tx * C::DW_S + kx;
                  const int pj = ROWB == 128 ? (j ^ (hp & 7)) : (j ^ ((hp >> 1) & 3));
                  const float4 x = *reinterpret_cast<const float4*>(halo + hp * ROWB + (pj << 4));
                  const float4 w = __ldg(reinterpret_cast<const float4*>(
                      dwk + (ky * C::DW_KW + kx) * C::CI + c0 + 4 * j));
                  acc.x = add(acc.x, mul(x.x, w.x)); acc.y = add(acc.y, mul(x.y, w.y));
                  acc.z = add(acc.z, mul(x.z, w.z)); acc.w = add(acc.w, mul(x.w, w.w));
                }
              const int c = c0 + 4 * j;
              a[4 * jj + 0] = finish<C::DW_ACT, EMODE, C::DW_POST>(acc.x, dps, dpo, c);
              a[4 * jj + 1] = finish<C::DW_ACT, EMODE, C::DW_POST>(acc.y, dps, dpo, c + 1);
              a[4 * jj + 2] = finish<C::DW_ACT, EMODE, C::DW_POST>(acc.z, dps, dpo, c + 2);
              a[4 * jj + 3] = finish<C::DW_ACT, EMODE, C::DW_POST>(acc.w, dps, dpo, c + 3);
            }
            if constexpr (TA) {
              u32 hi[16], lo[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                hi[i] = split_hi(a[i]);
                lo[i] = __float_as_uint(a[i] - __uint_as_float(hi[i]));
              }
              tmem_st<16>(ta + hh * 16, hi);
              tmem_st<16>(ta + BK + hh * 16, lo);
            } else {
              // raw value as A (the tensor core truncates it) and lo = a - trunc(a)
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                const int j = hh * 4 + jj;
                const int pj = ROWB == 128 ? (j ^ (r & 7)) : (j ^ ((r >> 1) & 3));
                const float4 full4 = make_float4(a[4 * jj], a[4 * jj + 1], a[4 * jj + 2], a[4 * jj + 3]);
                float4 v = full4, l;
                if (C::RN_SS) {            // RN hi written as the A value, lo = a - hi
                  v = make_float4(__uint_as_float(split_hi(full4.x)), __uint_as_float(split_hi(full4.y)),
                                  __uint_as_float(split_hi(full4.z)), __uint_as_float(split_hi(full4.w)));
                  l.x = full4.x - v.x; l.y = full4.y - v.y; l.z = full4.z - v.z; l.w = full4.w - v.w;
                } else {
                  l.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
                  l.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
                  l.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
                  l.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
                }
                *reinterpret_cast<float4*>(arow + (pj << 4)) = v;
                *reinterpret_cast<float4*>(arow + A_BYTES + (pj << 4)) = l;
              }
            }
          }
          if constexpr (TA) {
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
          } else {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          }
          arrive_mma(&lo_ready[s]);
          if (++s == C::NS) { s = 0; ph ^= 1; }
        }
      }
     } else if constexpr (TA) {
      // ---------------- converter: A row -> (hi, lo) columns in TMEM ----------------
      const int q = warp & 3, r = q * 32 + lane;      // this thread's tile row = TMEM lane
      int s = 0;
      u32 ph = 0;
      for (int t = t0; t < tiles; t += tstep) {
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[s], ph);
          if (NNB_TC_DBG & 4) {
            arrive_mma(&lo_ready[s]);
            if (++s == C::NS) { s = 0; ph ^= 1; }
            continue;
          }
          const unsigned char* row = smem + s * STAGE + r * ROWB;
          const u32 ta = tmem + ((u32)(q * 32) << 16) + A_TCOL + s * 2 * BK;
#pragma unroll
          for (int hh = 0; hh < BK / 16; ++hh) {      // 16 columns at a time (registers)
            u32 hi[16], lo[16];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {          // 16-byte chunk j of the swizzled row
              const int j = hh * 4 + jj;
              // SW128: chunk ^= row & 7; SW64: chunk ^= (row >> 1) & 3
              const int pj = ROWB == 128 ? (j ^ (r & 7)) : (j ^ ((r >> 1) & 3));
              const float4 v = *reinterpret_cast<const float4*>(row + (pj << 4));
              const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const u32 h = split_hi(e[i]);
                hi[4 * jj + i] = h;
                lo[4 * jj + i] = __float_as_uint(e[i] - __uint_as_float(h));
              }
            }
            tmem_st<16>(ta + hh * 16, hi);
            tmem_st<16>(ta + BK + hh * 16, lo);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          arrive_mma(&lo_ready[s]);
          if (++s == C::NS) { s = 0; ph ^= 1; }
        }
      }
     } else if constexpr (AL) {
      // ---------------- loader: cp.async gather of A, then split in place ----------------
      constexpr int CH = BK / 4;                       // 16-byte chunks per row
      constexpr int PER = BM * CH / 128;               // chunks per loader thread
      constexpr int D = C::NS - 1;                     // k-blocks in flight
      const int lt = threadIdx.x - 64;                 // 0..127
      const int my_tiles = blockIdx.x < tiles ? (tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
      const int total = my_tiles * KB;
      const float* a0 = at<float>(arena, C::IN_OFF);
      const float* a1 = at<float>(arena, C::IN1_OFF);
      auto issue = [&](int it) {
        const int t = blockIdx.x + (it / KB) * gridDim.x, kb = it % KB, mb = t / NTN;
        const int stg = it % C::NS;
        mbar_wait(&empty[stg], ((it / C::NS) & 1) ^ 1);
        const u32 sbase = smem_u32(smem + stg * STAGE);
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          const int e = j * 128 + lt, row = e / CH, ch = e % CH;
          const float* src = a0;
          bool ok;
          if (C::CONV) {
            const int img = mb / TPI, tt = mb % TPI;
            const int tap = kb / CB, cb = kb % CB;
            const int kx = KP ? 0 : tap % C::KW, ky = KP ? tap : tap / C::KW;
            const int iy = (tt / TX) * THO + row / TW + ky - C::PT;
            const int ix = (tt % TX) * OW + row % TW + kx - C::PL;
            ok = iy >= 0 && iy < C::H && ix >= 0 && ix < C::W;
            const bool second = C::CONCAT && cb >= CB0;
            const int cis = second ? C::CI - C::C0 : C::C0;
            const long long off = (long long)img * ((second ? C::IN1_IMG : C::IN_IMG) / 4) +
                                  ((long long)iy * C::W + ix) * cis +
                                  (second ? cb - CB0 : cb) * BK + ch * 4;
            if (ok) src = (second ? a1 : a0) + off;
          } else {
            const long long m = (long long)mb * BM + row;
            const int k = kb * BK + ch * 4;
            ok = m < rows && k < C::K;
            if (ok) src = a0 + m * C::K + k;
          }
          const u32 pj = ROWB == 128 ? (ch ^ (row & 7)) : (ch ^ ((row >> 1) & 3));
          const u32 dst = sbase + row * ROWB + (pj << 4);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                       "r"(ok ? 16 : 0) : "memory");
        }
      };
      // prologue: D k-blocks in flight; afterwards convert k-block `it`, hand it
      // to the MMA, then refill the stage of `it-1` (free once MMA(it-1) is done,
      // while MMA(it) already runs).  Exactly one commit group per k-block.
      for (int it = 0; it < D; ++it) {
        if (it < total) issue(it);
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
      for (int it = 0; it < total; ++it) {
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
        // this thread's own chunks of k-block `it` have landed: split in place
        const int stg = it % C::NS;
        unsigned char* sb = smem + stg * STAGE;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          const int e = j * 128 + lt, row = e / CH, ch = e % CH;
          const int pj = ROWB == 128 ? (ch ^ (row & 7)) : (ch ^ ((row >> 1) & 3));
          float4* pa = reinterpret_cast<float4*>(sb + row * ROWB + (pj << 4));
          float4* pl = reinterpret_cast<float4*>(sb + A_BYTES + row * ROWB + (pj << 4));
          float4 v = *pa, h, l;
          h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u); l.x = v.x - h.x;
          h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u); l.y = v.y - h.y;
          h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u); l.z = v.z - h.z;
          h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u); l.w = v.w - h.w;
          if (NNB_HI_INPLACE) *pa = h;
          *pl = l;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&lo_ready[stg]);
        if (it + D < total) issue(it + D);
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
     } else {
      // ---------------- converter: A -> (hi, lo) ----------------
      const int ct = threadIdx.x - 64;   // 0 .. 32 * CONV_WARPS - 1
      int s = 0;
      u32 ph = 0;
      for (int t = t0; t < tiles; t += tstep) {
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[s], ph);
          // EARLY: the peer's A / B halves of this stage have landed -- the
          // leader may issue the main products before the split is done
          if (EARLY && PAIR && rank != 0 && ct == 0) mbar_arrive_leader(&pfull[s]);
          float4* a = reinterpret_cast<float4*>(smem + s * STAGE);
          float4* lo = reinterpret_cast<float4*>(smem + s * STAGE + A_BYTES);
          if constexpr (CB16) {
            // k-step g of row `row` = logical 16-byte chunks 2g, 2g+1 of the
            // 128B-swizzled row (physical chunk = logical ^ (row & 7)); the
            // A_corr row keeps the same swizzle: bf16(hi) x 8 in chunk 2g,
            // bf16(lo) x 8 in chunk 2g+1
            uint4* corr = reinterpret_cast<uint4*>(lo);
#pragma unroll (SPLIT_UNROLL)
            for (int i = ct; i < ((NNB_TC_DBG & 4) ? 0 : A_BYTES / 32); i += 32 * CONV_WARPS) {
              const int row = i >> 2, g = i & 3, x = row & 7;
              const int p0 = row * 8 + ((2 * g) ^ x), p1 = row * 8 + ((2 * g + 1) ^ x);
              const float4 v0 = a[p0], v1 = a[p1];
              float4 h0, h1;
              h0.x = __uint_as_float(cb16_hi(v0.x)); h0.y = __uint_as_float(cb16_hi(v0.y));
              h0.z = __uint_as_float(cb16_hi(v0.z)); h0.w = __uint_as_float(cb16_hi(v0.w));
              h1.x = __uint_as_float(cb16_hi(v1.x)); h1.y = __uint_as_float(cb16_hi(v1.y));
              h1.z = __uint_as_float(cb16_hi(v1.z)); h1.w = __uint_as_float(cb16_hi(v1.w));
              if (NNB_CB16_WB) {
                a[p0] = h0;
                a[p1] = h1;
              }
              corr[p0] = make_uint4(bf16x2_rn(h0.x, h0.y), bf16x2_rn(h0.z, h0.w),
                                    bf16x2_rn(h1.x, h1.y), bf16x2_rn(h1.z, h1.w));
              corr[p1] = make_uint4(bf16x2_rn(v0.x - h0.x, v0.y - h0.y), bf16x2_rn(v0.z - h0.z, v0.w - h0.w),
                                    bf16x2_rn(v1.x - h1.x, v1.y - h1.y), bf16x2_rn(v1.z - h1.z, v1.w - h1.w));
            }
          } else {
#pragma unroll 4
          for (int i = ct; i < ((NNB_TC_DBG & 4) ? 0 : A_BYTES / 16); i += 32 * CONV_WARPS) {
            float4 v = a[i], h, l;
            if (C::RN_SS == 2) {
              // truncated hi left to the hardware (the raw tile), lo rounded
              // to TF32 here: its rounding error is unbiased and the tile is
              // not written back (one store per 4 elements instead of two)
              float4 r;
              r.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
              r.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
              r.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
              r.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
              l.x = __uint_as_float(split_hi(r.x)); l.y = __uint_as_float(split_hi(r.y));
              l.z = __uint_as_float(split_hi(r.z)); l.w = __uint_as_float(split_hi(r.w));
              lo[i] = l;
              continue;
            }
            if (C::RN_SS) {
              // round-to-nearest split written back: lo of either sign, so
              // its own TF32 truncation is unbiased (the raw tile would be
              // truncated by the hardware, leaving lo >= 0 and biased)
              h.x = __uint_as_float(split_hi(v.x)); h.y = __uint_as_float(split_hi(v.y));
              h.z = __uint_as_float(split_hi(v.z)); h.w = __uint_as_float(split_hi(v.w));
            } else {
              h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
              h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
              h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
              h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
            }
            l.x = v.x - h.x; l.y = v.y - h.y; l.z = v.z - h.z; l.w = v.w - h.w;
            if (NNB_HI_INPLACE || C::RN_SS) a[i] = h;
            lo[i] = l;
          }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          arrive_mma(&lo_ready[s]);
          if (++s == C::NS) { s = 0; ph ^= 1; }
        }
      }
     }
    } else {
      NNB_SETREG_INC();
      // ---------------- epilogue ----------------
      const int q = warp & 3;                    // TMEM lane quarter of this warp
      const int r = q * 32 + lane;               // row within the tile
      const int cbeg = ((warp - EPI_W0) >> 2) * EPI_COLS;
      const float* bias = at<float>(pool, C::B_OFF);
      const float* ps = at<float>(pool, C::PS_OFF);
      const float* po = at<float>(pool, C::PO_OFF);
      float* out = at<float>(arena, C::OUT_OFF);
      const int ew = warp - EPI_W0;
      float4* ebuf = epi_stage + ew * NBUF * 128;      // this warp's 2 KB boxes
      int acc = 0;
      u32 aph = 0, rph = 0;
      constexpr int ECQ = C::BN / 4, ETAPS = EDW ? C::E_KH * C::E_KW : 1;
      const int et = threadIdx.x - 32 * EPI_W0, ecq = et % ECQ;
      for (int t = t0; t < tiles; t += tstep) {
        const int mb = mb_of(t), nb = t % NTN;
        // TMA box (32 rows of this warp x 16 columns from `col`) load / store
        auto box_io = [&](bool load, float4* b, int col) {
          if (C::CONV) {       // rows = 2 image rows x 16 pixels of the 8 x 16 tile
            const int img = mb / TPI, tt = mb % TPI;
            const int x = (tt % TX) * TW, y = (tt / TX) * TH + 2 * q;
            if (load) tma_load_4d(b, tmR, &rbar[ew], col, x, y, img);
            else tma_store_4d(tmO, b, col, x, y, img);
          } else {
            if (load) tma_load_2d(b, tmR, &rbar[ew], col, mb * BM + q * 32);
            else tma_store_2d(tmO, b, col, mb * BM + q * 32);
          }
        };
        int ngrp = 0;                                   // live 16-column groups (warp-uniform)
#pragma unroll
        for (int g = 0; g < EGRP; ++g)
          ngrp += (cbeg + g * 16 < C::BN && nb * C::BN + cbeg + g * 16 < C::N) ? 1 : 0;
        if constexpr (ET && C::RES) {
          // prefetch the residual boxes; they land while the MMAs run
          if (lane == 0 && ngrp > 0) {
            bulk_wait_read<0>();                        // last tile's stores have read them
            mbar_expect_tx(&rbar[ew], ngrp * 2048);
            for (int g = 0; g < ngrp; ++g) box_io(true, ebuf + g * 128, nb * C::BN + cbeg + g * 16);
          }
        }
        if constexpr (K9) {
          // ---- all taps packed: D''[pixel][ky][kx][co] -> out ----
          constexpr int GCO = C::CO / 2;                 // output channels per warp group (8)
          constexpr int NT = C::KH * C::KW;
          const int g = (warp - EPI_W0) >> 2;
          float d[NT][GCO];
#pragma unroll
          for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int i = 0; i < GCO; ++i) d[t][i] = 0.f;
          for (int ch = 0; ch < NCHUNK; ++ch) {
            mbar_wait(&tfull[acc], aph);
            tc_fence_after();
            if (!(NNB_TC_DBG & 8)) {
              u32 rv[NT][GCO];
#pragma unroll
              for (int t = 0; t < NT; ++t)
                tmem_ld_async<GCO>(tmem + ((u32)(q * 32) << 16) + acc * ACC_COLS + t * C::CO + g * GCO,
                                   rv[t]);
              tmem_wait_ld();
#pragma unroll
              for (int t = 0; t < NT; ++t) {
                tmem_pin_n<GCO>(rv[t]);
#pragma unroll
                for (int i = 0; i < GCO; ++i) d[t][i] += __uint_as_float(rv[t][i]);
              }
            }
            tc_fence_before();
            arrive_mma(&tempty[acc]);
            if (++acc == ABUF) { acc = 0; aph ^= 1; }
          }
          // horizontal: h[ky] = sum_kx D''(column + kx)[ky][kx] (lanes of one image row)
          float h[C::KH][GCO];
#pragma unroll
          for (int ky = 0; ky < C::KH; ++ky)
#pragma unroll
            for (int i = 0; i < GCO; ++i) {
              float v = d[ky * C::KW][i];
#pragma unroll
              for (int kx = 1; kx < C::KW; ++kx)
                v += __shfl_down_sync(0xffffffffu, d[ky * C::KW + kx][i], kx);
              h[ky][i] = v;
            }
          // vertical: out(row) = h[0](row) + h[1](row + 1) + h[2](row + 2); rows
          // two apart live in the next warp quarter, so h[1..] go through the
          // group's half of the staging area ([ky-1][tile row][column][GCO])
          float* hx = reinterpret_cast<float*>(epi_stage) + g * ((C::KH - 1) * 8 * 16 * GCO);
          const int rr = q * 32 + lane, trow = rr / TW, tcol = rr % TW;
          named_sync128(9 + g);                          // last tile's reads are done
#pragma unroll
          for (int ky = 1; ky < C::KH; ++ky)
#pragma unroll
            for (int i = 0; i < GCO; i += 4)
              *reinterpret_cast<float4*>(hx + (((ky - 1) * 8 + trow) * 16 + tcol) * GCO + i) =
                  make_float4(h[ky][i], h[ky][i + 1], h[ky][i + 2], h[ky][i + 3]);
          named_sync128(9 + g);                          // this tile's partial rows stored
          if (NNB_TC_DBG & 16) continue;
          const int img = mb / TPI, tt = mb % TPI;
          const int oy = (tt / TX) * THO + trow, ox = (tt % TX) * OW + tcol;
          if (trow < THO && tcol < OW && img < n && oy < C::HO && ox < C::WO) {
            float y[GCO];
#pragma unroll
            for (int i = 0; i < GCO; ++i) {
              float v = h[0][i];
#pragma unroll
              for (int ky = 1; ky < C::KH; ++ky)
                v += hx[(((ky - 1) * 8 + trow + ky) * 16 + tcol) * GCO + i];
              const int col = g * GCO + i;
              y[i] = finish<C::ACT, EMODE, C::POST>(v + __ldg(bias + col), ps, po, col);
            }
            float* dst = out + (long long)img * (C::OUT_IMG / 4) + ((long long)oy * C::WO + ox) * C::CO +
                         g * GCO;
#pragma unroll
            for (int i = 0; i < GCO; i += 4)
              *reinterpret_cast<float4*>(dst + i) = make_float4(y[i], y[i + 1], y[i + 2], y[i + 3]);
          }
          continue;
        }
        if constexpr (KP && C::CO / 2 > 16 && NCHUNK == 1 && NACC == 1) {
          // ---- packed horizontal taps, wide groups (CO = 64: N = 192): one
          // chunk, so each 16-channel group is drained, combined, finished and
          // stored on its own (registers: KW x 16 loaded values at a time) ----
          constexpr int GCO = C::CO / 2;
          const int g = (warp - EPI_W0) >> 2;
          const int img = mb / TPI, tt = mb % TPI;
          const int rr0 = q * 32 + lane, w0 = rr0 % TW;
          auto pix = [&](int rr, long long& ob) {
            const int w = rr % TW;
            const int oy = (tt / TX) * TH + rr / TW, ox = (tt % TX) * OW + w;
            ob = (long long)img * (C::OUT_IMG / 4) +
                 ((long long)(oy * C::UPF) * C::WO * C::UPF + ox * C::UPF) * C::CO + g * GCO;
            return img < n && w < OW && oy < C::HO && ox < C::WO;
          };
          mbar_wait(&tfull[acc], aph);
          tc_fence_after();
#pragma unroll 1
          for (int h = 0; h < GCO / 16; ++h) {
            u32 rv[C::KW][16], rc[C::KW][16];
#pragma unroll
            for (int kx = 0; kx < C::KW; ++kx) {
              const u32 ta = tmem + ((u32)(q * 32) << 16) + acc * ACC_COLS + kx * C::CO + g * GCO + h * 16;
              tmem_ld16_async(ta, rv[kx]);
              if (CS) tmem_ld16_async(ta + C::BN, rc[kx]);
            }
            tmem_wait_ld();
            float y[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              float part[C::KW];
#pragma unroll
              for (int kx = 0; kx < C::KW; ++kx) {
                tmem_pin_n<16>(rv[kx]);
                if (CS) tmem_pin_n<16>(rc[kx]);
                part[kx] = CS ? __uint_as_float(rv[kx][i]) + __uint_as_float(rc[kx][i])
                              : __uint_as_float(rv[kx][i]);
              }
              float sacc = part[0];
#pragma unroll
              for (int kx = 1; kx < C::KW; ++kx) sacc += __shfl_down_sync(0xffffffffu, part[kx], kx);
              const int col = g * GCO + h * 16 + i;
              y[i] = finish<C::ACT, EMODE, C::POST>(sacc + __ldg(bias + col), ps, po, col);
            }
            if (NNB_TC_DBG & 16) continue;
            if constexpr (C::DPOOL) {
              dual_pool_store<16>(arena, y, (rr0 & 17) == 0 && w0 + 1 < OW, img,
                                  (tt / TX) * TH + rr0 / TW, (tt % TX) * OW + w0, g * GCO + h * 16, n);
            }
            float4* st = epi_stage + (warp - EPI_W0) * 128;
            stage_rows<16>(st, y, lane);
#pragma unroll
            for (int p = 0; p < 4; ++p) {
              const int row = p * 8 + lane / 4, c = lane % 4;
              long long ob;
              if (pix(q * 32 + row, ob)) {
                const float4 x = st[stage_slot<16>(row, c)];
#pragma unroll
                for (int rep = 0; rep < C::UPF * C::UPF; ++rep)
                  *reinterpret_cast<float4*>(
                      out + ob + ((long long)(rep / C::UPF) * C::WO * C::UPF + rep % C::UPF) * C::CO +
                      h * 16 + 4 * c) = x;
              }
            }
            __syncwarp();
          }
          tc_fence_before();
          arrive_mma(&tempty[acc]);
          if (++acc == ABUF) { acc = 0; aph ^= 1; }
          continue;
        }
        if constexpr (KP && !(C::CO / 2 > 16 && NCHUNK == 1 && NACC == 1)) {
          // ---- packed horizontal taps: reduce chunks, combine across lanes ----
          constexpr int GCO = C::CO / EPI_GROUPS;        // output channels per warp group
          static_assert(GCO == 8 || GCO % 16 == 0, "KPACK staged store width");
          const int g = (warp - EPI_W0) >> 2;
          float run[C::KW][GCO];
#pragma unroll
          for (int kx = 0; kx < C::KW; ++kx)
#pragma unroll
            for (int i = 0; i < GCO; ++i) run[kx][i] = 0.f;
          for (int ch = 0; ch < NCHUNK; ++ch) {
            mbar_wait(&tfull[acc], aph);
            tc_fence_after();
            const int ksteps = (ch == NCHUNK - 1 ? KB - ch * CHUNK_KB : CHUNK_KB) * KSTEPS;
            // every tap of a chain in flight, one wait (the drain is the KPACK
            // epilogue's critical path: 12 serial load+wait pairs per tile before)
#pragma unroll
            for (int c = 0; c < ((NNB_TC_DBG & 8) ? 0 : NACC); ++c) {
              if (c >= ksteps) break;
              u32 rv[C::KW][GCO], rc[C::KW][GCO];
#pragma unroll
              for (int kx = 0; kx < C::KW; ++kx) {
                const u32 ta = tmem + ((u32)(q * 32) << 16) + acc * ACC_COLS + c * CW +
                               kx * C::CO + g * GCO;
                tmem_ld_async<GCO>(ta, rv[kx]);
                if (CS) tmem_ld_async<GCO>(ta + C::BN, rc[kx]);
              }
              tmem_wait_ld();
#pragma unroll
              for (int kx = 0; kx < C::KW; ++kx) {
                tmem_pin_n<GCO>(rv[kx]);
                if (CS) tmem_pin_n<GCO>(rc[kx]);
#pragma unroll
                for (int i = 0; i < GCO; ++i)
                  run[kx][i] += CS ? __uint_as_float(rv[kx][i]) + __uint_as_float(rc[kx][i])
                                   : __uint_as_float(rv[kx][i]);
              }
            }
            tc_fence_before();
            arrive_mma(&tempty[acc]);
            if (++acc == ABUF) { acc = 0; aph ^= 1; }
          }
          if (NNB_TC_DBG & 16) continue;
          const int img = mb / TPI, tt = mb % TPI;
          // output pixel of tile row rr (16 input columns per tile row)
          auto pix = [&](int rr, long long& ob) {
            const int w = rr % TW;
            const int oy = (tt / TX) * TH + rr / TW, ox = (tt % TX) * OW + w;
            ob = (long long)img * (C::OUT_IMG / 4) +
                 ((long long)(oy * C::UPF) * C::WO * C::UPF + ox * C::UPF) * C::CO + g * GCO;
            return img < n && w < OW && oy < C::HO && ox < C::WO;
          };
          float y[GCO];
#pragma unroll
          for (int i = 0; i < GCO; ++i) {
            float sacc = run[0][i];
#pragma unroll
            for (int kx = 1; kx < C::KW; ++kx) sacc += __shfl_down_sync(0xffffffffu, run[kx][i], kx);
            const int col = g * GCO + i;
            y[i] = finish<C::ACT, EMODE, C::POST>(sacc + __ldg(bias + col), ps, po, col);
          }
          if constexpr (C::DPOOL) {
            const int rr = q * 32 + lane, w = rr % TW;
            dual_pool_store<GCO>(arena, y, (rr & 17) == 0 && w + 1 < OW, img,
                                 (tt / TX) * TH + rr / TW, (tt % TX) * OW + w, g * GCO, n);
          }
#pragma unroll
          for (int h = 0; h < (GCO + 15) / 16; ++h) {
            constexpr int NC = GCO < 16 ? GCO : 16;
            constexpr int CPR = NC / 4;
            float4* st = epi_stage + (warp - EPI_W0) * 128;
            stage_rows<NC>(st, y + h * 16, lane);
#pragma unroll
            for (int p = 0; p < CPR; ++p) {
              const int row = p * (32 / CPR) + lane / CPR, c = lane % CPR;
              long long ob;
              if (pix(q * 32 + row, ob)) {
                const float4 x = st[stage_slot<NC>(row, c)];
#pragma unroll
                for (int rep = 0; rep < C::UPF * C::UPF; ++rep)
                  *reinterpret_cast<float4*>(
                      out + ob + ((long long)(rep / C::UPF) * C::WO * C::UPF + rep % C::UPF) * C::CO +
                      h * 16 + 4 * c) = x;
              }
            }
            __syncwarp();
          }
          continue;
        }
        // FP32 (round-to-nearest) reduction of the per-chunk tensor-core sums
        float run[EPI_COLS];
#pragma unroll
        for (int i = 0; i < EPI_COLS; ++i) run[i] = 0.f;
        for (int ch = 0; ch < NCHUNK; ++ch) {
          mbar_wait(&tfull[acc], aph);
          tc_fence_after();
          // chains written in this chunk (a short last chunk may not reach all)
          const int ksteps = (ch == NCHUNK - 1 ? KB - ch * CHUNK_KB : CHUNK_KB) * KSTEPS;
          // batches of GB 16-column groups: all their loads in flight, one wait
          // (32 loaded registers per batch: the 64-column running sums stay in
          // registers next to them)
          constexpr int GB = (EPI_COLS / 16 >= 2 && !CS) ? 2 : 1;
          const bool rd_c = CS && (!C::CORR_WHOLE || ch == NCHUNK - 1);   // correction read
          if constexpr (C::CORR_WHOLE && NACC == 1 && NNB_DRAIN2 && EPI_COLS % 32 == 0) {
            // mid-tile chunk of a whole-K correction chain: only the main
            // columns are read, two 16-column groups per wait (the correction
            // registers hold the second) -- half the load round trips while
            // the MMAs wait for this drain
            if (!rd_c) {
#pragma unroll
              for (int g0 = 0; g0 < ((NNB_TC_DBG & 8) ? 0 : EPI_COLS / 16); g0 += 2) {
                if (cbeg + g0 * 16 < C::BN) {
                  u32 rv[16], rw[16];
                  const u32 ta = tmem + ((u32)(q * 32) << 16) + acc * ACC_COLS + cbeg + g0 * 16;
                  tmem_ld16_async(ta, rv);
                  tmem_ld16_async(ta + 16, rw);
                  tmem_wait_ld();
                  tmem_pin(rv);
                  tmem_pin(rw);
#pragma unroll
                  for (int i = 0; i < 16; ++i) {
                    run[g0 * 16 + i] += __uint_as_float(rv[i]);
                    run[g0 * 16 + 16 + i] += __uint_as_float(rw[i]);
                  }
                }
              }
              tc_fence_before();
              arrive_mma(&tempty[acc]);
              if (++acc == ABUF) { acc = 0; aph ^= 1; }
              continue;
            }
          }
#pragma unroll
          for (int g0 = 0; g0 < ((NNB_TC_DBG & 8) ? 0 : EPI_COLS / 16); g0 += GB) {
            if (cbeg + g0 * 16 < C::BN) {            // warp-uniform (whole batch valid)
#pragma unroll
              for (int c = 0; c < NACC; ++c) {
                if (c >= ksteps) break;
                u32 rv[GB][16], rc[GB][16];
#pragma unroll
                for (int b = 0; b < GB; ++b) {
                  const u32 ta = tmem + ((u32)(q * 32) << 16) + acc * ACC_COLS + c * CW +
                                 cbeg + (g0 + b) * 16;
                  tmem_ld16_async(ta, rv[b]);
                  if (rd_c) tmem_ld16_async(ta + C::BN, rc[b]);
                }
                tmem_wait_ld();
#pragma unroll
                for (int b = 0; b < GB; ++b) {
                  tmem_pin(rv[b]);
                  if (rd_c) tmem_pin(rc[b]);
#pragma unroll
                  for (int i = 0; i < 16; ++i)
                    run[(g0 + b) * 16 + i] += rd_c ? __uint_as_float(rv[b][i]) + __uint_as_float(rc[b][i])
                                                   : __uint_as_float(rv[b][i]);
                }
              }
            }
          }
          tc_fence_before();
          arrive_mma(&tempty[acc]);
          if (++acc == ABUF) { acc = 0; aph ^= 1; }
        }
        if (NNB_TC_DBG & 16) continue;
        // output position of tile row rr: element offset of its first channel
        auto rowpos = [&](int rr, long long& obase) {
          bool live;
          if (C::CONV) {
            const int img = mb / TPI, tt = mb % TPI;
            const int oy = (tt / TX) * TH + rr / TW, ox = (tt % TX) * TW + rr % TW;
            live = img < n && oy < C::HO && ox < C::WO;
            obase = (long long)img * (C::OUT_IMG / 4) + ((long long)oy * C::WO + ox) * C::N;
            if (C::UPF > 1)     // fused nearest upsampling: first replica of the pixel
              obase = (long long)img * (C::OUT_IMG / 4) +
                      ((long long)(oy * C::UPF) * C::WO * C::UPF + ox * C::UPF) * C::N;
            if (C::POOL) {      // pooled row index of the 2x2 window this row leads
              const int py = (tt / TX) * (TH / 2) + (rr / TW) / 2,
                        px = (tt % TX) * (TW / 2) + (rr % TW) / 2;
              live = img < n && py < C::PHO && px < C::PWO && (rr & 17) == 0;
              obase = (long long)img * (C::OUT_IMG / 4) + ((long long)py * C::PWO + px) * C::N;
            }
          } else {
            const long long m = (long long)mb * BM + rr;
            live = m < rows;
            obase = m * C::N;
            if (C::UPF > 1) {   // 1x1 conv rows: pixel (oy, ox) of image m / ROWS
              const long long img = m / C::ROWS;
              const int ri = (int)(m - img * C::ROWS), oy = ri / C::WO, ox = ri % C::WO;
              obase = img * (C::OUT_IMG / 4) +
                      ((long long)(oy * C::UPF) * C::WO * C::UPF + ox * C::UPF) * C::N;
            }
          }
          return live;
        };
        const float* res = at<float>(arena, C::RES_OFF);
        if constexpr (HEAD) {
#pragma unroll
          for (int i = 0; i < EPI_COLS; i += 2) {
            const int c0 = cbeg + i < C::N ? cbeg + i : C::N - 1;
            const int c1 = cbeg + i + 1 < C::N ? cbeg + i + 1 : C::N - 1;
            const float2 y = finish2<C::ACT, EMODE, C::POST>(
                make_float2(run[i] + __ldg(bias + c0), run[i + 1] + __ldg(bias + c1)), ps, po, c0, c1);
            run[i] = y.x;
            run[i + 1] = y.y;
          }
          float hp[C::HN];
          float* xch = reinterpret_cast<float*>(epi_stage + (ew & 3) * NBUF * 128);   // [HN][32]
          if (cbeg == 0) {
#pragma unroll
            for (int j = 0; j < C::HN; ++j) hp[j] = C::hbias(j);
            head_dot<0>(run, hp);
            named_sync64(1 + q);                     // partials stored
#pragma unroll
            for (int j = 0; j < C::HN; ++j) hp[j] = add(hp[j], xch[j * 32 + lane]);
            named_sync64(5 + q);                     // partials consumed
            const float* hps = at<float>(pool, C::H_PS_OFF);
            const float* hpo = at<float>(pool, C::H_PO_OFF);
            float hv[C::HN];
#pragma unroll
            for (int j = 0; j < C::HN; ++j) hv[j] = finish<C::H_ACT, EMODE, C::H_POST>(hp[j], hps, hpo, j);
            if (C::H_SOFTMAX) {
              softmax_row_regs<C::HN, C::HN, C::H_SMEXP>(hv);
            }
            const long long m = (long long)mb * BM + r;
            if (m < rows) {
              float* d = at<float>(arena, C::H_OUT_OFF) + m * C::HN;
#pragma unroll
              for (int j = 0; j < C::HN; ++j) d[j] = hv[j];
            }
          } else {
#pragma unroll
            for (int j = 0; j < C::HN; ++j) hp[j] = 0.f;
            if (cbeg < C::N) head_dot<EPI_COLS>(run, hp);
#pragma unroll
            for (int j = 0; j < C::HN; ++j) xch[j * 32 + lane] = hp[j];
            named_sync64(1 + q);
            named_sync64(5 + q);
          }
          continue;
        }
#pragma unroll
        for (int g = 0; g < EPI_COLS / 16; ++g) {
          const int col0 = nb * C::BN + cbeg + g * 16;
          if (cbeg + g * 16 >= C::BN || col0 >= C::N) continue;   // warp-uniform
          float* v = run + g * 16;
          if constexpr (paired_act<C::ACT, EMODE>() && !C::POOL) {
            // two columns per f32x2 instruction (nnb_common.cuh finish2)
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
              const int c0 = col0 + i < C::N ? col0 + i : C::N - 1;
              const int c1 = col0 + i + 1 < C::N ? col0 + i + 1 : C::N - 1;
              float2 y = make_float2(v[i] + __ldg(bias + c0), v[i + 1] + __ldg(bias + c1));
              if (!(NNB_TC_DBG & 32)) y = finish2<C::ACT, EMODE, C::POST>(y, ps, po, c0, c1);
              v[i] = y.x;
              v[i + 1] = y.y;
            }
          } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int col = col0 + i < C::N ? col0 + i : C::N - 1;
            float y = v[i] + __ldg(bias + col);
            if (!(NNB_TC_DBG & 32)) y = finish<C::ACT, EMODE, C::POST>(y, ps, po, col);
            if (C::POOL) {     // lanes w, w^1 (same image row), w^16 (next row)
              y = fmaxf(y, __shfl_xor_sync(0xffffffffu, y, 1));
              y = fmaxf(y, __shfl_xor_sync(0xffffffffu, y, 16));
            }
            v[i] = y;
          }
          }
          if constexpr (C::DPOOL && C::CONV) {
            const int img = mb / TPI, tt = mb % TPI;
            dual_pool_store<16>(arena, v, (r & 17) == 0, img, (tt / TX) * TH + r / TW,
                                (tt % TX) * TW + r % TW, col0, n);
          }
          if constexpr (EDW) {
            float* trow = reinterpret_cast<float*>(epi_stage) + r * ETS + cbeg + g * 16;
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<float4*>(trow + 4 * j) =
                  make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          } else if constexpr (ET) {
            float4* b = ebuf + (g % NBUF) * 128;
            if (C::RES) {
              if (g == 0) mbar_wait(&rbar[ew], rph);
            } else {
              if (lane == 0) bulk_wait_read<NBUF - 1>();  // the box's previous store has read it
              __syncwarp();
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int sl = stage_slot<16>(lane, j);
              float4 x = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
              if (C::RES) {
                const float4 rv = b[sl];
                x.x = add(x.x, rv.x); x.y = add(x.y, rv.y);
                x.z = add(x.z, rv.z); x.w = add(x.w, rv.w);
              }
              b[sl] = x;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              box_io(false, b, col0);
              bulk_commit();
            }
          } else if constexpr (C::N % 16 == 0 && C::EPI_ST) {
            // coalesced: 8 lanes per row segment of 16 columns (residual too)
            float4* st = epi_stage + (warp - EPI_W0) * 128;
            stage_rows<16>(st, v, lane);
#pragma unroll
            for (int p = 0; p < 4; ++p) {
              const int row = p * 8 + (lane >> 2), c = lane & 3;
              long long ob;
              if (rowpos(q * 32 + row, ob)) {
                float4 x = st[stage_slot<16>(row, c)];
                if (C::RES) {
                  const float4 rv = __ldg(reinterpret_cast<const float4*>(res + ob + col0 + 4 * c));
                  x.x = add(x.x, rv.x); x.y = add(x.y, rv.y);
                  x.z = add(x.z, rv.z); x.w = add(x.w, rv.w);
                }
#pragma unroll
                for (int rep = 0; rep < C::UPF * C::UPF; ++rep)
                  *reinterpret_cast<float4*>(
                      out + ob + ((long long)(rep / C::UPF) * C::WO * C::UPF + rep % C::UPF) * C::N +
                      col0 + 4 * c) = x;
              }
            }
            __syncwarp();
          } else {
            long long ob;
            const bool live = rowpos(r, ob);
            if (live) {
#pragma unroll
              for (int rep = 0; rep < C::UPF * C::UPF; ++rep) {
                float* d = out + ob + ((long long)(rep / C::UPF) * C::WO * C::UPF + rep % C::UPF) * C::N;
                if (C::RES) {
#pragma unroll
                  for (int i = 0; i < 16; ++i)
                    if (col0 + i < C::N) v[i] = add(v[i], __ldg(res + ob + col0 + i));
                }
                if (C::N % 16 == 0) {
#pragma unroll
                  for (int i = 0; i < 16; i += 4)
                    *reinterpret_cast<float4*>(d + col0 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                } else {
#pragma unroll
                  for (int i = 0; i < 16; ++i)
                    if (col0 + i < C::N) d[col0 + i] = v[i];
                }
              }
            }
          }
        }
        if constexpr (EDW) {
          // this thread's channel quad of the depthwise kernel and bias (the
          // same for every row task it takes); the loads fly across the barrier
          const int ch = nb * C::BN + 4 * ecq;
          const int chl = ch < C::N ? ch : 0;
          float4 ewq[ETAPS];
#pragma unroll
          for (int k = 0; k < ETAPS; ++k)
            ewq[k] = __ldg(reinterpret_cast<const float4*>(at<float>(pool, C::E_W_OFF) + k * C::N + chl));
          const float4 eb4 = __ldg(reinterpret_cast<const float4*>(at<float>(pool, C::E_B_OFF) + chl));
          named_sync256(9);                          // the tile is parked
          constexpr int IMGS = EBAND ? 1 : BM / EP;
          if constexpr (C::E_GAP != 0) {
            // global average pool: (image of the tile, channel quad) tasks sum the
            // image's parked rows in pixel order and divide by the count (the Pool
            // kernel's operations, pkg/src/nnjit/interpreter.py:85-95)
            constexpr int TPG = EPI_THREADS / ECQ;
            const float* Tg = reinterpret_cast<const float*>(epi_stage) + 4 * ecq;
#pragma unroll 1
            for (int li = et < TPG * ECQ ? et / ECQ : IMGS; li < IMGS; li += TPG) {
              const long long img = (long long)mb * IMGS + li;
              if (img >= n || ch >= C::N) continue;
              float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
              for (int p = 0; p < EP; ++p) {
                const float4 v = *reinterpret_cast<const float4*>(Tg + (li * EP + p) * ETS);
                a.x = add(a.x, v.x); a.y = add(a.y, v.y); a.z = add(a.z, v.z); a.w = add(a.w, v.w);
              }
              const float cf = (float)EP;
              *reinterpret_cast<float4*>(at<float>(arena, C::E_OUT_OFF + img * C::E_OUT_IMG) + ch) =
                  make_float4(dvd(a.x, cf), dvd(a.y, cf), dvd(a.z, cf), dvd(a.w, cf));
            }
          } else {
          constexpr int RT = EBAND ? EB_OT : IMGS * C::E_HO;   // output rows of the tile
          constexpr int OXC = C::E_WO < 4 ? C::E_WO : 4;       // outputs per register window
          constexpr int NWIN = (C::E_WO + OXC - 1) / OXC;      // windows per output row
          constexpr int XW = (OXC - 1) * C::E_S + C::E_KW;     // input columns of a window
          constexpr int TPR = EPI_THREADS / ECQ;               // (row, window) tasks in flight
          const float* T = reinterpret_cast<const float*>(epi_stage) + 4 * ecq;
          const float* eps = at<float>(pool, C::E_PS_OFF);
          const float* epo = at<float>(pool, C::E_PO_OFF);
#pragma unroll 1
          for (int rw = et < TPR * ECQ ? et / ECQ : RT * NWIN; rw < RT * NWIN; rw += TPR) {
            const int rt = rw / NWIN, ox0 = (rw - rt * NWIN) * OXC;
            int li, oy, trow;          // image of the tile, output row, tile row of input row iy = 0
            long long img;
            if (EBAND) {
              const int tt = mb % EB_TPI;
              li = 0; oy = tt * EB_OT + rt; img = mb / EB_TPI;
              trow = -(tt * EB_OT * C::E_S - C::E_PT);
              if (oy >= C::E_HO) continue;
            } else {
              li = rt / C::E_HO; oy = rt - li * C::E_HO; img = (long long)mb * IMGS + li;
              trow = li * C::E_H;
            }
            if (img >= n || ch >= C::N) continue;
            const int ixb = ox0 * C::E_S - C::E_PL;              // first input column of the window
            float4 a[OXC];
#pragma unroll
            for (int o = 0; o < OXC; ++o) a[o] = eb4;
#pragma unroll
            for (int ky = 0; ky < C::E_KH; ++ky) {
              const int iy = oy * C::E_S - C::E_PT + ky;
              if (iy < 0 || iy >= C::E_H) continue;              // taps outside the image are skipped
              const float* row = T + ((trow + iy) * C::E_W + ixb) * ETS;
              float4 x[XW];
#pragma unroll
              for (int j = 0; j < XW; ++j)                        // ... or read as zeros
                x[j] = (ixb + j >= 0 && ixb + j < C::E_W) ? *reinterpret_cast<const float4*>(row + j * ETS)
                                                          : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
              for (int kx = 0; kx < C::E_KW; ++kx) {
                const float4 w4 = ewq[ky * C::E_KW + kx];
#pragma unroll
                for (int o = 0; o < OXC; ++o) {
                  const int j = o * C::E_S + kx;
                  if (C::E_FMA) {     // one rounding per tap (within the FP32 gate), FFMA2
                    const float2 lo = __ffma2_rn(make_float2(x[j].x, x[j].y), make_float2(w4.x, w4.y),
                                                 make_float2(a[o].x, a[o].y));
                    const float2 hi = __ffma2_rn(make_float2(x[j].z, x[j].w), make_float2(w4.z, w4.w),
                                                 make_float2(a[o].z, a[o].w));
                    a[o] = make_float4(lo.x, lo.y, hi.x, hi.y);
                  } else {            // the interpreter's mul-then-add
                    a[o].x = add(a[o].x, mul(x[j].x, w4.x)); a[o].y = add(a[o].y, mul(x[j].y, w4.y));
                    a[o].z = add(a[o].z, mul(x[j].z, w4.z)); a[o].w = add(a[o].w, mul(x[j].w, w4.w));
                  }
                }
              }
            }
            float* d = at<float>(arena, C::E_OUT_OFF + img * C::E_OUT_IMG) +
                       ((long long)oy * C::E_WO + ox0) * C::N + ch;
#pragma unroll
            for (int o = 0; o < OXC; ++o)
              if (ox0 + o < C::E_WO)
                *reinterpret_cast<float4*>(d + o * C::N) = make_float4(
                    finish<C::E_ACT, EMODE, C::E_POST>(a[o].x, eps, epo, ch),
                    finish<C::E_ACT, EMODE, C::E_POST>(a[o].y, eps, epo, ch + 1),
                    finish<C::E_ACT, EMODE, C::E_POST>(a[o].z, eps, epo, ch + 2),
                    finish<C::E_ACT, EMODE, C::E_POST>(a[o].w, eps, epo, ch + 3));
          }
          }
          if (t + tstep < tiles) named_sync256(9);   // the next tile parks over this one
        }
        if (C::RES && ngrp > 0) rph ^= 1;
      }
      if (ET && lane == 0) bulk_wait_all();        // boxes stay valid until stored
    }
    tc_fence_before();
    if (PAIR) cluster_sync();          // neither CTA leaves while its peer may still use it
    else __syncthreads();
    if (warp == 1) {
      tc_fence_after();
      if (PAIR)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(TMEM_COLS));
      else
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(TMEM_COLS));
    }
  }
};

}  // namespace nnb
