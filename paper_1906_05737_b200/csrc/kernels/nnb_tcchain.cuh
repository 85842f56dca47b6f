// nnb_tcchain.cuh -- the 8x8 stage of a MobileNet-style net (alternating
// depthwise 3x3 and pointwise 1x1 layers, planner.fuse_tc_chain) in one
// launch on the tensor cores: one CTA holds two images (2 x 64 pixels = the
// 128 rows of a tcgen05 M=128 tile) for the whole run.
//
// Per layer pair, all inside the CTA, no HBM traffic between layers:
//   depthwise  CUDA cores: thread (pixel row r = TMEM lane, 16 channels)
//              accumulates the taps in the interpreter's order (bias, then
//              (ky, kx), out-of-image taps skipped -- pkg/src/nnjit/
//              interpreter.py:65-73; FFMA2, two channels per instruction,
//              since this output only feeds the MMA), applies the activation /
//              post-BN, splits a = hi + lo (hi = a rounded to TF32, lo exact)
//              and writes both into TMEM (tcgen05.st) as the A operand;
//   pointwise  one thread issues the 3xTF32 MMAs (kind::tf32, A from TMEM:
//              a_hi*b_hi into the main accumulator, a_hi*b_lo + a_lo*b_hi
//              into the correction accumulator -- the split of
//              nnb_gemm_tc.cuh, error bound DESIGN.md section 4) over weight
//              blocks streamed by bulk copies into a shared-memory ring;
//   epilogue   8 warps read the accumulators (tcgen05.ld; warp w owns lanes
//              32*(w%4).. and half the columns), add main + correction in FP32,
//              bias, activation / post-BN, and store the layer's output into a
//              shared-memory activation buffer [image][pixel][channel] whose
//              pixel stride C+4 keeps the next depthwise's float4 reads
//              conflict-free.
// The weights of each pointwise layer are split and pre-swizzled at compile
// time into the exact shared-memory image of a K-major SW128 operand (one
// 1-D bulk copy per 32-wide k-block: [B_hi | B_lo]); the next layer's blocks
// are issued as soon as the current layer's MMAs have completed, so they land
// while the epilogue and the next depthwise run.  The first step may read
// its input from the arena (HWC), the last writes its output there.
// TMEM: 512 columns = D_main [0, N) + D_corr [N, 2N) + A_hi [256, 256+K) +
// A_lo [256+K, 256+2K), K, N <= 128.
#pragma once
#include "nnb_gemm_tc.cuh"

// NNB_TCC_DBG (diagnostics only, results are garbage): bit 0 skips the
// depthwise taps, bit 1 the MMAs (barriers still complete), bit 2 the weight
// bulk copies (and their waits)
#ifndef NNB_TCC_DBG
#define NNB_TCC_DBG 0
#endif

namespace nnb {

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<u64>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct TcChainCtx {
  u32 tmem;
  u64* full;             // [NSTAGE] weight block landed
  u64* dready;           // accumulators complete
  unsigned char* ring;   // NSTAGE x STAGE_BYTES, 1024-aligned
  float* act;            // [2][64][AS]
  const float* pool;
  const float* src;      // chain input of image 0 of this CTA (HWC, arena)
  float* dst;            // chain output of image 0 (HWC, arena)
  int nimg;              // live images of this CTA (1 or 2)
  u32 full_ph;           // thread 0: expected parity bit per stage
  u32 dready_ph;
  int next_blk;          // thread 0: next weight block of the stream to issue
};

// C: NSTAGE, STAGE_BYTES, NBLK and blk_off(i) / blk_bytes(i) / blk_layer(i):
// the weight stream.  Thread 0 issues blocks while their stage is free,
// i.e. blocks of `layer` (stages are free at a layer boundary).
template <class C>
__device__ __forceinline__ void tcc_issue(TcChainCtx& x, int layer) {
  if (threadIdx.x != 0 || (NNB_TCC_DBG & 4)) return;
  while (x.next_blk < C::NBLK && C::blk_layer(x.next_blk) == layer) {
    const int b = x.next_blk, s = C::blk_stage(b);
    mbar_expect_tx(&x.full[s], (u32)C::blk_bytes(b));
    bulk_g2s(x.ring + s * C::STAGE_BYTES, at<unsigned char>(x.pool, C::blk_off(b)),
             (u32)C::blk_bytes(b), &x.full[s]);
    ++x.next_blk;
  }
}

// depthwise producing the A operand of the next pointwise layer.
// S: H, W, C, HO (=8), WO (=8), KH, KW, S, PT, PL, W_OFF, B_OFF, ACT, MODE, POST,
//    PS_OFF, PO_OFF, SRC_GLOBAL, SRC_IMG (bytes per image of a global source),
//    AS_IN (activation-buffer pixel stride of a shared source), KA (= C, the
//    next layer's K)
template <class S>
struct TccDwA {
  // The depthwise output here only feeds the next layer's 3xTF32 MMA (it is
  // never stored), so its taps use FFMA2 (two channels per instruction, one
  // rounding per tap) -- within the FP32 gate like every other contraction
  // of this path; the stored depthwise layers (TccDwOut, the standalone
  // kernels) keep the interpreter's mul-then-add order.
  __device__ static __forceinline__ void run(TcChainCtx& x) {
    constexpr int T = S::KH * S::KW;
    constexpr int PS = S::SRC_GLOBAL ? S::C : S::AS_IN;     // floats per source pixel
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3, half = warp >> 2;
    const int r = q * 32 + lane, img = r >> 6, p = r & 63;
    const int oy = p / S::WO, ox = p % S::WO;
    const bool live = img < x.nimg && p < S::HO * S::WO;
    const float* wk = at<float>(x.pool, S::W_OFF);
    const float* bs = at<float>(x.pool, S::B_OFF);
    const float* ps = at<float>(x.pool, S::PS_OFF);
    const float* po = at<float>(x.pool, S::PO_OFF);
    const float* src = S::SRC_GLOBAL ? at<float>(x.src, (long long)(img < x.nimg ? img : 0) * S::SRC_IMG)
                                     : x.act + img * 64 * S::AS_IN;
    // the pixel's taps: source offsets (clamped in-bounds, so every load is
    // valid and they issue together) and which taps lie inside the image
    int off[T];
    bool ok[T];
#pragma unroll
    for (int ky = 0; ky < S::KH; ++ky) {
      const int iy = oy * S::S - S::PT + ky;
#pragma unroll
      for (int kx = 0; kx < S::KW; ++kx) {
        const int ix = ox * S::S - S::PL + kx;
        const int t = ky * S::KW + kx;
        ok[t] = live && iy >= 0 && iy < S::H && ix >= 0 && ix < S::W && !(NNB_TCC_DBG & 1);
        const int cy = iy < 0 ? 0 : (iy >= S::H ? S::H - 1 : iy);
        const int cx = ix < 0 ? 0 : (ix >= S::W ? S::W - 1 : ix);
        off[t] = (cy * S::W + cx) * PS;
      }
    }
    constexpr int CH = S::C / 2;                     // channels of this warp's half
    const u32 trow = (u32)(q * 32) << 16;
#pragma unroll 1
    for (int c0 = half * CH; c0 < (half + 1) * CH; c0 += 16) {
      float a[16];
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        const float4 b4 = __ldg(reinterpret_cast<const float4*>(bs + c0 + j));
        float2 a01 = make_float2(b4.x, b4.y), a23 = make_float2(b4.z, b4.w);
        float4 wt[T], xv[T];
#pragma unroll
        for (int t = 0; t < T; ++t) {
          wt[t] = __ldg(reinterpret_cast<const float4*>(wk + t * S::C + c0 + j));
          const float* pv = src + off[t] + c0 + j;
          xv[t] = S::SRC_GLOBAL ? lda(reinterpret_cast<const float4*>(pv))
                                : *reinterpret_cast<const float4*>(pv);
        }
#pragma unroll
        for (int t = 0; t < T; ++t) {
          if (ok[t]) {
            a01 = __ffma2_rn(make_float2(xv[t].x, xv[t].y), make_float2(wt[t].x, wt[t].y), a01);
            a23 = __ffma2_rn(make_float2(xv[t].z, xv[t].w), make_float2(wt[t].z, wt[t].w), a23);
          }
        }
        a[j + 0] = finish<S::ACT, S::MODE, S::POST>(a01.x, ps, po, c0 + j);
        a[j + 1] = finish<S::ACT, S::MODE, S::POST>(a01.y, ps, po, c0 + j + 1);
        a[j + 2] = finish<S::ACT, S::MODE, S::POST>(a23.x, ps, po, c0 + j + 2);
        a[j + 3] = finish<S::ACT, S::MODE, S::POST>(a23.y, ps, po, c0 + j + 3);
      }
      u32 hi[16], lo[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float v = live ? a[i] : 0.f;
        hi[i] = split_hi(v);
        lo[i] = __float_as_uint(v - __uint_as_float(hi[i]));
      }
      tmem_st<16>(x.tmem + trow + 256 + c0, hi);
      tmem_st<16>(x.tmem + trow + 256 + S::KA + c0, lo);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
  }
};

// the chain's first layer is a pointwise one: its input (<= 64 pixels x K,
// HWC in the arena) becomes the A operand directly -- thread (pixel row r,
// its half of the channels) loads its pixel's channels (independent
// coalesced float4 loads), splits them and writes both halves to TMEM.
// S: P (pixels), K, SRC_IMG (bytes per image)
template <class S>
struct TccLoadA {
  __device__ static __forceinline__ void run(TcChainCtx& x) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3, half = warp >> 2;
    const int r = q * 32 + lane, img = r >> 6, p = r & 63;
    const bool live = img < x.nimg && p < S::P;
    const float* src = at<float>(x.src, (long long)(img < x.nimg ? img : 0) * S::SRC_IMG) +
                       (p < S::P ? p : 0) * S::K;
    constexpr int CH = S::K / 2;
    const u32 trow = (u32)(q * 32) << 16;
#pragma unroll
    for (int c0 = half * CH; c0 < (half + 1) * CH; c0 += 16) {
      u32 hi[16], lo[16];
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        const float4 v4 = lda(reinterpret_cast<const float4*>(src + c0 + j));
        const float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float a = live ? v[i] : 0.f;
          hi[j + i] = split_hi(a);
          lo[j + i] = __float_as_uint(a - __uint_as_float(hi[j + i]));
        }
      }
      tmem_st<16>(x.tmem + trow + 256 + c0, hi);
      tmem_st<16>(x.tmem + trow + 256 + S::K + c0, lo);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
  }
};

// pointwise: MMAs over the streamed weight blocks, then the epilogue into
// the activation buffer (or the arena when LAST).
// S: K, N, P (output pixels), LAYER (index in the weight stream), BLK0 (its first block),
//    B_OFF, ACT, MODE, POST, PS_OFF, PO_OFF, AS_OUT, LAST, OUT_IMG (bytes)
template <class C, class S>
struct TccPw {
  static constexpr u32 IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((u32)(S::N >> 3) << 17) |
                               ((u32)(128 >> 4) << 24);
  __device__ static __forceinline__ void run(TcChainCtx& x) {
    __syncthreads();                                 // A (TMEM) complete in every warp
    tc_fence_after();
    if (threadIdx.x == 0) {
#pragma unroll 1
      for (int kb = 0; kb < S::K / 32; ++kb) {
        const int s = C::blk_stage(S::BLK0 + kb);
        if (!(NNB_TCC_DBG & 4)) mbar_wait(&x.full[s], (x.full_ph >> s) & 1u);
        x.full_ph ^= 1u << s;
        tc_fence_after();
        const u32 b_hi = smem_u32(x.ring + s * C::STAGE_BYTES);
        const u32 b_lo = b_hi + S::N * 128;
#pragma unroll
        for (int k = 0; k < ((NNB_TCC_DBG & 2) ? 0 : 4); ++k) {
          const u32 ta = x.tmem + 256 + kb * 32 + 8 * k;
          const u32 accum = (kb | k) != 0;
          mma_tf32_ts(x.tmem, ta, kmajor_desc<128>(b_hi + 32 * k), IDESC, accum);
          mma_tf32_ts(x.tmem + S::N, ta, kmajor_desc<128>(b_lo + 32 * k), IDESC, accum);
          mma_tf32_ts(x.tmem + S::N, ta + S::K, kmajor_desc<128>(b_hi + 32 * k), IDESC, 1);
        }
      }
      mma_commit(x.dready);
      mbar_wait(x.dready, x.dready_ph);
    }
    x.dready_ph ^= 1u;
    __syncthreads();                                 // accumulators ready, ring free
    tc_fence_after();
    tcc_issue<C>(x, S::LAYER + 1);                   // next layer's weights land meanwhile
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3, half = warp >> 2;
    const int r = q * 32 + lane, img = r >> 6, p = r & 63;
    const float* bias = at<float>(x.pool, S::B_OFF);
    const float* ps = at<float>(x.pool, S::PS_OFF);
    const float* po = at<float>(x.pool, S::PO_OFF);
    constexpr int CH = S::N / 2;
    const u32 trow = (u32)(q * 32) << 16;
#pragma unroll 1
    for (int c0 = half * CH; c0 < (half + 1) * CH; c0 += 16) {
      u32 m[16], cr[16];
      float bv[16];
#pragma unroll
      for (int i = 0; i < 16; i += 4) {
        const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + c0 + i));
        bv[i] = b4.x; bv[i + 1] = b4.y; bv[i + 2] = b4.z; bv[i + 3] = b4.w;
      }
      tmem_ld16_async(x.tmem + trow + c0, m);
      tmem_ld16_async(x.tmem + trow + S::N + c0, cr);
      tmem_wait_ld();
      tmem_pin(m);
      tmem_pin(cr);
      float y[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        y[i] = finish<S::ACT, S::MODE, S::POST>(
            __uint_as_float(m[i]) + __uint_as_float(cr[i]) + bv[i], ps, po, c0 + i);
      float* d = S::LAST ? (img < x.nimg && p < S::P
                                ? at<float>(x.dst, (long long)img * S::OUT_IMG) + p * S::N + c0
                                : nullptr)
                         : x.act + (img * 64 + p) * S::AS_OUT + c0;
      if (d) {
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          *reinterpret_cast<float4*>(d + i) = make_float4(y[i], y[i + 1], y[i + 2], y[i + 3]);
      }
    }
    tc_fence_before();
    __syncthreads();                                 // activation buffer complete
  }
};

// closing depthwise from the activation buffer to the arena (HWC).
// S: H, W, C, HO, WO, KH, KW, S, PT, PL, W_OFF, B_OFF, ACT, MODE, POST,
//    PS_OFF, PO_OFF, AS_IN, OUT_IMG (bytes)
template <class S>
struct TccDwOut {
  __device__ static __forceinline__ void run(TcChainCtx& x) {
    constexpr int C4 = S::C / 4, PO = S::HO * S::WO;
    const float* wk = at<float>(x.pool, S::W_OFF);
    const float* bs = at<float>(x.pool, S::B_OFF);
    const float* ps = at<float>(x.pool, S::PS_OFF);
    const float* po = at<float>(x.pool, S::PO_OFF);
    for (int e = threadIdx.x; e < x.nimg * PO * C4; e += blockDim.x) {
      const int img = e / (PO * C4), rem = e % (PO * C4), p = rem / C4, c = 4 * (rem % C4);
      const int oy = p / S::WO, ox = p % S::WO;
      const float* src = x.act + img * 64 * S::AS_IN;
      float4 acc = __ldg(reinterpret_cast<const float4*>(bs + c));
      float4 wt[S::KH * S::KW];
#pragma unroll
      for (int t = 0; t < S::KH * S::KW; ++t)
        wt[t] = __ldg(reinterpret_cast<const float4*>(wk + t * S::C + c));
#pragma unroll
      for (int ky = 0; ky < S::KH; ++ky) {
        const int iy = oy * S::S - S::PT + ky;
#pragma unroll
        for (int kx = 0; kx < S::KW; ++kx) {
          const int ix = ox * S::S - S::PL + kx;
          if (iy >= 0 && iy < S::H && ix >= 0 && ix < S::W) {
            const float4 w4 = wt[ky * S::KW + kx];
            const float4 v = *reinterpret_cast<const float4*>(src + (iy * S::W + ix) * S::AS_IN + c);
            acc.x = add(acc.x, mul(v.x, w4.x)); acc.y = add(acc.y, mul(v.y, w4.y));
            acc.z = add(acc.z, mul(v.z, w4.z)); acc.w = add(acc.w, mul(v.w, w4.w));
          }
        }
      }
      float* d = at<float>(x.dst, (long long)img * S::OUT_IMG) + p * S::C + c;
      *reinterpret_cast<float4*>(d) = make_float4(
          finish<S::ACT, S::MODE, S::POST>(acc.x, ps, po, c),
          finish<S::ACT, S::MODE, S::POST>(acc.y, ps, po, c + 1),
          finish<S::ACT, S::MODE, S::POST>(acc.z, ps, po, c + 2),
          finish<S::ACT, S::MODE, S::POST>(acc.w, ps, po, c + 3));
    }
  }
};

// C: IN_OFF, IN_IMG, OUT_OFF, OUT_IMG, NSTAGE, STAGE_BYTES, ACT_FLOATS, the
//    weight stream and the generated body(TcChainCtx&)
template <class C>
struct TcChain {
  static constexpr int SMEM = 1024 + C::NSTAGE * C::STAGE_BYTES + 4 * C::ACT_FLOATS + 256;
  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena, int n) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<u64>(smem_raw) + 1023) & ~(u64)1023);
    TcChainCtx x;
    x.ring = base;
    x.act = reinterpret_cast<float*>(base + C::NSTAGE * C::STAGE_BYTES);
    u64* bars = reinterpret_cast<u64*>(base + C::NSTAGE * C::STAGE_BYTES + 4 * C::ACT_FLOATS);
    x.full = bars;
    x.dready = bars + C::NSTAGE;
    u32* tmem_slot = reinterpret_cast<u32*>(bars + C::NSTAGE + 1);
    if (blockDim.x != 256) __trap();
    if (threadIdx.x == 0) {
      for (int s = 0; s < C::NSTAGE; ++s) mbar_init(&x.full[s], 1);
      mbar_init(x.dready, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if ((threadIdx.x >> 5) == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    x.tmem = *tmem_slot;
    x.pool = pool;
    x.full_ph = 0;
    x.dready_ph = 0;
    x.next_blk = 0;
    const long long img0 = 2ll * blockIdx.x;
    x.nimg = n - img0 >= 2 ? 2 : (int)(n - img0);
    x.src = at<float>(arena, C::IN_OFF + img0 * C::IN_IMG);
    x.dst = at<float>(arena, C::OUT_OFF + img0 * C::OUT_IMG);
    tcc_issue<C>(x, 0);                              // the first layer's weights
    C::body(x);
    tc_fence_before();
    __syncthreads();
    if ((threadIdx.x >> 5) == 1) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(x.tmem), "r"(512));
    }
  }
};

}  // namespace nnb
