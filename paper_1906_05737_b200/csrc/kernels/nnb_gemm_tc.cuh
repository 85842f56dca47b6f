// nnb_gemm_tc.cuh -- tcgen05 (5th-gen tensor core) GEMM for Dense and 1x1
// convolutions, FP32-accurate through the 3xTF32 split.
//
//   C[m, j] = sum_k A[m, k] * B[k, j]            A: activations  [M, K] row-major
//                                                B: weights, stored transposed
//                                                   [Npad, Kpad] (K-major)
// FP32 parity (rtol 1e-4 / atol 1e-5, BASELINE.json north_star) with TF32
// inputs: every operand is split a = hi + lo with hi = a with the 13 low
// mantissa bits cleared (exactly representable in TF32) and lo = a - hi
// (exact in FP32), and the product is a_hi*b_hi + a_hi*b_lo + a_lo*b_hi
// accumulated in FP32 in tensor memory -- the dropped a_lo*b_lo term and the
// TF32 rounding of lo are below 2^-21 relative.  Weights are split once at
// compile() time (B_hi, B_lo in the device pool); activations are split in
// shared memory by two converter warps while the tensor core works on the
// previous stage.
//
// Warp roles (384 threads, one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer: A tile [128 x 32] and B_hi/B_lo tiles [BN x 32],
//               128B-swizzled, into an NS-stage ring (mbarrier full/empty)
//   warp 1      TMEM allocator + single-thread MMA issuer:
//               tcgen05.mma.cta_group::1.kind::tf32, M=128, N=BN, K=8
//   warps 2-3   converter: A -> (A_hi in place, A_lo) in the same swizzled
//               layout (elementwise, so the layout is preserved)
//   warps 4-11  epilogue: warp w reads TMEM lanes 32*(w%4).. (the hardware's
//               lane-quarter rule) and half of the tile's columns;
//               tcgen05.ld 32 lanes x 16 columns, bias, activation,
//               post-affine, residual, float4 stores.  The accumulator is
//               double-buffered in TMEM so the epilogue of tile t overlaps the
//               MMAs of tile t+1.
#pragma once
#include "nnb_common.cuh"

namespace nnb {

struct __align__(64) TmaDesc { unsigned long long opaque[16]; };

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

__device__ __forceinline__ void tma_load_4d(void* dst, const TmaDesc* map, u64* bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<u64>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// K-major operand, 128-byte swizzle, rows of 128 B, 8-row atoms 1024 B apart.
__device__ __forceinline__ u64 sw128_desc(u32 saddr) {
  return (u64)((saddr >> 4) & 0x3FFF) | ((u64)1 << 16) | ((u64)(1024 >> 4) << 32) |
         ((u64)1 << 46) | ((u64)2 << 61);
}

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

// C: K, N, NPAD (multiple of BN), BN (32..256, multiple of 16), NS (stages),
//    ROWS (GEMM rows per image), IN/OUT offsets, B_OFF (bias), epilogue fields.
template <class C>
struct GemmTc {
  static constexpr int BM = 128, BK = 32;
  static constexpr int A_BYTES = BM * BK * 4;            // 16 KiB
  static constexpr int B_BYTES = C::BN * BK * 4;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int KB = (C::K + BK - 1) / BK;
  static constexpr int NTN = C::NPAD / C::BN;
  // One accumulator buffer = main (a_hi*b_hi) + correction (a_hi*b_lo + a_lo*b_hi)
  // columns.  Tensor-core accumulation truncates once per MMA instruction, so the
  // error grows with the number of accumulate steps into a large running sum;
  // keeping the two small correction products out of the main sum cuts the
  // truncations on it by 3x, and the two are added in FP32 (round-to-nearest)
  // in the epilogue.
  static constexpr int ACC_COLS = 2 * C::BN;              // fp32 columns per buffer
  static constexpr int TMEM_COLS = 2 * ACC_COLS <= 32 ? 32 : 2 * ACC_COLS <= 64 ? 64
                                 : 2 * ACC_COLS <= 128 ? 128 : 2 * ACC_COLS <= 256 ? 256 : 512;
  static constexpr u32 IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((u32)(C::BN >> 3) << 17) |
                               ((u32)(BM >> 4) << 24);
  static constexpr int SMEM = C::NS * STAGE + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int EPI_WARPS = 8, EPI_THREADS = 32 * EPI_WARPS;
  static constexpr int THREADS = 128 + EPI_THREADS;
  static constexpr int EPI_COLS = C::BN >= 32 ? C::BN / 2 : 16;  // columns per epilogue warp
  static constexpr int CHUNK_KB = 8;                 // k-blocks (K = 256) per TMEM chunk
  static constexpr int NCHUNK = (KB + CHUNK_KB - 1) / CHUNK_KB;
  static_assert(C::BN % 16 == 0 && C::BN >= 16 && C::BN <= 128, "UMMA N / TMEM budget");
  // spatial (implicit-GEMM convolution) tiling: 8 x 16 output pixels per tile
  static constexpr int TH = 8, TW = 16;
  static constexpr int TX = C::CONV ? (C::WO + TW - 1) / TW : 1;
  static constexpr int TPI = C::CONV ? ((C::HO + TH - 1) / TH) * TX : 1;
  static constexpr int CB = C::CONV ? C::CI / BK : 1;       // channel blocks per tap
  static_assert(!C::CONV || C::CI % BK == 0, "conv tiles need CI % 32 == 0");
  static_assert(STAGE % 1024 == 0, "stage alignment");

  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena, int n,
                             const TmaDesc* tmA, const TmaDesc* tmB, const TmaDesc* tmBlo) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<u64>(smem_raw) + 1023) & ~(u64)1023);
    u64* bars = reinterpret_cast<u64*>(smem + C::NS * STAGE);
    u64* full = bars;                 // [NS]  TMA landed
    u64* lo_ready = bars + C::NS;     // [NS]  A split done (64 converter arrivals)
    u64* empty = bars + 2 * C::NS;    // [NS]  MMA finished reading the stage
    u64* tfull = bars + 3 * C::NS;    // [2]   accumulator ready
    u64* tempty = tfull + 2;          // [2]   accumulator drained (128 arrivals)
    u32* tmem_slot = reinterpret_cast<u32*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long rows = (long long)n * C::ROWS;
    const int mtiles = C::CONV ? n * TPI : (int)((rows + BM - 1) / BM);
    const int tiles = mtiles * NTN;

    if (threadIdx.x == 0) {
      for (int s = 0; s < C::NS; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&lo_ready[s], 64);
        mbar_init(&empty[s], 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(&tfull[a], 1);
        mbar_init(&tempty[a], EPI_THREADS);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const u32 tmem = *tmem_slot;

    if (warp == 0) {
      // ---------------- TMA producer ----------------
      if (lane == 0) {
        int s = 0;
        u32 ph = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
          const int mb = t / NTN, nb = t % NTN;
          for (int kb = 0; kb < KB; ++kb) {
            mbar_wait(&empty[s], ph ^ 1);
            unsigned char* st = smem + s * STAGE;
            mbar_expect_tx(&full[s], A_BYTES + 2 * B_BYTES);
            if (C::CONV) {
              // tap (ky, kx) and channel block cb of an 8x16 output-pixel tile;
              // out-of-image coordinates are zero-filled = 'same' padding
              const int img = mb / TPI, tt = mb % TPI;
              const int tap = kb / CB, cb = kb % CB;
              tma_load_4d(st, tmA, &full[s], cb * BK, (tt % TX) * TW + tap % C::KW - C::PL,
                          (tt / TX) * TH + tap / C::KW - C::PT, img);
            } else {
              tma_load_2d(st, tmA, &full[s], kb * BK, mb * BM);
            }
            tma_load_2d(st + 2 * A_BYTES, tmB, &full[s], kb * BK, nb * C::BN);
            tma_load_2d(st + 2 * A_BYTES + B_BYTES, tmBlo, &full[s], kb * BK, nb * C::BN);
            if (++s == C::NS) { s = 0; ph ^= 1; }
          }
        }
      }
    } else if (warp == 1) {
      // ---------------- MMA issuer ----------------
      // K is consumed in chunks of CHUNK_KB k-blocks; every chunk starts a fresh
      // (main, correction) accumulator pair in the next TMEM buffer and is
      // reduced in FP32 by the epilogue warps (split-K inside the CTA).
      int s = 0, acc = 0;
      u32 ph = 0, aph = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        for (int kb = 0; kb < KB; ++kb) {
          const int kc = kb % CHUNK_KB;
          if (kc == 0) {
            mbar_wait(&tempty[acc], aph ^ 1);
            tc_fence_after();
          }
          const u32 d = tmem + acc * ACC_COLS;
          mbar_wait(&lo_ready[s], ph);
          tc_fence_after();
          if (lane == 0) {
            const u32 base = smem_u32(smem + s * STAGE);
            const u32 a_hi = base, a_lo = base + A_BYTES;
            const u32 b_hi = base + 2 * A_BYTES, b_lo = b_hi + B_BYTES;
#pragma unroll
            for (int k = 0; k < BK / 8; ++k) {
              const u32 o = k * 32;   // 8 tf32 = 32 bytes along the swizzled row
              const u32 accum = (kc | k) != 0;
              mma_tf32(d, sw128_desc(a_hi + o), sw128_desc(b_hi + o), IDESC, accum);
              mma_tf32(d + C::BN, sw128_desc(a_hi + o), sw128_desc(b_lo + o), IDESC, accum);
              mma_tf32(d + C::BN, sw128_desc(a_lo + o), sw128_desc(b_hi + o), IDESC, 1);
            }
            mma_commit(&empty[s]);
            if (kc == CHUNK_KB - 1 || kb == KB - 1) mma_commit(&tfull[acc]);
          }
          __syncwarp();
          if (++s == C::NS) { s = 0; ph ^= 1; }
          if (kc == CHUNK_KB - 1 || kb == KB - 1) {
            if (++acc == 2) { acc = 0; aph ^= 1; }
          }
        }
      }
    } else if (warp < 4) {
      // ---------------- converter: A -> (hi, lo) ----------------
      const int ct = threadIdx.x - 64;   // 0..63
      int s = 0;
      u32 ph = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[s], ph);
          float4* a = reinterpret_cast<float4*>(smem + s * STAGE);
          float4* lo = reinterpret_cast<float4*>(smem + s * STAGE + A_BYTES);
#pragma unroll 4
          for (int i = ct; i < A_BYTES / 16; i += 64) {
            float4 v = a[i], h, l;
            h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u); l.x = v.x - h.x;
            h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u); l.y = v.y - h.y;
            h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u); l.z = v.z - h.z;
            h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u); l.w = v.w - h.w;
            a[i] = h;
            lo[i] = l;
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(&lo_ready[s]);
          if (++s == C::NS) { s = 0; ph ^= 1; }
        }
      }
    } else {
      // ---------------- epilogue ----------------
      const int q = warp & 3;                    // TMEM lane quarter of this warp
      const int r = q * 32 + lane;               // row within the tile
      const int cbeg = ((warp - 4) >> 2) * EPI_COLS;
      const float* bias = at<float>(pool, C::B_OFF);
      const float* ps = at<float>(pool, C::PS_OFF);
      const float* po = at<float>(pool, C::PO_OFF);
      float* out = at<float>(arena, C::OUT_OFF);
      int acc = 0;
      u32 aph = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int mb = t / NTN, nb = t % NTN;
        // FP32 (round-to-nearest) reduction of the per-chunk tensor-core sums
        float run[EPI_COLS];
#pragma unroll
        for (int i = 0; i < EPI_COLS; ++i) run[i] = 0.f;
        for (int ch = 0; ch < NCHUNK; ++ch) {
          mbar_wait(&tfull[acc], aph);
          tc_fence_after();
#pragma unroll
          for (int g = 0; g < EPI_COLS / 16; ++g) {
            if (cbeg + g * 16 < C::BN) {             // warp-uniform
              float v[16], cr[16];
              const u32 ta = tmem + ((u32)(q * 32) << 16) + acc * ACC_COLS + cbeg + g * 16;
              tmem_ld16(ta, v);
              tmem_ld16(ta + C::BN, cr);
#pragma unroll
              for (int i = 0; i < 16; ++i) run[g * 16 + i] += v[i] + cr[i];
            }
          }
          tc_fence_before();
          mbar_arrive(&tempty[acc]);
          if (++acc == 2) { acc = 0; aph ^= 1; }
        }
        // output position of this thread's row
        long long obase;            // element offset of the row's first channel
        bool live;
        if (C::CONV) {
          const int img = mb / TPI, tt = mb % TPI;
          const int oy = (tt / TX) * TH + r / TW, ox = (tt % TX) * TW + r % TW;
          live = img < n && oy < C::HO && ox < C::WO;
          obase = (long long)img * (C::OUT_IMG / 4) + ((long long)oy * C::WO + ox) * C::N;
          if (C::POOL) {      // pooled row index of the 2x2 window this lane leads
            const int py = (tt / TX) * (TH / 2) + (r / TW) / 2, px = (tt % TX) * (TW / 2) + (r % TW) / 2;
            live = img < n && py < C::PHO && px < C::PWO && (lane & 17) == 0;
            obase = (long long)img * (C::OUT_IMG / 4) + ((long long)py * C::PWO + px) * C::N;
          }
        } else {
          const long long m = (long long)mb * BM + r;
          live = m < rows;
          obase = m * C::N;
        }
        float* dst = out + obase;
        const float* res = at<float>(arena, C::RES_OFF) + obase;
#pragma unroll
        for (int g = 0; g < EPI_COLS / 16; ++g) {
          const int col0 = nb * C::BN + cbeg + g * 16;
          if (cbeg + g * 16 >= C::BN || col0 >= C::N) continue;   // warp-uniform
          float* v = run + g * 16;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int col = col0 + i < C::N ? col0 + i : C::N - 1;
            float y = v[i] + __ldg(bias + col);
            y = finish<C::ACT, C::MODE, C::POST>(y, ps, po, col);
            if (C::RES && live) y = add(y, __ldg(res + col));
            if (C::POOL) {     // lanes w, w^1 (same image row), w^16 (next row)
              y = fmaxf(y, __shfl_xor_sync(0xffffffffu, y, 1));
              y = fmaxf(y, __shfl_xor_sync(0xffffffffu, y, 16));
            }
            v[i] = y;
          }
          if (live) {
            if (C::N % 16 == 0) {
#pragma unroll
              for (int i = 0; i < 16; i += 4)
                *reinterpret_cast<float4*>(dst + col0 + i) =
                    make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (col0 + i < C::N) dst[col0 + i] = v[i];
            }
          }
        }
      }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(TMEM_COLS));
    }
  }
};

}  // namespace nnb
