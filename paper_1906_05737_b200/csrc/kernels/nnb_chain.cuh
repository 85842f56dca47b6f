// nnb_chain.cuh -- a run of small depthwise / pointwise convolutions (the
// 16x16 / 8x8 / 4x4 tail of a MobileNet-style net, planner.fuse_chain) in one
// launch: one CTA per image keeps every intermediate activation in shared
// memory, so the run costs one HBM read of its input and one write of its
// output instead of a round trip (and a launch) per layer.
//
// Reference semantics per step: depthwise pkg/src/nnjit/interpreter.py:65-73
// (bias, then the taps (ky, kx) of the zero-padded input, channel-wise, each
// product and sum rounded -- here __fmul_rn / __fadd_rn with out-of-image taps
// skipped, bit-identical to the interpreter), pointwise :52-62 (a per-pixel
// dot over the channels, bias first, k ascending -- here with fmaf, inside
// the FP32 gate), global average pool :85-95 (in-order sum, divided by the
// tap count), each followed by the unit's activation / post-BN (finish()).
//
// Shared-memory layout: channel-major, channel stride CS = pixels | 1 (odd),
// so a warp whose lanes read one pixel of 32 channels (the staging transpose)
// and a warp whose lanes read 32 pixels of one channel (depthwise, stores)
// are both conflict-free.  Buffers: X (the staged chain input), A and B (ping-
// pong intermediates).
//   * stage: the HWC input of the image is read with coalesced float4 loads
//     and transposed into X;
//   * depthwise: warp w takes channels w, w + 8, ..., its 9 (KH*KW) weights in
//     registers; lanes walk the output pixels;
//   * pointwise: thread (pixel group, channel group) owns a TP x TC register
//     tile; per k it reads TP activations (warp broadcasts: the 32 lanes span
//     <= 4 pixel groups) and TC weights (two coalesced float4 LDGs, L1-resident
//     after the first image) and issues TP*TC FFMAs;
//   * the last step writes the output to the arena (HWC, coalesced) or, for a
//     closing global average pool, C floats per image.
#pragma once
#include "nnb_common.cuh"

namespace nnb {

__device__ __forceinline__ constexpr int chain_cs(int pixels) { return pixels | 1; }

// HWC image in the arena -> channel-major shared memory
template <int H, int W, int C>
__device__ __forceinline__ void chain_stage(const float* __restrict__ src, float* __restrict__ dst) {
  constexpr int P = H * W, CS = chain_cs(P);
  if constexpr (C % 4 == 0) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    for (int e = threadIdx.x; e < P * C / 4; e += blockDim.x) {
      const float4 v = lda(s4 + e);
      const int p = (4 * e) / C, c = (4 * e) % C;
      dst[c * CS + p] = v.x;
      dst[(c + 1) * CS + p] = v.y;
      dst[(c + 2) * CS + p] = v.z;
      dst[(c + 3) * CS + p] = v.w;
    }
  } else {
    for (int e = threadIdx.x; e < P * C; e += blockDim.x) dst[(e % C) * CS + e / C] = lda(src + e);
  }
}

// S: H, W, C, HO, WO, KH, KW, S, PT, PL, W_OFF (kh, kw, c), B_OFF, ACT, MODE,
//    POST, PS_OFF, PO_OFF
template <class S>
struct ChainDw {
  __device__ static __forceinline__ void run(const float* __restrict__ pool,
                                             const float* __restrict__ in, float* __restrict__ out) {
    constexpr int PO = S::HO * S::WO, CSI = chain_cs(S::H * S::W), CSO = chain_cs(PO);
    constexpr int T = S::KH * S::KW;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const float* wk = at<float>(pool, S::W_OFF);
    const float* bs = at<float>(pool, S::B_OFF);
    const float* ps = at<float>(pool, S::PS_OFF);
    const float* po = at<float>(pool, S::PO_OFF);
    for (int c = warp; c < S::C; c += nw) {
      float w[T];
#pragma unroll
      for (int t = 0; t < T; ++t) w[t] = __ldg(wk + t * S::C + c);
      const float b = __ldg(bs + c);
      const float* ic = in + c * CSI;
#pragma unroll 2
      for (int p = lane; p < PO; p += 32) {
        const int oy = p / S::WO, ox = p - oy * S::WO;
        float acc = b;
#pragma unroll
        for (int ky = 0; ky < S::KH; ++ky) {
          const int iy = oy * S::S - S::PT + ky;
#pragma unroll
          for (int kx = 0; kx < S::KW; ++kx) {
            const int ix = ox * S::S - S::PL + kx;
            if (iy >= 0 && iy < S::H && ix >= 0 && ix < S::W)
              acc = add(acc, mul(ic[iy * S::W + ix], w[ky * S::KW + kx]));
          }
        }
        out[c * CSO + p] = finish<S::ACT, S::MODE, S::POST>(acc, ps, po, c);
      }
    }
  }
};

// S: P (pixels), CI, CO, TP, TC, W_OFF (CI x CO row-major), B_OFF, ACT, MODE,
//    POST, PS_OFF, PO_OFF
template <class S>
struct ChainPw {
  static constexpr int NCG = S::CO / S::TC;                 // channel groups
  static_assert(NCG * (S::P / S::TP) == 256 && S::P % S::TP == 0, "chain pointwise tile");
  static_assert(S::TC == 4 || S::TC == 8, "chain pointwise channel tile");
  __device__ static __forceinline__ void run(const float* __restrict__ pool,
                                             const float* __restrict__ in, float* __restrict__ out) {
    constexpr int CS = chain_cs(S::P);
    const int t = threadIdx.x;
    const int co0 = (t % NCG) * S::TC, p0 = (t / NCG) * S::TP;
    const float* wg = at<float>(pool, S::W_OFF) + co0;
    const float* bs = at<float>(pool, S::B_OFF);
    float acc[S::TP][S::TC];
#pragma unroll
    for (int j = 0; j < S::TC; ++j) {
      const float b = __ldg(bs + co0 + j);
#pragma unroll
      for (int i = 0; i < S::TP; ++i) acc[i][j] = b;
    }
    const float* xin = in + p0;
#pragma unroll 4
    for (int k = 0; k < S::CI; ++k) {
      float w[S::TC];
      const float4 w0 = __ldg(reinterpret_cast<const float4*>(wg + k * S::CO));
      w[0] = w0.x; w[1] = w0.y; w[2] = w0.z; w[3] = w0.w;
      if constexpr (S::TC == 8) {
        const float4 w1 = __ldg(reinterpret_cast<const float4*>(wg + k * S::CO + 4));
        w[4] = w1.x; w[5] = w1.y; w[6] = w1.z; w[7] = w1.w;
      }
      float x[S::TP];
#pragma unroll
      for (int i = 0; i < S::TP; ++i) x[i] = xin[k * CS + i];
#pragma unroll
      for (int i = 0; i < S::TP; ++i)
#pragma unroll
        for (int j = 0; j < S::TC; ++j) acc[i][j] = fmaf(x[i], w[j], acc[i][j]);
    }
    const float* ps = at<float>(pool, S::PS_OFF);
    const float* po = at<float>(pool, S::PO_OFF);
#pragma unroll
    for (int j = 0; j < S::TC; ++j)
#pragma unroll
      for (int i = 0; i < S::TP; ++i)
        out[(co0 + j) * CS + p0 + i] = finish<S::ACT, S::MODE, S::POST>(acc[i][j], ps, po, co0 + j);
  }
};

// the chain's last activation (P pixels x C channels, channel-major) to the
// arena as HWC
template <int P, int C>
__device__ __forceinline__ void chain_store(const float* __restrict__ in, float* __restrict__ dst) {
  constexpr int CS = chain_cs(P);
  for (int e = threadIdx.x; e < P * C; e += blockDim.x) dst[e] = in[(e % C) * CS + e / C];
}

// global average pool closing the chain: C floats per image
template <int P, int C>
__device__ __forceinline__ void chain_gap(const float* __restrict__ in, float* __restrict__ dst) {
  constexpr int CS = chain_cs(P);
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float s = 0.f;
#pragma unroll 4
    for (int p = 0; p < P; ++p) s = add(s, in[c * CS + p]);
    dst[c] = dvd(s, (float)P);
  }
}

// C: IN_OFF, IN_IMG, OUT_OFF, OUT_IMG, X_FLOATS, AB_FLOATS and the generated
//    body(pool, in_img, out_img, x, a, b) running the steps
template <class C>
struct Chain {
  struct Smem {
    float x[C::X_FLOATS];
    float a[C::AB_FLOATS];
    float b[C::AB_FLOATS];
  };
  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena, int n,
                             Smem& sm) {
    for (i64 img = nnb_bid(); img < n; img += gridDim.x) {
      C::body(pool, at<float>(arena, C::IN_OFF + img * C::IN_IMG),
              at<float>(arena, C::OUT_OFF + img * C::OUT_IMG), sm.x, sm.a, sm.b);
      nnb_sync();     // the next image restages X
    }
  }
};

}  // namespace nnb
