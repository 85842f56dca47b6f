// nnb_tiny.cuh -- the whole network in ONE kernel for small batches of a
// small net (kernels.py Specializer._tiny): one CTA per image runs every
// launch unit in order over a shared-memory copy of that image's arena --
// the same per-image layout and byte offsets the buffer planner gave the
// device arena -- so a batch-1 inference is one launch whose layers are
// separated by __syncthreads instead of kernel boundaries (the paper's own
// model: one compiled function per network, here one CTA per image).
//
// Reference semantics per step as in the per-layer kernels: convolution and
// Dense accumulate bias first, taps / inputs in the interpreter's order
// (pkg/src/nnjit/interpreter.py:45-62) with fmaf (inside the FP32 gate like
// the FFMA GEMM); pooling, elementwise and depthwise steps use the
// interpreter's op-by-op rounding (bit-exact).  The weights are staged into
// shared memory once per CTA (the selection bounds their size).
#pragma once
#include "nnb_common.cuh"
#include "nnb_softmax.cuh"

namespace nnb {

template <int BYTES>
__device__ __forceinline__ void tiny_copy(float* __restrict__ dst, const float* __restrict__ src) {
  if constexpr (BYTES % 16 == 0) {
    const float4* s = reinterpret_cast<const float4*>(src);
    float4* d = reinterpret_cast<float4*>(dst);
    for (int i = threadIdx.x; i < BYTES / 16; i += blockDim.x) d[i] = s[i];
  } else {
    for (int i = threadIdx.x; i < BYTES / 4; i += blockDim.x) dst[i] = src[i];
  }
}

// Conv2D (NHWC in shared memory), optional fused 2x2/2 max-pool, residual.
// S: H, W, CI, HO, WO, CO, KH, KW, S, PT, PL, POOL, PHO, PWO, IN, OUT, RES
//    (byte offsets in the image arena; RES < 0: none), W_OFF (kh,kw,ci,co),
//    B_OFF, ACT, MODE, POST, PS_OFF, PO_OFF
template <class S>
struct TinyConv {
  static constexpr int CQ = (S::CO + 3) / 4;
  __device__ static __forceinline__ void run(const float* __restrict__ pool, const float* w, float* a) {
    const float* in = a + S::IN / 4;
    float* out = a + S::OUT / 4;
    const float* wk = at<float>(w, S::W_OFF);
    const float* bs = at<float>(w, S::B_OFF);
    const float* ps = at<float>(pool, S::PS_OFF);
    const float* po = at<float>(pool, S::PO_OFF);
    constexpr int NP = S::POOL ? 4 : 1;
    constexpr int ITEMS = (S::POOL ? S::PHO * S::PWO : S::HO * S::WO) * CQ;
    static_assert(S::CO % 4 == 0, "tiny conv: channel quads");
    for (int it = threadIdx.x; it < ITEMS; it += blockDim.x) {
      const int q = it % CQ, pix = it / CQ, co = 4 * q;
      const int py = S::POOL ? pix / S::PWO : pix / S::WO, px = S::POOL ? pix % S::PWO : pix % S::WO;
      // a thread owns a channel quad of NP pixels (a whole pool window): each
      // tap's weight quad is one float4 load feeding 4*NP FFMAs
      float acc[NP][4];
      {
        const float4 b4 = *reinterpret_cast<const float4*>(bs + co);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          acc[p][0] = b4.x; acc[p][1] = b4.y; acc[p][2] = b4.z; acc[p][3] = b4.w;
        }
      }
      for (int ky = 0; ky < S::KH; ++ky) {
        for (int kx = 0; kx < S::KW; ++kx) {
          int off[NP];
          bool ok[NP];
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            const int oy = S::POOL ? 2 * py + p / 2 : py, ox = S::POOL ? 2 * px + p % 2 : px;
            const int iy = oy * S::S - S::PT + ky, ix = ox * S::S - S::PL + kx;
            ok[p] = iy >= 0 && iy < S::H && ix >= 0 && ix < S::W;
            off[p] = ok[p] ? (iy * S::W + ix) * S::CI : 0;
          }
          const float* wr = wk + ((ky * S::KW + kx) * S::CI) * S::CO + co;
#pragma unroll 2
          for (int ci = 0; ci < S::CI; ++ci) {
            const float4 w4 = *reinterpret_cast<const float4*>(wr + ci * S::CO);
#pragma unroll
            for (int p = 0; p < NP; ++p) {
              if (ok[p]) {
                const float x = in[off[p] + ci];
                acc[p][0] = fmaf(x, w4.x, acc[p][0]); acc[p][1] = fmaf(x, w4.y, acc[p][1]);
                acc[p][2] = fmaf(x, w4.z, acc[p][2]); acc[p][3] = fmaf(x, w4.w, acc[p][3]);
              }
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float y = finish<S::ACT, S::MODE, S::POST>(acc[0][j], ps, po, co + j);
#pragma unroll
        for (int p = 1; p < NP; ++p) y = fmaxf(y, finish<S::ACT, S::MODE, S::POST>(acc[p][j], ps, po, co + j));
        const int o = pix * S::CO + co + j;
        out[o] = S::RES >= 0 ? add(y, a[S::RES / 4 + o]) : y;
      }
    }
  }
};

// DepthwiseConv2D: bias, then the taps in (ky, kx) order with __fmul_rn /
// __fadd_rn, out-of-image taps skipped -- the interpreter's result bit for bit.
// S: H, W, C, HO, WO, KH, KW, S, PT, PL, IN, OUT, W_OFF (kh,kw,c), B_OFF, ACT,
//    MODE, POST, PS_OFF, PO_OFF
template <class S>
struct TinyDw {
  __device__ static __forceinline__ void run(const float* __restrict__ pool, const float* w, float* a) {
    const float* in = a + S::IN / 4;
    float* out = a + S::OUT / 4;
    const float* wk = at<float>(w, S::W_OFF);
    const float* bs = at<float>(w, S::B_OFF);
    const float* ps = at<float>(pool, S::PS_OFF);
    const float* po = at<float>(pool, S::PO_OFF);
    for (int it = threadIdx.x; it < S::HO * S::WO * S::C; it += blockDim.x) {
      const int c = it % S::C, pix = it / S::C, oy = pix / S::WO, ox = pix % S::WO;
      float acc = bs[c];
      for (int ky = 0; ky < S::KH; ++ky) {
        const int iy = oy * S::S - S::PT + ky;
        if (iy < 0 || iy >= S::H) continue;
        for (int kx = 0; kx < S::KW; ++kx) {
          const int ix = ox * S::S - S::PL + kx;
          if (ix < 0 || ix >= S::W) continue;
          acc = add(acc, mul(in[(iy * S::W + ix) * S::C + c], wk[(ky * S::KW + kx) * S::C + c]));
        }
      }
      out[it] = finish<S::ACT, S::MODE, S::POST>(acc, ps, po, c);
    }
  }
};

// Dense K -> CO (+ residual, + softmax over the row when SOFTMAX, CO <= 32).
// Lanes take 32 consecutive outputs (coalesced weight rows), the 8 warps
// split K into slices whose partial sums are added in slice order after the
// bias.
// S: K, CO, IN, OUT, RES, W_OFF (K, CO), B_OFF, ACT, MODE, POST, PS_OFF,
//    PO_OFF, SOFTMAX, SMEXP
template <class S>
struct TinyDense {
  __device__ static __forceinline__ void run(const float* __restrict__ pool, const float* w, float* a) {
    __shared__ float part[8][33];
    const float* in = a + S::IN / 4;
    float* out = a + S::OUT / 4;
    const float* wk = at<float>(w, S::W_OFF);
    const float* bs = at<float>(w, S::B_OFF);
    const float* ps = at<float>(pool, S::PS_OFF);
    const float* po = at<float>(pool, S::PO_OFF);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int KS = S::K >= 128 ? 8 : S::K >= 32 ? 4 : 1;        // K slices
    constexpr int KL = (S::K + KS - 1) / KS;
    for (int j0 = 0; j0 < S::CO; j0 += 32) {
      const int j = j0 + lane;
      if (warp < KS) {
        float s = 0.f;
        const int k0 = warp * KL, k1 = k0 + KL < S::K ? k0 + KL : S::K;
        if (j < S::CO) {
#pragma unroll 4
          for (int k = k0; k < k1; ++k) s = fmaf(in[k], wk[k * S::CO + j], s);
        }
        part[warp][lane] = s;
      }
      __syncthreads();
      if (warp == 0 && j < S::CO) {
        float y = bs[j];
#pragma unroll
        for (int sl = 0; sl < KS; ++sl) y = add(y, part[sl][lane]);
        y = finish<S::ACT, S::MODE, S::POST>(y, ps, po, j);
        if (S::RES >= 0) y = add(y, a[S::RES / 4 + j]);
        out[j] = y;
      }
      __syncthreads();
    }
    if constexpr (S::SOFTMAX) {
      if (warp == 0) {
        const float v = softmax_warp_row<S::SMEXP>(lane < S::CO ? out[lane] : 0.f, lane < S::CO);
        if (lane < S::CO) out[lane] = v;
      }
    }
  }
};

// Pool (max: taps in order with fmaxf; avg: in-bounds sum / in-bound count).
// S: H, W, C, HO, WO, PH, PW, S, PT, PL, AVG, IN, OUT
template <class S>
struct TinyPool {
  __device__ static __forceinline__ void run(const float* __restrict__, const float*, float* a) {
    const float* in = a + S::IN / 4;
    float* out = a + S::OUT / 4;
    for (int it = threadIdx.x; it < S::HO * S::WO * S::C; it += blockDim.x) {
      const int c = it % S::C, pix = it / S::C, oy = pix / S::WO, ox = pix % S::WO;
      float acc = S::AVG ? 0.f : -__int_as_float(0x7f800000);
      int cnt = 0;
      for (int ky = 0; ky < S::PH; ++ky) {
        const int iy = oy * S::S - S::PT + ky;
        if (iy < 0 || iy >= S::H) continue;
        for (int kx = 0; kx < S::PW; ++kx) {
          const int ix = ox * S::S - S::PL + kx;
          if (ix < 0 || ix >= S::W) continue;
          const float x = in[(iy * S::W + ix) * S::C + c];
          acc = S::AVG ? add(acc, x) : fmaxf(acc, x);
          ++cnt;
        }
      }
      out[it] = S::AVG ? dvd(acc, (float)cnt) : acc;
    }
  }
};

// Elementwise: y = x0 (+ x1 + ...), then scale/offset (BatchNorm), then the
// activation -- the interpreter's op order.
// S: N (elements), C (channels), NIN, IN0..IN3, OUT, AFFINE, SC_OFF, OF_OFF, ACT, MODE
template <class S>
struct TinyElem {
  __device__ static __forceinline__ void run(const float* __restrict__ pool, const float* w, float* a) {
    const float* sc = at<float>(w, S::SC_OFF);
    const float* of = at<float>(w, S::OF_OFF);
    for (int i = threadIdx.x; i < S::N; i += blockDim.x) {
      float y = a[S::IN0 / 4 + i];
      if (S::NIN > 1) y = add(y, a[S::IN1 / 4 + i]);
      if (S::NIN > 2) y = add(y, a[S::IN2 / 4 + i]);
      if (S::NIN > 3) y = add(y, a[S::IN3 / 4 + i]);
      if (S::AFFINE) y = add(mul(y, sc[i % S::C]), of[i % S::C]);
      a[S::OUT / 4 + i] = activate<S::ACT, S::MODE>(y);
    }
  }
};

// rank-1 softmax over L values by one warp per row pass
// S: L, IN, OUT, SMEXP
template <class S>
struct TinySoftmax {
  __device__ static __forceinline__ void run(const float* __restrict__, const float*, float* a) {
    if ((threadIdx.x >> 5) != 0) return;
    const int lane = threadIdx.x & 31;
    static_assert(S::L <= 32, "tiny softmax: one warp");
    const float v = softmax_warp_row<S::SMEXP>(lane < S::L ? a[S::IN / 4 + lane] : 0.f, lane < S::L);
    if (lane < S::L) a[S::OUT / 4 + lane] = v;
  }
};

// C: ARENA_FLOATS and the generated load(arena, img, a) / body(pool, a) /
//    store(arena, img, a)
// The kernel's weights and biases are the first W_BYTES of the pool (the
// TinyNet is specialised before any other unit) and are copied into shared
// memory once per CTA: every layer then reads them at shared-memory latency
// (from global memory each (tap, channel) row is a fresh L2 round trip -- all
// items read the same rows at the same time, so L1 never hits: 94 us for cfg0
// at batch 1 before).  Post-BN vectors stay in global memory (finish()).
template <class C>
struct TinyNet {
  struct Smem { float w[C::W_FLOATS]; float a[C::ARENA_FLOATS]; };
  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena, int n,
                             Smem& sm) {
    if (blockIdx.x < n) tiny_copy<C::W_FLOATS * 4>(sm.w, pool);
    for (int img = blockIdx.x; img < n; img += gridDim.x) {
      C::load(arena, img, sm.a);
      __syncthreads();
      C::body(pool, sm.w, sm.a);
      __syncthreads();
      C::store(arena, img, sm.a);
      __syncthreads();
    }
  }
};

}  // namespace nnb
