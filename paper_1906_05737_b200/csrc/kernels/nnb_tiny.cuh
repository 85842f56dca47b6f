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
// interpreter's op-by-op rounding (bit-exact).  Weights are read through L1
// (__ldg; they are small by construction: the selection bounds them).
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
  __device__ static __forceinline__ void run(const float* __restrict__ pool, float* a) {
    const float* in = a + S::IN / 4;
    float* out = a + S::OUT / 4;
    const float* wk = at<float>(pool, S::W_OFF);
    const float* bs = at<float>(pool, S::B_OFF);
    const float* ps = at<float>(pool, S::PS_OFF);
    const float* po = at<float>(pool, S::PO_OFF);
    constexpr int NP = S::POOL ? 4 : 1;
    constexpr int ITEMS = (S::POOL ? S::PHO * S::PWO : S::HO * S::WO) * CQ;
    for (int it = threadIdx.x; it < ITEMS; it += blockDim.x) {
      const int q = it % CQ, pix = it / CQ, co = 4 * q;
      const int py = S::POOL ? pix / S::PWO : pix / S::WO, px = S::POOL ? pix % S::PWO : pix % S::WO;
      float bias[4], m[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        bias[j] = co + j < S::CO ? __ldg(bs + co + j) : 0.f;
        m[j] = 0.f;
      }
      // the pixels of a pool window one after the other (rolled: NVRTC time);
      // each is finished (activation / post-BN) before the max, as unfused
#pragma unroll 1
      for (int p = 0; p < NP; ++p) {
        const int oy = S::POOL ? 2 * py + p / 2 : py, ox = S::POOL ? 2 * px + p % 2 : px;
        float acc[4] = {bias[0], bias[1], bias[2], bias[3]};
        for (int ky = 0; ky < S::KH; ++ky) {
          const int iy = oy * S::S - S::PT + ky;
          if (iy < 0 || iy >= S::H) continue;
          for (int kx = 0; kx < S::KW; ++kx) {
            const int ix = ox * S::S - S::PL + kx;
            if (ix < 0 || ix >= S::W) continue;
            const float* xin = in + (iy * S::W + ix) * S::CI;
            const float* wr = wk + ((ky * S::KW + kx) * S::CI) * S::CO + co;
#pragma unroll 4
            for (int ci = 0; ci < S::CI; ++ci) {
              const float x = xin[ci];
#pragma unroll
              for (int j = 0; j < 4; ++j)
                if (co + j < S::CO) acc[j] = fmaf(x, __ldg(wr + ci * S::CO + j), acc[j]);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float y = finish<S::ACT, S::MODE, S::POST>(acc[j], ps, po, co + j < S::CO ? co + j : 0);
          m[j] = p == 0 ? y : fmaxf(m[j], y);
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (co + j >= S::CO) continue;
        const int o = pix * S::CO + co + j;
        out[o] = S::RES >= 0 ? add(m[j], a[S::RES / 4 + o]) : m[j];
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
  __device__ static __forceinline__ void run(const float* __restrict__ pool, float* a) {
    const float* in = a + S::IN / 4;
    float* out = a + S::OUT / 4;
    const float* wk = at<float>(pool, S::W_OFF);
    const float* bs = at<float>(pool, S::B_OFF);
    const float* ps = at<float>(pool, S::PS_OFF);
    const float* po = at<float>(pool, S::PO_OFF);
    for (int it = threadIdx.x; it < S::HO * S::WO * S::C; it += blockDim.x) {
      const int c = it % S::C, pix = it / S::C, oy = pix / S::WO, ox = pix % S::WO;
      float acc = __ldg(bs + c);
      for (int ky = 0; ky < S::KH; ++ky) {
        const int iy = oy * S::S - S::PT + ky;
        if (iy < 0 || iy >= S::H) continue;
        for (int kx = 0; kx < S::KW; ++kx) {
          const int ix = ox * S::S - S::PL + kx;
          if (ix < 0 || ix >= S::W) continue;
          acc = add(acc, mul(in[(iy * S::W + ix) * S::C + c], __ldg(wk + (ky * S::KW + kx) * S::C + c)));
        }
      }
      out[it] = finish<S::ACT, S::MODE, S::POST>(acc, ps, po, c);
    }
  }
};

// Dense K -> CO (+ residual, + softmax over the row when SOFTMAX, CO <= 32).
// A warp per output: lanes split K, partial sums added in a fixed tree order.
// S: K, CO, IN, OUT, RES, W_OFF (K, CO), B_OFF, ACT, MODE, POST, PS_OFF,
//    PO_OFF, SOFTMAX, SMEXP
template <class S>
struct TinyDense {
  __device__ static __forceinline__ void run(const float* __restrict__ pool, float* a) {
    const float* in = a + S::IN / 4;
    float* out = a + S::OUT / 4;
    const float* wk = at<float>(pool, S::W_OFF);
    const float* bs = at<float>(pool, S::B_OFF);
    const float* ps = at<float>(pool, S::PS_OFF);
    const float* po = at<float>(pool, S::PO_OFF);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int j = warp; j < S::CO; j += nw) {
      float s = 0.f;
#pragma unroll 4
      for (int k = lane; k < S::K; k += 32) s = fmaf(in[k], __ldg(wk + k * S::CO + j), s);
      s = warp_sum(s);
      if (lane == 0) {
        float y = finish<S::ACT, S::MODE, S::POST>(add(__ldg(bs + j), s), ps, po, j);
        if (S::RES >= 0) y = add(y, a[S::RES / 4 + j]);
        out[j] = y;
      }
    }
    if constexpr (S::SOFTMAX) {
      __syncthreads();
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
  __device__ static __forceinline__ void run(const float* __restrict__, float* a) {
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
  __device__ static __forceinline__ void run(const float* __restrict__ pool, float* a) {
    const float* sc = at<float>(pool, S::SC_OFF);
    const float* of = at<float>(pool, S::OF_OFF);
    for (int i = threadIdx.x; i < S::N; i += blockDim.x) {
      float y = a[S::IN0 / 4 + i];
      if (S::NIN > 1) y = add(y, a[S::IN1 / 4 + i]);
      if (S::NIN > 2) y = add(y, a[S::IN2 / 4 + i]);
      if (S::NIN > 3) y = add(y, a[S::IN3 / 4 + i]);
      if (S::AFFINE) y = add(mul(y, __ldg(sc + i % S::C)), __ldg(of + i % S::C));
      a[S::OUT / 4 + i] = activate<S::ACT, S::MODE>(y);
    }
  }
};

// rank-1 softmax over L values by one warp per row pass
// S: L, IN, OUT, SMEXP
template <class S>
struct TinySoftmax {
  __device__ static __forceinline__ void run(const float* __restrict__, float* a) {
    if ((threadIdx.x >> 5) != 0) return;
    const int lane = threadIdx.x & 31;
    static_assert(S::L <= 32, "tiny softmax: one warp");
    const float v = softmax_warp_row<S::SMEXP>(lane < S::L ? a[S::IN / 4 + lane] : 0.f, lane < S::L);
    if (lane < S::L) a[S::OUT / 4 + lane] = v;
  }
};

// C: ARENA_FLOATS and the generated load(arena, img, a) / body(pool, a) /
//    store(arena, img, a)
template <class C>
struct TinyNet {
  struct Smem { float a[C::ARENA_FLOATS]; };
  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena, int n,
                             Smem& sm) {
    for (int img = blockIdx.x; img < n; img += gridDim.x) {
      C::load(arena, img, sm.a);
      __syncthreads();
      C::body(pool, sm.a);
      __syncthreads();
      C::store(arena, img, sm.a);
      __syncthreads();
    }
  }
};

}  // namespace nnb
