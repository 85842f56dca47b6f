// nnb_small.cuh -- memory-bound launch units (one thread per output vector).
//
// Every kernel here is HBM-bound at the BASELINE shapes, so
// the design rules are: one pass over the data, float4 along the innermost
// (channel) axis whenever C % 4 == 0, consecutive threads on consecutive
// addresses, and no shared memory.  Arithmetic is written with explicit *_rn
// intrinsics in the reference's operation order, which makes depthwise,
// pooling, BatchNorm, Add, upsample and concat bit-identical to the
// interpreter (pkg/src/nnjit/interpreter.py:65-99, 121-122, 166-172).
#pragma once
#include "nnb_common.cuh"
#include "nnb_softmax.cuh"

namespace nnb {

template <int V> struct Vec;
template <> struct Vec<1> { typedef float T; };
template <> struct Vec<4> { typedef float4 T; };

__device__ __forceinline__ float lane(const float& v, int) { return v; }
__device__ __forceinline__ float lane(const float4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}
__device__ __forceinline__ void set_lane(float& v, int, float x) { v = x; }
__device__ __forceinline__ void set_lane(float4& v, int i, float x) {
  if (i == 0) v.x = x; else if (i == 1) v.y = x; else if (i == 2) v.z = x; else v.w = x;
}
template <int V> __device__ __forceinline__ typename Vec<V>::T vzero();
template <> __device__ __forceinline__ float vzero<1>() { return 0.f; }
template <> __device__ __forceinline__ float4 vzero<4>() { return make_float4(0.f, 0.f, 0.f, 0.f); }

__device__ __forceinline__ i64 gtid() { return nnb_bid() * nnb_bdim() + threadIdx.x; }

// ---------------------------------------------------------------------------
// Dense / 1x1 convolution for a handful of rows (batch-1 latency path): MB
// rows and 32 output columns per block, KS warps split K, partial sums
// reduced in a fixed order.  Row m is pixel m % ROWS of image m / ROWS
// (ROWS = 1 for Dense).
template <class C>
struct DenseSmallM {
  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena, int n) {
#if NNB_MEGA
    extern __shared__ __align__(16) unsigned char nnb_dyn_smem[];
    float (*red)[C::MB][32] = reinterpret_cast<float (*)[C::MB][32]>(nnb_dyn_smem);
#else
    __shared__ float red[C::KS][C::MB][32];
#endif
    const int lane_ = threadIdx.x & 31, ks = threadIdx.x >> 5;
    constexpr int NJ = (C::CO + 31) / 32;
    const int jb = (int)(nnb_bid() % NJ);
    const int row0 = (int)(nnb_bid() / NJ) * C::MB;
    const int j = jb * 32 + lane_;
    const float* x = at<float>(arena, C::IN_OFF);
    const float* w = at<float>(pool, C::W_OFF);
    const i64 nrows = (i64)n * C::ROWS;
    auto in_row = [](i64 m) { return (m / C::ROWS) * (C::IN_IMG / 4) + (m % C::ROWS) * C::K; };
    auto out_row = [](i64 m) { return (m / C::ROWS) * (C::OUT_IMG / 4) + (m % C::ROWS) * C::CO; };
    constexpr int KPER = (C::K + C::KS - 1) / C::KS;
    const int k0 = ks * KPER;
    const int k1 = k0 + KPER < C::K ? k0 + KPER : C::K;
    float acc[C::MB];
    const float* xr[C::MB];
#pragma unroll
    for (int r = 0; r < C::MB; ++r) {
      acc[r] = 0.f;
      xr[r] = x + (row0 + r < nrows ? in_row(row0 + r) : 0);
    }
    // float4 row loads when every warp's k range is 4-aligned (same fmaf
    // order as the scalar loop, so results are identical)
    constexpr bool V4 = C::K % (4 * C::KS) == 0 && C::IN_IMG % 16 == 0;
    if (j < C::CO && V4) {
#pragma unroll 2
      for (int k = k0; k < k1; k += 4) {
        float wv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) wv[q] = __ldg(w + (i64)(k + q) * C::CO + j);
#pragma unroll
        for (int r = 0; r < C::MB; ++r)
          if (row0 + r < nrows) {
            const float4 xv = lda(reinterpret_cast<const float4*>(xr[r] + k));
            acc[r] = fmaf(xv.x, wv[0], acc[r]);
            acc[r] = fmaf(xv.y, wv[1], acc[r]);
            acc[r] = fmaf(xv.z, wv[2], acc[r]);
            acc[r] = fmaf(xv.w, wv[3], acc[r]);
          }
      }
    } else if (j < C::CO) {
#pragma unroll 4
      for (int k = k0; k < k1; ++k) {
        float wv = __ldg(w + (i64)k * C::CO + j);
#pragma unroll
        for (int r = 0; r < C::MB; ++r)
          if (row0 + r < nrows) acc[r] = fmaf(lda(xr[r] + k), wv, acc[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < C::MB; ++r) red[ks][r][lane_] = acc[r];
    nnb_sync();
    if (ks != 0) return;                       // warp 0 finishes all rows
    const bool live = j < C::CO;
    const float* ps = at<float>(pool, C::PS_OFF);
    const float* po = at<float>(pool, C::PO_OFF);
    float* out = at<float>(arena, C::OUT_OFF);
    const float b = live ? __ldg(at<float>(pool, C::B_OFF) + j) : 0.f;
#pragma unroll
    for (int r = 0; r < C::MB; ++r) {
      if (row0 + r >= nrows) break;
      float s = b;
      for (int q = 0; q < C::KS; ++q) s = s + red[q][r][lane_];
      float v = finish<C::ACT, C::MODE, C::POST>(s, ps, po, live ? j : 0);
      if (C::RES && live)
        v = add(v, lda(at<float>(arena, C::RES_OFF) + out_row(row0 + r) + j));
      if (C::SOFTMAX) v = softmax_warp_row<C::SMEXP>(v, live);   // CO <= 32
      if (live) out[out_row(row0 + r) + j] = v;
    }
  }
};

// ---------------------------------------------------------------------------
// DepthwiseConv2D: acc = bias; taps (ky, kx) in order; mul then add.
// A thread owns PX horizontally adjacent output pixels of one channel vector:
// the (PX-1)*S + KW input columns of each kernel row are loaded once into
// registers and shared by the PX outputs (PX=4, 3x3 stride 1: 18 loads for 4
// pixels instead of 36).  Out-of-image taps are skipped, not zero-multiplied,
// as in the reference.  IDX32: the launch's index space fits in 32 bits.
template <class C>
struct Depthwise {
  static constexpr int V = C::VEC, PX = C::PX;
  typedef typename Vec<V>::T T;
  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena, int n) {
    constexpr int CG = C::C / V, XG = (C::WO + PX - 1) / PX;
    constexpr int NCOL = (PX - 1) * C::S + C::KW;
    const i64 t = gtid();
    if (t >= (i64)n * C::HO * XG * CG) return;
    int cg, xg, oy;
    i64 img;
    if (C::IDX32) {
      unsigned q = (unsigned)t;
      cg = (int)(q % CG); q /= CG;
      xg = (int)(q % XG); q /= XG;
      oy = (int)(q % C::HO); img = q / C::HO;
    } else {
      i64 q = t;
      cg = (int)(q % CG); q /= CG;
      xg = (int)(q % XG); q /= XG;
      oy = (int)(q % C::HO); img = q / C::HO;
    }
    const T* in = at<T>(arena, C::IN_OFF + img * C::IN_IMG);
    const T* wk = at<T>(pool, C::W_OFF);
    const T b = at<T>(pool, C::B_OFF)[cg];
    T acc[PX];
#pragma unroll
    for (int p = 0; p < PX; ++p) acc[p] = b;
    const int ox0 = xg * PX;
    const int iy0 = oy * C::S - C::PT, ix0 = ox0 * C::S - C::PL;
#pragma unroll
    for (int ky = 0; ky < C::KH; ++ky) {
      const int iy = iy0 + ky;
      if (iy < 0 || iy >= C::H) continue;
      const T* row = in + (i64)iy * C::W * CG + cg;
      T xv[NCOL];
#pragma unroll
      for (int j = 0; j < NCOL; ++j) {
        const int ix = ix0 + j;
        xv[j] = (ix >= 0 && ix < C::W) ? lda(row + ix * CG) : vzero<V>();
      }
#pragma unroll
      for (int kx = 0; kx < C::KW; ++kx) {
        const T wv = __ldg(wk + (ky * C::KW + kx) * CG + cg);
#pragma unroll
        for (int p = 0; p < PX; ++p) {
          const int ix = ix0 + p * C::S + kx;
          if (ix < 0 || ix >= C::W) continue;
#pragma unroll
          for (int l = 0; l < V; ++l)
            set_lane(acc[p], l, add(lane(acc[p], l), mul(lane(xv[p * C::S + kx], l), lane(wv, l))));
        }
      }
    }
    const float* ps = at<float>(pool, C::PS_OFF);
    const float* po = at<float>(pool, C::PO_OFF);
    T* out = at<T>(arena, C::OUT_OFF + img * C::OUT_IMG) + ((i64)oy * C::WO + ox0) * CG + cg;
#pragma unroll
    for (int p = 0; p < PX; ++p) {
      if (ox0 + p >= C::WO) break;
#pragma unroll
      for (int l = 0; l < V; ++l)
        set_lane(acc[p], l, finish<C::ACT, C::MODE, C::POST>(lane(acc[p], l), ps, po, cg * V + l));
      out[p * CG] = acc[p];
    }
  }
};

// ---------------------------------------------------------------------------
// Max / average pooling over in-bounds taps (avg divides by their count,
// pkg/src/nnjit/interpreter.py:85-95).  Global average pooling is the
// whole-image window.
template <class C>
struct Pool {
  static constexpr int V = C::VEC;
  typedef typename Vec<V>::T T;
  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena, int n) {
    constexpr int CG = C::C / V;
    const i64 t = gtid();
    if (t >= (i64)n * C::HO * C::WO * CG) return;
    const int cg = (int)(t % CG);
    const i64 p = t / CG;
    const int ox = (int)(p % C::WO);
    const int oy = (int)((p / C::WO) % C::HO);
    const i64 img = p / ((i64)C::HO * C::WO);
    const T* in = at<T>(arena, C::IN_OFF + img * C::IN_IMG);
    const int iy0 = oy * C::S - C::PT, ix0 = ox * C::S - C::PL;
    T acc;
    const float ninf = -__int_as_float(0x7f800000);
#pragma unroll
    for (int l = 0; l < V; ++l) set_lane(acc, l, C::AVG ? 0.f : ninf);
    int count = 0;
    for (int ky = 0; ky < C::PH; ++ky) {
      const int iy = iy0 + ky;
      if (iy < 0 || iy >= C::H) continue;
      for (int kx = 0; kx < C::PW; ++kx) {
        const int ix = ix0 + kx;
        if (ix < 0 || ix >= C::W) continue;
        T xv = lda(in + ((i64)iy * C::W + ix) * CG + cg);
        ++count;
#pragma unroll
        for (int l = 0; l < V; ++l)
          set_lane(acc, l, C::AVG ? add(lane(acc, l), lane(xv, l)) : fmaxf(lane(acc, l), lane(xv, l)));
      }
    }
    if (C::AVG) {
      const float cf = (float)count;
#pragma unroll
      for (int l = 0; l < V; ++l) set_lane(acc, l, dvd(lane(acc, l), cf));
    }
    T* out = at<T>(arena, C::OUT_OFF + img * C::OUT_IMG);
    if (C::UPF > 1) {             // fused nearest upsampling of the pooled map
#pragma unroll
      for (int rep = 0; rep < C::UPF * C::UPF; ++rep)
        out[((i64)(oy * C::UPF + rep / C::UPF) * C::WO * C::UPF + ox * C::UPF + rep % C::UPF) * CG + cg] = acc;
      return;
    }
    out[p % ((i64)C::HO * C::WO) * CG + cg] = acc;
  }
};

// ---------------------------------------------------------------------------
// GlobalAveragePooling2D + the narrow Dense consuming it (planner.
// fuse_gap_dense: a classifier / regression head such as cfg2's 128 -> 4),
// one warp per image: lanes own channel quads and sum them over the pixels in
// (y, x) order, divide by the count (the Pool kernel's operations, pkg/src/
// nnjit/interpreter.py:85-95), park the pooled row in shared memory, then
// lane j forms output j = bias, k ascending (interpreter.py:45-50), applies
// the activation / post-BN / softmax and stores it.  One launch instead of two
// that each move a few kilobytes per image.
template <class C>
struct GapDense {
  static constexpr int CQ = C::CH / 4, QPL = (CQ + 31) / 32, WPB = 4;   // quads, quads per lane, warps
  static_assert(C::CH % 4 == 0 && C::CO <= 32, "pooled row in channel quads, one output per lane");
  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena, int n) {
    __shared__ __align__(16) float row[WPB][C::CH];
    const int lane_ = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const i64 img = nnb_bid() * WPB + wp;
    if (img >= n) return;
    const float4* in = at<float4>(arena, C::IN_OFF + img * C::IN_IMG);
    float4 s[QPL];
#pragma unroll
    for (int i = 0; i < QPL; ++i) s[i] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int p = 0; p < C::H * C::W; ++p) {
#pragma unroll
      for (int i = 0; i < QPL; ++i) {
        const int q = lane_ + 32 * i;
        if (q < CQ) {
          const float4 v = lda(in + (i64)p * CQ + q);
          s[i].x = add(s[i].x, v.x); s[i].y = add(s[i].y, v.y);
          s[i].z = add(s[i].z, v.z); s[i].w = add(s[i].w, v.w);
        }
      }
    }
    const float cf = (float)(C::H * C::W);
#pragma unroll
    for (int i = 0; i < QPL; ++i) {
      const int q = lane_ + 32 * i;
      if (q < CQ)
        *reinterpret_cast<float4*>(&row[wp][4 * q]) =
            make_float4(dvd(s[i].x, cf), dvd(s[i].y, cf), dvd(s[i].z, cf), dvd(s[i].w, cf));
    }
    __syncwarp();
    const bool live = lane_ < C::CO;
    const int j = live ? lane_ : 0;
    const float* w = at<float>(pool, C::W_OFF) + j;
    float acc = __ldg(at<float>(pool, C::B_OFF) + j);
#pragma unroll 4
    for (int k = 0; k < C::CH; k += 4) {
      const float4 a = *reinterpret_cast<const float4*>(&row[wp][k]);
      acc = fmaf(a.x, __ldg(w + (i64)k * C::CO), acc);
      acc = fmaf(a.y, __ldg(w + (i64)(k + 1) * C::CO), acc);
      acc = fmaf(a.z, __ldg(w + (i64)(k + 2) * C::CO), acc);
      acc = fmaf(a.w, __ldg(w + (i64)(k + 3) * C::CO), acc);
    }
    float v = finish<C::ACT, C::MODE, C::POST>(acc, at<float>(pool, C::PS_OFF), at<float>(pool, C::PO_OFF), j);
    if (C::SOFTMAX) v = softmax_warp_row<C::SMEXP>(v, live);
    if (live) at<float>(arena, C::OUT_OFF + img * C::OUT_IMG)[j] = v;
  }
};

// ---------------------------------------------------------------------------
// Elementwise: n-ary Add (left to right), BatchNorm affine (x*s + o, two
// roundings), activation -- in the order of emitters.py:115-121.
template <class C>
struct Elementwise {
  static constexpr int V = C::VEC;
  typedef typename Vec<V>::T T;
  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena, int n) {
    const i64 t = gtid();
    constexpr i64 PER = C::ELEMS / V;
    if (t >= (i64)n * PER) return;
    const i64 img = t / PER, e = t % PER;
    T v = at<T>(arena, C::IN0_OFF + img * C::IMG)[e];
    if (C::NIN > 1) { T w = at<T>(arena, C::IN1_OFF + img * C::IMG)[e];
#pragma unroll
      for (int l = 0; l < V; ++l) set_lane(v, l, add(lane(v, l), lane(w, l))); }
    if (C::NIN > 2) { T w = at<T>(arena, C::IN2_OFF + img * C::IMG)[e];
#pragma unroll
      for (int l = 0; l < V; ++l) set_lane(v, l, add(lane(v, l), lane(w, l))); }
    if (C::NIN > 3) { T w = at<T>(arena, C::IN3_OFF + img * C::IMG)[e];
#pragma unroll
      for (int l = 0; l < V; ++l) set_lane(v, l, add(lane(v, l), lane(w, l))); }
    const float* sc = at<float>(pool, C::S_OFF);
    const float* of = at<float>(pool, C::O_OFF);
#pragma unroll
    for (int l = 0; l < V; ++l) {
      float x = lane(v, l);
      if (C::AFFINE) {
        const int ch = (int)((e * V + l) % C::CH);
        x = add(mul(x, __ldg(sc + ch)), __ldg(of + ch));
      }
      set_lane(v, l, activate<C::ACT, C::MODE>(x));
    }
    at<T>(arena, C::OUT_OFF + img * C::IMG)[e] = v;
  }
};

// ---------------------------------------------------------------------------
// Nearest-neighbour upsampling by an integer factor.
template <class C>
struct Upsample {
  static constexpr int V = C::VEC;
  typedef typename Vec<V>::T T;
  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena, int n) {
    constexpr int CG = C::C / V;
    constexpr int HO = C::H * C::F, WO = C::W * C::F;
    const i64 t = gtid();
    if (t >= (i64)n * HO * WO * CG) return;
    const int cg = (int)(t % CG);
    const i64 p = t / CG;
    const int ox = (int)(p % WO), oy = (int)((p / WO) % HO);
    const i64 img = p / ((i64)HO * WO);
    const T* in = at<T>(arena, C::IN_OFF + img * C::IN_IMG);
    at<T>(arena, C::OUT_OFF + img * C::OUT_IMG)[((i64)oy * WO + ox) * CG + cg] =
        in[((i64)(oy / C::F) * C::W + ox / C::F) * CG + cg];
  }
};

// ---------------------------------------------------------------------------
// Channel concatenation of up to four sources (rank-1 concat is P == 1).
template <class C>
struct Concat {
  static constexpr int V = C::VEC;
  typedef typename Vec<V>::T T;
  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena, int n) {
    constexpr int CG = C::CT / V;
    const i64 t = gtid();
    if (t >= (i64)n * C::P * CG) return;
    const int cg = (int)(t % CG);
    const i64 p = t / CG;
    const i64 img = p / C::P, q = p % C::P;
    int c = cg * V;
    T v;
    if (c < C::C0) {
      v = at<T>(arena, C::OFF0 + img * C::C0 * C::P * 4)[(q * C::C0 + c) / V];
    } else if (C::NIN < 3 || c < C::C0 + C::C1) {
      c -= C::C0;
      v = at<T>(arena, C::OFF1 + img * C::C1 * C::P * 4)[(q * C::C1 + c) / V];
    } else if (C::NIN < 4 || c < C::C0 + C::C1 + C::C2) {
      c -= C::C0 + C::C1;
      v = at<T>(arena, C::OFF2 + img * C::C2 * C::P * 4)[(q * C::C2 + c) / V];
    } else {
      c -= C::C0 + C::C1 + C::C2;
      v = at<T>(arena, C::OFF3 + img * C::C3 * C::P * 4)[(q * C::C3 + c) / V];
    }
    at<T>(arena, C::OUT_OFF + img * C::CT * C::P * 4)[p % C::P * CG + cg] = v;
  }
};

// ---------------------------------------------------------------------------
// ZeroPadding2D (and plain copies when all pads are zero).
template <class C>
struct Pad {
  static constexpr int V = C::VEC;
  typedef typename Vec<V>::T T;
  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena, int n) {
    constexpr int CG = C::C / V;
    const i64 t = gtid();
    if (t >= (i64)n * C::HO * C::WO * CG) return;
    const int cg = (int)(t % CG);
    const i64 p = t / CG;
    const int ox = (int)(p % C::WO), oy = (int)((p / C::WO) % C::HO);
    const i64 img = p / ((i64)C::HO * C::WO);
    const int iy = oy - C::PT, ix = ox - C::PL;
    T v = vzero<V>();
    if (iy >= 0 && iy < C::H && ix >= 0 && ix < C::W)
      v = at<T>(arena, C::IN_OFF + img * C::IN_IMG)[((i64)iy * C::W + ix) * CG + cg];
    at<T>(arena, C::OUT_OFF + img * C::OUT_IMG)[((i64)oy * C::WO + ox) * CG + cg] = v;
  }
};

}  // namespace nnb
