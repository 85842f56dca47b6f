// nnb_softmax.cuh -- softmax over the last axis (rank-1 per image, or per
// pixel over channels for a rank-3 tensor).
//
// Three numeric flavours (options.py):
//   exact   : exp(x - max) and the sum in float64, one division, one rounding
//             to float32 -- the interpreter (pkg/src/nnjit/interpreter.py:115-118)
//   precise : float32 Cody-Waite exp, float32 sum, one reciprocal, multiply
//   fast    : float32 Schraudolph exp, same reduction
// precise/fast follow the three passes of the reference emitter
// (pkg/src/nnjit/codegen/emitters.py:489-545): stabilising max, exponentials
// and their sum, then a single reciprocal that scales every element.
#pragma once
#include "nnb_common.cuh"

namespace nnb {

template <int SMEXP>
__device__ __forceinline__ float sm_exp32(float d) {
  return SMEXP == SMEXP_FAST ? exp_fast(d) : exp_precise(d);
}

// Whole row held by one thread in registers (L <= TN).
template <int TN, int L, int SMEXP>
__device__ __forceinline__ void softmax_row_regs(float (&v)[TN]) {
  float m = v[0];
#pragma unroll
  for (int j = 1; j < L; ++j) m = fmaxf(m, v[j]);
  if (SMEXP == SMEXP_EXACT) {
    double e[L];
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < L; ++j) { e[j] = d_exp((double)v[j] - (double)m); s += e[j]; }
#pragma unroll
    for (int j = 0; j < L; ++j) v[j] = (float)(e[j] / s);
  } else {
    float s = 0.0f;
#pragma unroll
    for (int j = 0; j < L; ++j) { v[j] = sm_exp32<SMEXP>(sub(v[j], m)); s = add(s, v[j]); }
    float inv = dvd(1.0f, s);
#pragma unroll
    for (int j = 0; j < L; ++j) v[j] = mul(v[j], inv);
  }
}

// One row spread across a warp, one value per lane (lanes with live == false
// hold padding and do not contribute).
template <int SMEXP>
__device__ __forceinline__ float softmax_warp_row(float v, bool live) {
  const float ninf = -__int_as_float(0x7f800000);
  float m = warp_max(live ? v : ninf);
  if (SMEXP == SMEXP_EXACT) {
    double e = live ? d_exp((double)v - (double)m) : 0.0;
    double s = warp_sum(e);
    return (float)(e / s);
  }
  float e = live ? sm_exp32<SMEXP>(sub(v, m)) : 0.0f;
  float s = warp_sum(e);
  return mul(e, dvd(1.0f, s));
}

// Standalone kernel body.  C: IN_OFF, OUT_OFF, ROWS (rows per image),
// L (row length), SMEXP, PER_THREAD (1: thread per row, 0: warp per row).
template <class C>
struct SoftmaxRows {
  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena, int n) {
    const float* in = at<float>(arena, C::IN_OFF);
    float* out = at<float>(arena, C::OUT_OFF);
    const i64 rows = (i64)n * C::ROWS;
    if (C::PER_THREAD) {
      i64 r = nnb_bid() * nnb_bdim() + threadIdx.x;
      if (r >= rows) return;
      float v[C::L];
#pragma unroll
      for (int j = 0; j < C::L; ++j) v[j] = in[r * C::L + j];
      softmax_row_regs<C::L, C::L, C::SMEXP>(v);
#pragma unroll
      for (int j = 0; j < C::L; ++j) out[r * C::L + j] = v[j];
      return;
    }
    const int lane = threadIdx.x & 31;
    i64 r = (nnb_bid() * nnb_bdim() + threadIdx.x) >> 5;
    if (r >= rows) return;
    const float* x = in + r * C::L;
    float* y = out + r * C::L;
    constexpr int PER = (C::L + 31) / 32;
    float v[PER];
    float m = -__int_as_float(0x7f800000);
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      int j = lane + 32 * t;
      v[t] = j < C::L ? x[j] : -__int_as_float(0x7f800000);
      m = fmaxf(m, v[t]);
    }
    m = warp_max(m);
    if (C::SMEXP == SMEXP_EXACT) {
      double e[PER];
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < PER; ++t) {
        int j = lane + 32 * t;
        e[t] = j < C::L ? d_exp((double)v[t] - (double)m) : 0.0;
        s += e[t];
      }
      s = warp_sum(s);
#pragma unroll
      for (int t = 0; t < PER; ++t) {
        int j = lane + 32 * t;
        if (j < C::L) y[j] = (float)(e[t] / s);
      }
    } else {
      float s = 0.0f;
#pragma unroll
      for (int t = 0; t < PER; ++t) {
        int j = lane + 32 * t;
        v[t] = j < C::L ? sm_exp32<C::SMEXP>(sub(v[t], m)) : 0.0f;
        s = add(s, v[t]);
      }
      s = warp_sum(s);
      float inv = dvd(1.0f, s);
#pragma unroll
      for (int t = 0; t < PER; ++t) {
        int j = lane + 32 * t;
        if (j < C::L) y[j] = mul(v[t], inv);
      }
    }
  }
};

}  // namespace nnb
