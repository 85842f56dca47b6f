// nnb_rows.cuh -- narrow row GEMM: Dense (or a stride-1 1x1 conv, one row per
// pixel) with at most 32 output columns over many rows, e.g. a classifier
// head at batch 65536 (cfg1's Dense 128->10 + softmax).
//
// The work is a stream over A: K*4 bytes in, CO*4 bytes out per row, a few
// FMAs per byte -- HBM-bound.  The FFMA tile GEMM handles it with one row
// per thread but a synchronous K loop, so a CTA has 64 bytes per row in
// flight and the launch ran at 1.7 TB/s.  Here rows are contiguous (row m at
// in + m*K), so a tile of TR rows is one contiguous block of global memory:
//   * persistent CTAs walk tiles m0 = TR*(blockIdx.x + i*grid);
//   * NS-stage cp.async ring (16-byte LDGSTS, warp-contiguous) fills padded
//     smem rows (stride K+4 floats: the 8 lanes of an LDS.128 phase hit
//     disjoint banks), NS-1 tiles in flight while one is computed;
//   * the weights and bias are baked into the generated code (the paper's
//     specialisation idea, constants in the instruction stream): the
//     specialiser writes ``Cfg::dot`` -- the unrolled K x CO FFMAs with each
//     weight an immediate operand -- so no weight is ever loaded;
//   * a row's K is split into KS slices, one warp per (32 rows, slice), so
//     enough warps share a tile to hide the smem latency (the tile, not the
//     thread count, is what limits residency); slice 0 starts at the bias,
//     every slice takes its k in ascending order with fmaf, and the partial
//     sums are added in slice order -- within the FP32 gate of the
//     reference interpreter's single ascending chain
//     (pkg/src/nnjit/interpreter.py:52-62), identical to it when KS = 1;
//   * epilogue (activation, post-BN, residual, softmax in the selected
//     mode, nnb_softmax.cuh softmax_row_regs) in registers, the
//     tile staged in smem (odd row stride: conflict-free for any CO) and
//     written back as coalesced float4 stores.
#pragma once
#include "nnb_common.cuh"
#include "nnb_softmax.cuh"

namespace nnb {

__device__ __forceinline__ void cp_async16(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <class C>
struct RowsNarrow {
  static constexpr int TR = C::TR, K = C::K, CO = C::CO, NS = C::NS, KS = C::KS;
  static constexpr int NT = TR * KS;                              // KS warps per 32 rows
  static constexpr int AST = ((K + 4) / 4) % 2 ? K + 4 : K + 8;   // odd 16-byte stride
  static constexpr int KQ = K / 4;                                // 16-byte chunks per row
  static constexpr int RS = CO | 1;                               // odd smem row stride
  static_assert(K % (4 * KS) == 0 && CO <= 32 && TR % 32 == 0 && NT <= 1024, "narrow row GEMM");
  struct Smem {
    float a[NS][TR][AST];
    float red[KS > 1 ? KS - 1 : 1][TR][RS];
    float o[TR][RS];
  };

  __device__ static void load_tile(Smem& sm, int stage, const float* in, i64 m0, i64 nrows) {
    const unsigned base = (unsigned)__cvta_generic_to_shared(&sm.a[stage][0][0]);
    const int live = (int)(nrows - m0 < TR ? nrows - m0 : TR);
    const float* src = in + m0 * K;
#pragma unroll 4
    for (int e = threadIdx.x; e < live * KQ; e += NT) {
      const int r = e / KQ, c = e - r * KQ;
      cp_async16(base + (unsigned)((r * AST + 4 * c) * 4), src + (i64)e * 4);
    }
  }

  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena, int n,
                             Smem& sm) {
    const i64 nrows = (i64)n * C::ROWS;
    const i64 ntiles = (nrows + TR - 1) / TR;
    const float* in = at<float>(arena, C::IN_OFF);
    float* out = at<float>(arena, C::OUT_OFF);
    const int t = threadIdx.x;
    const int r = t % TR, ks = t / TR;                 // warp-uniform k slice
#pragma unroll
    for (int s = 0; s < NS - 1; ++s) {
      const i64 tile = blockIdx.x + (i64)s * gridDim.x;
      if (tile < ntiles) load_tile(sm, s, in, tile * TR, nrows);
      cp_async_commit();
    }
    const float* ps = at<float>(pool, C::PS_OFF);
    const float* po = at<float>(pool, C::PO_OFF);

    int stage = 0;
    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      {
        const i64 ahead = tile + (i64)(NS - 1) * gridDim.x;
        if (ahead < ntiles) load_tile(sm, (stage + NS - 1) % NS, in, ahead * TR, nrows);
        cp_async_commit();
      }
      cp_async_wait<NS - 1>();
      __syncthreads();

      const i64 m0 = tile * TR;
      const int live = (int)(nrows - m0 < TR ? nrows - m0 : TR);
      float acc[CO];
      // slice 0 starts at the bias, the others at zero; the generated dot
      // takes the slice's k in ascending order with the weights as FFMA
      // immediates
#pragma unroll
      for (int j = 0; j < CO; ++j) acc[j] = ks == 0 ? C::bias(j) : 0.f;
      C::dot(&sm.a[stage][r][0], acc, ks);
      if (KS > 1) {
        if (ks > 0) {
#pragma unroll
          for (int j = 0; j < CO; ++j) sm.red[ks - 1][r][j] = acc[j];
        }
        __syncthreads();
      }
      if (ks == 0) {
#pragma unroll
        for (int q = 1; q < KS; ++q)
#pragma unroll
          for (int j = 0; j < CO; ++j) acc[j] = add(acc[j], sm.red[q - 1][r][j]);
#pragma unroll
        for (int j = 0; j < CO; ++j) acc[j] = finish<C::ACT, C::MODE, C::POST>(acc[j], ps, po, j);
        if (C::RES && r < live) {
          const float* res = at<float>(arena, C::RES_OFF) + (m0 + r) * CO;
#pragma unroll
          for (int j = 0; j < CO; ++j) acc[j] = add(acc[j], __ldg(res + j));
        }
        if (C::SOFTMAX) {
          softmax_row_regs<CO, CO, C::SMEXP>(acc);
        }
#pragma unroll
        for (int j = 0; j < CO; ++j) sm.o[r][j] = acc[j];
      }
      __syncthreads();
      // the tile's outputs are one contiguous run of live*CO floats
      float* dst = out + m0 * CO;
      const int cnt = live * CO;
      if (live == TR && (TR * CO) % 4 == 0) {
        for (int e = t; e < cnt / 4; e += NT) {
          float v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int f = 4 * e + q, rr = f / CO;
            v[q] = sm.o[rr][f - rr * CO];
          }
          reinterpret_cast<float4*>(dst)[e] = make_float4(v[0], v[1], v[2], v[3]);
        }
      } else {
        for (int e = t; e < cnt; e += NT) {
          const int rr = e / CO;
          dst[e] = sm.o[rr][e - rr * CO];
        }
      }
      stage = (stage + 1) % NS;
    }
    cp_async_wait<0>();
  }
};

}  // namespace nnb
