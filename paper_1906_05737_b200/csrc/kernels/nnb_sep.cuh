// nnb_sep.cuh -- depthwise conv fused with a narrow pointwise conv (the
// depthwise-separable block of cfg2/cfg3 whose 1x1 conv has <= 32 output
// channels): one launch instead of two, and the depthwise tensor never
// reaches memory.
//
// Reference semantics: pkg/src/nnjit/interpreter.py:65-73 (depthwise: bias,
// then every tap (ky, kx) of the zero-padded input, channel-wise) followed by
// :52-62 (the 1x1 conv as a per-pixel dot over the channels).  At these
// widths both layers are a few FLOPs per byte: the fused kernel's floor is the
// depthwise input in + the pointwise output out, and its other limit is the
// instruction stream.
//   * a tile is TH output rows x the full output width of one image; its
//     (TH-1)*S+KH input rows are one contiguous run of global memory, copied
//     by an NS-stage cp.async ring (16-byte LDGSTS, coalesced) into a band
//     whose halo columns are zero and whose out-of-image rows are zeroed, so
//     every tap is accumulated branch-free exactly as the interpreter does
//     over its zero-padded input; pixels sit at an odd 16-byte stride
//     (conflict-free float4 reads);
//   * persistent CTAs walk tiles blockIdx.x + i*gridDim.x, NS-1 in flight;
//   * one thread per output pixel: depthwise taps in (ky, kx) order with
//     __fmul_rn/__fadd_rn, weights and bias as immediates (Cfg::dww/dwb) --
//     bit-identical to the interpreter's depthwise -- then the depthwise
//     epilogue, then the pointwise dot with its weights as FFMA immediates
//     (Cfg::dotr, bias first, k ascending: RowsNarrow's order with one K
//     slice), its epilogue and residual;
//   * the tile's outputs (contiguous rows) are staged in shared memory as
//     16-byte rows and written back as coalesced float4 stores (storing each
//     pixel's CO floats straight from registers was 5-10% slower).
//   * SP = 2 (wide layers, whose band leaves room for only a few CTAs per SM):
//     two threads per pixel in neighbouring WARPS -- each runs the depthwise
//     taps of half the channels, the halves meet in a shared-memory exchange
//     row, and each forms half of the pointwise outputs -- so the same band
//     feeds twice the warps (cfg3's 32-channel blocks ran 8 warps per SM).
// Measured alternatives (cfg3 @256, dw 64x64x8 + pw 16): a band version with
// per-tap bounds checks and weights loaded from shared memory spent 700
// instructions per pixel (36.9 us, 64% issue-busy); a register version with
// PX pixels per thread and channel-vector loads straight from global memory
// (uncoalesced: a lane per pixel group) ran at 60 us.
#pragma once
#include "nnb_common.cuh"
#include "nnb_rows.cuh"

namespace nnb {

template <class C>
struct SepNarrow {
  static constexpr int H = C::H, W = C::W, CI = C::CI, S = C::S, KH = C::KH, KW = C::KW;
  static constexpr int HO = C::HO, WO = C::WO, CO = C::CO, TH = C::TH, NS = C::NS, NT = C::NT;
  static constexpr int CP = ((CI + 4) / 4) % 2 ? CI + 4 : CI + 8;   // odd 16-byte pixel stride
  static constexpr int RI = (TH - 1) * S + KH;                      // band rows per tile
  static constexpr int WB = (WO - 1) * S + KW;                      // band columns (with halo)
  static constexpr int TPI = (HO + TH - 1) / TH;                    // tiles per image
  static constexpr int PXT = TH * WO;                               // output pixels per tile
  static constexpr int CQ = CI / 4;
  static constexpr int BAND = RI * WB * CP;                         // floats per stage
  static constexpr int SP = C::SP;                                  // threads per pixel
  static constexpr int CQH = CQ / SP, COH = CO / SP;                // quads / outputs per thread
  static_assert(CI % 4 == 0 && CI <= 128 && CO <= 128 && SP * PXT <= NT && NT % (32 * SP) == 0 &&
                NT <= 1024 && (SP == 1 || (SP == 2 && CQ % 2 == 0 && CO % 8 == 0)),
                "depthwise + narrow pointwise");
  // staging row stride: 16-byte rows at an odd 16-byte stride (conflict-free
  // float4 writes) when CO % 4 == 0, else an odd float stride
  static constexpr int RS = CO % 4 ? (CO | 1) : (((CO + 4) / 4) % 2 ? CO + 4 : CO + 8);
  struct Smem {
    float a[NS][BAND];
    // output staging; with SP = 2 first the exchange rows of the depthwise
    // outputs (one padded row per pixel), read back before any output lands
    float o[PXT * (SP == 2 && CP > RS ? CP : RS)];
  };

  __device__ static void load_tile(Smem& sm, int stage, const float* in, i64 tile) {
    const i64 img = tile / TPI;
    const int oy0 = (int)(tile - img * TPI) * TH;
    const int iy_lo = oy0 * S - C::PT;
    const int r0 = iy_lo > 0 ? iy_lo : 0, r1 = iy_lo + RI < H ? iy_lo + RI : H;
    float* band = &sm.a[stage][0];
    // out-of-image rows of this band read as zeros (interior columns; the
    // halo columns are zero from the start)
    if (iy_lo < 0 || iy_lo + RI > H) {
      for (int e = threadIdx.x; e < RI * W * CQ; e += NT) {
        const int p = e / CQ, q = e - p * CQ;
        const int rr = p / W, x = p - rr * W;
        const int iy = iy_lo + rr;
        if (iy < 0 || iy >= H)
          *reinterpret_cast<float4*>(band + (rr * WB + C::PL + x) * CP + 4 * q) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    if (r1 <= r0) return;
    // interior: in-image rows r0..r1-1, one contiguous run of global memory
    // (16-byte chunks; the remap to the padded layout is per chunk)
    const float* src = in + (img * H + r0) * (i64)(W * CI);
    const unsigned base = (unsigned)__cvta_generic_to_shared(band);
    const int cnt = (r1 - r0) * W * CQ;
#pragma unroll 4
    for (int e = threadIdx.x; e < cnt; e += NT) {
      const int p = e / CQ, q = e - p * CQ;          // p: pixel over the rows r0..
      const int rr = p / W, x = p - rr * W;
      cp_async16(base + (unsigned)((((r0 - iy_lo + rr) * WB + C::PL + x) * CP + 4 * q) * 4),
                 src + (i64)e * 4);
    }
  }

  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena, int n,
                             Smem& sm) {
    const i64 ntiles = (i64)n * TPI;
    const float* in = at<float>(arena, C::IN_OFF);
    float* out = at<float>(arena, C::OUT_OFF);
    const int t = threadIdx.x;
    // zero every band once: halo columns stay zero for the whole launch
    for (int e = t; e < NS * BAND / 4; e += NT)
      reinterpret_cast<float4*>(&sm.a[0][0])[e] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
#pragma unroll
    for (int s = 0; s < NS - 1; ++s) {
      const i64 tile = blockIdx.x + (i64)s * gridDim.x;
      if (tile < ntiles) load_tile(sm, s, in, tile);
      cp_async_commit();
    }
    const float* dps = at<float>(pool, C::DW_PS_OFF);
    const float* dpo = at<float>(pool, C::DW_PO_OFF);
    const float* ps = at<float>(pool, C::PS_OFF);
    const float* po = at<float>(pool, C::PO_OFF);
    // SP = 2: warps 2g and 2g + 1 own the same 32 pixels, half the channels each
    const int h = SP == 2 ? (t >> 5) & 1 : 0;
    const int pix = SP == 2 ? ((t >> 6) << 5) + (t & 31) : t;
    const int py = pix / WO, ox = pix - py * WO;
    const int boff = (py * S * WB + ox * S) * CP;       // the pixel's first tap in the band

    int stage = 0;
    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      {
        const i64 ahead = tile + (i64)(NS - 1) * gridDim.x;
        if (ahead < ntiles) load_tile(sm, (stage + NS - 1) % NS, in, ahead);
        cp_async_commit();
      }
      cp_async_wait<NS - 1>();
      __syncthreads();

      const i64 img = tile / TPI;
      const int oy0 = (int)(tile - img * TPI) * TH;
      const int live = (HO - oy0 < TH ? HO - oy0 : TH) * WO;
      const i64 p0 = img * (HO * WO) + (i64)oy0 * WO;      // first output pixel of the tile
      float a[CI];
      if (pix < live) {
        const float* band = &sm.a[stage][boff];
#pragma unroll
        for (int qq = 0; qq < CQH; ++qq) {
          // (the two halves branch on the warp's parity so that every weight
          // index below is a compile-time constant)
          float4 r4;
#pragma unroll
          for (int hh = 0; hh < SP; ++hh) {
            if (hh != h) continue;
            const int q = hh * CQH + qq;
            float4 acc = make_float4(C::dwb(4 * q), C::dwb(4 * q + 1), C::dwb(4 * q + 2), C::dwb(4 * q + 3));
#pragma unroll
            for (int ky = 0; ky < KH; ++ky)
#pragma unroll
              for (int kx = 0; kx < KW; ++kx) {
                const float4 x = *reinterpret_cast<const float4*>(band + (ky * WB + kx) * CP + 4 * q);
                const int wi = (ky * KW + kx) * CI + 4 * q;
                if (C::DW_FMA) {       // one rounding per tap (within the FP32 gate)
                  acc.x = fmaf(x.x, C::dww(wi + 0), acc.x);
                  acc.y = fmaf(x.y, C::dww(wi + 1), acc.y);
                  acc.z = fmaf(x.z, C::dww(wi + 2), acc.z);
                  acc.w = fmaf(x.w, C::dww(wi + 3), acc.w);
                } else {               // the interpreter's mul-then-add: bit-exact
                  acc.x = add(acc.x, mul(x.x, C::dww(wi + 0)));
                  acc.y = add(acc.y, mul(x.y, C::dww(wi + 1)));
                  acc.z = add(acc.z, mul(x.z, C::dww(wi + 2)));
                  acc.w = add(acc.w, mul(x.w, C::dww(wi + 3)));
                }
              }
            r4.x = finish<C::DW_ACT, C::MODE, C::DW_POST>(acc.x, dps, dpo, 4 * q + 0);
            r4.y = finish<C::DW_ACT, C::MODE, C::DW_POST>(acc.y, dps, dpo, 4 * q + 1);
            r4.z = finish<C::DW_ACT, C::MODE, C::DW_POST>(acc.z, dps, dpo, 4 * q + 2);
            r4.w = finish<C::DW_ACT, C::MODE, C::DW_POST>(acc.w, dps, dpo, 4 * q + 3);
            if (SP == 2) {
              *reinterpret_cast<float4*>(&sm.o[pix * CP + 4 * q]) = r4;
            } else {
              a[4 * q + 0] = r4.x; a[4 * q + 1] = r4.y; a[4 * q + 2] = r4.z; a[4 * q + 3] = r4.w;
            }
          }
        }
      }
      if (SP == 2) __syncthreads();          // both halves of every pixel's depthwise row stored
      if (SP == 2) {
        if (pix < live) {
#pragma unroll
          for (int q = 0; q < CQ; ++q) {
            const float4 v = *reinterpret_cast<const float4*>(&sm.o[pix * CP + 4 * q]);
            a[4 * q + 0] = v.x; a[4 * q + 1] = v.y; a[4 * q + 2] = v.z; a[4 * q + 3] = v.w;
          }
        }
        __syncthreads();                     // the exchange rows are read: outputs may land
      }
      if (pix < live) {
        float acc[COH];
        bool upper = false;
        if constexpr (SP == 2) {
          if (h == 1) {          // the upper half of the output channels
            upper = true;
#pragma unroll
            for (int j = 0; j < COH; ++j) acc[j] = C::bias(COH + j);
            C::dotr1(a, acc);
          }
        }
        if (!upper) {
#pragma unroll
          for (int j = 0; j < COH; ++j) acc[j] = C::bias(j);
          C::dotr(a, acc);
        }
        const int j0 = h * COH;
#pragma unroll
        for (int j = 0; j < COH; ++j) acc[j] = finish<C::ACT, C::MODE, C::POST>(acc[j], ps, po, j0 + j);
        if (C::RES) {
          const float* res = at<float>(arena, C::RES_OFF) + (p0 + pix) * CO + j0;
#pragma unroll
          for (int j = 0; j < COH; ++j) acc[j] = add(acc[j], __ldg(res + j));
        }
        if (COH % 4 == 0) {
#pragma unroll
          for (int j = 0; j < COH; j += 4)
            *reinterpret_cast<float4*>(&sm.o[pix * RS + j0 + j]) =
                make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < COH; ++j) sm.o[pix * RS + j0 + j] = acc[j];
        }
      }
      __syncthreads();
      // the tile's outputs are one contiguous run of live*CO floats
      float* dst = out + p0 * CO;
      if (CO % 4 == 0) {
        constexpr int C4 = CO / 4;
        for (int e = t; e < live * C4; e += NT) {
          const int r = e / C4, c = e - r * C4;
          reinterpret_cast<float4*>(dst)[e] = *reinterpret_cast<const float4*>(&sm.o[r * RS + 4 * c]);
        }
      } else {
        for (int e = t; e < live * CO; e += NT) {
          const int r = e / CO;
          dst[e] = sm.o[r * RS + e - r * CO];
        }
      }
      __syncthreads();             // the next iteration refills this stage and the staging
      stage = (stage + 1) % NS;
    }
    cp_async_wait<0>();
  }
};

}  // namespace nnb
