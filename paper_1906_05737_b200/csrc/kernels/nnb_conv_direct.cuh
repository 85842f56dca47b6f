// nnb_conv_direct.cuh -- direct FFMA convolution for narrow inputs (CI <= 16,
// CO <= 32): the network stems and the small encoder layers.
//
// At K = KH*KW*CI <= 144 an implicit GEMM spends its time on tile staging and
// index arithmetic, not on FMAs.  Here every thread owns NP output pixels
// and all CO output channels in registers, walks the taps in the interpreter's
// (ky, kx, ci) order (accumulators start at the bias; pkg/src/nnjit/
// interpreter.py:52-62) with float4 loads along the channels when CI % 4 == 0,
// and reads the (kh, kw, ci, co) weights as warp-uniform broadcasts from
// shared memory.  The epilogue fuses activation, post-BN, residual Add and the
// 2x2/2 max-pool (a thread owns a whole pool window when POOL).
#pragma once
#include "nnb_common.cuh"

namespace nnb {

template <class C>
struct ConvDirect {
  // PSPLIT: a 2x2 pool window is shared by two lanes (2l: top row, 2l+1:
  // bottom row), halving the unrolled FFMAs per thread (NVRTC time) at the
  // same instruction mix; the window max crosses lanes with one shuffle
  // PSPLIT = 4: one pixel per lane, a window over lanes 4l..4l+3 (max by two
  // shuffles) -- a quarter of the unrolled body again.
  static constexpr int NSPLIT = C::POOL ? (C::PSPLIT == 4 ? 4 : C::PSPLIT ? 2 : 1) : 1;
  static constexpr bool PSPLIT = NSPLIT > 1;
  static constexpr int PY = C::POOL && NSPLIT == 1 ? 2 : 1;
  static constexpr int PX = C::POOL ? (NSPLIT == 4 ? 1 : 2) : C::PXT;
  static constexpr int NP = PY * PX;
  static constexpr int CV = (C::CI % 4 == 0) ? 4 : 1;        // channels per load
  static constexpr int WN = C::KH * C::KW * C::CI * C::CO;   // weight floats
  static constexpr int CELLS_Y = C::POOL ? C::PHO : C::HO;
  static constexpr int CELLS_X = C::POOL ? C::PWO : (C::WO + PX - 1) / PX;

  struct Smem { alignas(16) float w[C::WIMM ? 4 : WN]; float b[C::CO]; };

  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena, int n,
                             Smem& sm) {
    if (!C::WIMM) {
      const float* wg = at<float>(pool, C::W_OFF);
      for (int i = threadIdx.x; i < WN; i += nnb_bdim()) sm.w[i] = __ldg(wg + i);
      for (int i = threadIdx.x; i < C::CO; i += nnb_bdim()) sm.b[i] = __ldg(at<float>(pool, C::B_OFF) + i);
      nnb_sync();
    }

    // Pixel ownership.  POOL: a thread owns one 2x2 window (consecutive lanes,
    // consecutive windows).  Otherwise the PX pixels of a thread are 32 apart
    // in the flattened (image, row, column) order and consecutive lanes take
    // consecutive pixels, so every warp load covers 32 neighbouring pixels
    // (PX adjacent pixels per thread made lanes PX*S pixels apart: 4-8x the
    // cache lines per load).
    const i64 cell = nnb_bid() * nnb_bdim() + threadIdx.x;
    int oyp[NP], oxp[NP];
    const float* inp[NP];
    i64 imgp[NP];
    bool live[NP];
    if (C::POOL) {
      const int half = (int)(cell & (NSPLIT - 1));
      const i64 win = cell / NSPLIT;
      const bool ok = win < (i64)n * CELLS_Y * CELLS_X;
      const int cx = (int)(win % CELLS_X);
      const int cy = (int)((win / CELLS_X) % CELLS_Y);
      const i64 img = ok ? win / ((i64)CELLS_X * CELLS_Y) : 0;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        oyp[p] = cy * 2 + (NSPLIT == 4 ? half >> 1 : NSPLIT == 2 ? half : p / PX);
        oxp[p] = NSPLIT == 4 ? cx * 2 + (half & 1) : cx * PX + p % PX;
        imgp[p] = img;
        live[p] = ok;
      }
      if (!ok) return;
    } else {
      constexpr i64 HW = (i64)C::HO * C::WO;
      const i64 base = (cell >> 5) * (32 * PX) + (cell & 31);
      bool any = false;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const i64 q = base + 32 * p;
        live[p] = q < (i64)n * HW;
        any |= live[p];
        const i64 qq = live[p] ? q : 0;
        imgp[p] = qq / HW;
        const int r = (int)(qq - imgp[p] * HW);
        oyp[p] = r / C::WO;
        oxp[p] = r % C::WO;
      }
      if (!any) return;
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) inp[p] = at<float>(arena, C::IN_OFF + imgp[p] * C::IN_IMG);

    float acc[NP][C::CO];
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int o = 0; o < C::CO; ++o) {
        if constexpr (C::WIMM) acc[p][o] = C::bias(o);
        else acc[p][o] = sm.b[o];
      }

    // weights as immediates (Cfg::wt, WIMM): every loop below is unrolled,
    // so each FFMA takes its weight from the instruction stream; otherwise
    // warp-uniform LDS.128 broadcasts from shared memory, and the kernel-row
    // loop stays rolled (ROLL_KY) when the unrolled body would make NVRTC
    // slow (kernels.py DIRECT_UNROLL_MAX)
    // ROLL_KY = 1: the ky loop is rolled; 2: ky and kx are (one rolled loop
    // over the KH*KW taps)
    // PATCH: a stride-1 pooled window over <= 4 channels reads its whole
    // (PY+KH-1) x (PX+KW-1) input patch once into registers (16 loads for a
    // 3x3 conv instead of 36 per-tap loads with their bounds arithmetic --
    // the stems were issue-bound: cfg0's 32x32x1 -> 8 conv 79% issue-active
    // at 50% FMA-pipe use); the FFMAs keep the (ky, kx, ci) order
    constexpr bool PATCH = C::POOL && NSPLIT == 1 && C::S == 1 && C::CI <= 4 && C::WIMM &&
                           C::ROLL_KY == 0;
    constexpr int PR = PATCH ? PY + C::KH - 1 : 1, PCC = PATCH ? PX + C::KW - 1 : 1;
    float pt[PR][PCC][PATCH ? C::CI : 1];
    if constexpr (PATCH) {
      const int iy0 = oyp[0] - C::PT, ix0 = oxp[0] - C::PL;
#pragma unroll
      for (int r = 0; r < PR; ++r)
#pragma unroll
        for (int c = 0; c < PCC; ++c) {
          const int iy = iy0 + r, ix = ix0 + c;
          const bool ok = iy >= 0 && iy < C::H && ix >= 0 && ix < C::W;
          const float* src = inp[0] + ((i64)(ok ? iy : 0) * C::W + (ok ? ix : 0)) * C::CI;
#pragma unroll
          for (int ci = 0; ci < C::CI; ++ci) pt[r][c][ci] = ok ? lda(src + ci) : 0.f;
        }
    }
    // RUN: the KW * CI floats a kernel row reads for one pixel are one
    // contiguous run of the input; with CI % 4 != 0 (the RGB stems) the
    // per-tap path issued one scalar load with its own bounds arithmetic per
    // (tap, channel) -- 27 loads for a 3x3x3 window, and the stems are
    // issue-bound.  Here each kernel row's run is read once per pixel, as
    // 8-byte loads where the run starts 8-byte aligned (even S*CI, W*CI,
    // PL*CI: the stride-2 stems), with one row test and one test per column;
    // the FFMAs keep the (ky, kx, ci) order.
    constexpr bool RUN = !PATCH && CV == 1 && C::WIMM && C::ROLL_KY == 0 && C::KW * C::CI <= 16 &&
                         C::KW * C::CI > 1;
    constexpr bool RUN2 = RUN && (C::S * C::CI) % 2 == 0 && (C::W * C::CI) % 2 == 0 &&
                          (C::PL * C::CI) % 2 == 0 && C::IN_IMG % 8 == 0 && C::IN_OFF % 8 == 0;
    constexpr int RL = RUN ? C::KW * C::CI : 1;
    constexpr int TAPS_ROLLED = C::ROLL_KY == 2 ? C::KH * C::KW : C::ROLL_KY == 1 ? C::KH : 1;
    constexpr int KX_UNROLLED = C::ROLL_KY == 2 ? 1 : C::KW;
#pragma unroll
    for (int ky = 0; ky < C::KH * C::KW / (TAPS_ROLLED * KX_UNROLLED); ++ky) {
     float rn[NP][RL];
     if constexpr (RUN) {
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const int iy = oyp[p] * C::S - C::PT + ky;
        const int ix0 = oxp[p] * C::S - C::PL;
        const bool rowok = iy >= 0 && iy < C::H;
        const float* src = inp[p] + ((i64)(rowok ? iy : 0) * C::W + ix0) * C::CI;
        bool ok[C::KW];
#pragma unroll
        for (int c = 0; c < C::KW; ++c) ok[c] = rowok && ix0 + c >= 0 && ix0 + c < C::W;
#pragma unroll
        for (int e = 0; e < RL; e += (RUN2 ? 2 : 1)) {
          if (RUN2 && e + 1 < RL) {
            const bool o0 = ok[e / C::CI], o1 = ok[(e + 1) / C::CI];
            float2 v = make_float2(0.f, 0.f);
            if (o0 && o1) v = lda(reinterpret_cast<const float2*>(src + e));
            else if (o0) v.x = lda(src + e);
            else if (o1) v.y = lda(src + e + 1);
            rn[p][e] = v.x;
            rn[p][e + 1] = v.y;
          } else {
            rn[p][e] = ok[e / C::CI] ? lda(src + e) : 0.f;
          }
        }
      }
     }
#pragma unroll 1
     for (int tr = 0; tr < TAPS_ROLLED; ++tr) {
#pragma unroll
      for (int kxu = 0; kxu < KX_UNROLLED; ++kxu) {
        const int ky_ = C::ROLL_KY == 2 ? tr / C::KW : C::ROLL_KY == 1 ? tr : ky;
        const int kx = C::ROLL_KY == 2 ? tr % C::KW : kxu;
#pragma unroll
        for (int c0 = 0; c0 < C::CI; c0 += CV) {
          float xv[NP][CV];
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            if constexpr (PATCH) {
#pragma unroll
              for (int c = 0; c < CV; ++c) xv[p][c] = pt[p / PX + ky_][p % PX + kx][c0 + c];
              continue;
            }
            if constexpr (RUN) {
              xv[p][0] = rn[p][kx * C::CI + c0];
              continue;
            }
            const int iy = oyp[p] * C::S - C::PT + ky_;
            const int ix = oxp[p] * C::S - C::PL + kx;
            const bool ok = iy >= 0 && iy < C::H && ix >= 0 && ix < C::W;
            const float* src = inp[p] + ((i64)iy * C::W + ix) * C::CI + c0;
            if (CV == 4) {
              float4 v = ok ? lda(reinterpret_cast<const float4*>(src)) : make_float4(0.f, 0.f, 0.f, 0.f);
              xv[p][0] = v.x; xv[p][CV > 1 ? 1 : 0] = v.y; xv[p][CV > 2 ? 2 : 0] = v.z; xv[p][CV > 3 ? 3 : 0] = v.w;
            } else {
              xv[p][0] = ok ? lda(src) : 0.f;
            }
          }
#pragma unroll
          for (int c = 0; c < CV; ++c) {
            const int wi = ((ky_ * C::KW + kx) * C::CI + c0 + c) * C::CO;
            const float* wr = sm.w + wi;
            if constexpr (C::WIMM) {
#pragma unroll
              for (int o = 0; o < C::CO; ++o) {
                const float wv = C::wt(wi + o);
#pragma unroll
                for (int p = 0; p < NP; ++p) acc[p][o] = fmaf(xv[p][c], wv, acc[p][o]);
              }
            } else if (C::CO % 4 == 0) {      // one LDS.128 broadcast feeds 4*NP FMAs
#pragma unroll
              for (int o = 0; o < C::CO; o += 4) {
                const float4 w4 = *reinterpret_cast<const float4*>(wr + o);
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                  acc[p][o] = fmaf(xv[p][c], w4.x, acc[p][o]);
                  acc[p][o + 1] = fmaf(xv[p][c], w4.y, acc[p][o + 1]);
                  acc[p][o + 2] = fmaf(xv[p][c], w4.z, acc[p][o + 2]);
                  acc[p][o + 3] = fmaf(xv[p][c], w4.w, acc[p][o + 3]);
                }
              }
            } else {
#pragma unroll
              for (int o = 0; o < C::CO; ++o) {
                const float wv = wr[o];
#pragma unroll
                for (int p = 0; p < NP; ++p) acc[p][o] = fmaf(xv[p][c], wv, acc[p][o]);
              }
            }
          }
        }
      }
     }
    }

    const float* ps = at<float>(pool, C::PS_OFF);
    const float* po = at<float>(pool, C::PO_OFF);
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int o = 0; o < C::CO; ++o) acc[p][o] = finish<C::ACT, C::MODE, C::POST>(acc[p][o], ps, po, o);

    if (PSPLIT) {
      // both lanes of a window are live or neither (the early return above
      // is per window), so the pair exchange needs no full-warp mask
      const unsigned mask = __activemask();
      float* dst = at<float>(arena, C::OUT_OFF + imgp[0] * C::OUT_IMG) +
                   ((i64)(oyp[0] / 2) * C::PWO + oxp[0] / 2) * C::CO;
      const bool top = (oyp[0] & 1) == 0 && (NSPLIT == 2 || (oxp[0] & 1) == 0);
#pragma unroll
      for (int o = 0; o < C::CO; o += 4) {
        float m4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (o + i < C::CO) {
            float m = NP > 1 ? fmaxf(acc[0][o + i], acc[NP > 1 ? 1 : 0][o + i]) : acc[0][o + i];
            m = fmaxf(m, __shfl_xor_sync(mask, m, 1));
            if (NSPLIT == 4) m = fmaxf(m, __shfl_xor_sync(mask, m, 2));
            m4[i] = m;
          }
        }
        if (top) {
          if (C::CO % 4 == 0) {
            *reinterpret_cast<float4*>(dst + o) = make_float4(m4[0], m4[1], m4[2], m4[3]);
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (o + i < C::CO) dst[o + i] = m4[i];
          }
        }
      }
      return;
    }
    if (C::POOL) {
      float* dst = at<float>(arena, C::OUT_OFF + imgp[0] * C::OUT_IMG) +
                   ((i64)(oyp[0] / 2) * C::PWO + oxp[0] / 2) * C::CO;
      if (C::CO % 4 == 0) {
#pragma unroll
        for (int o = 0; o < C::CO; o += 4) {
          float m4[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            m4[i] = fmaxf(fmaxf(acc[0][o + i], acc[1][o + i]), fmaxf(acc[2][o + i], acc[3][o + i]));
          *reinterpret_cast<float4*>(dst + o) = make_float4(m4[0], m4[1], m4[2], m4[3]);
        }
      } else {
#pragma unroll
        for (int o = 0; o < C::CO; ++o)
          dst[o] = fmaxf(fmaxf(acc[0][o], acc[1][o]), fmaxf(acc[2][o], acc[3][o]));
      }
      return;
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const int oy = oyp[p], ox = oxp[p];
      if (!live[p]) continue;
      float* out = at<float>(arena, C::OUT_OFF + imgp[p] * C::OUT_IMG);
      const i64 pix = (i64)oy * C::WO + ox;
      float* dst = out + (C::UPF > 1 ? ((i64)(oy * C::UPF) * C::WO * C::UPF + ox * C::UPF) : pix) * C::CO;
      if (C::RES) {
        const float* res = at<float>(arena, C::RES_OFF + imgp[p] * C::OUT_IMG) + pix * C::CO;
#pragma unroll
        for (int o = 0; o < C::CO; ++o) acc[p][o] = add(acc[p][o], lda(res + o));
      }
#pragma unroll
      for (int rep = 0; rep < C::UPF * C::UPF; ++rep) {
        float* d = dst + ((i64)(rep / C::UPF) * C::WO * C::UPF + rep % C::UPF) * C::CO;
        if (C::CO % 4 == 0) {
#pragma unroll
          for (int o = 0; o < C::CO; o += 4)
            *reinterpret_cast<float4*>(d + o) = make_float4(acc[p][o], acc[p][o + 1], acc[p][o + 2], acc[p][o + 3]);
        } else {
#pragma unroll
          for (int o = 0; o < C::CO; ++o) d[o] = acc[p][o];
        }
      }
    }
  }
};

}  // namespace nnb
