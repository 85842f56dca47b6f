// nnb_gemm_simt.cuh -- FFMA implicit-GEMM for Conv2D / 1x1 conv / Dense.
//
// GEMM view of a convolution (NHWC, batch-major arena):
//   row m    = one output pixel  (img, oy, ox)           M = n * ROWS
//   column j = one output channel                          N = CO
//   k        = one tap (ky, kx, ci), lexicographic         K = KH*KW*CI
// A[m,k] is gathered on the fly (zero outside the image = TF 'same' padding,
// graph.py same_padding), B[k,j] is the (kh,kw,cin,cout) kernel read as a
// (K, CO) row-major matrix, exactly the layout of the container blob.
//
// Accumulators start at the bias and take the taps in ascending k, the
// accumulation order of the reference interpreter (pkg/src/nnjit/
// interpreter.py:52-62); the only difference is the fused multiply-add
// rounding, which the FP32 parity gate (rtol 1e-4 / atol 1e-5) absorbs.
//
// Fused epilogue (planner.py): activation, post-BN affine, residual Add,
// 2x2/2 max-pool (rows are numbered so four consecutive rows form one pool
// window and a thread owns whole windows), and a per-row softmax when a
// thread owns the entire row (TN >= CO).
#pragma once
#include "nnb_common.cuh"
#include "nnb_softmax.cuh"

namespace nnb {

template <class C>
struct GemmSimt {
  static constexpr int NTX = C::BN / C::TN;            // threads along N
  static constexpr int NTY = C::BM / C::TM;            // threads along M
  static constexpr int NT = NTX * NTY;
  static constexpr int APAD = 4;
  static constexpr int AST = C::BM + APAD;             // As row stride
  static constexpr int BST = C::BN + 4;                // Bs row stride
  static constexpr bool AVEC = (C::CI % 4 == 0) && (C::BK % 4 == 0);
  static constexpr int AKV = AVEC ? 4 : 1;             // k elements per A load
  static constexpr int A_LOADS = C::BM * C::BK / AKV / NT;
  static constexpr bool BVEC = (C::CO % 4 == 0) && (C::BN % 4 == 0);
  static constexpr int BJV = BVEC ? 4 : 1;
  static constexpr int B_LOADS = (C::BK * C::BN / BJV + NT - 1) / NT;
  static constexpr int KCH = (C::K + C::BK - 1) / C::BK;
  static_assert(C::BM * C::BK % (AKV * NT) == 0, "A tile must split evenly");
  static_assert(C::TN <= C::BN && C::TM % (C::POOL ? 4 : 1) == 0, "tile");

  struct Smem {
    float a[2][C::BK][AST];
    float b[2][C::BK][BST];
  };

  // pixel coordinates of GEMM row r inside one image
  __device__ static __forceinline__ void row_pixel(int r, int& oy, int& ox) {
    if (C::POOL) {
      int w = r >> 2, q = r & 3;
      oy = 2 * (w / C::PWO) + (q >> 1);
      ox = 2 * (w % C::PWO) + (q & 1);
    } else {
      oy = r / C::WO;
      ox = r % C::WO;
    }
  }

  // depthwise output at pixel (oy, ox) of its output map, channels c..c+3:
  // bias, taps (ky, kx) as FMAs, then its own activation / post-BN
  __device__ static __forceinline__ float4 dw_point(const float* __restrict__ pool,
                                                    const float* img, int oy, int ox, int c) {
    const float* wk = at<float>(pool, C::DW_W_OFF);
    float4 acc = __ldg(reinterpret_cast<const float4*>(at<float>(pool, C::DW_B_OFF) + c));
#pragma unroll
    for (int ky = 0; ky < C::DW_KH; ++ky) {
      const int y = oy * C::DW_S - C::DW_PT + ky;
      if (y < 0 || y >= C::DW_H) continue;
#pragma unroll
      for (int kx = 0; kx < C::DW_KW; ++kx) {
        const int x = ox * C::DW_S - C::DW_PL + kx;
        if (x < 0 || x >= C::DW_W) continue;
        const float4 v = lda(reinterpret_cast<const float4*>(img + ((i64)y * C::DW_W + x) * C::CI + c));
        const float4 w = __ldg(reinterpret_cast<const float4*>(wk + (ky * C::DW_KW + kx) * C::CI + c));
        acc.x = fmaf(v.x, w.x, acc.x); acc.y = fmaf(v.y, w.y, acc.y);
        acc.z = fmaf(v.z, w.z, acc.z); acc.w = fmaf(v.w, w.w, acc.w);
      }
    }
    const float* ps = at<float>(pool, C::DW_PS_OFF);
    const float* po = at<float>(pool, C::DW_PO_OFF);
    acc.x = finish<C::DW_ACT, C::MODE, C::DW_POST>(acc.x, ps, po, c);
    acc.y = finish<C::DW_ACT, C::MODE, C::DW_POST>(acc.y, ps, po, c + 1);
    acc.z = finish<C::DW_ACT, C::MODE, C::DW_POST>(acc.z, ps, po, c + 2);
    acc.w = finish<C::DW_ACT, C::MODE, C::DW_POST>(acc.w, ps, po, c + 3);
    return acc;
  }

  __device__ static void run(const float* __restrict__ pool, float* __restrict__ arena,
                             int n, Smem& sm) {
    const int tid = threadIdx.x;
    const int tx = tid % NTX, ty = tid / NTX;
    const i64 mtotal = (i64)n * C::ROWS;
    const int ntile_n = (C::CO + C::BN - 1) / C::BN;
    const i64 m0 = (i64)(nnb_bid() / ntile_n) * C::BM;
    const int n0 = (int)(nnb_bid() % ntile_n) * C::BN;
    if (m0 >= mtotal) return;

    const float* __restrict__ in = at<float>(arena, C::IN_OFF);
    const float* __restrict__ wk = at<float>(pool, C::W_OFF);

    // ---- per-thread A-load rows (fixed across the K loop) ----
    constexpr int KQ = C::BK / AKV;          // load slots per row
    int a_mi[A_LOADS], a_kq[A_LOADS];
    const float* a_base[A_LOADS];          // image base of source 0 (or the only source)
    int a_iy[A_LOADS], a_ix[A_LOADS];
    i64 a_img[A_LOADS];
#pragma unroll
    for (int l = 0; l < A_LOADS; ++l) {
      int e = tid + l * NT;
      a_kq[l] = e % KQ;
      a_mi[l] = e / KQ;
      i64 m = m0 + a_mi[l];
      if (m < mtotal) {
        i64 img = m / C::ROWS;
        int r = (int)(m - img * C::ROWS);
        int oy, ox;
        row_pixel(r, oy, ox);
        a_base[l] = in + img * (C::IN_IMG / 4);
        a_img[l] = img;
        a_iy[l] = oy * C::S - C::PT;
        a_ix[l] = ox * C::S - C::PL;
      } else {
        a_base[l] = nullptr;
        a_iy[l] = a_ix[l] = 0;
        a_img[l] = 0;
      }
    }

    float ra[A_LOADS][AKV];
    float rb[B_LOADS][BJV];

    auto load_a = [&](int k0) {
#pragma unroll
      for (int l = 0; l < A_LOADS; ++l) {
        int k = k0 + a_kq[l] * AKV;
        bool ok = a_base[l] != nullptr && k < C::K;
        int ky = k / (C::KW * C::CI);
        int kx = (k / C::CI) % C::KW;
        int ci = k % C::CI;
        int iy = a_iy[l] + ky, ix = a_ix[l] + kx;
        ok = ok && iy >= 0 && iy < C::H && ix >= 0 && ix < C::W;
        if (C::DW) {
          // fused depthwise producer: A[pixel, ci..ci+3] = dw(x)(iy, ix, ci..ci+3)
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (ok) v = dw_point(pool, a_base[l], iy, ix, ci);
          ra[l][0] = v.x; if (AKV > 1) { ra[l][1 % AKV] = v.y; ra[l][2 % AKV] = v.z; ra[l][3 % AKV] = v.w; }
          continue;
        }
        // channel-concat loader: channels [0, C0) from source 0, the rest from source 1
        const float* src = a_base[l] + (iy * C::W + ix) * C::C0 + ci;
        if (C::CONCAT && ci >= C::C0)
          src = at<float>(arena, C::IN1_OFF) + a_img[l] * (C::IN1_IMG / 4) +
                (iy * C::W + ix) * (C::CI - C::C0) + (ci - C::C0);
        if (AVEC) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (ok) v = lda(reinterpret_cast<const float4*>(src));
          ra[l][0] = v.x; if (AKV > 1) { ra[l][1 % AKV] = v.y; ra[l][2 % AKV] = v.z; ra[l][3 % AKV] = v.w; }
        } else {
          ra[l][0] = ok ? lda(src) : 0.f;
        }
      }
    };
    auto store_a = [&](int buf) {
#pragma unroll
      for (int l = 0; l < A_LOADS; ++l)
#pragma unroll
        for (int v = 0; v < AKV; ++v) sm.a[buf][a_kq[l] * AKV + v][a_mi[l]] = ra[l][v];
    };
    auto load_b = [&](int k0) {
#pragma unroll
      for (int l = 0; l < B_LOADS; ++l) {
        int e = tid + l * NT;
        int kk = e / (C::BN / BJV), jq = e % (C::BN / BJV);
        int k = k0 + kk, j = n0 + jq * BJV;
        bool ok = (e < C::BK * C::BN / BJV) && k < C::K;
        if (BVEC) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (ok && j < C::CO) v = __ldg(reinterpret_cast<const float4*>(wk + (i64)k * C::CO + j));
          rb[l][0] = v.x; if (BJV > 1) { rb[l][1 % BJV] = v.y; rb[l][2 % BJV] = v.z; rb[l][3 % BJV] = v.w; }
        } else {
          rb[l][0] = (ok && j < C::CO) ? __ldg(wk + (i64)k * C::CO + j) : 0.f;
        }
      }
    };
    auto store_b = [&](int buf) {
#pragma unroll
      for (int l = 0; l < B_LOADS; ++l) {
        int e = tid + l * NT;
        if (e < C::BK * C::BN / BJV) {
          int kk = e / (C::BN / BJV), jq = e % (C::BN / BJV);
#pragma unroll
          for (int v = 0; v < BJV; ++v) sm.b[buf][kk][jq * BJV + v] = rb[l][v];
        }
      }
    };

    // ---- accumulators start at the bias ----
    float acc[C::TM][C::TN];
    {
      const float* bias = at<float>(pool, C::B_OFF);
#pragma unroll
      for (int j = 0; j < C::TN; ++j) {
        int col = n0 + tx * C::TN + j;
        float bv = col < C::CO ? __ldg(bias + col) : 0.f;
#pragma unroll
        for (int i = 0; i < C::TM; ++i) acc[i][j] = bv;
      }
    }

    load_a(0);
    load_b(0);
    store_a(0);
    store_b(0);
    nnb_sync();
    for (int kc = 0; kc < KCH; ++kc) {
      const int buf = kc & 1;
      if (kc + 1 < KCH) {
        load_a((kc + 1) * C::BK);
        load_b((kc + 1) * C::BK);
      }
#pragma unroll
      for (int kk = 0; kk < C::BK; ++kk) {
        float av[C::TM], bv[C::TN];
#pragma unroll
        for (int i = 0; i < C::TM; ++i) av[i] = sm.a[buf][kk][ty * C::TM + i];
#pragma unroll
        for (int j = 0; j < C::TN; ++j) bv[j] = sm.b[buf][kk][tx * C::TN + j];
#pragma unroll
        for (int i = 0; i < C::TM; ++i)
#pragma unroll
          for (int j = 0; j < C::TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      if (kc + 1 < KCH) {
        store_a(buf ^ 1);
        store_b(buf ^ 1);
      }
      nnb_sync();
    }

    // ---- epilogue ----
    const float* ps = at<float>(pool, C::PS_OFF);
    const float* po = at<float>(pool, C::PO_OFF);
    float* out = at<float>(arena, C::OUT_OFF);
#pragma unroll
    for (int i = 0; i < C::TM; ++i)
#pragma unroll
      for (int j = 0; j < C::TN; ++j) {
        int col = n0 + tx * C::TN + j;
        acc[i][j] = finish<C::ACT, C::MODE, C::POST>(acc[i][j], ps, po, col < C::CO ? col : 0);
      }

    if (C::POOL) {
      // 4 consecutive rows = one 2x2 window; max is exact in any order
#pragma unroll
      for (int g = 0; g < C::TM / 4; ++g) {
        i64 m = m0 + ty * C::TM + 4 * g;
        if (m >= mtotal) continue;
        i64 img = m / C::ROWS;
        int w = (int)(m - img * C::ROWS) >> 2;
        float* dst = out + img * (C::OUT_IMG / 4) + (i64)w * C::CO;
#pragma unroll
        for (int j = 0; j < C::TN; ++j) {
          int col = n0 + tx * C::TN + j;
          float v = fmaxf(fmaxf(acc[4 * g][j], acc[4 * g + 1][j]),
                          fmaxf(acc[4 * g + 2][j], acc[4 * g + 3][j]));
          if (col < C::CO) dst[col] = v;
        }
      }
      return;
    }

#pragma unroll
    for (int i = 0; i < C::TM; ++i) {
      i64 m = m0 + ty * C::TM + i;
      if (m >= mtotal) continue;
      i64 img = m / C::ROWS;
      int r = (int)(m - img * C::ROWS);
      float* dst = out + img * (C::OUT_IMG / 4) + (i64)r * C::CO;
      if (C::UPF > 1) {       // fused nearest upsampling: the pixel's first replica
        const int oy = r / C::WO, ox = r % C::WO;
        dst = out + img * (C::OUT_IMG / 4) + ((i64)(oy * C::UPF) * C::WO * C::UPF + ox * C::UPF) * C::CO;
      }
      if (C::RES) {
        const float* res = at<float>(arena, C::RES_OFF) + img * (C::OUT_IMG / 4) + (i64)r * C::CO;
#pragma unroll
        for (int j = 0; j < C::TN; ++j) {
          int col = n0 + tx * C::TN + j;
          if (col < C::CO) acc[i][j] = C::RES_FIRST ? add(lda(res + col), acc[i][j])
                                                     : add(acc[i][j], lda(res + col));
        }
      }
      if (C::SOFTMAX) {
        // the thread owns the whole row (planner guarantees TN >= CO, NTX == 1)
        softmax_row_regs<C::TN, C::CO, C::SMEXP>(acc[i]);
      }
#pragma unroll
      for (int rep = 0; rep < C::UPF * C::UPF; ++rep) {
        float* d = dst + ((i64)(rep / C::UPF) * C::WO * C::UPF + rep % C::UPF) * C::CO;
        if (BVEC && C::TN % 4 == 0 && C::CO % 4 == 0) {
#pragma unroll
          for (int j = 0; j < C::TN; j += 4) {
            int col = n0 + tx * C::TN + j;
            if (col < C::CO)
              *reinterpret_cast<float4*>(d + col) =
                  make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < C::TN; ++j) {
            int col = n0 + tx * C::TN + j;
            if (col < C::CO) d[col] = acc[i][j];
          }
        }
      }
    }
  }
};

}  // namespace nnb
