/* nnoracle.c -- CPU oracle for the CompiledNN forward pass.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker or the reported CPU baseline -- never as the product
 * path.
 *
 * A plain-C restatement of the reference interpreter
 * (pkg/src/nnjit/interpreter.py), batched over images and threaded over
 * them with pthreads.  Every multiply and add rounds to float32 in the
 * interpreter's documented order (interpreter.py:1-19); build with
 * -ffp-contract=off and without -ffast-math so the compiler cannot fuse or
 * reassociate:
 *   dense      acc_j = bias_j; acc_j += x_i * K[i,j], i ascending        (:45-49)
 *   conv2d     acc = bias; taps (ky, kx, ci) lexicographic over the
 *              zero-padded input                                          (:52-62)
 *   depthwise  acc = bias; taps (ky, kx)                                  (:65-73)
 *   max pool   -inf start, padded taps are -inf                           (:76-82)
 *   avg pool   sum over the zero-padded window / count of in-bounds taps  (:85-95)
 *   batchnorm  x*scale + offset                                           (:98-99)
 *   tanh/sigmoid/softmax in float64, rounded once                         (:102-118)
 * Extensions (not in the reference, pinned by tests/test_oracle.py's naive
 * loops): relu6, elu (float64 expm1), per-pixel channel softmax, zero padding.
 *
 * The approximation models of pkg/src/nnjit/codegen/approx.py:72-128
 * (rational/fast tanh and sigmoid, fast and precise exp) are restated
 * operation by operation for the "compiled path" semantics (oracle B). */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { int lo, hi; void *ctx; void (*fn)(void *, int, int); } job_t;

static void *job_main(void *p) {
  job_t *j = (job_t *)p;
  j->fn(j->ctx, j->lo, j->hi);
  return NULL;
}

/* split [0, n) over up to nthreads workers */
static void parallel(int n, int nthreads, void *ctx, void (*fn)(void *, int, int)) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > n) nthreads = n;
  if (nthreads <= 1) { fn(ctx, 0, n); return; }
  pthread_t th[256];
  job_t jobs[256];
  if (nthreads > 256) nthreads = 256;
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].lo = (int)((long)n * t / nthreads);
    jobs[t].hi = (int)((long)n * (t + 1) / nthreads);
    jobs[t].ctx = ctx;
    jobs[t].fn = fn;
    pthread_create(&th[t], NULL, job_main, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* ------------------------------------------------------------------ approx */
#define TANH_CLAMP 5.7f
static float f32_bits(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }
static uint32_t bits_f32(float f) { uint32_t b; memcpy(&b, &f, 4); return b; }

static float pade(float x) {
  float t = x * x;
  float num = t * 36.0f + 6930.0f;
  num = num * t + 270270.0f;
  num = num * t + 2027025.0f;
  num = num * x;
  float den = t + 630.0f;
  den = den * t + 51975.0f;
  den = den * t + 945945.0f;
  den = den * t + 2027025.0f;
  return num / den;
}

static float np_max(float a, float b) { return (a >= b || a != a) ? a : b; }
static float np_min(float a, float b) { return (a <= b || a != a) ? a : b; }

float nno_tanh_rational(float x) {
  static float at_clamp = 0.0f, delta = 0.0f;
  if (at_clamp == 0.0f) { at_clamp = pade(TANH_CLAMP); delta = 1.0f - at_clamp; }
  x = np_min(np_max(x, -TANH_CLAMP), TANH_CLAMP);
  float p = pade(x);
  float adj = fabsf(p) == at_clamp ? delta : 0.0f;
  return p + copysignf(adj, p);
}

float nno_sigmoid_rational(float x) {
  float y = nno_tanh_rational(x * 0.5f);
  return y * 0.5f + 0.5f;
}

#define EXP_A ((float)12102203.161561485)
#define EXP_BIAS ((127 << 23) - 366000)
#define EXP_CLAMP 80.0f

float nno_exp_fast(float x) {
  x = np_min(np_max(x, -EXP_CLAMP), EXP_CLAMP);
  float prod = x * EXP_A;
  int32_t b = (int32_t)rintf(prod) + EXP_BIAS;
  return f32_bits((uint32_t)b);
}

float nno_sigmoid_fast(float x) { return 1.0f / (nno_exp_fast(-x) + 1.0f); }
float nno_tanh_fast(float x) { return 2.0f / (nno_exp_fast(x * -2.0f) + 1.0f) - 1.0f; }

float nno_exp_precise(float x) {
  const float inv_ln2 = (float)1.4426950408889634;
  const float ln2_hi = 0.693359375f;
  const float ln2_lo = (float)(0.6931471805599453 - 0.693359375);
  const float poly[8] = {(float)(1.0 / 5040), (float)(1.0 / 720), (float)(1.0 / 120),
                         (float)(1.0 / 24), (float)(1.0 / 6), 0.5f, 1.0f, 1.0f};
  x = np_min(np_max(x, -EXP_CLAMP), EXP_CLAMP);
  int32_t k = (int32_t)rintf(x * inv_ln2);
  float two_k = f32_bits((uint32_t)((k + 127) << 23));
  float kf = (float)k;
  float r = (x - kf * ln2_hi) - kf * ln2_lo;
  float p = r * poly[0] + poly[1];
  for (int i = 2; i < 8; ++i) p = p * r + poly[i];
  return p * two_k;
}

/* activation codes: 0 linear 1 relu 2 sigmoid 3 tanh 4 relu6 5 elu
 * modes: 0 rational 1 fast 2 exact */
static float act1(float x, int act, int mode) {
  switch (act) {
    case 1: return np_max(x, 0.0f);
    case 4: return np_min(np_max(x, 0.0f), 6.0f);
    case 5: return x > 0.0f ? x : (float)expm1((double)x);
    case 3:
      if (mode == 0) return nno_tanh_rational(x);
      if (mode == 1) return nno_tanh_fast(x);
      return (float)tanh((double)x);
    case 2:
      if (mode == 0) return nno_sigmoid_rational(x);
      if (mode == 1) return nno_sigmoid_fast(x);
      return (float)(1.0 / (1.0 + exp(-(double)x)));
    default: return x;
  }
}

void nno_activation(const float *x, float *y, long count, int act, int mode) {
  for (long i = 0; i < count; ++i) y[i] = act1(x[i], act, mode);
}

/* ------------------------------------------------------------------- dense */
typedef struct { const float *x, *w, *b; float *y; int k, u; } dense_t;

static void dense_rows(void *p, int lo, int hi) {
  dense_t *d = (dense_t *)p;
  for (int r = lo; r < hi; ++r) {
    const float *x = d->x + (long)r * d->k;
    float *acc = d->y + (long)r * d->u;
    for (int j = 0; j < d->u; ++j) acc[j] = d->b[j];
    for (int i = 0; i < d->k; ++i) {
      const float xi = x[i];
      const float *wr = d->w + (long)i * d->u;
      for (int j = 0; j < d->u; ++j) acc[j] = acc[j] + xi * wr[j];
    }
  }
}

void nno_dense(const float *x, int n, int k, const float *w, const float *b, int u, float *y,
               int nthreads) {
  dense_t d = {x, w, b, y, k, u};
  parallel(n, nthreads, &d, dense_rows);
}

/* ------------------------------------------------------------------ conv2d */
typedef struct {
  const float *x, *w, *b; float *y;
  int h, wd, ci, kh, kw, co, s, pt, pl, ho, wo, depthwise;
} conv_t;

static void conv_images(void *p, int lo, int hi) {
  conv_t *c = (conv_t *)p;
  float *acc = (float *)malloc(sizeof(float) * (c->depthwise ? c->ci : c->co));
  for (int img = lo; img < hi; ++img) {
    const float *x = c->x + (long)img * c->h * c->wd * c->ci;
    for (int oy = 0; oy < c->ho; ++oy)
      for (int ox = 0; ox < c->wo; ++ox) {
        float *out = c->y + (((long)img * c->ho + oy) * c->wo + ox) * (c->depthwise ? c->ci : c->co);
        if (!c->depthwise) {
          for (int o = 0; o < c->co; ++o) acc[o] = c->b[o];
          for (int ky = 0; ky < c->kh; ++ky)
            for (int kx = 0; kx < c->kw; ++kx) {
              int iy = oy * c->s - c->pt + ky, ix = ox * c->s - c->pl + kx;
              int in = iy >= 0 && iy < c->h && ix >= 0 && ix < c->wd;
              for (int ci = 0; ci < c->ci; ++ci) {
                float v = in ? x[((long)iy * c->wd + ix) * c->ci + ci] : 0.0f;
                const float *wr = c->w + (((long)ky * c->kw + kx) * c->ci + ci) * c->co;
                for (int o = 0; o < c->co; ++o) acc[o] = acc[o] + v * wr[o];
              }
            }
          memcpy(out, acc, sizeof(float) * c->co);
        } else {
          for (int ch = 0; ch < c->ci; ++ch) acc[ch] = c->b[ch];
          for (int ky = 0; ky < c->kh; ++ky)
            for (int kx = 0; kx < c->kw; ++kx) {
              int iy = oy * c->s - c->pt + ky, ix = ox * c->s - c->pl + kx;
              int in = iy >= 0 && iy < c->h && ix >= 0 && ix < c->wd;
              const float *wr = c->w + ((long)ky * c->kw + kx) * c->ci;
              for (int ch = 0; ch < c->ci; ++ch) {
                float v = in ? x[((long)iy * c->wd + ix) * c->ci + ch] : 0.0f;
                acc[ch] = acc[ch] + v * wr[ch];
              }
            }
          memcpy(out, acc, sizeof(float) * c->ci);
        }
      }
  }
  free(acc);
}

void nno_conv2d(const float *x, int n, int h, int w, int ci, const float *k, const float *b,
                int kh, int kw, int co, int s, int pt, int pl, int ho, int wo, float *y,
                int depthwise, int nthreads) {
  conv_t c = {x, k, b, y, h, w, ci, kh, kw, co, s, pt, pl, ho, wo, depthwise};
  parallel(n, nthreads, &c, conv_images);
}

/* -------------------------------------------------------------------- pool */
void nno_pool(const float *x, int n, int h, int w, int c, int ph, int pw, int s, int pt, int pl,
              int ho, int wo, int avg, float *y) {
  for (long img = 0; img < n; ++img)
    for (int oy = 0; oy < ho; ++oy)
      for (int ox = 0; ox < wo; ++ox)
        for (int ch = 0; ch < c; ++ch) {
          float acc = avg ? 0.0f : -INFINITY, cnt = 0.0f;
          for (int ky = 0; ky < ph; ++ky)
            for (int kx = 0; kx < pw; ++kx) {
              int iy = oy * s - pt + ky, ix = ox * s - pl + kx;
              int in = iy >= 0 && iy < h && ix >= 0 && ix < w;
              float v = in ? x[(((img * h) + iy) * (long)w + ix) * c + ch] : (avg ? 0.0f : -INFINITY);
              if (avg) { acc = acc + v; cnt = cnt + (in ? 1.0f : 0.0f); }
              else acc = np_max(acc, v);
            }
          y[(((img * ho) + oy) * (long)wo + ox) * c + ch] = avg ? acc / cnt : acc;
        }
}

/* ------------------------------------------------------------- elementwise */
void nno_affine(const float *x, float *y, long count, const float *scale, const float *offset, int c) {
  for (long i = 0; i < count; ++i) y[i] = x[i] * scale[i % c] + offset[i % c];
}

void nno_add(float *acc, const float *x, long count) {
  for (long i = 0; i < count; ++i) acc[i] = acc[i] + x[i];
}

/* softmax over rows of length l.  smexp: 0 fast, 1 precise (float32 models,
 * sequential sum, one reciprocal), 2 exact (interpreter, float64). */
void nno_softmax(const float *x, float *y, long rows, int l, int smexp) {
  double *e = (double *)malloc(sizeof(double) * (size_t)l);
  for (long r = 0; r < rows; ++r) {
    const float *v = x + r * l;
    float *o = y + r * l;
    float m = v[0];
    for (int j = 1; j < l; ++j) m = np_max(m, v[j]);
    if (smexp == 2) {
      double s = 0.0;
      for (int j = 0; j < l; ++j) { e[j] = exp((double)v[j] - (double)m); s += e[j]; }
      for (int j = 0; j < l; ++j) o[j] = (float)(e[j] / s);
    } else {
      float s = 0.0f;
      for (int j = 0; j < l; ++j) {
        float d = v[j] - m;
        o[j] = smexp == 0 ? nno_exp_fast(d) : nno_exp_precise(d);
        s = s + o[j];
      }
      float inv = 1.0f / s;
      for (int j = 0; j < l; ++j) o[j] = o[j] * inv;
    }
  }
  free(e);
}

/* ------------------------------------------------------------ data movement */
void nno_upsample(const float *x, int n, int h, int w, int c, int f, float *y) {
  for (long img = 0; img < n; ++img)
    for (int oy = 0; oy < h * f; ++oy)
      for (int ox = 0; ox < w * f; ++ox)
        memcpy(y + (((img * h * f) + oy) * (long)w * f + ox) * c,
               x + (((img * h) + oy / f) * (long)w + ox / f) * c, sizeof(float) * c);
}

/* copy a [n, p, cs] source into channels [c0, c0+cs) of a [n, p, ct] tensor */
void nno_concat_part(const float *x, int n, long p, int cs, float *y, int ct, int c0) {
  for (long img = 0; img < n; ++img)
    for (long q = 0; q < p; ++q)
      memcpy(y + (img * p + q) * ct + c0, x + (img * p + q) * cs, sizeof(float) * cs);
}

void nno_zeropad(const float *x, int n, int h, int w, int c, int pt, int pl, int ho, int wo, float *y) {
  memset(y, 0, sizeof(float) * (size_t)n * ho * wo * c);
  for (long img = 0; img < n; ++img)
    for (int iy = 0; iy < h; ++iy)
      memcpy(y + (((img * ho) + iy + pt) * (long)wo + pl) * c, x + ((img * h) + iy) * (long)w * c,
             sizeof(float) * (size_t)w * c);
}

uint32_t nno_bits(float f) { return bits_f32(f); }
