/*
 * oracle/lopt_oracle.c -- CPU restatement of the reference learned-optimizer
 * step (PyLO "lopt" package, numpy + numba).
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * kernels and the CPU baseline timed by bench.py.  Only tests/, the smoke()
 * entry in __graft_entry__.py and bench.py (cpu_baseline leg and
 * `--impl reference`) may load it.  The product path never links it.
 *
 * It restates, operation for operation, the reference functions named in the
 * comments (paths relative to the reference repository root), so that for
 * the same inputs it reproduces the reference bit for bit:
 *
 *   - f32 EMA algebra without contraction (state.py:77-113), compiled with
 *     -ffp-contract=off;
 *   - numpy's f64 reduction orders: pairwise summation along a contiguous
 *     axis, sequential accumulation along axis 0 of a matrix, and 8192-element
 *     buffered chunks when a f32 array is reduced with dtype=float64
 *     (state.py:108-110, features.py:133-135); these orders were checked
 *     against numpy 2.3 in tests/golden/gen_golden.py's self-check;
 *   - the streaming engine's lane blocking (64 lanes that never cross a row),
 *     worker partition and binary-tree merge of f64 partials
 *     (engine.py:431-438, 483-514, 597-616);
 *   - the MLP as a per-output sequential FMA chain starting from the bias
 *     (engine.py:441-480, numba fastmath={"contract"});
 *   - glibc expf through libm, which is what numba's np.exp on float32 calls
 *     (engine.py:537).
 *
 * Pinned against the reference itself: tests/test_oracle_golden.py compares
 * this file's outputs with fixtures produced by importing the reference
 * (tests/golden/gen_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define LO_SMALL_FC_LOPT 0
#define LO_VELO_MLP 1
#define LO_LANES 64            /* engine.py:56 */
#define LO_MAX_FEAT 39
#define LO_MAX_HIDDEN 256

/* status codes shared with oracle.py */
#define LO_OK 0
#define LO_ERR_NONFINITE_GRAD 1
#define LO_ERR_OVERFLOW 2
#define LO_ERR_SHAPE 3
#define LO_ERR_ALLOC 4

static const float EPS_RECIP = 1e-12f;   /* features.py:66 */
static const double EPS_NORM = 1e-5;     /* features.py:67 */
static const float CLIP_BOUND = 0.1f;    /* features.py:82 */

int lo_d_feat(int kind) { return kind == LO_SMALL_FC_LOPT ? 39 : 29; }

/* libm expf over an array (what numba's np.exp on float32 calls). */
void lo_expf_array(const float *x, float *y, int64_t n) {
  for (int64_t i = 0; i < n; i++) y[i] = expf(x[i]);
}

/* ------------------------------------------------------------------ */
/* numpy f64 reduction orders                                           */

/* numpy pairwise_sum for a contiguous f64 run (umath loops, PW_BLOCKSIZE
 * 128, 8 partial accumulators). */
static double pw_sum(const double *a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; i++) res = res + a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    for (int k = 0; k < 8; k++) r[k] = a[k];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; k++) r[k] = r[k] + a[i + k];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res = res + a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pw_sum(a, n2) + pw_sum(a + n2, n - n2);
  }
}

/* np.add.reduce(f32 array, dtype=float64): the cast goes through the
 * iterator's 8192-element buffer, each buffer is pairwise-summed and the
 * buffer sums are accumulated in order. */
static double cast_sum_f32(const float *a, int64_t n) {
  double buf[8192];
  double acc = 0.0;
  for (int64_t s = 0; s < n; s += 8192) {
    int64_t e = s + 8192 < n ? s + 8192 : n;
    for (int64_t i = s; i < e; i++) buf[i - s] = (double)a[i];
    acc = acc + pw_sum(buf, e - s);
  }
  return acc;
}

/* features.py:133-135 factor_means: F32(np.mean(r_i, dtype=float64)). */
float lo_factor_mean(const float *r, int64_t m) {
  return (float)(cast_sum_f32(r, m) / (double)m);
}

/* ------------------------------------------------------------------ */
/* accumulators (state.py)                                             */

/* state.py:116-130 state_step, in place.  betas[0..2] momentum,
 * betas[3] second moment, betas[4..6] adafactor.  Returns LO_OK or
 * LO_ERR_NONFINITE_GRAD (nothing modified in that case). */
int lo_state_step(int64_t m, int64_t n, const float *g, float *M0, float *M1,
                  float *M2, float *V, float *r0, float *r1, float *r2,
                  float *c0, float *c1, float *c2, const double *betas) {
  const int64_t mn = m * n;
  for (int64_t i = 0; i < mn; i++)
    if (!isfinite(g[i])) return LO_ERR_NONFINITE_GRAD;
  float *M[3] = {M0, M1, M2};
  float *r[3] = {r0, r1, r2};
  float *c[3] = {c0, c1, c2};
  /* update_momentum, state.py:77-82: b*M + (1-b)*g in f32 */
  for (int k = 0; k < 3; k++) {
    const float b = (float)betas[k];
    const float omb = 1.0f - b;
    for (int64_t i = 0; i < mn; i++) {
      float t1 = b * M[k][i];
      float t2 = omb * g[i];
      M[k][i] = t1 + t2;
    }
  }
  /* update_second_moment, state.py:85-90: b*V + (1-b)*g^2 */
  {
    const float b = (float)betas[3];
    const float omb = 1.0f - b;
    for (int64_t i = 0; i < mn; i++) {
      float gg = g[i] * g[i];
      float t1 = b * V[i];
      float t2 = omb * gg;
      V[i] = t1 + t2;
    }
  }
  /* update_adafactor, state.py:93-113: row/col means of g^2 in f64 */
  double *row_mean = (double *)malloc(sizeof(double) * (size_t)m);
  double *col_mean = (double *)calloc((size_t)n, sizeof(double));
  double *tmp = (double *)malloc(sizeof(double) * (size_t)(m > n ? m : n));
  if (!row_mean || !col_mean || !tmp) {
    free(row_mean); free(col_mean); free(tmp);
    return LO_ERR_ALLOC;
  }
  for (int64_t a = 0; a < m; a++) {
    for (int64_t b = 0; b < n; b++) {
      double v = (double)g[a * n + b];
      tmp[b] = v * v;
    }
    row_mean[a] = pw_sum(tmp, n) / (double)n;   /* axis=1: contiguous, pairwise */
  }
  if (n == 1) {
    /* an (m,1) array reduced over axis 0 is contiguous: pairwise */
    for (int64_t a = 0; a < m; a++) {
      double v = (double)g[a];
      tmp[a] = v * v;
    }
    col_mean[0] = pw_sum(tmp, m) / (double)m;
  } else {
    /* axis=0 of a C-contiguous matrix: rows accumulated in order */
    for (int64_t a = 0; a < m; a++)
      for (int64_t b = 0; b < n; b++) {
        double v = (double)g[a * n + b];
        col_mean[b] = col_mean[b] + v * v;
      }
    for (int64_t b = 0; b < n; b++) col_mean[b] = col_mean[b] / (double)m;
  }
  for (int k = 0; k < 3; k++) {
    const float b = (float)betas[4 + k];
    const float omb = 1.0f - b;
    for (int64_t a = 0; a < m; a++) {
      float t1 = b * r[k][a];
      float t2 = omb * (float)row_mean[a];
      r[k][a] = t1 + t2;
    }
    for (int64_t j = 0; j < n; j++) {
      float t1 = b * c[k][j];
      float t2 = omb * (float)col_mean[j];
      c[k][j] = t1 + t2;
    }
  }
  free(row_mean); free(col_mean); free(tmp);
  return LO_OK;
}

/* ------------------------------------------------------------------ */
/* features (features.py:147-195, engine.py:313-428)                   */

typedef struct {
  int64_t m, n;
  const float *W, *g, *M[3], *V, *r[3], *c[3];
  float mr[3];
  float tf[11];
  int kind;
} lo_view;

/* Fill feat[0..d_feat) for element (a, b); the expression trees are those
 * of features.py:_gathered_columns, strict f32. */
static void fill_features(const lo_view *s, int64_t a, int64_t b, float *feat) {
  const float eps = EPS_RECIP, one = 1.0f;
  const int64_t i = a * s->n + b;
  const float wv = s->W[i], gv = s->g[i];
  const float m1 = s->M[0][i], m2 = s->M[1][i], m3 = s->M[2][i], v = s->V[i];
  const float rv5 = s->r[0][a], rv6 = s->r[1][a], rv7 = s->r[2][a];
  const float cv5 = s->c[0][b], cv6 = s->c[1][b], cv7 = s->c[2][b];
  const float sv = sqrtf(v + eps);
  feat[0] = m1; feat[1] = m2; feat[2] = m3; feat[3] = v;
  feat[4] = rv5; feat[5] = rv6; feat[6] = rv7;
  feat[7] = cv5; feat[8] = cv6; feat[9] = cv7;
  feat[10] = m1 / sv; feat[11] = m2 / sv; feat[12] = m3 / sv;
  feat[13] = one / sv;
  feat[14] = one / sqrtf(rv5 + eps);
  feat[15] = one / sqrtf(rv6 + eps);
  feat[16] = one / sqrtf(rv7 + eps);
  feat[17] = one / sqrtf(cv5 + eps);
  feat[18] = one / sqrtf(cv6 + eps);
  feat[19] = one / sqrtf(cv7 + eps);
  const float p5 = rv5 * cv5, p6 = rv6 * cv6, p7 = rv7 * cv7;
  const float s5 = sqrtf(s->mr[0] / (p5 + eps));
  const float s6 = sqrtf(s->mr[1] / (p6 + eps));
  const float s7 = sqrtf(s->mr[2] / (p7 + eps));
  feat[20] = gv * s5; feat[21] = gv * s6; feat[22] = gv * s7;
  feat[23] = m1 * s5; feat[24] = m2 * s6; feat[25] = m3 * s7;
  if (s->kind == LO_SMALL_FC_LOPT) {
    for (int k = 0; k < 11; k++) feat[26 + k] = s->tf[k];
    feat[37] = wv;
    feat[38] = gv;
  } else {
    feat[26] = wv;
    feat[27] = gv;
    float cg = gv;
    if (cg > CLIP_BOUND) cg = CLIP_BOUND;
    else if (cg < -CLIP_BOUND) cg = -CLIP_BOUND;
    feat[28] = cg;
  }
}

static void make_view(lo_view *s, int kind, int64_t m, int64_t n, const float *W,
                      const float *g, const float *M0, const float *M1,
                      const float *M2, const float *V, const float *r0,
                      const float *r1, const float *r2, const float *c0,
                      const float *c1, const float *c2, const float *tf) {
  s->kind = kind; s->m = m; s->n = n; s->W = W; s->g = g;
  s->M[0] = M0; s->M[1] = M1; s->M[2] = M2; s->V = V;
  s->r[0] = r0; s->r[1] = r1; s->r[2] = r2;
  s->c[0] = c0; s->c[1] = c1; s->c[2] = c2;
  for (int k = 0; k < 3; k++) s->mr[k] = lo_factor_mean(s->r[k], m);
  for (int k = 0; k < 11; k++) s->tf[k] = tf ? tf[k] : 0.0f;
}

/* features.py:304-315 construct_features_at, for one flat index. */
void lo_features_at(int kind, int64_t m, int64_t n, const float *W, const float *g,
                    const float *M0, const float *M1, const float *M2, const float *V,
                    const float *r0, const float *r1, const float *r2, const float *c0,
                    const float *c1, const float *c2, const float *tf, int64_t idx,
                    float *feat) {
  lo_view s;
  make_view(&s, kind, m, n, W, g, M0, M1, M2, V, r0, r1, r2, c0, c1, c2, tf);
  fill_features(&s, idx / n, idx % n, feat);
}

/* engine.py:597-605 worker_ranges */
static void worker_range(int64_t lo, int64_t hi, int64_t workers, int64_t w,
                         int64_t *wlo, int64_t *whi) {
  const int64_t span = hi - lo;
  *wlo = lo + span * w / workers;
  *whi = lo + span * (w + 1) / workers;
}

/* engine.py:619-654 fused_stats (pass 1): worker-private f64 partials over
 * 64-lane blocks, merged by engine.py:608-616's fixed binary tree. */
static int stats_view(const lo_view *s, int64_t lo, int64_t hi, int64_t workers,
                      double *sumsq) {
  const int d = lo_d_feat(s->kind);
  double *partials = (double *)calloc((size_t)(workers * d), sizeof(double));
  if (!partials) return LO_ERR_ALLOC;
  float featT[LO_MAX_FEAT][LO_LANES];
  float feat[LO_MAX_FEAT];
  const int64_t n = s->n;
  for (int64_t w = 0; w < workers; w++) {
    int64_t i, whi;
    worker_range(lo, hi, workers, w, &i, &whi);
    while (i < whi) {
      const int64_t a = i / n, b0 = i - a * n;
      int64_t nl = LO_LANES;
      if (n - b0 < nl) nl = n - b0;
      if (whi - i < nl) nl = whi - i;
      for (int64_t l = 0; l < nl; l++) {
        fill_features(s, a, b0 + l, feat);
        for (int k = 0; k < d; k++) featT[k][l] = feat[k];
      }
      /* engine.py:431-438 _accum_sq */
      for (int k = 0; k < d; k++) {
        double acc = 0.0;
        for (int64_t l = 0; l < nl; l++) {
          double fv = (double)featT[k][l];
          acc = acc + fv * fv;
        }
        partials[w * d + k] = partials[w * d + k] + acc;
      }
      i += nl;
    }
  }
  /* merge_partials_tree */
  for (int64_t step = 1; step < workers; step *= 2)
    for (int64_t p = 0; p < workers - step; p += 2 * step)
      for (int k = 0; k < d; k++)
        partials[p * d + k] = partials[p * d + k] + partials[(p + step) * d + k];
  for (int k = 0; k < d; k++) sumsq[k] = partials[k];
  free(partials);
  return LO_OK;
}

int lo_fused_stats(int kind, int64_t m, int64_t n, const float *W, const float *g,
                   const float *M0, const float *M1, const float *M2, const float *V,
                   const float *r0, const float *r1, const float *r2, const float *c0,
                   const float *c1, const float *c2, const float *tf, int64_t lo,
                   int64_t hi, int64_t workers, double *sumsq) {
  lo_view s;
  make_view(&s, kind, m, n, W, g, M0, M1, M2, V, r0, r1, r2, c0, c1, c2, tf);
  return stats_view(&s, lo, hi, workers, sumsq);
}

/* features.py:138-140 normalization_scale */
void lo_normalization_scale(int d, const double *sumsq, int64_t count, float *scale) {
  for (int k = 0; k < d; k++)
    scale[k] = (float)(1.0 / sqrt(sumsq[k] / (double)count + EPS_NORM));
}

/* MLP weights of the reference three-layer topology (engine.py:119-163):
 * w1 (H1, d), b1 (H1), w2 (H2, H1), b2 (H2), w3 (2, H2), b3 (2). */
typedef struct {
  int d, h1, h2;
  const float *w1, *b1, *w2, *b2, *w3, *b3;
  float alpha, beta_out;
  int update_sign;
} lo_mlp;

/* engine.py:441-480 _mlp_lanes for one lane: sequential fma chains. */
static void mlp_lane(const lo_mlp *w, const float *w1s, const float *x, float *dir,
                     float *mag) {
  float h1[LO_MAX_HIDDEN], h2[LO_MAX_HIDDEN];
  for (int o = 0; o < w->h1; o++) h1[o] = w->b1[o];
  for (int j = 0; j < w->d; j++)
    for (int o = 0; o < w->h1; o++) h1[o] = fmaf(w1s[o * w->d + j], x[j], h1[o]);
  for (int o = 0; o < w->h1; o++)
    if (h1[o] < 0.0f) h1[o] = 0.0f;
  for (int o = 0; o < w->h2; o++) h2[o] = w->b2[o];
  for (int j = 0; j < w->h1; j++)
    for (int o = 0; o < w->h2; o++) h2[o] = fmaf(w->w2[o * w->h1 + j], h1[j], h2[o]);
  for (int o = 0; o < w->h2; o++)
    if (h2[o] < 0.0f) h2[o] = 0.0f;
  float d = w->b3[0], mg = w->b3[1];
  for (int j = 0; j < w->h2; j++) {
    d = fmaf(w->w3[j], h2[j], d);
    mg = fmaf(w->w3[w->h2 + j], h2[j], mg);
  }
  *dir = d;
  *mag = mg;
}

/* engine.py:441-480 _mlp_lanes over LANES elements at once, as the
 * reference blocks them (64 lanes): every lane's outputs are the same
 * sequential fma chains as mlp_lane (bitwise), but the innermost loop runs
 * across lanes, so the compiler vectorizes it (8 lanes per AVX2 FMA). */
#define LANES 64
static void mlp_lanes(const lo_mlp *w, const float *w1s, const float (*x)[LANES], int nl,
                      float *dir, float *mag) {
  float h1[LO_MAX_HIDDEN][LANES], h2[LO_MAX_HIDDEN][LANES];
  for (int o = 0; o < w->h1; o++)
    for (int l = 0; l < LANES; l++) h1[o][l] = w->b1[o];
  for (int j = 0; j < w->d; j++)
    for (int o = 0; o < w->h1; o++) {
      const float c = w1s[o * w->d + j];
      for (int l = 0; l < LANES; l++) h1[o][l] = fmaf(c, x[j][l], h1[o][l]);
    }
  for (int o = 0; o < w->h1; o++)
    for (int l = 0; l < LANES; l++)
      if (h1[o][l] < 0.0f) h1[o][l] = 0.0f;
  for (int o = 0; o < w->h2; o++)
    for (int l = 0; l < LANES; l++) h2[o][l] = w->b2[o];
  for (int j = 0; j < w->h1; j++)
    for (int o = 0; o < w->h2; o++) {
      const float c = w->w2[o * w->h1 + j];
      for (int l = 0; l < LANES; l++) h2[o][l] = fmaf(c, h1[j][l], h2[o][l]);
    }
  for (int o = 0; o < w->h2; o++)
    for (int l = 0; l < LANES; l++)
      if (h2[o][l] < 0.0f) h2[o][l] = 0.0f;
  float d[LANES], mg[LANES];
  for (int l = 0; l < LANES; l++) {
    d[l] = w->b3[0];
    mg[l] = w->b3[1];
  }
  for (int j = 0; j < w->h2; j++) {
    const float cd = w->w3[j], cm = w->w3[w->h2 + j];
    for (int l = 0; l < LANES; l++) {
      d[l] = fmaf(cd, h2[j][l], d[l]);
      mg[l] = fmaf(cm, h2[j][l], mg[l]);
    }
  }
  for (int l = 0; l < nl; l++) {
    dir[l] = d[l];
    mag[l] = mg[l];
  }
}

/* engine.py:657-710 fused_apply (pass 2) over [lo, hi): writes out, returns
 * max |update| through *maxabs.  Elements go through the MLP 64 at a time. */
static int apply_view(const lo_view *s, const lo_mlp *w, const double *sumsq,
                      int64_t count, float lr, int64_t lo, int64_t hi, float *out,
                      float *maxabs_out) {
  const int d = lo_d_feat(s->kind);
  if (w->d != d || w->h1 > LO_MAX_HIDDEN || w->h2 > LO_MAX_HIDDEN) return LO_ERR_SHAPE;
  float scale[LO_MAX_FEAT];
  lo_normalization_scale(d, sumsq, count, scale);
  float *w1s = (float *)malloc(sizeof(float) * (size_t)(w->h1 * d));
  if (!w1s) return LO_ERR_ALLOC;
  for (int o = 0; o < w->h1; o++)
    for (int j = 0; j < d; j++) w1s[o * d + j] = w->w1[o * d + j] * scale[j];
  const float alpha = w->alpha, beta_out = w->beta_out;
  const float ds = (float)w->update_sign * lr;
  float feat[LO_MAX_FEAT];
  float x[LO_MAX_FEAT][LANES];
  float dir[LANES], mag[LANES];
  float maxabs = 0.0f;
  const int64_t n = s->n;
  for (int64_t i0 = lo; i0 < hi; i0 += LANES) {
    const int nl = (int)(hi - i0 < LANES ? hi - i0 : LANES);
    for (int l = 0; l < LANES; l++) {
      if (l < nl) {
        const int64_t i = i0 + l, a = i / n, b = i - a * n;
        fill_features(s, a, b, feat);
        for (int j = 0; j < d; j++) x[j][l] = feat[j];
      } else {
        for (int j = 0; j < d; j++) x[j][l] = 0.0f;
      }
    }
    mlp_lanes(w, w1s, (const float (*)[LANES])x, nl, dir, mag);
    for (int l = 0; l < nl; l++) {
      const int64_t i = i0 + l;
      const float t = mag[l] * alpha;
      const float e = expf(t);
      const float upd = (dir[l] * e) * beta_out;
      const float du = ds * upd;
      out[i] = s->W[i] + du;
      const float au = fabsf(du);
      if (au > maxabs) maxabs = au;
    }
  }
  free(w1s);
  *maxabs_out = maxabs;
  return LO_OK;
}

int lo_fused_apply(int kind, int64_t m, int64_t n, const float *W, const float *g,
                   const float *M0, const float *M1, const float *M2, const float *V,
                   const float *r0, const float *r1, const float *r2, const float *c0,
                   const float *c1, const float *c2, const float *tf, int h1, int h2,
                   const float *w1, const float *b1, const float *w2, const float *b2,
                   const float *w3, const float *b3, float alpha, float beta_out,
                   int update_sign, const double *sumsq, int64_t count, double lr,
                   int64_t lo, int64_t hi, float *out, float *maxabs) {
  lo_view s;
  make_view(&s, kind, m, n, W, g, M0, M1, M2, V, r0, r1, r2, c0, c1, c2, tf);
  lo_mlp w = {lo_d_feat(kind), h1, h2, w1, b1, w2, b2, w3, b3, alpha, beta_out,
              update_sign};
  return apply_view(&s, &w, sumsq, count, (float)lr, lo, hi, out, maxabs);
}

/* ------------------------------------------------------------------ */
/* multi-tensor facade (optim.py:144-180), used by the CPU baseline      */

typedef struct {
  int64_t m, n;
  float *W;
  const float *g;
  float *M0, *M1, *M2, *V, *r0, *r1, *r2, *c0, *c1, *c2;
  /* per-tensor MLP (the VeLO path may hand each tensor its own weights) */
  const float *w1, *b1, *w2, *b2, *w3, *b3;
} lo_tensor_desc;

/* One opt_step over `count` tensors with constant lr (the caller evaluates
 * schedule_lr(T) and the host time features, exactly as optim.py:156 and
 * features.py:125-130 do).  Tensors are independent, so they are spread over
 * `threads` OpenMP threads, largest first; results do not depend on the
 * thread count.  err_index receives the failing tensor on error. */
int lo_opt_step(int kind, int count, lo_tensor_desc *t, int h1, int h2, float alpha,
                float beta_out, int update_sign, const double *betas, double lr,
                double weight_decay, const float *tf, int64_t workers, int threads,
                int *err_index) {
  /* optim.py:160-165: every gradient is validated before anything changes */
  for (int j = 0; j < count; j++) {
    const int64_t mn = t[j].m * t[j].n;
    for (int64_t i = 0; i < mn; i++)
      if (!isfinite(t[j].g[i])) {
        *err_index = j;
        return LO_ERR_NONFINITE_GRAD;
      }
  }
  int *order = (int *)malloc(sizeof(int) * (size_t)(count > 0 ? count : 1));
  if (!order) return LO_ERR_ALLOC;
  for (int j = 0; j < count; j++) order[j] = j;
  for (int a = 1; a < count; a++) { /* insertion sort, largest first */
    int v = order[a], b = a - 1;
    while (b >= 0 && t[order[b]].m * t[order[b]].n < t[v].m * t[v].n) {
      order[b + 1] = order[b];
      b--;
    }
    order[b + 1] = v;
  }
  const float decay = (float)(1.0 - lr * weight_decay);
  int status = LO_OK;
  int bad = -1;
#ifdef _OPENMP
  if (threads < 1) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
#endif
  for (int q = 0; q < count; q++) {
    const int j = order[q];
    lo_tensor_desc *d = &t[j];
    const int64_t mn = d->m * d->n;
    int st = lo_state_step(d->m, d->n, d->g, d->M0, d->M1, d->M2, d->V, d->r0,
                           d->r1, d->r2, d->c0, d->c1, d->c2, betas);
    lo_view s;
    make_view(&s, kind, d->m, d->n, d->W, d->g, d->M0, d->M1, d->M2, d->V, d->r0,
              d->r1, d->r2, d->c0, d->c1, d->c2, tf);
    double sumsq[LO_MAX_FEAT];
    if (st == LO_OK) st = stats_view(&s, 0, mn, workers, sumsq);
    float maxabs = 0.0f;
    lo_mlp w = {lo_d_feat(kind), h1, h2, d->w1, d->b1, d->w2, d->b2, d->w3, d->b3,
                alpha, beta_out, update_sign};
    /* apply in place: pass 2 reads W[i] only for the element it writes */
    if (st == LO_OK) st = apply_view(&s, &w, sumsq, mn, (float)lr, 0, mn, d->W, &maxabs);
    if (st == LO_OK) {
      for (int64_t i = 0; i < mn; i++)
        if (!isfinite(d->W[i])) { st = LO_ERR_OVERFLOW; break; }
    }
    /* optim.py:171-172 decoupled decay, one f32 multiply after the update */
    if (st == LO_OK && weight_decay > 0.0)
      for (int64_t i = 0; i < mn; i++) d->W[i] = d->W[i] * decay;
    if (st != LO_OK) {
#ifdef _OPENMP
#pragma omp critical
#endif
      {
        if (bad < 0 || j < bad) { bad = j; status = st; }
      }
    }
  }
  free(order);
  if (status != LO_OK) *err_index = bad;
  return status;
}
