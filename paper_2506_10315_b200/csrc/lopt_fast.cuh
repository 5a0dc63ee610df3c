// lopt_fast.cuh -- definitions shared by the fast-mode kernels (lopt_fast.cu,
// lopt_apply_tc.cu): the per-tensor prepared operand image, the A-operand
// column order, and the per-element fast feature arithmetic.
#pragma once

#include "lopt_common.cuh"
#include "lopt_tc.cuh"

#include <cstddef>

namespace lopt {

constexpr int kTile = 128;

// B slices are K=16 x N fp16 in the canonical K-major no-swizzle layout:
// byte (k>>3)*(N*16) + (o>>3)*128 + (o&7)*16 + (k&7)*2 (N = 32 for layer 1,
// kN2 = 48 for layer 2; LBO = N*16 bytes, SBO = 128 bytes).
//
// Operands are fp16 two-term splits, x = x_hi + x_lo (relative residual
// 2^-22), and every product is formed as x_hi*W_hi + x_lo*W_hi + x_hi*W_lo by
// three MMAs that accumulate into the same f32 TMEM columns (the A operand of
// each MMA is just a different TMEM column range, so nothing is duplicated
// and the epilogue reads finished sums).  Layer 1 takes the NORMALIZED
// features x*scale (|x*scale| <= sqrt(m*n) < 65504 because
// sum_e (x*scale)^2 <= m*n), so W1 is used unscaled.  Layer 2 takes
// ReLU(h1) * 2^-s2 with s2 chosen per tensor from a bound on |h1| (s2 = 0 on
// every tensor of the benchmarked models): 2^-s2 is folded into W1 and the
// layer-1 bias (so the MMA emits h1 * 2^-s2), the layer-2 bias is pre-scaled
// by 2^-s2 and 2^s2 is folded into W3.
//
// Layer 3 without a ReLU pass: relu(h) = (h + |h|)/2, so
//   dir = b3 + 1/2 sum_o w3[o] h2[o] + 1/2 sum_o w3[o] |h2[o]|.
// The linear half is linear in relu(h1), so it rides on the layer-2 MMAs as
// two extra output rows v = 1/2 W2^T w3 (bias 1/2 w3.b2 + b3): layer 2 runs with
// N = 48 (rows 32, 33 = dir, mag; 34..47 zero) and the epilogue only forms
// sum (w3/2) |h2| with FFMA2's |x| operand modifier.
//
// A operands (per 128-element tile, TMEM, 2 fp16 per 32-bit column):
//   E_hi/E_lo  16 per-element features in elem_col order
//   B_hi/B_lo  r5 r6 r7 rr5 rr6 rr7 | c5 c6 c7 rc5 rc6 rc7 | clip | 1 | 0 0
//   H_hi/H_lo  32 hidden units of layer 1 (two K slices)
//   ONE        {1, 1, 0, ...}: selects the layer-2 bias slice (b2_hi + b2_lo)
// Layer 1 = 6 MMAs (M=128, N=32, K=16), layer 2 = 7 MMAs (M=128, N=48, K=16).
constexpr int kN2 = 48;     // layer-2 MMA width: 32 hidden + {dir, mag} linear halves + pad
struct __align__(128) PrepImage {
  uint16_t b1[4][512];      // W1 over E: hi, lo; W1 over B: hi, lo
  uint16_t b2[5][kN2 * 16]; // [W2|v]_hi[K0-15], _hi[K16-31], _lo[K0-15], _lo[K16-31], bias
  float w3h[16][4];         // {w3d[2q], w3m[2q], w3d[2q+1], w3m[2q+1]} * 2^s2 / 2
  float escale[20];         // normalization scale of the per-element columns (+ clip), float4-read
  float b3[2];
  float sqmr[3];            // sqrt(mean r_i)
  float s2_down;            // 2^-s2 (already folded into W1)
  float s2_up;              // 2^s2: scales layer 3's |h2| half when w3 comes from the launch
  float pad;
};
static_assert(offsetof(PrepImage, escale) % 16 == 0, "escale is read as float4");
static_assert(sizeof(PrepImage) % 16 == 0, "PrepImage must be 16-byte granular");

// canonical K-major no-swizzle index of (row o, k) in an N-row, K=16 slice
__device__ __forceinline__ int bslot(int o, int k, int N = 32) {
  return ((k >> 3) * (N * 16) + (o >> 3) * 128 + (o & 7) * 16 + (k & 7) * 2) >> 1;
}

// Element-wise column order of the A operand (reference column indices):
// M1 M2 M3 V M1/sv M2/sv M3/sv 1/sv gS5 gS6 gS7 M1S5 M2S6 M3S7 W g
__device__ __forceinline__ int elem_col(int kind, int q) {
  if (q < 4) return q;
  if (q < 8) return 6 + q;           // 10..13
  if (q < 14) return 12 + q;         // 20..25
  return kind == LOPT_SMALL_FC_LOPT ? 23 + q : 12 + q;   // W, g: 37,38 | 26,27
}
// Broadcast slice order: r5 r6 r7 rr5 rr6 rr7 c5 c6 c7 rc5 rc6 rc7 [clip] [bias]
__device__ __forceinline__ int bc_col(int q) {
  if (q < 3) return 4 + q;
  if (q < 6) return 11 + q;          // 14..16
  if (q < 9) return 1 + q;           // 7..9
  return 8 + q;                      // 17..19
}

struct FastIn {
  float w, g, m1, m2, m3, v;
};

// state.py:77-90 recomputed from the old accumulators, bit for bit, so the
// stored state stays exact in fast mode too.
__device__ __forceinline__ void advance(float g, float4 s, bool advanced, const float *beta,
                                        FastIn &x) {
  x.g = g;
  if (advanced) {
    x.m1 = s.x; x.m2 = s.y; x.m3 = s.z; x.v = s.w;
  } else {
    // state.py:77-90 bit for bit: both products rounded, then the sum
    // (packed f32x2 forms were measured to differ in the last bit: ptxas may
    // contract them, so the advance stays scalar with explicit rounding)
    x.m1 = ema(beta[0], __fsub_rn(1.0f, beta[0]), s.x, g);
    x.m2 = ema(beta[1], __fsub_rn(1.0f, beta[1]), s.y, g);
    x.m3 = ema(beta[2], __fsub_rn(1.0f, beta[2]), s.z, g);
    x.v = ema(beta[3], __fsub_rn(1.0f, beta[3]), s.w, __fmul_rn(g, g));
  }
}

// f[0..15] in elem_col order; rc = {r5, r6, r7} of the row, cc = {c5, c6, c7}.
// MUFU rsqrt replaces the correctly rounded div/sqrt of features.py:153-195.
// MUFU rsqrt without the denormal fix-up: every argument is >= 1e-12.
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void fast_features(const FastIn &x, const float *rc, const float *cc,
                                              const float *sqmr, float *f) {
  const float svi = rsqrt_ftz(x.v + kEpsRecip);
  const float2 rc01 = tc::fma2(make_float2(rc[0], rc[1]), make_float2(cc[0], cc[1]),
                               make_float2(kEpsRecip, kEpsRecip));
  const float rc2 = fmaf(rc[2], cc[2], kEpsRecip);
  const float2 s01 = tc::mul2(make_float2(sqmr[0], sqmr[1]),
                              make_float2(rsqrt_ftz(rc01.x), rsqrt_ftz(rc01.y)));
  const float s2 = sqmr[2] * rsqrt_ftz(rc2);
  const float2 m12 = make_float2(x.m1, x.m2);
  const float2 a = tc::mul2(m12, make_float2(svi, svi));
  const float2 b = tc::mul2(make_float2(x.g, x.g), s01);
  const float2 c = tc::mul2(m12, s01);
  f[0] = x.m1; f[1] = x.m2; f[2] = x.m3; f[3] = x.v;
  f[4] = a.x; f[5] = a.y; f[6] = x.m3 * svi; f[7] = svi;
  f[8] = b.x; f[9] = b.y; f[10] = x.g * s2;
  f[11] = c.x; f[12] = c.y; f[13] = x.m3 * s2;
  f[14] = x.w; f[15] = x.g;
}

__device__ __forceinline__ float clip01(float g) { return fminf(fmaxf(g, -kClip), kClip); }

// e = a*n + b for e < 2^53: one DMUL by the reciprocal and a +-1 correction.
__device__ __forceinline__ void divmod(int64_t e, int64_t n, double inv_n, int64_t &a, int64_t &b) {
  a = (int64_t)((double)e * inv_n);
  b = e - a * n;
  if (b < 0) {
    a--;
    b += n;
  } else if (b >= n) {
    a++;
    b -= n;
  }
}

}  // namespace lopt
