// lopt_common.cuh -- shared device definitions for the B200 learned-optimizer
// step: descriptor tables, work items, strict-IEEE feature arithmetic, the
// reference MLP as fma chains, and the glibc expf algorithm restated for the
// device.  Reference paths are relative to pkg/src/lopt/ of the reference.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/lopt_b200.h"

namespace lopt {

constexpr int kTimeFeatures = 11;
constexpr int kMaxFeat = 39;
constexpr int kMaxHidden = 32;        // compiled MLP width (reference optimizers use 32)
constexpr float kEpsRecip = 1e-12f;   // features.py:66
constexpr double kEpsNorm = 1e-5;     // features.py:67
constexpr float kClip = 0.1f;         // features.py:82
// row/col table entry (16 x 32-bit): f32 {x5, x6, x7, rsqrt(x5+eps) | rsqrt(x6+eps),
// rsqrt(x7+eps), 0, 0} then, for the fast path, the six values split into bf16
// hi/lo pairs {hi01, hi23, hi45, 0 | lo01, lo23, lo45, 0}
constexpr int kRowTab = 16;
constexpr int kWarpColumnBlocks = 32;   // factor reduce: warp-per-column threshold
constexpr int kMaxApplyCtas = 256;   // pair-kernel CTAs with a balance record

__host__ __device__ constexpr int d_feat(int kind) { return kind == LOPT_SMALL_FC_LOPT ? 39 : 29; }

// Device-side descriptor of one tensor (built by the host plan).
struct TensorDesc {
  float *theta;
  const float *grad;
  float4 *state;          // {M1, M2, M3, V} per element of [lo, hi)
  float *r;               // 3 x m  (r5 | r6 | r7)
  float *c;               // 3 x n
  int64_t m, n, lo, hi;
  // workspace views
  double *rowsum;         // [m]  sum over the call's elements of g^2, per row
  double *colsum;         // [n]
  double *rowpart;        // [nstrips x m] phase-0 partials
  double *colpart;        // [nrowblocks x n]
  float *rowtab;          // [m x 8] advanced r and 1/sqrt(r+eps)
  float *coltab;          // [n x 8]
  double *sumsq;          // [d_feat]
  int32_t nstrips, nrowblocks;
  int32_t weight_slot;
  int32_t stat_item0, stat_items;   // phase-1 items of this tensor (contiguous)
  int32_t apply_item0, apply_items; // phase-2 items of this tensor (contiguous)
  int32_t tiles;          // fast path: 128-lane tiles of this tensor
  int64_t tile0;          // fast path: first tile of this tensor in the plan
  // fast path tile shape: rowblock = 1 when n % 128 == 0; then tile q is row
  // a_lo + q % m_rows, columns [128 * (q / m_rows), +128) (column-block major,
  // so a run of tiles shares its column-table entries); otherwise tile q is
  // the flat elements [lo + 128 q, +128)
  int32_t rowblock, a_lo, m_rows;
  // pair kernel: tile pairs of this tensor and its first pair in the plan
  // (rowblock: rows 2r, 2r+1 of one column block; flat: tiles 2q, 2q+1; a
  // missing second tile is an empty tile)
  int32_t pairs;
  int64_t pair0;
  // element count behind the tensor's feature statistics for the apply
  // pass's normalization (features.py:138-140); 0 = the whole tensor, m * n
  int64_t stat_count;
};

// Phase-0 tile: rows [a0, a1) x columns [b0, b1) of one tensor.
struct FactorItem {
  int32_t tensor, strip, rowblock, pad_;
  int64_t a0, a1, b0, b1;
};

// Phase-1/2 chunk: flat elements [e0, e1) of one tensor, e0 >= lo, e1 <= hi.
// Fast-mode stats also use column strips (strip = 1): rows [e0 >> 32, e1 >> 32)
// x columns [e0 & 0xffffffff, e1 & 0xffffffff) of a tensor whose rows in that
// range lie entirely inside [lo, hi).
struct ChunkItem {
  int32_t tensor, strip;
  int64_t e0, e1;
};

// Per-step scalars, read by the kernels from device memory so a captured
// CUDA graph stays valid across steps.
struct StepScalars {
  float tf[kTimeFeatures];
  float lr_f32;           // f32(lr)
  float ds;               // f32(update_sign) * f32(lr)   (engine.py:695)
  float decay;            // f32(1 - lr * weight_decay)    (optim.py:100)
  int32_t apply_decay;    // weight_decay > 0               (optim.py:171)
  int32_t t;
  float loss[2];          // VeLO hypernetwork loss features (lopt_step_args.loss_features)
};

// Per-tensor device scalars produced on the device during the step.
struct TensorScalars {
  float mr[3];            // factor means of the advanced row factors
  float pad_;
};

struct DevicePlan {
  TensorDesc *tensors;
  FactorItem *factor_items;
  ChunkItem *stat_items;
  ChunkItem *apply_items;
  double *stat_part;      // [n_stat_items x d_feat]
  TensorScalars *tscal;
  StepScalars *step;
  const float *weights;   // [num_sets x weight_stride]
  uint32_t *status;       // [count]
  float *maxabs;          // [count]
  float *item_maxabs;     // [n_apply_items]
  uint32_t *abort_flag;   // any non-finite gradient in this step
  double *grad_flag;      // last slot of the factor-sum block: > 0 if any rank saw a
                          // non-finite gradient (all-reduced with the sums)
  int32_t count, n_factor_items, n_stat_items, n_apply_items;
  int32_t kind, mode, h1, h2;
  int32_t weight_stride, state_advanced;
  float beta[7];          // f32(beta) as the reference casts them (state.py:81)
  float alpha, beta_out;
  // fast path
  int64_t n_tiles;        // 128-element tiles over all tensors
  int64_t n_pairs;        // tile pairs over all tensors (pair kernel)
  // pair-kernel balance: CTA b steps pairs [pair_range[b], pair_range[b + 1]);
  // cta_perf[b] = {pairs, busy ns} of its last launch, from which prep
  // computes the next ranges (SMs differ in speed)
  int32_t *pair_range;    // [kMaxApplyCtas + 1]
  int64_t *cta_perf;      // [kMaxApplyCtas x 2], then [kMaxApplyCtas] f64 smoothed speeds
  int32_t apply_grid;     // pair-kernel CTAs (min(SMs, n_pairs))
  int32_t w3c_on;         // w3c holds the plan's one weight set's layer 3
  // layer 3 of a single-weight-set plan as a launch parameter, laid out like
  // PrepImage::w3h without the per-tensor 2^s2: the pair kernel's FFMA2s
  // take it from uniform registers instead of shared memory
  float w3c[16][4];
  unsigned char *prep;    // per-tensor PrepImage (B operands, layer-3 weights)
  double *bcsum;          // [count x d_feat] closed-form sums of broadcast features
  int32_t dbg, n_peers;   // dbg: timing experiments only (LOPT_APPLY_DEBUG), 0 in production
  int32_t peer_bulk, pad_peer;
  // flattened per-tensor work of the factor reduce / finalize kernels: tensor
  // j owns [red_prefix[j], red_prefix[j + 1]) = roundup(m, 32) rows then one
  // 32-thread warp per column, and [fin_prefix[j], fin_prefix[j + 1]) = m + n
  // (columns of tensors with more than kWarpColumnBlocks row blocks take a
  // warp each in the reduce, the others one thread)
  const int64_t *red_prefix, *fin_prefix;
  int64_t red_total, fin_total;   // every peer delta is 16-byte aligned: vector peer stores allowed
  int64_t peer_delta[LOPT_MAX_PEERS];   // fused all-gather: byte offsets of the peer copies
};

__host__ __device__ inline int weight_stride(int d, int h1, int h2) {
  return h1 * d + h1 + h2 * h1 + h2 + 2 * h2 + 2;
}

// ---------------------------------------------------------------------------
// glibc expf, restated for the device.
//
// numba lowers np.exp on float32 to libm expf (engine.py:537); on x86-64 with
// FMA, glibc 2.39 resolves it to the FMA build of the exp2f-table algorithm
// (32-entry table of 2^(i/32), degree-3 polynomial, double arithmetic).  The
// sequence below reproduces that build bit for bit on every float input; the
// check is tests/test_expf_port.py (exhaustive over all 2^32 inputs on the host
// build of the same arithmetic, see oracle/expf_check.c).
struct ExpTable {
  uint64_t t[32];
};

__device__ __forceinline__ float glibc_expf(float x, const uint64_t *tab) {
  const double kInvLn2N = 0x1.71547652b82fep+0 * 32;
  const double kShift = 0x1.8p+52;
  const double C0 = 0x1.c6af84b912394p-5 / 32 / 32 / 32;
  const double C1 = 0x1.ebfce50fac4f3p-3 / 32 / 32;
  const double C2 = 0x1.62e42ff0c52d6p-1 / 32;
  const uint32_t ux = __float_as_uint(x);
  const uint32_t abstop = (ux >> 20) & 0x7ffu;
  if (abstop >= 0x42bu) {                       // |x| >= 88 or nan
    if (ux == 0xff800000u) return 0.0f;         // -inf
    if (abstop >= 0x7f8u) return x + x;         // inf or nan
    if (x > 0x1.62e42ep6f) return __int_as_float(0x7f800000);
    if (x < -0x1.9fe368p6f) return 0.0f;
  }
  const double xd = (double)x;
  const double z = __dmul_rn(kInvLn2N, xd);
  double kd = __dadd_rn(z, kShift);
  const uint64_t ki = (uint64_t)__double_as_longlong(kd);
  kd = __dsub_rn(kd, kShift);
  const double r = __fma_rn(kInvLn2N, xd, -kd);
  uint64_t t = tab[ki & 31u];
  t += ki << 47;
  const double s = __longlong_as_double((long long)t);
  const double zz = __fma_rn(C0, r, C1);
  const double r2 = __dmul_rn(r, r);
  double y = __fma_rn(C2, r, 1.0);
  y = __fma_rn(zz, r2, y);
  y = __dmul_rn(y, s);
  return __double2float_rn(y);
}

// 2^(i/32) as doubles with the exponent bias folded (i << 47) subtracted.
__device__ __constant__ static const uint64_t kExp2Tab[32] = {
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL};

// ---------------------------------------------------------------------------
// strict f32 helpers (no contraction: every op is an explicit _rn intrinsic)

__device__ __forceinline__ float ema(float b, float omb, float prev, float x) {
  // state.py:81-82: b*prev + (1-b)*x, each product rounded, then the add
  return __fadd_rn(__fmul_rn(b, prev), __fmul_rn(omb, x));
}

__device__ __forceinline__ float rsqrt_strict(float x) {
  // one / np.sqrt(x + eps): sqrt then division, both correctly rounded
  return __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(x, kEpsRecip)));
}

// Per-element raw inputs after the accumulator advance.
struct Elem {
  float w, g, m1, m2, m3, v;
};

// features.py:147-195 / engine.py:313-428 for one element, strict.
// rowt/colt: {x5, x6, x7, rsqrt5, rsqrt6, rsqrt7} of the advanced factors.
template <int KIND>
__device__ __forceinline__ void strict_features(const Elem &e, const float *rowt, const float *colt,
                                                const float mr[3], const float *tf, float *f) {
  const float sv = __fsqrt_rn(__fadd_rn(e.v, kEpsRecip));
  f[0] = e.m1; f[1] = e.m2; f[2] = e.m3; f[3] = e.v;
  f[4] = rowt[0]; f[5] = rowt[1]; f[6] = rowt[2];
  f[7] = colt[0]; f[8] = colt[1]; f[9] = colt[2];
  f[10] = __fdiv_rn(e.m1, sv); f[11] = __fdiv_rn(e.m2, sv); f[12] = __fdiv_rn(e.m3, sv);
  f[13] = __fdiv_rn(1.0f, sv);
  f[14] = rowt[3]; f[15] = rowt[4]; f[16] = rowt[5];
  f[17] = colt[3]; f[18] = colt[4]; f[19] = colt[5];
  float s[3];
#pragma unroll
  for (int i = 0; i < 3; i++)
    s[i] = __fsqrt_rn(__fdiv_rn(mr[i], __fadd_rn(__fmul_rn(rowt[i], colt[i]), kEpsRecip)));
  f[20] = __fmul_rn(e.g, s[0]); f[21] = __fmul_rn(e.g, s[1]); f[22] = __fmul_rn(e.g, s[2]);
  f[23] = __fmul_rn(e.m1, s[0]); f[24] = __fmul_rn(e.m2, s[1]); f[25] = __fmul_rn(e.m3, s[2]);
  if (KIND == LOPT_SMALL_FC_LOPT) {
#pragma unroll
    for (int k = 0; k < kTimeFeatures; k++) f[26 + k] = tf[k];
    f[37] = e.w;
    f[38] = e.g;
  } else {
    f[26] = e.w;
    f[27] = e.g;
    float cg = e.g;
    if (cg > kClip) cg = kClip;
    else if (cg < -kClip) cg = -kClip;
    f[28] = cg;
  }
}

// ---------------------------------------------------------------------------
// block helpers

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace lopt
