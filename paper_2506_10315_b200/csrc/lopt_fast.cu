// lopt_fast.cu -- phases 1 and 2 in fast mode: the product path.
//
// Same pipeline as strict mode (engine.py:619-710 fused_stats/fused_apply,
// with the accumulator advance of state.py:77-90 fused in), re-planned for
// B200:
//
//  * features use MUFU rsqrt instead of correctly rounded div/sqrt, and only
//    the 16 (VeLO: 17) per-element columns are reduced per element; the 12
//    row/column-broadcast columns have closed-form sums (lopt_factors.cu) and
//    the 11 time columns are folded into the layer-1 bias;
//  * the two 32-wide MLP layers run on the 5th-generation tensor cores
//    (tcgen05.mma kind::f16, M=128 elements x N=32 hidden units, f32
//    accumulators in TMEM).  fp32 accuracy comes from a two-term bf16 split of
//    both operands (x = x_hi + x_lo, W = W_hi + W_lo; x_hi*W_hi + x_hi*W_lo +
//    x_lo*W_hi, error ~2^-16 relative), so the A operands are written straight
//    from registers into TMEM (tcgen05.st) and never touch shared memory;
//  * layer 3 (32 -> 2), the exp and the update stay on CUDA cores in f32, the
//    exp is the bit-exact glibc expf (lopt_common.cuh).
//
// The apply kernel is persistent: one CTA per SM with three independent
// 128-thread warpgroups, each streaming its own contiguous range of 128-element
// tiles, so one warpgroup's tensor-core latency is covered by the others'
// CUDA-core work.  Per-tensor B operands (normalization scale folded into W1,
// split, laid out in the canonical no-swizzle K-major UMMA layout) are built
// once per step by prep_kernel and copied into a warpgroup's shared memory
// when its tile stream enters a new tensor.
#include "lopt_common.cuh"
#include "lopt_tc.cuh"

namespace lopt {

constexpr int kFastStatThreads = 256;
constexpr int64_t kFastStatChunk = 8192;
constexpr int kTile = 128;
constexpr int kWGs = 3;
constexpr int kApplyThreads = 128 * kWGs;
constexpr uint32_t kTmemCols = 512;

// ---------------------------------------------------------------------------
// per-tensor prepared operands

// B slices are K=16 x N=32 bf16 in the canonical K-major no-swizzle layout:
// byte (k>>3)*512 + (o>>3)*128 + (o&7)*16 + (k&7)*2.
struct __align__(128) PrepImage {
  uint16_t b1[4][512];      // layer 1: We_hi, We_lo, Wbc_hi(+bias_hi), Wbc_lo(+bias_lo)
  uint16_t b2[5][512];      // layer 2: W2_hi[K0-15], W2_hi[K16-31], W2_lo x2, bias
  float w3[2][32];          // layer 3, f32
  float b3[2];
  float sqmr[3];            // sqrt(mean r_i)
  float pad[27];
};
static_assert(sizeof(PrepImage) % 16 == 0, "PrepImage must be 16-byte granular");

__device__ __forceinline__ int bslot(int o, int k) {
  return ((k >> 3) * 512 + (o >> 3) * 128 + (o & 7) * 16 + (k & 7) * 2) >> 1;
}

// Element-wise column order of the A operand (reference column indices):
// M1 M2 M3 V M1/sv M2/sv M3/sv 1/sv gS5 gS6 gS7 M1S5 M2S6 M3S7 W g
__device__ __forceinline__ int elem_col(int kind, int q) {
  const int base[14] = {0, 1, 2, 3, 10, 11, 12, 13, 20, 21, 22, 23, 24, 25};
  if (q < 14) return base[q];
  return kind == LOPT_SMALL_FC_LOPT ? 37 + (q - 14) : 26 + (q - 14);
}
// Broadcast slice order: r5 r6 r7 rr5 rr6 rr7 c5 c6 c7 rc5 rc6 rc7 [clip] [bias]
__device__ __forceinline__ int bc_col(int q) {
  const int c[12] = {4, 5, 6, 14, 15, 16, 7, 8, 9, 17, 18, 19};
  return c[q];
}

__device__ __forceinline__ uint16_t bf16_bits(float x) {
  return (uint16_t)(tc::pack_bf16x2(x, 0.0f) & 0xFFFFu);
}
__device__ __forceinline__ void split1(float x, uint16_t &hi, uint16_t &lo) {
  const uint32_t h = tc::pack_bf16x2(x, 0.0f) & 0xFFFFu;
  hi = (uint16_t)h;
  lo = bf16_bits(x - __uint_as_float(h << 16));
}

// One CTA per tensor: normalization scale, W1s = W1 * scale (engine.py:686),
// time columns folded into the bias, bf16 two-term split, canonical layout.
template <int KIND>
__global__ void __launch_bounds__(256) prep_kernel(DevicePlan P) {
  constexpr int D = d_feat(KIND);
  const int j = blockIdx.x;
  const TensorDesc T = P.tensors[j];
  PrepImage *img = reinterpret_cast<PrepImage *>(P.prep) + j;
  const float *wp = P.weights + (int64_t)T.weight_slot * P.weight_stride;
  const float *w1 = wp, *b1 = w1 + 32 * D, *w2 = b1 + 32, *b2 = w2 + 32 * 32, *w3 = b2 + 32,
              *b3 = w3 + 64;
  __shared__ float scale[kMaxFeat];
  __shared__ float w1s[32][kMaxFeat + 1];
  __shared__ float bias1[32];
  const int64_t count = T.m * T.n;
  for (int k = threadIdx.x; k < D; k += blockDim.x)
    scale[k] = (float)(1.0 / sqrt(T.sumsq[k] / (double)count + kEpsNorm));
  __syncthreads();
  for (int i = threadIdx.x; i < 32 * D; i += blockDim.x)
    w1s[i / D][i % D] = __fmul_rn(w1[i], scale[i % D]);
  __syncthreads();
  if (threadIdx.x < 32) {
    const int o = threadIdx.x;
    float b = b1[o];
    if (KIND == LOPT_SMALL_FC_LOPT) {
#pragma unroll
      for (int k = 0; k < kTimeFeatures; k++) b = __fmaf_rn(w1s[o][26 + k], P.step->tf[k], b);
    }
    bias1[o] = b;
  }
  __syncthreads();
  // layer 1 slices
  for (int i = threadIdx.x; i < 32 * 16; i += blockDim.x) {
    const int o = i >> 4, k = i & 15;
    uint16_t hi, lo;
    split1(w1s[o][elem_col(KIND, k)], hi, lo);
    img->b1[0][bslot(o, k)] = hi;
    img->b1[1][bslot(o, k)] = lo;
    float v = 0.0f;
    if (k < 12) v = w1s[o][bc_col(k)];
    else if (k == 12) v = (KIND == LOPT_VELO_MLP) ? w1s[o][28] : 0.0f;
    else if (k == 13) v = bias1[o];
    split1(v, hi, lo);
    img->b1[2][bslot(o, k)] = hi;
    img->b1[3][bslot(o, k)] = lo;
  }
  // layer 2 slices
  for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) {
    const int o = i >> 5, k = i & 31;
    uint16_t hi, lo;
    split1(w2[o * 32 + k], hi, lo);
    img->b2[k >> 4][bslot(o, k & 15)] = hi;
    img->b2[2 + (k >> 4)][bslot(o, k & 15)] = lo;
  }
  for (int i = threadIdx.x; i < 32 * 16; i += blockDim.x) {
    const int o = i >> 4, k = i & 15;
    uint16_t hi, lo;
    split1(b2[o], hi, lo);
    img->b2[4][bslot(o, k)] = k == 0 ? hi : (k == 1 ? lo : (uint16_t)0);
  }
  if (threadIdx.x < 64) img->w3[threadIdx.x >> 5][threadIdx.x & 31] = w3[threadIdx.x];
  if (threadIdx.x < 2) img->b3[threadIdx.x] = b3[threadIdx.x];
  if (threadIdx.x < 3) img->sqmr[threadIdx.x] = sqrtf(P.tscal[j].mr[threadIdx.x]);
}

// ---------------------------------------------------------------------------
// per-element fast features

struct FastIn {
  float w, g, m1, m2, m3, v;
};

__device__ __forceinline__ void load_fast(const TensorDesc &T, int64_t e, bool advanced,
                                          const float *beta, FastIn &x, float4 &ns) {
  x.w = __ldg(T.theta + e);
  x.g = __ldg(T.grad + e);
  const float4 s = T.state[e - T.lo];
  if (advanced) {
    x.m1 = s.x; x.m2 = s.y; x.m3 = s.z; x.v = s.w;
  } else {
    // state.py:77-90 bit for bit (the stored accumulators stay exact)
    x.m1 = ema(beta[0], __fsub_rn(1.0f, beta[0]), s.x, x.g);
    x.m2 = ema(beta[1], __fsub_rn(1.0f, beta[1]), s.y, x.g);
    x.m3 = ema(beta[2], __fsub_rn(1.0f, beta[2]), s.z, x.g);
    x.v = ema(beta[3], __fsub_rn(1.0f, beta[3]), s.w, __fmul_rn(x.g, x.g));
  }
  ns = make_float4(x.m1, x.m2, x.m3, x.v);
}

// f[0..15] in elem_col order; rc = {r5, r6, r7} of the row, cc = {c5, c6, c7}.
__device__ __forceinline__ void fast_features(const FastIn &x, const float *rc, const float *cc,
                                              const float *sqmr, float *f) {
  const float svi = rsqrtf(x.v + kEpsRecip);
  float s[3];
#pragma unroll
  for (int i = 0; i < 3; i++) s[i] = sqmr[i] * rsqrtf(fmaf(rc[i], cc[i], kEpsRecip));
  f[0] = x.m1; f[1] = x.m2; f[2] = x.m3; f[3] = x.v;
  f[4] = x.m1 * svi; f[5] = x.m2 * svi; f[6] = x.m3 * svi; f[7] = svi;
  f[8] = x.g * s[0]; f[9] = x.g * s[1]; f[10] = x.g * s[2];
  f[11] = x.m1 * s[0]; f[12] = x.m2 * s[1]; f[13] = x.m3 * s[2];
  f[14] = x.w; f[15] = x.g;
}

// e = a*n + b for e < 2^53: one DMUL by the reciprocal and a +-1 correction.
__device__ __forceinline__ void divmod(int64_t e, int64_t n, double inv_n, int64_t &a, int64_t &b) {
  a = (int64_t)((double)e * inv_n);
  b = e - a * n;
  if (b < 0) { a--; b += n; }
  else if (b >= n) { a++; b -= n; }
}

__device__ __forceinline__ float clip01(float g) { return fminf(fmaxf(g, -kClip), kClip); }

// ---------------------------------------------------------------------------
// phase 1: per-element column sums of squares

template <int KIND>
__global__ void __launch_bounds__(kFastStatThreads) stats_fast_kernel(DevicePlan P) {
  constexpr int D = d_feat(KIND);
  constexpr int NE = KIND == LOPT_VELO_MLP ? 17 : 16;
  const ChunkItem it = P.stat_items[blockIdx.x];
  const TensorDesc T = P.tensors[it.tensor];
  const TensorScalars ts = P.tscal[it.tensor];
  const float sqmr[3] = {sqrtf(ts.mr[0]), sqrtf(ts.mr[1]), sqrtf(ts.mr[2])};
  const double inv_n = 1.0 / (double)T.n;
  __shared__ double red[kFastStatThreads / 32][NE];
  float acc[NE];
#pragma unroll
  for (int k = 0; k < NE; k++) acc[k] = 0.0f;
  const bool adv = P.state_advanced != 0;
  for (int64_t e = it.e0 + threadIdx.x; e < it.e1; e += kFastStatThreads) {
    FastIn x;
    float4 ns;
    load_fast(T, e, adv, P.beta, x, ns);
    int64_t a, b;
    divmod(e, T.n, inv_n, a, b);
    const float4 rt = reinterpret_cast<const float4 *>(T.rowtab + a * kRowTab)[0];
    const float4 ct = reinterpret_cast<const float4 *>(T.coltab + b * kRowTab)[0];
    const float rc[3] = {rt.x, rt.y, rt.z}, cc[3] = {ct.x, ct.y, ct.z};
    float f[16];
    fast_features(x, rc, cc, sqmr, f);
#pragma unroll
    for (int k = 0; k < 16; k++) acc[k] = fmaf(f[k], f[k], acc[k]);
    if (KIND == LOPT_VELO_MLP) {
      const float cg = clip01(x.g);
      acc[NE - 1] = fmaf(cg, cg, acc[NE - 1]);
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NE; k++) {
    const double s = warp_sum((double)acc[k]);
    if (lane == 0) red[warp][k] = s;
  }
  __syncthreads();
  double *out = P.stat_part + (int64_t)blockIdx.x * D;
  for (int c = threadIdx.x; c < D; c += blockDim.x) out[c] = 0.0;
  __syncthreads();
  if (threadIdx.x < NE) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kFastStatThreads / 32; w++) s += red[w][threadIdx.x];
    const int col = threadIdx.x < 16 ? elem_col(KIND, threadIdx.x) : 28;
    out[col] = s;
  }
}

// Per-tensor sums: item partials (fixed order) + broadcast closed forms +
// time columns (count * tf^2).  Writes the all-reducible sumsq block.
__global__ void stats_reduce_fast_kernel(DevicePlan P) {
  const int j = blockIdx.x;
  const TensorDesc T = P.tensors[j];
  const int D = d_feat(P.kind);
  for (int k = threadIdx.x; k < D; k += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < T.stat_items; i++) s += P.stat_part[(int64_t)(T.stat_item0 + i) * D + k];
    s += P.bcsum[(int64_t)j * D + k];
    if (P.kind == LOPT_SMALL_FC_LOPT && k >= 26 && k < 37) {
      const double tf = (double)P.step->tf[k - 26];
      s += (double)(T.hi - T.lo) * tf * tf;
    }
    T.sumsq[k] = s;
  }
}

// ---------------------------------------------------------------------------
// phase 2: the tensor-core apply kernel

struct __align__(16) ApplySmem {
  PrepImage img[kWGs];
  uint64_t exptab[32];
  uint64_t bar_acc1[kWGs];
  uint64_t bar_acc2[kWGs];
  uint32_t tmem_base;
};

__device__ __forceinline__ uint32_t bf16_one_pair() { return 0x3F803F80u; }

template <int KIND>
__global__ void __launch_bounds__(kApplyThreads, 1) apply_fast_kernel(DevicePlan P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  ApplySmem &S = *reinterpret_cast<ApplySmem *>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, wg = warp >> 2, row = tid & 127;
  if (warp == 0) {
    tc::tmem_alloc(&S.tmem_base, kTmemCols);
    tc::tmem_relinquish();
  }
  if (tid < 32) S.exptab[tid] = kExp2Tab[tid];
  if (tid == 0) {
    for (int g = 0; g < kWGs; g++) {
      tc::mbar_init(&S.bar_acc1[g], 1);
      tc::mbar_init(&S.bar_acc2[g], 1);
    }
    tc::mbar_fence_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = S.tmem_base;
  const uint32_t lane_addr = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t cA1 = 96 * wg, cACC1 = 96 * wg + 32, cA2 = 96 * wg + 64, cONES = 288;
  // constant "ones" A slice for the layer-2 bias: K0 = K1 = 1
  if (wg == 0) {
    uint32_t r[16];
#pragma unroll
    for (int q = 0; q < 16; q++) r[q] = q == 0 ? bf16_one_pair() : 0u;
    tc::tmem_st16(tbase + lane_addr + cONES, r);
    tc::tmem_st_wait();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();

  const bool adv = P.state_advanced != 0;
  const float alpha = P.alpha, beta_out = P.beta_out;
  const float ds = P.step->ds, decay = P.step->decay;
  const bool apply_decay = P.step->apply_decay != 0;
  const bool aborted = *P.abort_flag != 0;
  constexpr uint32_t kIdesc = tc::idesc_bf16_f32(128, 32);
  PrepImage &img = S.img[wg];

  // contiguous tile range of this warpgroup
  const int64_t nwg = (int64_t)gridDim.x * kWGs;
  const int64_t gwg = (int64_t)blockIdx.x * kWGs + wg;
  const int64_t t_begin = P.n_tiles * gwg / nwg, t_end = P.n_tiles * (gwg + 1) / nwg;
  int cur = -1;
  int j = 0;
  uint32_t phase = 0;
  float maxabs = 0.0f;
  uint32_t bad = 0;
  TensorDesc T;
  double inv_n = 1.0;
  for (int64_t t = t_begin; t < t_end && !aborted; t++) {
    while (j + 1 < P.count && P.tensors[j + 1].tile0 <= t) j++;
    if (j != cur) {
      // flush the previous tensor's statistics, then load this tensor's operands
      if (cur >= 0) {
        if (maxabs > 0.0f) atomicMax(reinterpret_cast<unsigned int *>(&P.maxabs[cur]),
                                     __float_as_uint(maxabs));
        if (bad) atomicOr(&P.status[cur], LOPT_STATUS_NONFINITE_PARAM);
        maxabs = 0.0f;
        bad = 0;
      }
      // the previous tile's MMAs have completed (its acc2 wait), so the B
      // buffer is free once every thread of the warpgroup is here
      tc::bar_sync(1 + wg, 128);
      const uint4 *src = reinterpret_cast<const uint4 *>(reinterpret_cast<PrepImage *>(P.prep) + j);
      uint4 *dst = reinterpret_cast<uint4 *>(&img);
      for (int i = row; i < (int)(sizeof(PrepImage) / 16); i += 128) dst[i] = src[i];
      tc::fence_proxy_async_smem();
      tc::bar_sync(1 + wg, 128);
      cur = j;
      T = P.tensors[j];
      inv_n = 1.0 / (double)T.n;
    }
    const int64_t e = T.lo + (t - T.tile0) * kTile + row;
    const bool valid = e < T.hi;
    // ---- features -> A1 (TMEM) ----
    FastIn x{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float4 ns = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t a1[32];
    if (valid) {
      load_fast(T, e, adv, P.beta, x, ns);
      int64_t a, b;
      divmod(e, T.n, inv_n, a, b);
      const uint4 *rt = reinterpret_cast<const uint4 *>(T.rowtab + a * kRowTab);
      const uint4 *ct = reinterpret_cast<const uint4 *>(T.coltab + b * kRowTab);
      const uint4 r0 = rt[0], rh = rt[2], rl = rt[3];
      const uint4 c0 = ct[0], ch = ct[2], cl = ct[3];
      const float rc[3] = {__uint_as_float(r0.x), __uint_as_float(r0.y), __uint_as_float(r0.z)};
      const float cc[3] = {__uint_as_float(c0.x), __uint_as_float(c0.y), __uint_as_float(c0.z)};
      float f[16];
      fast_features(x, rc, cc, img.sqmr, f);
#pragma unroll
      for (int q = 0; q < 8; q++) tc::split_pair(f[2 * q], f[2 * q + 1], a1[q], a1[8 + q]);
      uint32_t xh = 0, xl = 0;
      if (KIND == LOPT_VELO_MLP) tc::split_pair(clip01(x.g), 0.0f, xh, xl);
      a1[16] = rh.x; a1[17] = rh.y; a1[18] = rh.z;
      a1[19] = ch.x; a1[20] = ch.y; a1[21] = ch.z;
      a1[22] = (xh & 0xFFFFu) | 0x3F800000u;   // K12 = clip hi, K13 = 1 (bias)
      a1[23] = 0u;
      a1[24] = rl.x; a1[25] = rl.y; a1[26] = rl.z;
      a1[27] = cl.x; a1[28] = cl.y; a1[29] = cl.z;
      a1[30] = xl & 0xFFFFu;
      a1[31] = 0u;
    } else {
#pragma unroll
      for (int q = 0; q < 32; q++) a1[q] = 0u;
    }
    tc::tmem_st32(tbase + lane_addr + cA1, a1);
    tc::tmem_st_wait();
    tc::fence_before_sync();
    tc::bar_sync(1 + wg, 128);
    if (row == 0) {
      tc::fence_after_sync();
      const uint32_t d = tbase + cACC1, a = tbase + cA1;
      const uint32_t b0 = tc::smem_u32(img.b1[0]), b1 = tc::smem_u32(img.b1[1]);
      const uint32_t b2 = tc::smem_u32(img.b1[2]), b3 = tc::smem_u32(img.b1[3]);
      tc::mma_ts(d, a + 0, tc::smem_desc_kmajor(b0, 512, 128), kIdesc, 0);   // f_hi  W_hi
      tc::mma_ts(d, a + 0, tc::smem_desc_kmajor(b1, 512, 128), kIdesc, 1);   // f_hi  W_lo
      tc::mma_ts(d, a + 8, tc::smem_desc_kmajor(b0, 512, 128), kIdesc, 1);   // f_lo  W_hi
      tc::mma_ts(d, a + 16, tc::smem_desc_kmajor(b2, 512, 128), kIdesc, 1);  // bc_hi Wbc_hi + bias_hi
      tc::mma_ts(d, a + 16, tc::smem_desc_kmajor(b3, 512, 128), kIdesc, 1);  // bc_hi Wbc_lo + bias_lo
      tc::mma_ts(d, a + 24, tc::smem_desc_kmajor(b2, 512, 128), kIdesc, 1);  // bc_lo Wbc_hi
      tc::mma_commit(&S.bar_acc1[wg]);
    }
    tc::mbar_wait(&S.bar_acc1[wg], phase);
    tc::fence_after_sync();
    // ---- layer-1 epilogue: ReLU + split -> A2 (TMEM) ----
    {
      uint32_t h[32];
      tc::tmem_ld32(tbase + lane_addr + cACC1, h);
      tc::tmem_ld_wait();
      uint32_t a2[32];
#pragma unroll
      for (int q = 0; q < 16; q++) {
        const float u = fmaxf(__uint_as_float(h[2 * q]), 0.0f);
        const float v = fmaxf(__uint_as_float(h[2 * q + 1]), 0.0f);
        tc::split_pair(u, v, a2[q], a2[16 + q]);
      }
      tc::tmem_st32(tbase + lane_addr + cA2, a2);
      tc::tmem_st_wait();
    }
    tc::fence_before_sync();
    tc::bar_sync(1 + wg, 128);
    if (row == 0) {
      tc::fence_after_sync();
      const uint32_t d = tbase + cA1, a = tbase + cA2;   // acc2 reuses the A1 columns
      uint32_t bb[5];
#pragma unroll
      for (int q = 0; q < 5; q++) bb[q] = tc::smem_u32(img.b2[q]);
      tc::mma_ts(d, a + 0, tc::smem_desc_kmajor(bb[0], 512, 128), kIdesc, 0);   // h_hi W_hi
      tc::mma_ts(d, a + 8, tc::smem_desc_kmajor(bb[1], 512, 128), kIdesc, 1);
      tc::mma_ts(d, a + 0, tc::smem_desc_kmajor(bb[2], 512, 128), kIdesc, 1);   // h_hi W_lo
      tc::mma_ts(d, a + 8, tc::smem_desc_kmajor(bb[3], 512, 128), kIdesc, 1);
      tc::mma_ts(d, a + 16, tc::smem_desc_kmajor(bb[0], 512, 128), kIdesc, 1);  // h_lo W_hi
      tc::mma_ts(d, a + 24, tc::smem_desc_kmajor(bb[1], 512, 128), kIdesc, 1);
      tc::mma_ts(d, tbase + cONES, tc::smem_desc_kmajor(bb[4], 512, 128), kIdesc, 1);  // + b2
      tc::mma_commit(&S.bar_acc2[wg]);
    }
    tc::mbar_wait(&S.bar_acc2[wg], phase);
    tc::fence_after_sync();
    phase ^= 1u;
    // ---- layer-2 epilogue: ReLU, layer 3, update ----
    uint32_t h2[32];
    tc::tmem_ld32(tbase + lane_addr + cA1, h2);
    tc::tmem_ld_wait();
    if (valid) {
      float dir = img.b3[0], mag = img.b3[1];
#pragma unroll
      for (int q = 0; q < 32; q++) {
        const float hv = fmaxf(__uint_as_float(h2[q]), 0.0f);
        dir = fmaf(img.w3[0][q], hv, dir);
        mag = fmaf(img.w3[1][q], hv, mag);
      }
      // engine.py:537-539
      const float ex = glibc_expf(__fmul_rn(mag, alpha), S.exptab);
      const float upd = __fmul_rn(__fmul_rn(dir, ex), beta_out);
      const float du = __fmul_rn(ds, upd);
      float out = __fadd_rn(x.w, du);
      maxabs = fmaxf(maxabs, fabsf(du));
      bad |= !isfinite(out);
      if (apply_decay) out = __fmul_rn(out, decay);   // optim.py:100-101
      T.theta[e] = out;
      if (!adv) T.state[e - T.lo] = ns;
    }
  }
  if (cur >= 0) {
    if (maxabs > 0.0f)
      atomicMax(reinterpret_cast<unsigned int *>(&P.maxabs[cur]), __float_as_uint(maxabs));
    if (bad) atomicOr(&P.status[cur], LOPT_STATUS_NONFINITE_PARAM);
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, kTmemCols);
}

// ---------------------------------------------------------------------------
// host launchers

int fast_supported(const DevicePlan &P) { return P.h1 == 32 && P.h2 == 32 ? 1 : 0; }
int64_t fast_stat_chunk() { return kFastStatChunk; }
int64_t fast_apply_chunk() { return kTile; }

void launch_fast_stats(const DevicePlan &P, cudaStream_t s) {
  if (P.n_stat_items > 0) {
    if (P.kind == LOPT_SMALL_FC_LOPT)
      stats_fast_kernel<LOPT_SMALL_FC_LOPT><<<P.n_stat_items, kFastStatThreads, 0, s>>>(P);
    else
      stats_fast_kernel<LOPT_VELO_MLP><<<P.n_stat_items, kFastStatThreads, 0, s>>>(P);
  }
  stats_reduce_fast_kernel<<<P.count, 64, 0, s>>>(P);
}

static int g_num_sms = 0;

void launch_fast_apply(const DevicePlan &P, cudaStream_t s) {
  if (P.kind == LOPT_SMALL_FC_LOPT)
    prep_kernel<LOPT_SMALL_FC_LOPT><<<P.count, 256, 0, s>>>(P);
  else
    prep_kernel<LOPT_VELO_MLP><<<P.count, 256, 0, s>>>(P);
  if (P.n_tiles == 0) return;
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  // > half of the SM's shared memory: one CTA per SM, which the 512-column
  // TMEM allocation needs anyway
  const size_t smem = std::max<size_t>(sizeof(ApplySmem) + 1024, 120 * 1024);
  const int grid = (int)std::min<int64_t>(g_num_sms, (P.n_tiles + kWGs - 1) / kWGs);
  if (P.kind == LOPT_SMALL_FC_LOPT) {
    cudaFuncSetAttribute(apply_fast_kernel<LOPT_SMALL_FC_LOPT>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    apply_fast_kernel<LOPT_SMALL_FC_LOPT><<<grid, kApplyThreads, smem, s>>>(P);
  } else {
    cudaFuncSetAttribute(apply_fast_kernel<LOPT_VELO_MLP>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    apply_fast_kernel<LOPT_VELO_MLP><<<grid, kApplyThreads, smem, s>>>(P);
  }
}

size_t prep_image_bytes() { return sizeof(PrepImage); }

}  // namespace lopt
