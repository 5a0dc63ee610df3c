// lopt_fast.cu -- fast mode (the product path): phase 1 and the per-tensor
// operand preparation for phase 2.
//
// Same pipeline as strict mode (engine.py:619-710 fused_stats/fused_apply,
// with the accumulator advance of state.py:77-90 fused in), re-planned for
// B200:
//
//  * features use MUFU rsqrt instead of correctly rounded div/sqrt, and only
//    the 16 (VeLO: 17) per-element columns are reduced per element; the 12
//    row/column-broadcast columns have closed-form sums (lopt_factors.cu) and
//    the 11 time columns are folded into the layer-1 bias;
//  * the two 32-wide MLP layers run on the tensor cores (lopt_apply_tc.cu)
//    from B operands prepared here once per tensor and step: the
//    normalization scale folded into W1 (engine.py:686), a two-term bf16
//    split of every weight, the canonical no-swizzle K-major UMMA layout.
#include "lopt_fast.cuh"

namespace lopt {

constexpr int kFastStatThreads = 256;
constexpr int64_t kFastStatChunk = 8192;

__device__ __forceinline__ void split1(float x, uint16_t &hi, uint16_t &lo) {
  uint32_t h, l;
  tc::split_pair_f16(x, 0.0f, h, l);
  hi = (uint16_t)(h & 0xFFFFu);
  lo = (uint16_t)(l & 0xFFFFu);
}

// Scaled fp16 operands of the six row (column) broadcast features, written
// into table entries 8..15: {hi01, hi23, hi45, 0 | lo01, lo23, lo45, 0}.
__device__ __forceinline__ void prep_tab(float *tab, const float *sc) {
  const float4 a = reinterpret_cast<const float4 *>(tab)[0];
  const float4 b = reinterpret_cast<const float4 *>(tab)[1];
  const float v[6] = {a.x * sc[0], a.y * sc[1], a.z * sc[2], a.w * sc[3], b.x * sc[4], b.y * sc[5]};
  uint32_t hi[3], lo[3];
#pragma unroll
  for (int q = 0; q < 3; q++) tc::split_pair_f16(v[2 * q], v[2 * q + 1], hi[q], lo[q]);
  reinterpret_cast<uint4 *>(tab)[2] = make_uint4(hi[0], hi[1], hi[2], 0u);
  reinterpret_cast<uint4 *>(tab)[3] = make_uint4(lo[0], lo[1], lo[2], 0u);
}

// One CTA per tensor, after the feature sums are final: normalization scale
// (features.py:138-140), the layer-1 bias with the time columns folded in,
// fp16 two-term splits of the weights in the UMMA layout, the layer-2 input
// exponent s2, and the scaled broadcast-feature operands of every row/column.
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
  __shared__ float bias1[32];
  __shared__ float bound[32];
  __shared__ float s2s[2];
  const int64_t count = T.m * T.n;
  for (int k = threadIdx.x; k < D; k += blockDim.x)
    scale[k] = (float)(1.0 / sqrt(T.sumsq[k] / (double)count + kEpsNorm));
  __syncthreads();
  if (threadIdx.x < 32) {
    const int o = threadIdx.x;
    float b = b1[o];
    if (KIND == LOPT_SMALL_FC_LOPT) {
#pragma unroll
      for (int k = 0; k < kTimeFeatures; k++)
        b = __fmaf_rn(w1[o * D + 26 + k], __fmul_rn(P.step->tf[k], scale[26 + k]), b);
    }
    bias1[o] = b;
    // |h1_o| <= |bias| + sum_k |w1[o,k]| * sqrt(m*n): normalized features are
    // bounded by sqrt(m*n)
    float l1 = 0.0f;
    for (int k = 0; k < D; k++) l1 += fabsf(w1[o * D + k]);
    bound[o] = fabsf(b) + 1.01f * l1 * sqrtf((float)count);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float mx = 0.0f;
    for (int o = 0; o < 32; o++) mx = fmaxf(mx, bound[o]);
    int s2 = 0;
    while (mx > 16384.0f && s2 < 60) {
      mx *= 0.5f;
      s2++;
    }
    s2s[0] = ldexpf(1.0f, -s2);
    s2s[1] = ldexpf(1.0f, s2);
  }
  __syncthreads();
  // layer 1 (see PrepImage): slices 0/1 = W1_hi/W1_lo over the per-element
  // features, slices 2/3 over the broadcast slice [12 row/col | clip | 1 | 0 0]
  for (int i = threadIdx.x; i < 2 * 32 * 16; i += blockDim.x) {
    const int s = i >> 9, o = (i >> 4) & 31, q = i & 15;
    float v = 0.0f;
    if (s == 0) {
      v = w1[o * D + elem_col(KIND, q)];
    } else if (q < 12) {
      v = w1[o * D + bc_col(q)];
    } else if (q == 12) {
      v = (KIND == LOPT_VELO_MLP) ? w1[o * D + 28] : 0.0f;   // clip(g)
    } else if (q == 13) {
      v = bias1[o];                                          // the constant-1 column
    }
    uint16_t hi, lo;
    split1(v, hi, lo);
    img->b1[2 * s][bslot(o, q)] = hi;
    img->b1[2 * s + 1][bslot(o, q)] = lo;
  }
  // layer 2: W2 hi/lo by K halves, then the bias slice (k = 0: hi, k = 1: lo)
  const float sd = s2s[0], su = s2s[1];
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
    split1(b2[o] * sd, hi, lo);
    img->b2[4][bslot(o, k)] = k == 0 ? hi : (k == 1 ? lo : (uint16_t)0);
  }
  if (threadIdx.x < 64) {
    const int o = threadIdx.x & 31, out = threadIdx.x >> 5;
    img->w3i[o >> 1][2 * out + (o & 1)] = w3[out * 32 + o] * su;
  }
  if (threadIdx.x < 2) img->b3[threadIdx.x] = b3[threadIdx.x];
  if (threadIdx.x < 3) img->sqmr[threadIdx.x] = sqrtf(P.tscal[j].mr[threadIdx.x]);
  if (threadIdx.x < 17)
    img->escale[threadIdx.x] = threadIdx.x < 16 ? scale[elem_col(KIND, threadIdx.x)]
                                                : (KIND == LOPT_VELO_MLP ? scale[28] : 0.0f);
  if (threadIdx.x >= 17 && threadIdx.x < 20) img->escale[threadIdx.x] = 0.0f;
  if (threadIdx.x == 0) {
    img->s2_down = sd;
    img->pad[0] = img->pad[1] = 0.0f;
  }
  // broadcast operands: rows r5 r6 r7 rr5 rr6 rr7, columns c5 c6 c7 rc5 rc6 rc7
  const float rs[6] = {scale[4], scale[5], scale[6], scale[14], scale[15], scale[16]};
  const float cs[6] = {scale[7], scale[8], scale[9], scale[17], scale[18], scale[19]};
  for (int64_t a = threadIdx.x; a < T.m; a += blockDim.x) prep_tab(T.rowtab + a * kRowTab, rs);
  for (int64_t b = threadIdx.x; b < T.n; b += blockDim.x) prep_tab(T.coltab + b * kRowTab, cs);
}

// Phase 1 (engine.py:619-654): per-element column sums of squares of the 16
// (VeLO 17) per-element features; f32 per thread over its 32 elements, then a
// fixed-order f64 block reduction.
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
  // four consecutive elements per thread per step: 16-byte loads of theta and
  // g when the chunk is aligned, one divmod per four elements
  const bool vec = ((it.e0 & 3) == 0) && ((reinterpret_cast<uintptr_t>(T.theta) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(T.grad) & 15) == 0);
  for (int64_t e = it.e0 + 4 * threadIdx.x; e < it.e1; e += 4 * kFastStatThreads) {
    const int cnt = it.e1 - e < 4 ? (int)(it.e1 - e) : 4;
    float w4[4], g4[4];
    if (vec && cnt == 4) {
      const float4 w = __ldg(reinterpret_cast<const float4 *>(T.theta + e));
      const float4 g = __ldg(reinterpret_cast<const float4 *>(T.grad + e));
      w4[0] = w.x; w4[1] = w.y; w4[2] = w.z; w4[3] = w.w;
      g4[0] = g.x; g4[1] = g.y; g4[2] = g.z; g4[3] = g.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; u++) {
        w4[u] = u < cnt ? __ldg(T.theta + e + u) : 0.0f;
        g4[u] = u < cnt ? __ldg(T.grad + e + u) : 0.0f;
      }
    }
    // every load of the four elements is issued before any arithmetic
    float4 s4[4], rt[4], ct[4];
    int64_t a, b;
    divmod(e, T.n, inv_n, a, b);
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const bool ok = u < cnt;
      s4[u] = __ldg(T.state + (ok ? e + u - T.lo : e - T.lo));
      rt[u] = __ldg(reinterpret_cast<const float4 *>(T.rowtab + a * kRowTab));
      ct[u] = __ldg(reinterpret_cast<const float4 *>(T.coltab + b * kRowTab));
      if (++b >= T.n) {
        b = 0;
        a = a + 1 < T.m ? a + 1 : a;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const float m = u < cnt ? 1.0f : 0.0f;   // masked lanes add zeros
      FastIn x;
      x.w = w4[u];
      advance(g4[u], s4[u], adv, P.beta, x);
      const float rc[3] = {rt[u].x, rt[u].y, rt[u].z}, cc[3] = {ct[u].x, ct[u].y, ct[u].z};
      float f[16];
      fast_features(x, rc, cc, sqmr, f);
#pragma unroll
      for (int k = 0; k < 16; k++) {
        const float fm = f[k] * m;
        acc[k] = fmaf(fm, fm, acc[k]);
      }
      if (KIND == LOPT_VELO_MLP) {
        const float cg = clip01(x.g) * m;
        acc[NE - 1] = fmaf(cg, cg, acc[NE - 1]);
      }
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
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    // reference column c <- per-element slot, or 0 for broadcast/time columns
    int q = -1;
    for (int s = 0; s < 16; s++)
      if (elem_col(KIND, s) == c) q = s;
    if (KIND == LOPT_VELO_MLP && c == 28) q = 16;
    double v = 0.0;
    if (q >= 0) {
#pragma unroll
      for (int w = 0; w < kFastStatThreads / 32; w++) v += red[w][q];
    }
    out[c] = v;
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
// host launchers

// The tensor-core apply kernel indexes with 32-bit integers.
int fast_supported(const DevicePlan &P) {
  return P.h1 == 32 && P.h2 == 32 && P.n_tiles < ((int64_t)1 << 31) ? 1 : 0;
}
int64_t fast_stat_chunk() { return kFastStatChunk; }
int64_t fast_apply_chunk() { return kTile; }
size_t prep_image_bytes() { return sizeof(PrepImage); }

void launch_fast_stats(const DevicePlan &P, cudaStream_t s) {
  if (P.n_stat_items > 0) {
    if (P.kind == LOPT_SMALL_FC_LOPT)
      stats_fast_kernel<LOPT_SMALL_FC_LOPT><<<P.n_stat_items, kFastStatThreads, 0, s>>>(P);
    else
      stats_fast_kernel<LOPT_VELO_MLP><<<P.n_stat_items, kFastStatThreads, 0, s>>>(P);
  }
  stats_reduce_fast_kernel<<<P.count, 64, 0, s>>>(P);
}

void launch_tc_apply(const DevicePlan &P, cudaStream_t s);

void launch_fast_apply(const DevicePlan &P, cudaStream_t s) {
  if (P.kind == LOPT_SMALL_FC_LOPT)
    prep_kernel<LOPT_SMALL_FC_LOPT><<<P.count, 256, 0, s>>>(P);
  else
    prep_kernel<LOPT_VELO_MLP><<<P.count, 256, 0, s>>>(P);
  if (P.n_tiles > 0) launch_tc_apply(P, s);
}

}  // namespace lopt
