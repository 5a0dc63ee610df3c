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
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "lopt_fast.cuh"

namespace lopt {

#ifndef LOPT_STAT_CHUNK
#define LOPT_STAT_CHUNK 8192   // elements per stats item (tuning builds override)
#endif
#ifndef LOPT_STAT_MINB
#define LOPT_STAT_MINB 4       // stats CTAs per SM the registers are sized for
#endif
#ifndef LOPT_STAT_THREADS
#define LOPT_STAT_THREADS 256   // stats CTA size (co-residency experiments override)
#endif
constexpr int kFastStatThreads = LOPT_STAT_THREADS;
constexpr int64_t kFastStatChunk = LOPT_STAT_CHUNK;

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
constexpr int kPrepThreads = 256;
constexpr int kPrepSplit = 16;   // CTAs per tensor: the row/column table loops are latency-bound
// The apply kernel's per-CTA pair ranges, from each CTA's measured speed
// (pairs / busy ns) in the plan's previous launches (halved-weight average).  The SMs do not run at one
// speed: over identical work ~12 % of them (the same CTA indices on every
// box measured) take ~6 % longer (tools/cta_balance.py), and an even split
// leaves the rest idle for their tail.  Speeds are clamped to [0.75, 1.33] x
// their mean; missing records (first launch, aborted step) take the mean, so
// the first launch splits evenly.  Any split gives identical results.
static_assert(kPrepThreads >= kMaxApplyCtas, "one thread per apply CTA");
__device__ void balance_pair_ranges(const DevicePlan &P) {
  using Scan = cub::BlockScan<double, kPrepThreads>;
  using Reduce = cub::BlockReduce<double, kPrepThreads>;
  __shared__ union {
    typename Scan::TempStorage scan;
    typename Reduce::TempStorage red;
  } tmp;
  __shared__ double mean_s;
  const int G = P.apply_grid, b = threadIdx.x;
  // smoothed speed: the mean of the last record and the previous estimate
  double *smooth = reinterpret_cast<double *>(P.cta_perf + 2 * kMaxApplyCtas);
  double v = 0.0;
  if (b < G) {
    const int64_t n = P.cta_perf[2 * b], ns = P.cta_perf[2 * b + 1];
    const double prev = smooth[b];
    if (n > 0 && ns > 0) {
      v = (double)n / (double)ns;
      if (prev > 0.0) v = 0.5 * (v + prev);
    } else {
      v = prev;
    }
    smooth[b] = v;
  }
  const double sum = Reduce(tmp.red).Sum(v);
  __syncthreads();
  const double cnt = Reduce(tmp.red).Sum(v > 0.0 ? 1.0 : 0.0);
  if (b == 0) mean_s = cnt > 0.0 ? sum / cnt : 1.0;
  __syncthreads();
  const double mean = mean_s;
  if (b < G) v = v > 0.0 ? fmin(fmax(v, 0.75 * mean), 1.33 * mean) : mean;
  double pre, total;
  Scan(tmp.scan).ExclusiveSum(v, pre, total);
  if (b < G) P.pair_range[b] = b == 0 ? 0 : (int32_t)((double)P.n_pairs * (pre / total));
  if (b == 0) P.pair_range[G] = (int32_t)P.n_pairs;
}

template <int KIND>
__global__ void __launch_bounds__(kPrepThreads) prep_kernel(DevicePlan P) {
  constexpr int D = d_feat(KIND);
  if (blockIdx.x == 0 && blockIdx.y == gridDim.y - 1 && P.apply_grid > 0) balance_pair_ranges(P);
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
  const int64_t count = T.stat_count > 0 ? T.stat_count : T.m * T.n;
  for (int k = threadIdx.x; k < D; k += blockDim.x)
    scale[k] = (float)(1.0 / sqrt(T.sumsq[k] / (double)count + kEpsNorm));
  __syncthreads();
  if (blockIdx.y == 0) {
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
    split1(v * s2s[0], hi, lo);   // 2^-s2 folded into layer 1 (exact power of two)
    img->b1[2 * s][bslot(o, q)] = hi;
    img->b1[2 * s + 1][bslot(o, q)] = lo;
  }
  // layer 2: [W2 | v] hi/lo by K halves, then the bias slice (k = 0: hi, k = 1: lo).
  // Rows 32/33 carry the linear half of layer 3 (see PrepImage): v_out[k] =
  // 1/2 * 2^s2 * sum_o w3[out,o] W2[o,k] (its input is relu(h1) * 2^-s2) and the
  // bias 1/2 * sum_o w3[out,o] b2[o] + b3[out]; summed in f64, rounded once.
  const float sd = s2s[0], su = s2s[1];
  __shared__ float vrow[2][32], vbias[2];
  if (threadIdx.x < 64) {
    const int out = threadIdx.x >> 5, k = threadIdx.x & 31;
    double acc = 0.0;
    for (int o = 0; o < 32; o++) acc += (double)w3[out * 32 + o] * (double)w2[o * 32 + k];
    vrow[out][k] = (float)(0.5 * (double)su * acc);
  } else if (threadIdx.x < 66) {
    const int out = threadIdx.x - 64;
    double acc = 0.0;
    for (int o = 0; o < 32; o++) acc += (double)w3[out * 32 + o] * (double)b2[o];
    vbias[out] = (float)(0.5 * acc + (double)b3[out]);   // b3 rides along
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kN2 * 32; i += blockDim.x) {
    const int o = i >> 5, k = i & 31;
    const float v = o < 32 ? w2[o * 32 + k] : (o < 34 ? vrow[o - 32][k] : 0.0f);
    uint16_t hi, lo;
    split1(v, hi, lo);
    img->b2[k >> 4][bslot(o, k & 15, kN2)] = hi;
    img->b2[2 + (k >> 4)][bslot(o, k & 15, kN2)] = lo;
  }
  for (int i = threadIdx.x; i < kN2 * 16; i += blockDim.x) {
    const int o = i >> 4, k = i & 15;
    const float b = o < 32 ? b2[o] * sd : (o < 34 ? vbias[o - 32] : 0.0f);
    uint16_t hi, lo;
    split1(b, hi, lo);
    img->b2[4][bslot(o, k, kN2)] = k == 0 ? hi : (k == 1 ? lo : (uint16_t)0);
  }
  if (threadIdx.x < 64) {
    const int o = threadIdx.x & 31, out = threadIdx.x >> 5;
    img->w3h[o >> 1][2 * (o & 1) + out] = w3[out * 32 + o] * su * 0.5f;
  }
  if (threadIdx.x < 2) img->b3[threadIdx.x] = b3[threadIdx.x];
  if (threadIdx.x < 3) img->sqmr[threadIdx.x] = sqrtf(P.tscal[j].mr[threadIdx.x]);
  if (threadIdx.x < 17)
    img->escale[threadIdx.x] = threadIdx.x < 16 ? scale[elem_col(KIND, threadIdx.x)]
                                                : (KIND == LOPT_VELO_MLP ? scale[28] : 0.0f);
  if (threadIdx.x >= 17 && threadIdx.x < 20) img->escale[threadIdx.x] = 0.0f;
  if (threadIdx.x == 0) {
    img->s2_down = sd;
    img->s2_up = su;
    img->pad = 0.0f;
  }
  }   // blockIdx.y == 0
  // broadcast operands: rows r5 r6 r7 rr5 rr6 rr7, columns c5 c6 c7 rc5 rc6 rc7
  const float rs[6] = {scale[4], scale[5], scale[6], scale[14], scale[15], scale[16]};
  const float cs[6] = {scale[7], scale[8], scale[9], scale[17], scale[18], scale[19]};
  const int64_t t0 = (int64_t)blockIdx.y * blockDim.x + threadIdx.x, ts = (int64_t)gridDim.y * blockDim.x;
  for (int64_t a = t0; a < T.m; a += ts) prep_tab(T.rowtab + a * kRowTab, rs);
  for (int64_t b = t0; b < T.n; b += ts) prep_tab(T.coltab + b * kRowTab, cs);
}

// Phase 1 (engine.py:619-654): per-element column sums of squares of the 16
// (VeLO 17) per-element features; f32 per thread, then a fixed-order f64 block
// reduction.  Four consecutive elements per thread per step with 16-byte loads
// of theta and g; full groups run unmasked, only a chunk's ragged end is
// masked, and the row-table entry is loaded once per group when the four
// elements share a row.
template <int KIND>
__device__ __forceinline__ void stats_accum(float w, float g, float4 st, const float4 &rt,
                                            const float4 &ct, bool adv, const float *beta,
                                            const float *sqmr, float m, float *acc) {
  constexpr int NE = KIND == LOPT_VELO_MLP ? 17 : 16;
  FastIn x;
  x.w = w;
  advance(g, st, adv, beta, x);
  const float rc[3] = {rt.x, rt.y, rt.z}, cc[3] = {ct.x, ct.y, ct.z};
  float f[16];
  fast_features(x, rc, cc, sqmr, f);
  if (m != 1.0f) {
#pragma unroll
    for (int k = 0; k < 16; k++) f[k] *= m;
  }
#pragma unroll
  for (int k = 0; k < 16; k++) acc[k] = fmaf(f[k], f[k], acc[k]);
  if (KIND == LOPT_VELO_MLP) {
    const float cg = clip01(x.g) * m;
    acc[NE - 1] = fmaf(cg, cg, acc[NE - 1]);
  }
}

template <int KIND>
__global__ void __launch_bounds__(kFastStatThreads, LOPT_STAT_MINB) stats_fast_kernel(DevicePlan P) {
  constexpr int D = d_feat(KIND);
  constexpr int NE = KIND == LOPT_VELO_MLP ? 17 : 16;
  const ChunkItem it = P.stat_items[blockIdx.x];
  const TensorDesc &T = P.tensors[it.tensor];
  const float *theta = T.theta, *grad = T.grad, *rowtab = T.rowtab, *coltab = T.coltab;
  const float4 *state = T.state;
  const int64_t n = T.n, lo = T.lo;
  const TensorScalars ts = P.tscal[it.tensor];
  const float sqmr[3] = {sqrtf(ts.mr[0]), sqrtf(ts.mr[1]), sqrtf(ts.mr[2])};
  const double inv_n = 1.0 / (double)n;
  __shared__ float red[kFastStatThreads / 32][NE];
  float acc[NE];
#pragma unroll
  for (int k = 0; k < NE; k++) acc[k] = 0.0f;
  const bool adv = P.state_advanced != 0;
  if (it.strip) {
    // column strip: this thread's column b for rows [ra, rb); its column
    // entry is loaded once, the row entry is the same for the whole warp
    const int64_t ra = it.e0 >> 32, rb = it.e1 >> 32;
    const int64_t b = (it.e0 & 0xffffffffll) + threadIdx.x;
    const float4 ct = __ldg(reinterpret_cast<const float4 *>(coltab + b * kRowTab));
    const float *tp = theta + ra * n + b, *gp = grad + ra * n + b;
    const float4 *sp = state + (ra * n + b - lo);
#pragma unroll 2
    for (int64_t a = ra; a < rb; a++) {
      const float4 rt = __ldg(reinterpret_cast<const float4 *>(rowtab + a * kRowTab));
      stats_accum<KIND>(__ldg(tp), __ldg(gp), __ldg(sp), rt, ct, adv, P.beta, sqmr, 1.0f, acc);
      tp += n;
      gp += n;
      sp += n;
    }
  } else {
  const bool vec = ((it.e0 & 1) == 0) && ((reinterpret_cast<uintptr_t>(theta) & 7) == 0) &&
                   ((reinterpret_cast<uintptr_t>(grad) & 7) == 0);
  // two consecutive elements per thread per step (64 registers: four CTAs
  // per SM keep enough loads in flight to cover HBM latency)
  int64_t e = it.e0 + 2 * threadIdx.x;
  for (; e < it.e1; e += 2 * kFastStatThreads) {
    const int cnt = it.e1 - e < 2 ? (int)(it.e1 - e) : 2;
    int64_t a, b;
    divmod(e, n, inv_n, a, b);
    if (cnt == 2 && vec) {
      const float2 w2 = __ldg(reinterpret_cast<const float2 *>(theta + e));
      const float2 g2 = __ldg(reinterpret_cast<const float2 *>(grad + e));
      const float4 *sp = state + (e - lo);
      const float4 s0 = __ldg(sp), s1 = __ldg(sp + 1);
      const float4 r0 = __ldg(reinterpret_cast<const float4 *>(rowtab + a * kRowTab));
      const float4 c0 = __ldg(reinterpret_cast<const float4 *>(coltab + b * kRowTab));
      float4 r1 = r0, c1;
      if (b + 1 < n) {
        c1 = __ldg(reinterpret_cast<const float4 *>(coltab + (b + 1) * kRowTab));
      } else {
        r1 = __ldg(reinterpret_cast<const float4 *>(rowtab + (a + 1) * kRowTab));
        c1 = __ldg(reinterpret_cast<const float4 *>(coltab));
      }
      stats_accum<KIND>(w2.x, g2.x, s0, r0, c0, adv, P.beta, sqmr, 1.0f, acc);
      stats_accum<KIND>(w2.y, g2.y, s1, r1, c1, adv, P.beta, sqmr, 1.0f, acc);
    } else {
      // ragged or unaligned pair: element by element, masked
      int64_t aa = a, bb = b;
      for (int u = 0; u < 2; u++) {
        const bool ok = u < cnt;
        const int64_t eu = ok ? e + u : e;
        const float4 rt = __ldg(reinterpret_cast<const float4 *>(rowtab + aa * kRowTab));
        const float4 ct = __ldg(reinterpret_cast<const float4 *>(coltab + bb * kRowTab));
        stats_accum<KIND>(__ldg(theta + eu), __ldg(grad + eu), __ldg(state + (eu - lo)), rt, ct,
                          adv, P.beta, sqmr, ok ? 1.0f : 0.0f, acc);
        if (++bb >= n) {
          bb = 0;
          aa = aa + 1 < T.m ? aa + 1 : aa;
        }
      }
    }
  }
  }
  // warp reduction in f32 (each lane holds at most 32 elements' worth), then
  // a fixed-order f64 block reduction
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NE; k++) {
    const float s = warp_sum(acc[k]);
    if (lane == 0) red[warp][k] = s;
  }
  __syncthreads();
  double *out = P.stat_part + (int64_t)blockIdx.x * D;
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    // reference column c <- per-element slot, or 0 for broadcast/time columns
    int q = -1;
    for (int s2 = 0; s2 < 16; s2++)
      if (elem_col(KIND, s2) == c) q = s2;
    if (KIND == LOPT_VELO_MLP && c == 28) q = 16;
    double v = 0.0;
    if (q >= 0) {
#pragma unroll
      for (int w = 0; w < kFastStatThreads / 32; w++) v += (double)red[w][q];
    }
    out[c] = v;
  }
}

// Per-tensor sums: item partials (fixed order) + broadcast closed forms +
// time columns (count * tf^2).  Writes the all-reducible sumsq block.
__global__ void __launch_bounds__(256) stats_reduce_fast_kernel(DevicePlan P) {
  // warp w sums items w, w+8, ... (lanes over features), then the 8 warp
  // partials are added in warp order: a fixed order, 8 short dependent chains
  // instead of one chain as long as the tensor's item count
  constexpr int kWarps = 8;
  __shared__ double part[kWarps][kMaxFeat];
  const int j = blockIdx.x;
  const TensorDesc T = P.tensors[j];
  const int D = d_feat(P.kind);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = lane; k < D; k += 32) {
    double s = 0.0;
    for (int i = warp; i < T.stat_items; i += kWarps)
      s += P.stat_part[(int64_t)(T.stat_item0 + i) * D + k];
    part[warp][k] = s;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < D; k += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; w++) s += part[w][k];
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
int64_t fast_stat_strip() { return kFastStatThreads; }
int fast_stat_min_blocks() { return LOPT_STAT_MINB; }
int64_t fast_apply_chunk() { return kTile; }
size_t prep_image_bytes() { return sizeof(PrepImage); }

void launch_fast_stats(const DevicePlan &P, cudaStream_t s) {
  if (P.n_stat_items > 0) {
    if (P.kind == LOPT_SMALL_FC_LOPT)
      stats_fast_kernel<LOPT_SMALL_FC_LOPT><<<P.n_stat_items, kFastStatThreads, 0, s>>>(P);
    else
      stats_fast_kernel<LOPT_VELO_MLP><<<P.n_stat_items, kFastStatThreads, 0, s>>>(P);
  }
  stats_reduce_fast_kernel<<<P.count, 256, 0, s>>>(P);
}

// strict mode: the same per-tensor reduction (item partials of the per-element
// columns + closed-form broadcast and time columns, all f64)
void launch_stats_reduce_closed(const DevicePlan &P, cudaStream_t s) {
  stats_reduce_fast_kernel<<<P.count, 256, 0, s>>>(P);
}

void launch_tc_apply(const DevicePlan &P, cudaStream_t s);

void launch_fast_apply(const DevicePlan &P, cudaStream_t s) {
  if (P.kind == LOPT_SMALL_FC_LOPT)
    prep_kernel<LOPT_SMALL_FC_LOPT><<<dim3(P.count, kPrepSplit), kPrepThreads, 0, s>>>(P);
  else
    prep_kernel<LOPT_VELO_MLP><<<dim3(P.count, kPrepSplit), kPrepThreads, 0, s>>>(P);
  if (P.n_tiles > 0) launch_tc_apply(P, s);
}

}  // namespace lopt
