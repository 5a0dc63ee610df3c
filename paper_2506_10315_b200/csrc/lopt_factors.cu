// lopt_factors.cu -- phase 0 of the step: the Adafactor row/column factors.
//
// Reference: state.py:93-113 update_adafactor (row/col means of g^2 in f64,
// rounded to f32, then an f32 EMA) and features.py:133-135 factor_means.
// The B200 pass reads g once (4 B/param) and produces f64 partial sums per
// (row, column strip) and per (row block, column); fixed-order reductions
// turn them into per-row / per-column f64 sums, which is also the block a
// multi-GPU caller all-reduces (distsim.py:448-474).  No float atomics: the
// result is bit-reproducible for a fixed plan.
#include "lopt_common.cuh"
#include "lopt_tc.cuh"

namespace lopt {

constexpr int kFactorThreads = 256;
constexpr int kFactorWarps = kFactorThreads / 32;
constexpr int kStripCols = 1024;     // 32 columns per lane

// One tile per CTA: rows [a0, a1) x columns [b0, b1).  Warps own rows (w, w+8,
// ...), lanes own columns (lane + 32k), so every g row segment is read
// coalesced exactly once.  Vector tensors (n == 1) take the thread-per-row path.
__global__ void __launch_bounds__(kFactorThreads)
factor_partials_kernel(DevicePlan P) {
  const FactorItem it = P.factor_items[blockIdx.x];
  const TensorDesc T = P.tensors[it.tensor];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ double colbuf[kStripCols];
  __shared__ double wsum[kFactorWarps];
  __shared__ uint32_t bad_s;
  if (tid == 0) bad_s = 0;
  __syncthreads();
  uint32_t bad = 0;
  const float *g = T.grad;

  if (T.n == 1) {
    // vector (m,1): row sum of row a is g[a]^2; the single column sums all rows
    double acc = 0.0;
    for (int64_t a = it.a0 + tid; a < it.a1; a += kFactorThreads) {
      double sq = 0.0;
      if (a >= T.lo && a < T.hi) {
        const float v = g[a];
        bad |= !isfinite(v);
        sq = (double)v * (double)v;
      }
      T.rowpart[a] = sq;   // strip 0
      acc += sq;
    }
    acc = warp_sum(acc);
    if (lane == 0) wsum[warp] = acc;
    if (bad) atomicOr(&bad_s, 1u);
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < kFactorWarps; w++) s += wsum[w];
      T.colpart[it.rowblock] = s;
      if (bad_s) {
        atomicOr(&P.status[it.tensor], LOPT_STATUS_NONFINITE_GRAD);
        atomicOr(P.abort_flag, 1u);
        *P.grad_flag = 1.0;
      }
    }
    return;
  }

  constexpr int K = kStripCols / 32;
  double colacc[K];
#pragma unroll
  for (int k = 0; k < K; k++) colacc[k] = 0.0;
  const int64_t n = T.n;
  for (int64_t a = it.a0 + warp; a < it.a1; a += kFactorWarps) {
    const float *grow = g + a * n;
    const int64_t rowbase = a * n;
    double rowp = 0.0;
#pragma unroll
    for (int k = 0; k < K; k++) {
      const int64_t b = it.b0 + lane + 32 * k;
      if (b < it.b1) {
        const int64_t e = rowbase + b;
        if (e >= T.lo && e < T.hi) {
          const float v = grow[b];
          bad |= !isfinite(v);
          const double sq = (double)v * (double)v;
          colacc[k] += sq;
          rowp += sq;
        }
      }
    }
    rowp = warp_sum(rowp);
    if (lane == 0) T.rowpart[(int64_t)it.strip * T.m + a] = rowp;
  }
  // combine the warps' column partials in warp order
  for (int w = 0; w < kFactorWarps; w++) {
    if (warp == w) {
#pragma unroll
      for (int k = 0; k < K; k++) {
        const int j = lane + 32 * k;
        colbuf[j] = (w == 0) ? colacc[k] : colbuf[j] + colacc[k];
      }
    }
    __syncthreads();
  }
  const int64_t width = it.b1 - it.b0;
  for (int j = tid; j < width; j += kFactorThreads)
    T.colpart[(int64_t)it.rowblock * n + it.b0 + j] = colbuf[j];
  if (bad) atomicOr(&bad_s, 1u);
  __syncthreads();
  if (tid == 0 && bad_s) {
    atomicOr(&P.status[it.tensor], LOPT_STATUS_NONFINITE_GRAD);
    atomicOr(P.abort_flag, 1u);
    *P.grad_flag = 1.0;
  }
}

// rowsum[a] = sum over strips of rowpart, colsum[b] = sum over row blocks of
// colpart, each in a fixed order.  grid: (ceil(max(m+n)/256), count).
__global__ void factor_reduce_kernel(DevicePlan P) {
  const TensorDesc T = P.tensors[blockIdx.y];
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < T.m) {
    double s = 0.0;
    for (int k = 0; k < T.nstrips; k++) s += T.rowpart[(int64_t)k * T.m + idx];
    T.rowsum[idx] = s;
  } else if (idx < T.m + T.n) {
    const int64_t b = idx - T.m;
    double s = 0.0;
    for (int k = 0; k < T.nrowblocks; k++) s += T.colpart[(int64_t)k * T.n + b];
    T.colsum[b] = s;
  }
}

// state.py:108-113: mean = f32(sum / len), r' = b*r + (1-b)*mean in f32; then
// the row/column tables the features read: {x5', x6', x7', 1/sqrt(x'+eps) x3}.
// With state_advanced the factors are taken as given.
__global__ void factor_finalize_kernel(DevicePlan P) {
  const TensorDesc T = P.tensors[blockIdx.y];
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= T.m + T.n) return;
  const bool is_row = idx < T.m;
  const int64_t i = is_row ? idx : idx - T.m;
  const int64_t len = is_row ? T.m : T.n;
  float *fac = is_row ? T.r : T.c;
  float *tab = (is_row ? T.rowtab : T.coltab) + i * kRowTab;
  float x[3];
  if (P.state_advanced) {
#pragma unroll
    for (int k = 0; k < 3; k++) x[k] = fac[k * len + i];
  } else {
    const double sum = is_row ? T.rowsum[i] : T.colsum[i];
    if (*P.grad_flag != 0.0) {
      // a non-finite gradient on any rank (the flag is all-reduced with the
      // sums): abort before any state is written (optim.py:160-165)
      if (!isfinite(sum)) atomicOr(&P.status[blockIdx.y], LOPT_STATUS_NONFINITE_GRAD);
      atomicOr(P.abort_flag, 1u);
      return;
    }
    const float mean = (float)(sum / (double)(is_row ? T.n : T.m));
#pragma unroll
    for (int k = 0; k < 3; k++) {
      const float b = P.beta[4 + k];
      const float omb = __fsub_rn(1.0f, b);
      x[k] = ema(b, omb, fac[k * len + i], mean);
      fac[k * len + i] = x[k];
    }
  }
  // entries 8..15 (the fast path's scaled fp16 operands) are written by
  // prep_kernel once the normalization scale is known
  float4 *t4 = reinterpret_cast<float4 *>(tab);
  t4[0] = make_float4(x[0], x[1], x[2], rsqrt_strict(x[0]));
  t4[1] = make_float4(rsqrt_strict(x[1]), rsqrt_strict(x[2]), 0.f, 0.f);
}

// features.py:133-135: mr_i = f32(mean_f64(r_i')).  One CTA per tensor,
// fixed-order f64 reduction.
// Fast mode also produces the closed-form feature sums of the 12 row/column
// broadcast columns over this call's elements [lo, hi): sum_a cnt_a * x(a)^2
// and sum_b cnt_b * y(b)^2, so phase 1 only has to reduce the per-element
// columns.
__global__ void __launch_bounds__(256) factor_means_kernel(DevicePlan P) {
  const TensorDesc T = P.tensors[blockIdx.x];
  constexpr int NW = 256 / 32;
  __shared__ double red[15][NW];
  const bool bc = P.bcsum != nullptr;
  double acc[15];
#pragma unroll
  for (int k = 0; k < 15; k++) acc[k] = 0.0;
  for (int64_t a = threadIdx.x; a < T.m; a += blockDim.x) {
    const float4 v = reinterpret_cast<const float4 *>(T.rowtab + a * kRowTab)[0];
    acc[0] += (double)v.x;
    acc[1] += (double)v.y;
    acc[2] += (double)v.z;
    if (bc) {
      const float4 w = reinterpret_cast<const float4 *>(T.rowtab + a * kRowTab)[1];
      const int64_t s0 = max(T.lo, a * T.n), s1 = min(T.hi, (a + 1) * T.n);
      const double cnt = s1 > s0 ? (double)(s1 - s0) : 0.0;
      const float x6[6] = {v.x, v.y, v.z, v.w, w.x, w.y};
#pragma unroll
      for (int k = 0; k < 6; k++) acc[3 + k] += cnt * (double)x6[k] * (double)x6[k];
    }
  }
  if (bc) {
    for (int64_t b = threadIdx.x; b < T.n; b += blockDim.x) {
      // rows a with lo <= a*n + b < hi
      const int64_t alo = T.lo > b ? (T.lo - b + T.n - 1) / T.n : 0;
      const int64_t ahi = T.hi - 1 >= b ? (T.hi - 1 - b) / T.n : -1;
      const double cnt = ahi >= alo ? (double)(ahi - alo + 1) : 0.0;
      const float4 v = reinterpret_cast<const float4 *>(T.coltab + b * kRowTab)[0];
      const float4 w = reinterpret_cast<const float4 *>(T.coltab + b * kRowTab)[1];
      const float y6[6] = {v.x, v.y, v.z, v.w, w.x, w.y};
#pragma unroll
      for (int k = 0; k < 6; k++) acc[9 + k] += cnt * (double)y6[k] * (double)y6[k];
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 15; k++) {
    const double s = warp_sum(acc[k]);
    if (lane == 0) red[k][warp] = s;
  }
  __syncthreads();
  if (threadIdx.x < 15) {
    double s = 0.0;
    for (int w = 0; w < NW; w++) s += red[threadIdx.x][w];
    const int k = threadIdx.x;
    if (k < 3) {
      P.tscal[blockIdx.x].mr[k] = (float)(s / (double)T.m);
    } else if (bc) {
      // reference columns: r5,r6,r7 -> 4,5,6; rsqrt r -> 14,15,16;
      // c5,c6,c7 -> 7,8,9; rsqrt c -> 17,18,19
      const int q = k - 3;
      const int col = q < 6 ? (q < 3 ? 4 + q : 11 + q) : (q < 9 ? 1 + q : 8 + q);
      P.bcsum[(int64_t)blockIdx.x * d_feat(P.kind) + col] = s;
    }
  }
}

}  // namespace lopt

namespace lopt {

void launch_factor_partials(const DevicePlan &P, cudaStream_t s) {
  if (P.n_factor_items > 0) factor_partials_kernel<<<P.n_factor_items, kFactorThreads, 0, s>>>(P);
}

void launch_factor_reduce(const DevicePlan &P, int64_t max_mn, cudaStream_t s) {
  dim3 grid((unsigned)((max_mn + 255) / 256), (unsigned)P.count);
  factor_reduce_kernel<<<grid, 256, 0, s>>>(P);
}

void launch_factor_finalize(const DevicePlan &P, int64_t max_mn, cudaStream_t s) {
  dim3 grid((unsigned)((max_mn + 255) / 256), (unsigned)P.count);
  factor_finalize_kernel<<<grid, 256, 0, s>>>(P);
}

void launch_factor_means(const DevicePlan &P, cudaStream_t s) {
  factor_means_kernel<<<P.count, 256, 0, s>>>(P);
}

}  // namespace lopt
