// lopt_factors.cu -- phase 0 of the step: the Adafactor row/column factors.
//
// Reference: state.py:93-113 update_adafactor (row/col means of g^2 in f64,
// rounded to f32, then an f32 EMA) and features.py:133-135 factor_means.
// The B200 pass reads g once (4 B/param) and produces f64 partial sums per
// (row, column strip) and per (row block, column); fixed-order reductions
// turn them into per-row / per-column f64 sums, which is also the block a
// multi-GPU caller all-reduces (distsim.py:448-474).  No float atomics: the
// result is bit-reproducible for a fixed plan.
#include <algorithm>

#include "lopt_common.cuh"
#include "lopt_tc.cuh"

namespace lopt {

constexpr int kFactorThreads = 256;
constexpr int kFactorWarps = kFactorThreads / 32;
constexpr int kStripCols = 512;      // columns per tile strip (16 per lane)

__device__ __forceinline__ void flag_nonfinite(const DevicePlan &P, int tensor) {
  atomicOr(&P.status[tensor], LOPT_STATUS_NONFINITE_GRAD);
  atomicOr(P.abort_flag, 1u);
  *P.grad_flag = 1.0;
}

// Loads one row segment of the strip into v[16]: VEC lanes own 4 consecutive
// columns per 128-column slab (16-byte loads), otherwise 1 column per 32.
template <bool VEC>
__device__ __forceinline__ void load_row(const float *grow, int64_t b0, int64_t b1, int lane,
                                         float (&v)[16]) {
  if (VEC) {
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int64_t b = b0 + 4 * lane + 128 * k;
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
      if (b < b1) x = __ldg(reinterpret_cast<const float4 *>(grow + b));
      v[4 * k + 0] = x.x; v[4 * k + 1] = x.y; v[4 * k + 2] = x.z; v[4 * k + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 16; k++) {
      const int64_t b = b0 + lane + 32 * k;
      v[k] = b < b1 ? __ldg(grow + b) : 0.0f;
    }
  }
}

template <bool VEC>
__device__ __forceinline__ int64_t col_of(int64_t b0, int lane, int k) {
  return VEC ? b0 + 4 * lane + 128 * (k >> 2) + (k & 3) : b0 + lane + 32 * k;
}

// One tile per CTA: rows [a0, a1) x columns [b0, b1), b1 - b0 <= 512.  Warp w
// owns rows a0+w, a0+w+8, ... and processes two rows per step so 2 x 16 loads
// are in flight per lane; lanes own fixed columns, so column partials stay in
// registers (f64) and are combined across warps once, in warp order.  The
// element-range mask of a sharded plan is applied only on rows that straddle
// [lo, hi).  A non-finite gradient shows up as a non-finite row sum.
template <bool VEC>
__device__ void factor_tile(const DevicePlan &P, const FactorItem &it, const TensorDesc &T,
                            double (*colbuf)[kStripCols]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ uint32_t bad_s;
  if (tid == 0) bad_s = 0;
  double colacc[16];
#pragma unroll
  for (int k = 0; k < 16; k++) colacc[k] = 0.0;
  const int64_t n = T.n;
  bool bad = false;
  for (int64_t a = it.a0 + warp; a < it.a1; a += 2 * kFactorWarps) {
    const int64_t a2 = a + kFactorWarps;
    const bool has2 = a2 < it.a1;
    float v[2][16];
    load_row<VEC>(T.grad + a * n, it.b0, it.b1, lane, v[0]);
    if (has2) load_row<VEC>(T.grad + a2 * n, it.b0, it.b1, lane, v[1]);
#pragma unroll
    for (int r = 0; r < 2; r++) {
      if (r == 1 && !has2) break;
      const int64_t row = r == 0 ? a : a2;
      const bool full = row * n >= T.lo && (row + 1) * n <= T.hi;
      double rowp2[2] = {0.0, 0.0};   // two chains: half the dependent DADD latency
#pragma unroll
      for (int k = 0; k < 16; k++) {
        double sq = (double)v[r][k] * (double)v[r][k];
        if (!full) {
          const int64_t e = row * n + col_of<VEC>(it.b0, lane, k);
          if (e < T.lo || e >= T.hi) sq = 0.0;
        }
        colacc[k] += sq;
        rowp2[k & 1] += sq;
      }
      double rowp = warp_sum(rowp2[0] + rowp2[1]);
      if (lane == 0) {
        T.rowpart[(int64_t)it.strip * T.m + row] = rowp;
        bad |= !isfinite(rowp);
      }
    }
  }
  // combine the warps' column partials: every warp parks its 16 columns in
  // its own row of shared memory, one barrier, then each thread sums the
  // warps in warp order (fixed order: bit-reproducible)
#pragma unroll
  for (int k = 0; k < 16; k++) colbuf[warp][(int)col_of<VEC>(0, lane, k)] = colacc[k];
  __syncthreads();
  const int64_t width = it.b1 - it.b0;
  for (int j = tid; j < width; j += kFactorThreads) {
    double c = colbuf[0][j];
#pragma unroll
    for (int w = 1; w < kFactorWarps; w++) c += colbuf[w][j];
    T.colpart[(int64_t)it.rowblock * n + it.b0 + j] = c;
  }
  if (bad) atomicOr(&bad_s, 1u);
  __syncthreads();
  if (tid == 0 && bad_s) flag_nonfinite(P, it.tensor);
}

// VEC tiles through a per-warp double buffer filled by cp.async (LDGSTS):
// every lane copies, and later reads back, only its own 16-byte column
// groups, so a lane waits on its own copy groups (no cross-lane sync) while
// the next row pair is already in flight -- twice the bytes in flight of the
// register-staged loop without registers to hold them.
#ifndef LOPT_FACTOR_BUFS
#define LOPT_FACTOR_BUFS 2   // row-pair buffers per warp (prefetch distance + 1)
#endif
constexpr int kFactorBufs = LOPT_FACTOR_BUFS;
struct FactorSmem {
  double colbuf[kFactorWarps][kStripCols];
  float4 rows[kFactorWarps][kFactorBufs][2][kStripCols / 4];
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(tc::smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// WFULL: the item spans a full 512-column strip (no per-column bounds)
template <bool WFULL>
__device__ void factor_tile_async(const DevicePlan &P, const FactorItem &it, const TensorDesc &T,
                                  FactorSmem &F) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ uint32_t bad_s;
  if (tid == 0) bad_s = 0;
  double colacc[16];
#pragma unroll
  for (int k = 0; k < 16; k++) colacc[k] = 0.0;
  const int64_t n = T.n, width = it.b1 - it.b0;
  // row pairs of this warp: (a0 + warp + 16 q, a0 + warp + 16 q + 8)
  const int64_t first = it.a0 + warp;
  const int npairs = first < it.a1 ? (int)((it.a1 - first + 2 * kFactorWarps - 1) / (2 * kFactorWarps)) : 0;
  auto issue = [&](int q) {
    const int buf = q % kFactorBufs;
#pragma unroll
    for (int r = 0; r < 2; r++) {
      const int64_t row = first + (int64_t)q * 2 * kFactorWarps + r * kFactorWarps;
      if (row < it.a1) {
        const float *g = T.grad + row * n + it.b0;
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const int b = 4 * lane + 128 * k;
          if (WFULL || b < width) cp_async16(&F.rows[warp][buf][r][lane + 32 * k], g + b);
        }
      }
    }
    cp_async_commit();
  };
  bool bad = false;
  constexpr int kAhead = kFactorBufs - 1;
#pragma unroll
  for (int q = 0; q < kAhead; q++)
    if (q < npairs) issue(q);
  for (int q = 0; q < npairs; q++) {
    if (q + kAhead < npairs) {
      issue(q + kAhead);
      cp_async_wait<kAhead>();
    } else {
      cp_async_wait<0>();
    }
    const int buf = q % kFactorBufs;
#pragma unroll
    for (int r = 0; r < 2; r++) {
      const int64_t row = first + (int64_t)q * 2 * kFactorWarps + r * kFactorWarps;
      if (row >= it.a1) break;
      float v[16];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int b = 4 * lane + 128 * k;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (WFULL || b < width) x = F.rows[warp][buf][r][lane + 32 * k];
        v[4 * k + 0] = x.x; v[4 * k + 1] = x.y; v[4 * k + 2] = x.z; v[4 * k + 3] = x.w;
      }
      const bool full = row * n >= T.lo && (row + 1) * n <= T.hi;
      if (!full) {
        // a row cut by the element range: elements outside it count zero
        // (masked once here, so the accumulation below has no branches)
#pragma unroll
        for (int k = 0; k < 16; k++) {
          const int64_t e = row * n + col_of<true>(it.b0, lane, k);
          if (e < T.lo || e >= T.hi) v[k] = 0.0f;
        }
      }
      double rowp2[2] = {0.0, 0.0};
#pragma unroll
      for (int k = 0; k < 16; k++) {
        const double sq = (double)v[k] * (double)v[k];
        colacc[k] += sq;
        rowp2[k & 1] += sq;
      }
      const double rowp = warp_sum(rowp2[0] + rowp2[1]);
      if (lane == 0) {
        T.rowpart[(int64_t)it.strip * T.m + row] = rowp;
        bad |= !isfinite(rowp);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 16; k++) F.colbuf[warp][(int)col_of<true>(0, lane, k)] = colacc[k];
  __syncthreads();
  for (int64_t j = tid; j < width; j += kFactorThreads) {
    double c = F.colbuf[0][j];
#pragma unroll
    for (int w = 1; w < kFactorWarps; w++) c += F.colbuf[w][j];
    T.colpart[(int64_t)it.rowblock * n + it.b0 + j] = c;
  }
  if (bad) atomicOr(&bad_s, 1u);
  __syncthreads();
  if (tid == 0 && bad_s) flag_nonfinite(P, it.tensor);
}

// Vector (m, 1): the row sum of row a is g[a]^2; the single column sums all
// rows.  Four rows per thread per step, loads first.
__device__ void factor_vector(const DevicePlan &P, const FactorItem &it, const TensorDesc &T) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ double wsum[kFactorWarps];
  __shared__ uint32_t bad_s;
  if (tid == 0) bad_s = 0;
  __syncthreads();
  double acc = 0.0;
  for (int64_t a = it.a0 + tid; a < it.a1; a += 4 * kFactorThreads) {
    float v[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int64_t r = a + u * kFactorThreads;
      v[u] = (r < it.a1 && r >= T.lo && r < T.hi) ? __ldg(T.grad + r) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int64_t r = a + u * kFactorThreads;
      if (r < it.a1) {
        const double sq = (double)v[u] * (double)v[u];
        T.rowpart[r] = sq;   // strip 0
        acc += sq;
      }
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) wsum[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < kFactorWarps; w++) s += wsum[w];
    T.colpart[it.rowblock] = s;
    if (!isfinite(s)) flag_nonfinite(P, it.tensor);
  }
}

// One CTA per item (the loop also allows a persistent launch).
__global__ void __launch_bounds__(kFactorThreads, 2) factor_partials_kernel(DevicePlan P) {
  extern __shared__ __align__(16) unsigned char factor_smem_raw[];
  FactorSmem &F = *reinterpret_cast<FactorSmem *>(factor_smem_raw);
  for (int item = blockIdx.x; item < P.n_factor_items; item += gridDim.x) {
    const FactorItem it = P.factor_items[item];
    const TensorDesc T = P.tensors[it.tensor];
    if (T.n == 1) {
      factor_vector(P, it, T);
    } else if ((T.n & 3) == 0 && (reinterpret_cast<uintptr_t>(T.grad) & 15) == 0) {
      if (it.b1 - it.b0 == kStripCols) factor_tile_async<true>(P, it, T, F);
      else factor_tile_async<false>(P, it, T, F);
    } else {
      factor_tile<false>(P, it, T, F.colbuf);
    }
    __syncthreads();   // shared scratch is reused by the next item
  }
}


// Tensor owning flattened work index idx: the last j with prefix[j] <= idx.
__device__ __forceinline__ int tensor_of(const int64_t *prefix, int count, int64_t idx) {
  int lo = 0, hi = count;   // prefix[lo] <= idx < prefix[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (prefix[mid] <= idx) lo = mid;
    else hi = mid;
  }
  return lo;
}

// rowsum[a] = sum over strips of rowpart, colsum[b] = sum over row blocks of
// colpart, each in a fixed order.  One flattened grid over every tensor's
// rows (one thread each, over the <= a few strips) and columns (one warp
// each: lanes take every 32nd row block, then a fixed shuffle tree -- the
// GPT-2 embedding has 197 row blocks per column).
__device__ __forceinline__ void finalize_one(const DevicePlan &P, int jt, const TensorDesc &T,
                                             bool is_row, int64_t i, double sum);
// FIN: each row / column sum is finalized by the thread that forms it
template <bool FIN>
__global__ void factor_reduce_kernel_t(DevicePlan P) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= P.red_total) return;   // whole warps: every segment is a multiple of 32
  const int j = tensor_of(P.red_prefix, P.count, idx);
  const TensorDesc &T = P.tensors[j];
  const int64_t local = idx - P.red_prefix[j], mpad = (T.m + 31) / 32 * 32;
  if (local < mpad) {
    if (local < T.m) {
      double s = 0.0;
      for (int k = 0; k < T.nstrips; k++) s += T.rowpart[(int64_t)k * T.m + local];
      T.rowsum[local] = s;
      if (FIN) finalize_one(P, j, T, true, local, s);
    }
    return;
  }
  if (T.nrowblocks <= kWarpColumnBlocks) {   // a thread per column, in order
    const int64_t b = local - mpad;
    if (b < T.n) {
      double s = 0.0;
      for (int k = 0; k < T.nrowblocks; k++) s += T.colpart[(int64_t)k * T.n + b];
      T.colsum[b] = s;
      if (FIN) finalize_one(P, j, T, false, b, s);
    }
    return;
  }
  const int64_t b = (local - mpad) >> 5;
  const int lane = (int)(local & 31);
  double s = 0.0;
  for (int k = lane; k < T.nrowblocks; k += 32) s += T.colpart[(int64_t)k * T.n + b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0) {
    T.colsum[b] = s;
    if (FIN) finalize_one(P, j, T, false, b, s);
  }
}

// state.py:108-113: mean = f32(sum / len), r' = b*r + (1-b)*mean in f32; then
// the row/column tables the features read: {x5', x6', x7', 1/sqrt(x'+eps) x3}.
// With state_advanced the factors are taken as given.
// One row (or column) i of tensor jt: the EMA of r' (c') from this step's f64
// sum of g^2 (state.py:108-113), or the already advanced factors, and the
// row (column) table entries the per-element features read.
__device__ __forceinline__ void finalize_one(const DevicePlan &P, int jt, const TensorDesc &T,
                                             bool is_row, int64_t i, double sum) {
  const int64_t len = is_row ? T.m : T.n;
  float *fac = is_row ? T.r : T.c;
  float *tab = (is_row ? T.rowtab : T.coltab) + i * kRowTab;
  float x[3];
  if (P.state_advanced) {
#pragma unroll
    for (int k = 0; k < 3; k++) x[k] = fac[k * len + i];
  } else {
    if (*P.grad_flag != 0.0) {
      // a non-finite gradient on any rank (the flag is all-reduced with the
      // sums): abort before any state is written (optim.py:160-165)
      if (!isfinite(sum)) atomicOr(&P.status[jt], LOPT_STATUS_NONFINITE_GRAD);
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

__global__ void factor_finalize_kernel(DevicePlan P) {
  const int64_t gidx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gidx >= P.fin_total) return;
  const int jt = tensor_of(P.fin_prefix, P.count, gidx);
  const TensorDesc &T = P.tensors[jt];
  const int64_t idx = gidx - P.fin_prefix[jt];
  const bool is_row = idx < T.m;
  const int64_t i = is_row ? idx : idx - T.m;
  const double sum = P.state_advanced ? 0.0 : (is_row ? T.rowsum[i] : T.colsum[i]);
  finalize_one(P, jt, T, is_row, i, sum);
}

// features.py:133-135: mr_i = f32(mean_f64(r_i')).  One CTA per tensor,
// fixed-order f64 reduction.
// Fast mode also produces the closed-form feature sums of the 12 row/column
// broadcast columns over this call's elements [lo, hi): sum_a cnt_a * x(a)^2
// and sum_b cnt_b * y(b)^2, so phase 1 only has to reduce the per-element
// columns.
constexpr int kMeansThreads = 1024;   // the row/column loops are latency-bound
__global__ void __launch_bounds__(kMeansThreads) factor_means_kernel(DevicePlan P) {
  const TensorDesc T = P.tensors[blockIdx.x];
  constexpr int NW = kMeansThreads / 32;
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

// ---------------------------------------------------------------------------
// host launchers

int64_t factor_strip_cols() { return kStripCols; }

static int g_factor_sms = 0;

void launch_factor_partials(const DevicePlan &P, cudaStream_t s) {
  if (g_factor_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_factor_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_factor_sms <= 0) g_factor_sms = 148;
  }
  // one CTA per item (measured faster than a persistent grid: items differ in
  // size, and short CTAs backfill)
  (void)g_factor_sms;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(factor_partials_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(FactorSmem));
    attr = true;
  }
  if (P.n_factor_items > 0)
    factor_partials_kernel<<<P.n_factor_items, kFactorThreads, sizeof(FactorSmem), s>>>(P);
}

void launch_factor_reduce(const DevicePlan &P, int64_t max_mn, cudaStream_t s) {
  (void)max_mn;
  if (P.red_total > 0)
    factor_reduce_kernel_t<false><<<(unsigned)((P.red_total + 255) / 256), 256, 0, s>>>(P);
}

// single-device step: the row / column sums finalized by the threads that
// reduce them (no cross-rank merge between the two)
void launch_factor_reduce_finalize(const DevicePlan &P, cudaStream_t s) {
  if (P.red_total > 0)
    factor_reduce_kernel_t<true><<<(unsigned)((P.red_total + 255) / 256), 256, 0, s>>>(P);
}

void launch_factor_finalize(const DevicePlan &P, int64_t max_mn, cudaStream_t s) {
  (void)max_mn;
  if (P.fin_total > 0)
    factor_finalize_kernel<<<(unsigned)((P.fin_total + 255) / 256), 256, 0, s>>>(P);
}

void launch_factor_means(const DevicePlan &P, cudaStream_t s) {
  factor_means_kernel<<<P.count, kMeansThreads, 0, s>>>(P);
}

}  // namespace lopt
