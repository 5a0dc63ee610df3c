// lopt_strict.cu -- phases 1 and 2 in strict mode (CUDA cores).
//
// Strict mode is the parity reference of the build: every feature is computed
// with correctly rounded f32 ops in the reference's expression order
// (features.py:147-195), the MLP is a per-output sequential fmaf chain from the
// bias (engine.py:441-480 under fastmath={"contract"}), and the exponential is
// the glibc expf algorithm (engine.py:537).  Given identical advanced state and
// identical f64 sums it reproduces fused_apply bit for bit.  The fast mode
// (lopt_fast.cu) is the product path; this one is the yardstick.
#include "lopt_common.cuh"
#include "lopt_tc.cuh"
#include "lopt_fast.cuh"

namespace lopt {

constexpr int kStrictThreads = 256;
// apply: two elements a thread (~214 registers, one CTA of 8 warps per SM;
// 192 threads x 2 CTAs at 168 registers spilled and ran 27% slower)
constexpr int kStrictApplyThreads = 256;

// Flat element index -> (row, col) for a chunk that starts at e0.
struct RowCol {
  int64_t a, b;
};
__device__ __forceinline__ RowCol split_index(int64_t e, int64_t n) {
  return {e / n, e % n};
}

// One element's global inputs, loaded before any of them is used so that a
// thread keeps two elements' loads in flight (the strict kernels run at one
// or two warps per scheduler and are otherwise load-latency bound).
struct RawElem {
  float w, g;
  float4 s, r0, r1, c0, c1;
};

__device__ __forceinline__ RawElem load_raw(const TensorDesc &T, int64_t e) {
  RawElem r;
  r.w = T.theta[e];
  r.g = T.grad[e];
  r.s = T.state[e - T.lo];
  const RowCol rc = split_index(e, T.n);
  const float4 *rt = reinterpret_cast<const float4 *>(T.rowtab + rc.a * kRowTab);
  const float4 *ct = reinterpret_cast<const float4 *>(T.coltab + rc.b * kRowTab);
  r.r0 = rt[0];
  r.r1 = rt[1];
  r.c0 = ct[0];
  r.c1 = ct[1];
  return r;
}

__device__ __forceinline__ void unpack_elem(const RawElem &r, bool advanced, const float *beta,
                                            Elem &x, float4 &newstate, float *rowt,
                                            float *colt) {
  x.w = r.w;
  x.g = r.g;
  const float4 s = r.s;
  if (advanced) {
    x.m1 = s.x; x.m2 = s.y; x.m3 = s.z; x.v = s.w;
  } else {
    // state.py:77-90, recomputed in registers from the old accumulators
    x.m1 = ema(beta[0], __fsub_rn(1.0f, beta[0]), s.x, x.g);
    x.m2 = ema(beta[1], __fsub_rn(1.0f, beta[1]), s.y, x.g);
    x.m3 = ema(beta[2], __fsub_rn(1.0f, beta[2]), s.z, x.g);
    x.v = ema(beta[3], __fsub_rn(1.0f, beta[3]), s.w, __fmul_rn(x.g, x.g));
  }
  newstate = make_float4(x.m1, x.m2, x.m3, x.v);
  rowt[0] = r.r0.x; rowt[1] = r.r0.y; rowt[2] = r.r0.z; rowt[3] = r.r0.w;
  rowt[4] = r.r1.x; rowt[5] = r.r1.y;
  colt[0] = r.c0.x; colt[1] = r.c0.y; colt[2] = r.c0.z; colt[3] = r.c0.w;
  colt[4] = r.c1.x; colt[5] = r.c1.y;
}

// Phase 1 (engine.py:619-654 fused_stats): per-element features, f64 sums of
// squares of the 16 (VeLO: 17) per-element columns -> stat_part[item][col]
// (0 for the others).  The 12 row/column-broadcast columns and the 11 time
// columns are per-row / per-column / per-tensor constants whose sums have
// closed forms (count x value^2, factor_means_kernel and
// stats_reduce_fast_kernel); any f64 summation order reproduces the f32
// normalization scale, so only the per-element
// columns need per-thread f64 accumulators -- 16 instead of 39 doubles,
// which is what lets the kernel hold two elements' loads in flight.
template <int KIND>
__global__ void __launch_bounds__(kStrictThreads, 3)
stats_strict_kernel(DevicePlan P) {
  constexpr int D = d_feat(KIND);
  constexpr int NE = KIND == LOPT_VELO_MLP ? 17 : 16;
  const ChunkItem it = P.stat_items[blockIdx.x];
  const TensorDesc T = P.tensors[it.tensor];
  const TensorScalars ts = P.tscal[it.tensor];
  __shared__ float tf[kTimeFeatures];
  __shared__ double red[kStrictThreads / 32][NE];
  if (threadIdx.x < kTimeFeatures) tf[threadIdx.x] = P.step->tf[threadIdx.x];
  __syncthreads();
  double acc[NE];
#pragma unroll
  for (int k = 0; k < NE; k++) acc[k] = 0.0;
  auto accumulate = [&](const RawElem &r) {
    Elem x;
    float4 ns;
    float rowt[6], colt[6], f[D];
    unpack_elem(r, P.state_advanced, P.beta, x, ns, rowt, colt);
    strict_features<KIND>(x, rowt, colt, ts.mr, tf, f);
#pragma unroll
    for (int q = 0; q < NE; q++) {
      const double fv = (double)f[q < 16 ? elem_col(KIND, q) : 28];
      acc[q] = __fma_rn(fv, fv, acc[q]);
    }
  };
  for (int64_t e = it.e0 + threadIdx.x; e < it.e1; e += 2 * kStrictThreads) {
    const int64_t eb = e + kStrictThreads;
    const bool has_b = eb < it.e1;
    const RawElem ra = load_raw(T, e);
    const RawElem rb = load_raw(T, has_b ? eb : e);
    accumulate(ra);
    if (has_b) accumulate(rb);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NE; q++) {
    const double s = warp_sum(acc[q]);
    if (lane == 0) red[warp][q] = s;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    int q = -1;
    for (int s2 = 0; s2 < 16; s2++)
      if (elem_col(KIND, s2) == c) q = s2;
    if (KIND == LOPT_VELO_MLP && c == 28) q = 16;
    double v = 0.0;
    if (q >= 0) {
      for (int w = 0; w < kStrictThreads / 32; w++) v += red[w][q];
    }
    P.stat_part[(int64_t)blockIdx.x * D + c] = v;
  }
}

// Shared-memory image of one tensor's MLP in strict mode.  W1 is stored
// transposed with the normalization scale folded in (engine.py:686:
// w1s = w1 * scale, one f32 multiply).
struct StrictMlpSmem {
  float w1sT[kMaxFeat][kMaxHidden];
  float b1[kMaxHidden];
  float w2T[kMaxHidden][kMaxHidden];
  float b2[kMaxHidden];
  float w3[2][kMaxHidden];
  float b3[2];
  uint64_t exptab[32];
};

template <int D>
__device__ void load_strict_mlp(const DevicePlan &P, const TensorDesc &T, StrictMlpSmem &S) {
  const int H1 = kMaxHidden, H2 = kMaxHidden;
  const float *wp = P.weights + (int64_t)T.weight_slot * P.weight_stride;
  const float *w1 = wp, *b1 = w1 + H1 * D, *w2 = b1 + H1, *b2 = w2 + H2 * H1, *w3 = b2 + H2,
              *b3 = w3 + 2 * H2;
  // features.py:138-140 normalization_scale, f64 then f32
  __shared__ float scale[kMaxFeat];
  const int64_t count = T.stat_count > 0 ? T.stat_count : T.m * T.n;
  for (int k = threadIdx.x; k < D; k += blockDim.x)
    scale[k] = (float)(1.0 / sqrt(T.sumsq[k] / (double)count + kEpsNorm));
  __syncthreads();
  for (int i = threadIdx.x; i < H1 * D; i += blockDim.x) {
    const int o = i / D, j = i % D;
    S.w1sT[j][o] = __fmul_rn(w1[i], scale[j]);
  }
  for (int i = threadIdx.x; i < H2 * H1; i += blockDim.x) {
    const int o = i / H1, j = i % H1;
    S.w2T[j][o] = w2[i];
  }
  for (int i = threadIdx.x; i < H1; i += blockDim.x) S.b1[i] = b1[i];
  for (int i = threadIdx.x; i < H2; i += blockDim.x) {
    S.b2[i] = b2[i];
    S.w3[0][i] = w3[i];
    S.w3[1][i] = w3[H2 + i];
  }
  if (threadIdx.x < 2) S.b3[threadIdx.x] = b3[threadIdx.x];
  if (threadIdx.x < 32) S.exptab[threadIdx.x] = kExp2Tab[threadIdx.x];
  __syncthreads();
}

// engine.py:441-480 _mlp_lanes, two elements a thread: lane .x is element A,
// lane .y element B.  fma.rn.f32x2 is two independent correctly rounded fmas
// and each weight is a broadcast operand (SASS FFMA2 R.F32), so every output
// is the reference's fmaf chain in input order, bit for bit, while one
// shared-memory weight load feeds four fmas and the FP32 pipe retires two
// per issue slot.
template <int D>
__device__ __forceinline__ void strict_mlp2(const StrictMlpSmem &S, const float *fa,
                                            const float *fb, float2 &dir, float2 &mag) {
  float2 h1[kMaxHidden];
#pragma unroll
  for (int o = 0; o < kMaxHidden; o++) h1[o] = make_float2(S.b1[o], S.b1[o]);
#pragma unroll
  for (int j = 0; j < D; j++) {
    const float2 xj = make_float2(fa[j], fb[j]);
    const float4 *wr = reinterpret_cast<const float4 *>(S.w1sT[j]);
#pragma unroll
    for (int q = 0; q < kMaxHidden / 4; q++) {
      const float4 w = wr[q];
      h1[4 * q + 0] = tc::fma2(make_float2(w.x, w.x), xj, h1[4 * q + 0]);
      h1[4 * q + 1] = tc::fma2(make_float2(w.y, w.y), xj, h1[4 * q + 1]);
      h1[4 * q + 2] = tc::fma2(make_float2(w.z, w.z), xj, h1[4 * q + 2]);
      h1[4 * q + 3] = tc::fma2(make_float2(w.w, w.w), xj, h1[4 * q + 3]);
    }
  }
#pragma unroll
  for (int o = 0; o < kMaxHidden; o++) {
    if (h1[o].x < 0.0f) h1[o].x = 0.0f;
    if (h1[o].y < 0.0f) h1[o].y = 0.0f;
  }
  float2 h2[kMaxHidden];
#pragma unroll
  for (int o = 0; o < kMaxHidden; o++) h2[o] = make_float2(S.b2[o], S.b2[o]);
#pragma unroll
  for (int j = 0; j < kMaxHidden; j++) {
    const float4 *wr = reinterpret_cast<const float4 *>(S.w2T[j]);
#pragma unroll
    for (int q = 0; q < kMaxHidden / 4; q++) {
      const float4 w = wr[q];
      h2[4 * q + 0] = tc::fma2(make_float2(w.x, w.x), h1[j], h2[4 * q + 0]);
      h2[4 * q + 1] = tc::fma2(make_float2(w.y, w.y), h1[j], h2[4 * q + 1]);
      h2[4 * q + 2] = tc::fma2(make_float2(w.z, w.z), h1[j], h2[4 * q + 2]);
      h2[4 * q + 3] = tc::fma2(make_float2(w.w, w.w), h1[j], h2[4 * q + 3]);
    }
  }
  float2 d = make_float2(S.b3[0], S.b3[0]), m = make_float2(S.b3[1], S.b3[1]);
#pragma unroll
  for (int j = 0; j < kMaxHidden; j++) {
    float2 hj = h2[j];
    if (hj.x < 0.0f) hj.x = 0.0f;
    if (hj.y < 0.0f) hj.y = 0.0f;
    d = tc::fma2(make_float2(S.w3[0][j], S.w3[0][j]), hj, d);
    m = tc::fma2(make_float2(S.w3[1][j], S.w3[1][j]), hj, m);
  }
  dir = d;
  mag = m;
}

// Phase 2 (engine.py:657-710 fused_apply + optim.py:171-172 decay): features,
// MLP, update, decay; writes theta and the advanced accumulators.
template <int KIND>
__global__ void __launch_bounds__(kStrictApplyThreads)
apply_strict_kernel(DevicePlan P) {
  constexpr int D = d_feat(KIND);
  const ChunkItem it = P.apply_items[blockIdx.x];
  const TensorDesc T = P.tensors[it.tensor];
  const TensorScalars ts = P.tscal[it.tensor];
  __shared__ __align__(16) StrictMlpSmem S;
  __shared__ float tf[kTimeFeatures];
  __shared__ float red[kStrictApplyThreads / 32];
  __shared__ uint32_t bad_s;
  if (threadIdx.x < kTimeFeatures) tf[threadIdx.x] = P.step->tf[threadIdx.x];
  if (threadIdx.x == 0) bad_s = 0;
  load_strict_mlp<D>(P, T, S);
  // a non-finite gradient anywhere aborts the whole step before any write
  // (optim.py:160-165 validates every gradient before committing)
  if (*P.abort_flag) return;
  const float alpha = P.alpha, beta_out = P.beta_out;
  const float ds = P.step->ds, decay = P.step->decay;
  const bool apply_decay = P.step->apply_decay != 0;
  float maxabs = 0.0f;
  uint32_t bad = 0;
  // element A = e, element B = e + kStrictApplyThreads (a duplicate of A, not
  // stored, when it falls past the item's end)
  auto features = [&](const RawElem &r, Elem &x, float4 &ns, float *f) {
    float rowt[6], colt[6];
    unpack_elem(r, P.state_advanced, P.beta, x, ns, rowt, colt);
    strict_features<KIND>(x, rowt, colt, ts.mr, tf, f);
  };
  // engine.py:537-539: upd = dir * exp(mag*alpha) * beta; out = W + ds*upd
  auto finish = [&](int64_t e, const Elem &x, const float4 &ns, float dir, float mag) {
    const float ex = glibc_expf(__fmul_rn(mag, alpha), S.exptab);
    const float upd = __fmul_rn(__fmul_rn(dir, ex), beta_out);
    const float du = __fmul_rn(ds, upd);
    float out = __fadd_rn(x.w, du);
    maxabs = fmaxf(maxabs, fabsf(du));
    bad |= !isfinite(out);
    if (apply_decay) out = __fmul_rn(out, decay);
    T.theta[e] = out;
    if (!P.state_advanced) T.state[e - T.lo] = ns;
  };
  for (int64_t e = it.e0 + threadIdx.x; e < it.e1; e += 2 * kStrictApplyThreads) {
    const int64_t eb = e + kStrictApplyThreads;
    const bool has_b = eb < it.e1;
    Elem xa, xb;
    float4 nsa, nsb;
    float fa[D], fb[D];
    const RawElem ra = load_raw(T, e);
    const RawElem rb = load_raw(T, has_b ? eb : e);
    features(ra, xa, nsa, fa);
    features(rb, xb, nsb, fb);
    float2 dir, mag;
    strict_mlp2<D>(S, fa, fb, dir, mag);
    finish(e, xa, nsa, dir.x, mag.x);
    if (has_b) finish(eb, xb, nsb, dir.y, mag.y);
  }
  maxabs = fmaxf(maxabs, __shfl_xor_sync(0xffffffffu, maxabs, 16));
  maxabs = fmaxf(maxabs, __shfl_xor_sync(0xffffffffu, maxabs, 8));
  maxabs = fmaxf(maxabs, __shfl_xor_sync(0xffffffffu, maxabs, 4));
  maxabs = fmaxf(maxabs, __shfl_xor_sync(0xffffffffu, maxabs, 2));
  maxabs = fmaxf(maxabs, __shfl_xor_sync(0xffffffffu, maxabs, 1));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = maxabs;
  if (bad) atomicOr(&bad_s, 1u);
  __syncthreads();
  if (threadIdx.x == 0) {
    float mx = 0.0f;
    for (int w = 0; w < kStrictApplyThreads / 32; w++) mx = fmaxf(mx, red[w]);
    P.item_maxabs[blockIdx.x] = mx;
    if (bad_s) atomicOr(&P.status[it.tensor], LOPT_STATUS_NONFINITE_PARAM);
  }
}

// Per-tensor max |update| over the tensor's apply items.
__global__ void maxabs_reduce_kernel(DevicePlan P) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P.count) return;
  const TensorDesc T = P.tensors[j];
  float mx = 0.0f;
  for (int i = 0; i < T.apply_items; i++) mx = fmaxf(mx, P.item_maxabs[T.apply_item0 + i]);
  P.maxabs[j] = mx;
}

template __global__ void stats_strict_kernel<LOPT_SMALL_FC_LOPT>(DevicePlan);
template __global__ void stats_strict_kernel<LOPT_VELO_MLP>(DevicePlan);
template __global__ void apply_strict_kernel<LOPT_SMALL_FC_LOPT>(DevicePlan);
template __global__ void apply_strict_kernel<LOPT_VELO_MLP>(DevicePlan);

}  // namespace lopt

namespace lopt {

void launch_strict_stats(const DevicePlan &P, cudaStream_t s) {
  if (P.n_stat_items == 0) return;
  if (P.kind == LOPT_SMALL_FC_LOPT)
    stats_strict_kernel<LOPT_SMALL_FC_LOPT><<<P.n_stat_items, kStrictThreads, 0, s>>>(P);
  else
    stats_strict_kernel<LOPT_VELO_MLP><<<P.n_stat_items, kStrictThreads, 0, s>>>(P);
}

void launch_stats_reduce_closed(const DevicePlan &P, cudaStream_t s);
void launch_stats_reduce(const DevicePlan &P, cudaStream_t s) {
  launch_stats_reduce_closed(P, s);
}

void launch_strict_apply(const DevicePlan &P, cudaStream_t s) {
  if (P.n_apply_items == 0) return;
  if (P.kind == LOPT_SMALL_FC_LOPT)
    apply_strict_kernel<LOPT_SMALL_FC_LOPT><<<P.n_apply_items, kStrictApplyThreads, 0, s>>>(P);
  else
    apply_strict_kernel<LOPT_VELO_MLP><<<P.n_apply_items, kStrictApplyThreads, 0, s>>>(P);
}

void launch_maxabs_reduce(const DevicePlan &P, cudaStream_t s) {
  maxabs_reduce_kernel<<<(P.count + 127) / 128, 128, 0, s>>>(P);
}

}  // namespace lopt
