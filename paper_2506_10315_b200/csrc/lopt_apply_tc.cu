// lopt_apply_tc.cu -- phase 2 of the fast path on the tensor cores.
//
// engine.py:657-710 fused_apply + state.py:77-90 + optim.py:171-172 for
// 128-element tiles: features -> layer 1 (tcgen05, M=128 elements) -> ReLU ->
// layer 2 (tcgen05, plus the linear half of layer 3 as two extra output rows)
// -> layer 3's |h2| half (CUDA cores, f32; relu(x) = (x + |x|)/2) -> exp ->
// update -> decay -> store theta and the advanced accumulators.
//
// fp32 accuracy on the f16 tensor-core path: every operand is split in two
// fp16 terms and each product is x_hi*W_hi + x_lo*W_hi + x_hi*W_lo with f32
// accumulation (see PrepImage in lopt_fast.cuh for the operand layout).
//
// Default kernel (apply_pair_kernel, LOPT_APPLY_VARIANT 3): persistent, one
// CTA per SM; three producer warps stage tile *pairs* (two 128-element tiles
// of one tensor) into a ring with TMA bulk copies, and three math warpgroups
// each carry every third pair through all stages in their own two TMEM slots:
// features -> E/B operands -> layer-1 MMAs -> ReLU + fp16 split -> layer-2
// MMAs -> layer 3, update, stores.  Each CTA's pair range comes from prep's
// balance of the previous launch's per-CTA speeds (pair_range / cta_perf);
// a single-weight-set plan takes layer 3's weights from the launch parameter
// (uniform registers, DevicePlan::w3c).  DESIGN.md section 3 has the details
// and the variants measured.
//
// The older role-specialized kernel (apply_tc_kernel, LOPT_APPLY_VARIANT 1),
// kept for A/B: a warp-specialized persistent kernel, one CTA per SM, that
// streams the CTA's contiguous range of tiles through a pipeline:
//
//   producer warps --TMA bulk copies-->  smem ring of kRing tile slots
//                  (theta, g, {M1,M2,M3,V} quads, row-table entry, and the
//                   tensor's operand image when the tensor changes)
//   WG_A (128 thr) features -> E/B operands in TMEM slot   --op_ready-->
//   MMA warp L1    6 x tcgen05.mma -> acc                  --acc1_full-->
//   WG_B (128 thr) ReLU + fp16 split of h1 -> H operand    --h_ready-->
//   MMA warp L2    7 x tcgen05.mma (N = 48) -> acc         --acc2_full-->
//   WG_C (128 thr) layer 3 (|h2| FFMA2s + MMA linear half), exp, update, store theta --slot_free/data_free-->
//
// Each role has two warpgroups taking alternate tiles; ring and TMEM-slot
// positions are computed from the tile index (Pos).  Thread i of a warpgroup
// owns TMEM lane i = lane i of its tiles.  TMEM holds kSlots tiles in flight
// (kSlotCols = 80 columns each: 32 operand, 48 accumulator), so
// MMA latency is hidden by the other tiles' CUDA-core work instead of being
// waited out.  All hand-offs are mbarriers; MMAs are issued by one elected
// lane of a converged warp (descriptors in uniform registers, back-to-back
// issue).
//
// Tiles of tensors with n % 128 == 0 are (row, 128-column block) pairs in
// column-block-major order, so consecutive tiles share their column-table
// entries; other tensors use flat 128-element tiles.
#include <cstddef>
#include <cstdio>
#include <cstdlib>

#include "lopt_fast.cuh"

namespace lopt {

constexpr int kRing = 16;      // smem tile slots (prefetch + in flight)
constexpr int kSlots = 6;      // TMEM tile slots
constexpr uint32_t kSlotCols = 80;   // per slot: 32 operand columns + 48 accumulator columns
constexpr int kImgs = 4;       // smem operand images (tensor switches in flight)
// warpgroups per role (tile i goes to warpgroup i % kWGs of the role) and
// producer warps (tile i staged by producer i % kProducers)
constexpr int kWGsA = 2, kWGsB = 2, kWGsC = 2, kProducers = 2;
constexpr int kApplyThreads = (kWGsA + kWGsB + kWGsC) * 128 + (kProducers + 2) * 32;
constexpr int kWarpA = 0, kWarpB = 4 * kWGsA, kWarpC = kWarpB + 4 * kWGsB;
constexpr int kWarpProducer = kWarpC + 4 * kWGsC;
constexpr int kWarpMma1 = kWarpProducer + kProducers, kWarpMma2 = kWarpMma1 + 1;
static_assert(kWGsA < kSlots && kWGsC < kSlots && kProducers < kRing, "cursor strides");
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kOneCol = kSlotCols * kSlots;   // shared constant slice
static_assert(kOneCol + 8 <= kTmemCols, "TMEM budget");

// kFlagTail: one of the last kWGsC tiles of its tensor -- the C warps publish
// their progress there (image-buffer reuse), nowhere else
constexpr int32_t kFlagRowblock = 1, kFlagSlow = 2, kFlagTail = 4;

// Written by the producer for every tile it stages.  Lane pointers are
// pre-offset to the tile's first element, so lane i uses ptr + i.
struct __align__(16) TileMeta {
  int32_t j;        // tensor
  int32_t flags;    // kFlagRowblock | kFlagSlow (lanes read theta/g/state from global)
  int32_t v0, v1;   // valid lanes [v0, v1)
  int32_t img;      // operand image buffer
  int32_t img_par;  // parity of that buffer's current load (img_full phase)
  int32_t b0;       // rowblock: first column of the tile (column-entry cache key)
  int32_t e0, n;    // flat: element of lane 0, columns (table indices)
  int32_t pad0[3];
  float *theta;     // &theta[e0]
  const float *grad;// &grad[e0]
  float4 *state;    // &state[e0 - lo]
  const float *rowtab, *coltab;
  void *pad;
};

struct __align__(128) Stage {
  float4 st[128];       // {M1, M2, M3, V}
  float th[128];
  float gr[128];
  uint4 rowent[4];      // rowblock: the tile row's table entry
  TileMeta meta;
};

struct __align__(1024) ApplySmem {
  PrepImage img[kImgs];
  Stage stage[kRing];
  uint64_t full[kRing];        // producer -> A, B, C: tile staged (TMA complete_tx)
  uint64_t data_free[kRing];   // C -> producer (128 arrivals)
  uint64_t op_ready[kSlots];   // A -> MMA1 (128)
  uint64_t acc1_full[kSlots];  // MMA1 -> B (commit)
  uint64_t h_ready[kSlots];    // B -> MMA2 (128)
  uint64_t acc2_full[kSlots];  // MMA2 -> C (commit)
  uint64_t slot_free[kSlots];  // C -> A (one arrival per warp)
  uint64_t img_full[kImgs];    // producer -> A: operand image loaded (TMA complete_tx)
  int32_t c_done[kWGsC][4];    // C warps: last tile finished (image-buffer reuse)
  uint32_t tmem_base;
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tc::smem_u32(bar)) : "memory");
}
// Hand-off arrival of a math warpgroup: every lane arrives (count 128), each
// after its own tcgen05.wait / fence, so no intra-warp sync is needed.
__device__ __forceinline__ void warp_arrive(uint64_t *bar) {
  // every thread arrives (barriers count 128 per warpgroup): one instruction
  // per lane instead of a syncwarp / elect / arrive / syncwarp sequence
  mbar_arrive(bar);
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(tc::smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// global -> shared bulk copy (TMA engine), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          tc::smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ uint64_t f2_bits(float2 v) { return *reinterpret_cast<uint64_t *>(&v); }
__device__ __forceinline__ float2 bits_f2(uint64_t v) { return *reinterpret_cast<float2 *>(&v); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;\n" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)), "l"(f2_bits(c)));
  return bits_f2(d);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;\n" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return bits_f2(d);
}

// Two-term fp16 split of a pair, x = hi + lo: hi rounds to nearest, the
// residual x - hi is formed exactly by a mixed f32 - f16 subtract (FHADD), so
// a pair costs four instructions (no f16 -> f32 unpack).
__device__ __forceinline__ void split2(float a, float b, uint32_t &hi, uint32_t &lo) {
  asm("{\n"
      ".reg .b16 h0, h1, n0, n1;\n"
      ".reg .f32 r0, r1;\n"
      "cvt.rn.f16x2.f32 %0, %3, %2;\n"
      "mov.b32 {h0, h1}, %0;\n"
      "neg.f16 n0, h0;\n"
      "neg.f16 n1, h1;\n"
      "add.rn.f32.f16 r0, n0, %2;\n"
      "add.rn.f32.f16 r1, n1, %3;\n"
      "cvt.rn.f16x2.f32 %1, r1, r0;\n"
      "}\n"
      : "=r"(hi), "=r"(lo)
      : "f"(a), "f"(b));
}
// ReLU fused into the split: hi truncates toward zero (so the residual of a
// positive value is non-negative) and both conversions clamp at 0.
__device__ __forceinline__ void relu_split2(float a, float b, uint32_t &hi, uint32_t &lo) {
  asm("{\n"
      ".reg .b16 h0, h1, n0, n1;\n"
      ".reg .f32 r0, r1;\n"
      "cvt.rz.relu.f16x2.f32 %0, %3, %2;\n"
      "mov.b32 {h0, h1}, %0;\n"
      "neg.f16 n0, h0;\n"
      "neg.f16 n1, h1;\n"
      "add.rn.f32.f16 r0, n0, %2;\n"
      "add.rn.f32.f16 r1, n1, %3;\n"
      "cvt.rn.relu.f16x2.f32 %1, r1, r0;\n"
      "}\n"
      : "=r"(hi), "=r"(lo)
      : "f"(a), "f"(b));
}

// The producer (one lane): walks the CTA's tiles in order and stages each one
// with bulk copies (theta, g, the state quads of the valid lanes, the row's
// table entry for row-block tiles, the tensor's operand image on a switch).
struct Producer {
  int j = -1;
  int32_t left = 0;               // tiles of tensor j still to stage
  int32_t a = 0, b0 = 0, e0 = 0;  // rowblock: row, first column; flat: first element
  int32_t n = 1, lo = 0, hi = 0, a_lo = 0, a_end = 0;
  bool rb = false, aligned = false;
  float *theta = nullptr;
  const float *grad = nullptr, *rowtab = nullptr, *coltab = nullptr;
  float4 *state = nullptr;

  __device__ __forceinline__ void load_tensor(const DevicePlan &P, int jj, int32_t q) {
    const TensorDesc *T = P.tensors + jj;
    j = jj;
    n = (int32_t)T->n;
    lo = (int32_t)T->lo;
    hi = (int32_t)T->hi;
    rb = T->rowblock != 0;
    a_lo = T->a_lo;
    a_end = T->a_lo + T->m_rows;
    theta = T->theta;
    grad = T->grad;
    state = T->state;
    rowtab = T->rowtab;
    coltab = T->coltab;
    aligned = ((reinterpret_cast<uintptr_t>(theta) | reinterpret_cast<uintptr_t>(grad)) & 15) == 0;
    left = T->tiles - q;
    if (rb) {
      const int32_t mr = T->m_rows;
      a = a_lo + q % mr;
      b0 = (q / mr) * kTile;
    } else {
      e0 = lo + q * kTile;
    }
  }

  __device__ __forceinline__ void seek(const DevicePlan &P, int32_t t) {
    int jj = 0;
    while (jj + 1 < P.count && P.tensors[jj + 1].tile0 <= t) jj++;
    while (P.tensors[jj].tiles == 0 && jj + 1 < P.count) jj++;
    load_tensor(P, jj, t - (int32_t)P.tensors[jj].tile0);
  }

  __device__ __forceinline__ void advance(const DevicePlan &P) {
    if (--left == 0) {
      int jj = j + 1;
      while (jj < P.count && P.tensors[jj].tiles == 0) jj++;
      if (jj < P.count) load_tensor(P, jj, 0);
      return;
    }
    if (rb) {
      if (++a == a_end) {
        a = a_lo;
        b0 += kTile;
      }
    } else {
      e0 += kTile;
    }
  }

  __device__ __forceinline__ void stage(Stage &st, uint64_t *full, int img, int img_par,
                                        int tail_tiles = kWGsC) {
    TileMeta mt;
    mt.j = j;
    mt.b0 = b0;
    const int32_t el0 = rb ? a * n + b0 : e0;
    mt.e0 = el0;
    mt.n = n;
    int32_t v0 = max(0, lo - el0), v1 = min(kTile, hi - el0);
    if (v1 <= v0) v0 = v1 = 0;
    mt.v0 = v0;
    mt.v1 = v1;
    const bool fast = aligned && ((el0 + v0) & 3) == 0 && ((v1 - v0) & 3) == 0;
    mt.flags = (rb ? kFlagRowblock : 0) | (fast ? 0 : kFlagSlow) | (left <= tail_tiles ? kFlagTail : 0);
    mt.img = img;
    mt.img_par = img_par;
    mt.pad0[0] = mt.pad0[1] = mt.pad0[2] = 0;
    mt.theta = theta + el0;
    mt.grad = grad + el0;
    mt.state = state + (el0 - lo);
    mt.rowtab = rowtab;
    mt.coltab = coltab;
    mt.pad = nullptr;
    st.meta = mt;
    const uint32_t nv = (uint32_t)(v1 - v0);
    const uint32_t bytes = (fast ? 24u * nv : 0u) + (rb ? 64u : 0u);
    mbar_arrive_tx(full, bytes);
    if (fast && nv > 0) {
      bulk_g2s(&st.th[v0], theta + el0 + v0, 4 * nv, full);
      bulk_g2s(&st.gr[v0], grad + el0 + v0, 4 * nv, full);
      bulk_g2s(&st.st[v0], state + (el0 + v0 - lo), 16 * nv, full);
    }
    if (rb) bulk_g2s(st.rowent, rowtab + (int64_t)a * kRowTab, 64, full);
  }
};

// x5 x6 x7 and the scaled fp16 hi/lo operand words of a row/column table entry
struct Entry {
  float x[3];
  uint32_t hi[3], lo[3];
};
__device__ __forceinline__ void load_entry(const float *tab, int32_t i, Entry &E) {
  const uint4 *p = reinterpret_cast<const uint4 *>(tab + (int64_t)i * kRowTab);
  const uint4 v = __ldg(p), h = __ldg(p + 2), l = __ldg(p + 3);
  E.x[0] = __uint_as_float(v.x); E.x[1] = __uint_as_float(v.y); E.x[2] = __uint_as_float(v.z);
  E.hi[0] = h.x; E.hi[1] = h.y; E.hi[2] = h.z;
  E.lo[0] = l.x; E.lo[1] = l.y; E.lo[2] = l.z;
}

// MMA issue.  `dimg` is the UMMA descriptor of the tile's operand image (its
// first byte); every B slice is a constant 16-byte offset from it, so a tile
// costs one uniform add per MMA instead of rebuilding descriptors.
constexpr uint64_t slice_off(size_t bytes) { return (uint64_t)(bytes >> 4); }
template <bool kCommit = true>
__device__ __forceinline__ void issue_layer1(uint64_t dimg, uint32_t op, uint32_t acc, uint64_t *bar) {
  constexpr uint32_t idesc = tc::idesc_f16_f32(128, 32);
  const uint64_t w_eh = dimg + slice_off(offsetof(PrepImage, b1[0]));
  const uint64_t w_el = dimg + slice_off(offsetof(PrepImage, b1[1]));
  const uint64_t w_bh = dimg + slice_off(offsetof(PrepImage, b1[2]));
  const uint64_t w_bl = dimg + slice_off(offsetof(PrepImage, b1[3]));
  tc::mma_ts(acc, op + 0, w_eh, idesc, 0);
  tc::mma_ts(acc, op + 8, w_eh, idesc, 1);
  tc::mma_ts(acc, op + 0, w_el, idesc, 1);
  tc::mma_ts(acc, op + 16, w_bh, idesc, 1);
  tc::mma_ts(acc, op + 24, w_bh, idesc, 1);
  tc::mma_ts(acc, op + 16, w_bl, idesc, 1);
  if (kCommit) tc::mma_commit(bar);
}
__device__ __forceinline__ void issue_layer1_nc(uint64_t dimg, uint32_t op, uint32_t acc) {
  issue_layer1<false>(dimg, op, acc, nullptr);
}

// H operand column layout: kHInter = false: [hi K0-15 | hi K16-31 | lo K0-15 |
// lo K16-31] (8 columns each); true: [hi K0-15 | lo K0-15 | hi K16-31 | lo
// K16-31], so each 16-unit half of the layer-1 epilogue is one 16-column store.
template <bool kCommit = true, bool kHInter = false>
__device__ __forceinline__ void issue_layer2(uint64_t dimg, uint32_t op, uint32_t acc,
                                             uint32_t one, uint64_t *bar) {
  constexpr uint32_t idesc = tc::idesc_f16_f32(128, kN2);
  const uint64_t h0 = dimg + slice_off(offsetof(PrepImage, b2[0]));
  const uint64_t h1 = dimg + slice_off(offsetof(PrepImage, b2[1]));
  const uint64_t l0 = dimg + slice_off(offsetof(PrepImage, b2[2]));
  const uint64_t l1 = dimg + slice_off(offsetof(PrepImage, b2[3]));
  const uint64_t bb = dimg + slice_off(offsetof(PrepImage, b2[4]));
  constexpr uint32_t kHi0 = 0, kHi1 = kHInter ? 16 : 8, kLo0 = kHInter ? 8 : 16, kLo1 = 24;
  tc::mma_ts(acc, op + kHi0, h0, idesc, 0);
  tc::mma_ts(acc, op + kHi1, h1, idesc, 1);
  tc::mma_ts(acc, op + kLo0, h0, idesc, 1);
  tc::mma_ts(acc, op + kLo1, h1, idesc, 1);
  tc::mma_ts(acc, op + kHi0, l0, idesc, 1);
  tc::mma_ts(acc, op + kHi1, l1, idesc, 1);
  tc::mma_ts(acc, one, bb, idesc, 1);
  if (kCommit) tc::mma_commit(bar);
}
__device__ __forceinline__ void issue_layer2_nc(uint64_t dimg, uint32_t op, uint32_t acc, uint32_t one) {
  issue_layer2<false, true>(dimg, op, acc, one, nullptr);
}

__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}
// max that propagates NaN (any non-finite update poisons the tensor's flag)
__device__ __forceinline__ float max_nan_abs(float m, float x) {
  float y;
  asm("max.NaN.f32 %0, %1, %2;\n" : "=f"(y) : "f"(m), "f"(fabsf(x)));
  return y;
}

// Timing trace (LOPT_APPLY_DEBUG & 32): CTA 0 records clock64 at the pipeline
// hand-offs of its first kTraceTiles tiles.
constexpr int kTraceTiles = 64;
constexpr int kTraceEvents = 12;
__device__ long long g_trace[kTraceTiles][kTraceEvents];
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace(const DevicePlan &P, int32_t i, int ev) {
#ifdef LOPT_TRACE
  if ((P.dbg & 32) && blockIdx.x == 0 && i < kTraceTiles && (threadIdx.x & 31) == 0)
    g_trace[i][ev] = clock64();
#endif
}

// Ring position of a role: slot index and phase parity, advanced per tile.
template <int N>
struct Cursor {
  int i = 0;
  uint32_t phase = 0;
  bool wrapped = false;
  __device__ __forceinline__ void next() {
    if (++i == N) {
      i = 0;
      phase ^= 1u;
      wrapped = true;
    }
  }
};

#ifdef LOPT_WATCHDOG
__device__ __forceinline__ void wd_wait(uint64_t *bar, uint32_t parity, int tag, int32_t i) {
  long long n = 0;
  while (!tc::mbar_try(bar, parity)) {
    if (++n == (1ll << 24) && blockIdx.x < 3 && (threadIdx.x & 31) == 0) {
      printf("apply hang: block %d warp %d tag %d tile %d parity %u\n", blockIdx.x,
             threadIdx.x >> 5, tag, i, parity);
    }
  }
}
#define WAIT(bar, par, tag) wd_wait(bar, par, tag, i)
#else
#define WAIT(bar, par, tag) tc::mbar_wait(bar, par)
#endif

// Ring / slot position of tile t, computed directly (a power-of-two ring is
// two bit operations, the 6-slot TMEM ring a multiply-high): cheaper than
// carrying wrap-around cursors through the loop.
template <int N>
struct Pos {
  int i;
  uint32_t phase;
  bool wrapped;
  __device__ __forceinline__ explicit Pos(int32_t t) {
    const uint32_t u = (uint32_t)t;
    i = (int)(u % (uint32_t)N);
    phase = (u / (uint32_t)N) & 1u;
    wrapped = u >= (uint32_t)N;
  }
};

template <int KIND>
__global__ void __launch_bounds__(kApplyThreads, 1) apply_tc_kernel(DevicePlan P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  ApplySmem &S = *reinterpret_cast<ApplySmem *>(smem_raw);
  const int tid = threadIdx.x;
  // warp-uniform role index the compiler can prove uniform
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int row = tid & 127;
  if (warp == 0) {
    tc::tmem_alloc(&S.tmem_base, kTmemCols);
    tc::tmem_relinquish();
  }
  if (tid == 0) {
    for (int r = 0; r < kRing; r++) {
      tc::mbar_init(&S.full[r], 1);
      tc::mbar_init(&S.data_free[r], 128);
    }
    for (int b = 0; b < kImgs; b++) tc::mbar_init(&S.img_full[b], 1);
    for (int w = 0; w < kWGsC; w++)
      for (int q = 0; q < 4; q++) S.c_done[w][q] = -1;
    for (int s = 0; s < kSlots; s++) {
      tc::mbar_init(&S.op_ready[s], 128);
      tc::mbar_init(&S.acc1_full[s], 1);
      tc::mbar_init(&S.h_ready[s], 128);
      tc::mbar_init(&S.acc2_full[s], 1);
      tc::mbar_init(&S.slot_free[s], 128);
    }
    tc::mbar_fence_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = S.tmem_base;
  const uint32_t lane_addr = (uint32_t)((warp & 3) * 32) << 16;
  if (warp >= kWarpC && warp < kWarpC + 4) {
    // the constant slice that selects the layer-2 bias: fp16 {1, 1, 0, ...}
    const uint32_t one[8] = {0x3C003C00u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    tc::tmem_st8(tbase + lane_addr + kOneCol, one);
    tc::tmem_st_wait();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const bool aborted = *P.abort_flag != 0;
  const int32_t tb = (int32_t)(P.n_tiles * blockIdx.x / gridDim.x);
  const int32_t te = (int32_t)(P.n_tiles * (blockIdx.x + 1) / gridDim.x);
  const int32_t nt = aborted ? 0 : te - tb;

  if (warp >= kWarpProducer && warp < kWarpProducer + kProducers) {
    // -------------------------------------------------------------- producers
    // Producer p stages the tiles of parity p; both walk every tile so they
    // agree on the tensor sequence (image buffer k % kImgs for the k-th
    // tensor of this CTA's range).  The producer whose tile opens a tensor
    // loads its operand image once the C warps are done with the buffer.
    const int p = warp - kWarpProducer;
    if (tc::elect_one() && nt > 0) {
      Producer pr;
      pr.seek(P, tb);
      int k = -1, img = 0, cur_j = -1;
      uint32_t par_bits = 0;
      int32_t first0 = 0, first1 = 0, first2 = 0, first3 = 0;   // first tile of the tensor in buffer b
      Cursor<kRing> rc;
      for (int32_t i = 0; i < nt; i++) {
        if (pr.j != cur_j) {
          cur_j = pr.j;
          k++;
          img = k & (kImgs - 1);
          const int32_t pf = img == 0 ? first0 : img == 1 ? first1 : img == 2 ? first2 : first3;
          const int nb = (k + 1) & (kImgs - 1);   // buffer of tensor k - 3
          const int32_t nf = nb == 0 ? first0 : nb == 1 ? first1 : nb == 2 ? first2 : first3;
          if (img == 0) first0 = i; else if (img == 1) first1 = i; else if (img == 2) first2 = i; else first3 = i;
          if (k >= kImgs) par_bits ^= 1u << img;
          if (i % kProducers == p) {
            if (k >= kImgs) {
              // tensor k - kImgs used tiles [pf, nf - 1]: every C warp must be
              // past the last tile of its parity in that range
              const int32_t last = nf - 1;
              for (int w = 0; w < kWGsC; w++) {
                const int32_t need = last - (((last - w) % kWGsC) + kWGsC) % kWGsC;
                if (need < pf) continue;
                for (int q = 0; q < 4; q++) {
                  int32_t d;
                  while (true) {
                    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];\n"
                                 : "=r"(d)
                                 : "r"(tc::smem_u32(&S.c_done[w][q]))
                                 : "memory");
                    if (d >= need) break;
                    __nanosleep(32);
                  }
                }
              }
            }
            mbar_arrive_tx(&S.img_full[img], (uint32_t)sizeof(PrepImage));
            bulk_g2s(&S.img[img], reinterpret_cast<const PrepImage *>(P.prep) + pr.j,
                     (uint32_t)sizeof(PrepImage), &S.img_full[img]);
          }
        }
        if (i % kProducers == p) {
          if (rc.wrapped) WAIT(&S.data_free[rc.i], rc.phase ^ 1u, 1);
          trace(P, i, 0);
          pr.stage(S.stage[rc.i], &S.full[rc.i], img, (int)((par_bits >> img) & 1u));
        }
        pr.advance(P);
        rc.next();
      }
    }
    __syncwarp();
  } else if (warp == kWarpMma1 || warp == kWarpMma2) {
    // --------------------------------------------------------------- MMA warps
    const bool l1 = warp == kWarpMma1;
    const uint32_t one = tbase + kOneCol;
    // layer-1 slices are N = 32 rows (LBO 512 B), layer-2 slices N = 48 (LBO 768 B)
    const uint64_t dimg0 = tc::smem_desc_kmajor(tc::smem_u32(&S.img[0]), l1 ? 512 : kN2 * 16, 128);
    for (int32_t i = 0; i < nt; i++) {
      const Pos<kRing> rc(i);
      const Pos<kSlots> sc(i);
      WAIT(l1 ? &S.op_ready[sc.i] : &S.h_ready[sc.i], sc.phase, 4);
      tc::fence_after_sync();
      trace(P, i, l1 ? 3 : 5);
      const uint64_t dimg =
          dimg0 + (uint64_t)((uint32_t)S.stage[rc.i].meta.img * (uint32_t)(sizeof(PrepImage) >> 4));
      const uint32_t op = tbase + kSlotCols * sc.i, acc = op + 32;
      if (tc::elect_one()) {
        if (l1) issue_layer1(dimg, op, acc, &S.acc1_full[sc.i]);
        else issue_layer2(dimg, op, acc, one, &S.acc2_full[sc.i]);
      }
      __syncwarp();
    }
  } else if (warp < kWarpB) {
    // ------------------------------------------ WG_A: features -> E/B operands
    const int r0 = (warp - kWarpA) >> 2;
    constexpr int kStep = kWGsA;
    const bool adv = P.state_advanced != 0;
    const float *beta = P.beta;
    int32_t col_j = -1, col_b0 = -1;   // rowblock: cached column entry of this lane
    int32_t a_img = -1, a_par = -1;    // operand image last waited for
    Entry ce;
    for (int32_t i = r0; i < nt; i += kStep) {
      const Pos<kRing> rc(i);
      const Pos<kSlots> sc(i);
      WAIT(&S.full[rc.i], rc.phase, 5);
      if (warp == 0) trace(P, i, 1);
      const Stage &st = S.stage[rc.i];
      const TileMeta &mt = st.meta;
      const int32_t flags = mt.flags;
      const bool valid = row >= mt.v0 && row < mt.v1;
      if (mt.img != a_img || mt.img_par != a_par) {   // a new operand image: wait for its load
        WAIT(&S.img_full[mt.img], (uint32_t)mt.img_par, 9);
        a_img = mt.img;
        a_par = mt.img_par;
      }
      const PrepImage &im = S.img[mt.img];
      float4 *sp = mt.state + row;
      float w, g;
      float4 sq4;
      if (!(flags & kFlagSlow)) {
        w = st.th[row];
        g = st.gr[row];
        sq4 = st.st[row];
      } else {
        w = valid ? mt.theta[row] : 0.0f;
        g = valid ? mt.grad[row] : 0.0f;
        sq4 = valid ? *sp : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      Entry re;
      if (flags & kFlagRowblock) {
        const uint4 v = st.rowent[0], hh = st.rowent[2], ll = st.rowent[3];
        re.x[0] = __uint_as_float(v.x); re.x[1] = __uint_as_float(v.y); re.x[2] = __uint_as_float(v.z);
        re.hi[0] = hh.x; re.hi[1] = hh.y; re.hi[2] = hh.z;
        re.lo[0] = ll.x; re.lo[1] = ll.y; re.lo[2] = ll.z;
        if (mt.j != col_j || mt.b0 != col_b0) {
          col_j = mt.j;
          col_b0 = mt.b0;
          load_entry(mt.coltab, mt.b0 + row, ce);
        }
      } else {
        const int32_t ec = mt.e0 + (valid ? row : (mt.v1 > mt.v0 ? mt.v0 : 0));
        const int32_t la = (int32_t)((uint32_t)ec / (uint32_t)mt.n);
        load_entry(mt.rowtab, la, re);
        load_entry(mt.coltab, ec - la * mt.n, ce);
        col_j = -1;
      }
      FastIn x;
      x.w = w;
      advance(g, sq4, adv, beta, x);
      // the accumulators do not depend on the MLP: store them right away
      if (valid && !adv) *sp = make_float4(x.m1, x.m2, x.m3, x.v);
      const float sq[3] = {im.sqmr[0], im.sqmr[1], im.sqmr[2]};
      float f[16];
      fast_features(x, re.x, ce.x, sq, f);
      // normalize (features.py:349-354) so every operand fits fp16
      const float4 *es = reinterpret_cast<const float4 *>(im.escale);
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const float4 e4 = es[q];
        const float2 p0 = fmul2(make_float2(f[4 * q], f[4 * q + 1]), make_float2(e4.x, e4.y));
        const float2 p1 = fmul2(make_float2(f[4 * q + 2], f[4 * q + 3]), make_float2(e4.z, e4.w));
        f[4 * q] = p0.x; f[4 * q + 1] = p0.y; f[4 * q + 2] = p1.x; f[4 * q + 3] = p1.y;
      }
      uint32_t ev[16];   // E_hi(8) E_lo(8)
#pragma unroll
      for (int q = 0; q < 8; q++) split2(f[2 * q], f[2 * q + 1], ev[q], ev[8 + q]);
      uint32_t xh = 0, xl = 0;
      if (KIND == LOPT_VELO_MLP) split2(clip01(x.g) * im.escale[16], 0.0f, xh, xl);
      uint32_t bv[16];   // B_hi(8) B_lo(8)
      bv[0] = re.hi[0]; bv[1] = re.hi[1]; bv[2] = re.hi[2];
      bv[3] = ce.hi[0]; bv[4] = ce.hi[1]; bv[5] = ce.hi[2];
      bv[6] = (xh & 0xFFFFu) | 0x3C000000u;   // clip_hi, fp16 1 (bias)
      bv[7] = 0u;
      bv[8] = re.lo[0]; bv[9] = re.lo[1]; bv[10] = re.lo[2];
      bv[11] = ce.lo[0]; bv[12] = ce.lo[1]; bv[13] = ce.lo[2];
      bv[14] = xl & 0xFFFFu;
      bv[15] = 0u;
      // TMEM slot is free once C has read the tile kSlots before
      if (warp == 0) trace(P, i, 8);
      if (sc.wrapped) WAIT(&S.slot_free[sc.i], sc.phase ^ 1u, 6);
      tc::fence_after_sync();
      const uint32_t ta = tbase + lane_addr + kSlotCols * sc.i;
      tc::tmem_st16(ta, ev);
      tc::tmem_st16(ta + 16, bv);
      tc::tmem_st_wait();
      tc::fence_before_sync();
      if (warp == 0) trace(P, i, 2);
      warp_arrive(&S.op_ready[sc.i]);
    }
  } else if (warp < kWarpC) {
    // ------------------------------------------- WG_B: layer-1 epilogue -> H
    const int r0 = (warp - kWarpB) >> 2;
    constexpr int kStep = kWGsB;
    for (int32_t i = r0; i < nt; i += kStep) {
      const Pos<kSlots> sc(i);
      // B touches neither the data ring nor the operand image (the layer-1
      // scale 2^-s2 is folded into W1): it waits for the accumulator only
      if (warp == kWarpB) trace(P, i, 10);
      WAIT(&S.acc1_full[sc.i], sc.phase, 7);
      tc::fence_after_sync();
      if (warp == kWarpB) trace(P, i, 4);
      const uint32_t ta = tbase + lane_addr + kSlotCols * sc.i;
#pragma unroll
      for (int half = 0; half < 2; half++) {
        uint32_t h[16];
        tc::tmem_ld16(ta + 32 + 16 * half, h);
        tc::tmem_ld_wait();
        uint32_t hi[8], lo[8];
#pragma unroll
        for (int q = 0; q < 8; q++)
          relu_split2(__uint_as_float(h[2 * q]), __uint_as_float(h[2 * q + 1]), hi[q], lo[q]);
        tc::tmem_st8(ta + 8 * half, hi);
        tc::tmem_st8(ta + 16 + 8 * half, lo);
      }
      tc::tmem_st_wait();
      tc::fence_before_sync();
      warp_arrive(&S.h_ready[sc.i]);
    }
  } else if (warp < kWarpProducer) {
    // ------------------------- WG_C: layer-2 epilogue, layer 3, update, store
    const int r0 = (warp - kWarpC) >> 2;
    constexpr int kStep = kWGsC;
    const float alpha_log2e = P.alpha * 1.4426950408889634f;
    const float dsb = P.step->ds * P.beta_out;
    const float decay = P.step->apply_decay != 0 ? P.step->decay : 1.0f;
    const int n_peers = P.n_peers;
    int red_j = -1;
    float red_max = 0.0f, red_out = 0.0f;   // max |delta|, NaN-propagating max |theta'|
    for (int32_t i = r0; i < nt; i += kStep) {
      const Pos<kRing> rc(i);
      const Pos<kSlots> sc(i);
      WAIT(&S.full[rc.i], rc.phase, 5);
      const Stage &st = S.stage[rc.i];
      const TileMeta &mt = st.meta;
      const int j = mt.j;
      const int32_t mt_flags = mt.flags;
      if (j != red_j) {
        if (red_j >= 0) {
          if (red_max > 0.0f)
            atomicMax(reinterpret_cast<unsigned int *>(&P.maxabs[red_j]), __float_as_uint(red_max));
          if (!(red_out <= 3.402823466e38f)) atomicOr(&P.status[red_j], LOPT_STATUS_NONFINITE_PARAM);
        }
        red_j = j;
        red_max = 0.0f;
        red_out = 0.0f;
      }
      const bool valid = row >= mt.v0 && row < mt.v1;
      float *tp = mt.theta + row;
      const float w = (mt.flags & kFlagSlow) ? (valid ? *tp : 0.0f) : st.th[row];
      const PrepImage &ip = S.img[mt.img];
      if (warp == kWarpC) trace(P, i, 9);
      WAIT(&S.acc2_full[sc.i], sc.phase, 8);
      tc::fence_after_sync();
      if (warp == kWarpC) trace(P, i, 6);
      // layer 3 in f32: (b3 + linear half, from the MMA) + sum (w3/2)|h2| as
      // {dir, mag} pairs -- |h2[j]| is a broadcast operand with the |x|
      // modifier, two chains (even / odd j); h2 is read in two 16-column
      // halves to stay within the register budget
      const uint32_t tc2 = tbase + lane_addr + kSlotCols * sc.i + 32;
      uint32_t h2[16], lin[2];
      tc::tmem_ld16(tc2, h2);
      tc::tmem_ld2(tc2 + 32, lin);
      tc::tmem_ld_wait();
      float2 de = make_float2(__uint_as_float(lin[0]), __uint_as_float(lin[1]));
      float2 dd = make_float2(0.0f, 0.0f);
      const float4 *w3 = reinterpret_cast<const float4 *>(ip.w3h);
#pragma unroll
      for (int half = 0; half < 2; half++) {
        if (half == 1) {
          tc::tmem_ld16(tc2 + 16, h2);
          tc::tmem_ld_wait();
          tc::fence_before_sync();
          warp_arrive(&S.slot_free[sc.i]);
        }
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const float4 w = w3[8 * half + q];
          const float he = fabsf(__uint_as_float(h2[2 * q])), ho = fabsf(__uint_as_float(h2[2 * q + 1]));
          de = ffma2(make_float2(he, he), make_float2(w.x, w.y), de);
          dd = ffma2(make_float2(ho, ho), make_float2(w.z, w.w), dd);
        }
      }
      // the data slot (theta, meta) and the image are no longer needed
      warp_arrive(&S.data_free[rc.i]);
      if ((mt_flags & kFlagTail) && (threadIdx.x & 31) == 0)
        asm volatile("st.release.cta.shared.b32 [%0], %1;\n" ::"r"(tc::smem_u32(&S.c_done[r0][warp & 3])),
                     "r"(i)
                     : "memory");
      const float dir = de.x + dd.x, mag = de.y + dd.y;
      // engine.py:537-539, exp on the SFU (fp32 tolerance path)
      const float du = dsb * (dir * ex2_ftz(mag * alpha_log2e));
      const float out = (w + du) * decay;   // optim.py:100-101 (decay = 1 without weight decay)
      if (valid) {
        red_max = fmaxf(red_max, fabsf(du));
        red_out = max_nan_abs(red_out, out);
        *tp = out;
        // fused all-gather: the same value into every peer's copy (NVLink
        // stores through the peers' mapped arenas)
        for (int q = 0; q < n_peers; q++)
          *reinterpret_cast<float *>(reinterpret_cast<char *>(tp) + P.peer_delta[q]) = out;
      }
      if (warp == kWarpC) trace(P, i, 7);
    }
    if (red_j >= 0) {
      if (red_max > 0.0f)
        atomicMax(reinterpret_cast<unsigned int *>(&P.maxabs[red_j]), __float_as_uint(red_max));
      if (!(red_out <= 3.402823466e38f)) atomicOr(&P.status[red_j], LOPT_STATUS_NONFINITE_PARAM);
    }
    if (n_peers > 0) __threadfence_system();   // peer stores performed before the caller's barrier
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, kTmemCols);
}

// ---------------------------------------------------------------------------
// Pair pipeline (the default; LOPT_APPLY_VARIANT=1 selects the role-specialized
// kernel above).  Every math warpgroup carries its own tiles through all
// stages -- features, layer-1 MMAs, layer-1 epilogue, layer-2 MMAs, layer 3 +
// update -- in its own TMEM slots, issuing its MMAs from an elected lane of its
// first warp; the warpgroups interleave, so while one waits for its MMAs the
// others compute, and there are no hand-offs between roles (the per-iteration
// waits are the warpgroup's TMA data and its two MMA commits).  Each iteration
// carries a PAIR of 128-element tiles in two TMEM slots (rowblock tensors: rows
// 2r and 2r+1 of one column block, so the pair shares its column-table entries;
// flat tensors: tiles 2q, 2q+1; a missing second tile is an empty tile): one
// data-ring wait, one image check, one w3 read, two MMA commits and two
// warpgroup barriers per 256 elements, and two independent elements per thread
// for ILP between the MMA waits.  Measured against the role-specialized kernel
// (ncu, ViT-B/16): 396 vs 516 thread-instructions per element, 1.61 vs 1.84 ms.
#ifndef LOPT_PRING
#define LOPT_PRING 9    // data-ring depth in pairs, 3 per warpgroup (same-box ncu: 12: +0.7 %, 6: +0.3 %)
#endif
#ifndef LOPT_ACC_SLEEP
#define LOPT_ACC_SLEEP 0   // MMA-commit waits parked in hardware (suspend hint)
#endif
#ifndef LOPT_STATE_EARLY
#define LOPT_STATE_EARLY 0 // advanced accumulators stored before the layer-1 issue
#endif
#ifndef LOPT_EPI_PREFETCH
#define LOPT_EPI_PREFETCH 0   // layer-1 epilogue: both halves' TMEM loads before one wait
#endif
#ifndef LOPT_L3_CHAINS8
#define LOPT_L3_CHAINS8 0   // layer 3: eight FFMA2 chains, all TMEM loads before one wait
#endif
#ifndef LOPT_L1_SPLIT
#define LOPT_L1_SPLIT 0   // tile 0's layer-1 MMAs issued before tile 1's features
#endif
#ifndef LOPT_FEAT_ILP
#define LOPT_FEAT_ILP 0   // both tiles' operands computed before their TMEM stores
#endif
#ifndef LOPT_PPROD
#define LOPT_PPROD 3    // producer warps, one per math warpgroup (same-box ncu A/B: 4: +0.7 %, 2: +4.5 %)
#endif
constexpr int kPWGs = 3;
constexpr int kPRing = LOPT_PRING;
constexpr int kPProducers = LOPT_PPROD;
constexpr int kPThreads = kPWGs * 128 + kPProducers * 32;
constexpr int kPWarpProducer = kPWGs * 4;
constexpr uint32_t kPOneCol = 2 * kSlotCols * kPWGs;
static_assert(kPOneCol + 8 <= kTmemCols, "TMEM budget");

struct __align__(128) PairStage {
  float4 st[2][128];     // {M1, M2, M3, V}
  float th[2][128];
  float gr[2][128];
  uint4 rowent[2][4];    // rowblock: each tile row's table entry
  TileMeta meta[2];
};

struct __align__(1024) PairSmem {
  PrepImage img[kImgs];
  PairStage stage[kPRing];
  uint64_t full[kPRing];       // producer -> WG: pair staged (TMA complete_tx)
  uint64_t data_free[kPRing];  // WG -> producer (128 arrivals)
  uint64_t acc[kPWGs];         // MMA commits of the WG (two phases per pair)
  uint64_t img_full[kImgs];    // producer -> WGs: operand image loaded
  int32_t done[kPWGs][4];      // WG warps: last pair finished (image-buffer reuse)
  uint32_t tmem_base;
  uint64_t t_start;            // CTA start (globaltimer), for the balance record
  // fused all-gather: each WG stages its pair's updated theta (double
  // buffered) for the 16-byte peer stores
  __align__(16) float peer_stage[kPWGs][2][2][128];
};

// Walks a CTA's pairs in order (one lane), staging both tiles of each.
struct PairProducer {
  int j = -1;
  int32_t left = 0;                 // pairs of tensor j still to stage
  int32_t hp = 1, rp = 0, b0 = 0;   // rowblock: row pairs per column block, row pair, first column
  int32_t e0 = 0;                   // flat: first element of the pair
  int32_t n = 1, lo = 0, hi = 0, a_lo = 0, mr = 0;
  bool rb = false, aligned = false;
  float *theta = nullptr;
  const float *grad = nullptr, *rowtab = nullptr, *coltab = nullptr;
  float4 *state = nullptr;

  __device__ __forceinline__ void load_tensor(const DevicePlan &P, int jj, int32_t q) {
    const TensorDesc *T = P.tensors + jj;
    j = jj;
    n = (int32_t)T->n;
    lo = (int32_t)T->lo;
    hi = (int32_t)T->hi;
    rb = T->rowblock != 0;
    a_lo = T->a_lo;
    mr = T->m_rows;
    theta = T->theta;
    grad = T->grad;
    state = T->state;
    rowtab = T->rowtab;
    coltab = T->coltab;
    aligned = ((reinterpret_cast<uintptr_t>(theta) | reinterpret_cast<uintptr_t>(grad)) & 15) == 0;
    left = T->pairs - q;
    if (rb) {
      hp = (mr + 1) >> 1;
      rp = q % hp;
      b0 = (q / hp) * kTile;
    } else {
      e0 = lo + q * 2 * kTile;
    }
  }
  __device__ __forceinline__ void seek(const DevicePlan &P, int32_t t) {
    // last tensor whose first pair is <= t (pair0 is non-decreasing)
    int jj = 0, hi_ = P.count - 1;
    while (jj < hi_) {
      const int mid = (jj + hi_ + 1) >> 1;
      if (P.tensors[mid].pair0 <= t) jj = mid;
      else hi_ = mid - 1;
    }
    while (P.tensors[jj].pairs == 0 && jj + 1 < P.count) jj++;
    load_tensor(P, jj, t - (int32_t)P.tensors[jj].pair0);
  }
  __device__ __forceinline__ void advance(const DevicePlan &P) {
    if (--left == 0) {
      int jj = j + 1;
      while (jj < P.count && P.tensors[jj].pairs == 0) jj++;
      if (jj < P.count) load_tensor(P, jj, 0);
      return;
    }
    if (rb) {
      if (++rp == hp) {
        rp = 0;
        b0 += kTile;
      }
    } else {
      e0 += 2 * kTile;
    }
  }
  __device__ __forceinline__ void stage(PairStage &st, uint64_t *full, int img, int img_par) {
    int32_t el[2], va[2], vb[2];
    bool fast[2], ex[2];
    int32_t arow[2];
    uint32_t bytes = 0;
#pragma unroll
    for (int k = 0; k < 2; k++) {
      if (rb) {
        ex[k] = 2 * rp + k < mr;
        arow[k] = a_lo + (ex[k] ? 2 * rp + k : 0);
        el[k] = arow[k] * n + b0;
      } else {
        el[k] = e0 + k * kTile;
        ex[k] = el[k] < hi;
        if (!ex[k]) el[k] = lo;
        arow[k] = 0;
      }
      int32_t v0 = max(0, lo - el[k]), v1 = min(kTile, hi - el[k]);
      if (!ex[k] || v1 <= v0) v0 = v1 = 0;
      va[k] = v0;
      vb[k] = v1;
      // an empty tile reads nothing: the slow path with no valid lanes yields zeros
      fast[k] = ex[k] && aligned && ((el[k] + v0) & 3) == 0 && ((v1 - v0) & 3) == 0;
      TileMeta mt;
      mt.j = j;
      mt.b0 = b0;
      mt.e0 = el[k];
      mt.n = n;
      mt.v0 = v0;
      mt.v1 = v1;
      mt.flags = (rb ? kFlagRowblock : 0) | (fast[k] ? 0 : kFlagSlow) | (left <= kPWGs ? kFlagTail : 0);
      mt.img = img;
      mt.img_par = img_par;
      mt.pad0[0] = mt.pad0[1] = mt.pad0[2] = 0;
      mt.theta = theta + el[k];
      mt.grad = grad + el[k];
      mt.state = state + (el[k] - lo);
      mt.rowtab = rowtab;
      mt.coltab = coltab;
      mt.pad = nullptr;
      st.meta[k] = mt;
      bytes += (fast[k] ? 24u * (uint32_t)(v1 - v0) : 0u) + (rb ? 64u : 0u);
    }
    mbar_arrive_tx(full, bytes);
#pragma unroll
    for (int k = 0; k < 2; k++) {
      const uint32_t nv = (uint32_t)(vb[k] - va[k]);
      if (fast[k] && nv > 0) {
        bulk_g2s(&st.th[k][va[k]], theta + el[k] + va[k], 4 * nv, full);
        bulk_g2s(&st.gr[k][va[k]], grad + el[k] + va[k], 4 * nv, full);
        bulk_g2s(&st.st[k][va[k]], state + (el[k] + va[k] - lo), 16 * nv, full);
      }
      if (rb) bulk_g2s(st.rowent[k], rowtab + (int64_t)arow[k] * kRowTab, 64, full);
    }
  }
};

// Features of one element -> the tile's E (hi | lo) operand words, stored to
// TMEM at `ta`, and the B operand words.
template <int KIND>
__device__ __forceinline__ void pair_operands(const FastIn &x, const Entry &re, const Entry &ce,
                                              const PrepImage &im, uint32_t ta,
                                              uint32_t (&bv)[16]) {
  const float sq[3] = {im.sqmr[0], im.sqmr[1], im.sqmr[2]};
  float f[16];
  fast_features(x, re.x, ce.x, sq, f);
  // normalize (features.py:349-354) so every operand fits fp16
  const float4 *es = reinterpret_cast<const float4 *>(im.escale);
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const float4 e4 = es[q];
    const float2 p0 = fmul2(make_float2(f[4 * q], f[4 * q + 1]), make_float2(e4.x, e4.y));
    const float2 p1 = fmul2(make_float2(f[4 * q + 2], f[4 * q + 3]), make_float2(e4.z, e4.w));
    f[4 * q] = p0.x; f[4 * q + 1] = p0.y; f[4 * q + 2] = p1.x; f[4 * q + 3] = p1.y;
  }
  uint32_t ev[16];
#pragma unroll
  for (int q = 0; q < 8; q++) split2(f[2 * q], f[2 * q + 1], ev[q], ev[8 + q]);
  tc::tmem_st16(ta, ev);
  uint32_t xh = 0, xl = 0;
  if (KIND == LOPT_VELO_MLP) split2(clip01(x.g) * im.escale[16], 0.0f, xh, xl);
  bv[0] = re.hi[0]; bv[1] = re.hi[1]; bv[2] = re.hi[2];
  bv[3] = ce.hi[0]; bv[4] = ce.hi[1]; bv[5] = ce.hi[2];
  bv[6] = (xh & 0xFFFFu) | 0x3C000000u;   // clip_hi, fp16 1 (bias)
  bv[7] = 0u;
  bv[8] = re.lo[0]; bv[9] = re.lo[1]; bv[10] = re.lo[2];
  bv[11] = ce.lo[0]; bv[12] = ce.lo[1]; bv[13] = ce.lo[2];
  bv[14] = xl & 0xFFFFu;
  bv[15] = 0u;
}

// pair_operands without the store: E words returned in ev (LOPT_FEAT_ILP)
template <int KIND>
__device__ __forceinline__ void pair_operands_regs(const FastIn &x, const Entry &re, const Entry &ce,
                                                   const PrepImage &im, uint32_t (&ev)[16],
                                                   uint32_t (&bv)[16]) {
  const float sq[3] = {im.sqmr[0], im.sqmr[1], im.sqmr[2]};
  float f[16];
  fast_features(x, re.x, ce.x, sq, f);
  const float4 *es = reinterpret_cast<const float4 *>(im.escale);
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const float4 e4 = es[q];
    const float2 p0 = fmul2(make_float2(f[4 * q], f[4 * q + 1]), make_float2(e4.x, e4.y));
    const float2 p1 = fmul2(make_float2(f[4 * q + 2], f[4 * q + 3]), make_float2(e4.z, e4.w));
    f[4 * q] = p0.x; f[4 * q + 1] = p0.y; f[4 * q + 2] = p1.x; f[4 * q + 3] = p1.y;
  }
#pragma unroll
  for (int q = 0; q < 8; q++) split2(f[2 * q], f[2 * q + 1], ev[q], ev[8 + q]);
  uint32_t xh = 0, xl = 0;
  if (KIND == LOPT_VELO_MLP) split2(clip01(x.g) * im.escale[16], 0.0f, xh, xl);
  bv[0] = re.hi[0]; bv[1] = re.hi[1]; bv[2] = re.hi[2];
  bv[3] = ce.hi[0]; bv[4] = ce.hi[1]; bv[5] = ce.hi[2];
  bv[6] = (xh & 0xFFFFu) | 0x3C000000u;
  bv[7] = 0u;
  bv[8] = re.lo[0]; bv[9] = re.lo[1]; bv[10] = re.lo[2];
  bv[11] = ce.lo[0]; bv[12] = ce.lo[1]; bv[13] = ce.lo[2];
  bv[14] = xl & 0xFFFFu;
  bv[15] = 0u;
}

// The producer warps' loop (one elected lane each): walk the CTA's pairs,
// load each tensor's operand image once its buffer is free, stage the pairs of
// parity p into the ring.
__device__ __forceinline__ void pair_producer_loop(const DevicePlan &P, PairSmem &S, int p,
                                                   int32_t pb, int32_t np) {
  if (tc::elect_one() && np > 0) {
    PairProducer pr;
    pr.seek(P, pb);
    int k = -1, img = 0, cur_j = -1;
    uint32_t par_bits = 0;
    int32_t first[kImgs] = {0, 0, 0, 0};
    Cursor<kPRing> rc;
    for (int32_t i = 0; i < np; i++) {
      if (pr.j != cur_j) {
        cur_j = pr.j;
        k++;
        img = k & (kImgs - 1);
        const int32_t pf = first[img];
        const int32_t nf = first[(k + 1) & (kImgs - 1)];
        first[img] = i;
        if (k >= kImgs) par_bits ^= 1u << img;
        if (i % kPProducers == p) {
          if (k >= kImgs) {
            // tensor k - kImgs used pairs [pf, nf - 1]: every warp of every
            // WG must be past its last pair in that range
            const int32_t last = nf - 1;
            for (int w = 0; w < kPWGs; w++) {
              const int32_t need = last - (((last - w) % kPWGs) + kPWGs) % kPWGs;
              if (need < pf) continue;
              for (int q = 0; q < 4; q++) {
                int32_t d;
                while (true) {
                  asm volatile("ld.acquire.cta.shared.b32 %0, [%1];\n"
                               : "=r"(d)
                               : "r"(tc::smem_u32(&S.done[w][q]))
                               : "memory");
                  if (d >= need) break;
                  __nanosleep(32);
                }
              }
            }
          }
          mbar_arrive_tx(&S.img_full[img], (uint32_t)sizeof(PrepImage));
          bulk_g2s(&S.img[img], reinterpret_cast<const PrepImage *>(P.prep) + pr.j,
                   (uint32_t)sizeof(PrepImage), &S.img_full[img]);
        }
      }
#ifdef LOPT_CTA_CLOCK
      if (p == 0) {
        long long *cp = &g_trace[0][0] + 5 * blockIdx.x;
        if (i == 0) cp[2] = cp[3] = cp[4] = 0;
        if (!pr.rb) cp[3]++;
        if (!pr.aligned) cp[4]++;
      }
#endif
      if (i % kPProducers == p) {
        // parked in hardware while the ring is full (no issue slots spent)
        if (rc.wrapped) tc::mbar_sleep(&S.data_free[rc.i], rc.phase ^ 1u);
        pr.stage(S.stage[rc.i], &S.full[rc.i], img, (int)((par_bits >> img) & 1u));
      }
      pr.advance(P);
      rc.next();
    }
#ifdef LOPT_CTA_CLOCK
    if (p == 0) (&g_trace[0][0] + 5 * blockIdx.x)[2] = k + 1;
#endif
  }
}

template <int KIND, bool W3C>
#ifdef LOPT_APPLY_MAXNREG
#define LOPT_PAIR_BOUNDS __maxnreg__(LOPT_APPLY_MAXNREG)   // leaves registers for a co-resident kernel
#else
#define LOPT_PAIR_BOUNDS __launch_bounds__(kPThreads, 1)
#endif
__global__ void LOPT_PAIR_BOUNDS apply_pair_kernel(DevicePlan P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  PairSmem &S = *reinterpret_cast<PairSmem *>(smem_raw);
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int row = tid & 127;
  if (warp == 0) {
    tc::tmem_alloc(&S.tmem_base, kTmemCols);
    tc::tmem_relinquish();
  }
  if (tid == 0) {
    for (int r = 0; r < kPRing; r++) {
      tc::mbar_init(&S.full[r], 1);
      tc::mbar_init(&S.data_free[r], 128);
    }
    for (int b = 0; b < kImgs; b++) tc::mbar_init(&S.img_full[b], 1);
    for (int w = 0; w < kPWGs; w++) {
      tc::mbar_init(&S.acc[w], 1);
      for (int q = 0; q < 4; q++) S.done[w][q] = -1;
    }
    tc::mbar_fence_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = S.tmem_base;
  const uint32_t lane_addr = (uint32_t)((warp & 3) * 32) << 16;
  if (warp < 4) {
    // the constant slice that selects the layer-2 bias: fp16 {1, 1, 0, ...}
    const uint32_t one[8] = {0x3C003C00u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    tc::tmem_st8(tbase + lane_addr + kPOneCol, one);
    tc::tmem_st_wait();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
#ifdef LOPT_CTA_CLOCK
  // per-CTA profile (balance experiments): start / end globaltimer, tensor
  // switches, flat pairs, slow tiles of the CTA's range
  long long *cta_prof = &g_trace[0][0] + 5 * blockIdx.x;
  if (tid == 0) cta_prof[0] = (long long)globaltimer_ns();
#endif
  const bool aborted = *P.abort_flag != 0;
  // this CTA's pairs: balanced by prep from the SMs' measured speeds
#ifdef LOPT_EVEN_SPLIT
  const int32_t pb = (int32_t)(P.n_pairs * blockIdx.x / gridDim.x);   // A/B reference
  const int32_t pe = (int32_t)(P.n_pairs * (blockIdx.x + 1) / gridDim.x);
#else
  const int32_t pb = P.pair_range[blockIdx.x], pe = P.pair_range[blockIdx.x + 1];
#endif
  if (tid == 0) S.t_start = globaltimer_ns();
  const int32_t np = aborted ? 0 : pe - pb;

  if (warp >= kPWarpProducer) {
    pair_producer_loop(P, S, warp - kPWarpProducer, pb, np);
    __syncwarp();
  } else {
    // ------------------------------------------------------ math warpgroups
    const int wg = warp >> 2;
    const bool issuer = (warp & 3) == 0;
    const uint32_t bar_id = 1 + wg;
    const uint32_t op0 = tbase + 2 * kSlotCols * wg, op1 = op0 + kSlotCols;
    const uint32_t ta0 = op0 + lane_addr, ta1 = op1 + lane_addr;
    const uint32_t one = tbase + kPOneCol;
    const uint64_t dimg1 = tc::smem_desc_kmajor(tc::smem_u32(&S.img[0]), 512, 128);
    const uint64_t dimg2 = tc::smem_desc_kmajor(tc::smem_u32(&S.img[0]), kN2 * 16, 128);
    const bool adv = P.state_advanced != 0;
    const float *beta = P.beta;
    const float alpha_log2e = P.alpha * 1.4426950408889634f;
    const float dsb = P.step->ds * P.beta_out;
    const float decay = P.step->apply_decay != 0 ? P.step->decay : 1.0f;
    const int n_peers = P.n_peers;
    int32_t col_j = -1, col_b0 = -1;
    int32_t a_img = -1, a_par = -1;
    int red_j = -1;
    float red_max = 0.0f, red_out = 0.0f;
    Entry ce, ce1;
    int32_t it = 0;   // this warpgroup's iteration count (peer staging buffer)
    for (int32_t i = wg; i < np; i += kPWGs) {
      const Pos<kPRing> rc(i);
      tc::mbar_wait(&S.full[rc.i], rc.phase);
      const PairStage &st = S.stage[rc.i];
      const TileMeta &m0 = st.meta[0];
      const int32_t flags0 = m0.flags, flags1 = st.meta[1].flags;
      const int j = m0.j;
      if (m0.img != a_img || m0.img_par != a_par) {
        tc::mbar_wait(&S.img_full[m0.img], (uint32_t)m0.img_par);
        a_img = m0.img;
        a_par = m0.img_par;
      }
      if (j != red_j) {
        if (red_j >= 0) {
          if (red_max > 0.0f)
            atomicMax(reinterpret_cast<unsigned int *>(&P.maxabs[red_j]), __float_as_uint(red_max));
          if (!(red_out <= 3.402823466e38f)) atomicOr(&P.status[red_j], LOPT_STATUS_NONFINITE_PARAM);
        }
        red_j = j;
        red_max = 0.0f;
        red_out = 0.0f;
      }
      const PrepImage &im = S.img[m0.img];
      const uint64_t doff = (uint64_t)((uint32_t)m0.img * (uint32_t)(sizeof(PrepImage) >> 4));
      // ---- inputs of both tiles
      bool valid[2];
      float w[2];
      float4 *sp[2];
      FastIn x[2];
      Entry re[2];
      if (flags0 & kFlagRowblock) {
        // both tiles are rows of one column block: one column entry (cached
        // across the pairs of the block; tile 1 reads its own copy)
        if (j != col_j || m0.b0 != col_b0) {
          col_j = j;
          col_b0 = m0.b0;
          load_entry(m0.coltab, m0.b0 + row, ce);
          load_entry(m0.coltab, m0.b0 + row, ce1);
        }
      } else {
        col_j = -1;
      }
#pragma unroll
      for (int k = 0; k < 2; k++) {
        const TileMeta &mt = st.meta[k];
        const int32_t fl = k == 0 ? flags0 : flags1;
        valid[k] = row >= mt.v0 && row < mt.v1;
        float g;
        float4 sq4;
        if (!(fl & kFlagSlow)) {
          w[k] = st.th[k][row];
          g = st.gr[k][row];
          sq4 = st.st[k][row];
        } else {
          w[k] = valid[k] ? mt.theta[row] : 0.0f;
          g = valid[k] ? mt.grad[row] : 0.0f;
          sq4 = valid[k] ? mt.state[row] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (fl & kFlagRowblock) {
          const uint4 v = st.rowent[k][0], hh = st.rowent[k][2], ll = st.rowent[k][3];
          re[k].x[0] = __uint_as_float(v.x); re[k].x[1] = __uint_as_float(v.y); re[k].x[2] = __uint_as_float(v.z);
          re[k].hi[0] = hh.x; re[k].hi[1] = hh.y; re[k].hi[2] = hh.z;
          re[k].lo[0] = ll.x; re[k].lo[1] = ll.y; re[k].lo[2] = ll.z;
        } else {
          const int32_t ec = mt.e0 + (valid[k] ? row : (mt.v1 > mt.v0 ? mt.v0 : 0));
          const int32_t la = (int32_t)((uint32_t)ec / (uint32_t)mt.n);
          load_entry(mt.rowtab, la, re[k]);
          load_entry(mt.coltab, ec - la * mt.n, k == 0 ? ce : ce1);
        }
        x[k].w = w[k];
        sp[k] = mt.state + row;
        advance(g, sq4, adv, beta, x[k]);
#if LOPT_STATE_EARLY
        if (valid[k] && !adv) *sp[k] = make_float4(x[k].m1, x[k].m2, x[k].m3, x[k].v);
#endif
      }
      // ---- features -> E/B operands of both tiles, layer-1 MMAs
#if LOPT_L1_SPLIT
      // tile 0's layer 1 runs while tile 1's features are computed (its own
      // named barrier: no warp waits on an MMA between the two issues)
      {
        uint32_t bv[16];
        pair_operands<KIND>(x[0], re[0], ce, im, ta0, bv);
        tc::tmem_st16(ta0 + 16, bv);
        tc::tmem_st_wait();
      }
      tc::fence_before_sync();
      if (issuer) {
        tc::bar_sync(7 + wg, 128);
        tc::fence_after_sync();
        if (tc::elect_one()) issue_layer1_nc(dimg1 + doff, op0, op0 + 32);
        __syncwarp();
      } else {
        tc::bar_arrive(7 + wg, 128);
      }
      {
        uint32_t bv[16];
        pair_operands<KIND>(x[1], re[1], ce1, im, ta1, bv);
        tc::tmem_st16(ta1 + 16, bv);
        tc::tmem_st_wait();
      }
      tc::fence_before_sync();
      if (issuer) {
        tc::bar_sync(bar_id, 128);
        tc::fence_after_sync();
        if (tc::elect_one()) issue_layer1(dimg1 + doff, op1, op1 + 32, &S.acc[wg]);
        __syncwarp();
      } else {
        tc::bar_arrive(bar_id, 128);
      }
#else
#if LOPT_FEAT_ILP
      {
        // both tiles' features computed before any store (interleavable)
        uint32_t e0[16], b0[16], e1[16], b1[16];
        pair_operands_regs<KIND>(x[0], re[0], ce, im, e0, b0);
        pair_operands_regs<KIND>(x[1], re[1], ce1, im, e1, b1);
        tc::tmem_st16(ta0, e0);
        tc::tmem_st16(ta0 + 16, b0);
        tc::tmem_st16(ta1, e1);
        tc::tmem_st16(ta1 + 16, b1);
        tc::tmem_st_wait();
      }
#else
      {
        uint32_t bv[16];
        pair_operands<KIND>(x[0], re[0], ce, im, ta0, bv);
        tc::tmem_st16(ta0 + 16, bv);
        pair_operands<KIND>(x[1], re[1], ce1, im, ta1, bv);
        tc::tmem_st16(ta1 + 16, bv);
        tc::tmem_st_wait();
      }
#endif
      tc::fence_before_sync();
      if (issuer) {
        tc::bar_sync(bar_id, 128);
        tc::fence_after_sync();
        if (tc::elect_one()) {
          issue_layer1_nc(dimg1 + doff, op0, op0 + 32);
          issue_layer1(dimg1 + doff, op1, op1 + 32, &S.acc[wg]);
        }
        __syncwarp();
      } else {
        tc::bar_arrive(bar_id, 128);
      }
#endif
#if !LOPT_STATE_EARLY
      // the accumulators do not depend on the MLP: stored while layer 1 runs
#pragma unroll
      for (int k = 0; k < 2; k++)
        if (valid[k] && !adv) *sp[k] = make_float4(x[k].m1, x[k].m2, x[k].m3, x[k].v);
#endif
#if LOPT_ACC_SLEEP
      tc::mbar_sleep(&S.acc[wg], 0u);
#else
      tc::mbar_wait(&S.acc[wg], 0u);
#endif
      tc::fence_after_sync();
      // ---- layer-1 epilogue (ReLU + split -> H) of both tiles, layer-2 MMAs
#if LOPT_EPI_PREFETCH
      // all four accumulator loads in flight before the first wait
      uint32_t hh[2][2][16];
#pragma unroll
      for (int half = 0; half < 2; half++) {
        tc::tmem_ld16(ta0 + 32 + 16 * half, hh[half][0]);
        tc::tmem_ld16(ta1 + 32 + 16 * half, hh[half][1]);
      }
      tc::tmem_ld_wait();
#endif
#pragma unroll
      for (int half = 0; half < 2; half++) {
#if LOPT_EPI_PREFETCH
        const uint32_t (&h0)[16] = hh[half][0];
        const uint32_t (&h1)[16] = hh[half][1];
#else
        uint32_t h0[16], h1[16];
        tc::tmem_ld16(ta0 + 32 + 16 * half, h0);
        tc::tmem_ld16(ta1 + 32 + 16 * half, h1);
        tc::tmem_ld_wait();
#endif
        uint32_t o0[16], o1[16];   // {hi(8) | lo(8)} of this 16-unit half
#pragma unroll
        for (int q = 0; q < 8; q++) {
          relu_split2(__uint_as_float(h0[2 * q]), __uint_as_float(h0[2 * q + 1]), o0[q], o0[8 + q]);
          relu_split2(__uint_as_float(h1[2 * q]), __uint_as_float(h1[2 * q + 1]), o1[q], o1[8 + q]);
        }
        tc::tmem_st16(ta0 + 16 * half, o0);
        tc::tmem_st16(ta1 + 16 * half, o1);
      }
      tc::tmem_st_wait();
      tc::fence_before_sync();
      if (issuer) {
        tc::bar_sync(bar_id, 128);
        tc::fence_after_sync();
        if (tc::elect_one()) {
          issue_layer2_nc(dimg2 + doff, op0, op0 + 32, one);
          issue_layer2<true, true>(dimg2 + doff, op1, op1 + 32, one, &S.acc[wg]);
        }
        __syncwarp();
      } else {
        tc::bar_arrive(bar_id, 128);
      }
#if LOPT_ACC_SLEEP
      tc::mbar_sleep(&S.acc[wg], 1u);
#else
      tc::mbar_wait(&S.acc[wg], 1u);
#endif
      tc::fence_after_sync();
#if LOPT_L3_CHAINS8
      // ---- layer 3 in f32: (b3 + linear half, from the MMA) + sum (w3/2)|h2|
      // as {dir, mag} pairs, eight independent chains (two tiles x two
      // 16-unit halves x even / odd units), all TMEM loads before one wait
      float2 de[2], dd[2];
      {
        uint32_t h0[16], h1[16], g0[16], g1[16], l0[2], l1[2];
        tc::tmem_ld16(ta0 + 32, h0);
        tc::tmem_ld16(ta1 + 32, h1);
        tc::tmem_ld16(ta0 + 48, g0);
        tc::tmem_ld16(ta1 + 48, g1);
        tc::tmem_ld2(ta0 + 64, l0);
        tc::tmem_ld2(ta1 + 64, l1);
        tc::tmem_ld_wait();
        float2 e2[2], d2[2];
        de[0] = make_float2(__uint_as_float(l0[0]), __uint_as_float(l0[1]));
        de[1] = make_float2(__uint_as_float(l1[0]), __uint_as_float(l1[1]));
        dd[0] = dd[1] = e2[0] = e2[1] = d2[0] = d2[1] = make_float2(0.0f, 0.0f);
        const float4 *w3 = reinterpret_cast<const float4 *>(im.w3h);
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const float4 wa = w3[q], wb = w3[8 + q];
          const float2 wda = make_float2(wa.x, wa.y), wma = make_float2(wa.z, wa.w);
          const float2 wdb = make_float2(wb.x, wb.y), wmb = make_float2(wb.z, wb.w);
          float he = fabsf(__uint_as_float(h0[2 * q])), ho = fabsf(__uint_as_float(h0[2 * q + 1]));
          de[0] = ffma2(make_float2(he, he), wda, de[0]);
          dd[0] = ffma2(make_float2(ho, ho), wma, dd[0]);
          he = fabsf(__uint_as_float(h1[2 * q]));
          ho = fabsf(__uint_as_float(h1[2 * q + 1]));
          de[1] = ffma2(make_float2(he, he), wda, de[1]);
          dd[1] = ffma2(make_float2(ho, ho), wma, dd[1]);
          he = fabsf(__uint_as_float(g0[2 * q]));
          ho = fabsf(__uint_as_float(g0[2 * q + 1]));
          e2[0] = ffma2(make_float2(he, he), wdb, e2[0]);
          d2[0] = ffma2(make_float2(ho, ho), wmb, d2[0]);
          he = fabsf(__uint_as_float(g1[2 * q]));
          ho = fabsf(__uint_as_float(g1[2 * q + 1]));
          e2[1] = ffma2(make_float2(he, he), wdb, e2[1]);
          d2[1] = ffma2(make_float2(ho, ho), wmb, d2[1]);
        }
#pragma unroll
        for (int k = 0; k < 2; k++) {
          de[k] = tc::add2(de[k], e2[k]);
          dd[k] = tc::add2(dd[k], d2[k]);
        }
      }
#else
      // ---- layer 3 in f32: (b3 + linear half, from the MMA) + sum (w3/2)|h2|
      float2 de[2], dd[2];
      {
        uint32_t h0[16], h1[16], l0[2], l1[2];
        tc::tmem_ld16(ta0 + 32, h0);
        tc::tmem_ld16(ta1 + 32, h1);
        tc::tmem_ld2(ta0 + 64, l0);
        tc::tmem_ld2(ta1 + 64, l1);
        tc::tmem_ld_wait();
        de[0] = make_float2(__uint_as_float(l0[0]), __uint_as_float(l0[1]));
        de[1] = make_float2(__uint_as_float(l1[0]), __uint_as_float(l1[1]));
        dd[0] = dd[1] = make_float2(0.0f, 0.0f);
        if (W3C) {
          // w3 from the launch parameter (uniform registers) lacks the
          // tensor's 2^s2: run the chains 2^-s2 down and scale the sum back
          // up -- powers of two, so every rounding is the image path's
          const float sdn = im.s2_down;
          de[0] = fmul2(de[0], make_float2(sdn, sdn));
          de[1] = fmul2(de[1], make_float2(sdn, sdn));
        }
        const float4 *w3 = W3C ? reinterpret_cast<const float4 *>(&P.w3c[0][0])
                               : reinterpret_cast<const float4 *>(im.w3h);
#pragma unroll
        for (int half = 0; half < 2; half++) {
          if (half == 1) {
            tc::tmem_ld16(ta0 + 48, h0);
            tc::tmem_ld16(ta1 + 48, h1);
            tc::tmem_ld_wait();
          }
#pragma unroll
          for (int q = 0; q < 8; q++) {
            const float4 wq = w3[8 * half + q];
            const float2 wd = make_float2(wq.x, wq.y), wm = make_float2(wq.z, wq.w);
            float he = fabsf(__uint_as_float(h0[2 * q])), ho = fabsf(__uint_as_float(h0[2 * q + 1]));
            de[0] = ffma2(make_float2(he, he), wd, de[0]);
            dd[0] = ffma2(make_float2(ho, ho), wm, dd[0]);
            he = fabsf(__uint_as_float(h1[2 * q]));
            ho = fabsf(__uint_as_float(h1[2 * q + 1]));
            de[1] = ffma2(make_float2(he, he), wd, de[1]);
            dd[1] = ffma2(make_float2(ho, ho), wm, dd[1]);
          }
        }
        if (W3C) {
          const float sup = im.s2_up;
#pragma unroll
          for (int k = 0; k < 2; k++) {
            de[k] = fmul2(de[k], make_float2(sup, sup));
            dd[k] = fmul2(dd[k], make_float2(sup, sup));
          }
        }
      }
#endif
      // ---- update and stores; the tile metadata and theta are re-read from
      // the data slot (not held in registers across the MMA waits)
      float out[2];
      float *tpk[2];
      bool vk[2];
      int32_t kv0[2], kv1[2], kfl[2];
#pragma unroll
      for (int k = 0; k < 2; k++) {
        const TileMeta &mt = st.meta[k];
        kv0[k] = mt.v0;
        kv1[k] = mt.v1;
        kfl[k] = mt.flags;
        vk[k] = row >= kv0[k] && row < kv1[k];
        tpk[k] = mt.theta + row;
        const float wk = !(kfl[k] & kFlagSlow) ? st.th[k][row] : (vk[k] ? *tpk[k] : 0.0f);
        const float dir = de[k].x + dd[k].x, mag = de[k].y + dd[k].y;
        const float du = dsb * (dir * ex2_ftz(mag * alpha_log2e));   // engine.py:537-539
        out[k] = (wk + du) * decay;                                  // optim.py:100-101
        if (vk[k]) {
          red_max = fmaxf(red_max, fabsf(du));
          red_out = max_nan_abs(red_out, out[k]);
          *tpk[k] = out[k];
        }
      }
      if (n_peers > 0) {
        // fused all-gather: the same values into every
        // peer's copy of the arena over NVLink.  Aligned tiles are staged in
        // shared memory and leave as 16-byte stores: thread t owns chunk
        // t % 64 (four elements of one tile) and sends it to peers t / 64,
        // t / 64 + 2, ... -- one shared load and n_peers / 2 vector stores
        // per thread instead of n_peers scalar stores per element.
        // Unaligned tiles store element by element.
        if (P.peer_bulk && !((kfl[0] | kfl[1]) & kFlagSlow)) {
          const int b = it & 1;   // double buffer: reused two pairs later,
                                  // past this pair's MMA barriers
          S.peer_stage[wg][b][0][row] = out[0];
          S.peer_stage[wg][b][1][row] = out[1];
          tc::bar_sync(4 + wg, 128);
          const int c = row & 63, kk = c >> 5, e = (c & 31) * 4;
          const int32_t lo_ = kk ? kv0[1] : kv0[0], hi_ = kk ? kv1[1] : kv1[0];
          if (e >= lo_ && e + 4 <= hi_) {
            const float4 v4 = *reinterpret_cast<const float4 *>(&S.peer_stage[wg][b][kk][e]);
            char *dst = reinterpret_cast<char *>((kk ? tpk[1] : tpk[0]) - row + e);
            for (int q = row >> 6; q < n_peers; q += 2)
              *reinterpret_cast<float4 *>(dst + P.peer_delta[q]) = v4;
          }
        } else {
#pragma unroll
          for (int k = 0; k < 2; k++)
            if (vk[k])
              for (int q = 0; q < n_peers; q++)
                *reinterpret_cast<float *>(reinterpret_cast<char *>(tpk[k]) + P.peer_delta[q]) = out[k];
        }
      }
      // the data slot and (for the producer's image reuse) this pair are done
      mbar_arrive(&S.data_free[rc.i]);
      __syncwarp();   // every lane's image reads precede lane 0's release
      if ((flags0 & kFlagTail) && (threadIdx.x & 31) == 0)
        asm volatile("st.release.cta.shared.b32 [%0], %1;\n" ::"r"(tc::smem_u32(&S.done[wg][warp & 3])),
                     "r"(i)
                     : "memory");
      it++;
    }
    if (red_j >= 0) {
      if (red_max > 0.0f)
        atomicMax(reinterpret_cast<unsigned int *>(&P.maxabs[red_j]), __float_as_uint(red_max));
      if (!(red_out <= 3.402823466e38f)) atomicOr(&P.status[red_j], LOPT_STATUS_NONFINITE_PARAM);
    }
    if (n_peers > 0) __threadfence_system();
  }
  tc::fence_before_sync();
  __syncthreads();
#ifdef LOPT_CTA_CLOCK
  if (tid == 0) cta_prof[1] = (long long)globaltimer_ns();
#endif
  if (tid == 0) {
    // this launch's speed record for the next split (none for an aborted step)
    P.cta_perf[2 * blockIdx.x] = aborted ? 0 : pe - pb;
    P.cta_perf[2 * blockIdx.x + 1] = (int64_t)(globaltimer_ns() - S.t_start);
  }
  if (warp == 0) tc::tmem_dealloc(tbase, kTmemCols);
}

static int g_num_sms = 0;

void launch_tc_apply(const DevicePlan &P0, cudaStream_t s) {
  DevicePlan P = P0;
  if (const char *d = getenv("LOPT_APPLY_DEBUG")) P.dbg = atoi(d);   // timing experiments
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  // one CTA per SM (the 512-column TMEM allocation needs it anyway)
  const int grid = (int)std::min<int64_t>(g_num_sms, P.n_tiles);
  // development A/B switch (read per launch so one process can compare)
  const char *ve = getenv("LOPT_APPLY_VARIANT");
  const int variant = ve ? atoi(ve) : 3;
  if (variant == 3) {
    const size_t smem = sizeof(PairSmem) + 1024;
    const int pgrid = P.apply_grid;   // the grid prep balanced the ranges for
    if (P.kind == LOPT_SMALL_FC_LOPT) {
      if (P.w3c_on) {
        cudaFuncSetAttribute(apply_pair_kernel<LOPT_SMALL_FC_LOPT, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        apply_pair_kernel<LOPT_SMALL_FC_LOPT, true><<<pgrid, kPThreads, smem, s>>>(P);
      } else {
        cudaFuncSetAttribute(apply_pair_kernel<LOPT_SMALL_FC_LOPT, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        apply_pair_kernel<LOPT_SMALL_FC_LOPT, false><<<pgrid, kPThreads, smem, s>>>(P);
      }
    } else {
      if (P.w3c_on) {
        cudaFuncSetAttribute(apply_pair_kernel<LOPT_VELO_MLP, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        apply_pair_kernel<LOPT_VELO_MLP, true><<<pgrid, kPThreads, smem, s>>>(P);
      } else {
        cudaFuncSetAttribute(apply_pair_kernel<LOPT_VELO_MLP, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        apply_pair_kernel<LOPT_VELO_MLP, false><<<pgrid, kPThreads, smem, s>>>(P);
      }
    }
    return;
  }
  const size_t smem = sizeof(ApplySmem) + 1024;
  if (P.kind == LOPT_SMALL_FC_LOPT) {
    cudaFuncSetAttribute(apply_tc_kernel<LOPT_SMALL_FC_LOPT>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    apply_tc_kernel<LOPT_SMALL_FC_LOPT><<<grid, kApplyThreads, smem, s>>>(P);
  } else {
    cudaFuncSetAttribute(apply_tc_kernel<LOPT_VELO_MLP>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    apply_tc_kernel<LOPT_VELO_MLP><<<grid, kApplyThreads, smem, s>>>(P);
  }
}

}  // namespace lopt

extern "C" int lopt_debug_apply_trace(long long *host, int32_t n) {
  if (!host || n < 0 || n > lopt::kTraceTiles * lopt::kTraceEvents) return LOPT_ERR_INVALID;
  return cudaMemcpyFromSymbol(host, lopt::g_trace, sizeof(long long) * n) == cudaSuccess
             ? LOPT_OK
             : LOPT_ERR_CUDA;
}
