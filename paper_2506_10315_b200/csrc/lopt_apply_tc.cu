// lopt_apply_tc.cu -- phase 2 of the fast path on the tensor cores.
//
// engine.py:657-710 fused_apply + state.py:77-90 + optim.py:171-172 for
// 128-element tiles: features -> layer 1 (tcgen05, M=128 elements) -> ReLU ->
// layer 2 (tcgen05) -> ReLU -> layer 3 (CUDA cores, f32) -> exp -> update ->
// decay -> store theta and the advanced accumulators.
//
// fp32 accuracy on the f16 tensor-core path: every operand is split in two
// fp16 terms (x = x_hi + x_lo, relative error 2^-22) and each product is formed
// as x_hi*W_hi + x_lo*W_hi + x_hi*W_lo with f32 accumulation.  Layer-1 inputs
// are the normalized features (bounded by sqrt(m*n), so they fit fp16); layer-2
// inputs are scaled by a per-tensor power of two chosen from a bound on |h1|.
// The A operands go from registers straight into tensor memory (tcgen05.st)
// and the MMAs read them there; only the per-tensor B operands live in smem.
//
// What bounds this kernel (measured with tools/probe_umma.py): an issuing
// thread can launch one tcgen05.mma only every ~100 cycles, flat in N up to
// 128, while the tensor pipe itself needs M*N/256 cycles.  So: few, wide MMAs
// (layer 1 is N-packed: 4 MMAs of N=64; layer 2: 6 MMAs of N=32), and one
// issuing warp per math warpgroup.
//
// Structure: persistent kernel, one CTA per SM = three 128-thread math
// warpgroups + three MMA-issue warps (one each).  Thread i of a warpgroup owns
// row i of every tile (TMEM lane i).  Each warpgroup software-pipelines its
// contiguous tile range three deep -- iteration k runs stage B of tile k-1
// (layer-1 epilogue), stage A of tile k (features; its HBM loads were issued
// one iteration earlier) and stage C of tile k-1 (layer-2 epilogue, update,
// stores) -- and hands operands to its issue warp through mbarriers (128
// arrivals), so math threads only ever wait for MMA results they consume.
#include "lopt_fast.cuh"

namespace lopt {

constexpr int kWGs = 3;
constexpr int kMathThreads = 128 * kWGs;
constexpr int kApplyThreads = kMathThreads + 32 * kWGs;
constexpr int kIssueWarp0 = kMathThreads / 32;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColsPerWG = 160;      // A1 32 | ACC1 64 | A2 32 | ACC2 32
constexpr uint32_t kA1 = 0, kACC1 = 32, kA2 = 96, kACC2 = 128;

struct __align__(128) ApplySmem {
  PrepImage img[kWGs][2];   // double-buffered per warpgroup (tensor switches)
  uint64_t a1_ready[kWGs], a2_ready[kWGs];     // 128 arrivals: operands in TMEM
  uint64_t acc1_full[kWGs], acc2_full[kWGs];   // tcgen05.commit: results in TMEM
  uint32_t a1_buf[kWGs], a2_buf[kWGs];         // PrepImage buffer of the pending MMA
  uint32_t tmem_base;
};

struct TileLoad {
  int j;
  bool valid;
  int32_t a, b;      // (row, column) of the element (clamped into the tensor)
  float *tp;         // &theta[e]
  float4 *sp;        // &state[e - lo]
  float w, g;
  float4 s;
};

// Walks a warpgroup's contiguous tile range: current tensor, tile origin
// (row a0, column b0) advanced incrementally from tile to tile.
// (32-bit indices: fast-mode plans require < 2^31 elements per tensor and tiles)
struct TileWalker {
  int j = -1;
  int32_t next_tile0 = -1, tile0 = 0, lo = 0, hi = 0, n = 1, t = -2, a0 = 0, b0 = 0;
  const float *theta = nullptr, *grad = nullptr;
  const float4 *state = nullptr;
};

__device__ __forceinline__ void walk_to(const DevicePlan &P, TileWalker &W, int32_t t) {
  if (t >= W.next_tile0) {
    int j = W.j < 0 ? 0 : W.j;
    while (j + 1 < P.count && P.tensors[j + 1].tile0 <= t) j++;
    const TensorDesc *T = P.tensors + j;
    W.j = j;
    W.tile0 = (int32_t)T->tile0;
    W.lo = (int32_t)T->lo;
    W.hi = (int32_t)T->hi;
    W.n = (int32_t)T->n;
    W.theta = T->theta;
    W.grad = T->grad;
    W.state = T->state;
    W.next_tile0 = j + 1 < P.count ? (int32_t)P.tensors[j + 1].tile0 : INT32_MAX;
    W.t = -2;
  }
  if (t == W.t + 1 && W.n >= kTile) {
    W.b0 += kTile;
    if (W.b0 >= W.n) {
      W.b0 -= W.n;
      W.a0++;
    }
  } else {
    const int32_t e0 = W.lo + (t - W.tile0) * kTile;
    W.a0 = (int32_t)((uint32_t)e0 / (uint32_t)W.n);
    W.b0 = e0 - W.a0 * W.n;
  }
  W.t = t;
}

__device__ __forceinline__ void load_tile(const DevicePlan &P, TileWalker &W, int32_t t, int row,
                                          TileLoad &L) {
  walk_to(P, W, t);
  L.j = W.j;
  const int32_t e0 = W.lo + (t - W.tile0) * kTile;
  L.valid = e0 + row < W.hi;
  // rows past the end of the tensor compute on a valid element and are masked
  // at the store; their A rows never influence other rows
  const int r = L.valid ? row : 0;
  int32_t b = W.b0 + r, a = W.a0;
  if (b >= W.n) {
    if (W.n >= kTile) {
      b -= W.n;
      a++;
    } else {
      const uint32_t q = (uint32_t)b / (uint32_t)W.n;
      a += (int32_t)q;
      b -= (int32_t)q * W.n;
    }
  }
  L.a = a;
  L.b = b;
  L.tp = const_cast<float *>(W.theta) + e0 + r;
  L.sp = const_cast<float4 *>(W.state) + (e0 + r - W.lo);
  L.w = __ldg(L.tp);
  L.g = __ldg(W.grad + e0 + r);
  L.s = __ldg(L.sp);
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tc::smem_u32(bar)) : "memory");
}

__device__ __forceinline__ uint64_t f2_bits(float2 v) { return *reinterpret_cast<uint64_t *>(&v); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;\n" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)), "l"(f2_bits(c)));
  return *reinterpret_cast<float2 *>(&d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;\n" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return *reinterpret_cast<float2 *>(&d);
}

// ReLU fused into a two-term fp16 split: hi truncates toward zero (so the
// residual of a positive value is non-negative), both conversions clamp at 0.
__device__ __forceinline__ void relu_split_f16(float a, float b, uint32_t &hi, uint32_t &lo) {
  asm("cvt.rz.relu.f16x2.f32 %0, %2, %1;\n" : "=r"(hi) : "f"(a), "f"(b));
  const float2 h = tc::unpack_f16x2(hi);
  asm("cvt.rn.relu.f16x2.f32 %0, %2, %1;\n" : "=r"(lo) : "f"(a - h.x), "f"(b - h.y));
}

// One issue warp per math warpgroup: lane 0 walks the warpgroup's event stream
// A1(tb), A2(tb), A1(tb+1), ..., A2(te-1).
__device__ void issue_loop(const DevicePlan &P, ApplySmem &S, uint32_t tbase, int g) {
  const uint32_t idesc64 = tc::idesc_f16_f32(128, 64), idesc32 = tc::idesc_f16_f32(128, 32);
  const int64_t nwg = (int64_t)gridDim.x * kWGs;
  const int64_t gwg = (int64_t)blockIdx.x * kWGs + g;
  const int32_t tb = (int32_t)(P.n_tiles * gwg / nwg), te = (int32_t)(P.n_tiles * (gwg + 1) / nwg);
  const uint32_t base = tbase + kColsPerWG * g;
  for (int32_t k = tb; k < te; k++) {
    const uint32_t par = (uint32_t)((k - tb) & 1);
    // layer 1: four N-packed MMAs
    tc::mbar_wait(&S.a1_ready[g], par);
    tc::fence_after_sync();
    {
      const PrepImage &im = S.img[g][S.a1_buf[g]];
#pragma unroll
      for (int s = 0; s < 4; s++)
        tc::mma_ts(base + kACC1, base + kA1 + 8 * s,
                   tc::smem_desc_kmajor(tc::smem_u32(im.b1[s]), 1024, 128), idesc64, s > 0);
      tc::mma_commit(&S.acc1_full[g]);
    }
    // layer 2: six MMAs (h_hi * W2_hi, h_hi * W2_lo, h_lo * W2_hi)
    tc::mbar_wait(&S.a2_ready[g], par);
    tc::fence_after_sync();
    {
      const PrepImage &im = S.img[g][S.a2_buf[g]];
      uint64_t bd[4];
#pragma unroll
      for (int q = 0; q < 4; q++) bd[q] = tc::smem_desc_kmajor(tc::smem_u32(im.b2[q]), 512, 128);
      const uint32_t d = base + kACC2, a = base + kA2;
      tc::mma_ts(d, a + 0, bd[0], idesc32, 0);
      tc::mma_ts(d, a + 8, bd[1], idesc32, 1);
      tc::mma_ts(d, a + 0, bd[2], idesc32, 1);
      tc::mma_ts(d, a + 8, bd[3], idesc32, 1);
      tc::mma_ts(d, a + 16, bd[0], idesc32, 1);
      tc::mma_ts(d, a + 24, bd[1], idesc32, 1);
      tc::mma_commit(&S.acc2_full[g]);
    }
  }
}

// Per-warpgroup pipeline state carried between the stages.
struct Carry {
  int buf = 0, j = -1;
  bool valid = false;
  float w = 0.0f;
  float *theta = nullptr;
};

struct Reduce {
  int j = -1;
  float maxabs = 0.0f;
  uint32_t bad = 0;
  __device__ __forceinline__ void flush(const DevicePlan &P) {
    if (j >= 0) {
      if (maxabs > 0.0f)
        atomicMax(reinterpret_cast<unsigned int *>(&P.maxabs[j]), __float_as_uint(maxabs));
      if (bad) atomicOr(&P.status[j], LOPT_STATUS_NONFINITE_PARAM);
    }
  }
};

template <int KIND>
__global__ void __launch_bounds__(kApplyThreads, 1) apply_tc_kernel(DevicePlan P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  ApplySmem &S = *reinterpret_cast<ApplySmem *>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == kIssueWarp0) {
    tc::tmem_alloc(&S.tmem_base, kTmemCols);
    tc::tmem_relinquish();
    if ((tid & 31) == 0) {
      for (int g = 0; g < kWGs; g++) {
        tc::mbar_init(&S.a1_ready[g], 128);
        tc::mbar_init(&S.a2_ready[g], 128);
        tc::mbar_init(&S.acc1_full[g], 1);
        tc::mbar_init(&S.acc2_full[g], 1);
      }
      tc::mbar_fence_init();
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = S.tmem_base;
  const bool aborted = *P.abort_flag != 0;

  if (warp >= kIssueWarp0) {
    if ((tid & 31) == 0 && !aborted) issue_loop(P, S, tbase, warp - kIssueWarp0);
    __syncwarp();
  } else if (!aborted) {
    const int wg = warp >> 2, row = tid & 127;
    const uint32_t lane_addr = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t cbase = tbase + lane_addr + kColsPerWG * wg;
    const bool adv = P.state_advanced != 0;
    const float alpha_log2e = P.alpha * 1.4426950408889634f;
    const float beta_out = P.beta_out;
    const float ds = P.step->ds, decay = P.step->decay;
    const bool apply_decay = P.step->apply_decay != 0;
    const int bar_id = 1 + wg;
    const int64_t nwg = (int64_t)gridDim.x * kWGs;
    const int64_t gwg = (int64_t)blockIdx.x * kWGs + wg;
    const int32_t tb = (int32_t)(P.n_tiles * gwg / nwg), te = (int32_t)(P.n_tiles * (gwg + 1) / nwg);

    TileWalker W;
    TileLoad cur, nxt;
    if (tb < te) load_tile(P, W, tb, row, cur);
    int bufA = 1, bufA_j = -1;
    const float *rowtabA = nullptr, *coltabA = nullptr;
    Carry prev;
    Reduce red;

    for (int32_t k = tb; k <= te; k++) {
      const bool hasA = k < te, hasBC = k > tb;
      const uint32_t par = (uint32_t)((k - 1 - tb) & 1);
      if (k + 1 < te) load_tile(P, W, k + 1, row, nxt);
      // ---- stage A prologue: tensor switch, table loads ------------------
      uint4 rt0 = make_uint4(0, 0, 0, 0), rth = rt0, rtl = rt0, ct0 = rt0, cth = rt0, ctl = rt0;
      if (hasA) {
        if (cur.j != bufA_j) {
          // every thread must be past its last read of the buffer being
          // replaced, then the copy must be complete before anyone reads it
          bufA ^= 1;
          bufA_j = cur.j;
          const TensorDesc *T = P.tensors + cur.j;
          rowtabA = T->rowtab;
          coltabA = T->coltab;
          tc::bar_sync(bar_id, 128);
          const uint4 *src =
              reinterpret_cast<const uint4 *>(reinterpret_cast<const PrepImage *>(P.prep) + cur.j);
          uint4 *dst = reinterpret_cast<uint4 *>(&S.img[wg][bufA]);
          for (int i = row; i < (int)(sizeof(PrepImage) / 16); i += 128) dst[i] = __ldg(src + i);
          tc::fence_proxy_async_smem();
          tc::bar_sync(bar_id, 128);
        }
        const uint4 *rt = reinterpret_cast<const uint4 *>(rowtabA + cur.a * kRowTab);
        const uint4 *ct = reinterpret_cast<const uint4 *>(coltabA + cur.b * kRowTab);
        rt0 = __ldg(rt); rth = __ldg(rt + 2); rtl = __ldg(rt + 3);
        ct0 = __ldg(ct); cth = __ldg(ct + 2); ctl = __ldg(ct + 3);
      }
      // ---- stage B (tile k-1): layer-1 epilogue -> A2 --------------------
      if (hasBC) {
        tc::mbar_wait(&S.acc1_full[wg], par);
        tc::fence_after_sync();
        const float sdown = S.img[wg][prev.buf].s2_down;
#pragma unroll
        for (int half = 0; half < 2; half++) {
          uint32_t lo[16], hi[16];
          tc::tmem_ld16(cbase + kACC1 + 16 * half, lo);        // x_hi*W_hi + x_lo*W_hi
          tc::tmem_ld16(cbase + kACC1 + 32 + 16 * half, hi);   // x_hi*W_lo
          tc::tmem_ld_wait();
          uint32_t ah[8], al[8];
#pragma unroll
          for (int q = 0; q < 8; q++) {
            float2 h = fadd2(make_float2(__uint_as_float(lo[2 * q]), __uint_as_float(lo[2 * q + 1])),
                             make_float2(__uint_as_float(hi[2 * q]), __uint_as_float(hi[2 * q + 1])));
            if (sdown != 1.0f) {
              h.x *= sdown;
              h.y *= sdown;
            }
            relu_split_f16(h.x, h.y, ah[q], al[q]);
          }
          tc::tmem_st8(cbase + kA2 + 8 * half, ah);
          tc::tmem_st8(cbase + kA2 + 16 + 8 * half, al);
        }
        tc::tmem_st_wait();
        tc::fence_before_sync();
        if (row == 0) S.a2_buf[wg] = (uint32_t)prev.buf;
        mbar_arrive(&S.a2_ready[wg]);
      }
      // ---- stage A (tile k): features -> A1, advanced state --------------
      if (hasA) {
        const PrepImage &im = S.img[wg][bufA];
        FastIn x;
        x.w = cur.w;
        advance(cur.g, cur.s, adv, P.beta, x);
        // the accumulators do not depend on the MLP: store them right away
        if (cur.valid && !adv) *cur.sp = make_float4(x.m1, x.m2, x.m3, x.v);
        const float rc[3] = {__uint_as_float(rt0.x), __uint_as_float(rt0.y), __uint_as_float(rt0.z)};
        const float cc[3] = {__uint_as_float(ct0.x), __uint_as_float(ct0.y), __uint_as_float(ct0.z)};
        const float sq[3] = {im.sqmr[0], im.sqmr[1], im.sqmr[2]};
        float f[16];
        fast_features(x, rc, cc, sq, f);
        // normalize (features.py:349-354) so every operand fits fp16
#pragma unroll
        for (int q = 0; q < 16; q++) f[q] *= im.escale[q];
        uint32_t a[16];
        // slice s: [hi pairs of features 8s..8s+7 | lo pairs]
#pragma unroll
        for (int s = 0; s < 2; s++)
#pragma unroll
          for (int q = 0; q < 4; q++)
            tc::split_pair_f16(f[8 * s + 2 * q], f[8 * s + 2 * q + 1], a[8 * s + q], a[8 * s + 4 + q]);
        tc::tmem_st16(cbase + kA1, a);
        uint32_t xh = 0, xl = 0;
        if (KIND == LOPT_VELO_MLP) tc::split_pair_f16(clip01(x.g) * im.escale[16], 0.0f, xh, xl);
        uint32_t b[16];
        b[0] = rth.x; b[1] = rth.y; b[2] = rth.z; b[3] = cth.x;          // r5 r6 r7 rr5 rr6 rr7 c5 c6
        b[4] = rtl.x; b[5] = rtl.y; b[6] = rtl.z; b[7] = ctl.x;
        b[8] = cth.y; b[9] = cth.z;                                      // c7 rc5 rc6 rc7
        b[10] = (xh & 0xFFFFu) | 0x3C000000u;                            // clip_hi, fp16 1 (bias)
        b[11] = 0u;
        b[12] = ctl.y; b[13] = ctl.z; b[14] = xl & 0xFFFFu; b[15] = 0u;
        tc::tmem_st16(cbase + kA1 + 16, b);
        tc::tmem_st_wait();
        tc::fence_before_sync();
        if (row == 0) S.a1_buf[wg] = (uint32_t)bufA;
        mbar_arrive(&S.a1_ready[wg]);
      }
      // ---- stage C (tile k-1): layer-2 epilogue, layer 3, update ---------
      if (hasBC) {
        tc::mbar_wait(&S.acc2_full[wg], par);
        tc::fence_after_sync();
        if (prev.j != red.j) {
          red.flush(P);
          red.j = prev.j;
          red.maxabs = 0.0f;
          red.bad = 0;
        }
        const PrepImage &im = S.img[wg][prev.buf];
        const float sup = im.s2_up;
        float2 d2 = make_float2(im.b3[0], 0.0f), m2 = make_float2(im.b3[1], 0.0f);
        const float4 *w30 = reinterpret_cast<const float4 *>(im.w3[0]);
        const float4 *w31 = reinterpret_cast<const float4 *>(im.w3[1]);
        const float4 *bb2 = reinterpret_cast<const float4 *>(im.b2f);
#pragma unroll
        for (int half = 0; half < 2; half++) {
          uint32_t h2[16];
          tc::tmem_ld16(cbase + kACC2 + 16 * half, h2);
          tc::tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const float4 wa = w30[4 * half + q], wb = w31[4 * half + q], bq = bb2[4 * half + q];
            const float2 h01 = make_float2(fmaxf(fmaf(__uint_as_float(h2[4 * q]), sup, bq.x), 0.0f),
                                           fmaxf(fmaf(__uint_as_float(h2[4 * q + 1]), sup, bq.y), 0.0f));
            const float2 h23 = make_float2(fmaxf(fmaf(__uint_as_float(h2[4 * q + 2]), sup, bq.z), 0.0f),
                                           fmaxf(fmaf(__uint_as_float(h2[4 * q + 3]), sup, bq.w), 0.0f));
            d2 = ffma2(h01, make_float2(wa.x, wa.y), d2);
            d2 = ffma2(h23, make_float2(wa.z, wa.w), d2);
            m2 = ffma2(h01, make_float2(wb.x, wb.y), m2);
            m2 = ffma2(h23, make_float2(wb.z, wb.w), m2);
          }
        }
        const float dir = d2.x + d2.y, mag = m2.x + m2.y;
        // engine.py:537-539, exp on the SFU (fp32 tolerance path)
        const float ex = exp2f(mag * alpha_log2e);
        const float du = ds * ((dir * ex) * beta_out);
        float out = prev.w + du;
        if (prev.valid) {
          red.maxabs = fmaxf(red.maxabs, fabsf(du));
          red.bad |= !isfinite(out);
          if (apply_decay) out *= decay;   // optim.py:100-101
          *prev.theta = out;
        }
      }
      // ---- shift the pipeline ---------------------------------------------
      if (hasA) {
        prev.buf = bufA;
        prev.j = cur.j;
        prev.valid = cur.valid;
        prev.w = cur.w;
        prev.theta = cur.tp;
        cur = nxt;
      }
    }
    red.flush(P);
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == kIssueWarp0) tc::tmem_dealloc(tbase, kTmemCols);
}

static int g_num_sms = 0;

void launch_tc_apply(const DevicePlan &P, cudaStream_t s) {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  // more than half of the SM's shared memory: one CTA per SM, which the
  // 512-column TMEM allocation needs anyway
  const size_t smem = std::max<size_t>(sizeof(ApplySmem) + 1024, 120 * 1024);
  const int grid = (int)std::min<int64_t>(g_num_sms, (P.n_tiles + kWGs - 1) / kWGs);
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
