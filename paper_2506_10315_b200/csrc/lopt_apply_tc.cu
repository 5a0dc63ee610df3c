// lopt_apply_tc.cu -- phase 2 of the fast path on the tensor cores.
//
// engine.py:657-710 fused_apply + state.py:77-90 + optim.py:171-172 for
// 128-element tiles: features -> layer 1 (tcgen05, M=128 x N=32) -> ReLU ->
// layer 2 (tcgen05) -> ReLU -> layer 3 (CUDA cores, f32) -> exp -> update ->
// decay -> store theta and the advanced accumulators.
//
// fp32 accuracy on the f16 tensor-core path: every operand is split in two
// fp16 terms (x = x_hi + x_lo, relative error 2^-22) and each product is formed
// as x_hi*W_hi + x_hi*W_lo + x_lo*W_hi with f32 accumulation.  Layer-1 inputs
// are the normalized features (bounded by sqrt(m*n), so they fit fp16); layer-2
// inputs are scaled by a per-tensor power of two chosen from a bound on |h1|.
// The A operands go from registers straight into tensor memory (tcgen05.st)
// and the MMAs read them there; only the per-tensor B operands live in smem.
//
// Structure: persistent kernel, one CTA per SM = three 128-thread math
// warpgroups + one MMA-issue warp.  Thread i of a warpgroup owns row i of each
// tile (TMEM lane i).  Each warpgroup software-pipelines its contiguous tile
// range three deep -- iteration k runs stage B of tile k-1 (layer-1 epilogue),
// stage A of tile k (loads prefetched one iteration earlier, features) and
// stage C of tile k-1 (layer-2 epilogue, update, stores) -- and hands operands
// to the issue warp through mbarriers (128 arrivals each), so no math thread
// ever waits for another; they only wait for the MMA results they consume.
#include "lopt_fast.cuh"

namespace lopt {

constexpr int kWGs = 3;
constexpr int kMathThreads = 128 * kWGs;
constexpr int kApplyThreads = kMathThreads + 32;
constexpr int kIssueWarp = kMathThreads / 32;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColsPerWG = 128;      // A1 | ACC1 | A2 | ACC2, 32 columns each
constexpr uint32_t kOnesCol = kColsPerWG * kWGs;

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
  if (W.j < 0 || t >= W.next_tile0) {
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
  const int32_t e0 = W.lo + (t - W.tile0) * kTile;
  if (t == W.t + 1 && W.n >= kTile) {
    W.b0 += kTile;
    if (W.b0 >= W.n) {
      W.b0 -= W.n;
      W.a0++;
    }
  } else {
    W.a0 = (int32_t)((uint32_t)e0 / (uint32_t)W.n);
    W.b0 = e0 - W.a0 * W.n;
  }
  W.t = t;
}

__device__ __forceinline__ void load_tile(const DevicePlan &P, TileWalker &W, int32_t t, int row,
                                          TileLoad &L) {
  walk_to(P, W, t);
  L.j = W.j;
  const int32_t e = W.lo + (t - W.tile0) * kTile + row;
  L.valid = e < W.hi;
  // rows past the end of the tensor compute on a valid element and are masked
  // at the store; their A rows never influence other rows
  const int r = L.valid ? row : 0;
  const int32_t ec = L.valid ? e : W.lo + (t - W.tile0) * kTile;
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
  L.tp = const_cast<float *>(W.theta) + ec;
  L.sp = const_cast<float4 *>(W.state) + (ec - W.lo);
  L.w = __ldg(L.tp);
  L.g = __ldg(W.grad + ec);
  L.s = __ldg(L.sp);
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tc::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(tc::smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ uint64_t f2_bits(float2 v) { return *reinterpret_cast<uint64_t *>(&v); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;\n" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)), "l"(f2_bits(c)));
  return *reinterpret_cast<float2 *>(&d);
}

// ReLU fused into a two-term fp16 split: hi truncates toward zero (so the
// residual of a positive value is non-negative), both conversions clamp at 0.
__device__ __forceinline__ void relu_split_f16(float a, float b, uint32_t &hi, uint32_t &lo) {
  asm("cvt.rz.relu.f16x2.f32 %0, %2, %1;\n" : "=r"(hi) : "f"(a), "f"(b));
  const float2 h = tc::unpack_f16x2(hi);
  asm("cvt.rn.relu.f16x2.f32 %0, %2, %1;\n" : "=r"(lo) : "f"(a - h.x), "f"(b - h.y));
}

// The MMA-issue warp: one elected lane walks every warpgroup's event stream
// (A1(tb), A2(tb), A1(tb+1), ..., A2(te-1)) and issues the corresponding
// layer-1 / layer-2 MMAs when the warpgroup's 128 arrivals are in.
__device__ void issue_loop(const DevicePlan &P, ApplySmem &S, uint32_t tbase) {
  constexpr uint32_t kIdesc = tc::idesc_f16_f32(128, 32);
  int64_t left[kWGs];
  uint32_t cnt[kWGs];
  int active = 0;
  const int64_t nwg = (int64_t)gridDim.x * kWGs;
  for (int g = 0; g < kWGs; g++) {
    const int64_t gwg = (int64_t)blockIdx.x * kWGs + g;
    const int64_t tb = P.n_tiles * gwg / nwg, te = P.n_tiles * (gwg + 1) / nwg;
    left[g] = 2 * (te - tb);
    cnt[g] = 0;
    active += left[g] > 0;
  }
  while (active > 0) {
    bool progressed = false;
    for (int g = 0; g < kWGs; g++) {
      if (left[g] == 0) continue;
      const bool is_a1 = (cnt[g] & 1u) == 0;
      const uint32_t parity = (cnt[g] >> 1) & 1u;
      uint64_t *bar = is_a1 ? &S.a1_ready[g] : &S.a2_ready[g];
      if (!mbar_test(bar, parity)) continue;
      tc::fence_after_sync();
      const uint32_t base = tbase + kColsPerWG * g;
      if (is_a1) {
        const PrepImage &im = S.img[g][S.a1_buf[g]];
        const uint32_t d = base + 32, a = base;
        const uint64_t b0 = tc::smem_desc_kmajor(tc::smem_u32(im.b1[0]), 512, 128);
        const uint64_t b1 = tc::smem_desc_kmajor(tc::smem_u32(im.b1[1]), 512, 128);
        const uint64_t b2 = tc::smem_desc_kmajor(tc::smem_u32(im.b1[2]), 512, 128);
        const uint64_t b3 = tc::smem_desc_kmajor(tc::smem_u32(im.b1[3]), 512, 128);
        tc::mma_ts(d, a + 0, b0, kIdesc, 0);    // f_hi  * We_hi
        tc::mma_ts(d, a + 0, b1, kIdesc, 1);    // f_hi  * We_lo
        tc::mma_ts(d, a + 8, b0, kIdesc, 1);    // f_lo  * We_hi
        tc::mma_ts(d, a + 16, b2, kIdesc, 1);   // bc_hi * Wbc_hi (+ bias_hi)
        tc::mma_ts(d, a + 16, b3, kIdesc, 1);   // bc_hi * Wbc_lo (+ bias_lo)
        tc::mma_ts(d, a + 24, b2, kIdesc, 1);   // bc_lo * Wbc_hi
        tc::mma_commit(&S.acc1_full[g]);
      } else {
        const PrepImage &im = S.img[g][S.a2_buf[g]];
        const uint32_t d = base + 96, a = base + 64;
        uint64_t bd[5];
#pragma unroll
        for (int q = 0; q < 5; q++) bd[q] = tc::smem_desc_kmajor(tc::smem_u32(im.b2[q]), 512, 128);
        tc::mma_ts(d, a + 0, bd[0], kIdesc, 0);    // h_hi * W2_hi
        tc::mma_ts(d, a + 8, bd[1], kIdesc, 1);
        tc::mma_ts(d, a + 0, bd[2], kIdesc, 1);    // h_hi * W2_lo
        tc::mma_ts(d, a + 8, bd[3], kIdesc, 1);
        tc::mma_ts(d, a + 16, bd[0], kIdesc, 1);   // h_lo * W2_hi
        tc::mma_ts(d, a + 24, bd[1], kIdesc, 1);
        tc::mma_ts(d, tbase + kOnesCol, bd[4], kIdesc, 1);  // + b2 (hi + lo)
        tc::mma_commit(&S.acc2_full[g]);
      }
      cnt[g]++;
      if (--left[g] == 0) active--;
      progressed = true;
    }
    if (!progressed) __nanosleep(20);
  }
}

template <int KIND>
__global__ void __launch_bounds__(kApplyThreads, 1) apply_tc_kernel(DevicePlan P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  ApplySmem &S = *reinterpret_cast<ApplySmem *>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, wg = warp >> 2, row = tid & 127;
  if (warp == kIssueWarp) {
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
  if (warp < 4 && !aborted) {
    // constant A slice for the layer-2 bias MMA: K0 = K1 = fp16 1
    uint32_t r[16];
#pragma unroll
    for (int q = 0; q < 16; q++) r[q] = q == 0 ? 0x3C003C00u : 0u;
    tc::tmem_st16(tbase + ((uint32_t)(warp * 32) << 16) + kOnesCol, r);
    tc::tmem_st_wait();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();

  if (warp == kIssueWarp) {
    if ((tid & 31) == 0 && !aborted) issue_loop(P, S, tbase);
    __syncwarp();
  } else if (!aborted) {
    const uint32_t lane_addr = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t cA1 = kColsPerWG * wg, cACC1 = cA1 + 32, cA2 = cA1 + 64, cACC2 = cA1 + 96;
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
    // carry from stage A(k-1) to stages B/C(k-1)
    int prev_buf = 0, prev_j = -1;
    bool prev_valid = false;
    float prev_w = 0.0f;
    float *prev_theta = nullptr;
    // per-tensor reductions of stage C
    int red_j = -1;
    float maxabs = 0.0f;
    uint32_t bad = 0;

    for (int32_t k = tb; k <= te; k++) {
      const bool hasA = k < te, hasBC = k > tb;
      const uint32_t par = (uint32_t)((k - 1 - tb) & 1);
      if (k + 1 < te) load_tile(P, W, k + 1, row, nxt);
      // ---- stage A prologue: tensor switch, table loads ------------------
      uint4 rt0, rth, rtl, ct0, cth, ctl;
      if (hasA) {
        if (cur.j != bufA_j) {
          // every thread must be past its last read of the buffer being
          // replaced (stage C two tiles back), then the copy must be complete
          // before anyone reads it
          bufA ^= 1;
          bufA_j = cur.j;
          const TensorDesc *T = P.tensors + cur.j;
          rowtabA = T->rowtab;
          coltabA = T->coltab;
          tc::bar_sync(bar_id, 128);
          const uint4 *src =
              reinterpret_cast<const uint4 *>(reinterpret_cast<const PrepImage *>(P.prep) + cur.j);
          uint4 *dst = reinterpret_cast<uint4 *>(&S.img[wg][bufA]);
          for (int i = row; i < (int)(sizeof(PrepImage) / 16); i += 128) dst[i] = src[i];
          tc::fence_proxy_async_smem();
          tc::bar_sync(bar_id, 128);
        }
        const uint4 *rt = reinterpret_cast<const uint4 *>(rowtabA + cur.a * kRowTab);
        const uint4 *ct = reinterpret_cast<const uint4 *>(coltabA + cur.b * kRowTab);
        rt0 = rt[0]; rth = rt[2]; rtl = rt[3];
        ct0 = ct[0]; cth = ct[2]; ctl = ct[3];
      }
      // ---- stage B (tile k-1): layer-1 epilogue -> A2 --------------------
      if (hasBC) {
        tc::mbar_wait(&S.acc1_full[wg], par);
        tc::fence_after_sync();
        const float sdown = S.img[wg][prev_buf].s2_down;
#pragma unroll
        for (int half = 0; half < 2; half++) {
          uint32_t h[16];
          tc::tmem_ld16(tbase + lane_addr + cACC1 + 16 * half, h);
          tc::tmem_ld_wait();
          if (sdown != 1.0f) {
#pragma unroll
            for (int q = 0; q < 16; q++) h[q] = __float_as_uint(__uint_as_float(h[q]) * sdown);
          }
          uint32_t hi8[8], lo8[8];
#pragma unroll
          for (int q = 0; q < 8; q++)
            relu_split_f16(__uint_as_float(h[2 * q]), __uint_as_float(h[2 * q + 1]), hi8[q], lo8[q]);
          tc::tmem_st8(tbase + lane_addr + cA2 + 8 * half, hi8);
          tc::tmem_st8(tbase + lane_addr + cA2 + 16 + 8 * half, lo8);
        }
        tc::tmem_st_wait();
        tc::fence_before_sync();
        if (row == 0) S.a2_buf[wg] = (uint32_t)prev_buf;
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
        uint32_t lo16[16], hi16[16];
#pragma unroll
        for (int q = 0; q < 8; q++) tc::split_pair_f16(f[2 * q], f[2 * q + 1], lo16[q], lo16[8 + q]);
        uint32_t xh = 0, xl = 0;
        if (KIND == LOPT_VELO_MLP) tc::split_pair_f16(clip01(x.g) * im.escale[16], 0.0f, xh, xl);
        hi16[0] = rth.x; hi16[1] = rth.y; hi16[2] = rth.z;
        hi16[3] = cth.x; hi16[4] = cth.y; hi16[5] = cth.z;
        hi16[6] = (xh & 0xFFFFu) | 0x3C000000u;   // K12 = clip_hi, K13 = fp16 1 (bias)
        hi16[7] = 0u;
        hi16[8] = rtl.x; hi16[9] = rtl.y; hi16[10] = rtl.z;
        hi16[11] = ctl.x; hi16[12] = ctl.y; hi16[13] = ctl.z;
        hi16[14] = xl & 0xFFFFu;
        hi16[15] = 0u;
        tc::tmem_st16(tbase + lane_addr + cA1, lo16);
        tc::tmem_st16(tbase + lane_addr + cA1 + 16, hi16);
        tc::tmem_st_wait();
        tc::fence_before_sync();
        if (row == 0) S.a1_buf[wg] = (uint32_t)bufA;
        mbar_arrive(&S.a1_ready[wg]);
      }
      // ---- stage C (tile k-1): layer-2 epilogue, layer 3, update ---------
      if (hasBC) {
        tc::mbar_wait(&S.acc2_full[wg], par);
        tc::fence_after_sync();
        if (prev_j != red_j) {
          if (red_j >= 0) {
            if (maxabs > 0.0f)
              atomicMax(reinterpret_cast<unsigned int *>(&P.maxabs[red_j]), __float_as_uint(maxabs));
            if (bad) atomicOr(&P.status[red_j], LOPT_STATUS_NONFINITE_PARAM);
          }
          red_j = prev_j;
          maxabs = 0.0f;
          bad = 0;
        }
        const PrepImage &im = S.img[wg][prev_buf];
        const float sup = im.s2_up;
        float2 d2 = make_float2(im.b3[0], 0.0f), m2 = make_float2(im.b3[1], 0.0f);
        const float4 *w30 = reinterpret_cast<const float4 *>(im.w3[0]);
        const float4 *w31 = reinterpret_cast<const float4 *>(im.w3[1]);
#pragma unroll
        for (int half = 0; half < 2; half++) {
          uint32_t h2[16];
          tc::tmem_ld16(tbase + lane_addr + cACC2 + 16 * half, h2);
          tc::tmem_ld_wait();
          if (sup != 1.0f) {
#pragma unroll
            for (int q = 0; q < 16; q++) h2[q] = __float_as_uint(__uint_as_float(h2[q]) * sup);
          }
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const float4 wa = w30[4 * half + q], wb = w31[4 * half + q];
            const float2 h01 = make_float2(fmaxf(__uint_as_float(h2[4 * q]), 0.0f),
                                           fmaxf(__uint_as_float(h2[4 * q + 1]), 0.0f));
            const float2 h23 = make_float2(fmaxf(__uint_as_float(h2[4 * q + 2]), 0.0f),
                                           fmaxf(__uint_as_float(h2[4 * q + 3]), 0.0f));
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
        float out = prev_w + du;
        if (prev_valid) {
          maxabs = fmaxf(maxabs, fabsf(du));
          bad |= !isfinite(out);
          if (apply_decay) out *= decay;   // optim.py:100-101
          *prev_theta = out;
        }
      }
      // ---- shift the pipeline ---------------------------------------------
      if (hasA) {
        prev_buf = bufA;
        prev_j = cur.j;
        prev_valid = cur.valid;
        prev_w = cur.w;
        prev_theta = cur.tp;
        cur = nxt;
      }
    }
    if (red_j >= 0) {
      if (maxabs > 0.0f)
        atomicMax(reinterpret_cast<unsigned int *>(&P.maxabs[red_j]), __float_as_uint(maxabs));
      if (bad) atomicOr(&P.status[red_j], LOPT_STATUS_NONFINITE_PARAM);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == kIssueWarp) tc::tmem_dealloc(tbase, kTmemCols);
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
