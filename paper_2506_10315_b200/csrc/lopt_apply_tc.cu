// lopt_apply_tc.cu -- phase 2 of the fast path on the tensor cores.
//
// engine.py:657-710 fused_apply + state.py:77-90 + optim.py:171-172 for
// 128-element tiles: features -> layer 1 (tcgen05, M=128 x N=32) -> ReLU ->
// layer 2 (tcgen05) -> ReLU -> layer 3 (CUDA cores, f32) -> exp -> update ->
// decay -> store theta and the advanced accumulators.
//
// fp32 accuracy on bf16 tensor cores: every operand is split in two bf16 terms
// (x = x_hi + x_lo) and each product is formed as x_hi*W_hi + x_hi*W_lo +
// x_lo*W_hi with f32 accumulation (relative error ~2^-16).  The A operands
// are written from registers straight into tensor memory (tcgen05.st) and the
// MMAs read them from there (A-in-TMEM form), so the per-element operands
// never cross shared memory; only the per-tensor B operands live in smem.
//
// Structure: persistent kernel, one CTA per SM, three independent 128-thread
// warpgroups.  Thread i of a warpgroup owns row i of every tile (TMEM lane i).
// Each warpgroup software-pipelines its contiguous tile range three deep:
// iteration k runs stage B of tile k-1 (layer-1 epilogue, issues layer 2),
// stage A of tile k (loads prefetched one iteration earlier, features,
// issues layer 1) and stage C of tile k-1 (layer-2 epilogue, update, stores),
// so every MMA has a full stage of CUDA-core work to hide behind, and the
// next tile's HBM loads are in flight during the whole iteration.
#include "lopt_fast.cuh"

namespace lopt {

constexpr int kWGs = 3;
constexpr int kApplyThreads = 128 * kWGs;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColsPerWG = 128;      // A1 | ACC1 | A2 | ACC2, 32 columns each
constexpr uint32_t kOnesCol = kColsPerWG * kWGs;

struct __align__(128) ApplySmem {
  PrepImage img[kWGs][2];   // double-buffered per warpgroup (tensor switches)
  uint64_t exptab[32];
  uint64_t bar_acc1[kWGs];
  uint64_t bar_acc2[kWGs];
  uint32_t tmem_base;
};

struct TileLoad {
  int j;
  bool valid;
  int64_t e, a, b;   // flat element and its (row, column)
  float w, g;
  float4 s;
};

// Walks a warpgroup's contiguous tile range: current tensor, tile origin
// (row a0, column b0) advanced incrementally from tile to tile.
struct TileWalker {
  int j = -1;
  int64_t next_tile0 = -1, tile0 = 0, lo = 0, hi = 0, n = 1, t = -2, a0 = 0, b0 = 0;
};

__device__ __forceinline__ void walk_to(const DevicePlan &P, TileWalker &W, int64_t t) {
  if (W.j < 0 || t >= W.next_tile0) {
    int j = W.j < 0 ? 0 : W.j;
    while (j + 1 < P.count && P.tensors[j + 1].tile0 <= t) j++;
    const TensorDesc *T = P.tensors + j;
    W.j = j;
    W.tile0 = T->tile0;
    W.lo = T->lo;
    W.hi = T->hi;
    W.n = T->n;
    W.next_tile0 = j + 1 < P.count ? P.tensors[j + 1].tile0 : INT64_MAX;
    W.t = -2;
  }
  const int64_t e0 = W.lo + (t - W.tile0) * kTile;
  if (t == W.t + 1 && W.n >= kTile) {
    W.b0 += kTile;
    if (W.b0 >= W.n) {
      W.b0 -= W.n;
      W.a0++;
      if (W.b0 >= W.n) {   // only when n < 2*kTile... keep exact
        W.a0 += W.b0 / W.n;
        W.b0 %= W.n;
      }
    }
  } else {
    W.a0 = e0 / W.n;
    W.b0 = e0 - W.a0 * W.n;
  }
  W.t = t;
}

__device__ __forceinline__ void load_tile(const DevicePlan &P, TileWalker &W, int64_t t, int row,
                                          TileLoad &L) {
  walk_to(P, W, t);
  const TensorDesc *T = P.tensors + W.j;
  L.j = W.j;
  L.e = W.lo + (t - W.tile0) * kTile + row;
  L.valid = L.e < W.hi;
  int64_t b = W.b0 + row, a = W.a0;
  if (b >= W.n) {
    if (W.n >= kTile) {
      b -= W.n;
      a++;
    } else {
      const uint32_t q = (uint32_t)b / (uint32_t)W.n;
      a += q;
      b -= (int64_t)q * W.n;
    }
  }
  L.a = a;
  L.b = b;
  if (L.valid) {
    L.w = __ldg(T->theta + L.e);
    L.g = __ldg(T->grad + L.e);
    L.s = __ldg(T->state + (L.e - W.lo));
  } else {
    L.w = L.g = 0.0f;
    L.s = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

template <int KIND>
__global__ void __launch_bounds__(kApplyThreads, 1) apply_tc_kernel(DevicePlan P) {
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
  const uint32_t cA1 = kColsPerWG * wg, cACC1 = cA1 + 32, cA2 = cA1 + 64, cACC2 = cA1 + 96;
  if (wg == 0) {
    // constant A slice for the layer-2 bias MMA: K0 = K1 = 1
    uint32_t r[16];
#pragma unroll
    for (int q = 0; q < 16; q++) r[q] = q == 0 ? 0x3C003C00u : 0u;   // fp16 {1, 1}
    tc::tmem_st16(tbase + lane_addr + kOnesCol, r);
    tc::tmem_st_wait();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();

  const bool adv = P.state_advanced != 0;
  const float alpha = P.alpha, beta_out = P.beta_out;
  const float ds = P.step->ds, decay = P.step->decay;
  const bool apply_decay = P.step->apply_decay != 0;
  constexpr uint32_t kIdesc = tc::idesc_f16_f32(128, 32);
  const int bar_id = 1 + wg;

  const int64_t nwg = (int64_t)gridDim.x * kWGs;
  const int64_t gwg = (int64_t)blockIdx.x * kWGs + wg;
  const int64_t tb = P.n_tiles * gwg / nwg, te = P.n_tiles * (gwg + 1) / nwg;
  if (*P.abort_flag != 0 || tb >= te) {
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tbase, kTmemCols);
    return;
  }

  int jwalk = 0;
  TileLoad cur, nxt;
  load_tile(P, jwalk, tb, row, cur);
  // stage-A tensor / buffer tracking
  int bufA = 1, bufA_j = -1;
  int64_t nA = 1;
  double inv_nA = 1.0;
  const float *rowtabA = nullptr, *coltabA = nullptr;
  // carry from stage A(k-1) to stages B/C(k-1)
  int prev_buf = 0, prev_j = -1;
  bool prev_valid = false;
  float prev_w = 0.0f;
  float4 prev_ns = make_float4(0.f, 0.f, 0.f, 0.f);
  float *prev_theta = nullptr;
  float4 *prev_state = nullptr;
  // per-tensor reductions of stage C
  int red_j = -1;
  float maxabs = 0.0f;
  uint32_t bad = 0;

  for (int64_t k = tb; k <= te; k++) {
    const bool hasA = k < te, hasBC = k > tb;
    const uint32_t par = (uint32_t)((k - 1 - tb) & 1);
    if (k + 1 < te) load_tile(P, jwalk, k + 1, row, nxt);
    // ---- stage A prologue: tensor switch, table loads --------------------
    uint4 rt0 = make_uint4(0, 0, 0, 0), rth = rt0, rtl = rt0, ct0 = rt0, cth = rt0, ctl = rt0;
    if (hasA) {
      if (cur.j != bufA_j) {
        bufA ^= 1;
        bufA_j = cur.j;
        const TensorDesc *T = P.tensors + cur.j;
        nA = T->n;
        inv_nA = 1.0 / (double)nA;
        rowtabA = T->rowtab;
        coltabA = T->coltab;
        // buffer bufA was last read by MMAs that completed before stage C of
        // an earlier iteration; all warps of the group must be past that
        tc::bar_sync(bar_id, 128);
        const uint4 *src = reinterpret_cast<const uint4 *>(reinterpret_cast<const PrepImage *>(P.prep) + cur.j);
        uint4 *dst = reinterpret_cast<uint4 *>(&S.img[wg][bufA]);
        for (int i = row; i < (int)(sizeof(PrepImage) / 16); i += 128) dst[i] = src[i];
        tc::fence_proxy_async_smem();
        tc::bar_sync(bar_id, 128);
      }
      if (cur.valid) {
        int64_t a, b;
        divmod(cur.e, nA, inv_nA, a, b);
        const uint4 *rt = reinterpret_cast<const uint4 *>(rowtabA + a * kRowTab);
        const uint4 *ct = reinterpret_cast<const uint4 *>(coltabA + b * kRowTab);
        rt0 = rt[0]; rth = rt[2]; rtl = rt[3];
        ct0 = ct[0]; cth = ct[2]; ctl = ct[3];
      }
    }
    // ---- stage B (tile k-1): layer-1 epilogue, issue layer 2 --------------
    if (hasBC) {
      tc::mbar_wait(&S.bar_acc1[wg], par);
      tc::fence_after_sync();
      uint32_t h[32];
      tc::tmem_ld32(tbase + lane_addr + cACC1, h);
      tc::tmem_ld_wait();
      uint32_t a2[32];
      const float sdown = S.img[wg][prev_buf].s2_down;
      if (sdown != 1.0f) {
#pragma unroll
        for (int q = 0; q < 32; q++) h[q] = __float_as_uint(__uint_as_float(h[q]) * sdown);
      }
#pragma unroll
      for (int q = 0; q < 16; q++) {
        const float u = fmaxf(__uint_as_float(h[2 * q]), 0.0f);
        const float v = fmaxf(__uint_as_float(h[2 * q + 1]), 0.0f);
        tc::split_pair_f16(u, v, a2[q], a2[16 + q]);
      }
      tc::tmem_st32(tbase + lane_addr + cA2, a2);
      tc::tmem_st_wait();
      tc::fence_before_sync();
      tc::bar_sync(bar_id, 128);
      if (row == 0) {
        tc::fence_after_sync();
        const PrepImage &im = S.img[wg][prev_buf];
        const uint32_t d = tbase + cACC2, a = tbase + cA2;
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
        tc::mma_commit(&S.bar_acc2[wg]);
      }
    }
    // ---- stage A (tile k): features -> A1, issue layer 1 -------------------
    float4 ns = make_float4(0.f, 0.f, 0.f, 0.f);
    if (hasA) {
      const PrepImage &im = S.img[wg][bufA];
      FastIn x;
      x.w = cur.w;
      advance(cur.g, cur.s, adv, P.beta, x);
      ns = make_float4(x.m1, x.m2, x.m3, x.v);
      uint32_t lo16[16], hi16[16];
      if (cur.valid) {
        const float rc[3] = {__uint_as_float(rt0.x), __uint_as_float(rt0.y), __uint_as_float(rt0.z)};
        const float cc[3] = {__uint_as_float(ct0.x), __uint_as_float(ct0.y), __uint_as_float(ct0.z)};
        const float sq[3] = {im.sqmr[0], im.sqmr[1], im.sqmr[2]};
        float f[16];
        fast_features(x, rc, cc, sq, f);
        // normalize (features.py:349-354) so every operand fits fp16
#pragma unroll
        for (int q = 0; q < 16; q++) f[q] *= im.escale[q];
#pragma unroll
        for (int q = 0; q < 8; q++)
          tc::split_pair_f16(f[2 * q], f[2 * q + 1], lo16[q], lo16[8 + q]);
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
      } else {
#pragma unroll
        for (int q = 0; q < 16; q++) lo16[q] = hi16[q] = 0u;
      }
      tc::tmem_st16(tbase + lane_addr + cA1, lo16);
      tc::tmem_st16(tbase + lane_addr + cA1 + 16, hi16);
      tc::tmem_st_wait();
      tc::fence_before_sync();
      tc::bar_sync(bar_id, 128);
      if (row == 0) {
        tc::fence_after_sync();
        const uint32_t d = tbase + cACC1, a = tbase + cA1;
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
        tc::mma_commit(&S.bar_acc1[wg]);
      }
    }
    // ---- stage C (tile k-1): layer-2 epilogue, layer 3, update -------------
    if (hasBC) {
      tc::mbar_wait(&S.bar_acc2[wg], par);
      tc::fence_after_sync();
      uint32_t h2[32];
      tc::tmem_ld32(tbase + lane_addr + cACC2, h2);
      tc::tmem_ld_wait();
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
      if (prev_valid) {
        const PrepImage &im = S.img[wg][prev_buf];
        float dir = im.b3[0], mag = im.b3[1];
        const float sup = im.s2_up;
#pragma unroll
        for (int q = 0; q < 32; q++) {
          const float hv = fmaxf(__uint_as_float(h2[q]) * sup, 0.0f);
          dir = fmaf(im.w3[0][q], hv, dir);
          mag = fmaf(im.w3[1][q], hv, mag);
        }
        // engine.py:537-539
        const float ex = glibc_expf(__fmul_rn(mag, alpha), S.exptab);
        const float upd = __fmul_rn(__fmul_rn(dir, ex), beta_out);
        const float du = __fmul_rn(ds, upd);
        float out = __fadd_rn(prev_w, du);
        maxabs = fmaxf(maxabs, fabsf(du));
        bad |= !isfinite(out);
        if (apply_decay) out = __fmul_rn(out, decay);   // optim.py:100-101
        *prev_theta = out;
        if (!adv) *prev_state = prev_ns;
      }
    }
    // ---- shift the pipeline -------------------------------------------------
    if (hasA) {
      const TensorDesc *T = P.tensors + cur.j;
      prev_buf = bufA;
      prev_j = cur.j;
      prev_valid = cur.valid;
      prev_w = cur.w;
      prev_ns = ns;
      prev_theta = T->theta + cur.e;
      prev_state = T->state + (cur.e - T->lo);
      cur = nxt;
    }
  }
  if (red_j >= 0) {
    if (maxabs > 0.0f)
      atomicMax(reinterpret_cast<unsigned int *>(&P.maxabs[red_j]), __float_as_uint(maxabs));
    if (bad) atomicOr(&P.status[red_j], LOPT_STATUS_NONFINITE_PARAM);
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, kTmemCols);
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
