// lopt_selftest.cu -- known-answer test of the tcgen05 building blocks the
// fast path relies on (descriptor encodings, TMEM layouts, commit/mbarrier
// hand-off).  D[128 x 32] = A[128 x K] * B[32 x K]^T with bf16 inputs and f32
// accumulation, A staged either in shared memory or in tensor memory.
#include "lopt_common.cuh"
#include "lopt_tc.cuh"

namespace lopt {

__global__ void __launch_bounds__(128) umma_selftest_kernel(int a_in_tmem, int fp16, int K,
                                                            const uint16_t *A, const uint16_t *B,
                                                            float *D) {
  __shared__ __align__(1024) uint16_t As[128 * 64];
  __shared__ __align__(1024) uint16_t Bs[32 * 64];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  const int slices = K / 16;
  // canonical K-major, no-swizzle layout: slice s (16 K) is [2 halves][rows/8][8 rows][8 k]
  for (int s = 0; s < slices; s++)
    for (int k = 0; k < 16; k++) {
      const int kk = s * 16 + k;
      As[s * 2048 + (k >> 3) * 1024 + (t >> 3) * 64 + (t & 7) * 8 + (k & 7)] = A[t * K + kk];
      if (t < 32) Bs[s * 512 + (k >> 3) * 256 + (t >> 3) * 64 + (t & 7) * 8 + (k & 7)] = B[t * K + kk];
    }
  if (warp == 0) {
    tc::tmem_alloc(&tbase, 128);
    tc::tmem_relinquish();
  }
  if (t == 0) {
    tc::mbar_init(&mbar, 1);
    tc::mbar_fence_init();
  }
  tc::fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t base = tbase;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  if (a_in_tmem) {
    // row t of A -> TMEM lane t, columns 64.. (two bf16 per 32-bit column)
    uint32_t r[32];
#pragma unroll
    for (int j = 0; j < 32; j++) {
      const int k0 = 2 * j;
      uint32_t lo = k0 < K ? A[t * K + k0] : 0, hi = k0 + 1 < K ? A[t * K + k0 + 1] : 0;
      r[j] = lo | (hi << 16);
    }
    tc::tmem_st32(base + lane_off + 64, r);
    tc::tmem_st_wait();
  }
  tc::fence_before_sync();
  __syncthreads();
  if (t == 0) {
    tc::fence_after_sync();
    const uint32_t idesc = fp16 ? tc::idesc_f16_f32(128, 32) : tc::idesc_bf16_f32(128, 32);
    for (int s = 0; s < slices; s++) {
      const uint64_t bdesc = tc::smem_desc_kmajor(tc::smem_u32(Bs + s * 512), 512, 128);
      if (a_in_tmem) {
        tc::mma_ts(base, base + 64 + s * 8, bdesc, idesc, s > 0);
      } else {
        const uint64_t adesc = tc::smem_desc_kmajor(tc::smem_u32(As + s * 2048), 2048, 128);
        tc::mma_ss(base, adesc, bdesc, idesc, s > 0);
      }
    }
    tc::mma_commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after_sync();
  uint32_t d[32];
  tc::tmem_ld32(base + lane_off, d);
  tc::tmem_ld_wait();
#pragma unroll
  for (int j = 0; j < 32; j++) D[t * 32 + j] = __uint_as_float(d[j]);
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(base, 128);
}

// Latency / throughput probe of the MMA shape the fast path uses
// (M=128, N=32, K=16, f16, A in TMEM): `batch` MMAs per commit, `rounds`
// commit->wait round trips, cycles reported per round in out[0].
__global__ void __launch_bounds__(128) umma_probe_kernel(int batch, int rounds, int N, int a_smem,
                                                         int issuers, int rotate, int warp_wide, long long *out) {
  __shared__ __align__(1024) uint16_t Bs[256 * 16];
  __shared__ __align__(1024) uint16_t As[128 * 16];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ __align__(8) uint64_t mbars[4];
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 256 * 16; i += 128) Bs[i] = 0x3C00;
  for (int i = t; i < 128 * 16; i += 128) As[i] = 0x3C00;
  if (warp == 0) {
    tc::tmem_alloc(&tbase, 512);
    tc::tmem_relinquish();
  }
  if (t == 0) {
    tc::mbar_init(&mbar, 1);
    for (int i = 0; i < 4; i++) tc::mbar_init(&mbars[i], 1);
    tc::mbar_fence_init();
  }
  tc::fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t base = tbase;
  if (warp_wide) {
    // `issuers` converged warps, each issuing through elect.sync into its own
    // accumulator columns, descriptors hoisted out of the loop
    if (warp < issuers) {
      const uint32_t idesc = tc::idesc_f16_f32(128, N);
      const uint64_t bdesc = tc::smem_desc_kmajor(tc::smem_u32(Bs), N * 16, 128);
      const uint64_t adesc = tc::smem_desc_kmajor(tc::smem_u32(As), 2048, 128);
      const uint32_t d = base + 64 * warp;
      long long t0 = clock64();
      for (int r = 0; r < rounds; r++) {
        if (tc::elect_one()) {
          for (int b = 0; b < batch; b++) {
            if (a_smem) tc::mma_ss(d, adesc, bdesc, idesc, b > 0);
            else tc::mma_ts(d, base + 256, bdesc, idesc, b > 0);
          }
          tc::mma_commit(&mbars[warp]);
        }
        __syncwarp();
        tc::mbar_wait(&mbars[warp], r & 1);
      }
      long long t1 = clock64();
      if ((t & 31) == 0) out[warp] = (t1 - t0) / rounds;
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(base, 512);
    return;
  }
  if (issuers > 1) {
    // `issuers` warps, lane 0 of each issuing its own MMA stream into its
    // own accumulator columns: does MMA throughput scale with issuers?
    if ((t & 31) == 0 && warp < issuers) {
      const uint32_t idesc = tc::idesc_f16_f32(128, N);
      const uint64_t bdesc = tc::smem_desc_kmajor(tc::smem_u32(Bs), N * 16, 128);
      const uint64_t adesc = tc::smem_desc_kmajor(tc::smem_u32(As), 2048, 128);
      const uint32_t d = base + 64 * warp;
      long long t0 = clock64();
      for (int r = 0; r < rounds; r++) {
#pragma unroll 1
        for (int b = 0; b < batch; b++) {
          if (a_smem) tc::mma_ss(d, adesc, bdesc, idesc, b > 0);
          else tc::mma_ts(d, base + 256, bdesc, idesc, b > 0);
        }
        tc::mma_commit(&mbars[warp]);
        tc::mbar_wait(&mbars[warp], r & 1);
      }
      long long t1 = clock64();
      out[warp] = (t1 - t0) / rounds;
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(base, 512);
    return;
  }
  if (t == 0) {
    const uint32_t idesc = tc::idesc_f16_f32(128, N);
    const uint64_t bdesc = tc::smem_desc_kmajor(tc::smem_u32(Bs), N * 16, 128);
    const uint64_t adesc = tc::smem_desc_kmajor(tc::smem_u32(As), 2048, 128);
    long long t0 = clock64();
    for (int r = 0; r < rounds; r++) {
      for (int b = 0; b < batch; b++) {
        if (a_smem) tc::mma_ss(base, adesc, bdesc, idesc, b > 0);
        else if (rotate) tc::mma_ts(base + (uint32_t)((b & 3) * 64), base + 256, bdesc, idesc, b > 3);
        else tc::mma_ts(base, base + 256, bdesc, idesc, b > 0);
      }
      tc::mma_commit(&mbar);
      tc::mbar_wait(&mbar, r & 1);
    }
    long long t1 = clock64();
    out[0] = (t1 - t0) / rounds;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(base, 512);
}


// TMEM load/store throughput probe: `warps` warps (multiple of 4) each run
// `rounds` iterations of `per` tcgen05.ld (mode 0: x16, 1: x32) or
// tcgen05.st (mode 2: x16) followed by one wait; out[w] = cycles of warp w.
__global__ void __launch_bounds__(1024) tmem_probe_kernel(int mode, int per, int rounds, long long *out) {
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  if (warp == 0) {
    tc::tmem_alloc(&tbase, 512);
    tc::tmem_relinquish();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t lane = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t col = (uint32_t)(((warp >> 2) * 32) & 511);
  const uint32_t ta = tbase + lane + col;
  uint32_t acc = 0;
  uint32_t r[32];
  for (int i = 0; i < 32; i++) r[i] = (uint32_t)(t * 7 + i);
  __syncthreads();
  long long t0 = clock64();
  for (int k = 0; k < rounds; k++) {
    if (mode == 0) {
      for (int q = 0; q < per; q++) {
        uint32_t h[16];
        tc::tmem_ld16(ta + (uint32_t)((q & 1) * 16), h);
        tc::tmem_ld_wait();
        acc ^= h[0] ^ h[15];
      }
    } else if (mode == 1) {
      for (int q = 0; q < per; q++) {
        tc::tmem_ld32(ta, r);
        tc::tmem_ld_wait();
        acc ^= r[0] ^ r[31];
      }
    } else {
      for (int q = 0; q < per; q++) {
        uint32_t h[16];
        for (int i = 0; i < 16; i++) h[i] = r[i] + (uint32_t)q;
        tc::tmem_st16(ta + (uint32_t)((q & 1) * 16), h);
      }
      tc::tmem_st_wait();
    }
  }
  long long t1 = clock64();
  if ((t & 31) == 0) out[warp] = t1 - t0;
  if (acc == 0x12345678u) out[63] = acc;
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

__global__ void expf_selftest_kernel(const float *x, float *y, int64_t n) {
  __shared__ uint64_t tab[32];
  if (threadIdx.x < 32) tab[threadIdx.x] = kExp2Tab[threadIdx.x];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = glibc_expf(x[i], tab);
}

}  // namespace lopt

extern "C" int lopt_selftest_expf(const float *x, float *y, int64_t n, void *stream) {
  if (!x || !y || n < 0) return LOPT_ERR_INVALID;
  lopt::expf_selftest_kernel<<<296, 256, 0, (cudaStream_t)stream>>>(x, y, n);
  return cudaGetLastError() == cudaSuccess ? LOPT_OK : LOPT_ERR_CUDA;
}

extern "C" int lopt_probe_umma(int32_t batch, int32_t rounds, long long *out, void *stream) {
  // batch: low 12 bits = MMAs per commit; bits 12..14 = issuing warps (1..4);
  // bits 16..27 = N (default 32); bit 28 = A from shared memory
  const int b = batch & 0xFFF, N = (batch >> 16) & 0xFFF ? (batch >> 16) & 0xFFF : 32;
  const int issuers = (batch >> 12) & 7 ? (batch >> 12) & 7 : 1;
  const int a_smem = (batch >> 28) & 1, rotate = (batch >> 29) & 1, warp_wide = (batch >> 30) & 1;
  if (N < 16 || N > 256 || N % 16 || issuers > 4) return LOPT_ERR_INVALID;
  lopt::umma_probe_kernel<<<1, 128, 0, (cudaStream_t)stream>>>(b, rounds, N, a_smem, issuers,
                                                               rotate, warp_wide, out);
  return cudaGetLastError() == cudaSuccess ? LOPT_OK : LOPT_ERR_CUDA;
}

extern "C" int lopt_probe_tmem(int32_t warps, int32_t mode, int32_t per, int32_t rounds, long long *out,
                               void *stream) {
  if (warps < 4 || warps > 32 || warps % 4 || mode < 0 || mode > 2 || per < 1) return LOPT_ERR_INVALID;
  lopt::tmem_probe_kernel<<<1, 32 * warps, 0, (cudaStream_t)stream>>>(mode, per, rounds, out);
  return cudaGetLastError() == cudaSuccess ? LOPT_OK : LOPT_ERR_CUDA;
}

extern "C" int lopt_selftest_umma(int32_t a_in_tmem, int32_t K, const void *A, const void *B,
                                  float *D, void *stream) {
  if (K < 16 || K > 64 || K % 16 != 0 || !A || !B || !D) return LOPT_ERR_INVALID;
  // bit 0: A in TMEM; bit 1: fp16 operands (else bf16)
  lopt::umma_selftest_kernel<<<1, 128, 0, (cudaStream_t)stream>>>(
      a_in_tmem & 1, (a_in_tmem >> 1) & 1, K, (const uint16_t *)A, (const uint16_t *)B, D);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? LOPT_OK : LOPT_ERR_CUDA;
}
