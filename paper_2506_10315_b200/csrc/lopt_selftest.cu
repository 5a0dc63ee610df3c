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

}  // namespace lopt

extern "C" int lopt_selftest_umma(int32_t a_in_tmem, int32_t K, const void *A, const void *B,
                                  float *D, void *stream) {
  if (K < 16 || K > 64 || K % 16 != 0 || !A || !B || !D) return LOPT_ERR_INVALID;
  // bit 0: A in TMEM; bit 1: fp16 operands (else bf16)
  lopt::umma_selftest_kernel<<<1, 128, 0, (cudaStream_t)stream>>>(
      a_in_tmem & 1, (a_in_tmem >> 1) & 1, K, (const uint16_t *)A, (const uint16_t *)B, D);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? LOPT_OK : LOPT_ERR_CUDA;
}
