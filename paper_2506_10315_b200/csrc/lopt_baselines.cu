// lopt_baselines.cu -- the reference's hand-designed baseline optimizers on the
// device, so the learned step's overhead is
// compared like for like with the reference's own conventions:
//
//   adam_step       optim.py:187-198  bias-corrected Adam, functional, one tensor
//   adafactor_step  optim.py:201-217  factored second moment (state.py:93-113
//                   update_adafactor + features.py:357-362 adafactor_scale),
//                   no momentum, plain step size
//
// Every f32 operation is the reference's, in its order, correctly rounded and
// never contracted (__f*_rn intrinsics), so Adam is bitwise the reference.
// Adafactor's f64 means use fixed (deterministic) orders -- warp trees for the
// row means and mean(r), 64-row chunks for the column means -- instead of
// numpy's pairwise / sequential ones, so they can differ from the reference in
// the last f64 bit; after the f32 rounding the factors agree except on rare
// ties (tests/test_gpu_baselines.py bounds the result at 1 f32 ulp).
#include <algorithm>

#include "lopt_common.cuh"

namespace lopt {

// theta, m, v in place.  omb1 = f32(1 - b1), bc1 = f32(1 - b1**t) etc. come
// from the host, computed with numpy's f32 scalar arithmetic like the reference.
__global__ void __launch_bounds__(256) adam_kernel(float *__restrict__ theta, const float *__restrict__ g,
                                                   float *__restrict__ m, float *__restrict__ v,
                                                   int64_t n, float b1, float omb1, float b2,
                                                   float omb2, float bc1, float bc2, float lr,
                                                   float eps) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    const float m2 = __fadd_rn(__fmul_rn(b1, m[i]), __fmul_rn(omb1, gi));            // optim.py:194
    const float v2 = __fadd_rn(__fmul_rn(b2, v[i]), __fmul_rn(omb2, __fmul_rn(gi, gi)));   // :195
    const float mhat = __fdiv_rn(m2, bc1);                                            // :196
    const float vhat = __fdiv_rn(v2, bc2);                                            // :197
    const float step = __fdiv_rn(__fmul_rn(lr, mhat), __fadd_rn(__fsqrt_rn(vhat), eps));   // :198
    theta[i] = __fsub_rn(theta[i], step);
    m[i] = m2;
    v[i] = v2;
  }
}

// Row means of g^2 (f64), one warp per row, then the EMA (state.py:108-113).
__global__ void __launch_bounds__(256) adafactor_rows_kernel(const float *__restrict__ g, float *__restrict__ r,
                                                             int64_t rows, int64_t cols, float b,
                                                             float omb) {
  const int64_t a = blockIdx.x * 8LL + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (a >= rows) return;
  const float *ga = g + a * cols;
  double s = 0.0;
  for (int64_t k = lane; k < cols; k += 32) {
    const double x = (double)ga[k];
    s += x * x;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    const float mean = (float)(s / (double)cols);
    r[a] = __fadd_rn(__fmul_rn(b, r[a]), __fmul_rn(omb, mean));
  }
}

// Column sums of g^2 over 64-row chunks (f64 partials, chunk q at
// part[q * cols + k]); adafactor_cols_finalize adds the chunks in order.
// (numpy's axis-0 mean adds all rows in sequence; the chunked order can differ
// in the last f64 bit.)
constexpr int kColChunk = 64;
__global__ void __launch_bounds__(256) adafactor_cols_kernel(const float *__restrict__ g,
                                                             double *__restrict__ part,
                                                             int64_t rows, int64_t cols) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= cols) return;
  const int64_t a0 = (int64_t)blockIdx.y * kColChunk, a1 = min(rows, a0 + kColChunk);
  double s = 0.0;
  for (int64_t a = a0; a < a1; a++) {
    const double x = (double)g[a * cols + k];
    s += x * x;
  }
  part[blockIdx.y * cols + k] = s;
}

__global__ void __launch_bounds__(256) adafactor_cols_finalize(const double *__restrict__ part,
                                                               float *__restrict__ c, int64_t rows,
                                                               int64_t cols, int nchunks, float b,
                                                               float omb) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= cols) return;
  double s = 0.0;
  for (int q = 0; q < nchunks; q++) s += part[q * cols + k];
  const float mean = (float)(s / (double)rows);
  c[k] = __fadd_rn(__fmul_rn(b, c[k]), __fmul_rn(omb, mean));   // state.py:111-113
}

// mean(r') in f64, rounded to f32 (features.py:361): one block, fixed order.
__global__ void __launch_bounds__(256) adafactor_meanr_kernel(const float *__restrict__ r, int64_t rows,
                                                              float *__restrict__ out) {
  __shared__ double part[256];
  double s = 0.0;
  for (int64_t a = threadIdx.x; a < rows; a += blockDim.x) s += (double)r[a];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = (float)(part[0] / (double)rows);
}

// theta' = theta - (lr * g) * sqrt(mean_r / (r[a] * c[b] + eps))   (optim.py:216)
__global__ void __launch_bounds__(256) adafactor_apply_kernel(float *__restrict__ theta,
                                                              const float *__restrict__ g,
                                                              const float *__restrict__ r,
                                                              const float *__restrict__ c,
                                                              const float *__restrict__ mean_r,
                                                              int64_t rows, int64_t cols, float lr,
                                                              float eps) {
  const float mr = *mean_r;
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = i / cols, k = i - a * cols;
    const float S = __fsqrt_rn(__fdiv_rn(mr, __fadd_rn(__fmul_rn(r[a], c[k]), eps)));
    theta[i] = __fsub_rn(theta[i], __fmul_rn(__fmul_rn(lr, g[i]), S));
  }
}

static int grid_for(int64_t n) {
  return (int)std::min<int64_t>(148 * 16, std::max<int64_t>(1, (n + 255) / 256));
}

}  // namespace lopt

extern "C" int lopt_adam_step(float *theta, const float *g, float *m, float *v, int64_t n,
                              const float *scalars, void *stream) {
  // scalars: {b1, 1-b1, b2, 1-b2, 1-b1**t, 1-b2**t, lr, eps} as f32
  if (!theta || !g || !m || !v || !scalars || n < 0) return LOPT_ERR_INVALID;
  if (n == 0) return LOPT_OK;
  const float *s = scalars;
  lopt::adam_kernel<<<lopt::grid_for(n), 256, 0, (cudaStream_t)stream>>>(
      theta, g, m, v, n, s[0], s[1], s[2], s[3], s[4], s[5], s[6], s[7]);
  return cudaGetLastError() == cudaSuccess ? LOPT_OK : LOPT_ERR_CUDA;
}

extern "C" int lopt_adafactor_step(float *theta, const float *g, float *r, float *c, int64_t rows,
                                   int64_t cols, const float *scalars, void *scratch,
                                   void *stream) {
  // scalars: {b, 1-b, lr, eps} as f32; scratch: device bytes >= lopt_adafactor_scratch_bytes
  if (!theta || !g || !r || !c || !scalars || !scratch) return LOPT_ERR_INVALID;
  if (rows < 1 || cols < 1) return LOPT_ERR_SHAPE;   // state.py:102-103
  cudaStream_t st = (cudaStream_t)stream;
  const float *s = scalars;
  const int nch = (int)((rows + lopt::kColChunk - 1) / lopt::kColChunk);
  double *part = static_cast<double *>(scratch);
  float *mean_r = reinterpret_cast<float *>(part + (int64_t)nch * cols);
  const unsigned cb = (unsigned)((cols + 255) / 256);
  lopt::adafactor_rows_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(g, r, rows, cols, s[0], s[1]);
  lopt::adafactor_cols_kernel<<<dim3(cb, (unsigned)nch), 256, 0, st>>>(g, part, rows, cols);
  lopt::adafactor_cols_finalize<<<cb, 256, 0, st>>>(part, c, rows, cols, nch, s[0], s[1]);
  lopt::adafactor_meanr_kernel<<<1, 256, 0, st>>>(r, rows, mean_r);
  lopt::adafactor_apply_kernel<<<lopt::grid_for(rows * cols), 256, 0, st>>>(theta, g, r, c, mean_r, rows,
                                                                           cols, s[2], s[3]);
  return cudaGetLastError() == cudaSuccess ? LOPT_OK : LOPT_ERR_CUDA;
}

extern "C" int64_t lopt_adafactor_scratch_bytes(int64_t rows, int64_t cols) {
  if (rows < 1 || cols < 1) return 0;
  return ((rows + lopt::kColChunk - 1) / lopt::kColChunk) * cols * 8 + 16;
}
