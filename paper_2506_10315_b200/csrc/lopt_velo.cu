// lopt_velo.cu -- the VeLO per-tensor hypernetwork (build-defined; the
// reference has none, SPEC.md:14 / SURVEY.md section 8(a) row 15).
//
// One CTA per tensor, between the (merged) phase-1 statistics and phase 2:
//   x   = [f32(log(sumsq_k / count + 1e-5)) for the 29 VeLO columns |
//          tanh(t/x) for the 11 horizons of features.py:52 | 2 loss features]
//   g   = b + W_x x + W_h h                   (f32 fma chains, inputs in order)
//   c'  = sig(g_f) c + sig(g_i) tanh(g_g),  h' = sig(g_o) tanh(c')
//   a   = softmax(b_o + W_o h')                (bank_size mixing weights)
//   W_j = sum_k a_k * bank_k                   (every layer, weights and biases)
// W_j is written into the plan's weight slot j, so the per-element kernels run
// a different MLP per tensor.  The numpy restatement that pins this is
// oracle/velo_lstm.py.
#include "lopt_common.cuh"

namespace lopt {

constexpr int kVeloIn = 42;
constexpr int kVeloMaxH = 64;
constexpr int kVeloMaxK = 16;

__device__ __forceinline__ float sigm(float z) { return 1.0f / (1.0f + expf(-z)); }

__global__ void __launch_bounds__(256) velo_mix_kernel(DevicePlan P, const float *hyper,
                                                       float *lstm_state, const float *bank,
                                                       const float *loss_feats, int H, int K,
                                                       float *mix_out) {
  // a non-finite gradient anywhere in the step (the flag is set by
  // factor_finalize from the all-reduced factor block) changes nothing --
  // optim.py:160-165 -- so the LSTM state must not advance either
  if (*P.abort_flag != 0) return;
  const int j = blockIdx.x;
  const TensorDesc T = P.tensors[j];
  __shared__ float x[kVeloIn];
  __shared__ float h[kVeloMaxH], c[kVeloMaxH], gates[4 * kVeloMaxH];
  __shared__ float logits[kVeloMaxK];
  const int D = d_feat(P.kind);
  const double count = (double)(T.m * T.n);
  const int tid = threadIdx.x;
  if (tid < D) x[tid] = (float)log(T.sumsq[tid] / count + kEpsNorm);
  if (tid < kTimeFeatures) x[29 + tid] = P.step->tf[tid];
  if (tid < 2) x[40 + tid] = loss_feats ? loss_feats[tid] : P.step->loss[tid];
  float *st = lstm_state + (int64_t)j * 2 * H;
  if (tid < H) {
    h[tid] = st[tid];
    c[tid] = st[H + tid];
  }
  __syncthreads();
  const float *Wx = hyper, *Wh = Wx + 4 * H * kVeloIn, *bg = Wh + 4 * H * H, *Wo = bg + 4 * H,
              *bo = Wo + K * H;
  for (int q = tid; q < 4 * H; q += blockDim.x) {
    float g = bg[q];
    for (int i = 0; i < kVeloIn; i++) g = __fmaf_rn(Wx[q * kVeloIn + i], x[i], g);
    for (int i = 0; i < H; i++) g = __fmaf_rn(Wh[q * H + i], h[i], g);
    gates[q] = g;
  }
  __syncthreads();
  if (tid < H) {
    const float ig = sigm(gates[tid]), fg = sigm(gates[H + tid]);
    const float gg = tanhf(gates[2 * H + tid]), og = sigm(gates[3 * H + tid]);
    const float cn = __fadd_rn(__fmul_rn(fg, c[tid]), __fmul_rn(ig, gg));
    const float hn = __fmul_rn(og, tanhf(cn));
    c[tid] = cn;
    st[H + tid] = cn;
    st[tid] = hn;
  }
  __syncthreads();
  if (tid < H) h[tid] = st[tid];
  __syncthreads();
  if (tid < K) {
    float l = bo[tid];
    for (int i = 0; i < H; i++) l = __fmaf_rn(Wo[tid * H + i], h[i], l);
    logits[tid] = l;
  }
  __syncthreads();
  __shared__ float alpha[kVeloMaxK];
  if (tid == 0) {
    float mx = logits[0];
    for (int k = 1; k < K; k++) mx = fmaxf(mx, logits[k]);
    float s = 0.0f;
    for (int k = 0; k < K; k++) {
      alpha[k] = expf(logits[k] - mx);
      s += alpha[k];
    }
    for (int k = 0; k < K; k++) alpha[k] = alpha[k] / s;
    if (mix_out)
      for (int k = 0; k < K; k++) mix_out[(int64_t)j * K + k] = alpha[k];
  }
  __syncthreads();
  float *dst = const_cast<float *>(P.weights) + (int64_t)T.weight_slot * P.weight_stride;
  for (int p = tid; p < P.weight_stride; p += blockDim.x) {
    float v = 0.0f;
    for (int k = 0; k < K; k++) v = __fmaf_rn(alpha[k], bank[(int64_t)k * P.weight_stride + p], v);
    dst[p] = v;
  }
}

int launch_velo_mix(const DevicePlan &P, const float *hyper, float *lstm_state, const float *bank,
                    const float *loss_feats, int H, int K, float *mix_out, cudaStream_t s) {
  if (H < 1 || H > kVeloMaxH || K < 1 || K > kVeloMaxK || P.kind != LOPT_VELO_MLP)
    return LOPT_ERR_INVALID;
  velo_mix_kernel<<<P.count, 256, 0, s>>>(P, hyper, lstm_state, bank, loss_feats, H, K, mix_out);
  return cudaGetLastError() == cudaSuccess ? LOPT_OK : LOPT_ERR_CUDA;
}

}  // namespace lopt
