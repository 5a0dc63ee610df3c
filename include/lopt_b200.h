/*
 * lopt_b200.h -- C ABI of the B200 learned-optimizer step.
 *
 * Plain pointers, sizes and a CUDA stream handle; no torch types.  Every entry
 * point is stream-ordered on the caller's stream and returns an int status
 * (LOPT_OK = 0).  Data-dependent conditions (non-finite gradient, non-finite
 * updated parameter) do not fail the call: they set per-tensor bits in the
 * device status words that lopt_read_status() returns.
 *
 * Reference interface each entry point replaces (paths relative to the
 * reference repository, pkg/src/lopt/):
 *
 *   lopt_plan_create      OptimizerHandle.fresh / __post_init__  optim.py:121-141
 *                         (shape checks of engine.py:583-594 _check_step_inputs)
 *   lopt_workspace_bytes  ScratchTracker accounting               engine.py:88-117
 *   lopt_set_weights      LoptWeights / weights_from_entries      engine.py:119-163, 212-228
 *   lopt_factor_partials  update_adafactor's f64 row/col sums     state.py:93-113
 *                         (and distsim's per-shard bincount partials distsim.py:448-453)
 *   lopt_factor_finalize  update_adafactor EMA + factor_means    state.py:108-113, features.py:133-135
 *                         (the coordinator merge of distsim.py:457-474)
 *   lopt_feature_stats    fused_stats (pass 1)                    engine.py:619-654
 *   lopt_apply            fused_apply (pass 2) + state_step's    engine.py:657-710,
 *                         M/V EMAs + apply_weight_decay          state.py:77-90, optim.py:92-101
 *   lopt_step             opt_step for one device                 optim.py:144-180
 *   lopt_read_status      UpdateOverflowError / OptimError        engine.py:737-738, optim.py:164-165
 *
 * Multi-GPU: lopt_factor_partials and lopt_feature_stats leave f64 partial
 * sums in two contiguous workspace blocks (lopt_factor_sums_ptr,
 * lopt_stat_sums_ptr); a caller that shards elements across ranks all-reduces
 * those blocks (sum, float64) between the phases -- the "factor merge" and
 * "stats merge" of distsim.py:427-499.
 */
#ifndef LOPT_B200_H
#define LOPT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define LOPT_OK 0
#define LOPT_ERR_INVALID 1      /* bad argument / descriptor */
#define LOPT_ERR_SHAPE 2        /* shape mismatch or empty tensor (EngineError) */
#define LOPT_ERR_WORKSPACE 3    /* workspace missing or too small (ScratchLimitError) */
#define LOPT_ERR_CUDA 4         /* a CUDA runtime call failed */
#define LOPT_ERR_UNSUPPORTED 5  /* topology / mode not compiled */

/* feature sets (features.py:52-104) */
#define LOPT_SMALL_FC_LOPT 0    /* 39 columns */
#define LOPT_VELO_MLP 1         /* 29 columns */

/* execution modes */
#define LOPT_MODE_STRICT 0      /* CUDA-core, bitwise features/MLP/expf */
#define LOPT_MODE_FAST 1        /* folded features, tcgen05 MLP, fp32 tolerance */

/* per-tensor status bits (lopt_read_status) */
#define LOPT_STATUS_NONFINITE_GRAD 1u
#define LOPT_STATUS_NONFINITE_PARAM 2u

/* One parameter tensor in its 2-D view (tensors.py:66-100: 1-D -> (n,1)).
 * theta/grad cover the whole m*n tensor; the call steps elements [lo, hi).
 * state holds 4 floats per stepped element {M1, M2, M3, V} for [lo, hi)
 * (state[4*(i-lo) + k]).  row_factors = r5|r6|r7 (3*m floats), col_factors =
 * c5|c6|c7 (3*n floats), full length on every rank. */
typedef struct lopt_tensor {
  int64_t m, n;
  int64_t lo, hi;
  float *theta;
  const float *grad;
  float *state;
  float *row_factors;
  float *col_factors;
  int32_t weight_slot;    /* index into the weight sets of lopt_set_weights */
  int32_t reserved;
} lopt_tensor;

typedef struct lopt_config {
  int32_t feature_set;    /* LOPT_SMALL_FC_LOPT | LOPT_VELO_MLP */
  int32_t mode;           /* LOPT_MODE_STRICT | LOPT_MODE_FAST */
  int32_t hidden1, hidden2;  /* MLP widths; 32,32 for the reference optimizers */
  int32_t num_weight_sets;   /* 1 = one global MLP; >1 = per-tensor sets (VeLO) */
  int32_t state_advanced; /* 1: state/factors already advanced for grad (engine-level
                             calls mirroring step_fused); 0: advance inside the step */
  double betas[7];        /* momentum x3, second moment, adafactor x3 (state.py:25-40) */
  float alpha, beta_out;  /* update rule constants (engine.py:61-62) */
  int32_t update_sign;    /* -1 or +1 */
  int32_t reserved;
} lopt_config;

/* Per-step host scalars, produced exactly as the reference does:
 * lr = schedule_lr(T) before the increment (optim.py:156), tf = numpy
 * tanh(f32(t)/x) at the post-increment t (features.py:125-130). */
typedef struct lopt_step_args {
  double lr;
  double weight_decay;
  float time_features[11];
  int32_t t;              /* post-increment step counter */
  /* VeLO hypernetwork loss inputs {log(loss), EMA of log(loss)} (build-defined,
   * no reference counterpart); read by the hypernetwork when it was registered
   * (lopt_set_velo / lopt_velo_mix) with loss_feats == NULL, else ignored. */
  float loss_features[2];
} lopt_step_args;

typedef struct lopt_plan lopt_plan;

int lopt_plan_create(const lopt_tensor *tensors, int32_t count, const lopt_config *cfg,
                     lopt_plan **out);
int lopt_plan_destroy(lopt_plan *plan);
int lopt_workspace_bytes(const lopt_plan *plan, size_t *bytes);
/* Binds caller-owned device memory and uploads the descriptor tables (on stream). */
int lopt_bind_workspace(lopt_plan *plan, void *dev_ptr, size_t bytes, void *stream);
/* Re-points theta/grad/state/factor pointers (e.g. torch re-allocated .grad)
 * without changing shapes or ranges; re-uploads the descriptor table. */
int lopt_rebind_tensors(lopt_plan *plan, const lopt_tensor *tensors, int32_t count, void *stream);
/* MLP weights for set `slot`, device or host pointer to the packed layout
 * w1 (h1 x d) | b1 (h1) | w2 (h2 x h1) | b2 (h2) | w3 (2 x h2) | b3 (2).
 * A fast plan with one weight set also keeps w3 on the host for the apply
 * kernel's launch parameter (a device source is read back synchronously on
 * `stream`). */
int lopt_set_weights(lopt_plan *plan, int32_t slot, const float *packed, int32_t is_device,
                     void *stream);
/* Device pointer to the per-set packed weights (for weights produced on the GPU,
 * e.g. the VeLO mixing kernel).  From the first call on, the plan reads layer 3
 * from device memory every step (writes through the pointer take effect). */
int lopt_weights_ptr(lopt_plan *plan, int32_t slot, float **dev_ptr);
int lopt_set_step_args(lopt_plan *plan, const lopt_step_args *args, void *stream);
/* Element count behind each tensor's feature statistics, used by the apply
 * pass's normalization 1/sqrt(sumsq/count + eps) (features.py:138-140) --
 * fused_apply's `stats.count` (engine.py:657-710), which the reference accepts
 * for a partial range; counts[j] == 0 or counts == NULL: the whole tensor. */
int lopt_set_stat_counts(lopt_plan *plan, const int64_t *counts, void *stream);

int lopt_factor_partials(lopt_plan *plan, void *stream);
int lopt_factor_finalize(lopt_plan *plan, void *stream);
int lopt_feature_stats(lopt_plan *plan, void *stream);
int lopt_apply(lopt_plan *plan, void *stream);
int lopt_step(lopt_plan *plan, const lopt_step_args *args, void *stream);
/* The same step (including a registered VeLO hypernetwork) replayed from a
 * CUDA graph captured on the first call: one launch per step instead of ~10,
 * the step scalars patched into the graph's first kernel.  The capture holds
 * the plan's device pointers; lopt_rebind_tensors / lopt_set_weights keep it
 * valid (they rewrite device tables), lopt_set_peers / lopt_set_velo drop it.
 * lopt_graph_reset drops it explicitly.  Replaces opt_step's per-step
 * dispatch (optim.py:144-180) for a launch-bound caller. */
int lopt_graph_step(lopt_plan *plan, const lopt_step_args *args, void *stream);
int lopt_graph_reset(lopt_plan *plan);
/* Phase timing for a benchmark (no reference counterpart).  With `slots` > 0
 * the plan owns slots x 5 timing events; each lopt_step / lopt_graph_step
 * uses the next set in turn and records it on its stream before phase 1a,
 * after 1a (factors), after 1b (feature statistics), after the VeLO
 * hypernetwork and after phase 2 (apply) -- phase times of the measured steps
 * themselves (a graph captured with timing holds event-record nodes,
 * re-pointed to the step's set before every launch).  slots 0 turns it off;
 * turning it on or off recaptures the graph.  lopt_phase_slot: the set the
 * next step uses; lopt_phase_elapsed: ms between marks k0 and k1 (0-4) of a
 * set, once that step completed. */
int lopt_set_phase_timing(lopt_plan *plan, int32_t slots);
int lopt_phase_slot(const lopt_plan *plan, int32_t *next_slot);
int lopt_phase_elapsed(lopt_plan *plan, int32_t slot, int32_t k0, int32_t k1, float *ms);

/* contiguous f64 blocks to all-reduce across element-sharded ranks */
int lopt_factor_sums_ptr(lopt_plan *plan, double **ptr, int64_t *count);
int lopt_stat_sums_ptr(lopt_plan *plan, double **ptr, int64_t *count);
/* per-tensor results: status bits and max |update| (UpdateReport.max_abs_update) */
int lopt_status_ptr(lopt_plan *plan, uint32_t **status, float **maxabs);
int lopt_read_status(lopt_plan *plan, uint32_t *status_host, float *maxabs_host, void *stream);
/* per-tensor f64 feature sums and f32 factor means (for parity tests) */
int lopt_debug_ptrs(lopt_plan *plan, double **sumsq, float **factor_means);

/* VeLO per-tensor hypernetwork (build-defined, no reference counterpart;
 * SURVEY.md section 8(a) row 15).  Runs between lopt_feature_stats (after any
 * cross-rank stats merge) and lopt_apply: for every tensor j one LSTM step on
 * x_j = [log(sumsq_j/count_j + 1e-5) (29) | tanh(t/x) (11) | loss features (2)],
 * softmax over a head -> mixing weights a_j (bank_size), and the per-tensor
 * MLP sum_k a_jk * bank_k written into weight slot j (the plan must have
 * num_weight_sets == count and tensor j using slot j).  All pointers are
 * device pointers: hyper = W_x (4H x 42) | W_h (4H x H) | b (4H) | W_o (K x H)
 * | b_o (K); lstm_state = count x (h[H] | c[H]), updated in place; bank = K
 * packed MLPs (lopt_set_weights layout); loss_feats = 2 floats; mix_out =
 * count x K mixing weights (may be NULL).  hidden <= 64, bank_size <= 16. */
int lopt_velo_mix(lopt_plan *plan, const float *hyper, float *lstm_state, const float *bank,
                  const float *loss_feats, int32_t hidden, int32_t bank_size, float *mix_out,
                  void *stream);

/* Registers the VeLO hypernetwork (same arguments as lopt_velo_mix) so that
 * lopt_step / lopt_graph_step run it between phases 1 and 2 of a one-device
 * step; hyper = NULL unregisters.  Element-sharded callers merge the stats
 * first and call lopt_velo_mix themselves. */
int lopt_set_velo(lopt_plan *plan, const float *hyper, float *lstm_state, const float *bank,
                  const float *loss_feats, int32_t hidden, int32_t bank_size, float *mix_out);

/* Known-answer test of the tcgen05 building blocks (device pointers):
 * D[128 x 32] f32 = A[128 x K] * B[32 x K]^T, K in {16,32,48,64}; flag bit 0:
 * A staged in tensor memory (else shared memory), bit 1: fp16 operands (else bf16). */
int lopt_selftest_umma(int32_t a_in_tmem, int32_t K, const void *A, const void *B, float *D,
                       void *stream);
/* The strict path's expf (glibc's algorithm restated, lopt_common.cuh) over a
 * device array, for the bitwise test against the host libm. */
int lopt_selftest_expf(const float *x, float *y, int64_t n, void *stream);
/* Micro-benchmark of the fast path's MMA shape: `batch` MMAs per commit,
 * `rounds` commit/wait round trips; out[0] = SM cycles per round. */
int lopt_probe_umma(int32_t batch, int32_t rounds, long long *out, void *stream);
/* ---- the reference's hand-designed baselines ----
 * adam_step, optim.py:187-198: theta, m, v (n f32 each) updated in place.
 * `scalars` (HOST pointer, 8 f32): {f32(b1), f32(1)-f32(b1), f32(b2), f32(1)-f32(b2),
 * f32(1)-f32(b1)**f32(t), f32(1)-f32(b2)**f32(t), f32(lr), f32(eps)} -- the
 * reference's numpy f32 scalars; every element op is the reference's, in order. */
int lopt_adam_step(float *theta, const float *g, float *m, float *v, int64_t n,
                   const float *scalars, void *stream);
/* adafactor_step, optim.py:201-217 (update_adafactor state.py:93-113,
 * adafactor_scale features.py:357-362): theta (rows x cols), r (rows), c (cols)
 * updated in place.  `scalars` (HOST pointer, 4 f32): {f32(beta),
 * f32(1)-f32(beta), f32(lr), f32(eps)}; `scratch`: device memory of
 * lopt_adafactor_scratch_bytes(rows, cols) bytes (8-byte aligned). */
int lopt_adafactor_step(float *theta, const float *g, float *r, float *c, int64_t rows,
                        int64_t cols, const float *scalars, void *scratch, void *stream);
int64_t lopt_adafactor_scratch_bytes(int64_t rows, int64_t cols);
/* TMEM ld/st throughput probe (development tool, no reference counterpart). */
int lopt_probe_tmem(int32_t warps, int32_t mode, int32_t per, int32_t rounds, long long *out, void *stream);

/* Fused parameter all-gather over NVLink (sharded step, replaces the
 * all-gather of distsim.py:523-530): every parameter the fast-mode apply pass
 * writes is also stored to `count` (<= LOPT_MAX_PEERS) peer copies at
 * byte offset deltas[p] from its local address -- the peers' parameter arenas
 * mapped into this process (CUDA IPC / symmetric memory), so the parameter
 * exchange rides on the apply kernel's own stores instead of a separate
 * collective.  count = 0 disables it.  The caller orders the peers' writes
 * before the next use of the parameters (a cross-rank barrier after the step). */
#define LOPT_MAX_PEERS 7
/* Enables the current device's kernels to access `peer_device`'s memory
 * (NVLink peer access), once per pair; LOPT_ERR_UNSUPPORTED without P2P.
 * The fused exchange calls it for every peer before lopt_set_peers. */
int lopt_enable_peer_access(int32_t peer_device);
int lopt_set_peers(lopt_plan *plan, int32_t count, const int64_t *deltas);

const char *lopt_version(void);
int lopt_num_kernels_launched_last_step(const lopt_plan *plan);

#ifdef __cplusplus
}
#endif
#endif
