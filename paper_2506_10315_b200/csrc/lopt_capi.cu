// lopt_capi.cu -- host side of the C ABI declared in include/lopt_b200.h.
//
// A plan is built once per parameter list (the OptimizerHandle of
// optim.py:104-141): it validates shapes, cuts every tensor into phase-0
// tiles and phase-1/2 element chunks, and lays out one caller-owned device
// workspace that holds the descriptor tables, the f64 partial sums and the
// per-step scalars.  Steps then only launch kernels on the caller's stream.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "lopt_common.cuh"

namespace lopt {
void launch_factor_partials(const DevicePlan &P, cudaStream_t s);
void launch_factor_reduce(const DevicePlan &P, int64_t max_mn, cudaStream_t s);
void launch_factor_finalize(const DevicePlan &P, int64_t max_mn, cudaStream_t s);
void launch_factor_means(const DevicePlan &P, cudaStream_t s);
void launch_factor_reduce_finalize(const DevicePlan &P, cudaStream_t s);
void launch_strict_stats(const DevicePlan &P, cudaStream_t s);
void launch_stats_reduce(const DevicePlan &P, cudaStream_t s);
void launch_strict_apply(const DevicePlan &P, cudaStream_t s);
void launch_maxabs_reduce(const DevicePlan &P, cudaStream_t s);
int fast_supported(const DevicePlan &P);
void launch_fast_stats(const DevicePlan &P, cudaStream_t s);
void launch_fast_apply(const DevicePlan &P, cudaStream_t s);
int64_t fast_stat_chunk();
int64_t fast_stat_strip();
int fast_stat_min_blocks();
int64_t fast_apply_chunk();
size_t prep_image_bytes();
int64_t factor_strip_cols();
int launch_velo_mix(const DevicePlan &P, const float *hyper, float *lstm_state, const float *bank,
                    const float *loss_feats, int H, int K, float *mix_out, cudaStream_t s);

// First kernel of every step: publishes the step scalars (by value, so the
// launch is stream-ordered and graph-capturable -- no pageable copy) and
// clears the per-step status words, max |update|, abort flag and the
// non-finite-gradient slot of the factor-sum block.
__global__ void __launch_bounds__(256) begin_step_kernel(DevicePlan P, StepScalars h,
                                                         int32_t write_scalars) {
  if (write_scalars && threadIdx.x == 0 && blockIdx.x == 0) *P.step = h;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P.count; j += gridDim.x * blockDim.x) {
    P.status[j] = 0u;
    P.maxabs[j] = 0.0f;
  }
  if (blockIdx.x == 0 && threadIdx.x < 4) P.abort_flag[threadIdx.x] = 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) *P.grad_flag = 0.0;
}
}  // namespace lopt

using namespace lopt;

namespace {

// strict-mode item sizes; LOPT_STRICT_CHUNKS="stat,apply" overrides them for
// tuning sweeps
int64_t strict_chunk(int which) {
  static int64_t v[2] = {0, 0};
  if (v[0] == 0) {
    v[0] = 8192;
    v[1] = 65536;   // 65536: -2 % vs 4096 (fewer per-item MLP smem fills)
    if (const char *e = getenv("LOPT_STRICT_CHUNKS")) {
      long long a = 0, b = 0;
      if (sscanf(e, "%lld,%lld", &a, &b) == 2 && a >= 256 && b >= 512) {
        v[0] = a;
        v[1] = b;
      }
    }
  }
  return v[which];
}
// elements per factor CTA (rows x <=512 columns); LOPT_FACTOR_TILE overrides
// it for tuning sweeps
int64_t factor_tile_elems() {
  static const int64_t v = [] {
    const char *e = getenv("LOPT_FACTOR_TILE");
    const long long x = e ? atoll(e) : 0;
    return x >= 512 ? (int64_t)x : (int64_t)131072;
  }();
  return v;
}

struct Region {
  size_t off = 0, bytes = 0;
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

struct lopt_plan {
  lopt_config cfg{};
  std::vector<lopt_tensor> tensors;
  std::vector<TensorDesc> descs;
  std::vector<FactorItem> fitems;
  std::vector<ChunkItem> sitems, aitems;
  int64_t max_mn = 0;        // max over tensors of m + n
  int64_t factor_sums = 0;   // f64 entries of the all-reducible factor block
  int64_t n_tiles = 0;       // fast path: 128-element tiles
  int64_t n_pairs = 0;       // fast path: tile pairs (pair kernel)
  // workspace regions
  Region r_desc, r_fitems, r_sitems, r_aitems, r_tscal, r_step, r_status, r_maxabs, r_imaxabs,
      r_abort, r_fsums, r_rowpart, r_colpart, r_rowtab, r_coltab, r_statpart, r_sumsq, r_weights,
      r_prep, r_bcsum, r_prefix, r_range, r_perf;
  std::vector<int64_t> prefixes;   // red_prefix (count + 1) then fin_prefix (count + 1)
  size_t ws_bytes = 0;
  char *ws = nullptr;
  DevicePlan dp{};
  int launches_last_step = 0;
  bool begun = false;        // lopt_set_step_args ran: the step's clears are done
  // VeLO hypernetwork registered with lopt_set_velo: run between phases 1 and 2
  bool velo = false;
  const float *v_hyper = nullptr, *v_bank = nullptr, *v_loss = nullptr;
  float *v_lstm = nullptr, *v_mix = nullptr;
  int v_H = 0, v_K = 0;
  // captured step (lopt_graph_step)
  cudaStream_t cap_stream = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaGraphNode_t gbegin = nullptr;
  // benchmark phase timing (lopt_set_phase_timing): `ev_slots` sets of five
  // plan-owned events, one set per step in turn; a graph captured with timing
  // holds event-record nodes re-pointed to the step's set before each launch
  std::vector<cudaEvent_t> phase_ev;   // [ev_slots x 5]
  int ev_slots = 0;
  int64_t ev_step = 0;                 // steps recorded so far
  cudaGraphNode_t ev_node[5] = {};
  bool graph_ev = false;
  // layer 3 of a single-weight-set plan, kept on the host for the pair
  // kernel's launch parameter (DevicePlan::w3c); a plan whose weights were
  // exposed through lopt_weights_ptr (device-side writes) reads them from the
  // operand images instead
  float w3c[16][4] = {};
  bool w3_known = false, w3_exposed = false;
  void drop_events() {
    for (cudaEvent_t e : phase_ev) cudaEventDestroy(e);
    phase_ev.clear();
    ev_slots = 0;
  }
  void drop_graph() {
    if (gexec) cudaGraphExecDestroy(gexec);
    if (graph) cudaGraphDestroy(graph);
    gexec = nullptr;
    graph = nullptr;
    gbegin = nullptr;
    graph_ev = false;
  }
  ~lopt_plan() {
    drop_graph();
    drop_events();
    if (cap_stream) cudaStreamDestroy(cap_stream);
  }
};

static int check_cuda_at(cudaError_t e, int line) {
  if (e != cudaSuccess) {
    fprintf(stderr, "lopt_b200: CUDA error %s (lopt_capi.cu:%d)\n", cudaGetErrorString(e), line);
    return LOPT_ERR_CUDA;
  }
  return LOPT_OK;
}
#define check_cuda(e) check_cuda_at((e), __LINE__)

static int check_launch() { return check_cuda(cudaGetLastError()); }

// Fast stats items: the largest chunk (fewest items: each costs a block
// reduction and a partial-sum write) among 8-32 K elements (32-128 rows of a
// 256-column strip) whose items are >= 97 % full (rows divide evenly) and
// still fill >= 6 waves of the stats grid (LOPT_STAT_MINB CTAs x SMs).
// Same-box ncu sweep on ViT-B/16: 8 K 352 us, 12 K 341, 16 K 337, 20 K 344
// (partial items), 24 K 330 (the pick), 32 K 343 (4.6 waves).
static int64_t pick_stat_chunk(const lopt_tensor *tensors, int32_t count) {
  if (getenv("LOPT_STAT_CHUNK_FIXED")) return fast_stat_chunk();
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
    sms = 148;
  cudaGetLastError();   // no device (CPU tests): not an error here
  const int64_t slots = (int64_t)sms * fast_stat_min_blocks();
  const int64_t strip_w = fast_stat_strip();
  int64_t best = fast_stat_chunk();
  for (int64_t c = 8192; c <= 32768; c += 4096) {
    int64_t items = 0, elems = 0;
    auto flat = [&](int64_t e0, int64_t e1) {
      if (e1 > e0) {
        items += (e1 - e0 + c - 1) / c;
        elems += e1 - e0;
      }
    };
    for (int j = 0; j < count; j++) {
      const lopt_tensor &t = tensors[j];
      if (t.n % strip_w == 0 && t.hi > t.lo) {
        const int64_t a0 = (t.lo + t.n - 1) / t.n, a1 = t.hi / t.n;
        if (a1 > a0) {
          flat(t.lo, a0 * t.n);
          const int64_t rows = std::max<int64_t>(1, c / strip_w);
          items += (t.n / strip_w) * ((a1 - a0 + rows - 1) / rows);
          elems += (a1 - a0) * t.n;
          flat(a1 * t.n, t.hi);
        } else {
          flat(t.lo, t.hi);
        }
      } else {
        flat(t.lo, t.hi);
      }
    }
    if (items == 0) continue;
    const double fill = (double)elems / ((double)items * (double)c);
    if (fill >= 0.97 && items >= 6 * slots) best = c;
  }
  return best;
}

extern "C" {

const char *lopt_version(void) { return "lopt_b200 0.1 (sm_100a)"; }

int lopt_plan_create(const lopt_tensor *tensors, int32_t count, const lopt_config *cfg,
                     lopt_plan **out) {
  if (!tensors || !cfg || !out || count < 1) return LOPT_ERR_INVALID;
  if (cfg->feature_set != LOPT_SMALL_FC_LOPT && cfg->feature_set != LOPT_VELO_MLP)
    return LOPT_ERR_INVALID;
  if (cfg->mode != LOPT_MODE_STRICT && cfg->mode != LOPT_MODE_FAST) return LOPT_ERR_INVALID;
  if (cfg->hidden1 != kMaxHidden || cfg->hidden2 != kMaxHidden) return LOPT_ERR_UNSUPPORTED;
  if (cfg->num_weight_sets < 1) return LOPT_ERR_INVALID;
  if (cfg->update_sign != 1 && cfg->update_sign != -1) return LOPT_ERR_INVALID;
  for (int k = 0; k < 7; k++)
    if (!(cfg->betas[k] >= 0.0 && cfg->betas[k] <= 1.0)) return LOPT_ERR_INVALID;
  for (int j = 0; j < count; j++) {
    const lopt_tensor &t = tensors[j];
    // engine.py:583-594: empty tensors are an EngineError
    if (t.m < 1 || t.n < 1) return LOPT_ERR_SHAPE;
    if (t.lo < 0 || t.hi < t.lo || t.hi > t.m * t.n) return LOPT_ERR_SHAPE;
    if (t.n > (int64_t)1 << 31 || t.m > (int64_t)1 << 40) return LOPT_ERR_SHAPE;
    // the tensor-core kernel indexes elements with 32-bit integers
    if (cfg->mode == LOPT_MODE_FAST && t.m * t.n >= ((int64_t)1 << 31)) return LOPT_ERR_UNSUPPORTED;
    if (!t.theta || !t.grad || !t.row_factors || !t.col_factors) return LOPT_ERR_INVALID;
    if (t.hi > t.lo && !t.state) return LOPT_ERR_INVALID;
    if ((reinterpret_cast<uintptr_t>(t.state) & 15) != 0) return LOPT_ERR_INVALID;
    if (t.weight_slot < 0 || t.weight_slot >= cfg->num_weight_sets) return LOPT_ERR_INVALID;
  }
  lopt_plan *p = new (std::nothrow) lopt_plan();
  if (!p) return LOPT_ERR_INVALID;
  p->cfg = *cfg;
  p->tensors.assign(tensors, tensors + count);
  p->descs.resize(count);
  const int D = d_feat(cfg->feature_set);
  const bool fast = cfg->mode == LOPT_MODE_FAST;
  const int64_t stat_chunk = fast ? pick_stat_chunk(tensors, count) : strict_chunk(0);
  const int64_t apply_chunk = fast ? fast_apply_chunk() : strict_chunk(1);
  const int64_t ftile = factor_tile_elems();
  int64_t rowpart = 0, colpart = 0, rows = 0, cols = 0;
  for (int j = 0; j < count; j++) {
    const lopt_tensor &t = tensors[j];
    TensorDesc &d = p->descs[j];
    memset(&d, 0, sizeof(d));
    d.m = t.m;
    d.n = t.n;
    d.lo = t.lo;
    d.hi = t.hi;
    d.weight_slot = t.weight_slot;
    p->max_mn = std::max<int64_t>(p->max_mn, t.m + t.n);
    if (!cfg->state_advanced) {
      if (t.n == 1) {
        d.nstrips = 1;
        d.nrowblocks = (int32_t)((t.m + ftile - 1) / ftile);
        for (int rb = 0; rb < d.nrowblocks; rb++) {
          // row blocks outside this call's element range keep zero partials
          const int64_t r0 = rb * ftile, r1 = std::min<int64_t>(t.m, r0 + ftile);
          if (r1 <= t.lo || r0 >= t.hi) continue;
          FactorItem it{};
          it.tensor = j;
          it.strip = 0;
          it.rowblock = rb;
          it.a0 = rb * ftile;
          it.a1 = std::min<int64_t>(t.m, it.a0 + ftile);
          it.b0 = 0;
          it.b1 = 1;
          p->fitems.push_back(it);
        }
      } else {
        const int64_t strip = factor_strip_cols();
        d.nstrips = (int32_t)((t.n + strip - 1) / strip);
        const int64_t width = std::min<int64_t>(t.n, strip);
        int64_t R = ftile / width;
        R = std::max<int64_t>(8, (R + 7) / 8 * 8);
        d.nrowblocks = (int32_t)((t.m + R - 1) / R);
        for (int rb = 0; rb < d.nrowblocks; rb++)
          for (int s = 0; s < d.nstrips; s++) {
            const int64_t e0 = rb * R * t.n, e1 = std::min<int64_t>(t.m, (rb + 1) * R) * t.n;
            if (e1 <= t.lo || e0 >= t.hi) continue;
            FactorItem it{};
            it.tensor = j;
            it.strip = s;
            it.rowblock = rb;
            it.a0 = rb * R;
            it.a1 = std::min<int64_t>(t.m, it.a0 + R);
            it.b0 = s * strip;
            it.b1 = std::min<int64_t>(t.n, it.b0 + strip);
            p->fitems.push_back(it);
          }
      }
    }
    rowpart += (int64_t)d.nstrips * t.m;
    colpart += (int64_t)d.nrowblocks * t.n;
    rows += t.m;
    cols += t.n;
    d.stat_item0 = (int32_t)p->sitems.size();
    auto flat_items = [&](int64_t e0, int64_t e1) {
      for (int64_t e = e0; e < e1; e += stat_chunk)
        p->sitems.push_back(ChunkItem{j, 0, e, std::min<int64_t>(e1, e + stat_chunk)});
    };
    const int64_t strip_w = fast_stat_strip();
    if (fast && t.n % strip_w == 0 && t.hi > t.lo) {
      // full rows as column strips (stat_chunk / strip_w rows x strip_w columns),
      // a partial first / last row (element-range shards) as flat chunks
      const int64_t a0 = (t.lo + t.n - 1) / t.n, a1 = t.hi / t.n;
      if (a1 > a0) {
        flat_items(t.lo, a0 * t.n);
        const int64_t rows = std::max<int64_t>(1, stat_chunk / strip_w);
        for (int64_t b = 0; b < t.n; b += strip_w)
          for (int64_t a = a0; a < a1; a += rows)
            p->sitems.push_back(ChunkItem{j, 1, (a << 32) | b,
                                          (std::min<int64_t>(a1, a + rows) << 32) | (b + strip_w)});
        flat_items(a1 * t.n, t.hi);
      } else {
        flat_items(t.lo, t.hi);
      }
    } else {
      flat_items(t.lo, t.hi);
    }
    d.stat_items = (int32_t)p->sitems.size() - d.stat_item0;
    d.apply_item0 = (int32_t)p->aitems.size();
    d.tile0 = p->n_tiles;
    if (fast) {
      // the persistent tensor-core kernel walks 128-lane tiles implicitly
      int64_t tiles = 0;
      if (t.hi > t.lo && t.n % apply_chunk == 0) {
        d.rowblock = 1;
        d.a_lo = (int32_t)(t.lo / t.n);
        d.m_rows = (int32_t)((t.hi - 1) / t.n - t.lo / t.n + 1);
        tiles = (int64_t)d.m_rows * (t.n / apply_chunk);
      } else {
        tiles = (t.hi - t.lo + apply_chunk - 1) / apply_chunk;
      }
      d.tiles = (int32_t)tiles;
      p->n_tiles += tiles;
      d.pair0 = p->n_pairs;
      d.pairs = (int32_t)(d.rowblock ? (int64_t)((d.m_rows + 1) / 2) * (t.n / apply_chunk)
                                     : (tiles + 1) / 2);
      p->n_pairs += d.pairs;
    } else {
      for (int64_t e = t.lo; e < t.hi; e += apply_chunk)
        p->aitems.push_back(ChunkItem{j, 0, e, std::min<int64_t>(t.hi, e + apply_chunk)});
    }
    d.apply_items = (int32_t)p->aitems.size() - d.apply_item0;
  }
  p->factor_sums = rows + cols + 1;   // + the non-finite-gradient flag slot
  // workspace layout
  size_t off = 0;
  // largest factor items first: the hardware dispatches CTAs in index order,
  // so the small items (remainders, vectors) backfill the last wave.  Each
  // item writes its own partial slots: the order does not change results.
  std::stable_sort(p->fitems.begin(), p->fitems.end(), [](const FactorItem &x, const FactorItem &y) {
    return (x.a1 - x.a0) * (x.b1 - x.b0) > (y.a1 - y.a0) * (y.b1 - y.b0);
  });
  auto take = [&](Region &r, size_t bytes) {
    off = align_up(off, 256);
    r.off = off;
    r.bytes = bytes;
    off += bytes;
  };
  const int wstride = weight_stride(D, cfg->hidden1, cfg->hidden2);
  take(p->r_desc, sizeof(TensorDesc) * count);
  take(p->r_fitems, sizeof(FactorItem) * std::max<size_t>(1, p->fitems.size()));
  take(p->r_sitems, sizeof(ChunkItem) * std::max<size_t>(1, p->sitems.size()));
  take(p->r_aitems, sizeof(ChunkItem) * std::max<size_t>(1, p->aitems.size()));
  take(p->r_tscal, sizeof(TensorScalars) * count);
  take(p->r_step, sizeof(StepScalars));
  take(p->r_status, sizeof(uint32_t) * count);
  take(p->r_maxabs, sizeof(float) * count);
  take(p->r_imaxabs, sizeof(float) * std::max<size_t>(1, p->aitems.size()));
  take(p->r_abort, sizeof(uint32_t) * 4);
  take(p->r_range, sizeof(int32_t) * (kMaxApplyCtas + 1));
  take(p->r_perf, sizeof(int64_t) * 3 * kMaxApplyCtas);   // {pairs, ns} + smoothed speed
  take(p->r_fsums, sizeof(double) * (size_t)p->factor_sums);
  take(p->r_rowpart, sizeof(double) * (size_t)std::max<int64_t>(1, rowpart));
  take(p->r_colpart, sizeof(double) * (size_t)std::max<int64_t>(1, colpart));
  take(p->r_rowtab, sizeof(float) * kRowTab * (size_t)rows);
  take(p->r_coltab, sizeof(float) * kRowTab * (size_t)cols);
  take(p->r_statpart, sizeof(double) * D * std::max<size_t>(1, p->sitems.size()));
  take(p->r_sumsq, sizeof(double) * D * count);
  take(p->r_weights, sizeof(float) * (size_t)wstride * cfg->num_weight_sets);
  take(p->r_prep, fast ? prep_image_bytes() * count : 16);
  take(p->r_bcsum, sizeof(double) * D * count);   // closed-form broadcast sums (both modes)
  p->prefixes.assign(2 * (size_t)(count + 1), 0);
  for (int j = 0; j < count; j++) {
    const lopt_tensor &t = tensors[j];
    // columns with many row blocks get a warp each, the others a thread
    const bool wide = p->descs[j].nrowblocks > kWarpColumnBlocks;
    p->prefixes[j + 1] = p->prefixes[j] + (t.m + 31) / 32 * 32 + (wide ? 32 * t.n : (t.n + 31) / 32 * 32);
    p->prefixes[count + 1 + j + 1] = p->prefixes[count + 1 + j] + t.m + t.n;
  }
  take(p->r_prefix, sizeof(int64_t) * p->prefixes.size());
  p->ws_bytes = align_up(off, 256);
  // device plan (pointers filled at bind time)
  DevicePlan &P = p->dp;
  P.count = count;
  P.n_factor_items = (int32_t)p->fitems.size();
  P.n_stat_items = (int32_t)p->sitems.size();
  P.n_apply_items = (int32_t)p->aitems.size();
  P.kind = cfg->feature_set;
  P.mode = cfg->mode;
  P.h1 = cfg->hidden1;
  P.h2 = cfg->hidden2;
  P.weight_stride = wstride;
  P.state_advanced = cfg->state_advanced;
  for (int k = 0; k < 7; k++) P.beta[k] = (float)cfg->betas[k];
  P.alpha = cfg->alpha;
  P.beta_out = cfg->beta_out;
  P.n_tiles = p->n_tiles;
  P.red_total = p->prefixes[count];
  P.fin_total = p->prefixes[2 * (size_t)count + 1];
  P.n_pairs = p->n_pairs;
  {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
      sms = 148;
    cudaGetLastError();
    P.apply_grid = (int32_t)std::min<int64_t>(std::min(sms, kMaxApplyCtas), p->n_pairs);
  }
  if (fast && !fast_supported(P)) {
    delete p;
    return LOPT_ERR_UNSUPPORTED;
  }
  *out = p;
  return LOPT_OK;
}

int lopt_plan_destroy(lopt_plan *plan) {
  delete plan;
  return LOPT_OK;
}

int lopt_workspace_bytes(const lopt_plan *plan, size_t *bytes) {
  if (!plan || !bytes) return LOPT_ERR_INVALID;
  *bytes = plan->ws_bytes;
  return LOPT_OK;
}

int lopt_bind_workspace(lopt_plan *p, void *dev_ptr, size_t bytes, void *stream) {
  if (!p || !dev_ptr) return LOPT_ERR_INVALID;
  if (bytes < p->ws_bytes) return LOPT_ERR_WORKSPACE;
  if ((reinterpret_cast<uintptr_t>(dev_ptr) & 255) != 0) return LOPT_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  p->ws = (char *)dev_ptr;
  char *ws = p->ws;
  const int D = d_feat(p->cfg.feature_set);
  int64_t rowoff = 0, coloff = 0, rpoff = 0, cpoff = 0;
  double *fsums = (double *)(ws + p->r_fsums.off);
  int64_t fsoff = 0;
  for (size_t j = 0; j < p->descs.size(); j++) {
    TensorDesc &d = p->descs[j];
    const lopt_tensor &t = p->tensors[j];
    d.theta = t.theta;
    d.grad = t.grad;
    d.state = reinterpret_cast<float4 *>(t.state);
    d.r = t.row_factors;
    d.c = t.col_factors;
    d.rowsum = fsums + fsoff;
    d.colsum = fsums + fsoff + t.m;
    fsoff += t.m + t.n;
    d.rowpart = (double *)(ws + p->r_rowpart.off) + rpoff;
    d.colpart = (double *)(ws + p->r_colpart.off) + cpoff;
    rpoff += (int64_t)d.nstrips * t.m;
    cpoff += (int64_t)d.nrowblocks * t.n;
    d.rowtab = (float *)(ws + p->r_rowtab.off) + rowoff * kRowTab;
    d.coltab = (float *)(ws + p->r_coltab.off) + coloff * kRowTab;
    rowoff += t.m;
    coloff += t.n;
    d.sumsq = (double *)(ws + p->r_sumsq.off) + (int64_t)j * D;
  }
  DevicePlan &P = p->dp;
  P.tensors = (TensorDesc *)(ws + p->r_desc.off);
  P.factor_items = (FactorItem *)(ws + p->r_fitems.off);
  P.stat_items = (ChunkItem *)(ws + p->r_sitems.off);
  P.apply_items = (ChunkItem *)(ws + p->r_aitems.off);
  P.stat_part = (double *)(ws + p->r_statpart.off);
  P.tscal = (TensorScalars *)(ws + p->r_tscal.off);
  P.step = (StepScalars *)(ws + p->r_step.off);
  P.weights = (const float *)(ws + p->r_weights.off);
  P.status = (uint32_t *)(ws + p->r_status.off);
  P.maxabs = (float *)(ws + p->r_maxabs.off);
  P.item_maxabs = (float *)(ws + p->r_imaxabs.off);
  P.abort_flag = (uint32_t *)(ws + p->r_abort.off);
  P.pair_range = (int32_t *)(ws + p->r_range.off);
  P.cta_perf = (int64_t *)(ws + p->r_perf.off);
  P.grad_flag = fsums + (p->factor_sums - 1);
  const bool fast = p->cfg.mode == LOPT_MODE_FAST;
  P.prep = fast ? (unsigned char *)(ws + p->r_prep.off) : nullptr;
  P.bcsum = (double *)(ws + p->r_bcsum.off);
  P.red_prefix = (const int64_t *)(ws + p->r_prefix.off);
  P.fin_prefix = P.red_prefix + p->descs.size() + 1;
  int st;
  if ((st = check_cuda(cudaMemcpyAsync(ws + p->r_prefix.off, p->prefixes.data(),
                                       sizeof(int64_t) * p->prefixes.size(),
                                       cudaMemcpyHostToDevice, s))))
    return st;
  if ((st = check_cuda(cudaMemsetAsync(ws + p->r_bcsum.off, 0, p->r_bcsum.bytes, s)))) return st;
  // no launch measured yet: prep splits the pairs evenly
  if ((st = check_cuda(cudaMemsetAsync(ws + p->r_perf.off, 0, p->r_perf.bytes, s)))) return st;
  // descriptor uploads: pageable source, so the copies complete before return
  if ((st = check_cuda(cudaMemcpyAsync(P.tensors, p->descs.data(),
                                       sizeof(TensorDesc) * p->descs.size(),
                                       cudaMemcpyHostToDevice, s))))
    return st;
  if (!p->fitems.empty() &&
      (st = check_cuda(cudaMemcpyAsync(P.factor_items, p->fitems.data(),
                                       sizeof(FactorItem) * p->fitems.size(),
                                       cudaMemcpyHostToDevice, s))))
    return st;
  if (!p->sitems.empty() &&
      (st = check_cuda(cudaMemcpyAsync(P.stat_items, p->sitems.data(),
                                       sizeof(ChunkItem) * p->sitems.size(),
                                       cudaMemcpyHostToDevice, s))))
    return st;
  if (!p->aitems.empty() &&
      (st = check_cuda(cudaMemcpyAsync(P.apply_items, p->aitems.data(),
                                       sizeof(ChunkItem) * p->aitems.size(),
                                       cudaMemcpyHostToDevice, s))))
    return st;
  if ((st = check_cuda(cudaMemsetAsync(ws + p->r_rowpart.off, 0, p->r_rowpart.bytes, s))))
    return st;
  if ((st = check_cuda(cudaMemsetAsync(ws + p->r_colpart.off, 0, p->r_colpart.bytes, s))))
    return st;
  return check_cuda(cudaMemsetAsync(ws + p->r_status.off, 0, p->r_status.bytes, s));
}

int lopt_rebind_tensors(lopt_plan *p, const lopt_tensor *tensors, int32_t count, void *stream) {
  if (!p || !p->ws || !tensors || count != (int32_t)p->tensors.size()) return LOPT_ERR_INVALID;
  for (int j = 0; j < count; j++) {
    const lopt_tensor &a = tensors[j], &b = p->tensors[j];
    if (a.m != b.m || a.n != b.n || a.lo != b.lo || a.hi != b.hi) return LOPT_ERR_SHAPE;
    if (!a.theta || !a.grad || !a.row_factors || !a.col_factors) return LOPT_ERR_INVALID;
    if (a.hi > a.lo && (!a.state || (reinterpret_cast<uintptr_t>(a.state) & 15) != 0))
      return LOPT_ERR_INVALID;
  }
  for (int j = 0; j < count; j++) {
    p->tensors[j] = tensors[j];
    TensorDesc &d = p->descs[j];
    d.theta = tensors[j].theta;
    d.grad = tensors[j].grad;
    d.state = reinterpret_cast<float4 *>(tensors[j].state);
    d.r = tensors[j].row_factors;
    d.c = tensors[j].col_factors;
  }
  return check_cuda(cudaMemcpyAsync(p->dp.tensors, p->descs.data(),
                                    sizeof(TensorDesc) * p->descs.size(), cudaMemcpyHostToDevice,
                                    (cudaStream_t)stream));
}

int lopt_set_stat_counts(lopt_plan *p, const int64_t *counts, void *stream) {
  if (!p || !p->ws) return LOPT_ERR_INVALID;
  for (size_t j = 0; j < p->descs.size(); j++) {
    if (counts && counts[j] < 0) return LOPT_ERR_INVALID;
  }
  for (size_t j = 0; j < p->descs.size(); j++) p->descs[j].stat_count = counts ? counts[j] : 0;
  return check_cuda(cudaMemcpyAsync(p->dp.tensors, p->descs.data(),
                                    sizeof(TensorDesc) * p->descs.size(), cudaMemcpyHostToDevice,
                                    (cudaStream_t)stream));
}

int lopt_set_weights(lopt_plan *p, int32_t slot, const float *packed, int32_t is_device,
                     void *stream) {
  if (!p || !p->ws || !packed) return LOPT_ERR_INVALID;
  if (slot < 0 || slot >= p->cfg.num_weight_sets) return LOPT_ERR_INVALID;
  const size_t bytes = sizeof(float) * p->dp.weight_stride;
  float *dst = (float *)(p->ws + p->r_weights.off) + (int64_t)slot * p->dp.weight_stride;
  cudaStream_t s = (cudaStream_t)stream;
  int st;
  if ((st = check_cuda(cudaMemcpyAsync(dst, packed, bytes,
                                       is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                       s))))
    return st;
  if (p->cfg.num_weight_sets == 1 && p->cfg.mode == LOPT_MODE_FAST) {
    // w3 (2 x 32 after W1, b1, W2, b2) as the launch parameter, halved
    const int64_t off = 32 * (int64_t)d_feat(p->cfg.feature_set) + 32 + 32 * 32 + 32;
    float w3[64];
    if (is_device) {
      if ((st = check_cuda(cudaMemcpyAsync(w3, packed + off, sizeof(w3), cudaMemcpyDeviceToHost, s))) ||
          (st = check_cuda(cudaStreamSynchronize(s))))
        return st;
    } else {
      memcpy(w3, packed + off, sizeof(w3));
    }
    float c[16][4];
    for (int out = 0; out < 2; out++)
      for (int o = 0; o < 32; o++) c[o >> 1][2 * (o & 1) + out] = w3[out * 32 + o] * 0.5f;
    if (!p->w3_known || memcmp(c, p->w3c, sizeof(c)) != 0) {
      memcpy(p->w3c, c, sizeof(c));
      p->w3_known = true;
      p->drop_graph();   // the captured apply launch holds the old parameter
    }
  }
  return LOPT_OK;
}

int lopt_weights_ptr(lopt_plan *p, int32_t slot, float **dev_ptr) {
  if (!p || !p->ws || !dev_ptr || slot < 0 || slot >= p->cfg.num_weight_sets)
    return LOPT_ERR_INVALID;
  if (!p->w3_exposed) {
    p->w3_exposed = true;   // device-side writes: layer 3 from the operand images
    p->drop_graph();
  }
  *dev_ptr = (float *)(p->ws + p->r_weights.off) + (int64_t)slot * p->dp.weight_stride;
  return LOPT_OK;
}

static StepScalars make_scalars(const lopt_plan *p, const lopt_step_args *a) {
  StepScalars h{};
  for (int k = 0; k < kTimeFeatures; k++) h.tf[k] = a->time_features[k];
  h.lr_f32 = (float)a->lr;
  h.ds = (float)p->cfg.update_sign * (float)a->lr;             // engine.py:695
  h.decay = (float)(1.0 - a->lr * a->weight_decay);             // optim.py:100
  h.apply_decay = a->weight_decay > 0.0 ? 1 : 0;                // optim.py:171
  h.t = a->t;
  h.loss[0] = a->loss_features[0];
  h.loss[1] = a->loss_features[1];
  return h;
}

static int begin_blocks(const lopt_plan *p) {
  return (int)std::min<int64_t>(64, ((int64_t)p->tensors.size() + 255) / 256);
}

int lopt_set_step_args(lopt_plan *p, const lopt_step_args *a, void *stream) {
  if (!p || !p->ws || !a) return LOPT_ERR_INVALID;
  if (!(a->weight_decay >= 0.0)) return LOPT_ERR_INVALID;
  const StepScalars h = make_scalars(p, a);
  begin_step_kernel<<<begin_blocks(p), 256, 0, (cudaStream_t)stream>>>(p->dp, h, 1);
  p->begun = true;
  p->launches_last_step = 1;
  return check_launch();
}

int lopt_factor_partials(lopt_plan *p, void *stream) {
  if (!p || !p->ws) return LOPT_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  if (!p->begun) {   // scalars from an earlier call: only the per-step clears
    begin_step_kernel<<<begin_blocks(p), 256, 0, s>>>(p->dp, StepScalars{}, 0);
    p->launches_last_step = 1;
  }
  p->begun = false;
  if (p->cfg.state_advanced) return check_launch();
  launch_factor_partials(p->dp, s);
  launch_factor_reduce(p->dp, p->max_mn, s);
  p->launches_last_step += 2;
  return check_launch();
}

int lopt_factor_finalize(lopt_plan *p, void *stream) {
  if (!p || !p->ws) return LOPT_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  launch_factor_finalize(p->dp, p->max_mn, s);
  launch_factor_means(p->dp, s);
  p->launches_last_step += 2;
  return check_launch();
}

int lopt_feature_stats(lopt_plan *p, void *stream) {
  if (!p || !p->ws) return LOPT_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  if (p->cfg.mode == LOPT_MODE_FAST) {
    launch_fast_stats(p->dp, s);
  } else {
    launch_strict_stats(p->dp, s);
    launch_stats_reduce(p->dp, s);
  }
  p->launches_last_step += (p->dp.n_stat_items > 0) + 1;
  return check_launch();
}

int lopt_apply(lopt_plan *p, void *stream) {
  if (!p || !p->ws) return LOPT_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  if (p->cfg.mode == LOPT_MODE_FAST) {
    DevicePlan P = p->dp;
    static const bool no_w3c = getenv("LOPT_NO_W3C") != nullptr;   // A/B switch
    P.w3c_on = !no_w3c && p->w3_known && !p->w3_exposed && !p->velo && p->cfg.num_weight_sets == 1;
    if (P.w3c_on) memcpy(P.w3c, p->w3c, sizeof(P.w3c));
    launch_fast_apply(P, s);   // prep + persistent tensor-core apply
    p->launches_last_step += 1 + (p->dp.n_tiles > 0);
  } else {
    launch_strict_apply(p->dp, s);
    launch_maxabs_reduce(p->dp, s);
    p->launches_last_step += (p->dp.n_apply_items > 0) + 1;
  }
  return check_launch();
}

static int run_velo(lopt_plan *p, cudaStream_t s) {
  const int st = launch_velo_mix(p->dp, p->v_hyper, p->v_lstm, p->v_bank, p->v_loss, p->v_H,
                                 p->v_K, p->v_mix, s);
  if (st == LOPT_OK) p->launches_last_step += 1;
  return st;
}

int lopt_set_phase_timing(lopt_plan *p, int32_t slots) {
  if (!p || slots < 0 || slots > 4096) return LOPT_ERR_INVALID;
  // a captured step with(out) event nodes no longer matches: recapture
  if (p->gexec && (slots > 0) != p->graph_ev) p->drop_graph();
  p->drop_events();
  for (int i = 0; i < 5 * slots; i++) {
    cudaEvent_t e = nullptr;
    int st;
    if ((st = check_cuda(cudaEventCreate(&e)))) {
      p->drop_events();
      return st;
    }
    p->phase_ev.push_back(e);
  }
  p->ev_slots = slots;
  p->ev_step = 0;
  return LOPT_OK;
}

int lopt_phase_slot(const lopt_plan *p, int32_t *next_slot) {
  if (!p || !next_slot || p->ev_slots == 0) return LOPT_ERR_INVALID;
  *next_slot = (int32_t)(p->ev_step % p->ev_slots);
  return LOPT_OK;
}

int lopt_phase_elapsed(lopt_plan *p, int32_t slot, int32_t k0, int32_t k1, float *ms) {
  if (!p || !ms || slot < 0 || slot >= p->ev_slots || k0 < 0 || k1 < 0 || k0 > 4 || k1 > 4)
    return LOPT_ERR_INVALID;
  return check_cuda(cudaEventElapsedTime(ms, p->phase_ev[5 * slot + k0], p->phase_ev[5 * slot + k1]));
}

int lopt_step(lopt_plan *p, const lopt_step_args *args, void *stream) {
  int st;
  if (!p) return LOPT_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  const bool tev = p->ev_slots > 0;
  const int slot = tev ? (int)(p->ev_step % p->ev_slots) : 0;
  bool capturing = false;
  if (tev) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if ((st = check_cuda(cudaStreamIsCapturing(s, &cs)))) return st;
    capturing = cs != cudaStreamCaptureStatusNone;
  }
  // inside a capture the records become event-record nodes (external events)
  auto mark = [&](int k) {
    if (!tev) return LOPT_OK;
    cudaEvent_t e = p->phase_ev[5 * slot + k];
    return check_cuda(capturing ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
                                : cudaEventRecord(e, s));
  };
  if (args && (st = lopt_set_step_args(p, args, stream))) return st;
  if ((st = mark(0))) return st;
  if (p->cfg.state_advanced) {
    if ((st = lopt_factor_partials(p, stream))) return st;
    if ((st = lopt_factor_finalize(p, stream))) return st;
  } else {
    // one device: no merge between the reduce and the finalize -- one kernel
    if (!p->begun) {
      begin_step_kernel<<<begin_blocks(p), 256, 0, s>>>(p->dp, StepScalars{}, 0);
      p->launches_last_step = 1;
    }
    p->begun = false;
    launch_factor_partials(p->dp, s);
    launch_factor_reduce_finalize(p->dp, s);
    launch_factor_means(p->dp, s);
    p->launches_last_step += 3;
    if ((st = check_launch())) return st;
  }
  if ((st = mark(1))) return st;
  if ((st = lopt_feature_stats(p, stream))) return st;
  if ((st = mark(2))) return st;
  if (p->velo && (st = run_velo(p, s))) return st;
  if ((st = mark(3))) return st;
  if ((st = lopt_apply(p, stream))) return st;
  if ((st = mark(4))) return st;
  if (tev && !capturing) p->ev_step++;
  return LOPT_OK;
}

int lopt_graph_step(lopt_plan *p, const lopt_step_args *args, void *stream) {
  if (!p || !p->ws || !args) return LOPT_ERR_INVALID;
  if (!(args->weight_decay >= 0.0)) return LOPT_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  StepScalars h = make_scalars(p, args);
  int st;
  if (!p->gexec) {
    // capture on a private stream (the caller's may be the legacy default
    // stream, which cannot be captured); the graph is launched on the caller's
    if (!p->cap_stream &&
        (st = check_cuda(cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking))))
      return st;
    // the capture stream starts after the caller's prior work (descriptor
    // uploads of bind/rebind) -- captured work itself is only enqueued later
    if ((st = check_cuda(cudaStreamSynchronize(s)))) return st;
    if ((st = check_cuda(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeRelaxed))))
      return st;
    int rc = lopt_set_step_args(p, args, p->cap_stream);
    if (rc == LOPT_OK) rc = lopt_step(p, nullptr, p->cap_stream);
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(p->cap_stream, &g);
    if (rc != LOPT_OK || ce != cudaSuccess) {
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      return rc != LOPT_OK ? rc : check_cuda(ce);
    }
    p->graph = g;
    if ((st = check_cuda(cudaGraphInstantiate(&p->gexec, g, 0)))) {
      p->drop_graph();
      return st;
    }
    // the step-scalar kernel is the graph's only root
    size_t nroot = 1;
    cudaGraphNode_t root = nullptr;
    if ((st = check_cuda(cudaGraphGetRootNodes(g, &root, &nroot))) || nroot != 1) {
      p->drop_graph();
      return st ? st : LOPT_ERR_CUDA;
    }
    p->gbegin = root;
    if (p->ev_slots > 0) {
      // map the captured event-record nodes to the phase marks
      size_t nn = 0;
      if ((st = check_cuda(cudaGraphGetNodes(g, nullptr, &nn)))) return st;
      std::vector<cudaGraphNode_t> nodes(nn);
      if ((st = check_cuda(cudaGraphGetNodes(g, nodes.data(), &nn)))) return st;
      int found = 0;
      for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType ty;
        if (cudaGraphNodeGetType(nd, &ty) != cudaSuccess || ty != cudaGraphNodeTypeEventRecord) continue;
        cudaEvent_t ev = nullptr;
        if (cudaGraphEventRecordNodeGetEvent(nd, &ev) != cudaSuccess) continue;
        const int cs = (int)(p->ev_step % p->ev_slots);
        for (int k = 0; k < 5; k++)
          if (ev == p->phase_ev[5 * cs + k]) {
            p->ev_node[k] = nd;
            found |= 1 << k;
          }
      }
      if (found != 31) {
        p->drop_graph();
        return LOPT_ERR_CUDA;
      }
      p->graph_ev = true;
    }
  }
  if (p->graph_ev) {
    const int slot = (int)(p->ev_step % p->ev_slots);
    for (int k = 0; k < 5; k++)
      if ((st = check_cuda(cudaGraphExecEventRecordNodeSetEvent(p->gexec, p->ev_node[k],
                                                                  p->phase_ev[5 * slot + k]))))
        return st;
    p->ev_step++;
  }
  cudaKernelNodeParams kp{};
  if ((st = check_cuda(cudaGraphKernelNodeGetParams(p->gbegin, &kp)))) return st;
  int32_t one = 1;
  void *kargs[3] = {&p->dp, &h, &one};
  kp.kernelParams = kargs;
  kp.extra = nullptr;
  if ((st = check_cuda(cudaGraphExecKernelNodeSetParams(p->gexec, p->gbegin, &kp)))) return st;
  return check_cuda(cudaGraphLaunch(p->gexec, s));
}

int lopt_graph_reset(lopt_plan *p) {
  if (!p) return LOPT_ERR_INVALID;
  p->drop_graph();
  return LOPT_OK;
}

int lopt_set_velo(lopt_plan *p, const float *hyper, float *lstm_state, const float *bank,
                  const float *loss_feats, int32_t hidden, int32_t bank_size, float *mix_out) {
  if (!p || !p->ws) return LOPT_ERR_INVALID;
  p->drop_graph();   // the captured step changes
  if (!hyper) {      // unregister
    p->velo = false;
    return LOPT_OK;
  }
  // loss_feats == NULL: the loss features come with the step scalars
  if (!lstm_state || !bank || hidden < 1 || hidden > 64 || bank_size < 1 ||
      bank_size > 16 || p->cfg.feature_set != LOPT_VELO_MLP)
    return LOPT_ERR_INVALID;
  if (p->cfg.num_weight_sets != (int32_t)p->tensors.size()) return LOPT_ERR_INVALID;
  for (size_t j = 0; j < p->tensors.size(); j++)
    if (p->tensors[j].weight_slot != (int32_t)j) return LOPT_ERR_INVALID;
  p->velo = true;
  p->w3_exposed = true;   // the hypernetwork writes the weights on the device
  p->v_hyper = hyper;
  p->v_lstm = lstm_state;
  p->v_bank = bank;
  p->v_loss = loss_feats;
  p->v_H = hidden;
  p->v_K = bank_size;
  p->v_mix = mix_out;
  return LOPT_OK;
}

int lopt_factor_sums_ptr(lopt_plan *p, double **ptr, int64_t *count) {
  if (!p || !p->ws || !ptr || !count) return LOPT_ERR_INVALID;
  *ptr = (double *)(p->ws + p->r_fsums.off);
  *count = p->factor_sums;
  return LOPT_OK;
}

int lopt_stat_sums_ptr(lopt_plan *p, double **ptr, int64_t *count) {
  if (!p || !p->ws || !ptr || !count) return LOPT_ERR_INVALID;
  *ptr = (double *)(p->ws + p->r_sumsq.off);
  *count = (int64_t)d_feat(p->cfg.feature_set) * (int64_t)p->tensors.size();
  return LOPT_OK;
}

int lopt_status_ptr(lopt_plan *p, uint32_t **status, float **maxabs) {
  if (!p || !p->ws || !status || !maxabs) return LOPT_ERR_INVALID;
  *status = p->dp.status;
  *maxabs = p->dp.maxabs;
  return LOPT_OK;
}

int lopt_read_status(lopt_plan *p, uint32_t *status_host, float *maxabs_host, void *stream) {
  if (!p || !p->ws) return LOPT_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  int st;
  const size_t n = p->tensors.size();
  if (status_host &&
      (st = check_cuda(cudaMemcpyAsync(status_host, p->dp.status, sizeof(uint32_t) * n,
                                       cudaMemcpyDeviceToHost, s))))
    return st;
  if (maxabs_host &&
      (st = check_cuda(cudaMemcpyAsync(maxabs_host, p->dp.maxabs, sizeof(float) * n,
                                       cudaMemcpyDeviceToHost, s))))
    return st;
  return check_cuda(cudaStreamSynchronize(s));
}

int lopt_debug_ptrs(lopt_plan *p, double **sumsq, float **factor_means) {
  if (!p || !p->ws) return LOPT_ERR_INVALID;
  if (sumsq) *sumsq = (double *)(p->ws + p->r_sumsq.off);
  if (factor_means) *factor_means = (float *)(p->ws + p->r_tscal.off);
  return LOPT_OK;
}

int lopt_velo_mix(lopt_plan *p, const float *hyper, float *lstm_state, const float *bank,
                  const float *loss_feats, int32_t hidden, int32_t bank_size, float *mix_out,
                  void *stream) {
  if (!p || !p->ws || !hyper || !lstm_state || !bank) return LOPT_ERR_INVALID;
  if (p->cfg.num_weight_sets != (int32_t)p->tensors.size()) return LOPT_ERR_INVALID;
  for (size_t j = 0; j < p->tensors.size(); j++)
    if (p->tensors[j].weight_slot != (int32_t)j) return LOPT_ERR_INVALID;
  if (!p->w3_exposed) {
    // the hypernetwork writes the plan's weights on the device: layer 3 from
    // the operand images from now on
    p->w3_exposed = true;
    p->drop_graph();
  }
  const int st = launch_velo_mix(p->dp, hyper, lstm_state, bank, loss_feats, hidden, bank_size,
                                 mix_out, (cudaStream_t)stream);
  if (st == LOPT_OK) p->launches_last_step += 1;
  return st;
}

int lopt_enable_peer_access(int32_t peer_device) {
  int cur = 0, can = 0;
  if (cudaGetDevice(&cur) != cudaSuccess) return LOPT_ERR_CUDA;
  if (peer_device == cur) return LOPT_OK;
  if (cudaDeviceCanAccessPeer(&can, cur, peer_device) != cudaSuccess || !can) return LOPT_ERR_UNSUPPORTED;
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();   // not an error here: clear it
    return LOPT_OK;
  }
  return check_cuda(e);
}

int lopt_set_peers(lopt_plan *p, int32_t count, const int64_t *deltas) {
  if (!p || count < 0 || count > LOPT_MAX_PEERS || (count > 0 && !deltas)) return LOPT_ERR_INVALID;
  if (count > 0 && p->cfg.mode != LOPT_MODE_FAST) return LOPT_ERR_UNSUPPORTED;
  p->dp.n_peers = count;
  for (int k = 0; k < LOPT_MAX_PEERS; k++) p->dp.peer_delta[k] = k < count ? deltas[k] : 0;
  p->dp.peer_bulk = 1;
  for (int k = 0; k < count; k++)
    if (deltas[k] % 16 != 0) p->dp.peer_bulk = 0;
  if (getenv("LOPT_PEER_SCALAR")) p->dp.peer_bulk = 0;   // A/B of the element-wise path
  p->drop_graph();   // the plan is captured by value
  return LOPT_OK;
}

int lopt_num_kernels_launched_last_step(const lopt_plan *p) {
  return p ? p->launches_last_step : 0;
}

}  // extern "C"
