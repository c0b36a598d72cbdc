// cs_api.cpp — host runtime behind include/cyclescope_b200.h.
//
// Owns device memory (grow-only buffers sized for whole instances resident in
// HBM), the ctx stream, and the orchestration of the kernels in
// cs_kernels.cu.  Rare control-flow paths of the reference (ordered-fold
// anchor tie break, wrong speculative anchor, NoAnchorFound -> frequency
// fallback) are driven from here; every per-event / per-cycle / per-record
// computation runs on the device.  There is no CPU fallback: without a device
// every compute entry point fails with CS_E_NO_DEVICE.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <new>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdint>
#include <limits>
#include <map>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "cs_internal.h"
#include "cs_guard.h"
#include "cyclescope_b200.h"

using namespace csb;

// an NVTX range for the rest of the enclosing scope
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
};
#define CS_NVTX_SCOPE(name) NvtxScope nvtx_scope_(name)

// CS_HOST_PROFILE=1: host-side phase times of each push on stderr (tools) and
// of each cs_run; =2 also records an event on `stream` at every mark and
// prints the device timeline (the events themselves cost device time)
struct HostPhases {
  const char* label;
  int on = 0;
  cudaStream_t stream = nullptr;
  std::chrono::steady_clock::time_point t0;
  std::string line;
  std::vector<std::pair<const char*, cudaEvent_t>> gpu;
  explicit HostPhases(const char* l) : label(l) {
    const char* e = std::getenv("CS_HOST_PROFILE");
    on = e && (*e == '1' || *e == '2') ? *e - '0' : 0;
    if (on) t0 = std::chrono::steady_clock::now();
  }
  void mark(const char* name) {
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    line += std::string(name) + "=" +
            std::to_string(std::chrono::duration<double, std::micro>(t - t0).count()) + " ";
    if (on == 2 && stream) {
      cudaEvent_t ev;
      cudaEventCreate(&ev);
      cudaEventRecord(ev, stream);
      gpu.push_back({name, ev});
    }
  }
  ~HostPhases() {
    if (!on) return;
    std::fprintf(stderr, "%s_us %s\n", label, line.c_str());
    if (gpu.empty()) return;
    cudaEventSynchronize(gpu.back().second);
    std::string g;
    for (auto& [n, ev] : gpu) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, gpu.front().second, ev);
      g += std::string(n) + "=" + std::to_string(ms * 1e3) + " ";
    }
    for (auto& [n, ev] : gpu) cudaEventDestroy(ev);
    std::fprintf(stderr, "%s_gpu_us %s\n", label, g.c_str());
  }
};


namespace {

// Pinned host memory for the small host mirrors a run copies to / from the
// device (instance states, offsets, stream carries): their copies then run
// asynchronously instead of being staged through pageable memory.
template <typename T>
struct PinnedAlloc {
  using value_type = T;
  PinnedAlloc() = default;
  template <typename U>
  PinnedAlloc(const PinnedAlloc<U>&) {}
  T* allocate(size_t n) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, std::max<size_t>(1, n) * sizeof(T), cudaHostAllocDefault) != cudaSuccess)
      throw std::bad_alloc();
    return static_cast<T*>(p);
  }
  void deallocate(T* p, size_t) { cudaFreeHost(p); }
  template <typename U>
  bool operator==(const PinnedAlloc<U>&) const { return true; }
  template <typename U>
  bool operator!=(const PinnedAlloc<U>&) const { return false; }
};
template <typename T>
using pinned_vector = std::vector<T, PinnedAlloc<T>>;

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  // a first allocation is exact; a buffer that has to grow again (streaming
  // batches of varying size) grows by half at least, so reallocations (and
  // the device synchronisation cudaFree implies) die out
  void* get(size_t bytes) {
    if (bytes > cap) {
      const size_t want = cap ? std::max(bytes, cap + cap / 2) : bytes;
      if (p) cudaFree(p);
      p = nullptr;
      cap = 0;
      if (bytes == 0) return nullptr;
      if (cudaMalloc(&p, want) != cudaSuccess) {
        if (want == bytes || cudaMalloc(&p, bytes) != cudaSuccess) {
          p = nullptr;
          return nullptr;
        }
        cap = bytes;
        return p;
      }
      cap = want;
    }
    return p;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

struct PackedModel {
  uint32_t n_trees = 0, depth = 0, n_features = 0, degenerate = 0;
  std::vector<int32_t> feature_ids;  // CS_F_* or CS_F_EXTRA (resolved by name per run)
  std::vector<std::string> feature_names;
  std::vector<double> thr, leaf;   // leaf holds fl(lr * value)
  std::vector<int64_t> thr_i;       // floor(thr) for exact integer compares
  std::vector<uint8_t> feat;
  double base = 0, lr = 0, floor_ = 0, mu = 0, sigma = 0;
  DevBuf d_thr, d_thr_i, d_leaf, d_feat;
  // compiled ensemble (<= 2 features): distinct thresholds per feature, node
  // ranks into them, and the per-cell prediction table built on the device
  bool has_lut = false;
  std::vector<double> lut_thr[2];
  DevBuf d_lut_thr[2], d_rank, d_lut;
};

}  // namespace

// cs_detect_residuals: a one-instance record table of its own
struct DetScratch {
  DevBuf resid, stat, flags, rec_off, rec_cycle, cyc_off, alert_rec, alert_off, block_tmp, inst,
      model, labels, out;
};

constexpr uint32_t kMaxBoundInstances = 1u << 24;  // model bindings per ctx

struct cs_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  cs_cycle_config cyc{};
  cs_control_config ctl{};
  bool have_config = false;
  std::vector<cs_name_info> names;
  // inputs
  uint32_t n_inst = 0;
  uint64_t n_ev = 0, n_wl = 0;
  pinned_vector<uint64_t> inst_off;
  DevBuf d_ev, d_wl, d_names;
  DevBuf d_wire;  // cs_upload_wire staging (all columns in one allocation)
  // tiles
  // pinned: the layout's host->device copies are asynchronous (streaming pushes)
  pinned_vector<uint32_t> tile_inst, inst_first_tile;
  pinned_vector<uint64_t> tile_begin, tile_end;
  // the layout (instance offsets, tiles, sample tiles) goes up as ONE copy
  // from a pinned staging block; the p_* pointers are its device segments
  pinned_vector<unsigned char> h_layout;
  DevBuf d_layout;
  cudaEvent_t ev_layout = nullptr;  // the staging block's last copy (reuse waits for it)
  uint64_t* p_inst_off = nullptr;
  uint64_t* p_tile_begin = nullptr;
  uint64_t* p_tile_end = nullptr;
  uint32_t* p_tile_inst = nullptr;
  uint32_t* p_inst_first_tile = nullptr;
  uint32_t* p_sample_tiles = nullptr;
  DevBuf d_tile_cnt, d_tile_pref;
  DevBuf d_scan_tmp;
  // record extras (cs_upload_extras)
  std::vector<std::string> extra_keys;
  uint64_t n_extra_refs = 0;
  DevBuf d_extra_refs, d_extra_vals, d_rec_extra, d_rec_extra_has;
  DevBuf d_stage2, d_stage_changed, d_stage_lb, d_stage_ctl;  // k_stage_jacobi
  DevBuf d_any_unknown;
  // counter-weighted mu: metric slots derived from the name table
  uint32_t n_metrics = 0;
  DevBuf d_series_slot, d_class_metric, d_m_off, d_s_ts, d_s_val, d_mu, d_mu_has;
  // cs_stream_push: the carried trailing partial cycle of every instance stays
  // in the previous batch's event buffer (d_ev_prev); per instance its start
  // and length there
  std::vector<uint64_t> tail_start, tail_len;
  bool tails_on_device = false;
  DevBuf d_ev_prev, d_new_ev, d_assemble;
  // K0 (cs_upload_unsorted): unsorted input, event ids, radix-sort scratch and
  // the canonical -> input position map of the last sorted upload
  DevBuf d_sort_in, d_sort_ids, d_sort_scratch, d_sort_hist, d_sort_hist_tmp, d_sort_ext, d_order;
  bool have_order = false;
  void* pin_models = nullptr;  // pinned staging of the per-instance DevModel array
  size_t pin_models_cap = 0;
  std::vector<uint64_t> stage_off;
  pinned_vector<uint64_t> assemble_host, h_new_anchors;
  DevBuf d_new_anchors;
  cudaEvent_t ev_counted = nullptr;  // the new events' anchor counts are on the host
  DevBuf d_keep;
  pinned_vector<uint32_t> sample_tiles;
  DevBuf d_redo_tiles;
  // state
  DevBuf d_stats, d_inst, d_a_pos, d_a_start, d_a_end;
  pinned_vector<InstState> h_inst;
  // cycles
  pinned_vector<uint64_t> cyc_off;   // cycle-slot base per instance (+ total)
  std::vector<uint64_t> n_cyc;     // cycles per instance
  uint64_t n_cycles = 0;           // cycle slots
  int reduce_variant = 0;  // profiling hook (single variant today)
  bool allow_fused = true;   // CS_OPT_FUSED (default on; 0 selects the two-pass path)
  bool no_fused_score = false;  // option 95 (testing): score in its own kernel after compaction
  int phase_timings = -1;    // CS_OPT_PHASE_TIMINGS (-1: per phase except streaming pushes)
  bool used_fused = false;   // the last run segmented with k_segment_range
  // slot-count speculation of the single-read pass: a run over the same
  // upload and configuration as the last verified one takes its per-instance
  // slot counts as the sizing, skips the mid-run synchronisation and checks
  // them (with every other fallback condition) at the final one; a mismatch
  // re-runs without speculation
  uint64_t seg_gen = 1;               // bumped by uploads and configuration changes
  bool no_speculate = false;          // the re-run after a failed speculation
  uint64_t pred_gen = 0;              // seg_gen of the verified counts below
  uint32_t pred_beta = 0;             // CS_RUN_BETA of that run
  std::vector<uint64_t> pred_cyc_off;
  // the anchors the last completed run over this upload and configuration
  // verified: the next run speculates on them instead of sampling (the full
  // moments still rank every candidate and check the guess)
  uint64_t anchor_gen = 0;
  std::vector<uint32_t> pred_anchor;
  unsigned int* pin_ctl = nullptr;    // pinned: the pass's control words at the final sync
  // cs_set_cycles: caller-given cycles of instance 0 (CS_RUN_GIVEN)
  std::vector<cs_cycle> given;
  std::vector<int64_t> given_comp;   // n x n_phases, empty = recompute
  bool given_run = false;            // the last run used them (indices map through `given`)
  DetScratch det;                    // cs_detect_residuals
  uint64_t slot_cap = 0;     // cycle-slot capacity of the fused pass (grows to the last count)
  // k_segment_range ranges (<= range_events events of one instance), built by
  // the first fused run after an upload for the range size in force
  uint64_t ranges_built_for = 0;
  int64_t opt_range_events = 0;   // 0: ~kSegCycles cycles per range from the last run's density
  int64_t opt_prefetch = 0;       // L2 prefetch lookahead in ranges (0: the claimed range only; -1: the grid's warp count)
  double ev_per_cycle = 0.0;      // events per cycle slot of the last run
  std::vector<uint64_t> range_begin, range_end;
  std::vector<uint32_t> range_inst, inst_first_range;
  DevBuf d_range_begin, d_range_end, d_range_inst, d_inst_first_range, d_lb_state, d_range_prefix,
      d_seg_ctl;
  bool no_lut = false;       // CS_OPT_TRAVERSAL: score by tree traversal even with a cell table
  DevBuf d_cyc_off, c_start, c_end, c_apos, c_aend, c_first, c_last, c_inst, c_stage, c_local,
      c_wl, c_comp, c_beta_tot, c_coll, c_coll_n;
  // records
  DevBuf d_rec_off, rec_cycle, rec_pred, rec_resid, rec_stat, rec_flags, alert_rec, d_alert_off,
      block_tmp;
  pinned_vector<uint64_t> rec_off, alert_off;
  uint64_t n_records = 0;
  // models
  std::vector<PackedModel*> model_store;
  std::vector<int> model_of_inst;  // per instance index; -1: use default_model
  int default_model = -1;          // cs_load_model(ctx, UINT32_MAX, ...)
  int model_id(uint32_t i) const {
    const int id = i < model_of_inst.size() ? model_of_inst[i] : -1;
    return id >= 0 ? id : default_model;
  }
  DevBuf d_models;
  std::vector<DevModel> h_models;
  // the per-instance model table on the device is rebuilt only when what it
  // is made of changes: the instance -> model binding, a model load (model_gen)
  // or the control config (cs_redetect also invalidates it)
  uint64_t model_gen = 0;
  bool mt_valid = false;
  uint64_t mt_gen = 0;
  uint32_t mt_n_inst = 0;
  cs_control_config mt_ctl{};
  std::vector<int> mt_ids;
  // fold results per instance: name -> (mean, cv, score)
  std::vector<std::map<uint32_t, std::array<double, 4>>> folded;
  std::vector<int> inst_status;
  std::vector<int> used_fallback;
  std::vector<uint64_t> fallback_cycles;
  bool ran = false;
  uint32_t last_mask = 0;
  // timing
  cudaEvent_t ev[16]{};
  cudaEvent_t ev_copied = nullptr;  // end of the last upload's host->device copies
  bool nvtx_phase_open = false;
  std::vector<std::pair<std::string, std::pair<int, int>>> timed;
  uint64_t launches = 0;
  DevBuf d_scratch;
  // streaming (cs_stream_begin): carry in force for the current batch and the
  // one being produced for the next
  bool streaming = false, stream_fresh = false, stream_pending = false;
  int stream_cur = 0;
  DevBuf d_stream[2];
  DevBuf d_shist[2], d_sdur[2], d_sgap[2];  // carried histories, window-sized rows per instance
  uint32_t s_hw = 1, s_sw = 1;              // row lengths fixed at stream start
  pinned_vector<StreamCarry> h_stream;   // carry in force for the last batch
  pinned_vector<uint64_t> h_cyc_stage;   // pinned staging of cycle-table reads
  std::vector<uint32_t> stream_anchor;   // per instance, fixed after first batch
  // monitor_loop stops at the first NonPositiveLatency (main.cpp:162): an
  // instance whose stream saw a zero-length latency emits nothing afterwards.
  // stream_stopped: set by the run that saw it; stream_stopped_prior: the
  // state before the current run (that run's alerts are cut, later runs' dropped)
  std::vector<uint8_t> stream_stopped, stream_stopped_prior;
  bool stream_broken = false;  // a push failed after it started mutating state
  // steady-state micro-batches: anchor occurrences per instance predicted on
  // the host (carried tail + the new events, the anchor being fixed), so the
  // run sizes its cycle tables without waiting for the event scan; verified
  // against the device's count at the run's final synchronisation
  std::vector<uint64_t> tail_anchors;    // anchor occurrences in each carried tail
  pinned_vector<uint64_t> h_keep;        // tail starts + tail anchor counts (stream_commit)
  pinned_vector<cs_alert> h_alerts_all;  // a push's alerts (stream_commit)
  std::vector<uint64_t> pred_anchors;    // for the run in flight (empty: no prediction)
  bool pred_pending = false;             // pred_anchors = tail_anchors + h_new_anchors once ev_counted completes

  ~cs_ctx() {
    for (auto* m : model_store) delete m;
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (ev_copied) cudaEventDestroy(ev_copied);
    if (ev_layout) cudaEventDestroy(ev_layout);
    if (ev_counted) cudaEventDestroy(ev_counted);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

int fail(cs_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

#define CS_CUDA(call)                                                                \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      return fail(ctx, CS_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

double ucl_from_stats_host(double mu, double sigma, const cs_control_config& c) {
  // detector.cpp:57-60
  const double ucl = std::min(mu + c.sigma_k * sigma, c.theta_max);
  return std::max(ucl, c.min_ucl);
}

template <typename T>
T* dev(DevBuf& b, size_t n) {
  return static_cast<T*>(b.get(std::max<size_t>(1, n) * sizeof(T)));
}

DevBuffers make_buffers(cs_ctx* ctx) {
  DevBuffers b{};
  b.ev = static_cast<const cs_event*>(ctx->d_ev.p);
  b.wl = static_cast<const cs_workload*>(ctx->d_wl.p);
  b.names = static_cast<const cs_name_info*>(ctx->d_names.p);
  b.n_names = static_cast<uint32_t>(ctx->names.size());
  b.n_inst = ctx->n_inst;
  b.inst_off = ctx->p_inst_off;
  b.tile_inst = ctx->p_tile_inst;
  b.tile_begin = ctx->p_tile_begin;
  b.tile_end = ctx->p_tile_end;
  b.inst_first_tile = ctx->p_inst_first_tile;
  b.n_tiles = static_cast<uint32_t>(ctx->tile_inst.size());
  b.stats = static_cast<NameStat*>(ctx->d_stats.p);
  b.inst = static_cast<InstState*>(ctx->d_inst.p);
  b.tile_cnt = static_cast<uint64_t*>(ctx->d_tile_cnt.p);
  b.tile_pref = static_cast<uint64_t*>(ctx->d_tile_pref.p);
  b.scan_tmp = static_cast<uint64_t*>(ctx->d_scan_tmp.p);
  b.a_pos = static_cast<uint64_t*>(ctx->d_a_pos.p);
  b.a_start = static_cast<int64_t*>(ctx->d_a_start.p);
  b.a_end = static_cast<int64_t*>(ctx->d_a_end.p);
  b.cyc_off = static_cast<const uint64_t*>(ctx->d_cyc_off.p);
  b.n_cycles = ctx->n_cycles;
  b.c_start = static_cast<int64_t*>(ctx->c_start.p);
  b.c_end = static_cast<int64_t*>(ctx->c_end.p);
  b.c_apos = static_cast<uint64_t*>(ctx->c_apos.p);
  b.c_aend = static_cast<int64_t*>(ctx->c_aend.p);
  b.c_first = static_cast<uint64_t*>(ctx->c_first.p);
  b.c_last = static_cast<uint64_t*>(ctx->c_last.p);
  b.c_inst = static_cast<uint32_t*>(ctx->c_inst.p);
  b.c_stage = static_cast<uint8_t*>(ctx->c_stage.p);
  b.c_local = static_cast<uint8_t*>(ctx->c_local.p);
  b.c_wl = static_cast<int32_t*>(ctx->c_wl.p);
  b.c_comp = static_cast<int64_t*>(ctx->c_comp.p);
  b.c_beta_tot = static_cast<int64_t*>(ctx->c_beta_tot.p);
  b.c_coll = static_cast<double*>(ctx->c_coll.p);
  b.c_coll_n = static_cast<uint8_t*>(ctx->c_coll_n.p);
  b.rec_off = static_cast<uint64_t*>(ctx->d_rec_off.p);
  b.rec_cycle = static_cast<uint64_t*>(ctx->rec_cycle.p);
  b.rec_pred = static_cast<double*>(ctx->rec_pred.p);
  b.rec_resid = static_cast<double*>(ctx->rec_resid.p);
  b.rec_stat = static_cast<double*>(ctx->rec_stat.p);
  b.rec_flags = static_cast<uint8_t*>(ctx->rec_flags.p);
  b.alert_rec = static_cast<uint64_t*>(ctx->alert_rec.p);
  b.alert_off = static_cast<uint64_t*>(ctx->d_alert_off.p);
  b.block_tmp = static_cast<uint64_t*>(ctx->block_tmp.p);
  b.models = static_cast<const DevModel*>(ctx->d_models.p);
  b.series_slot = static_cast<const int8_t*>(ctx->d_series_slot.p);
  b.class_metric = static_cast<const int8_t*>(ctx->d_class_metric.p);
  b.n_metrics = ctx->n_metrics;
  b.m_off = static_cast<uint64_t*>(ctx->d_m_off.p);
  b.s_ts = static_cast<int64_t*>(ctx->d_s_ts.p);
  b.s_val = static_cast<double*>(ctx->d_s_val.p);
  b.c_mu = static_cast<double*>(ctx->d_mu.p);
  b.c_mu_has = static_cast<uint8_t*>(ctx->d_mu_has.p);
  b.stream = ctx->streaming ? static_cast<StreamCarry*>(ctx->d_stream[ctx->stream_cur].p) : nullptr;
  b.s_hist = ctx->streaming ? static_cast<const double*>(ctx->d_shist[ctx->stream_cur].p) : nullptr;
  b.s_dur = ctx->streaming ? static_cast<const double*>(ctx->d_sdur[ctx->stream_cur].p) : nullptr;
  b.s_gap = ctx->streaming ? static_cast<const double*>(ctx->d_sgap[ctx->stream_cur].p) : nullptr;
  b.s_hw = ctx->s_hw;
  b.s_sw = ctx->s_sw;
  b.any_unknown = static_cast<unsigned int*>(ctx->d_any_unknown.p);
  b.extra_refs = static_cast<const cs_extra_ref*>(ctx->d_extra_refs.p);
  b.n_extra_refs = ctx->n_extra_refs;
  b.extra_vals = static_cast<const cs_extra_value*>(ctx->d_extra_vals.p);
  b.n_extra_keys = static_cast<uint32_t>(ctx->extra_keys.size());
  b.rec_extra = static_cast<double*>(ctx->d_rec_extra.p);
  b.rec_extra_has = static_cast<uint8_t*>(ctx->d_rec_extra_has.p);
  return b;
}

int tree_depth(const cs_tree_node* nodes, uint32_t n, int32_t i, int d, int* out_max,
               int guard) {
  if (i < 0 || static_cast<uint32_t>(i) >= n || guard > 64) return -1;
  *out_max = std::max(*out_max, d);
  if (nodes[i].feature < 0) return 0;
  if (tree_depth(nodes, n, nodes[i].left, d + 1, out_max, guard + 1) < 0) return -1;
  if (tree_depth(nodes, n, nodes[i].right, d + 1, out_max, guard + 1) < 0) return -1;
  return 0;
}

void fill_complete(const cs_tree_node* nodes, int32_t i, uint32_t pos, int d, int D,
                   double* thr, uint8_t* feat, double* leaf, int32_t const* fmap) {
  const uint32_t ni = (1u << D) - 1;
  if (d == D) {
    leaf[pos - ni] = nodes[i].value;
    return;
  }
  if (nodes[i].feature < 0) {
    // leaf above the padded depth: always-left internal node, value copied
    // to every descendant leaf (all but the leftmost are unreachable)
    thr[pos] = std::numeric_limits<double>::infinity();
    feat[pos] = 0;
    fill_complete(nodes, i, 2 * pos + 1, d + 1, D, thr, feat, leaf, fmap);
    fill_complete(nodes, i, 2 * pos + 2, d + 1, D, thr, feat, leaf, fmap);
    return;
  }
  thr[pos] = nodes[i].threshold;
  feat[pos] = static_cast<uint8_t>(nodes[i].feature);
  fill_complete(nodes, nodes[i].left, 2 * pos + 1, d + 1, D, thr, feat, leaf, fmap);
  fill_complete(nodes, nodes[i].right, 2 * pos + 2, d + 1, D, thr, feat, leaf, fmap);
}

}  // namespace

extern "C" {

int cs_abi_version(void) { return CS_ABI_VERSION; }

const char* cs_status_type(int status) {
  switch (status) {
    case CS_OK: return "ok";
    case CS_E_INVALID_ARGUMENT: return "invalid_argument";
    case CS_E_NO_DEVICE: return "no_device";
    case CS_E_CUDA: return "cuda_error";
    case CS_E_NO_ANCHOR_FOUND: return "no_anchor_found";
    case CS_E_MISSING_WORKLOAD: return "missing_workload_args";
    case CS_E_FEATURE_MISMATCH: return "feature_mismatch";
    case CS_E_NON_POSITIVE_LATENCY: return "non_positive_latency";
    case CS_E_INSUFFICIENT_DATA: return "insufficient_data";
    case CS_E_INSUFFICIENT_CALIBRATION: return "insufficient_calibration";
    case CS_E_NO_LABELS: return "no_labels";
    case CS_E_MODEL_FORMAT: return "model_format_error";
    case CS_E_UNSUPPORTED: return "unsupported";
    case CS_E_CONFIG: return "config_error";
    case CS_E_INSUFFICIENT_CYCLES: return "insufficient_cycles";
    case CS_E_NO_BEACONS: return "no_beacons";
    case CS_E_INCONSISTENT_BEACONS: return "inconsistent_beacons";
    case CS_E_ALREADY_CALIBRATED: return "already_calibrated";
    default: return "internal";
  }
}

int cs_ctx_create(int device, cs_ctx** out) {
  if (!out) return CS_E_INVALID_ARGUMENT;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return CS_E_NO_DEVICE;
  }
  if (device < 0 || device >= n) return CS_E_INVALID_ARGUMENT;
  if (cudaSetDevice(device) != cudaSuccess) return CS_E_NO_DEVICE;
  auto* ctx = new cs_ctx();
  ctx->device = device;
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return CS_E_CUDA;
  }
  for (auto& e : ctx->ev) cudaEventCreate(&e);
  // defaults: CycleConfig / ControlConfig
  ctx->cyc.anchor_hint_name = -1;
  ctx->cyc.min_anchor_calls = 10;
  ctx->cyc.prefill_duration_factor = 3.0;
  ctx->cyc.prefill_gap_factor = 2.0;
  ctx->cyc.stage_window = 32;
  ctx->cyc.stage_min_history = 8;
  ctx->cyc.frequency_bin_ns = 1000000;
  ctx->cyc.latency_phase = -1;
  ctx->ctl.strategy = CS_DYNAMIC_WINDOW;
  ctx->ctl.window = 10;
  ctx->ctl.fixed_threshold = 0.15;
  ctx->ctl.sigma_k = 3.0;
  ctx->ctl.theta_max = 0.18;
  ctx->ctl.min_ucl = 0.02;
  ctx->ctl.warmup = 100;
  ctx->ctl.epsilon = 1e-9;
  *out = ctx;
  return CS_OK;
}

void cs_ctx_destroy(cs_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->pin_models) cudaFreeHost(ctx->pin_models);
  if (ctx->pin_ctl) cudaFreeHost(ctx->pin_ctl);
  delete ctx;
}

const char* cs_last_error(const cs_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

int cs_set_config(cs_ctx* ctx, const cs_cycle_config* cycle, const cs_control_config* control) {
  if (!ctx) return CS_E_INVALID_ARGUMENT;
  if (cycle) {
    if (cycle->n_phases < 0 || cycle->n_beta_slots < 0 || cycle->n_comm_slots < 0)
      return fail(ctx, CS_E_INVALID_ARGUMENT, "negative phase / class / collective slot count");
    if (cycle->stage_window == 0 || cycle->stage_window > 1600)
      return fail(ctx, CS_E_UNSUPPORTED, "stage_window must be in [1, 1600]");
    if (cycle->latency_phase >= cycle->n_phases)
      return fail(ctx, CS_E_INVALID_ARGUMENT, "latency_phase out of range");
    if (cycle->frequency_bin_ns <= 0)
      return fail(ctx, CS_E_INVALID_ARGUMENT, "frequency_bin_ns must be positive");
    ctx->cyc = *cycle;
    ++ctx->seg_gen;
  }
  if (control) {
    if (control->strategy < 0 || control->strategy > 2)
      return fail(ctx, CS_E_CONFIG, "unknown detector strategy");
    if (control->window == 0) return fail(ctx, CS_E_CONFIG, "window must be positive");
    ctx->ctl = *control;
  }
  ctx->have_config = true;
  return CS_OK;
}

static int cs_set_name_table_impl(cs_ctx* ctx, uint32_t n_names, const cs_name_info* names) {
  if (ctx) ++ctx->seg_gen;
  if (!ctx || (n_names && !names)) return CS_E_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  ctx->names.assign(names, names + n_names);
  void* d = ctx->d_names.get(std::max<size_t>(1, n_names) * sizeof(cs_name_info));
  if (!d) return fail(ctx, CS_E_CUDA, "cudaMalloc(names)");
  if (n_names) CS_CUDA(cudaMemcpyAsync(d, names, n_names * sizeof(cs_name_info),
                                       cudaMemcpyHostToDevice, ctx->stream));
  // metric slots for the counter-weighted mu: one per counter name a class maps to
  std::vector<int8_t> series(std::max<uint32_t>(1, n_names), -1), cls(std::max<uint32_t>(1, n_names), -1);
  std::map<uint32_t, int> slot_of;
  for (uint32_t i = 0; i < n_names; ++i) {
    const uint32_t m = names[i].metric;
    if (m == 0) continue;
    if (m > n_names) return fail(ctx, CS_E_INVALID_ARGUMENT, "metric name id out of range");
    auto it = slot_of.find(m - 1);
    if (it == slot_of.end()) {
      if (slot_of.size() >= static_cast<size_t>(kMaxMetrics))
        return fail(ctx, CS_E_UNSUPPORTED, "at most 16 counter metrics");
      it = slot_of.emplace(m - 1, static_cast<int>(slot_of.size())).first;
      series[m - 1] = static_cast<int8_t>(it->second);
    }
    cls[i] = static_cast<int8_t>(it->second);
  }
  ctx->n_metrics = static_cast<uint32_t>(slot_of.size());
  void* ds = ctx->d_series_slot.get(series.size());
  void* dc = ctx->d_class_metric.get(cls.size());
  if (!ds || !dc) return fail(ctx, CS_E_CUDA, "cudaMalloc(metrics)");
  CS_CUDA(cudaMemcpy(ds, series.data(), series.size(), cudaMemcpyHostToDevice));
  CS_CUDA(cudaMemcpy(dc, cls.data(), cls.size(), cudaMemcpyHostToDevice));
  return CS_OK;
}

int cs_set_name_table(cs_ctx* ctx, uint32_t n_names, const cs_name_info* names) {
  return cs_guard([&] { return cs_set_name_table_impl(ctx, n_names, names); });
}

}  // extern "C"

namespace {

// Shared by cs_upload / cs_upload_wire: validates the instance layout,
// allocates the event array, uploads workloads and offsets, and builds the
// instance-aligned tiles (= wire blocks).  The caller fills d_ev.
int upload_layout(cs_ctx* ctx, uint32_t n_inst, const uint64_t* inst_offsets, bool have_ev,
                  uint64_t n_workloads, const cs_workload* wl) {
  if (!ctx || !inst_offsets || n_inst == 0) return CS_E_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  if (inst_offsets[0] != 0) return fail(ctx, CS_E_INVALID_ARGUMENT, "inst_offsets[0] must be 0");
  for (uint32_t i = 0; i < n_inst; ++i)
    if (inst_offsets[i + 1] < inst_offsets[i])
      return fail(ctx, CS_E_INVALID_ARGUMENT, "inst_offsets must be non-decreasing");
  const uint64_t n_ev = inst_offsets[n_inst];
  if (n_ev && !have_ev) return CS_E_INVALID_ARGUMENT;
  if (n_workloads && !wl) return CS_E_INVALID_ARGUMENT;
  ctx->n_inst = n_inst;
  ctx->n_ev = n_ev;
  if (n_workloads || wl) ctx->n_wl = n_workloads;  // none given: keep the previous table
  ctx->inst_off.assign(inst_offsets, inst_offsets + n_inst + 1);
  void* de = ctx->d_ev.get(std::max<uint64_t>(1, n_ev) * sizeof(cs_event));
  void* dw = ctx->d_wl.get(std::max<uint64_t>(1, n_workloads) * sizeof(cs_workload));
  if (!de || !dw) return fail(ctx, CS_E_CUDA, "cudaMalloc(events)");
  if (n_workloads)
    CS_CUDA(cudaMemcpyAsync(dw, wl, n_workloads * sizeof(cs_workload), cudaMemcpyHostToDevice,
                            ctx->stream));
  // instance-aligned tiles
  ctx->tile_inst.clear();
  ctx->tile_begin.clear();
  ctx->tile_end.clear();
  ctx->inst_first_tile.assign(n_inst, 0);
  for (uint32_t i = 0; i < n_inst; ++i) {
    ctx->inst_first_tile[i] = static_cast<uint32_t>(ctx->tile_inst.size());
    for (uint64_t t = inst_offsets[i]; t < inst_offsets[i + 1]; t += kTileEvents) {
      ctx->tile_inst.push_back(i);
      ctx->tile_begin.push_back(t);
      ctx->tile_end.push_back(std::min<uint64_t>(t + kTileEvents, inst_offsets[i + 1]));
    }
  }
  const size_t nt = ctx->tile_inst.size();
  if (nt > 0xffffffffull) return fail(ctx, CS_E_UNSUPPORTED, "too many tiles");
  ctx->sample_tiles.clear();
  for (size_t t = 0; t < nt; ++t)
    if (ctx->tile_begin[t] < inst_offsets[ctx->tile_inst[t]] + kSampleEvents)
      ctx->sample_tiles.push_back(static_cast<uint32_t>(t));
  // one staging block, one copy: [inst_off | tile_begin | tile_end | tile_inst |
  // inst_first_tile | sample_tiles], each segment 16-byte aligned
  const size_t ns = ctx->sample_tiles.size();
  if (ctx->ev_layout) CS_CUDA(cudaEventSynchronize(ctx->ev_layout));  // staging block free again
  else if (cudaEventCreateWithFlags(&ctx->ev_layout, cudaEventDisableTiming) != cudaSuccess)
    return fail(ctx, CS_E_CUDA, "cudaEventCreate");
  auto al = [](size_t x) { return (x + 15) & ~static_cast<size_t>(15); };
  const size_t o_off = 0, o_tb = al((n_inst + 1) * 8), o_te = o_tb + al(nt * 8), o_ti = o_te + al(nt * 8),
               o_ft = o_ti + al(nt * 4), o_st = o_ft + al(n_inst * 4u), total = o_st + al(std::max<size_t>(1, ns) * 4);
  ctx->h_layout.resize(total);
  unsigned char* hl = ctx->h_layout.data();
  std::memcpy(hl + o_off, ctx->inst_off.data(), (n_inst + 1) * 8);
  if (nt) {
    std::memcpy(hl + o_tb, ctx->tile_begin.data(), nt * 8);
    std::memcpy(hl + o_te, ctx->tile_end.data(), nt * 8);
    std::memcpy(hl + o_ti, ctx->tile_inst.data(), nt * 4);
  }
  std::memcpy(hl + o_ft, ctx->inst_first_tile.data(), n_inst * 4u);
  if (ns) std::memcpy(hl + o_st, ctx->sample_tiles.data(), ns * 4);
  auto* dl = static_cast<unsigned char*>(ctx->d_layout.get(total));
  if (!dl || !dev<uint64_t>(ctx->d_tile_cnt, nt) || !dev<uint64_t>(ctx->d_tile_pref, nt + 1) ||
      !dev<uint64_t>(ctx->d_scan_tmp, nt / 1024 + 2))
    return fail(ctx, CS_E_CUDA, "cudaMalloc(tiles)");
  CS_CUDA(cudaMemcpyAsync(dl, hl, total, cudaMemcpyHostToDevice, ctx->stream));
  CS_CUDA(cudaEventRecord(ctx->ev_layout, ctx->stream));
  ctx->p_inst_off = reinterpret_cast<uint64_t*>(dl + o_off);
  ctx->p_tile_begin = reinterpret_cast<uint64_t*>(dl + o_tb);
  ctx->p_tile_end = reinterpret_cast<uint64_t*>(dl + o_te);
  ctx->p_tile_inst = reinterpret_cast<uint32_t*>(dl + o_ti);
  ctx->p_inst_first_tile = reinterpret_cast<uint32_t*>(dl + o_ft);
  ctx->p_sample_tiles = reinterpret_cast<uint32_t*>(dl + o_st);
  ctx->ranges_built_for = 0;  // k_segment_range ranges are rebuilt by the next fused run
  ++ctx->seg_gen;
  if (!ctx->extra_keys.empty()) ctx->mt_valid = false;  // extras resolve per upload
  ctx->extra_keys.clear();
  ctx->n_extra_refs = 0;
  // bindings are by instance index and survive re-uploads (streaming pushes)
  if (ctx->model_of_inst.size() < n_inst) ctx->model_of_inst.resize(n_inst, -1);
  ctx->ran = false;
  return CS_OK;
}

}  // namespace

extern "C" {

// An upload returns once its host->device copies have completed: the
// caller's buffers may be reused, and a caller driving two contexts can hand
// the link to the other context's upload while this one's analysis runs.
int wait_copied(cs_ctx* ctx) {
  if (!ctx->ev_copied && cudaEventCreateWithFlags(&ctx->ev_copied, cudaEventDisableTiming) != cudaSuccess)
    return fail(ctx, CS_E_CUDA, "cudaEventCreate");
  CS_CUDA(cudaEventRecord(ctx->ev_copied, ctx->stream));
  return CS_OK;
}

static int cs_upload_unsorted_impl(cs_ctx* ctx, uint32_t n_inst, const uint64_t* inst_offsets,
                                   const cs_event* ev, const uint64_t* event_ids, uint64_t n_workloads,
                                   const cs_workload* wl) {
  CS_NVTX_SCOPE("cs_upload_unsorted");
  if (ctx) ctx->tails_on_device = false;
  if (ctx && ctx->streaming) return fail(ctx, CS_E_INVALID_ARGUMENT, "cs_upload_unsorted mid-stream");
  const int rc = upload_layout(ctx, n_inst, inst_offsets, ev != nullptr, n_workloads, wl);
  if (rc != CS_OK) return rc;
  ctx->have_order = false;
  const uint64_t n = ctx->n_ev;
  auto* din = dev<cs_event>(ctx->d_sort_in, n);
  auto* dids = event_ids ? dev<uint64_t>(ctx->d_sort_ids, n) : nullptr;
  auto* dsc = dev<unsigned long long>(ctx->d_sort_scratch, 4 * std::max<uint64_t>(1, n));
  const uint64_t n_tiles = (n + kSortTile - 1) / kSortTile;
  auto* dh = dev<uint64_t>(ctx->d_sort_hist, 256 * std::max<uint64_t>(1, n_tiles));
  auto* dht = dev<uint64_t>(ctx->d_sort_hist_tmp, 256 * n_tiles / 1024 + 4);
  auto* dex = dev<unsigned long long>(ctx->d_sort_ext, 4);
  auto* dord = dev<uint64_t>(ctx->d_order, n);
  if (!din || (event_ids && !dids) || !dsc || !dh || !dht || !dex || !dord)
    return fail(ctx, CS_E_CUDA, "cudaMalloc(sort)");
  if (n) {
    CS_CUDA(cudaMemcpyAsync(din, ev, n * sizeof(cs_event), cudaMemcpyHostToDevice, ctx->stream));
    if (event_ids)
      CS_CUDA(cudaMemcpyAsync(dids, event_ids, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  }
  if (wait_copied(ctx) != CS_OK) return CS_E_CUDA;
  uint64_t launches = 0;
  if (sort_events_device(din, dids, ctx->p_inst_off, n_inst, n,
                         static_cast<cs_event*>(ctx->d_ev.p), dord, dsc, dh, dht, dex, ctx->stream,
                         &launches) != 0)
    return fail(ctx, CS_E_CUDA, std::string("device sort: ") + cudaGetErrorString(cudaGetLastError()));
  CS_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->have_order = true;
  return CS_OK;
}

int cs_upload_unsorted(cs_ctx* ctx, uint32_t n_inst, const uint64_t* inst_offsets, const cs_event* ev,
                       const uint64_t* event_ids, uint64_t n_workloads, const cs_workload* wl) {
  return cs_guard(
      [&] { return cs_upload_unsorted_impl(ctx, n_inst, inst_offsets, ev, event_ids, n_workloads, wl); });
}

int cs_get_order(cs_ctx* ctx, uint32_t inst, uint64_t* buf, size_t cap, size_t* n) {
  if (!ctx || inst >= ctx->n_inst) return CS_E_INVALID_ARGUMENT;
  if (!ctx->have_order) return fail(ctx, CS_E_INVALID_ARGUMENT, "no cs_upload_unsorted since the last upload");
  const uint64_t b = ctx->inst_off[inst], m = ctx->inst_off[inst + 1] - b;
  if (n) *n = m;
  if (!buf) return CS_OK;
  if (cap < m) return fail(ctx, CS_E_INVALID_ARGUMENT, "buffer too small");
  if (m)
    CS_CUDA(cudaMemcpyAsync(buf, static_cast<const uint64_t*>(ctx->d_order.p) + b, m * 8,
                            cudaMemcpyDeviceToHost, ctx->stream));
  CS_CUDA(cudaStreamSynchronize(ctx->stream));
  return CS_OK;
}

int cs_upload_extras(cs_ctx* ctx, uint32_t n_keys, const char* keys, const cs_extra_ref* refs,
                     uint64_t n_refs, const cs_extra_value* values, uint64_t n_values) {
  if (!ctx || (n_keys && !keys) || (n_refs && !refs) || (n_values && !values)) return CS_E_INVALID_ARGUMENT;
  std::vector<std::string> k;
  const char* p = keys;
  for (uint32_t i = 0; i < n_keys; ++i) {
    k.emplace_back(p);
    p += k.back().size() + 1;
    if (i && !(k[i - 1] < k[i])) return fail(ctx, CS_E_INVALID_ARGUMENT, "extras keys must be sorted and distinct");
  }
  for (uint64_t r = 0; r < n_refs; ++r) {
    if (refs[r].event >= ctx->n_ev || (r && refs[r].event <= refs[r - 1].event))
      return fail(ctx, CS_E_INVALID_ARGUMENT, "extras refs must be sorted by event and inside the upload");
    if (static_cast<uint64_t>(refs[r].first) + refs[r].count > n_values)
      return fail(ctx, CS_E_INVALID_ARGUMENT, "extras ref out of range");
  }
  for (uint64_t v = 0; v < n_values; ++v)
    if (values[v].key >= n_keys) return fail(ctx, CS_E_INVALID_ARGUMENT, "extras key id out of range");
  CS_CUDA(cudaSetDevice(ctx->device));
  void* dr = ctx->d_extra_refs.get(std::max<uint64_t>(1, n_refs) * sizeof(cs_extra_ref));
  void* dv = ctx->d_extra_vals.get(std::max<uint64_t>(1, n_values) * sizeof(cs_extra_value));
  if (!dr || !dv) return fail(ctx, CS_E_CUDA, "cudaMalloc(extras)");
  if (n_refs) CS_CUDA(cudaMemcpyAsync(dr, refs, n_refs * sizeof(cs_extra_ref), cudaMemcpyHostToDevice, ctx->stream));
  if (n_values)
    CS_CUDA(cudaMemcpyAsync(dv, values, n_values * sizeof(cs_extra_value), cudaMemcpyHostToDevice, ctx->stream));
  CS_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->extra_keys = std::move(k);
  ctx->n_extra_refs = n_refs;
  ctx->mt_valid = false;  // model extras resolve against these keys
  return CS_OK;
}

int cs_get_record_extras(cs_ctx* ctx, uint32_t inst, double* values, uint8_t* present, size_t cap,
                         size_t* n) {
  if (!ctx || !ctx->ran || inst >= ctx->n_inst) return CS_E_INVALID_ARGUMENT;
  const uint64_t K = ctx->extra_keys.size();
  const uint64_t r0 = ctx->rec_off[inst], nr = ctx->rec_off[inst + 1] - r0;
  if (n) *n = nr * K;
  if (!values && !present) return CS_OK;
  if (cap < nr * K) return fail(ctx, CS_E_INVALID_ARGUMENT, "buffer too small");
  if (nr * K != 0) {
    if (values)
      CS_CUDA(cudaMemcpy(values, static_cast<const double*>(ctx->d_rec_extra.p) + r0 * K, nr * K * 8,
                         cudaMemcpyDeviceToHost));
    if (present)
      CS_CUDA(cudaMemcpy(present, static_cast<const uint8_t*>(ctx->d_rec_extra_has.p) + r0 * K, nr * K,
                         cudaMemcpyDeviceToHost));
  }
  return CS_OK;
}

int cs_set_cycles(cs_ctx* ctx, const cs_cycle* cycles, uint64_t n, const int64_t* components) {
  if (!ctx || (n && !cycles)) return CS_E_INVALID_ARGUMENT;
  ctx->given.assign(cycles, cycles + n);
  if (components) ctx->given_comp.assign(components, components + n * static_cast<uint64_t>(ctx->cyc.n_phases));
  else ctx->given_comp.clear();
  return CS_OK;
}

static int cs_upload_impl(cs_ctx* ctx, uint32_t n_inst, const uint64_t* inst_offsets, const cs_event* ev,
              uint64_t n_workloads, const cs_workload* wl) {
  CS_NVTX_SCOPE("cs_upload");
  if (ctx) ctx->tails_on_device = false;
  if (ctx) ctx->have_order = false;
  const int rc = upload_layout(ctx, n_inst, inst_offsets, ev != nullptr, n_workloads, wl);
  if (rc != CS_OK) return rc;
  if (ctx->n_ev)
    CS_CUDA(cudaMemcpyAsync(ctx->d_ev.p, ev, ctx->n_ev * sizeof(cs_event), cudaMemcpyHostToDevice,
                            ctx->stream));
  if (wait_copied(ctx) != CS_OK) return CS_E_CUDA;
  CS_CUDA(cudaEventSynchronize(ctx->ev_copied));
  return CS_OK;
}

int cs_upload(cs_ctx* ctx, uint32_t n_inst, const uint64_t* inst_offsets, const cs_event* ev,
              uint64_t n_workloads, const cs_workload* wl) {
  return cs_guard([&] { return cs_upload_impl(ctx, n_inst, inst_offsets, ev, n_workloads, wl); });
}

static int cs_upload_wire_impl(cs_ctx* ctx, uint32_t n_inst, const uint64_t* inst_offsets,
                   const cs_wire_batch* w, uint64_t n_workloads, const cs_workload* wl) {
  if (!w || !ctx) return CS_E_INVALID_ARGUMENT;
  CS_NVTX_SCOPE("cs_upload_wire");
  ctx->tails_on_device = false;
  ctx->have_order = false;
  const bool wl32 = w->workloads32 != nullptr;
  if (wl32 && (n_workloads || wl)) return CS_E_INVALID_ARGUMENT;
  const int rc = upload_layout(ctx, n_inst, inst_offsets, w->codes != nullptr && w->dt_lo && w->blocks,
                               n_workloads, wl);
  if (rc != CS_OK) return rc;
  if ((w->n_durations && (!w->dur_lo || !w->dur_hi)) || (w->n_pay8 && !w->pay8) ||
      (w->n_pay16 && !w->pay16) || (w->n_values && !w->values) || (w->n_escapes && !w->escapes) ||
      (w->n_dt_hi && !w->dt_hi) || w->n_dict > CS_WIRE_MAX_DICT || (w->n_dict && !w->dict))
    return CS_E_INVALID_ARGUMENT;
  const uint64_t n = ctx->n_ev;
  const size_t nt = ctx->tile_inst.size();
  const uint64_t n_wl32 = wl32 ? w->n_workloads32 : 0;
  // one staging allocation, sections 16-B aligned
  auto al = [](size_t x) { return (x + 15) & ~size_t{15}; };
  const size_t s_code = al(n), s_dtl = al(n * 2), s_dth = al(w->n_dt_hi), s_dict = al(w->n_dict * 4),
               s_blk = al(nt * sizeof(cs_wire_block)), s_lo = al(w->n_durations * 2), s_hi = al(w->n_durations),
               s_p8 = al(w->n_pay8), s_p16 = al(w->n_pay16 * 2), s_val = al(w->n_values * 8),
               s_esc = al(w->n_escapes * sizeof(cs_event)), s_wl = al(n_wl32 * 12);
  auto* d = static_cast<unsigned char*>(ctx->d_wire.get(std::max<size_t>(
      16, s_code + s_dtl + s_dth + s_dict + s_blk + s_lo + s_hi + s_p8 + s_p16 + s_val + s_esc + s_wl)));
  if (!d) return fail(ctx, CS_E_CUDA, "cudaMalloc(wire)");
  WireDev dv;
  size_t o = 0;
  auto put = [&](const void* src, size_t bytes, size_t span) -> void* {
    void* dst = d + o;
    if (bytes) cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream);
    o += span;
    return dst;
  };
  dv.codes = static_cast<const uint8_t*>(put(w->codes, n, s_code));
  dv.dt_lo = static_cast<const uint16_t*>(put(w->dt_lo, n * 2, s_dtl));
  dv.dt_hi = static_cast<const uint8_t*>(put(w->dt_hi, w->n_dt_hi, s_dth));
  dv.dict = static_cast<const uint32_t*>(put(w->dict, w->n_dict * 4, s_dict));
  dv.n_dict = w->n_dict;
  dv.blocks = static_cast<const cs_wire_block*>(put(w->blocks, nt * sizeof(cs_wire_block), s_blk));
  dv.dur_lo = static_cast<const uint16_t*>(put(w->dur_lo, w->n_durations * 2, s_lo));
  dv.dur_hi = static_cast<const uint8_t*>(put(w->dur_hi, w->n_durations, s_hi));
  dv.pay8 = static_cast<const uint8_t*>(put(w->pay8, w->n_pay8, s_p8));
  dv.pay16 = static_cast<const uint16_t*>(put(w->pay16, w->n_pay16 * 2, s_p16));
  dv.values = static_cast<const double*>(put(w->values, w->n_values * 8, s_val));
  dv.escapes = static_cast<const cs_event*>(put(w->escapes, w->n_escapes * sizeof(cs_event), s_esc));
  const uint32_t* dwl32 = static_cast<const uint32_t*>(put(w->workloads32, n_wl32 * 12, s_wl));
  CS_CUDA(cudaGetLastError());
  if (wait_copied(ctx) != CS_OK) return CS_E_CUDA;
  if (wl32) {
    void* dw = ctx->d_wl.get(std::max<uint64_t>(1, n_wl32) * sizeof(cs_workload));
    if (!dw) return fail(ctx, CS_E_CUDA, "cudaMalloc(workloads)");
    ctx->n_wl = n_wl32;
    launch_wl32_expand(dwl32, n_wl32, static_cast<cs_workload*>(dw), ctx->stream);
  }
  launch_wire_expand(dv, ctx->p_tile_begin, ctx->p_tile_end, static_cast<uint32_t>(nt),
                     static_cast<cs_event*>(ctx->d_ev.p), ctx->stream);
  CS_CUDA(cudaGetLastError());
  CS_CUDA(cudaEventSynchronize(ctx->ev_copied));  // the expand keeps running
  return CS_OK;
}

int cs_upload_wire(cs_ctx* ctx, uint32_t n_inst, const uint64_t* inst_offsets,
                   const cs_wire_batch* w, uint64_t n_workloads, const cs_workload* wl) {
  return cs_guard([&] { return cs_upload_wire_impl(ctx, n_inst, inst_offsets, w, n_workloads, wl); });
}

static int cs_load_model_impl(cs_ctx* ctx, uint32_t inst, const cs_model* m) {
  if (!ctx || !m) return CS_E_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  if (m->n_features > static_cast<uint32_t>(kMaxFeatures))
    return fail(ctx, CS_E_UNSUPPORTED, "at most 8 model features are supported on device");
  auto* pm = new PackedModel();
  pm->n_trees = m->n_trees;
  pm->n_features = m->n_features;
  pm->degenerate = m->degenerate ? 1u : 0u;
  pm->base = m->base;
  pm->lr = m->learning_rate;
  pm->floor_ = m->prediction_floor;
  pm->mu = m->mu_train;
  pm->sigma = m->sigma_train;
  for (uint32_t f = 0; f < m->n_features; ++f) {
    const int32_t id = m->feature_ids[f];
    const char* nm = m->feature_names ? m->feature_names[f] : nullptr;
    if (id < CS_F_BATCH || id > CS_F_STAGE) {
      // a record extra (main.cpp:70-75), resolved by name when a run scores
      if (!nm || !*nm) {
        delete pm;
        return fail(ctx, CS_E_FEATURE_MISMATCH,
                    "model feature is not one of batch/w_kv/input_len/output_len/stage and has no name");
      }
      pm->feature_ids.push_back(CS_F_EXTRA);
    } else {
      pm->feature_ids.push_back(id);
    }
    pm->feature_names.push_back(nm ? nm : "");
  }
  int D = 0;
  for (uint32_t t = 0; t < m->n_trees; ++t) {
    const uint32_t n = m->tree_offsets[t + 1] - m->tree_offsets[t];
    int dmax = 0;
    if (n == 0 || tree_depth(m->nodes + m->tree_offsets[t], n, 0, 0, &dmax, 0) < 0) {
      delete pm;
      return fail(ctx, CS_E_MODEL_FORMAT, "malformed tree " + std::to_string(t));
    }
    for (uint32_t k = 0; k < n; ++k) {
      const auto& nd = m->nodes[m->tree_offsets[t] + k];
      if (nd.feature >= static_cast<int32_t>(m->n_features)) {
        delete pm;
        return fail(ctx, CS_E_MODEL_FORMAT, "tree node feature out of range");
      }
    }
    D = std::max(D, dmax);
  }
  // complete-tree layout (2^D - 1 internal + 2^D leaves per tree) in HBM
  const double layout_bytes = static_cast<double>(m->n_trees) * std::ldexp(1.0, D) * 25.0;
  if (D > kMaxTreeDepth || layout_bytes > 4e9) {
    delete pm;
    return fail(ctx, CS_E_UNSUPPORTED, "tree too deep for the complete-tree device layout");
  }
  pm->depth = static_cast<uint32_t>(D);
  const uint32_t ni = (1u << D) - 1, nl = 1u << D;
  pm->thr.assign(static_cast<size_t>(m->n_trees) * ni, 0.0);
  pm->feat.assign(static_cast<size_t>(m->n_trees) * ni, 0);
  pm->leaf.assign(static_cast<size_t>(m->n_trees) * nl, 0.0);
  for (uint32_t t = 0; t < m->n_trees; ++t)
    fill_complete(m->nodes + m->tree_offsets[t], 0, 0, 0, D, pm->thr.data() + t * ni,
                  pm->feat.data() + t * ni, pm->leaf.data() + t * nl, nullptr);
  // premultiplied leaves: the reference adds fl(learning_rate * value)
  // (gbdt.cpp:178); integer thresholds: x <= t <=> x <= floor(t) for integer x
  pm->thr_i.resize(pm->thr.size());
  for (size_t k = 0; k < pm->thr.size(); ++k) {
    const double t = pm->thr[k];
    int64_t ti;
    if (std::isnan(t) || t < -9.2e18) ti = -(int64_t{1} << 62);
    else if (t >= 9.2e18) ti = INT64_MAX;
    else ti = static_cast<int64_t>(std::floor(t));
    pm->thr_i[k] = ti;
  }
  for (auto& v : pm->leaf) v = pm->lr * v;
  void* a = pm->d_thr.get(std::max<size_t>(8, pm->thr.size() * 8));
  void* ai = pm->d_thr_i.get(std::max<size_t>(8, pm->thr_i.size() * 8));
  void* b = pm->d_leaf.get(std::max<size_t>(8, pm->leaf.size() * 8));
  void* c = pm->d_feat.get(std::max<size_t>(8, pm->feat.size()));
  if (!a || !ai || !b || !c) {
    delete pm;
    return fail(ctx, CS_E_CUDA, "cudaMalloc(model)");
  }
  if (!pm->thr.empty()) cudaMemcpy(a, pm->thr.data(), pm->thr.size() * 8, cudaMemcpyHostToDevice);
  if (!pm->thr_i.empty()) cudaMemcpy(ai, pm->thr_i.data(), pm->thr_i.size() * 8, cudaMemcpyHostToDevice);
  if (!pm->leaf.empty()) cudaMemcpy(b, pm->leaf.data(), pm->leaf.size() * 8, cudaMemcpyHostToDevice);
  if (!pm->feat.empty()) cudaMemcpy(c, pm->feat.data(), pm->feat.size(), cudaMemcpyHostToDevice);
  // compile <= 2-feature ensembles into an exact cell table (k_lut_build)
  constexpr uint64_t kLutMaxCells = 8ull << 20;
  if (m->n_features >= 1 && m->n_features <= 2 && m->n_trees > 0) {
    for (size_t k = 0; k < pm->thr.size(); ++k) {
      const double t = pm->thr[k];
      if (std::isfinite(t)) pm->lut_thr[pm->feat[k]].push_back(t);
    }
    for (auto& v : pm->lut_thr) {
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
    }
    const uint64_t n0 = pm->lut_thr[0].size(), n1 = pm->lut_thr[1].size();
    const uint64_t cells = (n0 + 1) * (n1 + 1);
    if (cells <= kLutMaxCells) {
      std::vector<int32_t> rank(pm->thr.size());
      for (size_t k = 0; k < pm->thr.size(); ++k) {
        const double t = pm->thr[k];
        if (std::isnan(t) || t == -std::numeric_limits<double>::infinity()) rank[k] = -1;
        else if (t == std::numeric_limits<double>::infinity()) rank[k] = INT32_MAX;
        else {
          const auto& v = pm->lut_thr[pm->feat[k]];
          rank[k] = static_cast<int32_t>(std::lower_bound(v.begin(), v.end(), t) - v.begin());
        }
      }
      auto* d0 = static_cast<double*>(pm->d_lut_thr[0].get(std::max<uint64_t>(1, n0) * 8));
      auto* d1 = static_cast<double*>(pm->d_lut_thr[1].get(std::max<uint64_t>(1, n1) * 8));
      auto* dr = static_cast<int32_t*>(pm->d_rank.get(std::max<size_t>(1, rank.size()) * 4));
      auto* dl = static_cast<double*>(pm->d_lut.get(cells * 8));
      if (d0 && d1 && dr && dl) {
        if (n0) cudaMemcpy(d0, pm->lut_thr[0].data(), n0 * 8, cudaMemcpyHostToDevice);
        if (n1) cudaMemcpy(d1, pm->lut_thr[1].data(), n1 * 8, cudaMemcpyHostToDevice);
        if (!rank.empty()) cudaMemcpy(dr, rank.data(), rank.size() * 4, cudaMemcpyHostToDevice);
        launch_lut_build(static_cast<const uint8_t*>(pm->d_feat.p), dr,
                         static_cast<const double*>(pm->d_leaf.p), pm->n_trees, pm->depth,
                         pm->base, pm->floor_, static_cast<uint32_t>(n0), cells, dl,
                         ctx->stream);
        if (cudaStreamSynchronize(ctx->stream) == cudaSuccess) pm->has_lut = true;
      }
    }
  }
  ctx->model_store.push_back(pm);
  ++ctx->model_gen;
  const int id = static_cast<int>(ctx->model_store.size() - 1);
  if (inst == UINT32_MAX) {
    ctx->default_model = id;
    ctx->model_of_inst.assign(ctx->model_of_inst.size(), -1);
  } else {
    // an instance index may be bound before its first upload (streams)
    if (inst >= kMaxBoundInstances) return fail(ctx, CS_E_INVALID_ARGUMENT, "instance out of range");
    if (ctx->model_of_inst.size() <= inst) ctx->model_of_inst.resize(inst + 1, -1);
    ctx->model_of_inst[inst] = id;
  }
  return CS_OK;
}

int cs_load_model(cs_ctx* ctx, uint32_t inst, const cs_model* m) {
  return cs_guard([&] { return cs_load_model_impl(ctx, inst, m); });
}

}  // extern "C"

namespace {

// Each timing event also moves the NVTX range (nsys / ncu --nvtx): the
// range opened here names the phase whose launches follow the event.
const char* const kPhaseAfterEvent[16] = {"sample_and_setup", "scan_events", "prefix_rank", "bounds",
                                          "cycle_reduce", "stage_records", "score", "detect",
                                          "finish", "host_sizing", nullptr};
// CS_OPT_PHASE_TIMINGS: an event between two small kernels costs the device
// a few microseconds (it ends programmatic dependent launch overlap), so a
// streaming push records only the run's first and last unless asked; mode 2
// keeps the events around the segmentation pass (slots 1, 2 and 4, 5)
static bool phase_events(const cs_ctx* ctx) {
  return ctx->phase_timings == 1 || (ctx->phase_timings < 0 && !ctx->streaming);
}
static bool phase_event_on(const cs_ctx* ctx, int idx) {
  if (idx == 0 || phase_events(ctx)) return true;
  return ctx->phase_timings == 2 && (idx == 1 || idx == 2 || idx == 4 || idx == 5);
}

int record_event(cs_ctx* ctx, int idx) {
  if (!phase_event_on(ctx, idx)) return idx;
  cudaEventRecord(ctx->ev[idx], ctx->stream);
  if (ctx->nvtx_phase_open) nvtxRangePop();
  ctx->nvtx_phase_open = kPhaseAfterEvent[idx] != nullptr;
  if (ctx->nvtx_phase_open) nvtxRangePushA(kPhaseAfterEvent[idx]);
  return idx;
}

// cs_run's outer NVTX range; closes the phase range on every exit path
struct NvtxRun {
  cs_ctx* ctx;
  explicit NvtxRun(cs_ctx* c) : ctx(c) { nvtxRangePushA("cs_run"); }
  ~NvtxRun() {
    if (ctx->nvtx_phase_open) nvtxRangePop();
    ctx->nvtx_phase_open = false;
    nvtxRangePop();
  }
};

// Ranges of the single-read segmentation: consecutive events of one instance,
// about one cycle per lane of the warp that takes the range (the lane-per-cycle
// reduce then keeps every lane busy), built once per upload and range size.
int build_ranges(cs_ctx* ctx, uint64_t range_events) {
  if (ctx->ranges_built_for == range_events) return CS_OK;
  const uint32_t n_inst = ctx->n_inst;
  ctx->range_begin.clear();
  ctx->range_end.clear();
  ctx->range_inst.clear();
  ctx->inst_first_range.assign(n_inst + 1, 0);
  for (uint32_t i = 0; i < n_inst; ++i) {
    ctx->inst_first_range[i] = static_cast<uint32_t>(ctx->range_inst.size());
    for (uint64_t t = ctx->inst_off[i]; t < ctx->inst_off[i + 1]; t += range_events) {
      ctx->range_begin.push_back(t);
      ctx->range_end.push_back(std::min<uint64_t>(t + range_events, ctx->inst_off[i + 1]));
      ctx->range_inst.push_back(i);
    }
  }
  ctx->inst_first_range[n_inst] = static_cast<uint32_t>(ctx->range_inst.size());
  const size_t nr = ctx->range_inst.size();
  if (nr > 0x7fffffffull) return fail(ctx, CS_E_UNSUPPORTED, "too many segmentation ranges");
  auto* rb = dev<uint64_t>(ctx->d_range_begin, nr);
  auto* re = dev<uint64_t>(ctx->d_range_end, nr);
  auto* ri = dev<uint32_t>(ctx->d_range_inst, nr);
  auto* rf = dev<uint32_t>(ctx->d_inst_first_range, n_inst + 1);
  if (!rb || !re || !ri || !rf) return fail(ctx, CS_E_CUDA, "cudaMalloc(ranges)");
  if (nr) {
    CS_CUDA(cudaMemcpyAsync(rb, ctx->range_begin.data(), nr * 8, cudaMemcpyHostToDevice, ctx->stream));
    CS_CUDA(cudaMemcpyAsync(re, ctx->range_end.data(), nr * 8, cudaMemcpyHostToDevice, ctx->stream));
    CS_CUDA(cudaMemcpyAsync(ri, ctx->range_inst.data(), nr * 4, cudaMemcpyHostToDevice, ctx->stream));
  }
  CS_CUDA(cudaMemcpyAsync(rf, ctx->inst_first_range.data(), (n_inst + 1) * 4, cudaMemcpyHostToDevice,
                          ctx->stream));
  CS_CUDA(cudaStreamSynchronize(ctx->stream));  // host vectors may change before the copies ran
  ctx->ranges_built_for = range_events;
  return CS_OK;
}

// NoAnchorFound -> segment_by_frequency (cycles.cpp:283-343) for one instance.
// Returns the number of cycles (0 = still NoAnchorFound); fills t0/period.
int frequency_plan(cs_ctx* ctx, uint32_t i, int64_t* t0, int64_t* period, uint64_t* n) {
  *n = 0;
  const uint64_t b = ctx->inst_off[i], e = ctx->inst_off[i + 1];
  auto* ext = dev<unsigned long long>(ctx->d_scratch, 3);
  if (!ext) return fail(ctx, CS_E_CUDA, "cudaMalloc(scratch)");
  unsigned long long init[3] = {0, ~0ull, 0};
  CS_CUDA(cudaMemcpyAsync(ext, init, sizeof init, cudaMemcpyHostToDevice, ctx->stream));
  launch_gpu_kernel_extent(static_cast<const cs_event*>(ctx->d_ev.p), b, e, ext, ctx->stream,
                           &ctx->launches);
  unsigned long long h[3];
  CS_CUDA(cudaMemcpyAsync(h, ext, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  CS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h[0] < 4) return CS_OK;
  const int64_t lo = static_cast<int64_t>(h[1] ^ (1ull << 63));
  const int64_t hi = static_cast<int64_t>(h[2] ^ (1ull << 63));
  const int64_t bin = ctx->cyc.frequency_bin_ns;
  const uint64_t bins = static_cast<uint64_t>((hi - lo) / bin) + 1;
  if (bins < 4) return CS_OK;
  DevBuf hist, acc;
  auto* dh = static_cast<double*>(hist.get(bins * 2 * sizeof(double)));
  auto* da = static_cast<double*>(acc.get((bins / 2 + 1) * sizeof(double)));
  if (!dh || !da) return fail(ctx, CS_E_CUDA, "cudaMalloc(hist)");
  launch_freq_hist(static_cast<const cs_event*>(ctx->d_ev.p), b, e, lo, bin, bins, dh,
                   ctx->stream, &ctx->launches);
  launch_freq_autocorr(dh, bins, da, ctx->stream, &ctx->launches);
  std::vector<double> a(bins / 2 + 1, 0.0);
  CS_CUDA(cudaMemcpyAsync(a.data(), da, a.size() * sizeof(double), cudaMemcpyDeviceToHost,
                          ctx->stream));
  CS_CUDA(cudaStreamSynchronize(ctx->stream));
  double best = 0.0;
  uint64_t best_lag = 0;
  for (uint64_t lag = 1; lag <= bins / 2; ++lag)
    if (a[lag] > best) {
      best = a[lag];
      best_lag = lag;
    }
  if (best_lag == 0) return CS_OK;
  *period = static_cast<int64_t>(best_lag) * bin;
  *t0 = lo;
  *n = static_cast<uint64_t>((hi - lo) / *period);
  return CS_OK;
}

}  // namespace

extern "C" {

static int cs_run_impl(cs_ctx* ctx, uint32_t mask) {
  HostPhases hp("cs_run");
  if (ctx) hp.stream = ctx->stream;
  if (!ctx) return CS_E_INVALID_ARGUMENT;
  NvtxRun nvtx_run(ctx);
  if (mask & CS_RUN_MU) mask |= CS_RUN_BETA;  // mu divides by the class totals
  if ((mask & CS_RUN_MU) && ctx->streaming)
    return fail(ctx, CS_E_UNSUPPORTED, "mu needs whole-trace counter series (not per micro-batch)");
  if (!(mask & (CS_RUN_SEGMENT | CS_RUN_GIVEN)))
    return fail(ctx, CS_E_INVALID_ARGUMENT, "CS_RUN_SEGMENT (or CS_RUN_GIVEN) required");
  if (ctx->n_inst == 0) return fail(ctx, CS_E_INVALID_ARGUMENT, "nothing uploaded");
  CS_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  ctx->launches = 0;
  ctx->timed.clear();
  const uint32_t n_inst = ctx->n_inst;
  const uint32_t n_names = static_cast<uint32_t>(ctx->names.size());
  const int64_t hint = ctx->cyc.anchor_hint_name;
  if (hint >= static_cast<int64_t>(n_names))
    return fail(ctx, CS_E_INVALID_ARGUMENT, "anchor hint name id out of range");
  if (n_names == 0 && ctx->n_ev) return fail(ctx, CS_E_INVALID_ARGUMENT, "name table not set");
  // streaming: advance to the carry the previous micro-batch produced
  bool all_fixed = false;
  if (ctx->streaming) {
    const uint32_t hw = std::max<uint32_t>(1, ctx->ctl.strategy == CS_FIXED_POINT ? 1 : ctx->ctl.window - 1);
    const uint32_t sw = std::max<uint32_t>(1, ctx->cyc.stage_window);
    if (!ctx->stream_fresh && (hw > ctx->s_hw || sw > ctx->s_sw))
      return fail(ctx, CS_E_INVALID_ARGUMENT, "detector or stage window larger than at the stream's start");
    if (ctx->stream_fresh || ctx->h_stream.size() != n_inst) {
      if (!ctx->stream_fresh) return fail(ctx, CS_E_INVALID_ARGUMENT, "instance count changed mid-stream");
      ctx->s_hw = hw;
      ctx->s_sw = sw;
      for (auto& d : ctx->d_stream)
        if (!dev<StreamCarry>(d, n_inst)) return fail(ctx, CS_E_CUDA, "cudaMalloc(stream)");
      for (int k = 0; k < 2; ++k)
        if (!dev<double>(ctx->d_shist[k], static_cast<size_t>(n_inst) * hw) ||
            !dev<double>(ctx->d_sdur[k], static_cast<size_t>(n_inst) * sw) ||
            !dev<double>(ctx->d_sgap[k], static_cast<size_t>(n_inst) * sw))
          return fail(ctx, CS_E_CUDA, "cudaMalloc(stream histories)");
      CS_CUDA(cudaMemsetAsync(ctx->d_stream[0].p, 0, n_inst * sizeof(StreamCarry), s));
      ctx->stream_cur = 0;
      ctx->h_stream.assign(n_inst, StreamCarry{});
      ctx->stream_anchor.assign(n_inst, UINT32_MAX);
      ctx->stream_stopped.assign(n_inst, 0);
      ctx->stream_fresh = false;
      ctx->stream_pending = false;
    }
    if (ctx->stream_pending) {
      ctx->stream_cur ^= 1;
      ctx->stream_pending = false;
    }
    all_fixed = true;
    for (uint32_t a : ctx->stream_anchor) all_fixed &= a != UINT32_MAX;
  }
  // a host prediction of the anchor counts applies to this run only
  std::vector<uint64_t> pred;
  pred.swap(ctx->pred_anchors);
  const bool pred_deferred = ctx->pred_pending;
  ctx->pred_pending = false;
  const bool predicted = ctx->streaming && all_fixed && (pred.size() == n_inst || pred_deferred) &&
                         !(mask & CS_RUN_GIVEN);
  // per-instance state
  ctx->h_inst.assign(n_inst, InstState{});
  for (uint32_t i = 0; i < n_inst; ++i) {
    auto& st = ctx->h_inst[i];
    st.guess = hint >= 0 ? static_cast<uint32_t>(hint) : UINT32_MAX;
    if (ctx->streaming && ctx->stream_anchor[i] != UINT32_MAX) {
      st.guess = ctx->stream_anchor[i];
      st.fixed_anchor = 1;
    }
    st.anchor = UINT32_MAX;
    st.first_bad_record = UINT64_MAX;
    st.first_missing_record = UINT64_MAX;
  }
  // speculative anchors from the last verified run on this upload
  bool guessed = false;
  if (hint == -1 && !ctx->streaming && !(mask & CS_RUN_GIVEN) && ctx->anchor_gen == ctx->seg_gen &&
      ctx->pred_anchor.size() == n_inst) {
    guessed = true;
    for (uint32_t i = 0; i < n_inst; ++i) guessed &= ctx->pred_anchor[i] != UINT32_MAX;
    if (guessed)
      for (uint32_t i = 0; i < n_inst; ++i) ctx->h_inst[i].guess = ctx->pred_anchor[i];
  }
  auto* d_inst = dev<InstState>(ctx->d_inst, n_inst);
  auto* d_stats = dev<NameStat>(ctx->d_stats, static_cast<size_t>(n_inst) * std::max(1u, n_names));
  const size_t cap_ev = std::max<uint64_t>(1, ctx->n_ev);
  if (!d_inst || !d_stats || !dev<uint64_t>(ctx->d_a_pos, cap_ev) ||
      !dev<int64_t>(ctx->d_a_start, cap_ev) || !dev<int64_t>(ctx->d_a_end, cap_ev))
    return fail(ctx, CS_E_CUDA, "cudaMalloc(state)");
  CS_CUDA(cudaMemcpyAsync(d_inst, ctx->h_inst.data(), n_inst * sizeof(InstState),
                          cudaMemcpyHostToDevice, s));
  if (!dev<unsigned int>(ctx->d_any_unknown, 1)) return fail(ctx, CS_E_CUDA, "cudaMalloc(flag)");
  CS_CUDA(cudaMemsetAsync(ctx->d_any_unknown.p, 0, 4, s));
  hp.mark("state_up");
  const size_t stats_bytes = static_cast<size_t>(n_inst) * n_names * sizeof(NameStat);
  const size_t nt = ctx->tile_inst.size();
  DevConfig cfg{ctx->cyc, ctx->ctl, 0.0};
  DevBuffers b = make_buffers(ctx);

  const int e0 = record_event(ctx, 0);
  if (hint == -1 && !all_fixed && !guessed && !(mask & CS_RUN_GIVEN)) {
    // speculative anchor from a sample of every instance
    if (stats_bytes) CS_CUDA(cudaMemsetAsync(d_stats, 0, stats_bytes, s));
    launch_scan_events(b, cfg, 1, true, ctx->p_sample_tiles,
                       static_cast<uint32_t>(ctx->sample_tiles.size()), s, &ctx->launches);
    launch_rank(b, cfg, 0, s, &ctx->launches);
  }
  const int P = ctx->cyc.n_phases, C = ctx->cyc.n_beta_slots, R = ctx->cyc.n_comm_slots;
  auto alloc_cycles = [&](uint64_t n_slots) -> bool {
    const size_t nc1 = std::max<uint64_t>(1, n_slots);
    return dev<uint64_t>(ctx->d_cyc_off, n_inst + 1) && dev<int64_t>(ctx->c_start, nc1) &&
           dev<int64_t>(ctx->c_end, nc1) && dev<uint64_t>(ctx->c_apos, nc1) &&
           dev<int64_t>(ctx->c_aend, nc1) && dev<uint64_t>(ctx->c_first, nc1) &&
           dev<uint64_t>(ctx->c_last, nc1) && dev<uint32_t>(ctx->c_inst, nc1) &&
           dev<uint8_t>(ctx->c_stage, nc1) && dev<uint8_t>(ctx->c_local, nc1) &&
           dev<int32_t>(ctx->c_wl, nc1) && dev<int64_t>(ctx->c_comp, nc1 * std::max(P, 1)) &&
           dev<int64_t>(ctx->c_beta_tot, nc1 * std::max(C, 1)) &&
           dev<double>(ctx->c_coll, nc1 * std::max(R, 1)) &&
           dev<uint8_t>(ctx->c_coll_n, nc1 * std::max(R, 1)) &&
           dev<uint64_t>(ctx->d_rec_off, n_inst + 1) && dev<uint64_t>(ctx->rec_cycle, nc1) &&
           dev<double>(ctx->rec_pred, nc1) && dev<double>(ctx->rec_resid, nc1) &&
           dev<double>(ctx->rec_stat, nc1) && dev<uint8_t>(ctx->rec_flags, nc1) &&
           dev<uint64_t>(ctx->alert_rec, nc1) && dev<uint64_t>(ctx->d_alert_off, n_inst + 1) &&
           dev<uint64_t>(ctx->block_tmp, nc1 / 256 + 16);
  };
  ctx->n_cyc.assign(n_inst, 0);
  bool speculated = false;
  int e1 = -1, e2 = -1, e4 = -1, e5 = -1;
  ctx->used_fused = false;
  ctx->given_run = false;
  // ---------------- caller-given cycles (CS_RUN_GIVEN): no anchor discovery or
  // segmentation; the cycle table is the caller's (cycles.hpp:62-77)
  if (mask & CS_RUN_GIVEN) {
    if (n_inst != 1) return fail(ctx, CS_E_INVALID_ARGUMENT, "CS_RUN_GIVEN needs exactly one instance");
    if (ctx->streaming) return fail(ctx, CS_E_INVALID_ARGUMENT, "CS_RUN_GIVEN mid-stream");
    const uint64_t nc = ctx->given.size();
    for (const cs_cycle& c : ctx->given)
      if (c.first_event > c.last_event || c.last_event > ctx->n_ev ||
          (c.anchor_pos != UINT64_MAX && c.anchor_pos >= ctx->n_ev))
        return fail(ctx, CS_E_INVALID_ARGUMENT, "given cycle event range out of bounds");
    if (!alloc_cycles(nc)) return fail(ctx, CS_E_CUDA, "cudaMalloc(cycles)");
    ctx->cyc_off.assign({0, nc});
    ctx->n_cyc[0] = nc;
    ctx->n_cycles = nc;
    ctx->inst_status.assign(1, CS_OK);
    ctx->used_fallback.assign(1, 0);
    ctx->fallback_cycles.assign(1, 0);
    ctx->folded.assign(1, {});
    std::vector<int64_t> st(nc), en(nc), ae(nc);
    std::vector<uint64_t> ap(nc), fi(nc), la(nc);
    std::vector<uint8_t> sg(nc);
    for (uint64_t k = 0; k < nc; ++k) {
      const cs_cycle& c = ctx->given[k];
      st[k] = c.start_ts;
      en[k] = c.end_ts;
      ae[k] = c.anchor_span_end;
      ap[k] = c.anchor_pos == UINT64_MAX ? UINT64_MAX : c.anchor_pos;
      fi[k] = c.first_event;
      la[k] = c.last_event;
      sg[k] = static_cast<uint8_t>(c.stage);
    }
    if (nc) {
      CS_CUDA(cudaMemcpyAsync(ctx->c_start.p, st.data(), nc * 8, cudaMemcpyHostToDevice, s));
      CS_CUDA(cudaMemcpyAsync(ctx->c_end.p, en.data(), nc * 8, cudaMemcpyHostToDevice, s));
      CS_CUDA(cudaMemcpyAsync(ctx->c_aend.p, ae.data(), nc * 8, cudaMemcpyHostToDevice, s));
      CS_CUDA(cudaMemcpyAsync(ctx->c_apos.p, ap.data(), nc * 8, cudaMemcpyHostToDevice, s));
      CS_CUDA(cudaMemcpyAsync(ctx->c_first.p, fi.data(), nc * 8, cudaMemcpyHostToDevice, s));
      CS_CUDA(cudaMemcpyAsync(ctx->c_last.p, la.data(), nc * 8, cudaMemcpyHostToDevice, s));
      CS_CUDA(cudaMemsetAsync(ctx->c_inst.p, 0, nc * 4, s));
    }
    CS_CUDA(cudaMemcpyAsync(ctx->d_cyc_off.p, ctx->cyc_off.data(), 16, cudaMemcpyHostToDevice, s));
    b = make_buffers(ctx);
    e1 = e2 = e4 = record_event(ctx, 4);
    launch_cycle_reduce_tpc(b, cfg, (mask & CS_RUN_BETA) ? 1 : 0, s, &ctx->launches, ctx->reduce_variant);
    if (!ctx->given_comp.empty() && P)
      CS_CUDA(cudaMemcpyAsync(ctx->c_comp.p, ctx->given_comp.data(), nc * P * 8, cudaMemcpyHostToDevice, s));
    if (!(mask & CS_RUN_CLASSIFY) && nc)  // build_cycle_records(span): the caller's stages
      CS_CUDA(cudaMemcpyAsync(ctx->c_stage.p, sg.data(), nc, cudaMemcpyHostToDevice, s));
    e5 = record_event(ctx, 5);
    ctx->timed.push_back({"cycle_reduce", {e4, e5}});
    ctx->given_run = true;
    CS_CUDA(cudaStreamSynchronize(s));  // the host staging vectors above go out of scope
  }
  // ---------------- single-read segmentation (k_segment_range)
  if (!ctx->given_run && ctx->allow_fused && !ctx->streaming && ctx->n_ev &&
      segment_range_smem(cfg, (mask & CS_RUN_BETA) ? 1 : 0, static_cast<uint32_t>(ctx->names.size())) >= 0) {
    uint64_t range_events = static_cast<uint64_t>(ctx->opt_range_events);
    if (!range_events) {
      const double epc = ctx->ev_per_cycle > 0.0 ? ctx->ev_per_cycle : 16.0;
      range_events = static_cast<uint64_t>(epc * kSegCycles);
    }
    range_events = std::min<uint64_t>(std::max<uint64_t>((range_events + 31) / 32 * 32, 128), 65536);
    const int rc = build_ranges(ctx, range_events);
    if (rc != CS_OK) return rc;
  }
  const uint32_t n_ranges = static_cast<uint32_t>(ctx->range_inst.size());
  if (!ctx->given_run && ctx->allow_fused && !ctx->streaming && n_ranges && ctx->ranges_built_for &&
      segment_range_smem(cfg, (mask & CS_RUN_BETA) ? 1 : 0, static_cast<uint32_t>(ctx->names.size())) >= 0) {
    const std::vector<InstState> h_init(ctx->h_inst.begin(), ctx->h_inst.end());
    uint64_t cap = std::max<uint64_t>(ctx->slot_cap, ctx->n_ev / 8 + 1024);
    for (int attempt = 0; attempt < 2 && !ctx->used_fused; ++attempt) {
      if (!alloc_cycles(cap) || !dev<unsigned long long>(ctx->d_lb_state, n_ranges) ||
          !dev<uint64_t>(ctx->d_range_prefix, n_ranges) || !dev<unsigned int>(ctx->d_seg_ctl, 2))
        return fail(ctx, CS_E_CUDA, "cudaMalloc(segment)");
      ctx->slot_cap = cap;
      if (attempt) {  // overflow: back to the state after the anchor guess
        for (uint32_t i = 0; i < n_inst; ++i) {
          ctx->h_inst[i].n_anchors = ctx->h_inst[i].n_unknown = 0;
          ctx->h_inst[i].unsorted = 0;
        }
        CS_CUDA(cudaMemcpyAsync(d_inst, ctx->h_inst.data(), n_inst * sizeof(InstState),
                                cudaMemcpyHostToDevice, s));
      }
      if (stats_bytes) CS_CUDA(cudaMemsetAsync(d_stats, 0, stats_bytes, s));
      CS_CUDA(cudaMemsetAsync(ctx->d_lb_state.p, 0, n_ranges * 8ull, s));
      CS_CUDA(cudaMemsetAsync(ctx->d_seg_ctl.p, 0, 8, s));
      b = make_buffers(ctx);
      SegMeta sm{static_cast<const uint64_t*>(ctx->d_range_begin.p),
                 static_cast<const uint64_t*>(ctx->d_range_end.p),
                 static_cast<const uint32_t*>(ctx->d_range_inst.p), n_ranges,
                 static_cast<unsigned long long*>(ctx->d_lb_state.p),
                 static_cast<uint64_t*>(ctx->d_range_prefix.p),
                 static_cast<unsigned int*>(ctx->d_seg_ctl.p),
                 static_cast<unsigned int*>(ctx->d_seg_ctl.p) + 1, cap,
                 static_cast<uint32_t>(ctx->opt_prefetch < 0 ? 0xffffffffu : ctx->opt_prefetch)};
      e1 = record_event(ctx, 1);
      launch_segment_range(b, cfg, sm, (mask & CS_RUN_BETA) ? 1 : 0, s, &ctx->launches);
      e2 = record_event(ctx, 2);
      launch_range_inst(b, sm, static_cast<const uint32_t*>(ctx->d_inst_first_range.p),
                        static_cast<uint64_t*>(ctx->d_cyc_off.p), s, &ctx->launches);
      launch_rank(b, cfg, 1, s, &ctx->launches);
      const int e9 = record_event(ctx, 9);
      e5 = e9;
      ctx->timed.push_back({"segment_range", {e1, e2}});
      ctx->timed.push_back({"sample_and_setup", {e0, e1}});
      ctx->timed.push_back({"prefix_rank", {e2, e9}});
      const uint32_t beta_bit = (mask & CS_RUN_BETA) ? 1u : 0u;
      if (attempt == 0 && ctx->pred_gen == ctx->seg_gen && ctx->pred_beta == beta_bit &&
          ctx->pred_cyc_off.size() == n_inst + 1 && ctx->pred_cyc_off[n_inst] <= cap && !ctx->no_speculate) {
        // sized from the last verified run on this upload; verified at the final sync
        if (!ctx->pin_ctl && cudaHostAlloc(reinterpret_cast<void**>(&ctx->pin_ctl), 8, cudaHostAllocDefault) != cudaSuccess)
          return fail(ctx, CS_E_CUDA, "cudaHostAlloc(ctl)");
        CS_CUDA(cudaMemcpyAsync(ctx->pin_ctl, ctx->d_seg_ctl.p, 8, cudaMemcpyDeviceToHost, s));
        ctx->cyc_off.assign(ctx->pred_cyc_off.begin(), ctx->pred_cyc_off.end());
        for (uint32_t i = 0; i < n_inst; ++i) {
          const uint64_t na = ctx->cyc_off[i + 1] - ctx->cyc_off[i];
          ctx->n_cyc[i] = na >= 2 ? na - 1 : 0;
        }
        ctx->n_cycles = ctx->cyc_off[n_inst];
        ctx->inst_status.assign(n_inst, CS_OK);
        ctx->used_fallback.assign(n_inst, 0);
        ctx->fallback_cycles.assign(n_inst, 0);
        ctx->folded.assign(n_inst, {});
        ctx->used_fused = true;
        speculated = true;
        break;
      }
      unsigned int ctl[2] = {0, 0};
      CS_CUDA(cudaMemcpyAsync(ctx->h_inst.data(), d_inst, n_inst * sizeof(InstState),
                              cudaMemcpyDeviceToHost, s));
      CS_CUDA(cudaMemcpyAsync(ctl, ctx->d_seg_ctl.p, 8, cudaMemcpyDeviceToHost, s));
      hp.mark("segment_issued");
      CS_CUDA(cudaStreamSynchronize(s));
      hp.mark("segment_sync");
      CS_CUDA(cudaGetLastError());
      for (uint32_t i = 0; i < n_inst; ++i)
        if (ctx->h_inst[i].unsorted)
          return fail(ctx, CS_E_INVALID_ARGUMENT,
                      "events of instance " + std::to_string(i) +
                          " are not in canonical (start_ts, event_id) order (trace.cpp:103-109); "
                          "cs_upload_unsorted sorts them on the device");
      uint64_t slots = 0;
      for (uint32_t i = 0; i < n_inst; ++i) slots += ctx->h_inst[i].n_anchors;
      if (ctl[1] & 2u) break;  // a range denser than its anchor list: two-pass path
      if (ctl[1]) {  // more anchors than slots: exact capacity, once more
        cap = slots + 1024;
        continue;
      }
      bool ok = true;
      for (uint32_t i = 0; i < n_inst; ++i) {
        const auto& st = ctx->h_inst[i];
        ok &= !st.ambiguous && !st.redo && !st.no_anchor;
      }
      if (!ok) break;  // wrong guess / uncertified ranking / no anchor: two-pass path
      ctx->cyc_off.assign(n_inst + 1, 0);
      for (uint32_t i = 0; i < n_inst; ++i) {
        const uint64_t na = ctx->h_inst[i].n_anchors;
        ctx->cyc_off[i + 1] = ctx->cyc_off[i] + na;  // slots: cycles + the hole
        ctx->n_cyc[i] = na >= 2 ? na - 1 : 0;
      }
      ctx->n_cycles = slots;
      if (slots) ctx->ev_per_cycle = static_cast<double>(ctx->n_ev) / static_cast<double>(slots);
      ctx->inst_status.assign(n_inst, CS_OK);
      ctx->used_fallback.assign(n_inst, 0);
      ctx->fallback_cycles.assign(n_inst, 0);
      ctx->folded.assign(n_inst, {});
      ctx->used_fused = true;
      ctx->pred_cyc_off.assign(ctx->cyc_off.begin(), ctx->cyc_off.end());  // verified counts for the next run on this upload
      ctx->pred_gen = ctx->seg_gen;
      ctx->pred_beta = beta_bit;
    }
    if (!ctx->used_fused) {
      // rare: redo on the two-pass path from a fresh anchor guess
      ctx->timed.clear();
      ctx->h_inst.assign(h_init.begin(), h_init.end());
      CS_CUDA(cudaMemcpyAsync(d_inst, ctx->h_inst.data(), n_inst * sizeof(InstState),
                              cudaMemcpyHostToDevice, s));
      b = make_buffers(ctx);
      if (hint == -1) {
        if (stats_bytes) CS_CUDA(cudaMemsetAsync(d_stats, 0, stats_bytes, s));
        launch_scan_events(b, cfg, 1, true, ctx->p_sample_tiles,
                           static_cast<uint32_t>(ctx->sample_tiles.size()), s, &ctx->launches);
        launch_rank(b, cfg, 0, s, &ctx->launches);
      }
    }
  }
  if (!ctx->used_fused && !ctx->given_run) {
  if (stats_bytes) CS_CUDA(cudaMemsetAsync(d_stats, 0, stats_bytes, s));
  CS_CUDA(cudaMemsetAsync(ctx->d_tile_cnt.p, 0, std::max<size_t>(1, nt) * 8, s));
  e1 = record_event(ctx, 1);
  launch_scan_events(b, cfg, 3, false, nullptr, static_cast<uint32_t>(nt), s, &ctx->launches);
  e2 = record_event(ctx, 2);
  hp.mark("scan");
  launch_tile_order(b, s, &ctx->launches);
  launch_tile_prefix(b, s, &ctx->launches);
  hp.mark("tiles");
  ctx->timed.push_back({"scan_events", {e1, e2}});
  launch_rank(b, cfg, 1, s, &ctx->launches);
  const int e9 = record_event(ctx, 9);
  ctx->timed.push_back({"sample_and_setup", {e0, e1}});
  ctx->timed.push_back({"prefix_rank", {e2, e9}});
  // steady-state stream: every anchor is fixed and the host predicted the
  // occurrence counts, so the ranking cannot be ambiguous or redone and the
  // sizing needs nothing from the device (checked after the final sync)
  if (predicted) {
    if (pred_deferred) {
      CS_CUDA(cudaEventSynchronize(ctx->ev_counted));
      pred.assign(ctx->tail_anchors.begin(), ctx->tail_anchors.end());
      for (uint32_t i = 0; i < n_inst; ++i) pred[i] += ctx->h_new_anchors[i];
    }
    for (uint32_t i = 0; i < n_inst; ++i) {
      auto& st = ctx->h_inst[i];
      st.n_anchors = pred[i];
      st.anchor = st.n_anchors ? st.guess : UINT32_MAX;
      st.no_anchor = st.n_anchors ? 0u : 1u;
      st.ambiguous = st.redo = 0;
    }
    hp.mark("scan_issued");
  } else {
  CS_CUDA(cudaMemcpyAsync(ctx->h_inst.data(), d_inst, n_inst * sizeof(InstState),
                          cudaMemcpyDeviceToHost, s));
  hp.mark("scan_issued");
  CS_CUDA(cudaStreamSynchronize(s));
  hp.mark("scan_sync");
  CS_CUDA(cudaGetLastError());  // launch failures surface here, not as bad counts
  for (uint32_t i = 0; i < n_inst; ++i)
    if (ctx->h_inst[i].unsorted)
      return fail(ctx, CS_E_INVALID_ARGUMENT,
                  "events of instance " + std::to_string(i) +
                      " are not in canonical (start_ts, event_id) order (trace.cpp:103-109); "
                      "cs_upload_unsorted sorts them on the device");
  }

  // ---- rare paths: ordered fold for uncertified rankings
  ctx->folded.assign(n_inst, {});
  std::vector<uint32_t> pi, pn;
  std::vector<NameStat> hs;
  bool any_amb = false;
  for (uint32_t i = 0; i < n_inst; ++i) any_amb |= ctx->h_inst[i].ambiguous != 0;
  if (any_amb) {
    hs.resize(static_cast<size_t>(n_inst) * n_names);
    CS_CUDA(cudaMemcpy(hs.data(), d_stats, stats_bytes, cudaMemcpyDeviceToHost));
    for (uint32_t i = 0; i < n_inst; ++i) {
      if (!ctx->h_inst[i].ambiguous) continue;
      for (uint32_t n = 0; n < n_names; ++n) {
        const NameStat& st = hs[static_cast<size_t>(i) * n_names + n];
        if (st.count >= ctx->cyc.min_anchor_calls && st.count > 0) {
          pi.push_back(i);
          pn.push_back(n);
        }
      }
    }
    DevBuf dpi, dpn, dout;
    auto* a = static_cast<uint32_t*>(dpi.get(pi.size() * 4));
    auto* c = static_cast<uint32_t*>(dpn.get(pn.size() * 4));
    auto* o = static_cast<double*>(dout.get(pi.size() * 32));
    if (!a || !c || !o) return fail(ctx, CS_E_CUDA, "cudaMalloc(fold)");
    CS_CUDA(cudaMemcpy(a, pi.data(), pi.size() * 4, cudaMemcpyHostToDevice));
    CS_CUDA(cudaMemcpy(c, pn.data(), pn.size() * 4, cudaMemcpyHostToDevice));
    launch_fold(b, cfg, a, c, static_cast<uint32_t>(pi.size()), o, s, &ctx->launches);
    std::vector<double> res(pi.size() * 4);
    CS_CUDA(cudaMemcpyAsync(res.data(), o, res.size() * 8, cudaMemcpyDeviceToHost, s));
    CS_CUDA(cudaStreamSynchronize(s));
    std::vector<double> best_score(n_inst, -1.0);
    std::vector<uint32_t> best_name(n_inst, UINT32_MAX);
    for (size_t k = 0; k < pi.size(); ++k) {
      const uint32_t i = pi[k];
      ctx->folded[i][pn[k]] = {res[4 * k], res[4 * k + 1], res[4 * k + 2], res[4 * k + 3]};
      const double sc = res[4 * k + 2];
      // std::sort by score desc then name asc (cycles.cpp:81-85)
      if (sc > best_score[i] || (sc == best_score[i] && pn[k] < best_name[i])) {
        best_score[i] = sc;
        best_name[i] = pn[k];
      }
    }
    for (uint32_t i = 0; i < n_inst; ++i) {
      if (!ctx->h_inst[i].ambiguous) continue;
      auto& st = ctx->h_inst[i];
      st.anchor = best_name[i];
      st.no_anchor = best_name[i] == UINT32_MAX;
      st.redo = (!st.no_anchor && st.anchor != st.guess) ? 1u : 0u;
    }
  }
  // ---- wrong speculation: compact again for the right anchor
  bool any_redo = false;
  for (uint32_t i = 0; i < n_inst; ++i) any_redo |= ctx->h_inst[i].redo != 0;
  if (any_redo || any_amb) {
    CS_CUDA(cudaMemcpyAsync(d_inst, ctx->h_inst.data(), n_inst * sizeof(InstState),
                            cudaMemcpyHostToDevice, s));
  }
  if (any_redo) {
    std::vector<uint32_t> redo_tiles;
    for (size_t t = 0; t < nt; ++t)
      if (ctx->h_inst[ctx->tile_inst[t]].redo) redo_tiles.push_back(static_cast<uint32_t>(t));
    auto* drt = dev<uint32_t>(ctx->d_redo_tiles, redo_tiles.size());
    if (!drt) return fail(ctx, CS_E_CUDA, "cudaMalloc(redo)");
    CS_CUDA(cudaMemcpyAsync(drt, redo_tiles.data(), redo_tiles.size() * 4,
                            cudaMemcpyHostToDevice, s));
    launch_scan_events(b, cfg, 2 | 4, false, drt, static_cast<uint32_t>(redo_tiles.size()), s,
                       &ctx->launches);
    launch_tile_prefix(b, s, &ctx->launches);
    CS_CUDA(cudaMemcpyAsync(ctx->h_inst.data(), d_inst, n_inst * sizeof(InstState),
                            cudaMemcpyDeviceToHost, s));
    CS_CUDA(cudaStreamSynchronize(s));
  }
  // ---- cycles per instance (frequency fallback where no anchor)
  ctx->inst_status.assign(n_inst, CS_OK);
  ctx->used_fallback.assign(n_inst, 0);
  ctx->fallback_cycles.assign(n_inst, 0);
  std::vector<int64_t> f_t0(n_inst, 0), f_period(n_inst, 0);
  ctx->cyc_off.assign(n_inst + 1, 0);
  for (uint32_t i = 0; i < n_inst; ++i) {
    uint64_t nc = 0;
    const auto& st = ctx->h_inst[i];
    if (st.no_anchor && ctx->streaming) {
      ctx->inst_status[i] = CS_E_NO_ANCHOR_FOUND;  // no cycles in this micro-batch
    } else if (st.no_anchor) {
      int rc = frequency_plan(ctx, i, &f_t0[i], &f_period[i], &nc);
      if (rc != CS_OK) return rc;
      ctx->used_fallback[i] = 1;
      ctx->fallback_cycles[i] = nc;
      if (nc == 0) ctx->inst_status[i] = CS_E_NO_ANCHOR_FOUND;
    } else {
      nc = st.n_anchors >= 2 ? st.n_anchors - 1 : 0;
    }
    ctx->cyc_off[i + 1] = ctx->cyc_off[i] + nc;
    ctx->n_cyc[i] = nc;
  }
  const uint64_t n_cyc = ctx->cyc_off[n_inst];
  ctx->n_cycles = n_cyc;
  if (n_cyc) ctx->ev_per_cycle = static_cast<double>(ctx->n_ev) / static_cast<double>(n_cyc);
  if (!alloc_cycles(n_cyc)) return fail(ctx, CS_E_CUDA, "cudaMalloc(cycles)");
  CS_CUDA(cudaMemcpyAsync(ctx->d_cyc_off.p, ctx->cyc_off.data(), (n_inst + 1) * 8,
                          cudaMemcpyHostToDevice, s));
  b = make_buffers(ctx);
  const int e3 = record_event(ctx, 3);
  ctx->timed.push_back({"host_sizing", {e9, e3}});
  hp.mark("sized");
  launch_bounds(b, s, &ctx->launches);
  for (uint32_t i = 0; i < n_inst; ++i)
    if (ctx->used_fallback[i] && ctx->fallback_cycles[i])
      launch_freq_cycles(static_cast<const cs_event*>(ctx->d_ev.p), ctx->inst_off[i],
                         ctx->inst_off[i + 1], f_t0[i], f_period[i], ctx->fallback_cycles[i],
                         ctx->cyc_off[i], b, i, s, &ctx->launches);
  e4 = record_event(ctx, 4);
  launch_cycle_reduce_tpc(b, cfg, (mask & CS_RUN_BETA) ? 1 : 0, s, &ctx->launches,
                          ctx->reduce_variant);
  e5 = record_event(ctx, 5);
  hp.mark("reduce");
  ctx->timed.push_back({"bounds", {e3, e4}});
  ctx->timed.push_back({"cycle_reduce", {e4, e5}});
  }
  b = make_buffers(ctx);
  if ((!ctx->given_run || (mask & CS_RUN_CLASSIFY)) && ctx->n_cycles) {
    const uint64_t nch = (ctx->n_cycles + kStageChunkCycles - 1) / kStageChunkCycles;
    // no per-run initialisation: st[1] is fully written before it is read,
    // stale changed_iter entries only make a chunk recompute (always exact),
    // and the kernels leave the control words (barrier count, change flags)
    // as they found them; the control words are zeroed once, on allocation
    const void* ctl_before = ctx->d_stage_ctl.p;
    if (!dev<uint8_t>(ctx->d_stage2, ctx->n_cycles) || !dev<int32_t>(ctx->d_stage_changed, nch) ||
        !dev<uint64_t>(ctx->d_stage_lb, nch) || !dev<unsigned int>(ctx->d_stage_ctl, 8))
      return fail(ctx, CS_E_CUDA, "cudaMalloc(stage heuristic)");
    if (ctx->d_stage_ctl.p != ctl_before) CS_CUDA(cudaMemsetAsync(ctx->d_stage_ctl.p, 0, 32, s));
    auto* ctl = static_cast<unsigned int*>(ctx->d_stage_ctl.p);
    StageMeta sm{{static_cast<uint8_t*>(ctx->c_stage.p), static_cast<uint8_t*>(ctx->d_stage2.p)},
                 static_cast<uint32_t>(nch), static_cast<int32_t*>(ctx->d_stage_changed.p),
                 static_cast<uint64_t*>(ctx->d_stage_lb.p), ctl, ctl + 2, ctl + 3, ctl + 4,
                 static_cast<int>(nch) + 2};
    if (launch_stage_heuristic(b, cfg, sm, s, &ctx->launches) != 0)
      return fail(ctx, CS_E_UNSUPPORTED, "stage_window too large for the device heuristic (<= 1600)");
  }
  hp.mark("stage");
  // the per-instance model table first: record compaction can score the
  // records it writes (cell-table models without record extras)
  if (mask & (CS_RUN_SCORE | CS_RUN_DETECT)) {
    bool reuse = ctx->mt_valid && ctx->mt_gen == ctx->model_gen && ctx->mt_n_inst == n_inst &&
                 ctx->h_models.size() == n_inst &&
                 std::memcmp(&ctx->mt_ctl, &ctx->ctl, sizeof(cs_control_config)) == 0;
    for (uint32_t i = 0; i < n_inst && reuse; ++i) reuse = ctx->mt_ids[i] == ctx->model_id(i);
    if (!reuse) {
    ctx->mt_valid = false;
    ctx->h_models.assign(n_inst, DevModel{});
    for (uint32_t i = 0; i < n_inst; ++i) {
      const int id = ctx->model_id(i);
      if (id < 0) return fail(ctx, CS_E_INVALID_ARGUMENT, "no model loaded for an instance");
      const PackedModel* pm = ctx->model_store[id];
      DevModel& dm = ctx->h_models[i];
      dm.n_trees = pm->n_trees;
      dm.depth = pm->depth;
      dm.n_features = pm->n_features;
      dm.degenerate = pm->degenerate;
      for (uint32_t f = 0; f < pm->n_features; ++f) {
        int32_t id = pm->feature_ids[f];
        if (id == CS_F_EXTRA) {
          auto it = std::lower_bound(ctx->extra_keys.begin(), ctx->extra_keys.end(), pm->feature_names[f]);
          id = (it != ctx->extra_keys.end() && *it == pm->feature_names[f])
                   ? kFeatExtra + static_cast<int32_t>(it - ctx->extra_keys.begin())
                   : kFeatMissing;  // every record lacks it: FeatureMismatch at the first
        }
        dm.feature_ids[f] = id;
      }
      dm.base = pm->base;
      dm.lr = pm->lr;
      dm.floor_ = pm->floor_;
      dm.mu = pm->mu;
      dm.sigma = pm->sigma;
      dm.ucl = ctx->ctl.strategy == CS_DYNAMIC_WINDOW ? ucl_from_stats_host(pm->mu, pm->sigma, ctx->ctl)
                                                      : ctx->ctl.fixed_threshold;
      dm.thr = static_cast<const double*>(pm->d_thr.p);
      dm.thr_i = static_cast<const long long*>(pm->d_thr_i.p);
      dm.leaf = static_cast<const double*>(pm->d_leaf.p);
      dm.feat = static_cast<const uint8_t*>(pm->d_feat.p);
      dm.smem_bytes = static_cast<uint64_t>(pm->thr_i.size()) * 8 + pm->leaf.size() * 8 +
                      pm->feat.size();
      dm.lut = (pm->has_lut && !ctx->no_lut) ? static_cast<const double*>(pm->d_lut.p) : nullptr;
      for (int f = 0; f < 2; ++f) {
        dm.lut_thr[f] = static_cast<const double*>(pm->d_lut_thr[f].p);
        dm.lut_n[f] = static_cast<uint32_t>(pm->lut_thr[f].size());
      }
    }
    auto* dm = dev<DevModel>(ctx->d_models, n_inst);
    if (!dm) return fail(ctx, CS_E_CUDA, "cudaMalloc(models)");
    // pinned staging: a pageable copy here would stall the host on the stream
    const size_t mbytes = n_inst * sizeof(DevModel);
    if (mbytes > ctx->pin_models_cap) {
      if (ctx->pin_models) cudaFreeHost(ctx->pin_models);
      ctx->pin_models = nullptr;
      ctx->pin_models_cap = 0;
      if (cudaHostAlloc(&ctx->pin_models, mbytes, cudaHostAllocDefault) != cudaSuccess)
        return fail(ctx, CS_E_CUDA, "cudaHostAlloc(models)");
      ctx->pin_models_cap = mbytes;
    }
    std::memcpy(ctx->pin_models, ctx->h_models.data(), mbytes);
    CS_CUDA(cudaMemcpyAsync(dm, ctx->pin_models, mbytes, cudaMemcpyHostToDevice, s));
    ctx->mt_ids.resize(n_inst);
    for (uint32_t i = 0; i < n_inst; ++i) ctx->mt_ids[i] = ctx->model_id(i);
    ctx->mt_gen = ctx->model_gen;
    ctx->mt_n_inst = n_inst;
    ctx->mt_ctl = ctx->ctl;
    ctx->mt_valid = true;
    }  // rebuild
    b = make_buffers(ctx);
  }
  bool fuse_score = (mask & (CS_RUN_SCORE | CS_RUN_DETECT)) && ctx->extra_keys.empty() && !ctx->no_fused_score;
  for (uint32_t i = 0; i < n_inst && fuse_score; ++i) fuse_score = ctx->h_models[i].lut != nullptr;
  // scores written by compaction carry absolute record indices in
  // first_bad_record / first_missing_record (converted after the final sync)
  const bool score_abs = launch_records(b, cfg, fuse_score ? 1 : 0, s, &ctx->launches);
  hp.mark("records");
  if (!ctx->extra_keys.empty() && ctx->n_cycles) {
    const uint64_t K = ctx->extra_keys.size();
    if (!dev<double>(ctx->d_rec_extra, ctx->n_cycles * K) || !dev<uint8_t>(ctx->d_rec_extra_has, ctx->n_cycles * K))
      return fail(ctx, CS_E_CUDA, "cudaMalloc(record extras)");
    b = make_buffers(ctx);
    launch_record_extras(b, ctx->n_cycles, s, &ctx->launches);
  }
  const int e6m = record_event(ctx, 6);
  ctx->timed.push_back({"stage_records", {e5, e6m}});
  int e6 = e6m;
  // ---- counter-weighted mu (cycle_stats with a CounterTable, rca.cpp:97-126)
  if ((mask & CS_RUN_MU) && ctx->n_metrics && nt) {
    const uint64_t nm = static_cast<uint64_t>(ctx->n_metrics) * nt;
    if (!dev<uint64_t>(ctx->d_m_off, nm + 1) || !dev<uint64_t>(ctx->d_scan_tmp, nm / 1024 + 2))
      return fail(ctx, CS_E_CUDA, "cudaMalloc(counter series)");
    b = make_buffers(ctx);
    launch_counter_series(b, s, &ctx->launches);
    uint64_t n_samples = 0;
    CS_CUDA(cudaMemcpyAsync(&n_samples, static_cast<uint64_t*>(ctx->d_m_off.p) + nm, 8,
                            cudaMemcpyDeviceToHost, s));
    CS_CUDA(cudaStreamSynchronize(s));
    const size_t C = std::max<int32_t>(1, ctx->cyc.n_beta_slots);
    if (!dev<int64_t>(ctx->d_s_ts, std::max<uint64_t>(1, n_samples)) ||
        !dev<double>(ctx->d_s_val, std::max<uint64_t>(1, n_samples)) ||
        !dev<double>(ctx->d_mu, std::max<uint64_t>(1, ctx->n_cycles) * C) ||
        !dev<uint8_t>(ctx->d_mu_has, std::max<uint64_t>(1, ctx->n_cycles) * C))
      return fail(ctx, CS_E_CUDA, "cudaMalloc(mu)");
    b = make_buffers(ctx);
    launch_counter_scatter(b, s, &ctx->launches);
    launch_cycle_mu(b, cfg, s, &ctx->launches);
    e6 = record_event(ctx, 10);
    ctx->timed.push_back({"mu", {e6m, e6}});
  }
  // record counts stay on the device: scoring and detection launch over the
  // cycle count as capacity and clamp to rec_off[n_inst] (no host round trip)
  const uint64_t rec_cap = ctx->n_cycles;
  ctx->rec_off.assign(n_inst + 1, 0);
  int last = e6;
  // ---- score + detect
  if (mask & (CS_RUN_SCORE | CS_RUN_DETECT)) {
    b = make_buffers(ctx);
    if (!dev<uint64_t>(ctx->block_tmp, rec_cap / 256 + 16))
      return fail(ctx, CS_E_CUDA, "cudaMalloc(block_tmp)");
    b = make_buffers(ctx);
    hp.mark("models");
    if (!score_abs)
      launch_score(b, cfg, rec_cap, ctx->rec_off.data(), ctx->model_of_inst.data(),
                   ctx->h_models.data(), s, &ctx->launches);
    hp.mark("score");
    const int e7 = record_event(ctx, 7);
    ctx->timed.push_back({"score", {e6, e7}});
    last = e7;
    if (mask & CS_RUN_DETECT) {
      launch_detect(b, cfg, rec_cap, s, &ctx->launches);
      hp.mark("detect");
      const int e8 = record_event(ctx, 8);
      ctx->timed.push_back({"detect", {e7, e8}});
      last = e8;
    }
  }
  if (ctx->streaming) {
    launch_stream_update(b, cfg, static_cast<StreamCarry*>(ctx->d_stream[ctx->stream_cur ^ 1].p),
                         static_cast<double*>(ctx->d_shist[ctx->stream_cur ^ 1].p),
                         static_cast<double*>(ctx->d_sdur[ctx->stream_cur ^ 1].p),
                         static_cast<double*>(ctx->d_sgap[ctx->stream_cur ^ 1].p),
                         (mask & CS_RUN_DETECT) ? 1 : 0, s);
    ++ctx->launches;
    ctx->stream_pending = true;
    CS_CUDA(cudaMemcpyAsync(ctx->h_stream.data(), ctx->d_stream[ctx->stream_cur].p,
                            n_inst * sizeof(StreamCarry), cudaMemcpyDeviceToHost, s));
  }
  if (!phase_events(ctx)) {  // keep the phases whose events were recorded
    std::vector<std::pair<std::string, std::pair<int, int>>> kept;
    for (auto& t : ctx->timed)
      if (phase_event_on(ctx, t.second.first) && phase_event_on(ctx, t.second.second)) kept.push_back(t);
    ctx->timed.swap(kept);
    if (!phase_event_on(ctx, last)) cudaEventRecord(ctx->ev[last], ctx->stream);
  }
  ctx->timed.push_back({"total", {e0, last}});
  CS_CUDA(cudaMemcpyAsync(ctx->h_inst.data(), d_inst, n_inst * sizeof(InstState),
                          cudaMemcpyDeviceToHost, s));
  ctx->alert_off.assign(n_inst + 1, 0);
  if (mask & CS_RUN_DETECT)
    CS_CUDA(cudaMemcpyAsync(ctx->alert_off.data(), ctx->d_alert_off.p, (n_inst + 1) * 8,
                            cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaMemcpyAsync(ctx->rec_off.data(), ctx->d_rec_off.p, (n_inst + 1) * 8,
                          cudaMemcpyDeviceToHost, s));
  hp.mark("all_issued");
  CS_CUDA(cudaStreamSynchronize(s));
  hp.mark("final_sync");
  if (speculated) {
    bool ok = ctx->pin_ctl[1] == 0u;
    for (uint32_t i = 0; i < n_inst && ok; ++i) {
      const auto& st = ctx->h_inst[i];
      ok = !st.unsorted && !st.ambiguous && !st.redo && !st.no_anchor &&
           st.n_anchors == ctx->pred_cyc_off[i + 1] - ctx->pred_cyc_off[i];
    }
    if (!ok) {  // counts or a fallback condition changed: run again, sized from the device
      ctx->pred_gen = 0;
      ctx->no_speculate = true;
      const int rc = cs_run_impl(ctx, mask);
      ctx->no_speculate = false;
      return rc;
    }
  }
  if (std::getenv("CS_STAGE_ITERS") && ctx->d_stage_ctl.p) {  // profiling: Jacobi iterations of the stage heuristic
    unsigned int it = 0;
    cudaMemcpy(&it, static_cast<unsigned int*>(ctx->d_stage_ctl.p) + 5, 4, cudaMemcpyDeviceToHost);
    std::fprintf(stderr, "stage heuristic iterations: %u\n", it);
  }
  CS_CUDA(cudaGetLastError());
  if (predicted) {
    for (uint32_t i = 0; i < n_inst; ++i) {
      if (ctx->h_inst[i].unsorted)
        return fail(ctx, CS_E_INVALID_ARGUMENT,
                    "events of instance " + std::to_string(i) +
                        " are not in canonical (start_ts, event_id) order (trace.cpp:103-109)");
      if (ctx->h_inst[i].n_anchors != pred[i])
        return fail(ctx, CS_E_INTERNAL, "micro-batch anchor count differs from the host prediction");
    }
  }
  ctx->n_records = ctx->rec_off[n_inst];
  for (uint32_t i = 0; i < n_inst; ++i) {
    // monitor_loop stops at the first record whose features are missing
    // (FeatureMismatch, checked before ppe) or whose latency is <= 0
    InstState& st = ctx->h_inst[i];
    if (!(mask & (CS_RUN_SCORE | CS_RUN_DETECT))) continue;
    if (score_abs) {
      if (st.first_bad_record != UINT64_MAX) st.first_bad_record -= ctx->rec_off[i];
      if (st.first_missing_record != UINT64_MAX) st.first_missing_record -= ctx->rec_off[i];
    }
    const bool miss = st.first_missing_record != UINT64_MAX && st.first_missing_record <= st.first_bad_record;
    if (miss) st.first_bad_record = st.first_missing_record;
    if (ctx->inst_status[i] == CS_OK && st.first_bad_record != UINT64_MAX)
      ctx->inst_status[i] = miss ? CS_E_FEATURE_MISMATCH : CS_E_NON_POSITIVE_LATENCY;
  }
  if (ctx->streaming) {
    ctx->stream_stopped_prior = ctx->stream_stopped;
    for (uint32_t i = 0; i < n_inst; ++i) {
      if (ctx->stream_stopped_prior[i]) ctx->inst_status[i] = ctx->stream_stopped_prior[i];
      if (!ctx->stream_stopped[i] && ctx->h_inst[i].first_bad_record != UINT64_MAX &&
          (mask & (CS_RUN_SCORE | CS_RUN_DETECT)))
        ctx->stream_stopped[i] = static_cast<uint8_t>(ctx->inst_status[i]);  // the stop's status
    }
  } else {
    ctx->stream_stopped_prior.clear();
  }
  if (ctx->streaming)
    for (uint32_t i = 0; i < n_inst; ++i)
      if (ctx->stream_anchor[i] == UINT32_MAX && !ctx->h_inst[i].no_anchor &&
          ctx->h_inst[i].anchor != UINT32_MAX)
        ctx->stream_anchor[i] = ctx->h_inst[i].anchor;
  if (!ctx->streaming && hint == -1 && !(mask & CS_RUN_GIVEN)) {
    ctx->pred_anchor.assign(n_inst, UINT32_MAX);
    for (uint32_t i = 0; i < n_inst; ++i)
      if (!ctx->h_inst[i].no_anchor && !ctx->used_fallback[i]) ctx->pred_anchor[i] = ctx->h_inst[i].anchor;
    ctx->anchor_gen = ctx->seg_gen;
  }
  ctx->ran = true;
  ctx->last_mask = mask;
  hp.mark("done");
  return CS_OK;
}

int cs_run(cs_ctx* ctx, uint32_t mask) {
  return cs_guard([&] { return cs_run_impl(ctx, mask); });
}

int cs_stream_begin(cs_ctx* ctx) {
  if (!ctx) return CS_E_INVALID_ARGUMENT;
  ctx->streaming = true;
  ctx->stream_broken = false;
  ctx->stream_stopped.clear();
  ctx->stream_stopped_prior.clear();
  ctx->tail_len.clear();
  ctx->tail_start.clear();
  ctx->tail_anchors.clear();
  ctx->pred_anchors.clear();
  ctx->tails_on_device = false;
  ctx->stream_fresh = true;
  return CS_OK;
}

int cs_stream_end(cs_ctx* ctx) {
  if (!ctx) return CS_E_INVALID_ARGUMENT;
  ctx->streaming = false;
  ctx->stream_pending = false;
  return CS_OK;
}

int cs_stream_tail(cs_ctx* ctx, uint32_t inst, uint64_t* keep_from) {
  if (!ctx || !keep_from || !ctx->ran || inst >= ctx->n_inst) return CS_E_INVALID_ARGUMENT;
  if (!ctx->streaming) return fail(ctx, CS_E_INVALID_ARGUMENT, "not streaming");
  *keep_from = 0;
  if (ctx->n_cyc[inst] == 0) return CS_OK;
  const uint64_t g = ctx->cyc_off[inst] + ctx->n_cyc[inst] - 1;
  uint64_t last = 0;
  CS_CUDA(cudaMemcpy(&last, static_cast<const uint64_t*>(ctx->c_last.p) + g, 8,
                     cudaMemcpyDeviceToHost));
  *keep_from = last - ctx->inst_off[inst];
  return CS_OK;
}

// After a push's run: new tails (everything from the last closed cycle's end,
// cycles.cpp:147) and the alerts of every instance in instance order, cut at
// the first NonPositiveLatency of the stream (main.cpp:162).
static int stream_commit(cs_ctx* ctx, uint32_t n_inst, uint32_t mask, cs_alert* alerts, size_t cap,
                         size_t* n_alerts, HostPhases& hp) {
  auto* dk = dev<uint64_t>(ctx->d_keep, 2ull * n_inst);
  if (!dk) return fail(ctx, CS_E_CUDA, "cudaMalloc(keep)");
  launch_stream_keep(make_buffers(ctx), dk, ctx->stream);
  pinned_vector<uint64_t>& keep = ctx->h_keep;
  keep.resize(2ull * n_inst);
  CS_CUDA(cudaMemcpyAsync(keep.data(), dk, 2ull * n_inst * 8, cudaMemcpyDeviceToHost, ctx->stream));
  size_t na = 0;
  const bool det = (mask & CS_RUN_DETECT) != 0;
  pinned_vector<cs_alert>& all = ctx->h_alerts_all;
  if (det && ctx->alert_off[n_inst]) {
    const uint64_t n_all = ctx->alert_off[n_inst];
    auto* d = dev<cs_alert>(ctx->d_scratch, n_all);
    if (!d) return fail(ctx, CS_E_CUDA, "cudaMalloc(alerts)");
    DevConfig cfg{ctx->cyc, ctx->ctl, 0.0};
    launch_gather_alerts_all(make_buffers(ctx), cfg, n_all, d, ctx->stream);
    all.resize(n_all);
    CS_CUDA(cudaMemcpyAsync(all.data(), d, n_all * sizeof(cs_alert), cudaMemcpyDeviceToHost,
                            ctx->stream));
  }
  hp.mark("alerts_issued");
  CS_CUDA(cudaStreamSynchronize(ctx->stream));
  hp.mark("sync");
  for (uint32_t i = 0; i < n_inst && det; ++i) {
    if (ctx->stream_stopped_prior[i]) continue;  // stopped by an earlier push
    const uint64_t bad = ctx->h_inst[i].first_bad_record;
    for (uint64_t a = ctx->alert_off[i]; a < ctx->alert_off[i + 1]; ++a) {
      if (all[a].record_index >= bad) break;
      if (alerts && na < cap) alerts[na] = all[a];
      ++na;
    }
  }
  ctx->tail_anchors.resize(n_inst);
  for (uint32_t i = 0; i < n_inst; ++i) {
    const uint64_t len = ctx->stage_off[i + 1] - ctx->stage_off[i];
    const uint64_t k = std::min(keep[i], len);
    ctx->tail_start[i] = ctx->stage_off[i] + k;
    ctx->tail_len[i] = len - k;
    ctx->tail_anchors[i] = keep[n_inst + i];
  }
  ctx->tails_on_device = true;
  hp.mark("end");
  if (n_alerts) *n_alerts = na;
  if (alerts && na > cap)
    return fail(ctx, CS_E_INVALID_ARGUMENT,
                "alert buffer too small (the push is committed; cs_get_alerts reads its alerts)");
  return CS_OK;
}

static int cs_stream_push_impl(cs_ctx* ctx, uint32_t n_inst, const uint64_t* offsets, const cs_event* ev,
                   uint64_t n_workloads, const cs_workload* wl, uint32_t mask, cs_alert* alerts,
                   size_t cap, size_t* n_alerts) {
  HostPhases hp("cs_stream_push");
  if (ctx) hp.stream = ctx->stream;
  if (!ctx || !offsets || n_inst == 0) return CS_E_INVALID_ARGUMENT;
  if (!ctx->streaming) return fail(ctx, CS_E_INVALID_ARGUMENT, "not streaming (cs_stream_begin)");
  if (ctx->stream_broken)
    return fail(ctx, CS_E_INVALID_ARGUMENT, "stream broken by an earlier failed push (cs_stream_begin restarts it)");
  // every argument is checked before any state changes: a rejected push
  // leaves the stream exactly as it was
  if (offsets[0] != 0) return fail(ctx, CS_E_INVALID_ARGUMENT, "offsets[0] must be 0");
  for (uint32_t i = 0; i < n_inst; ++i)
    if (offsets[i + 1] < offsets[i]) return fail(ctx, CS_E_INVALID_ARGUMENT, "offsets must be non-decreasing");
  if (offsets[n_inst] && !ev) return fail(ctx, CS_E_INVALID_ARGUMENT, "events missing");
  if (n_workloads && !wl) return fail(ctx, CS_E_INVALID_ARGUMENT, "n_workloads > 0 needs wl");
  if (!ctx->tail_len.empty() && ctx->tail_len.size() != n_inst && !ctx->stream_fresh)
    return fail(ctx, CS_E_INVALID_ARGUMENT, "instance count changed mid-stream");
  if (ctx->tail_len.size() != n_inst) {
    if (!ctx->tail_len.empty() && !ctx->stream_fresh)
      return fail(ctx, CS_E_INVALID_ARGUMENT, "instance count changed mid-stream");
    ctx->tail_len.assign(n_inst, 0);
    ctx->tail_start.assign(n_inst, 0);
  }
  uint64_t carried = 0;
  for (uint32_t i = 0; i < n_inst; ++i) carried += ctx->tail_len[i];
  if (carried && !ctx->tails_on_device)
    return fail(ctx, CS_E_INVALID_ARGUMENT, "stream tails were replaced by cs_upload (use one streaming API)");
  // new layout: per instance the carried tail, then the new events
  ctx->stage_off.assign(n_inst + 1, 0);
  for (uint32_t i = 0; i < n_inst; ++i)
    ctx->stage_off[i + 1] = ctx->stage_off[i] + ctx->tail_len[i] + (offsets[i + 1] - offsets[i]);
  const uint64_t n_new = offsets[n_inst];
  // the previous batch's events (holding the tails) move to d_ev_prev; the
  // new batch is assembled on the device from them and the uploaded events.
  // From here on a failure (allocation, CUDA, run) leaves the carried tails
  // and detector carry inconsistent: the stream is marked broken and every
  // later push fails loudly instead of assembling from a stale buffer.
  std::swap(ctx->d_ev.p, ctx->d_ev_prev.p);
  std::swap(ctx->d_ev.cap, ctx->d_ev_prev.cap);
  auto broken = [&](int rc) {
    std::swap(ctx->d_ev.p, ctx->d_ev_prev.p);
    std::swap(ctx->d_ev.cap, ctx->d_ev_prev.cap);
    ctx->stream_broken = true;
    return rc;
  };
  hp.mark("pre");
  // the new events go up first; in steady state (every anchor fixed) a tiny
  // kernel counts their anchor occurrences while the host prepares the batch
  // layout, so the run can size its cycle tables without a mid-run sync
  // meta: 4 words per instance, then the fixed anchor ids (u32) when the
  // counts are predicted -- one copy
  bool predict = ctx->tail_anchors.size() == n_inst && ctx->stream_anchor.size() == n_inst && !ctx->stream_fresh;
  for (uint32_t i = 0; i < n_inst && predict; ++i) predict = ctx->stream_anchor[i] != UINT32_MAX;
  const size_t meta_words = 4ull * n_inst + (predict ? (n_inst + 1ull) / 2 : 0);
  auto* d_new = dev<cs_event>(ctx->d_new_ev, std::max<uint64_t>(1, n_new));
  auto* d_meta = dev<uint64_t>(ctx->d_assemble, meta_words);
  if (!d_new || !d_meta) return broken(fail(ctx, CS_E_CUDA, "cudaMalloc(stream)"));
  if (n_new && cudaMemcpyAsync(d_new, ev, n_new * sizeof(cs_event), cudaMemcpyHostToDevice,
                               ctx->stream) != cudaSuccess)
    return broken(fail(ctx, CS_E_CUDA, "cudaMemcpyAsync(stream events)"));
  auto& meta = ctx->assemble_host;
  meta.resize(meta_words);
  for (uint32_t i = 0; i < n_inst; ++i) {
    meta[4 * i + 0] = ctx->stage_off[i];
    meta[4 * i + 1] = ctx->tail_start[i];
    meta[4 * i + 2] = ctx->tail_len[i];
    meta[4 * i + 3] = offsets[i];
  }
  if (predict)
    std::memcpy(reinterpret_cast<uint32_t*>(meta.data() + 4ull * n_inst), ctx->stream_anchor.data(),
                n_inst * sizeof(uint32_t));
  if (cudaMemcpyAsync(d_meta, meta.data(), meta.size() * 8, cudaMemcpyHostToDevice, ctx->stream) !=
      cudaSuccess)
    return broken(fail(ctx, CS_E_CUDA, "cudaMemcpyAsync(stream meta)"));
  if (predict) {
    ctx->h_new_anchors.resize(n_inst);
    const uint32_t* da = reinterpret_cast<const uint32_t*>(d_meta + 4ull * n_inst);
    auto* dc = dev<uint64_t>(ctx->d_new_anchors, n_inst);
    if (!dc) return broken(fail(ctx, CS_E_CUDA, "cudaMalloc(stream count)"));
    if (!ctx->ev_counted && cudaEventCreateWithFlags(&ctx->ev_counted, cudaEventDisableTiming) != cudaSuccess)
      return broken(fail(ctx, CS_E_CUDA, "cudaEventCreate"));
    launch_stream_count(d_new, d_meta, da, n_inst, n_new, dc, ctx->stream);
    CS_CUDA(cudaMemcpyAsync(ctx->h_new_anchors.data(), dc, n_inst * 8ull, cudaMemcpyDeviceToHost, ctx->stream));
    CS_CUDA(cudaEventRecord(ctx->ev_counted, ctx->stream));
  }
  hp.mark("upload_new");
  int rc = upload_layout(ctx, n_inst, ctx->stage_off.data(), true, n_workloads, wl);
  if (rc != CS_OK) return broken(rc);
  hp.mark("layout");
  launch_stream_assemble(static_cast<const cs_event*>(ctx->d_ev_prev.p), d_new, d_meta, n_inst,
                         ctx->stage_off[n_inst], static_cast<cs_event*>(ctx->d_ev.p), ctx->stream);
  if (cudaGetLastError() != cudaSuccess) return broken(fail(ctx, CS_E_CUDA, "stream assemble"));
  ctx->pred_anchors.clear();
  // the run waits for the counts only where it sizes, after issuing its
  // first kernels (the count's round trip overlaps them)
  ctx->pred_pending = predict;
  hp.mark("assemble_count");
  rc = cs_run(ctx, mask);
  if (rc != CS_OK) return broken(rc);
  hp.mark("run");
  // the run has advanced the device carry: from here on the push commits
  // (the tails below move forward even when the alert buffer is too small;
  // the alerts of this push stay readable with cs_get_alerts until the next)
  rc = stream_commit(ctx, n_inst, mask, alerts, cap, n_alerts, hp);
  if (rc != CS_OK && rc != CS_E_INVALID_ARGUMENT) ctx->stream_broken = true;
  return rc;
}

int cs_stream_push(cs_ctx* ctx, uint32_t n_inst, const uint64_t* offsets, const cs_event* ev,
                   uint64_t n_workloads, const cs_workload* wl, uint32_t mask, cs_alert* alerts,
                   size_t cap, size_t* n_alerts) {
  return cs_guard([&] { return cs_stream_push_impl(ctx, n_inst, offsets, ev, n_workloads, wl, mask, alerts, cap, n_alerts); });
}

int cs_sync(cs_ctx* ctx) {
  if (!ctx) return CS_E_INVALID_ARGUMENT;
  CS_CUDA(cudaStreamSynchronize(ctx->stream));
  return CS_OK;
}

int cs_get_summary(cs_ctx* ctx, uint32_t inst, cs_instance_summary* out) {
  if (!ctx || !out || !ctx->ran || inst >= ctx->n_inst) return CS_E_INVALID_ARGUMENT;
  const auto& st = ctx->h_inst[inst];
  out->anchor_name_id = ctx->used_fallback[inst] ? UINT32_MAX : st.anchor;
  out->status = ctx->inst_status[inst];
  out->n_cycles = ctx->n_cyc[inst];
  out->n_records = ctx->rec_off[inst + 1] - ctx->rec_off[inst];
  out->n_alerts = ctx->alert_off[inst + 1] - ctx->alert_off[inst];
  out->first_bad_record = st.first_bad_record;
  out->ucl = inst < ctx->h_models.size() ? ctx->h_models[inst].ucl : 0.0;
  out->used_frequency_fallback = ctx->used_fallback[inst];
  out->anchor_ambiguous = static_cast<int32_t>(st.ambiguous);
  return CS_OK;
}

int cs_get_candidates(cs_ctx* ctx, uint32_t inst, cs_anchor_candidate* buf, size_t cap,
                      size_t* n) {
  if (!ctx || !ctx->ran || inst >= ctx->n_inst) return CS_E_INVALID_ARGUMENT;
  const uint32_t nn = static_cast<uint32_t>(ctx->names.size());
  std::vector<NameStat> hs(nn);
  if (nn)
    CS_CUDA(cudaMemcpy(hs.data(), static_cast<NameStat*>(ctx->d_stats.p) + static_cast<size_t>(inst) * nn,
                       nn * sizeof(NameStat), cudaMemcpyDeviceToHost));
  std::vector<cs_anchor_candidate> out;
  for (uint32_t k = 0; k < nn; ++k) {
    const NameStat& s = hs[k];
    if (s.count < ctx->cyc.min_anchor_calls || s.count == 0) continue;
    cs_anchor_candidate c{};
    c.name_id = k;
    c.call_count = s.count;
    auto it = ctx->folded[inst].find(k);
    if (it != ctx->folded[inst].end()) {
      c.mean_duration_ns = it->second[0];
      c.duration_cv = it->second[1];
      c.score = it->second[2];
      c.periodicity = it->second[3];
    } else {
      // exact moments; within a few ulps of the reference's ordered sums
      const double nd = static_cast<double>(s.count);
      const double sumsq = static_cast<double>(s.sumsq_hi) * 18446744073709551616.0 +
                           static_cast<double>(s.sumsq_lo);
      c.mean_duration_ns = static_cast<double>(static_cast<int64_t>(s.sum)) / nd;
      double cv = 0.0;
      if (c.mean_duration_ns > 0.0) {
        const double var = std::max(0.0, sumsq / nd - c.mean_duration_ns * c.mean_duration_ns);
        cv = std::sqrt(var) / c.mean_duration_ns;
      }
      c.duration_cv = cv;
      c.score = nd / (1.0 + cv);
      c.periodicity = std::numeric_limits<double>::quiet_NaN();  // cs_get_candidates_exact
    }
    out.push_back(c);
  }
  std::sort(out.begin(), out.end(), [](const cs_anchor_candidate& a, const cs_anchor_candidate& b) {
    if (a.score != b.score) return a.score > b.score;
    return a.name_id < b.name_id;
  });
  if (n) *n = out.size();
  if (!buf) return CS_OK;
  if (cap < out.size()) return fail(ctx, CS_E_INVALID_ARGUMENT, "buffer too small");
  std::copy(out.begin(), out.end(), buf);
  return CS_OK;
}

// rank_anchor_candidates (cycles.cpp:47-87) bit for bit: the ordered fold of
// every candidate name of the instance on the device (k_fold, warp per name:
// the reference's sequential sums of d, d*d and the start gaps), then the
// reference's sort (score desc, name asc).
int cs_get_candidates_exact(cs_ctx* ctx, uint32_t inst, cs_anchor_candidate* buf, size_t cap,
                            size_t* n) {
  if (!ctx || !ctx->ran || inst >= ctx->n_inst) return CS_E_INVALID_ARGUMENT;
  CS_CUDA(cudaSetDevice(ctx->device));
  const uint32_t nn = static_cast<uint32_t>(ctx->names.size());
  std::vector<NameStat> hs(nn);
  if (nn)
    CS_CUDA(cudaMemcpy(hs.data(), static_cast<NameStat*>(ctx->d_stats.p) + static_cast<size_t>(inst) * nn,
                       nn * sizeof(NameStat), cudaMemcpyDeviceToHost));
  std::vector<uint32_t> pi, pn;
  for (uint32_t k = 0; k < nn; ++k)
    if (hs[k].count >= ctx->cyc.min_anchor_calls && hs[k].count > 0) {
      pi.push_back(inst);
      pn.push_back(k);
    }
  std::vector<cs_anchor_candidate> out(pi.size());
  if (!pi.empty()) {
    DevBuf dpi, dpn, dout;
    auto* a = static_cast<uint32_t*>(dpi.get(pi.size() * 4));
    auto* c = static_cast<uint32_t*>(dpn.get(pn.size() * 4));
    auto* o = static_cast<double*>(dout.get(pi.size() * 32));
    if (!a || !c || !o) return fail(ctx, CS_E_CUDA, "cudaMalloc(fold)");
    CS_CUDA(cudaMemcpy(a, pi.data(), pi.size() * 4, cudaMemcpyHostToDevice));
    CS_CUDA(cudaMemcpy(c, pn.data(), pn.size() * 4, cudaMemcpyHostToDevice));
    DevConfig cfg{ctx->cyc, ctx->ctl, 0.0};
    launch_fold(make_buffers(ctx), cfg, a, c, static_cast<uint32_t>(pi.size()), o, ctx->stream,
                &ctx->launches);
    std::vector<double> res(pi.size() * 4);
    CS_CUDA(cudaMemcpyAsync(res.data(), o, res.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CS_CUDA(cudaStreamSynchronize(ctx->stream));
    for (size_t k = 0; k < pi.size(); ++k) {
      cs_anchor_candidate& x = out[k];
      x = cs_anchor_candidate{};
      x.name_id = pn[k];
      x.call_count = hs[pn[k]].count;
      x.mean_duration_ns = res[4 * k];
      x.duration_cv = res[4 * k + 1];
      x.score = res[4 * k + 2];
      x.periodicity = res[4 * k + 3];
    }
  }
  std::sort(out.begin(), out.end(), [](const cs_anchor_candidate& a, const cs_anchor_candidate& b) {
    if (a.score != b.score) return a.score > b.score;
    return a.name_id < b.name_id;
  });
  if (n) *n = out.size();
  if (!buf) return CS_OK;
  if (cap < out.size()) return fail(ctx, CS_E_INVALID_ARGUMENT, "buffer too small");
  std::copy(out.begin(), out.end(), buf);
  return CS_OK;
}

}  // extern "C"

namespace {

template <typename T>
int d2h(cs_ctx* ctx, std::vector<T>& v, const DevBuf& b, uint64_t off, uint64_t n) {
  v.resize(n);
  if (n) CS_CUDA(cudaMemcpy(v.data(), static_cast<const T*>(b.p) + off, n * sizeof(T),
                            cudaMemcpyDeviceToHost));
  return CS_OK;
}

}  // namespace

extern "C" {

static int cycles_to_host(cs_ctx* ctx, uint32_t inst, uint64_t first, uint64_t nc, cs_cycle* buf);

int cs_get_cycles(cs_ctx* ctx, uint32_t inst, cs_cycle* buf, size_t cap, size_t* n) {
  if (!ctx || !ctx->ran || inst >= ctx->n_inst) return CS_E_INVALID_ARGUMENT;
  const uint64_t nc = ctx->n_cyc[inst];
  if (n) *n = nc;
  if (!buf) return CS_OK;
  if (cap < nc) return fail(ctx, CS_E_INVALID_ARGUMENT, "buffer too small");
  return cycles_to_host(ctx, inst, 0, nc, buf);
}

int cs_get_cycle_range(cs_ctx* ctx, uint32_t inst, uint64_t first, uint64_t count, cs_cycle* buf) {
  if (!ctx || !ctx->ran || inst >= ctx->n_inst || (count && !buf)) return CS_E_INVALID_ARGUMENT;
  if (first > ctx->n_cyc[inst] || count > ctx->n_cyc[inst] - first)
    return fail(ctx, CS_E_INVALID_ARGUMENT, "cycle range out of bounds");
  return cycles_to_host(ctx, inst, first, count, buf);
}

static int cycles_to_host(cs_ctx* ctx, uint32_t inst, uint64_t first, uint64_t nc, cs_cycle* buf) {
  if (!nc) return CS_OK;
  const uint64_t c0 = ctx->cyc_off[inst] + first;
  // the eight columns land in one pinned staging area: async copies on the
  // ctx stream and one synchronize (pageable copies would each round-trip)
  ctx->h_cyc_stage.resize(7 * nc + (nc + 7) / 8 + 1);
  uint64_t* base = ctx->h_cyc_stage.data();
  auto* st = reinterpret_cast<int64_t*>(base);
  int64_t* en = st + nc;
  int64_t* ae = en + nc;
  auto* ap = reinterpret_cast<uint64_t*>(ae + nc);
  uint64_t* fi = ap + nc;
  uint64_t* la = fi + nc;
  auto* wl = reinterpret_cast<int32_t*>(la + nc);
  auto* sg = reinterpret_cast<uint8_t*>(wl + nc);
  auto col = [&](void* dst, const DevBuf& src, size_t elem) {
    return cudaMemcpyAsync(dst, static_cast<const uint8_t*>(src.p) + c0 * elem, nc * elem,
                           cudaMemcpyDeviceToHost, ctx->stream);
  };
  CS_CUDA(col(st, ctx->c_start, 8));
  CS_CUDA(col(en, ctx->c_end, 8));
  CS_CUDA(col(ae, ctx->c_aend, 8));
  CS_CUDA(col(ap, ctx->c_apos, 8));
  CS_CUDA(col(fi, ctx->c_first, 8));
  CS_CUDA(col(la, ctx->c_last, 8));
  CS_CUDA(col(wl, ctx->c_wl, 4));
  CS_CUDA(col(sg, ctx->c_stage, 1));
  CS_CUDA(cudaStreamSynchronize(ctx->stream));
  const uint64_t ib = ctx->inst_off[inst];
  const uint64_t idx0 = first + (ctx->streaming ? ctx->h_stream[inst].cycle_off : 0);
  for (uint64_t k = 0; k < nc; ++k) {
    cs_cycle& c = buf[k];
    c.index = ctx->given_run ? ctx->given[first + k].index : idx0 + k;
    c.start_ts = st[k];
    c.end_ts = en[k];
    c.anchor_pos = ap[k] == UINT64_MAX ? UINT64_MAX : ap[k] - ib;
    c.anchor_span_end = ae[k];
    c.first_event = fi[k] - ib;
    c.last_event = la[k] - ib;
    c.stage = sg[k];
    c.workload_status = wl[k] >= 0 ? 0 : (wl[k] == -1 ? 1 : 2);
  }
  return CS_OK;
}

int cs_get_components(cs_ctx* ctx, uint32_t inst, int64_t* buf, size_t cap, size_t* n) {
  if (!ctx || !ctx->ran || inst >= ctx->n_inst) return CS_E_INVALID_ARGUMENT;
  const uint64_t P = static_cast<uint64_t>(ctx->cyc.n_phases);
  const uint64_t c0 = ctx->cyc_off[inst], nc = ctx->n_cyc[inst];
  if (n) *n = nc * P;
  if (!buf) return CS_OK;
  if (cap < nc * P) return fail(ctx, CS_E_INVALID_ARGUMENT, "buffer too small");
  if (nc * P != 0)
    CS_CUDA(cudaMemcpy(buf, static_cast<int64_t*>(ctx->c_comp.p) + c0 * P, nc * P * 8,
                       cudaMemcpyDeviceToHost));
  return CS_OK;
}

int cs_get_beta(cs_ctx* ctx, uint32_t inst, int64_t* totals, double* beta, size_t cap, size_t* n) {
  if (!ctx || !ctx->ran || inst >= ctx->n_inst) return CS_E_INVALID_ARGUMENT;
  if (!(ctx->last_mask & CS_RUN_BETA)) return fail(ctx, CS_E_INVALID_ARGUMENT, "beta not computed");
  const uint64_t Cs = static_cast<uint64_t>(ctx->cyc.n_beta_slots);
  const uint64_t c0 = ctx->cyc_off[inst], nc = ctx->n_cyc[inst];
  if (n) *n = nc * Cs;
  if (cap < nc * Cs && (totals || beta)) return fail(ctx, CS_E_INVALID_ARGUMENT, "buffer too small");
  if (totals && nc * Cs != 0)
    CS_CUDA(cudaMemcpy(totals, static_cast<int64_t*>(ctx->c_beta_tot.p) + c0 * Cs, nc * Cs * 8,
                       cudaMemcpyDeviceToHost));
  if (beta && nc * Cs != 0) {
    // beta = total / cycle duration (rca.cpp:95-96, 119-121), formed here from
    // the device's totals (masked to positive durations) and cycle bounds:
    // one IEEE division, the same bits as a device __ddiv_rn
    std::vector<int64_t> tot(totals ? 0 : nc * Cs), st(nc), en(nc);
    int64_t* t = totals ? totals : tot.data();
    if (!totals)
      CS_CUDA(cudaMemcpy(t, static_cast<int64_t*>(ctx->c_beta_tot.p) + c0 * Cs, nc * Cs * 8,
                         cudaMemcpyDeviceToHost));
    CS_CUDA(cudaMemcpy(st.data(), static_cast<int64_t*>(ctx->c_start.p) + c0, nc * 8, cudaMemcpyDeviceToHost));
    CS_CUDA(cudaMemcpy(en.data(), static_cast<int64_t*>(ctx->c_end.p) + c0, nc * 8, cudaMemcpyDeviceToHost));
    for (uint64_t k = 0; k < nc; ++k) {
      const double dur = static_cast<double>(en[k] - st[k]);
      for (uint64_t c = 0; c < Cs; ++c) {
        const int64_t v = t[k * Cs + c];
        beta[k * Cs + c] = v > 0 ? static_cast<double>(v) / dur : 0.0;
      }
    }
  }
  return CS_OK;
}

int cs_get_collective_beta(cs_ctx* ctx, uint32_t inst, double* beta, uint8_t* present,
                           size_t cap, size_t* n) {
  if (!ctx || !ctx->ran || inst >= ctx->n_inst) return CS_E_INVALID_ARGUMENT;
  if (!(ctx->last_mask & CS_RUN_BETA)) return fail(ctx, CS_E_INVALID_ARGUMENT, "beta not computed");
  const uint64_t R = static_cast<uint64_t>(ctx->cyc.n_comm_slots);
  const uint64_t c0 = ctx->cyc_off[inst], nc = ctx->n_cyc[inst];
  if (n) *n = nc * R;
  if (cap < nc * R && (beta || present)) return fail(ctx, CS_E_INVALID_ARGUMENT, "buffer too small");
  if (beta && nc * R != 0)
    CS_CUDA(cudaMemcpy(beta, static_cast<double*>(ctx->c_coll.p) + c0 * R, nc * R * 8,
                       cudaMemcpyDeviceToHost));
  if (present && nc * R != 0) {
    CS_CUDA(cudaMemcpy(present, static_cast<uint8_t*>(ctx->c_coll_n.p) + c0 * R, nc * R,
                       cudaMemcpyDeviceToHost));
    for (uint64_t k = 0; k < nc * R; ++k) present[k] = present[k] ? 1 : 0;
  }
  return CS_OK;
}

static int cs_suspicion_rank_impl(cs_ctx* ctx, uint32_t inst, const uint64_t* normal_cycles, size_t n_normal,
                      const uint64_t* abnormal_cycles, size_t n_abnormal, const int32_t* comm_name,
                      const int32_t* comm_group, const int32_t* comm_rank,
                      const int32_t* comm_location, cs_suspect* out, size_t cap, size_t* n_out) {
  if (!ctx || !ctx->ran || inst >= ctx->n_inst || !n_out) return CS_E_INVALID_ARGUMENT;
  if (!(ctx->last_mask & CS_RUN_BETA)) return fail(ctx, CS_E_INVALID_ARGUMENT, "beta not computed");
  if ((n_normal && !normal_cycles) || (n_abnormal && !abnormal_cycles)) return CS_E_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  const uint32_t S = static_cast<uint32_t>(ctx->cyc.n_beta_slots), R = static_cast<uint32_t>(ctx->cyc.n_comm_slots);
  if (R && (!comm_name || !comm_group || !comm_rank)) return CS_E_INVALID_ARGUMENT;
  const uint64_t c0 = ctx->cyc_off[inst], nc = ctx->n_cyc[inst];
  const bool with_mu = (ctx->last_mask & CS_RUN_MU) != 0;
  // window rows, gathered cycle by cycle (windows are a few hundred cycles)
  struct Rows {
    std::vector<int64_t> totals;
    std::vector<double> beta, mu, coll;
    std::vector<uint8_t> mu_has, coll_n;
  };
  auto gather = [&](const uint64_t* idx, size_t n, Rows& w) -> int {
    w.totals.resize(n * S);
    w.beta.resize(n * S);
    w.coll.resize(n * R);
    w.coll_n.resize(n * R);
    if (with_mu) {
      w.mu.resize(n * S);
      w.mu_has.resize(n * S);
    }
    for (size_t k = 0; k < n; ++k) {
      if (idx[k] >= nc) return CS_E_INVALID_ARGUMENT;
      const uint64_t c = c0 + idx[k];
      if (S) {
        CS_CUDA(cudaMemcpy(&w.totals[k * S], static_cast<int64_t*>(ctx->c_beta_tot.p) + c * S, S * 8,
                           cudaMemcpyDeviceToHost));
        int64_t se[2];
        CS_CUDA(cudaMemcpy(&se[0], static_cast<int64_t*>(ctx->c_start.p) + c, 8, cudaMemcpyDeviceToHost));
        CS_CUDA(cudaMemcpy(&se[1], static_cast<int64_t*>(ctx->c_end.p) + c, 8, cudaMemcpyDeviceToHost));
        for (uint32_t q = 0; q < S; ++q) {  // beta = total / duration, formed on read
          const int64_t v = w.totals[k * S + q];
          w.beta[k * S + q] = v > 0 ? static_cast<double>(v) / static_cast<double>(se[1] - se[0]) : 0.0;
        }
        if (with_mu) {
          CS_CUDA(cudaMemcpy(&w.mu[k * S], static_cast<double*>(ctx->d_mu.p) + c * S, S * 8,
                             cudaMemcpyDeviceToHost));
          CS_CUDA(cudaMemcpy(&w.mu_has[k * S], static_cast<uint8_t*>(ctx->d_mu_has.p) + c * S, S,
                             cudaMemcpyDeviceToHost));
        }
      }
      if (R) {
        CS_CUDA(cudaMemcpy(&w.coll[k * R], static_cast<double*>(ctx->c_coll.p) + c * R, R * 8,
                           cudaMemcpyDeviceToHost));
        CS_CUDA(cudaMemcpy(&w.coll_n[k * R], static_cast<uint8_t*>(ctx->c_coll_n.p) + c * R, R,
                           cudaMemcpyDeviceToHost));
      }
    }
    for (auto& x : w.coll_n) x = x ? 1 : 0;
    return CS_OK;
  };
  Rows rn, ra;
  int rc = gather(normal_cycles, n_normal, rn);
  if (rc == CS_OK) rc = gather(abnormal_cycles, n_abnormal, ra);
  if (rc != CS_OK) return fail(ctx, rc, "cycle index out of range");
  auto window = [&](Rows& w, size_t n) {
    cs_rca_window v{};
    v.n_cycles = n;
    v.totals = w.totals.data();
    v.beta = w.beta.data();
    v.mu = with_mu ? w.mu.data() : nullptr;
    v.mu_has = with_mu ? w.mu_has.data() : nullptr;
    v.coll = w.coll.data();
    v.coll_present = w.coll_n.data();
    return v;
  };
  const cs_rca_window wn = window(rn, n_normal), wa = window(ra, n_abnormal);
  // per beta slot: its name's metric; per comm slot: its name's beta slot
  std::vector<int32_t> slot_metric(std::max<uint32_t>(S, 1), 0), comm_class(std::max<uint32_t>(R, 1), -1);
  for (const auto& ni : ctx->names)
    if (ni.beta_slot >= 0 && static_cast<uint32_t>(ni.beta_slot) < S) slot_metric[ni.beta_slot] = static_cast<int32_t>(ni.metric);
  for (uint32_t k = 0; k < R; ++k) {
    if (comm_name[k] < 0 || static_cast<size_t>(comm_name[k]) >= ctx->names.size()) return CS_E_INVALID_ARGUMENT;
    comm_class[k] = ctx->names[comm_name[k]].beta_slot;
  }
  cs_rca_layout lay{};
  lay.n_slots = S;
  lay.n_comm = R;
  lay.slot_metric = slot_metric.data();
  lay.comm_class = comm_class.data();
  lay.comm_group = comm_group;
  lay.comm_rank = comm_rank;
  lay.comm_location = comm_location;
  rc = cs_rank_suspects(&wn, &wa, &lay, out, cap, n_out);
  if (rc == CS_E_INSUFFICIENT_CYCLES)
    return fail(ctx, rc, "need >= 10 normal and >= 3 abnormal cycles, got " + std::to_string(n_normal) + "/" +
                             std::to_string(n_abnormal));
  return rc;
}

int cs_suspicion_rank(cs_ctx* ctx, uint32_t inst, const uint64_t* normal_cycles, size_t n_normal,
                      const uint64_t* abnormal_cycles, size_t n_abnormal, const int32_t* comm_name,
                      const int32_t* comm_group, const int32_t* comm_rank,
                      const int32_t* comm_location, cs_suspect* out, size_t cap, size_t* n_out) {
  return cs_guard([&] { return cs_suspicion_rank_impl(ctx, inst, normal_cycles, n_normal, abnormal_cycles, n_abnormal, comm_name, comm_group, comm_rank, comm_location, out, cap, n_out); });
}

int cs_get_mu(cs_ctx* ctx, uint32_t inst, double* mu, uint8_t* has, size_t cap, size_t* n) {
  if (!ctx || !ctx->ran || inst >= ctx->n_inst) return CS_E_INVALID_ARGUMENT;
  if (!(ctx->last_mask & CS_RUN_MU)) return fail(ctx, CS_E_INVALID_ARGUMENT, "mu not computed");
  const uint64_t C = static_cast<uint64_t>(ctx->cyc.n_beta_slots);
  const uint64_t c0 = ctx->cyc_off[inst], nc = ctx->n_cyc[inst];
  if (n) *n = nc * C;
  if (cap < nc * C && (mu || has)) return fail(ctx, CS_E_INVALID_ARGUMENT, "buffer too small");
  if (!ctx->n_metrics) {  // no class maps to a counter: beta-only entries everywhere
    if (mu) std::fill(mu, mu + nc * C, 0.0);
    if (has) std::fill(has, has + nc * C, 0);
    return CS_OK;
  }
  if (mu && nc * C != 0)
    CS_CUDA(cudaMemcpy(mu, static_cast<double*>(ctx->d_mu.p) + c0 * C, nc * C * 8, cudaMemcpyDeviceToHost));
  if (has && nc * C != 0)
    CS_CUDA(cudaMemcpy(has, static_cast<uint8_t*>(ctx->d_mu_has.p) + c0 * C, nc * C, cudaMemcpyDeviceToHost));
  return CS_OK;
}

}  // extern "C"

namespace {

int gather_records(cs_ctx* ctx, uint32_t inst, uint64_t r0, uint64_t nr, cs_record* out) {
  if (!nr) return CS_OK;
  auto* d = dev<cs_record>(ctx->d_scratch, nr);
  if (!d) return fail(ctx, CS_E_CUDA, "cudaMalloc(gather)");
  DevConfig cfg{ctx->cyc, ctx->ctl, 0.0};
  const bool scored = ctx->last_mask & (CS_RUN_SCORE | CS_RUN_DETECT);
  const bool det = ctx->last_mask & CS_RUN_DETECT;
  launch_gather_records(make_buffers(ctx), cfg, inst, r0, nr, scored, det, d, ctx->stream);
  CS_CUDA(cudaMemcpyAsync(out, d, nr * sizeof(cs_record), cudaMemcpyDeviceToHost, ctx->stream));
  CS_CUDA(cudaStreamSynchronize(ctx->stream));
  return CS_OK;
}

}  // namespace

extern "C" {

int cs_get_records(cs_ctx* ctx, uint32_t inst, cs_record* buf, size_t cap, size_t* n) {
  if (!ctx || !ctx->ran || inst >= ctx->n_inst) return CS_E_INVALID_ARGUMENT;
  const uint64_t r0 = ctx->rec_off[inst], nr = ctx->rec_off[inst + 1] - r0;
  if (n) *n = nr;
  if (!buf) return CS_OK;
  if (cap < nr) return fail(ctx, CS_E_INVALID_ARGUMENT, "buffer too small");
  int rc = gather_records(ctx, inst, r0, nr, buf);
  if (rc) return rc;
  if (ctx->given_run)
    for (uint64_t k = 0; k < nr; ++k) buf[k].cycle_index = ctx->given[buf[k].cycle_index].index;
  if (ctx->last_mask & CS_RUN_DETECT) {
    // episode ids: running alert count within the instance
    uint64_t ep = ctx->streaming ? ctx->h_stream[inst].episodes : 0;
    for (uint64_t k = 0; k < nr; ++k)
      if (buf[k].alert) buf[k].episode_id = ep++;
  }
  return CS_OK;
}

int cs_get_record_range(cs_ctx* ctx, uint32_t inst, uint64_t first, uint64_t count, cs_record* buf) {
  if (!ctx || !ctx->ran || inst >= ctx->n_inst || (count && !buf)) return CS_E_INVALID_ARGUMENT;
  const uint64_t r0 = ctx->rec_off[inst], nr = ctx->rec_off[inst + 1] - r0;
  if (first > nr || count > nr - first) return fail(ctx, CS_E_INVALID_ARGUMENT, "record range out of bounds");
  int rc = gather_records(ctx, inst, r0 + first, count, buf);
  if (rc) return rc;
  if ((ctx->last_mask & CS_RUN_DETECT) && count) {
    bool any = false;
    for (uint64_t k = 0; k < count && !any; ++k) any = buf[k].alert;
    if (any) {
      // episode ids: alerts before the range (the alerts are few)
      size_t na = 0;
      if ((rc = cs_get_alerts(ctx, inst, nullptr, 0, &na))) return rc;
      std::vector<cs_alert> al(na);
      if (na && (rc = cs_get_alerts(ctx, inst, al.data(), na, &na))) return rc;
      uint64_t ep = ctx->streaming ? ctx->h_stream[inst].episodes : 0;
      for (const cs_alert& a : al) ep += a.record_index < first;
      for (uint64_t k = 0; k < count; ++k)
        if (buf[k].alert) buf[k].episode_id = ep++;
    }
  }
  return CS_OK;
}

int cs_get_alerts(cs_ctx* ctx, uint32_t inst, cs_alert* buf, size_t cap, size_t* n) {
  if (!ctx || !ctx->ran || inst >= ctx->n_inst) return CS_E_INVALID_ARGUMENT;
  if (!(ctx->last_mask & CS_RUN_DETECT)) return fail(ctx, CS_E_INVALID_ARGUMENT, "detect not run");
  if (ctx->streaming && inst < ctx->stream_stopped_prior.size() && ctx->stream_stopped_prior[inst]) {
    if (n) *n = 0;  // the stream stopped at an earlier NonPositiveLatency
    return CS_OK;
  }
  const uint64_t a0 = ctx->alert_off[inst], na_all = ctx->alert_off[inst + 1] - a0;
  const uint64_t bad = ctx->h_inst[inst].first_bad_record;
  if (!buf && bad == UINT64_MAX) {  // a count query: no truncation to apply
    if (n) *n = na_all;
    return CS_OK;
  }
  std::vector<cs_alert> all(na_all);
  if (na_all) {
    auto* d = dev<cs_alert>(ctx->d_scratch, na_all);
    if (!d) return fail(ctx, CS_E_CUDA, "cudaMalloc(alerts)");
    DevConfig cfg{ctx->cyc, ctx->ctl, 0.0};
    launch_gather_alerts(make_buffers(ctx), cfg, inst, a0, na_all, d, ctx->stream);
    CS_CUDA(cudaMemcpyAsync(all.data(), d, na_all * sizeof(cs_alert), cudaMemcpyDeviceToHost,
                            ctx->stream));
    CS_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  if (ctx->given_run)
    for (auto& a : all) a.cycle = ctx->given[a.cycle].index;
  // monitor_loop stops at the first NonPositiveLatency (main.cpp:162)
  uint64_t na = 0;
  while (na < na_all && all[na].record_index < bad) ++na;
  if (n) *n = na;
  if (!buf) return CS_OK;
  if (cap < na) return fail(ctx, CS_E_INVALID_ARGUMENT, "buffer too small");
  std::copy(all.begin(), all.begin() + na, buf);
  return CS_OK;
}

int cs_redetect(cs_ctx* ctx, const cs_control_config* control) {
  if (!ctx || !control || !ctx->ran) return CS_E_INVALID_ARGUMENT;
  if (ctx->streaming) return fail(ctx, CS_E_UNSUPPORTED, "cs_redetect is not available mid-stream");
  if (!(ctx->last_mask & (CS_RUN_SCORE | CS_RUN_DETECT)))
    return fail(ctx, CS_E_INVALID_ARGUMENT, "cs_redetect needs a scored run");
  if (control->strategy < 0 || control->strategy > 2 || control->window == 0)
    return fail(ctx, CS_E_CONFIG, "invalid control config");
  const uint32_t n_inst = ctx->n_inst;
  // the limits come from the models the last run scored with (mt_ids), not
  // from the bindings now: a model loaded or rebound since would otherwise
  // mix its limits with the old model's residuals
  if (ctx->mt_ids.size() != n_inst || ctx->h_models.size() != n_inst)
    return fail(ctx, CS_E_INVALID_ARGUMENT, "cs_redetect needs the model table of the last run");
  CS_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  ctx->ctl = *control;
  ctx->mt_valid = false;  // the table below gets this config's limits
  for (uint32_t i = 0; i < n_inst; ++i) {
    const PackedModel* pm = ctx->model_store[ctx->mt_ids[i]];
    ctx->h_models[i].ucl = ctx->ctl.strategy == CS_DYNAMIC_WINDOW
                               ? ucl_from_stats_host(pm->mu, pm->sigma, ctx->ctl)
                               : ctx->ctl.fixed_threshold;
    ctx->h_inst[i].n_alerts = 0;
  }
  CS_CUDA(cudaMemcpyAsync(ctx->d_models.p, ctx->h_models.data(), n_inst * sizeof(DevModel),
                          cudaMemcpyHostToDevice, s));
  CS_CUDA(cudaMemcpyAsync(ctx->d_inst.p, ctx->h_inst.data(), n_inst * sizeof(InstState),
                          cudaMemcpyHostToDevice, s));
  DevConfig cfg{ctx->cyc, ctx->ctl, 0.0};
  launch_detect(make_buffers(ctx), cfg, ctx->n_records, s, &ctx->launches);
  CS_CUDA(cudaMemcpyAsync(ctx->alert_off.data(), ctx->d_alert_off.p, (n_inst + 1) * 8,
                          cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaStreamSynchronize(s));
  ctx->last_mask |= CS_RUN_DETECT;
  return CS_OK;
}

// StrategyMetrics from the device counts (tp, fp, fn, tn, alerts, lag sum,
// intervals): detector.cpp:193-222, same double arithmetic
static void fill_metrics(const unsigned long long* h, int32_t strategy, cs_strategy_metrics* out) {
  cs_strategy_metrics m{};
  m.strategy = strategy;
  m.tp = h[0];
  m.fp = h[1];
  m.fn = h[2];
  m.tn = h[3];
  m.alerts = h[4];
  const double tp = static_cast<double>(h[0]), fp = static_cast<double>(h[1]);
  const double fn = static_cast<double>(h[2]), tn = static_cast<double>(h[3]);
  m.precision = tp + fp > 0.0 ? tp / (tp + fp) : 0.0;
  m.recall = tp + fn > 0.0 ? tp / (tp + fn) : 0.0;
  m.f1 = m.precision + m.recall > 0.0 ? 2.0 * m.precision * m.recall / (m.precision + m.recall)
                                      : 0.0;
  m.fpr = fp + tn > 0.0 ? fp / (fp + tn) : 0.0;
  m.mean_lag = h[6] > 0 ? static_cast<double>(h[5]) / static_cast<double>(h[6]) : 0.0;
  *out = m;
}

// Detector::step over a caller's residual stream (detector.cpp:85-130) and
// evaluate_strategy (166-224) on the device, with the run's kernels
// (k_detect_flags / k_detect_scatter / k_eval_strategy) on a one-instance
// table whose record t is stream sample t.
int cs_detect_residuals(cs_ctx* ctx, const double* residuals, uint64_t n, const cs_control_config* ctl,
                        double dynamic_ucl, const uint8_t* labels, double* statistic, uint8_t* flags,
                        cs_strategy_metrics* metrics) {
  if (!ctx || !ctl || (n && !residuals)) return CS_E_INVALID_ARGUMENT;
  if (ctl->strategy < 0 || ctl->strategy > 2 || ctl->window == 0)
    return fail(ctx, CS_E_CONFIG, "invalid control config");
  if (metrics && (!labels || n == 0))
    return fail(ctx, CS_E_NO_LABELS, "labeled stream is empty or label count mismatches");
  CS_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const uint64_t n1 = std::max<uint64_t>(1, n);
  DetScratch& d = ctx->det;
  if (!dev<double>(d.resid, n1) || !dev<double>(d.stat, n1) || !dev<uint8_t>(d.flags, n1) ||
      !dev<uint64_t>(d.rec_off, 2) || !dev<uint64_t>(d.rec_cycle, n1) || !dev<uint64_t>(d.cyc_off, 2) ||
      !dev<uint64_t>(d.alert_rec, n1) || !dev<uint64_t>(d.alert_off, 2) ||
      !dev<uint64_t>(d.block_tmp, n1 / 256 + 16) || !dev<InstState>(d.inst, 1) ||
      !dev<DevModel>(d.model, 1) || !dev<uint8_t>(d.labels, n1) || !dev<unsigned long long>(d.out, 8))
    return fail(ctx, CS_E_CUDA, "cudaMalloc(detect)");
  const uint64_t off[2] = {0, n};
  std::vector<uint64_t> iota(n);
  for (uint64_t k = 0; k < n; ++k) iota[k] = k;
  InstState st{};
  st.first_bad_record = UINT64_MAX;
  DevModel m{};
  m.ucl = ctl->strategy == CS_DYNAMIC_WINDOW ? dynamic_ucl : ctl->fixed_threshold;
  if (n) {
    CS_CUDA(cudaMemcpyAsync(d.resid.p, residuals, n * 8, cudaMemcpyHostToDevice, s));
    CS_CUDA(cudaMemcpyAsync(d.rec_cycle.p, iota.data(), n * 8, cudaMemcpyHostToDevice, s));
  }
  CS_CUDA(cudaMemcpyAsync(d.rec_off.p, off, 16, cudaMemcpyHostToDevice, s));
  CS_CUDA(cudaMemsetAsync(d.cyc_off.p, 0, 16, s));
  CS_CUDA(cudaMemcpyAsync(d.inst.p, &st, sizeof st, cudaMemcpyHostToDevice, s));
  CS_CUDA(cudaMemcpyAsync(d.model.p, &m, sizeof m, cudaMemcpyHostToDevice, s));
  DevBuffers b{};
  b.n_inst = 1;
  b.rec_off = static_cast<uint64_t*>(d.rec_off.p);
  b.rec_cycle = static_cast<uint64_t*>(d.rec_cycle.p);
  b.rec_resid = static_cast<double*>(d.resid.p);
  b.rec_stat = static_cast<double*>(d.stat.p);
  b.rec_flags = static_cast<uint8_t*>(d.flags.p);
  b.alert_rec = static_cast<uint64_t*>(d.alert_rec.p);
  b.alert_off = static_cast<uint64_t*>(d.alert_off.p);
  b.block_tmp = static_cast<uint64_t*>(d.block_tmp.p);
  b.inst = static_cast<InstState*>(d.inst.p);
  b.models = static_cast<const DevModel*>(d.model.p);
  b.cyc_off = static_cast<const uint64_t*>(d.cyc_off.p);
  DevConfig cfg{ctx->cyc, *ctl, 0.0};
  launch_detect(b, cfg, n, s, &ctx->launches);
  if (statistic && n) CS_CUDA(cudaMemcpyAsync(statistic, d.stat.p, n * 8, cudaMemcpyDeviceToHost, s));
  if (flags && n) CS_CUDA(cudaMemcpyAsync(flags, d.flags.p, n, cudaMemcpyDeviceToHost, s));
  unsigned long long h[8] = {0};
  if (metrics) {
    CS_CUDA(cudaMemcpyAsync(d.labels.p, labels, n, cudaMemcpyHostToDevice, s));
    CS_CUDA(cudaMemsetAsync(d.out.p, 0, sizeof h, s));
    launch_eval_strategy(b, 0, static_cast<const uint8_t*>(d.labels.p), n, ctl->warmup,
                         static_cast<unsigned long long*>(d.out.p), s);
    CS_CUDA(cudaMemcpyAsync(h, d.out.p, sizeof h, cudaMemcpyDeviceToHost, s));
  }
  CS_CUDA(cudaStreamSynchronize(s));
  CS_CUDA(cudaGetLastError());
  if (metrics) fill_metrics(h, ctl->strategy, metrics);
  return CS_OK;
}

int cs_evaluate_strategy(cs_ctx* ctx, uint32_t inst, const uint8_t* labels, uint64_t n_labels,
                         cs_strategy_metrics* out) {
  if (!ctx || !out || !ctx->ran || inst >= ctx->n_inst || (n_labels && !labels))
    return CS_E_INVALID_ARGUMENT;
  if (!(ctx->last_mask & CS_RUN_DETECT)) return fail(ctx, CS_E_INVALID_ARGUMENT, "detect not run");
  const uint64_t nr = ctx->rec_off[inst + 1] - ctx->rec_off[inst];
  if (nr == 0 || n_labels == 0)
    return fail(ctx, CS_E_NO_LABELS, "labeled stream is empty or label count mismatches");
  CS_CUDA(cudaSetDevice(ctx->device));
  DevBuf dl, dout;
  auto* d_labels = static_cast<uint8_t*>(dl.get(n_labels));
  auto* d_out = static_cast<unsigned long long*>(dout.get(7 * 8));
  if (!d_labels || !d_out) return fail(ctx, CS_E_CUDA, "cudaMalloc(eval)");
  CS_CUDA(cudaMemcpyAsync(d_labels, labels, n_labels, cudaMemcpyHostToDevice, ctx->stream));
  CS_CUDA(cudaMemsetAsync(d_out, 0, 7 * 8, ctx->stream));
  launch_eval_strategy(make_buffers(ctx), inst, d_labels, n_labels, ctx->ctl.warmup, d_out,
                       ctx->stream);
  unsigned long long h[7];
  CS_CUDA(cudaMemcpyAsync(h, d_out, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  CS_CUDA(cudaStreamSynchronize(ctx->stream));
  fill_metrics(h, ctx->ctl.strategy, out);
  return CS_OK;
}

int cs_set_option(cs_ctx* ctx, int option, int64_t value) {
  if (!ctx) return CS_E_INVALID_ARGUMENT;
  if (option == CS_OPT_FUSED) {
    ctx->allow_fused = value != 0;
    return CS_OK;
  }
  if (option == CS_OPT_TRAVERSAL) {
    ctx->no_lut = value != 0;
    ctx->mt_valid = false;  // the per-instance model table carries the choice
    return CS_OK;
  }
  if (option == CS_OPT_PHASE_TIMINGS) {
    if (value < -1 || value > 2) return fail(ctx, CS_E_INVALID_ARGUMENT, "phase timings: -1, 0, 1 or 2");
    ctx->phase_timings = static_cast<int>(value);
    return CS_OK;
  }
  if (option == 95) {  // testing: 1 scores in k_score_lut_flat instead of during record compaction
    ctx->no_fused_score = value != 0;
    return CS_OK;
  }
  if (option == 96) {  // tuning: events per single-read segmentation range (0 = auto)
    ctx->opt_range_events = value;
    return CS_OK;
  }
  if (option == 97) {  // tuning: L2 prefetch lookahead in ranges (-1 = the grid's warps, 0 = the claimed range only)
    ctx->opt_prefetch = value;
    return CS_OK;
  }
  if (option == 98) {  // profiling: multi-kernel reduce variant
    ctx->reduce_variant = static_cast<int>(value);
    return CS_OK;
  }
  if (option == 99) {  // testing: skew the speculated slot counts by `value` (the next run must notice)
    if (ctx->pred_cyc_off.size() >= 2) ctx->pred_cyc_off.back() += static_cast<uint64_t>(value);
    return CS_OK;
  }
  return fail(ctx, CS_E_INVALID_ARGUMENT, "unknown option");
}

int cs_host_alloc(size_t bytes, void** out) {
  if (!out) return CS_E_INVALID_ARGUMENT;
  if (cudaHostAlloc(out, bytes, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    return CS_E_NO_DEVICE;
  }
  return CS_OK;
}

int cs_host_free(void* p) {
  if (p) cudaFreeHost(p);
  return CS_OK;
}

int cs_get_timings(cs_ctx* ctx, double* ms, size_t cap, size_t* n, char* names, size_t names_cap) {
  if (!ctx) return CS_E_INVALID_ARGUMENT;
  if (n) *n = ctx->timed.size();
  std::string all;
  for (size_t k = 0; k < ctx->timed.size(); ++k) {
    float t = 0.f;
    cudaEventElapsedTime(&t, ctx->ev[ctx->timed[k].second.first], ctx->ev[ctx->timed[k].second.second]);
    if (ms && k < cap) ms[k] = t;
    if (k) all += ",";
    all += ctx->timed[k].first;
  }
  if (names && names_cap) {
    std::strncpy(names, all.c_str(), names_cap - 1);
    names[names_cap - 1] = 0;
  }
  return CS_OK;
}

int cs_get_launch_count(cs_ctx* ctx, uint64_t* n) {
  if (!ctx || !n) return CS_E_INVALID_ARGUMENT;
  *n = ctx->launches;
  return CS_OK;
}

double cs_ucl_from_stats(double mu, double sigma, const cs_control_config* cfg) {
  return ucl_from_stats_host(mu, sigma, *cfg);
}

int cs_compute_ucl(const double* r, size_t n, double k, double theta_max, double min_ucl,
                   size_t min_n, double* out) {
  // detector.cpp:41-55, two-pass sample variance
  if (n < min_n) return CS_E_INSUFFICIENT_CALIBRATION;
  double mean = 0.0;
  for (size_t i = 0; i < n; ++i) mean += r[i];
  mean /= static_cast<double>(n);
  double var = 0.0;
  for (size_t i = 0; i < n; ++i) var += (r[i] - mean) * (r[i] - mean);
  var /= static_cast<double>(n - 1);
  *out = std::max(std::min(mean + k * std::sqrt(var), theta_max), min_ucl);
  return CS_OK;
}

}  // extern "C"
