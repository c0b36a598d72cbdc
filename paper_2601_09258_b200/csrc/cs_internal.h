// cs_internal.h — shared declarations between the host runtime (cs_api.cpp)
// and the sm_100a kernels (cs_kernels.cu).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "cyclescope_b200.h"

namespace csb {

// ------------------------------------------------------------ tiling
constexpr int kScanThreads = 512;               // 16 warps
constexpr int kTileEvents = 1024;               // 32 KiB tile, one TMA bulk copy
constexpr int kSmemNames = 512;                 // name stats staged in smem
constexpr int kMaxFeatures = 8;
constexpr int kMaxTreeDepth = 24;  // bounded in practice by the layout size (cs_load_model)
constexpr uint64_t kSampleEvents = 1u << 18;    // anchor-guess sample per instance (verified by the full pass)

// name-stat accumulator (per instance x name); exact integer moments
struct NameStat {
  unsigned long long count;
  unsigned long long sum;      // sum of durations, two's complement int64
  unsigned long long sumsq_lo; // unsigned 128-bit sum of squares
  unsigned long long sumsq_hi;
  unsigned long long span_count;  // Spans of this name in any category
  unsigned long long pad[3];
};

// per-instance device state
struct InstState {
  uint32_t guess;          // speculated anchor name id (UINT32_MAX none)
  uint32_t anchor;         // final anchor name id (UINT32_MAX: none)
  uint32_t redo;           // anchors compacted for a different name
  uint32_t ambiguous;      // ranking needs the ordered fold
  uint32_t no_anchor;      // NoAnchorFound
  uint32_t n_candidates;
  unsigned long long n_anchors;      // anchor occurrences compacted (for `anchor`)
  unsigned long long n_unknown;      // cycles whose local stage is Unknown
  unsigned long long first_bad_record;
  unsigned long long n_records;
  unsigned long long n_alerts;
  uint32_t fixed_anchor;   // streaming: `guess` is this instance's fixed anchor
  uint32_t unsorted;       // the event scan saw start_ts decrease (not canonical order)
  unsigned long long first_missing_record;  // FeatureMismatch: a model extra the record lacks
};

// flattened model in complete-binary-tree layout (see pack_model)
// feature ids in DevModel: CS_F_* (0..4), kFeatExtra + key for a record extra,
// kFeatMissing for an extra name the uploaded trace has no key for
constexpr int32_t kFeatExtra = 16;
constexpr int32_t kFeatMissing = 15;
struct DevModel {
  uint32_t n_trees;
  uint32_t depth;          // padded depth D: 2^D-1 internal, 2^D leaves per tree
  uint32_t n_features;
  uint32_t degenerate;
  int32_t feature_ids[kMaxFeatures];
  double base, lr, floor_, mu, sigma, ucl;
  // device pointers (SoA over trees): thr[t*(2^D-1)+n], feat[t*(2^D-1)+n],
  // leaf[t*2^D+l]
  const double* thr;       // f64 thresholds (fallback compare path)
  const long long* thr_i;  // floor(thr): exact compare for integer-valued x
  const uint8_t* feat;
  const double* leaf;      // fl(learning_rate * leaf value), as the reference adds
  uint64_t smem_bytes;     // bytes of thr_i+leaf+feat when staged
  // compiled ensemble (n_features <= 2): lut[k1 * (lut_n[0]+1) + k0]
  const double* lut;
  const double* lut_thr[2];
  uint32_t lut_n[2];
};

// Streaming (micro-batch) state carried per instance across cs_run calls:
// the detector's last W-1 residuals, samples seen, flagged state, episode
// count and the number of cycles already emitted.
// Per-instance state carried across micro-batches.  The histories live in
// window-sized per-instance rows beside it (DevBuffers::s_hist / s_dur /
// s_gap): any detector window and any stage window.
struct StreamCarry {
  unsigned long long seen;
  unsigned long long episodes;
  unsigned long long cycle_off;
  uint32_t n_hist;     // residuals carried for the detector window (oldest first)
  uint32_t prev_flag;
  // stage heuristic (cycles.cpp:204-250): counts of the carried durations /
  // gaps, most recent first
  uint32_t n_dur, n_gap;
  long long last_aend;
  uint32_t has_prev, pad;
};

struct DevConfig {
  cs_cycle_config cyc;
  cs_control_config ctl;
  double limit_unused;
};

// all device pointers of one run
struct DevBuffers {
  const cs_event* ev;
  const cs_workload* wl;
  const cs_name_info* names;
  uint32_t n_names;
  uint32_t n_inst;
  const uint64_t* inst_off;     // n_inst+1 event offsets
  // tiles over events (instance-aligned)
  const uint32_t* tile_inst;
  const uint64_t* tile_begin;   // n_tiles+1 (tile t = [begin[t], end[t]) )
  const uint64_t* tile_end;
  const uint32_t* inst_first_tile;
  uint32_t n_tiles;
  NameStat* stats;              // n_inst * n_names
  InstState* inst;
  uint64_t* tile_cnt;           // anchors per tile (tile-local compaction)
  uint64_t* tile_pref;          // exclusive prefix of tile_cnt, n_tiles+1
  uint64_t* scan_tmp;           // block sums of the multi-CTA scan (n_tiles/1024 + 2)
  // anchors (capacity = events; instance i at inst_off[i])
  uint64_t* a_pos;
  int64_t* a_start;
  int64_t* a_end;
  // cycles (instance i at cyc_off[i])
  const uint64_t* cyc_off;      // n_inst+1
  uint64_t n_cycles;
  int64_t* c_start;
  int64_t* c_end;
  uint64_t* c_apos;
  int64_t* c_aend;
  uint64_t* c_first;
  uint64_t* c_last;
  uint32_t* c_inst;
  uint8_t* c_stage;             // final stage
  uint8_t* c_local;             // local (args/keyword) stage
  int32_t* c_wl;                // workload index, -1 no carrier, -2 invalid carrier
  int64_t* c_comp;              // n_cycles x n_phases
  int64_t* c_beta_tot;          // n_cycles x n_beta
  double* c_coll;               // n_cycles x n_comm
  uint8_t* c_coll_n;            // contributions per (cycle, comm slot)
  // records (instance i at rec_off[i], device-computed)
  uint64_t* rec_off;            // n_inst+1
  uint64_t* rec_cycle;          // record -> global cycle index
  double* rec_pred;
  double* rec_resid;
  double* rec_stat;
  uint8_t* rec_flags;           // bit0 armed, bit1 flagged, bit2 alert
  uint64_t* alert_rec;          // alert -> record index
  uint64_t* alert_off;          // n_inst+1
  uint64_t* block_tmp;          // scratch for scans
  const DevModel* models;       // per instance (device array)
  // counter-weighted mu (CS_RUN_MU)
  const int8_t* series_slot;    // per name: metric slot of a counter series name, -1
  const int8_t* class_metric;   // per name: metric slot its class maps to, -1
  uint32_t n_metrics;
  uint64_t* m_off;              // [metric][tile] counts, then exclusive offsets (+ total)
  int64_t* s_ts;                // samples, metric-major, instances in tile order
  double* s_val;
  double* c_mu;                 // n_cycles x n_beta
  uint8_t* c_mu_has;
  StreamCarry* stream;          // per instance, null when not streaming
  const double* s_hist;         // [n_inst][s_hw]: carried residuals (oldest first)
  const double* s_dur;          // [n_inst][s_sw]: carried non-Prefill durations (most recent first)
  const double* s_gap;          // [n_inst][s_sw]: carried gaps
  uint32_t s_hw, s_sw;
  unsigned int* any_unknown;    // set by the reduces when any cycle's local stage is Unknown
  // record extras (cs_upload_extras): side table sorted by event, and the
  // per-record values / presence (n_records x n_extra_keys)
  const cs_extra_ref* extra_refs;
  uint64_t n_extra_refs;
  const cs_extra_value* extra_vals;
  uint32_t n_extra_keys;
  double* rec_extra;
  uint8_t* rec_extra_has;
};

// Single-read segmentation (k_segment_range, CS_OPT_FUSED): ranges of <= 4
// instance-aligned tiles claimed in order; per range the events are scanned
// (moments, order check, anchor compaction) and the range's cycles reduced
// right after, from L2.  Cycle slots = global anchor ranks (decoupled
// look-back over ranges), so each instance's last anchor leaves one hole slot
// (c_wl = kHoleWl, empty event range) after its cycles.
struct SegMeta {
  const uint64_t* range_begin;   // event index
  const uint64_t* range_end;
  const uint32_t* range_inst;
  uint32_t n_ranges;
  unsigned long long* lb_state;  // per range: look-back flag | value (zeroed per run)
  uint64_t* range_prefix;        // per range: global anchor rank of its first anchor
  unsigned int* ticket;          // zeroed per run
  unsigned int* overflow;        // zeroed per run; set when slots exceed `cap`
  uint64_t cap;                  // cycle slot capacity
  uint32_t prefetch_ahead;       // also prefetch range r + this into L2 (0xffffffff: the grid's warps)
};
constexpr int32_t kHoleWl = -3;
constexpr uint64_t kSegCycles = 31;  // target cycles per range (one warp, one cycle per lane; swept 28-33 on configs[1])

// launchers (cs_kernels.cu); all asynchronous on `s`
void launch_scan_events(const DevBuffers& b, const DevConfig& cfg, int mode, bool sample,
                        const uint32_t* list, uint32_t n_list, cudaStream_t s,
                        uint64_t* launches);
void launch_tile_prefix(const DevBuffers& b, cudaStream_t s, uint64_t* launches);
void launch_tile_order(const DevBuffers& b, cudaStream_t s, uint64_t* launches);
void launch_rank(const DevBuffers& b, const DevConfig& cfg, int final_pass, cudaStream_t s,
                 uint64_t* launches);
void launch_fold(const DevBuffers& b, const DevConfig& cfg, const uint32_t* pairs_inst,
                 const uint32_t* pairs_name, uint32_t n_pairs, double* out_scores,
                 cudaStream_t s, uint64_t* launches);
void launch_bounds(const DevBuffers& b, cudaStream_t s, uint64_t* launches);
void launch_cycle_reduce_tpc(const DevBuffers& b, const DevConfig& cfg, int do_beta,
                             cudaStream_t s, uint64_t* launches, int variant);
void launch_segment_range(const DevBuffers& b, const DevConfig& cfg, const SegMeta& sm, int do_beta,
                          cudaStream_t s, uint64_t* launches);
// per instance from the range prefixes: n_anchors (InstState) and slot offsets
void launch_range_inst(const DevBuffers& b, const SegMeta& sm, const uint32_t* inst_first_range,
                       uint64_t* slot_off, cudaStream_t s, uint64_t* launches);
// dynamic shared memory of k_segment_range for this configuration; -1 when the
// slot counts need the wide reduce (the fused pass is then not used)
int segment_range_smem(const DevConfig& cfg, int do_beta, uint32_t n_names);
// K4' (k_stage_jacobi): the stage heuristic over chunks of cycle slots with
// Jacobi refinement; st[0] = c_stage (holding the local stages), st[1] a
// scratch copy; *final_parity = index of the array with the result
// (0xffffffff: no fixed point within max_iter); final_parity[1] iterations
// run, [2] = 1 when K4b (k_stage_blocks) reached the fixed point, [3] K4b's
// out-of-range flag.
struct StageMeta {
  uint8_t* st[2];
  uint32_t n_chunks;
  int32_t* changed_iter;      // per chunk, zero-initialised to -1
  uint64_t* lookback_lo;      // per chunk
  unsigned int* any_changed;  // [2], zeroed
  unsigned int* bar_count;    // zeroed
  unsigned int* bar_gen;
  unsigned int* final_parity;
  int max_iter;
};
#ifndef CS_STAGE_CHUNK
#define CS_STAGE_CHUNK 256
#endif
constexpr uint32_t kStageChunkCycles = CS_STAGE_CHUNK;  // stage heuristic chunk (cycle slots)
// K4b (k_stage_blocks, windows <= 32, not streaming) runs first; K4' only
// when K4b could not (final_parity[2] == 0)
int launch_stage_heuristic(const DevBuffers& b, const DevConfig& cfg, const StageMeta& m, cudaStream_t s,
                           uint64_t* launches);
// record compaction; fuse_score != 0 also scores every record it writes
// (cell-table models, no record extras; first_bad / first_missing record are
// then absolute record indices).  Returns whether it scored.
bool launch_records(const DevBuffers& b, const DevConfig& cfg, int fuse_score, cudaStream_t s,
                    uint64_t* launches);
// per record: the extras of its cycle (last event carrying each key wins)
void launch_record_extras(const DevBuffers& b, uint64_t n_records_cap, cudaStream_t s, uint64_t* launches);
void launch_score(const DevBuffers& b, const DevConfig& cfg, uint64_t n_records_total,
                  const uint64_t* h_rec_off, const int* h_model_of_inst, const DevModel* h_models,
                  cudaStream_t s, uint64_t* launches);
void launch_detect(const DevBuffers& b, const DevConfig& cfg, uint64_t n_records_total,
                   cudaStream_t s, uint64_t* launches);
void launch_freq_hist(const cs_event* ev, uint64_t begin, uint64_t end, int64_t t0,
                      int64_t bin_ns, uint64_t bins, double* hist, cudaStream_t s,
                      uint64_t* launches);
void launch_freq_autocorr(const double* hist, uint64_t bins, double* acc, cudaStream_t s,
                          uint64_t* launches);
void launch_gpu_kernel_extent(const cs_event* ev, uint64_t begin, uint64_t end,
                              unsigned long long* out3, cudaStream_t s, uint64_t* launches);
void launch_freq_cycles(const cs_event* ev, uint64_t begin, uint64_t end, int64_t t0,
                        int64_t period, uint64_t n, uint64_t cyc_base, const DevBuffers& b,
                        uint32_t inst, cudaStream_t s, uint64_t* launches);

// device copies of a cs_wire_batch (cs_upload_wire)
struct WireDev {
  const uint8_t* codes;
  const uint16_t* dt_lo;
  const uint8_t* dt_hi;
  const uint32_t* dict;
  uint32_t n_dict;
  const cs_wire_block* blocks;
  const uint16_t* dur_lo;
  const uint8_t* dur_hi;
  const uint8_t* pay8;
  const uint16_t* pay16;
  const double* values;
  const cs_event* escapes;
};
void launch_wl32_expand(const uint32_t* wl32, uint64_t n, cs_workload* out, cudaStream_t s);
void launch_wire_expand(const WireDev& w, const uint64_t* tile_begin, const uint64_t* tile_end,
                        uint32_t n_tiles, cs_event* out, cudaStream_t s);
void launch_stream_keep(const DevBuffers& b, uint64_t* keep, cudaStream_t s);
void launch_stream_count(const cs_event* fresh, const uint64_t* meta, const uint32_t* anchor, uint32_t n_inst,
                         uint64_t n_new, uint64_t* out, cudaStream_t s);
// streaming batch assembly: per instance i (meta[4i..4i+3] = dst offset, tail
// start in prev, tail length, new-event offset) out[dst..] = prev tail, then
// the instance's new events
void launch_stream_assemble(const cs_event* prev, const cs_event* fresh, const uint64_t* meta,
                            uint32_t n_inst, uint64_t total, cs_event* out, cudaStream_t s);
void launch_counter_series(const DevBuffers& b, cudaStream_t s, uint64_t* launches);
void launch_counter_scatter(const DevBuffers& b, cudaStream_t s, uint64_t* launches);
void launch_cycle_mu(const DevBuffers& b, const DevConfig& cfg, cudaStream_t s, uint64_t* launches);
constexpr int kMaxMetrics = 16;
void launch_lut_build(const uint8_t* feat, const int32_t* rank, const double* leafp,
                      uint32_t n_trees, uint32_t D, double base, double floor_, uint32_t n0,
                      uint64_t cells, double* lut, cudaStream_t s);
void launch_exclusive_scan(uint64_t* v, uint64_t n, uint64_t* total, uint64_t* tmp, cudaStream_t s,
                           uint64_t* launches);
// K0 (cs_sort.cu): stable per-instance sort by (start_ts, event_id) (ids may be
// null: input position breaks ties); scratch = 4n u64, hist = 256 * ceil(n /
// 4096) u64, hist_tmp = its scan scratch, extent = 4 u64.  Returns 0 on success.
int sort_events_device(const cs_event* in, const uint64_t* ids, const uint64_t* d_off,
                       uint32_t n_inst, uint64_t n, cs_event* out, uint64_t* order,
                       unsigned long long* scratch, uint64_t* hist, uint64_t* hist_tmp,
                       unsigned long long* extent, cudaStream_t s, uint64_t* launches);
constexpr uint64_t kSortTile = 4096;
void launch_eval_strategy(const DevBuffers& b, uint32_t inst, const uint8_t* labels,
                          uint64_t n_labels, uint64_t warmup, unsigned long long* out,
                          cudaStream_t s);
void launch_stream_update(const DevBuffers& b, const DevConfig& cfg, StreamCarry* out, double* out_hist,
                          double* out_dur, double* out_gap, int detected,
                          cudaStream_t s);
void launch_gather_records(const DevBuffers& b, const DevConfig& cfg, uint32_t inst, uint64_t r0,
                           uint64_t nr, int scored, int det, cs_record* out, cudaStream_t s);
void launch_gather_alerts(const DevBuffers& b, const DevConfig& cfg, uint32_t inst, uint64_t a0,
                          uint64_t na, cs_alert* out, cudaStream_t s);
void launch_gather_alerts_all(const DevBuffers& b, const DevConfig& cfg, uint64_t n_all, cs_alert* out,
                              cudaStream_t s);

}  // namespace csb
