/*
 * cyclescope_b200.h — C ABI of the B200-native trace-analysis core.
 *
 * This is the drop-in boundary for the reference's analysis hot path
 * (`/root/reference/proj/include/cyclescope/{cycles,detector,baseline,rca}.hpp`).
 * The reference exposes that path as C++ functions over `Trace`; it has no
 * FFI.  The entry points below are what a C++ shim (or cgo/ctypes/JNI
 * binding) re-implementing those functions binds to.  Each entry cites the
 * reference interface it replaces.
 *
 * Conventions
 *  - Every function returns an int status: CS_OK (0) or a CS_E_* code whose
 *    machine-readable type string (cs_status_type) equals the reference's
 *    EngineError::type() (errors.hpp:12-85).  No exception crosses the ABI;
 *    the message of the last error is available from cs_last_error(ctx).
 *  - Inputs are borrowed, plain pointers + sizes.  Outputs go to
 *    caller-owned buffers with an explicit capacity and a size_t* count.
 *  - Events are in the reference's canonical order (start_ts, event_id)
 *    (trace.hpp:110-113).  All event indices returned (first_event,
 *    last_event, anchor position) are indices into that order, i.e. into the
 *    caller's Trace::events (cycles.hpp:71-73).
 *  - There is no CPU fallback: without a CUDA device every compute entry
 *    point returns CS_E_NO_DEVICE.
 */
#ifndef CYCLESCOPE_B200_H_
#define CYCLESCOPE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CS_ABI_VERSION 2

/* ------------------------------------------------------------------ status */
enum cs_status {
  CS_OK = 0,
  CS_E_INVALID_ARGUMENT = 1,   /* "invalid_argument" (ABI misuse)            */
  CS_E_NO_DEVICE = 2,          /* "no_device": no CUDA device / ext missing   */
  CS_E_CUDA = 3,               /* "cuda_error"                               */
  CS_E_NO_ANCHOR_FOUND = 4,    /* "no_anchor_found"        errors.hpp:41-43  */
  CS_E_MISSING_WORKLOAD = 5,   /* "missing_workload_args"  errors.hpp:44-46  */
  CS_E_FEATURE_MISMATCH = 6,   /* "feature_mismatch"       errors.hpp:50-52  */
  CS_E_NON_POSITIVE_LATENCY = 7, /* "non_positive_latency" errors.hpp:56-58  */
  CS_E_INSUFFICIENT_DATA = 8,  /* "insufficient_data"      errors.hpp:47-49  */
  CS_E_INSUFFICIENT_CALIBRATION = 9, /* "insufficient_calibration" 59-61     */
  CS_E_NO_LABELS = 10,         /* "no_labels"              errors.hpp:62-64  */
  CS_E_MODEL_FORMAT = 11,      /* "model_format_error"     errors.hpp:80-82  */
  CS_E_UNSUPPORTED = 12,       /* "unsupported": outside the device limits   */
  CS_E_CONFIG = 13,            /* "config_error"           errors.hpp:77-79  */
  CS_E_INTERNAL = 14,          /* "internal"                                 */
  CS_E_INSUFFICIENT_CYCLES = 15, /* "insufficient_cycles"  errors.hpp:68-70  */
  CS_E_NO_BEACONS = 16,         /* "no_beacons"             errors.hpp:26-28  */
  CS_E_INCONSISTENT_BEACONS = 17, /* "inconsistent_beacons" errors.hpp:29-31  */
  CS_E_ALREADY_CALIBRATED = 18  /* "already_calibrated"     errors.hpp:32-34  */
};

/* ------------------------------------------------------- event record (A1)
 * 32-byte record, 16-byte aligned: two 16-B vector loads per event.
 * Replaces TraceEvent (trace.hpp:67-81) + the std::map args the hot path
 * reads (arg_int/arg_string/arg_number, trace.cpp:76-101); the host interns
 * strings at ingest, the device never sees them.
 */
typedef struct cs_event {
  int64_t start_ts;   /* ns, canonical order key                          */
  int64_t duration;   /* ns for Span; for Counter: bit pattern of the f64
                         `value` arg (CS_EV_HAS_VALUE); 0 otherwise         */
  uint32_t name_id;   /* index into the name table (names interned in
                         lexicographic byte order, so name_id == lex rank)  */
  uint8_t kind;       /* cs_kind                                          */
  uint8_t category;   /* cs_category                                      */
  uint16_t flags;     /* CS_EV_* bits                                     */
  uint64_t payload;   /* low 32: workload-table index (CS_EV_HAS_BATCH)
                         high 32: collective slot (CS_EV_HAS_COMM)          */
} cs_event;

enum cs_kind { CS_SPAN = 0, CS_INSTANT = 1, CS_COUNTER = 2, CS_FLOW = 3 };
enum cs_category { /* trace.hpp:22-31 */
  CS_CAT_PYTHON_CALL = 0, CS_CAT_RUNTIME_API = 1, CS_CAT_GPU_KERNEL = 2,
  CS_CAT_MEM_COPY = 3, CS_CAT_OS_SCHED = 4, CS_CAT_NET_IO = 5,
  CS_CAT_COUNTER_TELEMETRY = 6, CS_CAT_COLLECTIVE_COMM = 7
};

/* forward_mode class of arg_string(e, forward_mode_key) after tolower
 * (cycles.cpp:205-220): none / contains prefill|extend / contains decode /
 * any other string (stops the first-forward_mode search, decides nothing). */
#define CS_EV_FM_MASK      0x0003u
#define CS_EV_FM_NONE      0u
#define CS_EV_FM_PREFILL   1u
#define CS_EV_FM_DECODE    2u
#define CS_EV_FM_OTHER     3u
#define CS_EV_HAS_BATCH    0x0004u /* arg_int(batch_size_key) present        */
#define CS_EV_WL_OK        0x0008u /* + input/output lens present, all >= 0  */
#define CS_EV_HAS_COMM     0x0010u /* CollectiveComm span w/ commHash + rank */
#define CS_EV_HAS_VALUE    0x0020u /* Counter with numeric `value`           */

/* One entry per batch-size carrier event.  input_len/output_len are
 * INT64_MIN when the arg is absent (MissingWorkloadArgs, cycles.cpp:264-267). */
typedef struct cs_workload { /* WorkloadFeatures (cycles.hpp:92-100) */
  int64_t batch;
  int64_t input_len;
  int64_t output_len;
} cs_workload;

/* Per interned name. Derived on the host from CycleConfig (cycles.hpp:18-43)
 * and the set of span names. */
typedef struct cs_name_info {
  uint32_t flags;      /* CS_NAME_* */
  int32_t phase;       /* index into CycleConfig::phase_functions, -1 none */
  int32_t beta_slot;   /* dense class slot for stage attribution, -1 none  */
  uint32_t metric;     /* 1 + name id of the counter series MetricMap maps this
                          class to (rca.cpp:55-69, RunConfig metric_map); 0 none */
} cs_name_info;
#define CS_NAME_PREFILL_KW 0x1u /* name contains a prefill keyword (174-179) */
#define CS_NAME_DECODE_KW  0x2u /* name contains a decode keyword            */

/* ------------------------------------------------------------- configs */
typedef struct cs_cycle_config { /* CycleConfig + PipelineOptions */
  int64_t anchor_hint_name;       /* name id, -1 = discover (cycles.hpp:20)
                                     -2 = hint given but not in name table */
  uint64_t min_anchor_calls;      /* 10 */
  double prefill_duration_factor; /* 3.0 */
  double prefill_gap_factor;      /* 2.0 */
  uint64_t stage_window;          /* 32 */
  uint64_t stage_min_history;     /* 8  */
  int64_t frequency_bin_ns;       /* 1'000'000 */
  int32_t n_phases;               /* |phase_functions| after dedup         */
  int32_t latency_phase;          /* PipelineOptions::latency_component as
                                     phase index; -1 = full cycle span      */
  int32_t include_prefill;        /* PipelineOptions::include_prefill       */
  int32_t n_beta_slots;           /* number of dense class slots            */
  int32_t n_comm_slots;           /* collective (name,comm,rank) slots      */
  int32_t monitor_from_cycle;     /* records (and the detector stream) start
                                     at this cycle index: evaluate_trial's
                                     train/monitor split (simkit.cpp:837-841) */
} cs_cycle_config;

enum cs_strategy { CS_FIXED_POINT = 0, CS_FIXED_WINDOW = 1, CS_DYNAMIC_WINDOW = 2 };

typedef struct cs_control_config { /* ControlConfig detector.hpp:25-34 */
  int32_t strategy;
  int32_t reserved;
  uint64_t window;         /* 10   */
  double fixed_threshold;  /* 0.15 */
  double sigma_k;          /* 3.0  */
  double theta_max;        /* 0.18 */
  double min_ucl;          /* 0.02 */
  uint64_t warmup;         /* 100  */
  double epsilon;          /* 1e-9 */
} cs_control_config;

/* Feature ids a model may request (main.cpp:59-78 features_by_name).  Any
 * other feature name is a record `extra` (the post_* args of the Full feature
 * set, cycles.cpp:392-405 / baseline.cpp:43-76), resolved by name against the
 * extras keys of the uploaded trace (cs_upload_extras) when a run scores. */
enum cs_feature { CS_F_BATCH = 0, CS_F_W_KV = 1, CS_F_INPUT_LEN = 2,
                  CS_F_OUTPUT_LEN = 3, CS_F_STAGE = 4, CS_F_EXTRA = -1 };

/* Flattened GbdtModel (gbdt.hpp:33-84) + LatencyModel stats (baseline.hpp:50-67).
 * Trees are concatenated node arrays; tree t owns nodes
 * [tree_offsets[t], tree_offsets[t+1]); child indices are tree-local. */
typedef struct cs_tree_node {
  int32_t feature;   /* -1 = leaf */
  int32_t left;
  int32_t right;
  int32_t reserved;
  double threshold;  /* go left iff x[feature] <= threshold */
  double value;      /* leaf output */
} cs_tree_node;

typedef struct cs_model {
  uint32_t n_features;
  uint32_t n_trees;
  const int32_t* feature_ids;     /* n_features cs_feature ids */
  const uint32_t* tree_offsets;   /* n_trees + 1 */
  const cs_tree_node* nodes;
  double base;
  double learning_rate;
  double prediction_floor;
  double mu_train;
  double sigma_train;
  int32_t degenerate;
  int32_t reserved;
  const char* const* feature_names; /* n_features names (NULL: ids only); needed
                                       for CS_F_EXTRA features */
} cs_model;

/* ------------------------------------------------------------- outputs */
enum cs_stage { CS_STAGE_PREFILL = 0, CS_STAGE_DECODE = 1, CS_STAGE_UNKNOWN = 2 };

typedef struct cs_cycle { /* Cycle (cycles.hpp:62-77) */
  uint64_t index;
  int64_t start_ts;
  int64_t end_ts;
  uint64_t anchor_pos;     /* canonical index of the anchor occurrence;
                              UINT64_MAX for frequency-fallback cycles */
  int64_t anchor_span_end;
  uint64_t first_event;
  uint64_t last_event;
  int32_t stage;
  int32_t workload_status; /* 0 ok, 1 no carrier, 2 carrier w/o lens/neg */
} cs_cycle;

typedef struct cs_record { /* CycleRecord (cycles.hpp:114-121) + ResidualSample
                              + StepResult (detector.hpp:43-73) */
  uint64_t cycle_index;
  int64_t start_ts;
  int64_t batch;
  int64_t input_len;
  int64_t output_len;
  double latency_s;
  double predicted_s;
  double residual;         /* ppe */
  double statistic;        /* E_t or window mean */
  int32_t stage;
  uint8_t armed;
  uint8_t flagged;
  uint8_t alert;
  uint8_t reserved;
  uint64_t episode_id;     /* valid when alert */
} cs_record;

typedef struct cs_alert { /* Alert (detector.hpp:52-63) */
  uint64_t cycle;
  int64_t ts;
  double smoothed_error;
  double limit;
  int32_t strategy;
  int32_t reserved;
  int64_t batch;
  int64_t input_len;
  int64_t output_len;
  uint64_t episode_id;
  uint64_t record_index;
} cs_alert;

typedef struct cs_anchor_candidate { /* AnchorCandidate (cycles.hpp:45-52) */
  uint32_t name_id;
  uint32_t reserved;
  uint64_t call_count;
  double mean_duration_ns;
  double duration_cv;
  double score;
  double periodicity;  /* 1 / (1 + CV of inter-start gaps) (cycles.cpp:76);
                          cs_get_candidates_exact only (NaN otherwise) */
} cs_anchor_candidate;

typedef struct cs_instance_summary {
  uint32_t anchor_name_id;   /* UINT32_MAX when frequency fallback used */
  int32_t status;            /* per-instance cs_status of the analysis    */
  uint64_t n_cycles;
  uint64_t n_records;
  uint64_t n_alerts;
  uint64_t first_bad_record; /* first record where monitor_loop stops: latency
                                <= 0 (NonPositiveLatency) or a model feature the
                                record lacks (FeatureMismatch); UINT64_MAX none */
  double ucl;                /* detector limit in force                   */
  int32_t used_frequency_fallback;
  int32_t anchor_ambiguous;  /* exact-stat ranking needed the ordered fold */
} cs_instance_summary;

/* ----------------------------------------------------------- context API */
typedef struct cs_ctx cs_ctx;

/* Stage mask for cs_run. */
#define CS_RUN_SEGMENT   0x1u  /* anchor + segment + classify + records  */
#define CS_RUN_BETA      0x2u  /* per-cycle class occupancy beta         */
#define CS_RUN_SCORE     0x4u  /* GBDT predict + ppe                     */
#define CS_RUN_DETECT    0x8u  /* control chart + alerts                 */
#define CS_RUN_ALL       0xFu
#define CS_RUN_GIVEN     0x20u /* use the cs_set_cycles table instead of anchor
                                  discovery + segmentation (one instance):
                                  local stage signals, workloads, components,
                                  beta / mu, records, score and detect run on
                                  the caller's cycles                      */
#define CS_RUN_CLASSIFY  0x40u /* with CS_RUN_GIVEN: classify_stages from
                                  scratch (cycles.cpp:190-254); without it the
                                  given cycles keep their stage            */
#define CS_RUN_MU        0x10u /* counter-weighted mu per (cycle, class):
                                  cycle_stats with a CounterTable
                                  (rca.cpp:97-106, 123-126); implies BETA  */

int cs_abi_version(void);
const char* cs_status_type(int status);

int cs_ctx_create(int device, cs_ctx** out);
void cs_ctx_destroy(cs_ctx* ctx);
const char* cs_last_error(const cs_ctx* ctx);

/* CycleConfig/PipelineOptions (cycles.hpp:18-43,123-128) and ControlConfig
 * (detector.hpp:25-34). */
int cs_set_config(cs_ctx* ctx, const cs_cycle_config* cycle,
                  const cs_control_config* control);

/* Name table: one entry per interned name id. */
int cs_set_name_table(cs_ctx* ctx, uint32_t n_names, const cs_name_info* names);

/* Upload a batch of monitored instances (events of instance i are
 * ev[inst_offsets[i] .. inst_offsets[i+1]) ).  H2D copy on the ctx stream;
 * host buffers may be pinned (cs_host_alloc) for full link bandwidth. */
int cs_upload(cs_ctx* ctx, uint32_t n_inst, const uint64_t* inst_offsets,
              const cs_event* ev, uint64_t n_workloads, const cs_workload* wl);
/* (n_workloads = 0 with wl = NULL keeps the previously uploaded workload table.) */

/* K0: canonical order on the device (Trace::sort_events, trace.cpp:103-105).
 * cs_upload / cs_upload_wire / cs_stream_push take events already in the
 * reference's canonical order (start_ts, event_id) per instance; cs_run
 * verifies it inside its first event pass (trace.cpp:107-109 is_sorted) and
 * returns CS_E_INVALID_ARGUMENT when an instance's start_ts ever decreases,
 * instead of producing wrong cycles.  cs_upload_unsorted accepts any order:
 * every instance's events are stably sorted on the device by (start_ts,
 * event_id) (event_ids NULL: the input position breaks ties, i.e. ids ascend
 * in input order), exactly the order sort_events gives.  All indices returned
 * afterwards (first_event, last_event, anchor_pos, ...) are canonical
 * positions; cs_get_order maps them back: buf[k] = the input position (within
 * the instance) of canonical position k. */
int cs_upload_unsorted(cs_ctx* ctx, uint32_t n_inst, const uint64_t* inst_offsets,
                       const cs_event* ev, const uint64_t* event_ids, uint64_t n_workloads,
                       const cs_workload* wl);
int cs_get_order(cs_ctx* ctx, uint32_t inst, uint64_t* buf, size_t cap, size_t* n);

/* ------------------------------------------------- wire format (host link)
 * Columnar wire format for the host->device leg: the H2D copy is what bounds
 * an end-to-end run, so the producer (ingest / collector) emits this instead
 * of cs_event and the device expands it in HBM (k_wire_expand).  Events are
 * grouped in instance-aligned blocks of CS_WIRE_BLOCK records (block b of
 * instance i covers events [inst_offsets[i] + b*CS_WIRE_BLOCK, ...)).
 *   codes[]      one byte per event: a dict code (< n_dict) or CS_WIRE_ESCAPE,
 *                | CS_WIRE_LONG_DT when the start_ts delta needs 17..24 bits;
 *   dt_lo[]      one u16 per event: the low 16 bits of dt = start_ts - the
 *                previous event's start_ts in the block (the block's first
 *                event: start_ts - blocks[b].base_ts, which the encoder makes
 *                0).  Events are canonically ordered, so dt >= 0;
 *   dt_hi[]      one byte per CS_WIRE_LONG_DT event: dt >> 16;
 *   dict[]       the packed name id (16 bits) | kind << 16 | category << 20 |
 *                CS_EV_* flags << 24 | CS_WIRE_WIDE (payload in pay16) of
 *                each code;
 *   dur_lo[], dur_hi[]  one 24-bit duration per Span in event order (low
 *                16 bits, high 8 bits);
 *   pay8[], pay16[]  one entry per event with CS_EV_HAS_COMM (collective
 *                slot = cs_event.payload >> 32) or CS_EV_HAS_BATCH (workload
 *                index - blocks[b].batch_base), in the column its code's
 *                CS_WIRE_WIDE bit selects;
 *   values[]     one f64 per Counter with CS_EV_HAS_VALUE;
 *   blocks[]     per block: base timestamp, batch_base, and the index of its
 *                first entry in every column;
 *   escapes[]    full cs_event, in event order, for records that do not fit
 *                (dt or span duration >= 2^24, negative duration, a non-Span
 *                non-value duration, info not in dict, payload out of range,
 *                both HAS_BATCH and HAS_COMM).  The next event's dt is taken
 *                from an escaped event's start_ts like any other;
 *   workloads32[]  optional: the workload table as (batch, input_len,
 *                output_len) u32 triples, 0xffffffff = absent (INT64_MIN). */
#define CS_WIRE_BLOCK 1024u
#define CS_WIRE_ESCAPE 0x7fu
#define CS_WIRE_LONG_DT 0x80u
#define CS_WIRE_MAX_DICT 127u
#define CS_WIRE_WIDE (1u << 30)
typedef struct cs_wire_block {
  int64_t base_ts;
  uint64_t dur, pay8, pay16, val, dt_hi, esc;  /* first entry of the block per column */
  uint32_t batch_base;
  uint32_t reserved;
} cs_wire_block;

typedef struct cs_wire_batch {
  const uint8_t* codes;          /* inst_offsets[n_inst] each */
  const uint16_t* dt_lo;
  const uint8_t* dt_hi;
  uint64_t n_dt_hi;
  const uint32_t* dict;          /* n_dict <= CS_WIRE_MAX_DICT */
  uint32_t n_dict;
  uint32_t reserved;
  const cs_wire_block* blocks;   /* n_blocks */
  const uint16_t* dur_lo;
  const uint8_t* dur_hi;
  uint64_t n_durations;
  const uint8_t* pay8;
  uint64_t n_pay8;
  const uint16_t* pay16;
  uint64_t n_pay16;
  const double* values;
  uint64_t n_values;
  const cs_event* escapes;
  uint64_t n_escapes;
  const uint32_t* workloads32;   /* NULL: the cs_upload_wire workload arguments */
  uint64_t n_workloads32;
} cs_wire_batch;

/* Upload a batch in the wire format (same instance layout and semantics as
 * cs_upload; expanded on the device into the same cs_event records).
 * cs_upload and cs_upload_wire return once the host->device copies have
 * completed (the host buffers may be reused); the expansion and everything
 * queued after it run asynchronously.  Two contexts whose uploads are issued
 * one after the other keep the host link busy while the other analyses.
 * With wire->workloads32 set, n_workloads / wl must be 0 / NULL. */
int cs_upload_wire(cs_ctx* ctx, uint32_t n_inst, const uint64_t* inst_offsets,
                   const cs_wire_batch* wire, uint64_t n_workloads, const cs_workload* wl);

/* Host encoder (multi-threaded) from cs_event to the wire format; the
 * producer side of cs_upload_wire.  Buffers are owned by the returned
 * object; cs_wire_view fills a cs_wire_batch pointing at them. */
typedef struct cs_wire_trace cs_wire_trace;
int cs_wire_pack(uint32_t n_inst, const uint64_t* inst_offsets, const cs_event* ev,
                 uint64_t n_workloads, const cs_workload* workloads, uint32_t n_threads,
                 cs_wire_trace** out);
int cs_wire_view(const cs_wire_trace* w, cs_wire_batch* out, uint64_t* n_blocks);
void cs_wire_free(cs_wire_trace* w);

/* ------------------------------------------- Chrome-trace JSON ingest
 * Native replacement of parse_trace_json (trace_io.cpp:162-206) + the
 * interning every exporter does: a Chrome-trace JSON document (an event array
 * or an object with "traceEvents") -> canonically ordered cs_event records,
 * event ids, names (lexicographic, packed NUL-separated), workload table and
 * (name, commHash, rank) collective slots.  Records parse in parallel on
 * n_threads host threads; semantics (number classification, duplicate keys,
 * args flattening, us -> ns rounding, fallback ids, skipped records) follow
 * the reference as built with nlohmann/json.  n_issues counts the reference's
 * ValidationIssue entries (an invalid document: empty trace, one issue). */
typedef struct cs_ingest_keys { /* CycleConfig arg keys (cycles.hpp:28-39); NULL = default */
  const char* forward_mode;
  const char* batch_size;
  const char* input_len;
  const char* output_len;
} cs_ingest_keys;
typedef struct cs_ingest_result cs_ingest_result;
int cs_ingest_chrome_json(const char* text, size_t len, const cs_ingest_keys* keys,
                          uint32_t n_threads, cs_ingest_result** out);
int cs_ingest_view(const cs_ingest_result* r, const cs_event** ev, const uint64_t** event_ids,
                   uint64_t* n_ev, const cs_workload** wl, uint64_t* n_wl, const char** names,
                   size_t* names_bytes, uint32_t* n_names, const int32_t** comm_name,
                   const int32_t** comm_rank, const char** comm_hash, size_t* comm_bytes,
                   uint32_t* n_comm, uint64_t* n_issues);
void cs_ingest_free(cs_ingest_result* r);

/* The ingest's ValidationReport (trace.hpp:129-148): the parse issues in
 * document order followed by validate_trace's checks (trace.cpp:239-276:
 * duplicate event ids, negative span durations, correlation ids, counter
 * values and per-series monotonicity) in canonical event order, as
 * (severity, stable code, event id).  category_counts is indexed by
 * cs_category; a report with n_errors == 0 is what load_validated
 * (main.cpp:41-56) accepts. */
enum cs_issue_code {
  CS_ISSUE_MALFORMED_EVENT = 0,
  CS_ISSUE_MALFORMED_ARGS = 1,
  CS_ISSUE_DUPLICATE_EVENT_ID = 2,
  CS_ISSUE_NEGATIVE_DURATION = 3,
  CS_ISSUE_DUPLICATE_CORRELATION = 4,
  CS_ISSUE_UNMATCHED_CORRELATION = 5,
  CS_ISSUE_NON_MONOTONE_COUNTER = 6
};
enum cs_severity { CS_SEV_ERROR = 0, CS_SEV_WARNING = 1 };
typedef struct cs_ingest_issue {
  uint8_t severity;      /* cs_severity */
  uint8_t code;          /* cs_issue_code */
  uint8_t has_event_id;
  uint8_t reserved[5];
  uint64_t event_id;
} cs_ingest_issue;
/* cmd_ingest's clock unification (main.cpp:80-97): the inputs' inline beacons
 * (Instant "beacon" events with an integer args.reference_ts, extract_beacons)
 * calibrate every clock domain (src.clock; calibrate, align.cpp:22-84: offset
 * from one beacon, the mean offset, or a least-squares drift fit), each input
 * is mapped onto the reference timeline (apply_calibration, 97-113:
 * llround(offset + drift * ts), span durations scaled by drift) and re-sorted,
 * and the inputs are merged (merge_traces, 193-206: stable canonical sort,
 * event ids renumbered from 1).  *out is a new ingest result for the merged
 * trace (names, collective slots, workloads and topology re-interned; no
 * ValidationReport); CS_E_NO_BEACONS / CS_E_INCONSISTENT_BEACONS /
 * CS_E_ALREADY_CALIBRATED as the reference throws them. */
typedef struct cs_calibration_options { /* CalibrationOptions (align.hpp) */
  const char* reference_domain;  /* NULL = "reference" */
  double tolerance_ns;           /* 1000 */
  int32_t estimate_drift;        /* 0 */
  int32_t reserved;
} cs_calibration_options;
int cs_ingest_merge(const cs_ingest_result* const* inputs, uint32_t n_inputs,
                    const cs_calibration_options* options, uint32_t n_threads,
                    cs_ingest_result** out, char* err, size_t err_cap);
/* resolve_topology (align.cpp:178-191) from the same records: a location per
 * comm slot (index into the locations, -1 unmapped); locations are distinct
 * (hostname, device) pairs, hostnames NUL-separated.  *conflicting != 0 when a
 * (commHash, rank) maps to two locations (the reference's ConflictingTopology). */
int cs_ingest_topology(const cs_ingest_result* r, const int32_t** comm_location,
                       const char** loc_nodes, size_t* loc_nodes_bytes, const int32_t** loc_device,
                       uint32_t* n_locations, int* conflicting);
int cs_ingest_report(const cs_ingest_result* r, const cs_ingest_issue** issues, uint64_t* n_issues,
                     uint64_t* n_parse_issues, uint64_t category_counts[8], uint64_t* n_errors);

/* Record extras (PipelineOptions::extra_args_prefix, cycles.cpp:392-405): the
 * numeric args with the prefix ("post_" by default) of the uploaded events, as
 * a side table sorted by event: refs[k] = {canonical event index (batch-wide),
 * first value, count}, values = {key id, value} with key ids into the n_keys
 * keys (lexicographic order, `keys` NUL-separated).  A record's extra[key] is
 * the value of the LAST event of its cycle carrying the key (map assignment in
 * event order).  Call after the events' upload (an upload clears the table). */
typedef struct cs_extra_ref {
  uint64_t event;
  uint32_t first;
  uint32_t count;
} cs_extra_ref;
typedef struct cs_extra_value {
  uint32_t key;
  uint32_t reserved;
  double value;
} cs_extra_value;
int cs_upload_extras(cs_ctx* ctx, uint32_t n_keys, const char* keys, const cs_extra_ref* refs,
                     uint64_t n_refs, const cs_extra_value* values, uint64_t n_values);
/* The records' extras of the last run: n_records x n_keys values and presence
 * bytes (present == 0: the record's cycle has no event with that key). */
int cs_get_record_extras(cs_ctx* ctx, uint32_t inst, double* values, uint8_t* present, size_t cap,
                         size_t* n);

/* Latency model for instance `inst` (UINT32_MAX = default for every instance
 * without its own binding).  Bindings are by instance index, may precede the
 * first cs_upload and survive re-uploads (streams).
 * Replaces LatencyModel::load/predict (baseline.cpp:288-317, gbdt.cpp:173-184). */
int cs_load_model(cs_ctx* ctx, uint32_t inst, const cs_model* model);

/* Runs the selected stages on the device for every uploaded instance.
 * Replaces segment_and_classify + build_cycle_records (cycles.cpp:345-409),
 * cycle_stats beta (rca.cpp:71-130), predict + ppe, Detector::step
 * (detector.cpp:14-19, 91-130).  Asynchronous w.r.t. the host until a getter
 * or cs_sync is called. */
int cs_run(cs_ctx* ctx, uint32_t stage_mask);
int cs_sync(cs_ctx* ctx);

/* Caller-given cycles for the next cs_run(CS_RUN_GIVEN | ...): the span
 * overloads of the reference (build_cycle_records(trace, span<const Cycle>,
 * ...) cycles.cpp:366-409, classify_stages 190-254, extract_workload 256-281,
 * cycle_stats rca.cpp:71-130) take cycles the caller built or edited.  Event
 * positions are canonical indices of the uploaded instance 0; anchor_pos =
 * UINT64_MAX marks a cycle without components (frequency fallback).
 * `components` (n x n_phases, may be NULL) are the cycles' own
 * component_durations, used for the latency target instead of recomputing
 * them.  Getters report the given `index` values. */
int cs_set_cycles(cs_ctx* ctx, const cs_cycle* cycles, uint64_t n, const int64_t* components);

int cs_get_summary(cs_ctx* ctx, uint32_t inst, cs_instance_summary* out);
/* Anchor candidates of the last run (cycles.cpp:47-87), best first.  The
 * scores come from the exact integer moments (within a few ulps of the
 * reference's ordered sums); cs_get_candidates_exact recomputes every
 * candidate with the reference's own sequential arithmetic on the device
 * (incl. periodicity) and is bit-identical to rank_anchor_candidates. */
int cs_get_candidates(cs_ctx* ctx, uint32_t inst, cs_anchor_candidate* buf,
                      size_t cap, size_t* n);
int cs_get_candidates_exact(cs_ctx* ctx, uint32_t inst, cs_anchor_candidate* buf,
                            size_t cap, size_t* n);
int cs_get_cycles(cs_ctx* ctx, uint32_t inst, cs_cycle* buf, size_t cap, size_t* n);
/* component_durations: n_cycles x n_phases int64, row-major */
int cs_get_components(cs_ctx* ctx, uint32_t inst, int64_t* buf, size_t cap, size_t* n);
/* stage attribution: n_cycles x n_beta_slots; total clipped span ns (int64)
 * and beta (f64); a class is absent from the reference's map iff total == 0 */
int cs_get_beta(cs_ctx* ctx, uint32_t inst, int64_t* totals, double* beta,
                size_t cap, size_t* n);
/* collective per-(name,comm,rank) beta: n_cycles x n_comm_slots f64;
 * presence mask: n_cycles x n_comm_slots uint8 */
int cs_get_collective_beta(cs_ctx* ctx, uint32_t inst, double* beta,
                           uint8_t* present, size_t cap, size_t* n);
/* Counter-weighted mean per (cycle, class slot) (CS_RUN_MU): for every Span of
 * the class with duration > 0 and positive clipped overlap whose class maps
 * to a counter series of the instance, interpolate_mean over [start,
 * clipped end) (rca.cpp:17-53) weighted by the overlap, divided by the class
 * total (ClassStat::mu); has[k] = 0 where the reference leaves mu unset. */
int cs_get_mu(cs_ctx* ctx, uint32_t inst, double* mu, uint8_t* has, size_t cap, size_t* n);
int cs_get_records(cs_ctx* ctx, uint32_t inst, cs_record* buf, size_t cap, size_t* n);
/* Row ranges [first, first + count) of the cycle / record tables above (the
 * same rows, `index` and `episode_id` as the whole-table getters).  Used by
 * the sharded single-instance run (halo.py) to read a shard's halo and tail
 * without copying its whole tables; no reference counterpart.  count rows
 * must fit in buf; a range past the table is CS_E_INVALID_ARGUMENT. */
int cs_get_cycle_range(cs_ctx* ctx, uint32_t inst, uint64_t first, uint64_t count, cs_cycle* buf);
int cs_get_record_range(cs_ctx* ctx, uint32_t inst, uint64_t first, uint64_t count, cs_record* buf);
int cs_get_alerts(cs_ctx* ctx, uint32_t inst, cs_alert* buf, size_t cap, size_t* n);

/* ------------------------------------------- post-alert root cause (§8f #4)
 * suspicion_rank + attribute_straggler (rca.cpp:220-353) over a normal and an
 * abnormal window of cycles, from the stage attribution of the last cs_run
 * (CS_RUN_BETA; CS_RUN_MU for the mu terms).  One entry per event class (beta
 * slot) present in either window, sorted by score (descending), ties by class
 * name; welch_p is the two-sided Welch test on beta.  Collective classes get
 * the rank whose mean per-rank beta shifted most between the windows, within
 * communicator groups with >= 2 ranks in the abnormal window.
 * CS_E_INSUFFICIENT_CYCLES below 10 normal / 3 abnormal cycles. */
typedef struct cs_suspect {
  int32_t beta_slot;           /* event class (its name = the slot's name)      */
  int32_t metric;              /* 1 + name id of the counter behind mu, 0 none  */
  double beta_norm, beta_abn, delta_beta, z_beta, z_log_mu, score;
  double mu_norm, mu_abn, delta_mu, welch_p;
  int32_t straggler_slot;      /* comm slot (class, commHash, rank), -1 none    */
  int32_t straggler_location;  /* comm_location[straggler_slot], -1 unmapped    */
  double rank_beta_shift;
} cs_suspect;
/* Host form, on window rows (row c = one cycle of the window, in window order):
 * totals / beta / mu / mu_has: n_cycles x n_slots; coll / coll_present:
 * n_cycles x n_comm. */
typedef struct cs_rca_window {
  uint64_t n_cycles;
  const int64_t* totals;
  const double* beta;
  const double* mu;            /* NULL: no mu terms */
  const uint8_t* mu_has;
  const double* coll;
  const uint8_t* coll_present;
} cs_rca_window;
typedef struct cs_rca_layout {
  uint32_t n_slots;
  uint32_t n_comm;
  const int32_t* slot_metric;    /* per beta slot: 1 + metric name id, 0 none  */
  const int32_t* comm_class;     /* per comm slot: beta slot of its name       */
  const int32_t* comm_group;     /* per comm slot: equal for equal (name, hash) */
  const int32_t* comm_rank;      /* per comm slot: rank                        */
  const int32_t* comm_location;  /* per comm slot: caller's (node, device) id, -1 unmapped; may be NULL */
} cs_rca_layout;
int cs_rank_suspects(const cs_rca_window* normal, const cs_rca_window* abnormal,
                     const cs_rca_layout* layout, cs_suspect* out, size_t cap, size_t* n_out);
/* Device form: the windows are cycle indices of instance `inst`; the rows are
 * gathered from the device.  comm_group / comm_rank / comm_location describe
 * the comm slots (comm_class comes from the name table). */
int cs_suspicion_rank(cs_ctx* ctx, uint32_t inst, const uint64_t* normal_cycles, size_t n_normal,
                      const uint64_t* abnormal_cycles, size_t n_abnormal, const int32_t* comm_name,
                      const int32_t* comm_group, const int32_t* comm_rank,
                      const int32_t* comm_location, cs_suspect* out, size_t cap, size_t* n_out);
/* welch_p_value (rca.cpp:206-218). */
double cs_welch_p_value(double mean_a, double var_a, uint64_t n_a, double mean_b, double var_b,
                        uint64_t n_b);

/* Re-run only the control chart over the residuals of the last cs_run with a
 * different ControlConfig (strategy / window / warmup / thresholds); the
 * evaluate_strategies loop of evaluate_trial (simkit.cpp:867-872). */
int cs_redetect(cs_ctx* ctx, const cs_control_config* control);

/* StrategyMetrics (detector.hpp:138-153) of the last detection for instance
 * `inst` against per-cycle ground-truth labels (labels[cycle_index] != 0),
 * computed on the device: confusion counts over armed records from the
 * flagged bits, lag per contiguous anomaly interval (detector.cpp:166-224). */
typedef struct cs_strategy_metrics {
  int32_t strategy;
  int32_t reserved;
  double precision, recall, f1, fpr, mean_lag;
  uint64_t alerts, tp, fp, fn, tn;
} cs_strategy_metrics;
int cs_evaluate_strategy(cs_ctx* ctx, uint32_t inst, const uint8_t* cycle_labels,
                         uint64_t n_labels, cs_strategy_metrics* out);

/* Detector::step over a residual stream (detector.cpp:85-130; one Detector,
 * samples in order) and, with per-sample labels, evaluate_strategy
 * (detector.cpp:166-224) — the batched detector of evaluate_trial / the
 * drop-in's evaluate_strategy.  The limit is dynamic_ucl for DynamicWindow and
 * ctl->fixed_threshold otherwise (the Detector constructor).  Optional
 * outputs: the statistic and flags (bit0 armed, bit1 flagged, bit2 alert) per
 * sample, metrics (needs labels; CS_E_NO_LABELS for an empty stream). */
int cs_detect_residuals(cs_ctx* ctx, const double* residuals, uint64_t n, const cs_control_config* ctl,
                        double dynamic_ucl, const uint8_t* labels, double* statistic, uint8_t* flags,
                        cs_strategy_metrics* metrics);

/* Alert sink of monitor_loop (main.cpp:151-177): Alert::to_json records
 * (detector.cpp:72-83) as NDJSON, with the Escalator's retain/mode fields on
 * Sentinel->DeepDive edges (detector.cpp:132-150, EscalationPolicy
 * pre/post roll).  `buf` receives the text; *n its length + 1. */
int cs_alerts_to_ndjson(const cs_alert* alerts, uint64_t n_alerts, uint64_t pre_roll,
                        uint64_t post_roll, char* buf, size_t cap, size_t* n);

/* Streaming (BASELINE config 5; the monitor_loop of main.cpp:151-177 fed by
 * time-sliced micro-batches).  Between cs_stream_begin and cs_stream_end every
 * cs_run continues one logical trace per instance:
 *  - the anchor chosen by the first batch (or the hint) is kept;
 *  - the detector window, warm-up count, flagged state and episode count
 *    carry over (any window; the windows in force at the stream's first
 *    batch bound later ones), as does the stage heuristic's history;
 *  - cycle indices and episode ids continue across batches.
 * The caller resubmits each instance's trailing partial cycle with the next
 * batch: events [keep_from, n) of the last upload, where cs_stream_tail gives
 * keep_from.  The result equals one cs_run over the whole trace, minus the
 * final partial cycle.  cs_redetect is unavailable mid-stream. */
int cs_stream_begin(cs_ctx* ctx);
int cs_stream_end(cs_ctx* ctx);
int cs_stream_tail(cs_ctx* ctx, uint32_t inst, uint64_t* keep_from);
/* One micro-batch of monitor_loop (main.cpp:151-177) natively: per instance,
 * the carried trailing partial cycle of the previous push is prepended to the
 * new events ev[offsets[i] .. offsets[i+1]), the batch is uploaded and run
 * with `stage_mask`, the new trailing partial cycle is kept, and the alerts
 * of every instance (instance order) are copied to `alerts`.  Passing
 * n_workloads = 0 and wl = NULL keeps the previously uploaded workload table
 * (event payloads index it).  Per-batch alert latency = this call. */
int cs_stream_push(cs_ctx* ctx, uint32_t n_inst, const uint64_t* offsets, const cs_event* ev,
                   uint64_t n_workloads, const cs_workload* wl, uint32_t stage_mask,
                   cs_alert* alerts, size_t cap, size_t* n_alerts);

/* Execution options.  CS_OPT_FUSED (default 1): the single-read segmentation
 * pass (events read from HBM once per run) when applicable, 0 the two-pass
 * path (warp-streaming event scan + thread-per-cycle reduce).  The single-read
 * pass falls back to the two-pass path by itself for a wrong anchor guess,
 * equal-timestamp groups at anchors, ranges denser than its anchor list and
 * streaming pushes.  Both are bit-identical; the tests run both. */
#define CS_OPT_FUSED 1
/* CS_OPT_TRAVERSAL (default 0): 1 scores every model by tree traversal
 * (k_score) even where a compiled cell table exists (k_score_lut); both are
 * bit-identical to GbdtModel::predict, the tests run both. */
#define CS_OPT_TRAVERSAL 2
/* CS_OPT_PHASE_TIMINGS (default -1): which device phases cs_get_timings
 * reports.  -1: every phase for cs_run, only "total" for cs_stream_push (an
 * event between a micro-batch's small kernels costs device time: it ends
 * the overlap of one kernel's launch with its predecessor); 1: every phase
 * always; 0: "total" only; 2: "total" and the segmentation pass
 * ("segment_range", or "scan_events" and "cycle_reduce" on the two-pass
 * path). */
#define CS_OPT_PHASE_TIMINGS 3
int cs_set_option(cs_ctx* ctx, int option, int64_t value);

/* Pinned host memory helpers (cudaHostAlloc) for the e2e path. */
int cs_host_alloc(size_t bytes, void** out);
int cs_host_free(void* p);

/* Device timing of the last cs_run per kernel family (ms, CUDA events on the
 * ctx stream).  names: comma-separated list written to `names` (cap bytes). */
int cs_get_timings(cs_ctx* ctx, double* ms, size_t cap, size_t* n,
                   char* names, size_t names_cap);
/* Number of kernels launched by the last cs_run. */
int cs_get_launch_count(cs_ctx* ctx, uint64_t* n);

/* ----------------------------------------------------- host-side services */
/* Deterministic GBDT fit (fit_latency_model, baseline.cpp:168-208 and
 * fit_gbdt, gbdt.cpp:40-171), bit-identical to the reference.  Host C++,
 * reported separately from events/s.  x: n x n_features
 * row-major; y: latency seconds.  The result is kept in an opaque handle. */
typedef struct cs_fitted_model cs_fitted_model;
typedef struct cs_gbdt_params { /* GbdtParams gbdt.hpp:25-31 */
  uint64_t n_trees;
  uint64_t max_depth;
  double learning_rate;
  uint64_t min_samples_leaf;
  double prediction_floor;
} cs_gbdt_params;
typedef struct cs_fit_options { /* FitOptions baseline.hpp:42-47 */
  double calibration_fraction;
  double ppe_epsilon;
  int32_t stratify_col;     /* column index of the stratify feature, -1 = 0 */
  int32_t reserved;
  uint64_t min_samples;
} cs_fit_options;
int cs_fit_latency_model(uint64_t n, uint32_t n_features, const int32_t* feature_ids,
                         const double* x, const double* y,
                         const cs_gbdt_params* params, const cs_fit_options* opt,
                         cs_fitted_model** out, char* err, size_t err_cap);
/* The same fit with feature NAMES (the Full feature set's extras columns,
 * to_sample_set baseline.cpp:43-78): names are stored in the model as given. */
int cs_fit_latency_model_named(uint64_t n, uint32_t n_features, const char* const* feature_names,
                               const double* x, const double* y, const cs_gbdt_params* params,
                               const cs_fit_options* opt, cs_fitted_model** out, char* err,
                               size_t err_cap);
/* Batched fit_latency_model on the device: n_models
 * independent sample sets (model m: rows [offsets[m], offsets[m+1]) of x / y,
 * x row-major), each fitted exactly as cs_fit_latency_model would (the model
 * JSON is byte-identical).  Checks, split_calibration and the holdout
 * statistics run on n_threads host threads; the boosting rounds of every
 * model run in one kernel, one CTA per model (k_gbdt_fit: libstdc++'s sort
 * order restated for the split search, sequential sums kept sequential).
 * status[m] is model m's cs_status; out[m] is NULL unless it is CS_OK.
 * device_ms (optional) receives the kernel time.  Supports max_depth <= 8 and
 * 1..8 features (CS_E_UNSUPPORTED otherwise). */
int cs_fit_latency_models(int device, uint32_t n_models, const uint64_t* offsets,
                          uint32_t n_features, const int32_t* feature_ids, const double* x,
                          const double* y, const cs_gbdt_params* params, const cs_fit_options* opt,
                          uint32_t n_threads, cs_fitted_model** out, int32_t* status,
                          float* device_ms);
/* Parse a LatencyModel JSON document (baseline.cpp:288-302). */
int cs_model_from_json(const char* json, cs_fitted_model** out, char* err, size_t err_cap);
/* Serialize to the reference's LatencyModel JSON (baseline.cpp:277-286). */
int cs_model_to_json(const cs_fitted_model* m, char* buf, size_t cap, size_t* n);
int cs_model_view(const cs_fitted_model* m, cs_model* view);
void cs_model_free(cs_fitted_model* m);

/* Single-record host helpers with the reference's exact arithmetic, used by
 * the C++ drop-in shim for ppe / ucl_from_stats / compute_ucl
 * (detector.cpp:14-19, 41-60). */
double cs_ucl_from_stats(double mu, double sigma, const cs_control_config* cfg);
int cs_compute_ucl(const double* residuals, size_t n, double k, double theta_max,
                   double min_ucl, size_t min_n, double* out);

/* RunConfig JSON (the reference's schema, config.cpp:78-188; unknown keys are
 * rejected with CS_E_CONFIG) -> device configs + name table.  `names` are the
 * interned names in id order; name_is_span marks names occurring as Spans
 * (they receive dense beta slots in name order).  Replaces the CycleConfig /
 * PipelineOptions / ControlConfig plumbing of monitor_loop (main.cpp:142-214). */
int cs_config_from_json(const char* run_config_json, uint32_t n_names,
                        const char* const* names, const uint8_t* name_is_span,
                        uint32_t n_comm_slots, cs_name_info* out_names,
                        cs_cycle_config* out_cycle, cs_control_config* out_control,
                        char* err, size_t err_cap);

#ifdef __cplusplus
}
#endif
#endif /* CYCLESCOPE_B200_H_ */
