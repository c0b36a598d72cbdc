"""numpy / ctypes mirrors of the structs in include/cyclescope_b200.h.

Pure layout definitions: no compute happens here.  The dtypes are used to
hand host buffers to the C ABI without copies and to read results back.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

EVENT_DTYPE = np.dtype(
    [("start_ts", "<i8"), ("duration", "<i8"), ("name_id", "<u4"), ("kind", "u1"),
     ("category", "u1"), ("flags", "<u2"), ("payload", "<u8")], align=True)
assert EVENT_DTYPE.itemsize == 32

# wire format (cs_wire_event header, 8 bytes): the host->device format
ISSUE_DTYPE = np.dtype([("severity", "u1"), ("code", "u1"), ("has_event_id", "u1"),
                        ("reserved", "u1", (5,)), ("event_id", "<u8")])
assert ISSUE_DTYPE.itemsize == 16
SEV_ERROR, SEV_WARNING = 0, 1
ISSUE_CODES = ("malformed_event", "malformed_args", "duplicate_event_id", "negative_duration",
               "duplicate_correlation", "unmatched_correlation", "non_monotone_counter")

WIRE_BLOCK = 1024
WIRE_ESCAPE = 0x7F          # code of an escaped event
WIRE_LONG_DT = 0x80         # code bit: the delta's high byte is in dt_hi
WIRE_MAX_DICT = 127
WIRE_WIDE = 1 << 30         # dictionary bit: the payload is in pay16
WIRE_BLOCK_DTYPE = np.dtype([("base_ts", "<i8"), ("dur", "<u8"), ("pay8", "<u8"), ("pay16", "<u8"),
                             ("val", "<u8"), ("dt_hi", "<u8"), ("esc", "<u8"), ("batch_base", "<u4"),
                             ("reserved", "<u4")])
assert WIRE_BLOCK_DTYPE.itemsize == 64

WORKLOAD_DTYPE = np.dtype([("batch", "<i8"), ("input_len", "<i8"), ("output_len", "<i8")])
EXTRA_REF_DTYPE = np.dtype([("event", "<u8"), ("first", "<u4"), ("count", "<u4")])
EXTRA_VALUE_DTYPE = np.dtype([("key", "<u4"), ("reserved", "<u4"), ("value", "<f8")])
NAME_INFO_DTYPE = np.dtype(
    [("flags", "<u4"), ("phase", "<i4"), ("beta_slot", "<i4"), ("metric", "<u4")])

CYCLE_DTYPE = np.dtype(
    [("index", "<u8"), ("start_ts", "<i8"), ("end_ts", "<i8"), ("anchor_pos", "<u8"),
     ("anchor_span_end", "<i8"), ("first_event", "<u8"), ("last_event", "<u8"),
     ("stage", "<i4"), ("workload_status", "<i4")], align=True)
RECORD_DTYPE = np.dtype(
    [("cycle_index", "<u8"), ("start_ts", "<i8"), ("batch", "<i8"), ("input_len", "<i8"),
     ("output_len", "<i8"), ("latency_s", "<f8"), ("predicted_s", "<f8"),
     ("residual", "<f8"), ("statistic", "<f8"), ("stage", "<i4"), ("armed", "u1"),
     ("flagged", "u1"), ("alert", "u1"), ("reserved", "u1"), ("episode_id", "<u8")],
    align=True)
ALERT_DTYPE = np.dtype(
    [("cycle", "<u8"), ("ts", "<i8"), ("smoothed_error", "<f8"), ("limit", "<f8"),
     ("strategy", "<i4"), ("reserved", "<i4"), ("batch", "<i8"), ("input_len", "<i8"),
     ("output_len", "<i8"), ("episode_id", "<u8"), ("record_index", "<u8")], align=True)
CANDIDATE_DTYPE = np.dtype(
    [("name_id", "<u4"), ("reserved", "<u4"), ("call_count", "<u8"),
     ("mean_duration_ns", "<f8"), ("duration_cv", "<f8"), ("score", "<f8"),
     ("periodicity", "<f8")], align=True)
TREE_NODE_DTYPE = np.dtype(
    [("feature", "<i4"), ("left", "<i4"), ("right", "<i4"), ("reserved", "<i4"),
     ("threshold", "<f8"), ("value", "<f8")], align=True)

# kinds / categories / flags (trace.hpp:20-31)
SPAN, INSTANT, COUNTER, FLOW = 0, 1, 2, 3
CAT = dict(python_call=0, runtime_api=1, gpu_kernel=2, mem_copy=3, os_sched=4,
           net_io=5, counter_telemetry=6, collective_comm=7)
FM_NONE, FM_PREFILL, FM_DECODE, FM_OTHER = 0, 1, 2, 3
EV_HAS_BATCH, EV_WL_OK, EV_HAS_COMM, EV_HAS_VALUE = 0x4, 0x8, 0x10, 0x20
NAME_PREFILL_KW, NAME_DECODE_KW = 0x1, 0x2
STAGE_PREFILL, STAGE_DECODE, STAGE_UNKNOWN = 0, 1, 2
FIXED_POINT, FIXED_WINDOW, DYNAMIC_WINDOW = 0, 1, 2
F_BATCH, F_W_KV, F_INPUT_LEN, F_OUTPUT_LEN, F_STAGE = 0, 1, 2, 3, 4
FEATURE_IDS = {"batch": F_BATCH, "w_kv": F_W_KV, "input_len": F_INPUT_LEN,
               "output_len": F_OUTPUT_LEN, "stage": F_STAGE}

RUN_SEGMENT, RUN_BETA, RUN_SCORE, RUN_DETECT, RUN_ALL = 0x1, 0x2, 0x4, 0x8, 0xF
RUN_MU = 0x10  # counter-weighted mu (cycle_stats with a CounterTable)
RUN_GIVEN = 0x20  # caller-given cycles (cs_set_cycles) instead of segmentation
RUN_CLASSIFY = 0x40  # with RUN_GIVEN: classify_stages from scratch

CS_ABI_VERSION = 2  # include/cyclescope_b200.h

STATUS_TYPES = {
    0: "ok", 1: "invalid_argument", 2: "no_device", 3: "cuda_error",
    4: "no_anchor_found", 5: "missing_workload_args", 6: "feature_mismatch",
    7: "non_positive_latency", 8: "insufficient_data", 9: "insufficient_calibration",
    10: "no_labels", 11: "model_format_error", 12: "unsupported", 13: "config_error",
    14: "internal", 15: "insufficient_cycles", 16: "no_beacons", 17: "inconsistent_beacons",
    18: "already_calibrated",
}
U64_MAX = (1 << 64) - 1
U32_MAX = (1 << 32) - 1


class CycleConfig(C.Structure):
    _fields_ = [("anchor_hint_name", C.c_int64), ("min_anchor_calls", C.c_uint64),
                ("prefill_duration_factor", C.c_double), ("prefill_gap_factor", C.c_double),
                ("stage_window", C.c_uint64), ("stage_min_history", C.c_uint64),
                ("frequency_bin_ns", C.c_int64), ("n_phases", C.c_int32),
                ("latency_phase", C.c_int32), ("include_prefill", C.c_int32),
                ("n_beta_slots", C.c_int32), ("n_comm_slots", C.c_int32),
                ("monitor_from_cycle", C.c_int32)]


class ControlConfig(C.Structure):
    _fields_ = [("strategy", C.c_int32), ("reserved", C.c_int32), ("window", C.c_uint64),
                ("fixed_threshold", C.c_double), ("sigma_k", C.c_double),
                ("theta_max", C.c_double), ("min_ucl", C.c_double),
                ("warmup", C.c_uint64), ("epsilon", C.c_double)]


class Model(C.Structure):
    _fields_ = [("n_features", C.c_uint32), ("n_trees", C.c_uint32),
                ("feature_ids", C.POINTER(C.c_int32)), ("tree_offsets", C.POINTER(C.c_uint32)),
                ("nodes", C.c_void_p), ("base", C.c_double), ("learning_rate", C.c_double),
                ("prediction_floor", C.c_double), ("mu_train", C.c_double),
                ("sigma_train", C.c_double), ("degenerate", C.c_int32),
                ("reserved", C.c_int32), ("feature_names", C.POINTER(C.c_char_p))]


class InstanceSummary(C.Structure):
    _fields_ = [("anchor_name_id", C.c_uint32), ("status", C.c_int32),
                ("n_cycles", C.c_uint64), ("n_records", C.c_uint64),
                ("n_alerts", C.c_uint64), ("first_bad_record", C.c_uint64),
                ("ucl", C.c_double), ("used_frequency_fallback", C.c_int32),
                ("anchor_ambiguous", C.c_int32)]


class GbdtParams(C.Structure):
    _fields_ = [("n_trees", C.c_uint64), ("max_depth", C.c_uint64),
                ("learning_rate", C.c_double), ("min_samples_leaf", C.c_uint64),
                ("prediction_floor", C.c_double)]


class FitOptions(C.Structure):
    _fields_ = [("calibration_fraction", C.c_double), ("ppe_epsilon", C.c_double),
                ("stratify_col", C.c_int32), ("reserved", C.c_int32),
                ("min_samples", C.c_uint64)]


def default_gbdt_params() -> GbdtParams:
    """GbdtParams defaults (gbdt.hpp:25-31)."""
    return GbdtParams(200, 5, 0.1, 5, 1e-6)


def default_fit_options(n_features: int = 2) -> FitOptions:
    """FitOptions defaults (baseline.hpp:42-47); stratify on w_kv (column 1)."""
    return FitOptions(0.2, 1e-9, 1 if n_features > 1 else 0, 0, 20)


def default_control(strategy: int = DYNAMIC_WINDOW) -> ControlConfig:
    """ControlConfig defaults (detector.hpp:25-34)."""
    return ControlConfig(strategy, 0, 10, 0.15, 3.0, 0.18, 0.02, 100, 1e-9)


class WireBatch(C.Structure):  # cs_wire_batch
    _fields_ = [("codes", C.c_void_p), ("dt_lo", C.c_void_p), ("dt_hi", C.c_void_p), ("n_dt_hi", C.c_uint64),
                ("dict", C.c_void_p), ("n_dict", C.c_uint32), ("reserved", C.c_uint32),
                ("blocks", C.c_void_p), ("dur_lo", C.c_void_p), ("dur_hi", C.c_void_p),
                ("n_durations", C.c_uint64), ("pay8", C.c_void_p), ("n_pay8", C.c_uint64),
                ("pay16", C.c_void_p), ("n_pay16", C.c_uint64), ("values", C.c_void_p),
                ("n_values", C.c_uint64), ("escapes", C.c_void_p), ("n_escapes", C.c_uint64),
                ("workloads32", C.c_void_p), ("n_workloads32", C.c_uint64)]


SUSPECT_DTYPE = np.dtype([("beta_slot", "<i4"), ("metric", "<i4"), ("beta_norm", "<f8"),
                          ("beta_abn", "<f8"), ("delta_beta", "<f8"), ("z_beta", "<f8"),
                          ("z_log_mu", "<f8"), ("score", "<f8"), ("mu_norm", "<f8"), ("mu_abn", "<f8"),
                          ("delta_mu", "<f8"), ("welch_p", "<f8"), ("straggler_slot", "<i4"),
                          ("straggler_location", "<i4"), ("rank_beta_shift", "<f8")])
assert SUSPECT_DTYPE.itemsize == 104


class Suspect(C.Structure):  # cs_suspect
    _fields_ = [("beta_slot", C.c_int32), ("metric", C.c_int32), ("beta_norm", C.c_double),
                ("beta_abn", C.c_double), ("delta_beta", C.c_double), ("z_beta", C.c_double),
                ("z_log_mu", C.c_double), ("score", C.c_double), ("mu_norm", C.c_double),
                ("mu_abn", C.c_double), ("delta_mu", C.c_double), ("welch_p", C.c_double),
                ("straggler_slot", C.c_int32), ("straggler_location", C.c_int32),
                ("rank_beta_shift", C.c_double)]


class CalibrationOptions(C.Structure):  # cs_calibration_options
    _fields_ = [("reference_domain", C.c_char_p), ("tolerance_ns", C.c_double),
                ("estimate_drift", C.c_int32), ("reserved", C.c_int32)]


class RcaWindow(C.Structure):  # cs_rca_window
    _fields_ = [("n_cycles", C.c_uint64), ("totals", C.c_void_p), ("beta", C.c_void_p),
                ("mu", C.c_void_p), ("mu_has", C.c_void_p), ("coll", C.c_void_p),
                ("coll_present", C.c_void_p)]


class RcaLayout(C.Structure):  # cs_rca_layout
    _fields_ = [("n_slots", C.c_uint32), ("n_comm", C.c_uint32), ("slot_metric", C.c_void_p),
                ("comm_class", C.c_void_p), ("comm_group", C.c_void_p), ("comm_rank", C.c_void_p),
                ("comm_location", C.c_void_p)]


class StrategyMetrics(C.Structure):
    _fields_ = [("strategy", C.c_int32), ("reserved", C.c_int32), ("precision", C.c_double),
                ("recall", C.c_double), ("f1", C.c_double), ("fpr", C.c_double),
                ("mean_lag", C.c_double), ("alerts", C.c_uint64), ("tp", C.c_uint64),
                ("fp", C.c_uint64), ("fn", C.c_uint64), ("tn", C.c_uint64)]
