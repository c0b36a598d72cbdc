"""ctypes binding of libcyclescope_b200.so (the C ABI in include/cyclescope_b200.h).

This is plumbing for tests, bench.py and __graft_entry__: every computation
happens in the native library (sm_100a kernels + host C++).  There is no
Python or CPU fallback — if the library or a CUDA device is missing the calls
raise.

Names mirror the reference's C++ API (cycles.hpp / detector.hpp /
baseline.hpp): `Analyzer.run` is segment_and_classify + build_cycle_records +
cycle_stats(beta) + LatencyModel::predict + ppe + Detector::step over a batch
of instances; `fit_latency_model` is the reference's deterministic fit.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass

import numpy as np

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcyclescope_b200.so")

_lib = None


class EngineError(RuntimeError):
    """Mirrors cyclescope::EngineError: .type is the reference's type() string."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.type = abi.STATUS_TYPES.get(status, "internal")
        super().__init__(f"{self.type}: {message}")


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: build it with __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    vp, sz, u32, u64 = C.c_void_p, C.c_size_t, C.c_uint32, C.c_uint64
    psz = C.POINTER(sz)
    L.cs_abi_version.restype = C.c_int
    L.cs_status_type.restype = C.c_char_p
    L.cs_status_type.argtypes = [C.c_int]
    L.cs_ctx_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.cs_ctx_destroy.argtypes = [vp]
    L.cs_last_error.restype = C.c_char_p
    L.cs_last_error.argtypes = [vp]
    L.cs_set_config.argtypes = [vp, C.POINTER(abi.CycleConfig), C.POINTER(abi.ControlConfig)]
    L.cs_set_name_table.argtypes = [vp, u32, vp]
    L.cs_upload.argtypes = [vp, u32, vp, vp, u64, vp]
    L.cs_upload_unsorted.argtypes = [vp, u32, vp, vp, vp, u64, vp]
    L.cs_get_order.argtypes = [vp, u32, vp, sz, psz]
    L.cs_set_cycles.argtypes = [vp, vp, u64, vp]
    L.cs_upload_extras.argtypes = [vp, u32, C.c_char_p, vp, u64, vp, u64]
    L.cs_get_record_extras.argtypes = [vp, u32, vp, vp, sz, psz]
    L.cs_fit_latency_model_named.argtypes = [u64, u32, C.POINTER(C.c_char_p), vp, vp,
                                             C.POINTER(abi.GbdtParams), C.POINTER(abi.FitOptions),
                                             C.POINTER(vp), C.c_char_p, sz]
    L.cs_detect_residuals.argtypes = [vp, vp, u64, C.POINTER(abi.ControlConfig), C.c_double, vp, vp, vp,
                                      C.POINTER(abi.StrategyMetrics)]
    L.cs_get_cycle_range.argtypes = [vp, u32, u64, u64, vp]
    L.cs_get_record_range.argtypes = [vp, u32, u64, u64, vp]
    L.cs_upload_wire.argtypes = [vp, u32, vp, C.POINTER(abi.WireBatch), u64, vp]
    L.cs_wire_pack.argtypes = [u32, vp, vp, u64, vp, u32, C.POINTER(vp)]
    L.cs_wire_view.argtypes = [vp, C.POINTER(abi.WireBatch), C.POINTER(u64)]
    L.cs_wire_free.argtypes = [vp]
    L.cs_ingest_chrome_json.argtypes = [C.c_char_p, sz, vp, u32, C.POINTER(vp)]
    L.cs_ingest_view.argtypes = [vp] + [C.POINTER(vp)] * 2 + [C.POINTER(u64), C.POINTER(vp),
                                 C.POINTER(u64), C.POINTER(vp), psz, C.POINTER(u32),
                                 C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), psz, C.POINTER(u32),
                                 C.POINTER(u64)]
    L.cs_ingest_free.argtypes = [vp]
    L.cs_rank_suspects.argtypes = [C.POINTER(abi.RcaWindow), C.POINTER(abi.RcaWindow),
                                   C.POINTER(abi.RcaLayout), vp, C.c_size_t, C.POINTER(C.c_size_t)]
    L.cs_suspicion_rank.argtypes = [vp, u32, vp, C.c_size_t, vp, C.c_size_t, vp, vp, vp, vp, vp,
                                    C.c_size_t, C.POINTER(C.c_size_t)]
    L.cs_welch_p_value.restype = C.c_double
    L.cs_welch_p_value.argtypes = [C.c_double, C.c_double, u64, C.c_double, C.c_double, u64]
    L.cs_ingest_topology.argtypes = [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(C.c_size_t), C.POINTER(vp),
                                     C.POINTER(u32), C.POINTER(C.c_int)]
    L.cs_ingest_merge.argtypes = [vp, u32, C.POINTER(abi.CalibrationOptions), u32, C.POINTER(vp),
                                  C.c_char_p, C.c_size_t]
    L.cs_ingest_report.argtypes = [vp, C.POINTER(vp), C.POINTER(u64), C.POINTER(u64), vp, C.POINTER(u64)]
    L.cs_load_model.argtypes = [vp, u32, C.POINTER(abi.Model)]
    L.cs_run.argtypes = [vp, u32]
    L.cs_sync.argtypes = [vp]
    L.cs_get_summary.argtypes = [vp, u32, C.POINTER(abi.InstanceSummary)]
    for fn in ("cs_get_candidates", "cs_get_candidates_exact", "cs_get_cycles", "cs_get_components", "cs_get_records",
               "cs_get_alerts"):
        getattr(L, fn).argtypes = [vp, u32, vp, sz, psz]
    L.cs_get_beta.argtypes = [vp, u32, vp, vp, sz, psz]
    L.cs_get_collective_beta.argtypes = [vp, u32, vp, vp, sz, psz]
    L.cs_get_mu.argtypes = [vp, u32, vp, vp, sz, psz]
    L.cs_set_option.argtypes = [vp, C.c_int, C.c_int64]
    L.cs_redetect.argtypes = [vp, C.POINTER(abi.ControlConfig)]
    L.cs_stream_begin.argtypes = [vp]
    L.cs_stream_end.argtypes = [vp]
    L.cs_stream_tail.argtypes = [vp, u32, C.POINTER(C.c_uint64)]
    L.cs_stream_push.argtypes = [vp, u32, vp, vp, u64, vp, u32, vp, sz, psz]
    L.cs_evaluate_strategy.argtypes = [vp, u32, vp, u64, C.POINTER(abi.StrategyMetrics)]
    L.cs_alerts_to_ndjson.argtypes = [vp, u64, u64, u64, vp, sz, psz]
    L.cs_host_alloc.argtypes = [sz, C.POINTER(vp)]
    L.cs_host_free.argtypes = [vp]
    L.cs_get_timings.argtypes = [vp, vp, sz, psz, C.c_char_p, sz]
    L.cs_get_launch_count.argtypes = [vp, C.POINTER(u64)]
    L.cs_fit_latency_models.argtypes = [C.c_int, u32, vp, u32, vp, vp, vp, C.POINTER(abi.GbdtParams),
                                        C.POINTER(abi.FitOptions), u32, vp, vp, C.POINTER(C.c_float)]
    L.cs_fit_latency_model.argtypes = [u64, u32, vp, vp, vp, C.POINTER(abi.GbdtParams),
                                       C.POINTER(abi.FitOptions), C.POINTER(vp), C.c_char_p, sz]
    L.cs_model_from_json.argtypes = [C.c_char_p, C.POINTER(vp), C.c_char_p, sz]
    L.cs_model_to_json.argtypes = [vp, vp, sz, psz]
    L.cs_model_view.argtypes = [vp, C.POINTER(abi.Model)]
    L.cs_model_free.argtypes = [vp]
    L.cs_ucl_from_stats.restype = C.c_double
    L.cs_ucl_from_stats.argtypes = [C.c_double, C.c_double, C.POINTER(abi.ControlConfig)]
    L.cs_config_from_json.argtypes = [C.c_char_p, u32, vp, vp, u32, vp,
                                      C.POINTER(abi.CycleConfig), C.POINTER(abi.ControlConfig),
                                      C.c_char_p, sz]
    _lib = L
    return L


EXPORTED_SYMBOLS = [
    "cs_abi_version", "cs_status_type", "cs_ctx_create", "cs_ctx_destroy", "cs_last_error",
    "cs_set_config", "cs_set_name_table", "cs_upload", "cs_upload_unsorted", "cs_get_order", "cs_set_cycles", "cs_detect_residuals", "cs_upload_extras", "cs_get_record_extras",
    "cs_fit_latency_model_named", "cs_upload_wire", "cs_wire_pack",
    "cs_wire_view", "cs_wire_free", "cs_ingest_chrome_json", "cs_ingest_view", "cs_ingest_free", "cs_ingest_report", "cs_ingest_topology", "cs_ingest_merge", "cs_rank_suspects",
    "cs_suspicion_rank", "cs_welch_p_value", "cs_load_model", "cs_run", "cs_sync",
    "cs_get_summary", "cs_get_candidates", "cs_get_candidates_exact", "cs_get_cycles", "cs_get_components", "cs_get_beta",
    "cs_get_collective_beta", "cs_get_mu", "cs_get_records", "cs_get_alerts", "cs_host_alloc",
    "cs_host_free", "cs_get_timings", "cs_get_launch_count", "cs_fit_latency_model", "cs_fit_latency_models",
    "cs_model_from_json", "cs_model_to_json", "cs_model_view", "cs_model_free",
    "cs_ucl_from_stats", "cs_compute_ucl", "cs_config_from_json", "cs_set_option",
    "cs_redetect", "cs_evaluate_strategy", "cs_alerts_to_ndjson", "cs_stream_begin",
    "cs_stream_end", "cs_stream_tail", "cs_stream_push",
]


def _check(rc: int, ctx=None, msg: str = ""):
    if rc != 0:
        detail = msg
        if ctx is not None:
            detail = (lib().cs_last_error(ctx) or b"").decode() or msg
        raise EngineError(rc, detail)


def _ptr(a: np.ndarray | None):
    return None if a is None or a.size == 0 else a.ctypes.data


# ---------------------------------------------------------------- models
class LatencyModel:
    """Handle on a fitted / loaded LatencyModel (baseline.hpp:50-67)."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.cs_model_free(self.h)
            self.h = None

    @classmethod
    def from_json(cls, text: str) -> "LatencyModel":
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        rc = lib().cs_model_from_json(text.encode(), C.byref(h), err, 1024)
        if rc:
            raise EngineError(rc, err.value.decode())
        return cls(h)

    def to_json(self) -> str:
        n = C.c_size_t(0)
        lib().cs_model_to_json(self.h, None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value)
        _check(lib().cs_model_to_json(self.h, buf, n.value, C.byref(n)))
        return buf.value.decode()

    def view(self) -> abi.Model:
        v = abi.Model()
        _check(lib().cs_model_view(self.h, C.byref(v)))
        return v

    @property
    def mu_train(self) -> float:
        return self.view().mu_train

    @property
    def sigma_train(self) -> float:
        return self.view().sigma_train


def fit_latency_model(x: np.ndarray, y: np.ndarray, feature_names=("batch", "w_kv"),
                      params: abi.GbdtParams | None = None,
                      options: abi.FitOptions | None = None) -> LatencyModel:
    """fit_latency_model (baseline.cpp:168-208): deterministic host C++ fit.
    Feature names outside batch/w_kv/input_len/output_len/stage are record
    extras (the Full feature set's post_* columns)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    names = list(feature_names)
    params = params or abi.default_gbdt_params()
    if options is None:
        options = abi.default_fit_options(len(names))
        options.stratify_col = names.index("w_kv") if "w_kv" in names else 0
    h = C.c_void_p()
    err = C.create_string_buffer(1024)
    if all(n in abi.FEATURE_IDS for n in names):
        ids = np.array([abi.FEATURE_IDS[n] for n in names], dtype=np.int32)
        rc = lib().cs_fit_latency_model(len(y), len(ids), ids.ctypes.data, _ptr(x), _ptr(y),
                                        C.byref(params), C.byref(options), C.byref(h), err, 1024)
    else:
        arr = (C.c_char_p * len(names))(*[n.encode() for n in names])
        rc = lib().cs_fit_latency_model_named(len(y), len(names), arr, _ptr(x), _ptr(y),
                                              C.byref(params), C.byref(options), C.byref(h), err, 1024)
    if rc:
        raise EngineError(rc, err.value.decode())
    return LatencyModel(h)


def fit_latency_models(xs, ys, feature_names=("batch", "w_kv"),
                       params: abi.GbdtParams | None = None,
                       options: abi.FitOptions | None = None, device: int = 0, n_threads=None):
    """Batched fit_latency_model on the device (cs_fit_latency_models): one model
    per (x, y) pair, each identical to fit_latency_model's.  Returns (models,
    device_ms); a model that cannot be fitted is an EngineError in the list."""
    ids = np.array([abi.FEATURE_IDS[n] for n in feature_names], dtype=np.int32)
    params = params or abi.default_gbdt_params()
    if options is None:
        options = abi.default_fit_options(len(ids))
        options.stratify_col = list(feature_names).index("w_kv") if "w_kv" in feature_names else 0
    xs = [np.ascontiguousarray(x, dtype=np.float64).reshape(-1, len(ids)) for x in xs]
    ys = [np.ascontiguousarray(y, dtype=np.float64) for y in ys]
    off = np.concatenate([[0], np.cumsum([len(y) for y in ys])]).astype(np.uint64)
    x = np.ascontiguousarray(np.concatenate(xs) if xs else np.zeros((0, len(ids))))
    y = np.ascontiguousarray(np.concatenate(ys) if ys else np.zeros(0))
    M = len(ys)
    out = (C.c_void_p * max(M, 1))()
    status = np.zeros(max(M, 1), np.int32)
    ms = C.c_float(0)
    _check(lib().cs_fit_latency_models(device, M, off.ctypes.data, len(ids), ids.ctypes.data, _ptr(x),
                                       _ptr(y), C.byref(params), C.byref(options),
                                       n_threads or os.cpu_count() or 1, out, status.ctypes.data,
                                       C.byref(ms)))
    models = [LatencyModel(C.c_void_p(out[m])) if status[m] == 0 else EngineError(int(status[m]), "fit failed")
              for m in range(M)]
    return models, ms.value


def _i32(a, n):
    return np.ascontiguousarray(np.asarray(a if a is not None else np.full(n, -1), dtype=np.int32))


def comm_groups(comm_name, comm_hash) -> np.ndarray:
    """Group id per comm slot: equal for equal (name, commHash) (cs_rca_layout)."""
    out, last, g = np.zeros(len(comm_name), np.int32), None, -1
    for k, key in enumerate(zip(comm_name, comm_hash)):
        if key != last:
            g, last = g + 1, key
        out[k] = g
    return out


def rank_suspects(normal: dict, abnormal: dict, n_slots: int, n_comm: int, slot_metric=None,
                  comm_class=None, comm_group=None, comm_rank=None, comm_location=None) -> np.ndarray:
    """cs_rank_suspects on window rows: dicts with totals, beta, [mu, mu_has],
    coll, coll_present (rows = cycles of the window, in window order)."""
    keep = []

    def win(d):
        arrs = {k: np.ascontiguousarray(d[k]) for k in d if d[k] is not None}
        keep.append(arrs)
        n = len(arrs["totals"]) // max(n_slots, 1) if n_slots else len(arrs.get("coll", [])) // max(n_comm, 1)
        return abi.RcaWindow(n, _ptr(arrs["totals"]), _ptr(arrs["beta"]), _ptr(arrs.get("mu")),
                             _ptr(arrs.get("mu_has")), _ptr(arrs.get("coll")), _ptr(arrs.get("coll_present")))

    wn, wa = win(normal), win(abnormal)
    lay_arrs = [_i32(slot_metric, n_slots) if slot_metric is not None else None, _i32(comm_class, n_comm),
                _i32(comm_group, n_comm), _i32(comm_rank, n_comm),
                _i32(comm_location, n_comm) if comm_location is not None else None]
    lay = abi.RcaLayout(n_slots, n_comm, *[_ptr(a) if a is not None else None for a in lay_arrs])
    n = C.c_size_t(0)
    _check(lib().cs_rank_suspects(C.byref(wn), C.byref(wa), C.byref(lay), None, 0, C.byref(n)))
    out = np.zeros(n.value, abi.SUSPECT_DTYPE)
    _check(lib().cs_rank_suspects(C.byref(wn), C.byref(wa), C.byref(lay), _ptr(out), n.value, C.byref(n)))
    return out


def suspects_report(entries: np.ndarray, slot_names, names, comm_hash=(), comm_rank=(), locations=()):
    """render_json_report's "suspects" list (rca.cpp:355-385) from cs_suspect records."""
    out = []
    for e in entries:
        d = {"class": slot_names[e["beta_slot"]], "beta_norm": float(e["beta_norm"]),
             "beta_abn": float(e["beta_abn"]), "delta_beta": float(e["delta_beta"]),
             "delta_beta_pct": 100.0 * float(e["delta_beta"]), "z_beta": float(e["z_beta"]),
             "z_log_mu": float(e["z_log_mu"]), "score": float(e["score"]),
             "metric": names[e["metric"] - 1] if e["metric"] > 0 else "",
             "mu_norm": float(e["mu_norm"]), "mu_abn": float(e["mu_abn"]), "delta_mu": float(e["delta_mu"]),
             "p_value": float(e["welch_p"])}
        k = int(e["straggler_slot"])
        if k >= 0:
            st = {"comm": comm_hash[k], "rank": int(comm_rank[k]), "beta_shift": float(e["rank_beta_shift"])}
            loc = locations[e["straggler_location"]] if e["straggler_location"] >= 0 else None
            if loc is None:
                st["node"] = "unmapped"
            else:
                st["node"], st["device"] = loc
            d["straggler"] = st
        out.append(d)
    return out


def diagnose_windows(records: np.ndarray, episode: int = 0, max_normal: int = 300):
    """cmd_diagnose's windows (main.cpp:262-298) from detector records in
    order: flagged runs are episodes, armed unflagged cycles are normal (the
    last max_normal kept).  Returns (normal, abnormal) cycle indices."""
    episodes, normal, open_ = [], [], False
    for r in records:
        if r["flagged"]:
            if not open_:
                episodes.append([])
            open_ = True
            episodes[-1].append(int(r["cycle_index"]))
        else:
            open_ = False
            if r["armed"]:
                normal.append(int(r["cycle_index"]))
    if not episodes:
        raise EngineError(15, "no alert episodes found in this trace")
    if episode >= len(episodes):
        raise EngineError(13, f"episode {episode} out of range, {len(episodes)} episode(s) found")
    return normal[-max_normal:], episodes[episode]


def welch_p_value(mean_a, var_a, n_a, mean_b, var_b, n_b) -> float:
    return lib().cs_welch_p_value(mean_a, var_a, n_a, mean_b, var_b, n_b)


def ucl_from_stats(mu: float, sigma: float, control: abi.ControlConfig) -> float:
    return lib().cs_ucl_from_stats(mu, sigma, C.byref(control))


# ---------------------------------------------------------------- configs
def configs_from_json(run_config: dict | str | None, names, name_is_span, n_comm_slots=0):
    """RunConfig JSON -> (CycleConfig, ControlConfig, name table) via the library."""
    text = run_config if isinstance(run_config, str) else json.dumps(run_config or {})
    n = len(names)
    arr = (C.c_char_p * max(n, 1))(*[s.encode() for s in names])
    span = np.ascontiguousarray(np.asarray(name_is_span, dtype=np.uint8))
    table = np.zeros(n, dtype=abi.NAME_INFO_DTYPE)
    cyc, ctl = abi.CycleConfig(), abi.ControlConfig()
    err = C.create_string_buffer(1024)
    rc = lib().cs_config_from_json(text.encode(), n, C.cast(arr, C.c_void_p) if n else None,
                                   _ptr(span), n_comm_slots, _ptr(table), C.byref(cyc),
                                   C.byref(ctl), err, 1024)
    if rc:
        raise EngineError(rc, err.value.decode())
    return cyc, ctl, table


def span_names_mask(events: np.ndarray, n_names: int) -> np.ndarray:
    """Which interned names occur as Spans (host ingest bookkeeping)."""
    m = np.zeros(n_names, dtype=np.uint8)
    ids = np.unique(events["name_id"][events["kind"] == abi.SPAN])
    m[ids] = 1
    return m


# ---------------------------------------------------------------- synth
@dataclass
class SynthTrace:
    events: np.ndarray
    event_ids: np.ndarray
    workloads: np.ndarray
    labels: np.ndarray
    names: list
    n_comm: int


class SynthParams(C.Structure):
    _fields_ = [("n_cycles", C.c_uint64), ("workload_seed", C.c_uint64),
                ("synth_seed", C.c_uint64), ("fault_family", C.c_int32),
                ("target_rank", C.c_int32), ("fault_onset", C.c_uint64),
                ("fault_duration", C.c_uint64), ("severity", C.c_double),
                ("n_ranks", C.c_uint64), ("noise", C.c_double)]


FAULT_FAMILIES = ["cpu_contention", "cpu_freq_drop", "gpu_contention", "gpu_clock_lock",
                  "memory_thrash", "nvlink_saturation", "pcie_bottleneck", "bus_contention"]


BENCH_LIB_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "benchlib",
                              "libcs_bench.so")
_bench = None


def bench_lib():
    """benchlib/libcs_bench.so: the synthetic trace producer and the HBM
    microbenchmark (benchmark support; never part of the analysis path)."""
    global _bench
    if _bench is None:
        if not os.path.exists(BENCH_LIB_PATH):
            raise RuntimeError(f"{BENCH_LIB_PATH} missing: build it with __graft_entry__.build()")
        B = C.CDLL(BENCH_LIB_PATH)
        vp, sz, u32, u64 = C.c_void_p, C.c_size_t, C.c_uint32, C.c_uint64
        B.cs_synth_generate.argtypes = [vp, u32, u32, C.c_int, C.POINTER(vp)]
        B.cs_synth_view.argtypes = [vp] + [C.POINTER(vp), C.POINTER(u64), C.POINTER(vp),
                                           C.POINTER(vp), C.POINTER(u64), C.POINTER(vp), C.POINTER(u64)]
        B.cs_synth_names.argtypes = [vp, C.POINTER(C.c_char_p), C.POINTER(sz), C.POINTER(u32), C.POINTER(u32)]
        B.cs_synth_free.argtypes = [vp]
        B.cs_microbench.argtypes = [C.c_int, vp, u64, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.POINTER(C.c_double)]
        _bench = B
    return _bench


def synth_trace(n_cycles, workload_seed, synth_seed, fault=None, onset=0, duration=0,
                severity=-1.0, target_rank=0, n_ranks=1, noise=-1.0, n_chunks=1,
                n_threads=None, compact_names=True) -> SynthTrace:
    """Synthetic trace from the simkit restatement (cs_synth.cpp)."""
    fam = -1 if fault is None else (FAULT_FAMILIES.index(fault) if isinstance(fault, str) else int(fault))
    p = SynthParams(n_cycles, workload_seed, synth_seed, fam, target_rank, onset, duration,
                    severity, n_ranks, noise)
    L = bench_lib()
    h = C.c_void_p()
    _check(L.cs_synth_generate(C.byref(p), n_chunks, n_threads or os.cpu_count() or 1,
                               int(compact_names), C.byref(h)))
    try:
        ev, ids, wl, lab = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        nev, nwl, ncyc = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(L.cs_synth_view(h, C.byref(ev), C.byref(nev), C.byref(ids), C.byref(wl),
                               C.byref(nwl), C.byref(lab), C.byref(ncyc)))

        def arr(ptr, n, dtype):
            if n == 0:
                return np.zeros(0, dtype=dtype)
            nbytes = n * np.dtype(dtype).itemsize
            return np.frombuffer((C.c_char * nbytes).from_address(ptr.value), dtype=dtype).copy()

        events = arr(ev, nev.value, abi.EVENT_DTYPE)
        event_ids = arr(ids, nev.value, np.uint64)
        workloads = arr(wl, nwl.value, abi.WORKLOAD_DTYPE)
        labels = arr(lab, ncyc.value, np.uint8).astype(bool)
        packed, nb, nn, nc = C.c_char_p(), C.c_size_t(), C.c_uint32(), C.c_uint32()
        _check(L.cs_synth_names(h, C.byref(packed), C.byref(nb), C.byref(nn), C.byref(nc)))
        raw = C.string_at(packed, nb.value)
        names = [s.decode() for s in raw.split(b"\0")[:nn.value]]
        return SynthTrace(events, event_ids, workloads, labels, names, nc.value)
    finally:
        L.cs_synth_free(h)


@dataclass
class IngestedTrace:
    """cs_ingest_chrome_json output: what an exporter produces from a Trace."""
    events: np.ndarray
    event_ids: np.ndarray
    workloads: np.ndarray
    names: list
    comm_name: np.ndarray
    comm_rank: np.ndarray
    comm_hash: list
    n_issues: int                  # parse issues (parse_trace_json's ValidationIssue count)
    issues: np.ndarray = None      # ISSUE_DTYPE: parse issues, then validate_trace's
    category_counts: np.ndarray = None
    n_errors: int = 0
    comm_location: np.ndarray = None  # per comm slot: index into locations, -1 unmapped
    locations: list = None            # (hostname, device)
    topology_conflict: bool = False

    @property
    def ok(self) -> bool:
        """ValidationReport::ok(): what load_validated (main.cpp:41-56) accepts."""
        return self.n_errors == 0

    @property
    def n_comm(self) -> int:
        return len(self.comm_name)


def ingest_chrome_json(text: bytes, n_threads=None) -> IngestedTrace:
    """Native Chrome-trace JSON ingest (parse_trace_json + interning)."""
    L = lib()
    h = C.c_void_p()
    _check(L.cs_ingest_chrome_json(text, len(text), None, n_threads or os.cpu_count() or 1,
                                   C.byref(h)))
    try:
        return _ingest_extract(h)
    finally:
        L.cs_ingest_free(h)


def ingest_merge(texts, reference_domain="reference", tolerance_ns=1000.0, estimate_drift=False,
                 n_threads=None) -> IngestedTrace:
    """cmd_ingest (main.cpp:80-97) natively: ingest each document, calibrate
    the clock domains from their beacons, apply, merge (cs_ingest_merge)."""
    L = lib()
    nt = n_threads or os.cpu_count() or 1
    hs = []
    try:
        for t in texts:
            h = C.c_void_p()
            _check(L.cs_ingest_chrome_json(t, len(t), None, nt, C.byref(h)))
            hs.append(h)
        arr = (C.c_void_p * max(1, len(hs)))(*[h.value for h in hs])
        opt = abi.CalibrationOptions(reference_domain.encode(), tolerance_ns, int(estimate_drift), 0)
        out = C.c_void_p()
        err = C.create_string_buffer(512)
        rc = L.cs_ingest_merge(arr, len(hs), C.byref(opt), nt, C.byref(out), err, 512)
        if rc:
            raise EngineError(rc, err.value.decode())
        try:
            return _ingest_extract(out)
        finally:
            L.cs_ingest_free(out)
    finally:
        for h in hs:
            L.cs_ingest_free(h)


def _ingest_extract(h) -> IngestedTrace:
    """IngestedTrace from a cs_ingest_result handle (copied out)."""
    L = lib()
    ev, ids, wl, nm, cn, cr, ch = (C.c_void_p() for _ in range(7))
    nev, nwl, iss = C.c_uint64(), C.c_uint64(), C.c_uint64()
    nb, cb = C.c_size_t(), C.c_size_t()
    nn, nc = C.c_uint32(), C.c_uint32()
    _check(L.cs_ingest_view(h, C.byref(ev), C.byref(ids), C.byref(nev), C.byref(wl), C.byref(nwl),
                            C.byref(nm), C.byref(nb), C.byref(nn), C.byref(cn), C.byref(cr),
                            C.byref(ch), C.byref(cb), C.byref(nc), C.byref(iss)))

    def arr(ptr, n, dtype):
        if n == 0 or not ptr.value:
            return np.zeros(0, dtype=dtype)
        nbytes = n * np.dtype(dtype).itemsize
        return np.frombuffer((C.c_char * nbytes).from_address(ptr.value), dtype=dtype).copy()

    names = C.string_at(nm, nb.value).split(b"\0")[:nn.value] if nb.value else []
    hashes = C.string_at(ch, cb.value).split(b"\0")[:nc.value] if cb.value else []
    ip, ni, npi, ne = C.c_void_p(), C.c_uint64(), C.c_uint64(), C.c_uint64()
    cats = np.zeros(8, np.uint64)
    _check(L.cs_ingest_report(h, C.byref(ip), C.byref(ni), C.byref(npi), cats.ctypes.data, C.byref(ne)))
    cl, lnp, ld = C.c_void_p(), C.c_void_p(), C.c_void_p()
    lnb, nloc, conf = C.c_size_t(), C.c_uint32(), C.c_int()
    _check(L.cs_ingest_topology(h, C.byref(cl), C.byref(lnp), C.byref(lnb), C.byref(ld), C.byref(nloc),
                                C.byref(conf)))
    nodes = C.string_at(lnp, lnb.value).split(b"\0")[:nloc.value] if lnb.value else []
    devs = arr(ld, nloc.value, np.int32)
    return IngestedTrace(arr(ev, nev.value, abi.EVENT_DTYPE), arr(ids, nev.value, np.uint64),
                         arr(wl, nwl.value, abi.WORKLOAD_DTYPE), [x.decode() for x in names],
                         arr(cn, nc.value, np.int32), arr(cr, nc.value, np.int32),
                         [x.decode() for x in hashes], iss.value,
                         arr(ip, ni.value, abi.ISSUE_DTYPE), cats, ne.value,
                         arr(cl, nc.value, np.int32), [(x.decode(), int(d)) for x, d in zip(nodes, devs)],
                         bool(conf.value))


@dataclass
class WireTrace:
    """A batch of instances in the columnar wire format (cs_wire_pack)."""
    codes: np.ndarray        # uint8 per event: dictionary code | WIRE_LONG_DT (WIRE_ESCAPE: escaped)
    dt_lo: np.ndarray        # uint16 per event: low 16 bits of the start_ts delta
    dt_hi: np.ndarray        # uint8 per long-delta event: delta >> 16
    dict: np.ndarray         # uint32 info words (name | kind << 16 | category << 20 | flags << 24 | WIDE)
    blocks: np.ndarray       # WIRE_BLOCK_DTYPE per instance-aligned block of WIRE_BLOCK records
    dur_lo: np.ndarray       # uint16, one per Span
    dur_hi: np.ndarray       # uint8, one per Span
    pay8: np.ndarray         # uint8 payloads (narrow codes)
    pay16: np.ndarray        # uint16 payloads (WIDE codes)
    values: np.ndarray       # float64, one per valued Counter
    escapes: np.ndarray      # EVENT_DTYPE records that do not fit
    workloads32: np.ndarray  # uint32 (n, 3) workload table, or None (the i64 table is sent)
    inst_offsets: np.ndarray

    COLUMNS = ("codes", "dt_lo", "dt_hi", "dict", "blocks", "dur_lo", "dur_hi", "pay8", "pay16",
               "values", "escapes", "workloads32")

    @property
    def nbytes(self) -> int:
        return sum(getattr(self, c).nbytes for c in self.COLUMNS if getattr(self, c) is not None)

    def batch(self) -> abi.WireBatch:
        w32 = self.workloads32
        return abi.WireBatch(_ptr(self.codes), _ptr(self.dt_lo), _ptr(self.dt_hi), len(self.dt_hi),
                             _ptr(self.dict), len(self.dict), 0, _ptr(self.blocks), _ptr(self.dur_lo),
                             _ptr(self.dur_hi), len(self.dur_lo), _ptr(self.pay8), len(self.pay8),
                             _ptr(self.pay16), len(self.pay16), _ptr(self.values), len(self.values),
                             _ptr(self.escapes), len(self.escapes),
                             _ptr(w32) if w32 is not None else None, 0 if w32 is None else len(w32))


def wire_pack(events: np.ndarray, inst_offsets, workloads=None, n_threads=None) -> WireTrace:
    """cs_wire_pack: cs_event records (+ workload table) -> wire format (the producer side)."""
    events = np.ascontiguousarray(events, dtype=abi.EVENT_DTYPE)
    off = np.ascontiguousarray(np.asarray(inst_offsets, dtype=np.uint64))
    wl = np.ascontiguousarray(workloads if workloads is not None else np.zeros(0, abi.WORKLOAD_DTYPE),
                              dtype=abi.WORKLOAD_DTYPE)
    L = lib()
    h = C.c_void_p()
    _check(L.cs_wire_pack(len(off) - 1, off.ctypes.data, _ptr(events), len(wl), _ptr(wl),
                          n_threads or os.cpu_count() or 1, C.byref(h)))
    try:
        v, nb = abi.WireBatch(), C.c_uint64()
        _check(L.cs_wire_view(h, C.byref(v), C.byref(nb)))

        def arr(ptr, n, dtype):
            if n == 0 or not ptr:
                return np.zeros(0, dtype=dtype)
            nbytes = n * np.dtype(dtype).itemsize
            return np.frombuffer((C.c_char * nbytes).from_address(ptr), dtype=dtype).copy()

        n = int(off[-1])
        w32 = arr(v.workloads32, 3 * v.n_workloads32, np.uint32).reshape(-1, 3) if v.workloads32 else None
        return WireTrace(arr(v.codes, n, np.uint8), arr(v.dt_lo, n, np.uint16), arr(v.dt_hi, v.n_dt_hi, np.uint8),
                         arr(v.dict, v.n_dict, np.uint32), arr(v.blocks, nb.value, abi.WIRE_BLOCK_DTYPE),
                         arr(v.dur_lo, v.n_durations, np.uint16), arr(v.dur_hi, v.n_durations, np.uint8),
                         arr(v.pay8, v.n_pay8, np.uint8), arr(v.pay16, v.n_pay16, np.uint16),
                         arr(v.values, v.n_values, np.float64), arr(v.escapes, v.n_escapes, abi.EVENT_DTYPE),
                         w32, off)
    finally:
        L.cs_wire_free(h)


# ---------------------------------------------------------------- analyzer
@dataclass
class InstanceResult:
    summary: abi.InstanceSummary
    cycles: np.ndarray
    components: np.ndarray
    beta_totals: np.ndarray | None
    beta: np.ndarray | None
    coll_beta: np.ndarray | None
    coll_present: np.ndarray | None
    records: np.ndarray
    alerts: np.ndarray
    candidates: np.ndarray

    @property
    def status_type(self) -> str:
        return abi.STATUS_TYPES.get(self.summary.status, "internal")


class Analyzer:
    """One device context (cs_ctx): a batch of monitored instances on one GPU."""

    def __init__(self, device: int = 0):
        self.L = lib()
        h = C.c_void_p()
        rc = self.L.cs_ctx_create(device, C.byref(h))
        if rc:
            raise EngineError(rc, "cs_ctx_create failed (no CUDA device?)")
        self.h = h
        self.cycle = abi.CycleConfig()
        self.control = abi.ControlConfig()
        self.names: list = []
        self._keep = []

    def close(self):
        if getattr(self, "h", None):
            self.L.cs_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def _ck(self, rc):
        _check(rc, self.h)

    def configure(self, names, name_is_span, n_comm_slots=0, run_config=None):
        cyc, ctl, table = configs_from_json(run_config, names, name_is_span, n_comm_slots)
        self.set_config(cyc, ctl)
        self.set_name_table(table)
        self.names = list(names)
        self.name_table = np.ascontiguousarray(table, dtype=abi.NAME_INFO_DTYPE)
        return cyc, ctl, table

    def set_config(self, cycle: abi.CycleConfig, control: abi.ControlConfig):
        self.cycle, self.control = cycle, control
        self._ck(self.L.cs_set_config(self.h, C.byref(cycle), C.byref(control)))

    def set_name_table(self, table: np.ndarray):
        table = np.ascontiguousarray(table, dtype=abi.NAME_INFO_DTYPE)
        self._ck(self.L.cs_set_name_table(self.h, len(table), _ptr(table)))

    def upload(self, events: np.ndarray, inst_offsets, workloads: np.ndarray):
        events = np.ascontiguousarray(events, dtype=abi.EVENT_DTYPE)
        off = np.ascontiguousarray(np.asarray(inst_offsets, dtype=np.uint64))
        wl = np.ascontiguousarray(workloads, dtype=abi.WORKLOAD_DTYPE)
        self._ck(self.L.cs_upload(self.h, len(off) - 1, off.ctypes.data, _ptr(events), len(wl),
                                  _ptr(wl)))
        self.n_inst = len(off) - 1

    def upload_unsorted(self, events: np.ndarray, inst_offsets, workloads: np.ndarray,
                        event_ids: np.ndarray | None = None):
        """cs_upload_unsorted (K0): any event order; each instance is sorted on
        the device by (start_ts, event_id) like Trace::sort_events."""
        events = np.ascontiguousarray(events, dtype=abi.EVENT_DTYPE)
        off = np.ascontiguousarray(np.asarray(inst_offsets, dtype=np.uint64))
        wl = np.ascontiguousarray(workloads, dtype=abi.WORKLOAD_DTYPE)
        ids = None if event_ids is None else np.ascontiguousarray(event_ids, dtype=np.uint64)
        self._ck(self.L.cs_upload_unsorted(self.h, len(off) - 1, off.ctypes.data, _ptr(events),
                                           _ptr(ids), len(wl), _ptr(wl)))
        self.n_inst = len(off) - 1

    def order(self, inst: int = 0) -> np.ndarray:
        """cs_get_order: canonical position -> input position within the instance."""
        return self._get(self.L.cs_get_order, inst, np.uint64)

    def upload_extras(self, keys, refs: np.ndarray, values: np.ndarray):
        """cs_upload_extras: the record-extras side table of the uploaded events
        (keys sorted, refs sorted by event, values per ref)."""
        packed = b"".join(k.encode() + b"\0" for k in keys) or b"\0"
        r = np.ascontiguousarray(refs, dtype=abi.EXTRA_REF_DTYPE)
        v = np.ascontiguousarray(values, dtype=abi.EXTRA_VALUE_DTYPE)
        self._keep_extras = (packed, r, v)
        self._ck(self.L.cs_upload_extras(self.h, len(keys), packed, _ptr(r), len(r), _ptr(v), len(v)))
        self.extra_keys = list(keys)

    def record_extras(self, inst=0):
        """cs_get_record_extras: (values, present), n_records x n_keys."""
        n = C.c_size_t()
        self._ck(self.L.cs_get_record_extras(self.h, inst, None, None, 0, C.byref(n)))
        k = len(getattr(self, "extra_keys", []))
        vals = np.zeros(n.value, np.float64)
        has = np.zeros(n.value, np.uint8)
        if n.value:
            self._ck(self.L.cs_get_record_extras(self.h, inst, vals.ctypes.data, has.ctypes.data, n.value,
                                                 C.byref(n)))
        return vals.reshape(-1, k) if k else vals.reshape(0, 0), has.reshape(-1, k) if k else has.reshape(0, 0)

    def set_cycles(self, cycles: np.ndarray, components: np.ndarray | None = None):
        """cs_set_cycles: caller-given cycles (CYCLE_DTYPE rows, canonical event
        positions of instance 0) for the next run(RUN_GIVEN | ...)."""
        cc = np.ascontiguousarray(cycles, dtype=abi.CYCLE_DTYPE)
        comp = None if components is None else np.ascontiguousarray(components, dtype=np.int64)
        self._keep_cycles = (cc, comp)
        self._ck(self.L.cs_set_cycles(self.h, _ptr(cc), len(cc), _ptr(comp)))

    def detect_residuals(self, residuals, control: abi.ControlConfig, dynamic_ucl: float,
                         labels=None):
        """cs_detect_residuals: Detector::step over a residual stream (+
        evaluate_strategy with labels).  Returns (statistic, flags, metrics|None)."""
        r = np.ascontiguousarray(residuals, dtype=np.float64)
        st = np.zeros(len(r), np.float64)
        fl = np.zeros(len(r), np.uint8)
        lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.uint8)
        m = abi.StrategyMetrics()
        self._ck(self.L.cs_detect_residuals(self.h, _ptr(r), len(r), C.byref(control), dynamic_ucl,
                                            _ptr(lab), _ptr(st), _ptr(fl),
                                            C.byref(m) if lab is not None else None))
        return st, fl, (m if lab is not None else None)

    def upload_wire(self, w: WireTrace, workloads: np.ndarray | None = None):
        """cs_upload_wire: same batch as upload(), sent in the columnar wire
        format (the workload table travels in it when packed with one)."""
        b = w.batch()
        if w.workloads32 is not None:
            self._ck(self.L.cs_upload_wire(self.h, len(w.inst_offsets) - 1, w.inst_offsets.ctypes.data,
                                           C.byref(b), 0, None))
        else:
            wl = np.ascontiguousarray(workloads if workloads is not None else np.zeros(0, abi.WORKLOAD_DTYPE),
                                      dtype=abi.WORKLOAD_DTYPE)
            self._ck(self.L.cs_upload_wire(self.h, len(w.inst_offsets) - 1, w.inst_offsets.ctypes.data,
                                           C.byref(b), len(wl), _ptr(wl) if len(wl) else None))
        self.n_inst = len(w.inst_offsets) - 1

    def sync(self):
        """cs_sync: wait for the context's queued work."""
        self._ck(self.L.cs_sync(self.h))

    def load_model(self, model: LatencyModel, inst: int | None = None):
        v = model.view()
        self._keep.append(model)
        self._ck(self.L.cs_load_model(self.h, 0xFFFFFFFF if inst is None else inst, C.byref(v)))

    def set_fused(self, enabled: bool):
        self._ck(self.L.cs_set_option(self.h, 1, int(bool(enabled))))

    def set_traversal(self, enabled: bool):
        """CS_OPT_TRAVERSAL: score by tree traversal (k_score) even when the
        model has a compiled cell table."""
        self._ck(self.L.cs_set_option(self.h, 2, int(bool(enabled))))

    def set_phase_timings(self, mode: int):
        """CS_OPT_PHASE_TIMINGS: -1 per phase except streaming pushes
        (default), 1 per phase always, 0 the run total only, 2 the total and
        the segmentation pass."""
        self._ck(self.L.cs_set_option(self.h, 3, int(mode)))

    def run(self, mask: int = abi.RUN_ALL):
        self._ck(self.L.cs_run(self.h, mask))

    def redetect(self, control: abi.ControlConfig):
        """Control chart only, new ControlConfig, same residuals."""
        self.control = control
        self._ck(self.L.cs_redetect(self.h, C.byref(control)))

    def stream(self) -> "Stream":
        """Begin a micro-batched stream on this analyzer (cs_stream_begin)."""
        return Stream(self)

    def evaluate_strategy(self, labels, inst=0) -> abi.StrategyMetrics:
        """StrategyMetrics vs per-cycle labels (detector.cpp:166-224)."""
        lab = np.ascontiguousarray(np.asarray(labels, dtype=np.uint8))
        m = abi.StrategyMetrics()
        self._ck(self.L.cs_evaluate_strategy(self.h, inst, _ptr(lab), len(lab), C.byref(m)))
        return m

    def launches(self) -> int:
        n = C.c_uint64()
        self._ck(self.L.cs_get_launch_count(self.h, C.byref(n)))
        return n.value

    def timings(self) -> dict:
        ms = np.zeros(32, np.float64)
        n = C.c_size_t()
        names = C.create_string_buffer(1024)
        self._ck(self.L.cs_get_timings(self.h, ms.ctypes.data, 32, C.byref(n), names, 1024))
        keys = names.value.decode().split(",") if n.value else []
        return {k: float(ms[i]) for i, k in enumerate(keys)}

    def summary(self, inst: int = 0) -> abi.InstanceSummary:
        s = abi.InstanceSummary()
        self._ck(self.L.cs_get_summary(self.h, inst, C.byref(s)))
        return s

    def _get(self, fn, inst, dtype):
        n = C.c_size_t()
        self._ck(fn(self.h, inst, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=dtype)
        if n.value:
            self._ck(fn(self.h, inst, out.ctypes.data, n.value, C.byref(n)))
        return out

    def cycles(self, inst=0):
        return self._get(self.L.cs_get_cycles, inst, abi.CYCLE_DTYPE)

    def components(self, inst=0):
        return self._get(self.L.cs_get_components, inst, np.int64)

    def records(self, inst=0):
        return self._get(self.L.cs_get_records, inst, abi.RECORD_DTYPE)

    def cycle_range(self, first: int, count: int, inst=0):
        """Rows [first, first + count) of cycles() (cs_get_cycle_range)."""
        out = np.zeros(count, abi.CYCLE_DTYPE)
        self._ck(self.L.cs_get_cycle_range(self.h, inst, first, count, out.ctypes.data if count else None))
        return out

    def record_range(self, first: int, count: int, inst=0):
        """Rows [first, first + count) of records() (cs_get_record_range)."""
        out = np.zeros(count, abi.RECORD_DTYPE)
        self._ck(self.L.cs_get_record_range(self.h, inst, first, count, out.ctypes.data if count else None))
        return out

    def suspicion_rank(self, normal_cycles, abnormal_cycles, comm_name=(), comm_group=(),
                       comm_rank=(), comm_location=None, inst=0) -> np.ndarray:
        """cs_suspicion_rank: suspects over two windows of cycle indices."""
        nrm = np.ascontiguousarray(np.asarray(normal_cycles, dtype=np.uint64))
        abn = np.ascontiguousarray(np.asarray(abnormal_cycles, dtype=np.uint64))
        cn, cg, cr = (np.ascontiguousarray(np.asarray(a, dtype=np.int32)) for a in (comm_name, comm_group, comm_rank))
        cl = None if comm_location is None else np.ascontiguousarray(np.asarray(comm_location, dtype=np.int32))
        n = C.c_size_t(0)
        args = [self.h, inst, _ptr(nrm), len(nrm), _ptr(abn), len(abn), _ptr(cn), _ptr(cg), _ptr(cr),
                _ptr(cl) if cl is not None else None]
        self._ck(self.L.cs_suspicion_rank(*args, None, 0, C.byref(n)))
        out = np.zeros(n.value, abi.SUSPECT_DTYPE)
        self._ck(self.L.cs_suspicion_rank(*args, _ptr(out), n.value, C.byref(n)))
        return out

    def alerts(self, inst=0):
        return self._get(self.L.cs_get_alerts, inst, abi.ALERT_DTYPE)

    def candidates(self, inst=0):
        return self._get(self.L.cs_get_candidates, inst, abi.CANDIDATE_DTYPE)

    def candidates_exact(self, inst=0):
        """rank_anchor_candidates bit for bit, periodicity included (cs_get_candidates_exact)."""
        return self._get(self.L.cs_get_candidates_exact, inst, abi.CANDIDATE_DTYPE)

    def beta(self, inst=0):
        n = C.c_size_t()
        self._ck(self.L.cs_get_beta(self.h, inst, None, None, 0, C.byref(n)))
        t = np.zeros(n.value, np.int64)
        b = np.zeros(n.value, np.float64)
        if n.value:
            self._ck(self.L.cs_get_beta(self.h, inst, t.ctypes.data, b.ctypes.data, n.value,
                                        C.byref(n)))
        return t, b

    def collective_beta(self, inst=0):
        n = C.c_size_t()
        self._ck(self.L.cs_get_collective_beta(self.h, inst, None, None, 0, C.byref(n)))
        b = np.zeros(n.value, np.float64)
        p = np.zeros(n.value, np.uint8)
        if n.value:
            self._ck(self.L.cs_get_collective_beta(self.h, inst, b.ctypes.data, p.ctypes.data,
                                                   n.value, C.byref(n)))
        return b, p

    def mu(self, inst=0):
        """Counter-weighted mu per (cycle, class slot) and its presence (CS_RUN_MU)."""
        n = C.c_size_t()
        self._ck(self.L.cs_get_mu(self.h, inst, None, None, 0, C.byref(n)))
        m = np.zeros(n.value, np.float64)
        h = np.zeros(n.value, np.uint8)
        if n.value:
            self._ck(self.L.cs_get_mu(self.h, inst, m.ctypes.data, h.ctypes.data, n.value, C.byref(n)))
        return m, h

    def result(self, inst=0, beta=True, scored=True) -> InstanceResult:
        s = self.summary(inst)
        bt = bb = cb = cp = None
        if beta:
            bt, bb = self.beta(inst)
            cb, cp = self.collective_beta(inst)
        return InstanceResult(s, self.cycles(inst), self.components(inst), bt, bb, cb, cp,
                              self.records(inst), self.alerts(inst) if scored else
                              np.zeros(0, abi.ALERT_DTYPE), self.candidates(inst))


def host_alloc(nbytes: int) -> tuple[int, np.ndarray]:
    """Pinned host buffer (cudaHostAlloc) viewed as uint8; returns (ptr, array)."""
    p = C.c_void_p()
    _check(lib().cs_host_alloc(nbytes, C.byref(p)))
    arr = np.frombuffer((C.c_char * nbytes).from_address(p.value), dtype=np.uint8)
    return p.value, arr


def host_free(ptr: int):
    lib().cs_host_free(C.c_void_p(ptr))


def pool_strategy_metrics(per_trial) -> np.ndarray:
    """evaluate_suite's aggregate (simkit.cpp:1038-1068): confusion counts
    pooled over trials per strategy, precision / recall / F1 / FPR from the
    pooled counts, mean lag averaged over trials (in trial order).

    per_trial: per trial, 3 rows (strategies in order) of
    [tp, fp, fn, tn, alerts, ..., mean_lag] — StrategyMetrics or array rows
    with mean_lag last.  Returns (3, 10) float64:
    [tp, fp, fn, tn, alerts, precision, recall, f1, fpr, mean_lag]."""
    out = np.zeros((3, 10), np.float64)
    n = len(per_trial)
    for s in range(3):
        tp = fp = fn = tn = alerts = 0
        lag_sum = 0.0
        for rows in per_trial:
            m = rows[s]
            if isinstance(m, abi.StrategyMetrics):
                v = (m.tp, m.fp, m.fn, m.tn, m.alerts, m.mean_lag)
            else:
                v = (int(m[0]), int(m[1]), int(m[2]), int(m[3]), int(m[4]), float(m[-1]))
            tp, fp, fn, tn, alerts = tp + v[0], fp + v[1], fn + v[2], tn + v[3], alerts + v[4]
            lag_sum += v[5]
        tpf, fpf, fnf, tnf = float(tp), float(fp), float(fn), float(tn)
        precision = tpf / (tpf + fpf) if tpf + fpf > 0.0 else 0.0
        recall = tpf / (tpf + fnf) if tpf + fnf > 0.0 else 0.0
        f1 = 2.0 * precision * recall / (precision + recall) if precision + recall > 0.0 else 0.0
        fpr = fpf / (fpf + tnf) if fpf + tnf > 0.0 else 0.0
        lag = lag_sum / float(n) if n else 0.0
        out[s] = [tp, fp, fn, tn, alerts, precision, recall, f1, fpr, lag]
    return out


def alerts_to_ndjson(alerts: np.ndarray, pre_roll: int = 5, post_roll: int = 20) -> str:
    """monitor_loop's NDJSON alert sink incl. escalation (main.cpp:151-177)."""
    a = np.ascontiguousarray(alerts, dtype=abi.ALERT_DTYPE)
    n = C.c_size_t()
    L = lib()
    _check(L.cs_alerts_to_ndjson(_ptr(a), len(a), pre_roll, post_roll, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value)
    _check(L.cs_alerts_to_ndjson(_ptr(a), len(a), pre_roll, post_roll, buf, n.value, C.byref(n)))
    return buf.value.decode()


class Stream:
    """monitor_loop over time-sliced micro-batches (BASELINE config 5).

    Each push() uploads, per instance, the carried trailing partial cycle of
    the previous batch followed by the new events, runs the path, and keeps
    the new trailing partial cycle (cs_stream_tail).  Detector, stage
    heuristic, cycle indices and episode ids continue across pushes on the
    device; the union of all pushes equals one whole-trace run minus the
    final partial cycle."""

    def __init__(self, analyzer: Analyzer):
        self.an = analyzer
        self.tails: list[np.ndarray] | None = None
        _check(lib().cs_stream_begin(analyzer.h), analyzer.h)

    def push(self, events_per_inst, workloads, mask: int = abi.RUN_ALL):
        if self.tails is None:
            self.tails = [np.zeros(0, abi.EVENT_DTYPE) for _ in events_per_inst]
        if len(events_per_inst) != len(self.tails):
            raise ValueError("instance count changed mid-stream")
        parts = [np.concatenate([t, np.asarray(e, dtype=abi.EVENT_DTYPE)])
                 for t, e in zip(self.tails, events_per_inst)]
        off = np.zeros(len(parts) + 1, np.uint64)
        off[1:] = np.cumsum([len(p) for p in parts])
        ev = np.concatenate(parts) if parts else np.zeros(0, abi.EVENT_DTYPE)
        self.an.upload(ev, off, workloads)
        self.an.run(mask)
        out = [self.an.result(i, beta=bool(mask & abi.RUN_BETA), scored=bool(mask & abi.RUN_DETECT))
               for i in range(len(parts))]
        keep = C.c_uint64(0)
        for i, p in enumerate(parts):
            _check(lib().cs_stream_tail(self.an.h, i, C.byref(keep)), self.an.h)
            self.tails[i] = p[keep.value:].copy()
        return out

    def push_native(self, events_per_inst, workloads=None, mask: int = abi.RUN_ALL,
                    max_alerts: int = 1 << 16) -> np.ndarray:
        """cs_stream_push: the same micro-batch step done in the library (tails,
        upload, run, alert gather in one call); returns every instance's alerts
        in instance order.  workloads=None keeps the uploaded table."""
        parts = [np.asarray(e, dtype=abi.EVENT_DTYPE) for e in events_per_inst]
        off = np.zeros(len(parts) + 1, np.uint64)
        off[1:] = np.cumsum([len(p) for p in parts])
        ev = np.ascontiguousarray(np.concatenate(parts)) if parts else np.zeros(0, abi.EVENT_DTYPE)
        return self.push_packed(ev, off, workloads, mask, max_alerts)

    def push_packed(self, ev: np.ndarray, off: np.ndarray, workloads=None, mask: int = abi.RUN_ALL,
                    max_alerts: int = 1 << 16) -> np.ndarray:
        """push_native with the batch already concatenated (ev, per-instance offsets)."""
        wl = None if workloads is None else np.ascontiguousarray(workloads, dtype=abi.WORKLOAD_DTYPE)
        # one alert buffer per stream, reused (a fresh 5 MB zeroed array per
        # push cost ~0.2 ms of a ~0.55 ms micro-batch)
        out = getattr(self, "_alert_buf", None)
        if out is None or len(out) < max_alerts:
            out = self._alert_buf = np.empty(max_alerts, abi.ALERT_DTYPE)
        n = C.c_size_t()
        _check(lib().cs_stream_push(self.an.h, len(off) - 1, off.ctypes.data, _ptr(ev) or None,
                                    0 if wl is None else len(wl), _ptr(wl), mask, _ptr(out),
                                    max_alerts, C.byref(n)), self.an.h)
        return out[:n.value].copy()

    def close(self):
        _check(lib().cs_stream_end(self.an.h), self.an.h)
