"""TEST INFRASTRUCTURE ONLY — Python handle on oracle/_ref/libcsref.so.

The library is the reference implementation (/root/reference/proj/src)
compiled unmodified plus our bridge (oracle/ref_bridge.cpp).  Only tests/,
__graft_entry__.smoke() and bench.py's reference / cpu_baseline legs may use
it, and only as the checker or the timed CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field

import numpy as np

from paper_2601_09258_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libcsref.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run make -C oracle)")
        L = C.CDLL(LIB_PATH)
        vp, sz = C.c_void_p, C.c_size_t
        L.ref_synth.restype = vp
        L.ref_synth.argtypes = [C.c_void_p]
        L.ref_to_json.argtypes = [vp, C.c_char_p, sz, C.POINTER(sz)]
        L.ref_from_json.restype = vp
        L.ref_from_json.argtypes = [C.c_char_p, sz, C.POINTER(C.c_uint64)]
        L.ref_rca.argtypes = [vp, vp, sz, vp, sz, C.c_int, C.c_char_p, sz, C.POINTER(sz), C.c_char_p, sz]
        L.ref_merge.restype = vp
        L.ref_merge.argtypes = [vp, vp, C.c_uint32, C.c_char_p, C.c_double, C.c_int, C.c_char_p, sz]
        L.ref_topology.argtypes = [vp, C.c_char_p, sz, C.POINTER(sz)]
        L.ref_validate.argtypes = [vp, vp, sz, C.POINTER(sz), vp, C.POINTER(C.c_uint64)]
        L.ref_build.restype = vp
        L.ref_build.argtypes = [C.c_uint64, vp, vp, C.c_uint32, C.c_char_p, vp, C.c_uint32,
                                C.c_char_p, vp, C.c_int]
        L.ref_free.argtypes = [vp]
        L.ref_n_events.restype = C.c_uint64
        L.ref_n_events.argtypes = [vp]
        L.ref_export.argtypes = [vp, C.c_char_p]
        L.ref_run.argtypes = [vp, C.c_char_p, C.c_char_p, C.c_uint64, C.c_int]
        L.ref_status.argtypes = [vp, C.c_char_p, sz, C.c_char_p, sz]
        L.ref_anchor.argtypes = [vp, C.c_char_p, sz, C.POINTER(C.c_int)]
        L.ref_ucl.restype = C.c_double
        L.ref_ucl.argtypes = [vp]
        L.ref_seconds.restype = C.c_double
        L.ref_seconds.argtypes = [vp]
        L.ref_first_bad_record.restype = C.c_uint64
        L.ref_first_bad_record.argtypes = [vp]
        L.ref_trial_dataset.restype = vp
        L.ref_trial_dataset.argtypes = [C.c_uint64]
        L.ref_evaluate_trial.argtypes = [vp, C.c_uint64, vp, C.c_char_p, sz]
        for fn in ("ref_get_events", "ref_get_event_ids", "ref_get_workloads", "ref_labels",
                   "ref_get_candidates", "ref_get_cycles", "ref_get_components",
                   "ref_get_records", "ref_get_alerts", "ref_get_model_json",
                   "ref_get_ndjson"):
            getattr(L, fn).argtypes = [vp, vp, sz, C.POINTER(sz)]
        L.ref_get_names.argtypes = [vp, vp, sz, C.POINTER(sz), C.POINTER(C.c_uint32)]
        L.ref_get_extra_keys.argtypes = [vp, vp, sz, C.POINTER(sz), C.POINTER(C.c_uint32)]
        L.ref_get_extra_refs.argtypes = [vp, vp, sz, C.POINTER(sz)]
        L.ref_get_extra_values.argtypes = [vp, vp, sz, C.POINTER(sz)]
        L.ref_get_record_extras.argtypes = [vp, vp, sz, C.POINTER(sz), vp, vp, sz, C.POINTER(sz)]
        L.ref_get_comm.argtypes = [vp, vp, vp, vp, sz, C.POINTER(sz), C.POINTER(C.c_uint32)]
        L.ref_get_beta.argtypes = [vp, vp, vp, sz, C.POINTER(sz)]
        L.ref_get_collective_beta.argtypes = [vp, vp, vp, sz, C.POINTER(sz)]
        L.ref_get_mu.argtypes = [vp, vp, vp, sz, C.POINTER(sz)]
        L.ref_fit.argtypes = [C.c_uint64, C.c_uint32, C.c_char_p, vp, vp, vp, vp, vp, sz,
                              C.POINTER(sz), C.c_char_p, sz]
        L.ref_cpu_prepare.restype = vp
        L.ref_cpu_prepare.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64,
                                      C.c_uint64]
        L.ref_cpu_prepare_slices.restype = vp
        L.ref_cpu_prepare_slices.argtypes = [C.c_uint64, vp, vp, C.c_uint32, C.c_char_p, vp, C.c_uint32,
                                             C.c_char_p, vp, C.c_uint32, vp, vp, C.c_char_p, C.c_char_p,
                                             C.c_uint32]
        L.ref_cpu_events.restype = C.c_uint64
        L.ref_cpu_events.argtypes = [vp]
        L.ref_cpu_fit_seconds.restype = C.c_double
        L.ref_cpu_fit_seconds.argtypes = [vp]
        L.ref_cpu_free.argtypes = [vp]
        L.ref_full_parity.argtypes = [C.c_uint64, vp, C.c_uint32, C.c_char_p, vp, C.c_uint32, C.c_char_p,
                                      vp, vp, C.c_int32, C.c_int32, C.c_int32, C.c_char_p, C.c_char_p,
                                      C.c_uint32, C.c_uint64, C.c_uint64, vp, vp, vp, vp, vp, vp,
                                      C.c_uint64, vp, C.c_uint64, vp, vp, vp, vp, C.c_char_p, sz]
        L.ref_cpu_run.restype = C.c_double
        L.ref_cpu_run.argtypes = [vp, C.c_uint32, C.POINTER(C.c_uint64)]
        _lib = L
    return _lib


class SynthParams(C.Structure):
    _fields_ = [("n_cycles", C.c_uint64), ("workload_seed", C.c_uint64),
                ("synth_seed", C.c_uint64), ("fault_family", C.c_int32),
                ("target_rank", C.c_int32), ("fault_onset", C.c_uint64),
                ("fault_duration", C.c_uint64), ("severity", C.c_double),
                ("n_ranks", C.c_uint64), ("noise", C.c_double)]


FAULT_FAMILIES = ["cpu_contention", "cpu_freq_drop", "gpu_contention", "gpu_clock_lock",
                  "memory_thrash", "nvlink_saturation", "pcie_bottleneck", "bus_contention"]


def _get(fn, h, dtype, n_hint=None):
    n = C.c_size_t(0)
    fn(h, None, 0, C.byref(n))
    out = np.zeros(n.value, dtype=dtype)
    if n.value:
        fn(h, out.ctypes.data, n.value, C.byref(n))
    return out


@dataclass
class Exported:
    events: np.ndarray
    event_ids: np.ndarray
    workloads: np.ndarray
    names: list
    comm_name: np.ndarray
    comm_rank: np.ndarray
    comm_hash: list
    extra_keys: list = field(default_factory=list)
    extra_refs: np.ndarray = None
    extra_values: np.ndarray = None


@dataclass
class RefResult:
    status: int
    err_type: str
    err_msg: str
    anchor: str
    fallback: bool
    candidates: np.ndarray
    cycles: np.ndarray
    components: np.ndarray
    beta_totals: np.ndarray
    beta: np.ndarray
    coll_beta: np.ndarray
    coll_present: np.ndarray
    records: np.ndarray
    alerts: np.ndarray
    model_json: str
    ucl: float
    first_bad_record: int
    seconds: float
    extra: dict = field(default_factory=dict)


class RefTrace:
    """A reference `Trace` living in the oracle library."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_free(self.h)
            self.h = None

    @classmethod
    def synth(cls, n_cycles, workload_seed, synth_seed, fault=None, onset=0, duration=0,
              severity=-1.0, target_rank=0, n_ranks=1, noise=-1.0):
        fam = -1 if fault is None else (FAULT_FAMILIES.index(fault) if isinstance(fault, str) else int(fault))
        p = SynthParams(n_cycles, workload_seed, synth_seed, fam, target_rank, onset, duration,
                        severity, n_ranks, noise)
        return cls(lib().ref_synth(C.byref(p)))

    def to_json(self) -> bytes:
        """The reference's serialize_trace_json of this trace."""
        L = lib()
        n = C.c_size_t(0)
        L.ref_to_json(self.h, None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value)
        L.ref_to_json(self.h, buf, n.value, C.byref(n))
        return buf.raw[:n.value]

    def rca(self, normal, abnormal, mu=False):
        """suspicion_rank + attribute_straggler over cycle-index windows of the
        last run(): the parsed render_json_report, or ("error", type)."""
        L = lib()
        nrm = np.ascontiguousarray(np.asarray(normal, dtype=np.uint64))
        abn = np.ascontiguousarray(np.asarray(abnormal, dtype=np.uint64))
        n = C.c_size_t(0)
        err = C.create_string_buffer(256)
        rc = L.ref_rca(self.h, nrm.ctypes.data, len(nrm), abn.ctypes.data, len(abn), int(mu), None, 0,
                       C.byref(n), err, 256)
        if rc == 2:
            return ("error", err.value.decode())
        buf = C.create_string_buffer(n.value + 1)
        assert L.ref_rca(self.h, nrm.ctypes.data, len(nrm), abn.ctypes.data, len(abn), int(mu), buf,
                         n.value, C.byref(n), err, 256) == 0
        return json.loads(buf.raw[:n.value])

    def topology(self):
        """resolve_topology per exported comm slot: [node, device] or None."""
        L = lib()
        n = C.c_size_t(0)
        L.ref_topology(self.h, None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value + 1)
        L.ref_topology(self.h, buf, n.value, C.byref(n))
        return json.loads(buf.raw[:n.value])

    def validate(self):
        """validate_trace with the parse issues: (ISSUE_DTYPE records, category counts, n_errors)."""
        L = lib()
        n, ne = C.c_size_t(0), C.c_uint64(0)
        cats = np.zeros(8, np.uint64)
        L.ref_validate(self.h, None, 0, C.byref(n), cats.ctypes.data, C.byref(ne))
        out = np.zeros(n.value, abi.ISSUE_DTYPE)
        assert L.ref_validate(self.h, out.ctypes.data, n.value, C.byref(n), None, None) == 0
        return out, cats, ne.value

    @classmethod
    def merge(cls, texts, reference_domain="reference", tolerance_ns=1000.0, estimate_drift=False):
        """The reference's cmd_ingest pipeline on documents: a RefTrace of the
        merged trace, or ("error", type)."""
        L = lib()
        bufs = [C.create_string_buffer(t, len(t)) for t in texts]
        ptrs = (C.c_void_p * max(1, len(texts)))(*[C.addressof(b) for b in bufs])
        lens = (C.c_size_t * max(1, len(texts)))(*[len(t) for t in texts])
        err = C.create_string_buffer(256)
        h = L.ref_merge(ptrs, lens, len(texts), reference_domain.encode(), tolerance_ns,
                        int(estimate_drift), err, 256)
        if not h:
            return ("error", err.value.decode())
        return cls(h)

    @classmethod
    def from_json(cls, text: bytes):
        """A trace from the reference's parse_trace_json; returns (trace, n_issues)."""
        iss = C.c_uint64(0)
        return cls(lib().ref_from_json(text, len(text), C.byref(iss))), iss.value

    @classmethod
    def build(cls, events, names, workloads=None, comm_hash=(), comm_rank=(), event_ids=None,
              sort=True):
        events = np.ascontiguousarray(events, dtype=abi.EVENT_DTYPE)
        wl = np.ascontiguousarray(workloads if workloads is not None else
                                  np.zeros(0, abi.WORKLOAD_DTYPE), dtype=abi.WORKLOAD_DTYPE)
        packed = b"".join(n.encode() + b"\0" for n in names)
        cpacked = b"".join(c.encode() + b"\0" for c in comm_hash) or b"\0"
        crank = np.ascontiguousarray(np.asarray(comm_rank, dtype=np.int32))
        ids = None if event_ids is None else np.ascontiguousarray(event_ids, dtype=np.uint64)
        h = lib().ref_build(len(events), events.ctypes.data,
                            None if ids is None else ids.ctypes.data, len(names), packed,
                            wl.ctypes.data if len(wl) else None, len(comm_hash), cpacked,
                            crank.ctypes.data if len(crank) else None, int(sort))
        t = cls(h)
        t._keep = (events, wl, crank, ids)
        return t

    @classmethod
    def trial(cls, trial: int):
        """SuiteConfig{} trial dataset (simkit.cpp:760-792)."""
        return cls(lib().ref_trial_dataset(trial))

    def evaluate_trial(self, trial: int) -> np.ndarray:
        """Reference evaluate_trial: 3 x [tp, fp, fn, tn, alerts, f1, fpr, lag]."""
        out = np.zeros(24, np.float64)
        err = C.create_string_buffer(512)
        if lib().ref_evaluate_trial(self.h, trial, out.ctypes.data, err, 512):
            raise RuntimeError(err.value.decode())
        return out.reshape(3, 8)

    def n_events(self):
        return int(lib().ref_n_events(self.h))

    def labels(self):
        return _get(lib().ref_labels, self.h, np.uint8).astype(bool)

    def export(self, run_config: dict | None = None) -> Exported:
        L = lib()
        assert L.ref_export(self.h, json.dumps(run_config or {}).encode()) == 0
        ev = _get(L.ref_get_events, self.h, abi.EVENT_DTYPE)
        ids = _get(L.ref_get_event_ids, self.h, np.uint64)
        wl = _get(L.ref_get_workloads, self.h, abi.WORKLOAD_DTYPE)
        nb, nn = C.c_size_t(0), C.c_uint32(0)
        L.ref_get_names(self.h, None, 0, C.byref(nb), C.byref(nn))
        buf = C.create_string_buffer(nb.value + 1)
        L.ref_get_names(self.h, buf, nb.value, C.byref(nb), C.byref(nn))
        names = buf.raw[:nb.value].split(b"\0")[:nn.value]
        cb, nc = C.c_size_t(0), C.c_uint32(0)
        L.ref_get_comm(self.h, None, None, None, 0, C.byref(cb), C.byref(nc))
        cn = np.zeros(nc.value, np.int32)
        cr = np.zeros(nc.value, np.int32)
        cbuf = C.create_string_buffer(cb.value + 1)
        L.ref_get_comm(self.h, cn.ctypes.data, cr.ctypes.data, cbuf, cb.value, C.byref(cb),
                       C.byref(nc))
        hashes = cbuf.raw[:cb.value].split(b"\0")[:nc.value]
        kb, nk = C.c_size_t(0), C.c_uint32(0)
        L.ref_get_extra_keys(self.h, None, 0, C.byref(kb), C.byref(nk))
        kbuf = C.create_string_buffer(kb.value + 1)
        L.ref_get_extra_keys(self.h, kbuf, kb.value, C.byref(kb), C.byref(nk))
        keys = [k.decode() for k in kbuf.raw[:kb.value].split(b"\0")[:nk.value]]
        return Exported(ev, ids, wl, [n.decode() for n in names], cn, cr,
                        [h.decode() for h in hashes], keys,
                        _get(L.ref_get_extra_refs, self.h, abi.EXTRA_REF_DTYPE),
                        _get(L.ref_get_extra_values, self.h, abi.EXTRA_VALUE_DTYPE))

    def run(self, run_config: dict | None = None, model_json: str | None = None,
            train_cycles: int = 2400, beta: bool = True, mu: bool = False) -> RefResult:
        """mu=True: cycle_stats with the trace's CounterTable (O(cycles x samples)
        in the reference: keep traces small)."""
        L = lib()
        L.ref_run(self.h, json.dumps(run_config or {}).encode(),
                  (model_json or "").encode(), train_cycles, int(beta) | (2 if mu else 0))
        tb, mb = C.create_string_buffer(256), C.create_string_buffer(4096)
        status = L.ref_status(self.h, tb, 256, mb, 4096)
        ab, fb = C.create_string_buffer(4096), C.c_int(0)
        L.ref_anchor(self.h, ab, 4096, C.byref(fb))
        n = C.c_size_t(0)
        L.ref_get_beta(self.h, None, None, 0, C.byref(n))
        bt = np.zeros(n.value, np.int64)
        bb = np.zeros(n.value, np.float64)
        if n.value:
            L.ref_get_beta(self.h, bt.ctypes.data, bb.ctypes.data, n.value, C.byref(n))
        L.ref_get_collective_beta(self.h, None, None, 0, C.byref(n))
        cbeta = np.zeros(n.value, np.float64)
        cpres = np.zeros(n.value, np.uint8)
        if n.value:
            L.ref_get_collective_beta(self.h, cbeta.ctypes.data, cpres.ctypes.data, n.value,
                                      C.byref(n))
        L.ref_get_mu(self.h, None, None, 0, C.byref(n))
        mu_v = np.zeros(n.value, np.float64)
        mu_h = np.zeros(n.value, np.uint8)
        if n.value:
            L.ref_get_mu(self.h, mu_v.ctypes.data, mu_h.ctypes.data, n.value, C.byref(n))
        kb, nx = C.c_size_t(0), C.c_size_t(0)
        L.ref_get_record_extras(self.h, None, 0, C.byref(kb), None, None, 0, C.byref(nx))
        kbuf = C.create_string_buffer(kb.value + 1)
        rx = np.zeros(nx.value, np.float64)
        rh = np.zeros(nx.value, np.uint8)
        L.ref_get_record_extras(self.h, kbuf, kb.value, C.byref(kb), rx.ctypes.data, rh.ctypes.data, nx.value,
                                C.byref(nx))
        rkeys = [k.decode() for k in kbuf.raw[:kb.value].split(b"\0") if k]
        mj = _get(L.ref_get_model_json, self.h, np.uint8)
        nd = _get(L.ref_get_ndjson, self.h, np.uint8)
        return RefResult(
            status=status, err_type=tb.value.decode(), err_msg=mb.value.decode(),
            anchor=ab.value.decode(), fallback=bool(fb.value),
            candidates=_get(L.ref_get_candidates, self.h, abi.CANDIDATE_DTYPE),
            cycles=_get(L.ref_get_cycles, self.h, abi.CYCLE_DTYPE),
            components=_get(L.ref_get_components, self.h, np.int64),
            beta_totals=bt, beta=bb, coll_beta=cbeta, coll_present=cpres,
            records=_get(L.ref_get_records, self.h, abi.RECORD_DTYPE),
            alerts=_get(L.ref_get_alerts, self.h, abi.ALERT_DTYPE),
            model_json=bytes(mj[:-1]).decode() if len(mj) else "",
            ucl=L.ref_ucl(self.h), first_bad_record=int(L.ref_first_bad_record(self.h)),
            seconds=L.ref_seconds(self.h),
            extra={"ndjson": bytes(nd[:-1]).decode() if len(nd) else "", "mu": mu_v,
                   "mu_has": mu_h, "rec_extra_keys": rkeys,
                   "rec_extra": rx.reshape(-1, len(rkeys)) if rkeys else rx.reshape(0, 0),
                   "rec_extra_has": rh.reshape(-1, len(rkeys)) if rkeys else rh.reshape(0, 0)})


def ref_fit(x: np.ndarray, y: np.ndarray, feature_names, params=None, options=None) -> str:
    """Reference fit_latency_model on explicit samples -> model JSON."""
    L = lib()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    params = params or abi.default_gbdt_params()
    options = options or abi.default_fit_options(len(feature_names))
    packed = b"".join(n.encode() + b"\0" for n in feature_names)
    n = C.c_size_t(0)
    err = C.create_string_buffer(1024)
    cap = 1 << 24
    buf = C.create_string_buffer(cap)
    rc = L.ref_fit(len(y), len(feature_names), packed, x.ctypes.data, y.ctypes.data,
                   C.byref(params), C.byref(options), buf, cap, C.byref(n), err, 1024)
    if rc == 2:
        raise RuntimeError(err.value.decode())
    return buf.raw[:n.value - 1].decode()


class CpuBaseline:
    """Reference CPU analyzer on prepared simkit traces (one instance/thread)."""

    def __init__(self, n_instances, n_threads, cycles_per_instance, n_ranks, seed=42):
        self.n_threads = n_threads
        self.h = lib().ref_cpu_prepare(n_instances, n_threads, cycles_per_instance, n_ranks, seed)
        self.events = int(lib().ref_cpu_events(self.h))
        self.fit_seconds = lib().ref_cpu_fit_seconds(self.h)

    @classmethod
    def slices(cls, events, event_ids, names, workloads, comm_hash, comm_rank, lo, hi, model_json,
               anchor, n_threads):
        """Cycle-aligned slices [lo[k], hi[k]) of ONE trace, one reference
        Trace each (analysed on its own thread with `anchor` as the hint and
        one model)."""
        self = cls.__new__(cls)
        self.n_threads = n_threads
        ev = np.ascontiguousarray(events, dtype=abi.EVENT_DTYPE)
        ids = None if event_ids is None else np.ascontiguousarray(event_ids, dtype=np.uint64)
        wl = np.ascontiguousarray(workloads, dtype=abi.WORKLOAD_DTYPE)
        lo = np.ascontiguousarray(lo, dtype=np.uint64)
        hi = np.ascontiguousarray(hi, dtype=np.uint64)
        packed = b"".join(n.encode() + b"\0" for n in names)
        cpacked = b"".join(c.encode() + b"\0" for c in comm_hash) or b"\0"
        crank = np.ascontiguousarray(np.asarray(comm_rank, dtype=np.int32))
        self.h = lib().ref_cpu_prepare_slices(len(ev), ev.ctypes.data, None if ids is None else ids.ctypes.data,
                                              len(names), packed,
                                              wl.ctypes.data, len(comm_hash), cpacked,
                                              crank.ctypes.data if len(crank) else None, len(lo),
                                              lo.ctypes.data, hi.ctypes.data, model_json.encode(),
                                              anchor.encode(), n_threads)
        self.events = int(lib().ref_cpu_events(self.h))
        self.fit_seconds = 0.0
        return self

    def run(self):
        """One timed pass; returns (seconds, alerts)."""
        na = C.c_uint64(0)
        secs = lib().ref_cpu_run(self.h, self.n_threads, C.byref(na))
        return secs, int(na.value)

    def close(self):
        if self.h:
            lib().ref_cpu_free(self.h)
            self.h = None


def full_parity(an, events, names, workloads, n_comm, model_json, anchor, n_threads,
                chunk_events=1_000_000, inst=0):
    """The WHOLE trace through the reference (ref_full_parity: cycle-aligned
    chunks on n_threads threads, one Detector over every record in order)
    compared with the product's results for instance `inst` of analyzer `an`
    (after a RUN_ALL with beta).  Returns the summary dict bench.py reports;
    every comparison is bitwise."""
    ev = np.ascontiguousarray(events, dtype=abi.EVENT_DTYPE)
    wl = np.ascontiguousarray(workloads, dtype=abi.WORKLOAD_DTYPE)
    packed = b"".join(n.encode() + b"\0" for n in names)
    cpacked = b"".join(b"comm0\0" for _ in range(n_comm)) or b"\0"
    crank = np.arange(max(1, n_comm), dtype=np.int32)
    P, Cs, R = an.cycle.n_phases, an.cycle.n_beta_slots, an.cycle.n_comm_slots
    cyc = an.cycles(inst)
    recs = an.records(inst)
    alerts = an.alerts(inst)
    nc, nr = len(cyc), len(recs)
    cap_c, cap_r, cap_a = nc + 16, nr + 16, len(alerts) + 1024
    r_cyc = np.zeros(cap_c, abi.CYCLE_DTYPE)
    r_comp = np.zeros(cap_c * max(P, 1), np.int64)
    r_tot = np.zeros(cap_c * max(Cs, 1), np.int64)
    r_beta = np.zeros(cap_c * max(Cs, 1), np.float64)
    r_coll = np.zeros(cap_c * max(R, 1), np.float64)
    r_cp = np.zeros(cap_c * max(R, 1), np.uint8)
    r_rec = np.zeros(cap_r, abi.RECORD_DTYPE)
    r_al = np.zeros(cap_a, abi.ALERT_DTYPE)
    n_out = np.zeros(3, np.uint64)
    flags = C.c_uint32(0)
    secs = C.c_double(0)
    err = C.create_string_buffer(512)
    table = np.ascontiguousarray(an.name_table, dtype=abi.NAME_INFO_DTYPE)
    rc = lib().ref_full_parity(len(ev), ev.ctypes.data, len(names), packed, wl.ctypes.data, n_comm, cpacked,
                               crank.ctypes.data, table.ctypes.data, P, Cs, R, model_json.encode(),
                               anchor.encode(), n_threads, chunk_events, cap_c, r_cyc.ctypes.data,
                               r_comp.ctypes.data, r_tot.ctypes.data, r_beta.ctypes.data, r_coll.ctypes.data,
                               r_cp.ctypes.data, cap_r, r_rec.ctypes.data, cap_a, r_al.ctypes.data,
                               n_out.ctypes.data, C.byref(flags), C.byref(secs), err, 512)
    if rc != 0:
        raise RuntimeError(f"ref_full_parity: {err.value.decode()}")
    rn_c, rn_r, rn_a = (int(x) for x in n_out)
    r_cyc, r_rec, r_al = r_cyc[:rn_c], r_rec[:rn_r], r_al[:rn_a]

    def same(a, b):
        return a.shape == b.shape and a.tobytes() == b.tobytes()

    ok = {}
    ok["cycles"] = rn_c == nc and all(np.array_equal(r_cyc[f], cyc[f]) for f in abi.CYCLE_DTYPE.names)
    ok["components"] = same(r_comp[:rn_c * P], an.components(inst)[:nc * P])
    tot, beta = an.beta(inst)
    ok["beta"] = same(r_tot[:rn_c * Cs], tot) and same(r_beta[:rn_c * Cs], beta)
    cb, cp = an.collective_beta(inst)
    ok["collective_beta"] = same(r_coll[:rn_c * R], cb) and same(r_cp[:rn_c * R], cp)
    rec_fields = [f for f in abi.RECORD_DTYPE.names if f not in ("reserved", "episode_id")]
    def raw(a):
        return np.ascontiguousarray(a).view(np.uint8)

    ok["records"] = rn_r == nr and all(np.array_equal(raw(r_rec[f]), raw(recs[f])) for f in rec_fields)
    al_fields = [f for f in abi.ALERT_DTYPE.names if f != "reserved"]
    ok["alerts"] = rn_a == len(alerts) and all(
        np.array_equal(raw(r_al[f]), raw(alerts[f])) for f in al_fields)
    out = {"checked_against": "reference built unmodified from /root/reference (oracle/_ref)",
           "scope": "whole trace: cycle-aligned chunks through segment_and_classify / cycle_stats / "
                    "build_cycle_records / predict / ppe, one Detector over every record in order",
           "events_compared": int(len(ev)), "cycles_compared": nc, "records_compared": nr,
           "alerts_compared": int(rn_a), "reference_seconds": round(secs.value, 2),
           "reference_threads": int(n_threads),
           "stages_from_heuristic": bool(flags.value & 1)}
    out.update({f"{k}_identical": bool(v) for k, v in ok.items()})
    out["identical"] = all(ok.values())
    return out
