"""TEST INFRASTRUCTURE ONLY — Python handle on the C restatement oracle
(oracle/cs_oracle.c -> oracle/libcsoracle.so).

Derives the name table and configs from a RunConfig dict in plain Python
(independently of the product's cs_config_from_json) and parses the
LatencyModel JSON with the json module, so the oracle shares nothing with
the product beyond the record layout of include/cyclescope_b200.h.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

from paper_2601_09258_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcsoracle.so")
_lib = None

FEATURES = {"batch": 0, "w_kv": 1, "input_len": 2, "output_len": 3, "stage": 4}


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            import subprocess
            subprocess.run(["make", "-C", HERE, "cs_oracle"], check=True,
                           stdout=subprocess.DEVNULL)
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.cso_analyze.argtypes = [vp, C.c_uint64, vp, C.c_uint32, vp, C.POINTER(abi.CycleConfig),
                                  C.POINTER(abi.ControlConfig), C.POINTER(abi.Model),
                                  C.POINTER(vp)]
        L.cso_free.argtypes = [vp]
        for fn, rt in [("cso_status", C.c_int), ("cso_anchor", C.c_uint32),
                       ("cso_fallback", C.c_int), ("cso_ucl", C.c_double),
                       ("cso_first_bad", C.c_uint64), ("cso_n_candidates", C.c_uint64),
                       ("cso_n_cycles", C.c_uint64), ("cso_n_records", C.c_uint64),
                       ("cso_n_alerts", C.c_uint64)] + \
                [(f, vp) for f in ("cso_candidates", "cso_cycles", "cso_components",
                                   "cso_beta_totals", "cso_beta", "cso_coll",
                                   "cso_coll_present", "cso_mu", "cso_mu_has", "cso_records",
                                   "cso_alerts")]:
            getattr(L, fn).restype = rt
            getattr(L, fn).argtypes = [vp]
        _lib = L
    return _lib


def derive_config(run_config, names, name_is_span, n_comm):
    """CycleConfig/PipelineOptions/ControlConfig defaults (cycles.hpp:18-43,
    123-128; detector.hpp:25-34) overridden by a RunConfig dict."""
    rc = run_config or {}
    cy = rc.get("cycle", {})
    pl = rc.get("pipeline", {})
    de = rc.get("detector", {})
    phases = []
    for p in cy.get("phase_functions", ["run_batch", "process_batch_result",
                                        "get_next_batch_to_run"]):
        if p not in phases:
            phases.append(p)
    pkw = cy.get("prefill_keywords", ["forward_prefill"])
    dkw = cy.get("decode_keywords", ["process_batch_result_decode"])
    # MetricMap::defaults (rca.cpp:55-69), replaced by RunConfig metric_map
    metric_map = rc.get("metric_map", {
        "oncpu": "cpu_usage", "gemm_kernel": "gpu_usage", "attn_kernel": "gpu_clock",
        "reduce": "tx_bytes", "memcpy_h2d": "pcie_util", "memcpy_d2d": "bus_util",
        "run_batch": "gpu_usage", "process_batch_result": "cpu_usage",
        "get_next_batch_to_run": "cpu_usage"})
    table = np.zeros(len(names), dtype=abi.NAME_INFO_DTYPE)
    slot = 0
    for i, n in enumerate(names):
        m = metric_map.get(n)
        table[i]["metric"] = names.index(m) + 1 if m in names else 0
        table[i]["phase"] = phases.index(n) if n in phases else -1
        flags = 0
        if any(k in n for k in pkw):
            flags |= abi.NAME_PREFILL_KW
        if any(k in n for k in dkw):
            flags |= abi.NAME_DECODE_KW
        table[i]["flags"] = flags
        table[i]["beta_slot"] = slot if name_is_span[i] else -1
        slot += 1 if name_is_span[i] else 0
    hint = cy.get("anchor_hint", "")
    lc = pl.get("latency_component", "run_batch")
    cyc = abi.CycleConfig(
        anchor_hint_name=(-1 if not hint else (names.index(hint) if hint in names else -2)),
        min_anchor_calls=cy.get("min_anchor_calls", 10),
        prefill_duration_factor=cy.get("prefill_duration_factor", 3.0),
        prefill_gap_factor=cy.get("prefill_gap_factor", 2.0),
        stage_window=cy.get("stage_window", 32), stage_min_history=8,
        frequency_bin_ns=1_000_000, n_phases=len(phases),
        latency_phase=(phases.index(lc) if lc and lc in phases else -1),
        include_prefill=int(pl.get("include_prefill", False)), n_beta_slots=slot,
        n_comm_slots=n_comm)
    strat = {"fixed_point": 0, "fixed_window": 1, "dynamic_window": 2}[
        de.get("strategy", "dynamic_window")]
    ctl = abi.ControlConfig(strat, 0, de.get("window", 10), de.get("fixed_threshold", 0.15),
                            de.get("sigma_k", 3.0), de.get("theta_max", 0.18),
                            de.get("min_ucl", 0.02), de.get("warmup", 100),
                            de.get("epsilon", 1e-9))
    return cyc, ctl, table


def model_struct(model_json: str):
    j = json.loads(model_json)
    g = j["gbdt"]
    nodes, offs = [], [0]
    for t in g["trees"]:
        for n in t:
            nodes.append((n["f"], n["l"], n["r"], 0, n["t"], n["v"]))
        offs.append(len(nodes))
    nodes = np.array(nodes, dtype=abi.TREE_NODE_DTYPE) if nodes else np.zeros(1, abi.TREE_NODE_DTYPE)
    offs = np.array(offs, dtype=np.uint32)
    fids = np.array([FEATURES[f] for f in j["features"]], dtype=np.int32)
    m = abi.Model(len(fids), len(g["trees"]), fids.ctypes.data_as(C.POINTER(C.c_int32)),
                  offs.ctypes.data_as(C.POINTER(C.c_uint32)), nodes.ctypes.data,
                  g["base"], g["params"]["learning_rate"], g["params"]["prediction_floor"],
                  j["residual_stats"]["mu"], j["residual_stats"]["sigma"],
                  int(g["degenerate"]), 0)
    return m, (nodes, offs, fids)


def _arr(ptr, n, dtype):
    if not n:
        return np.zeros(0, dtype=dtype)
    nbytes = n * np.dtype(dtype).itemsize
    return np.frombuffer((C.c_char * nbytes).from_address(ptr), dtype=dtype).copy()


def analyze(events, names, workloads, n_comm=0, run_config=None, model_json=None, span=None):
    """The whole hot path on one instance; returns a dict of numpy arrays.
    `span`: which names are span names (beta slots); default: those with a
    span event in `events` (a shard of a trace passes the whole trace's)."""
    L = lib()
    events = np.ascontiguousarray(events, dtype=abi.EVENT_DTYPE)
    workloads = np.ascontiguousarray(workloads, dtype=abi.WORKLOAD_DTYPE)
    if span is None:
        span = np.zeros(len(names), np.uint8)
        span[np.unique(events["name_id"][events["kind"] == abi.SPAN])] = 1
    span = np.ascontiguousarray(span, dtype=np.uint8)
    cyc, ctl, table = derive_config(run_config, names, span, n_comm)
    mp = None
    if model_json:
        m, keep = model_struct(model_json)
        mp = C.byref(m)
    out = C.c_void_p()
    L.cso_analyze(events.ctypes.data if len(events) else None, len(events),
                  workloads.ctypes.data if len(workloads) else None, len(names),
                  table.ctypes.data if len(table) else None, C.byref(cyc), C.byref(ctl), mp,
                  C.byref(out))
    try:
        nc = L.cso_n_cycles(out)
        P, Cs, R = cyc.n_phases, cyc.n_beta_slots, cyc.n_comm_slots
        res = dict(
            status=L.cso_status(out), anchor=L.cso_anchor(out), fallback=bool(L.cso_fallback(out)),
            ucl=L.cso_ucl(out), first_bad_record=L.cso_first_bad(out),
            candidates=_arr(L.cso_candidates(out), L.cso_n_candidates(out), abi.CANDIDATE_DTYPE),
            cycles=_arr(L.cso_cycles(out), nc, abi.CYCLE_DTYPE),
            components=_arr(L.cso_components(out), nc * P, np.int64),
            beta_totals=_arr(L.cso_beta_totals(out), nc * Cs, np.int64),
            beta=_arr(L.cso_beta(out), nc * Cs, np.float64),
            coll_beta=_arr(L.cso_coll(out), nc * R, np.float64),
            coll_present=_arr(L.cso_coll_present(out), nc * R, np.uint8),
            mu=_arr(L.cso_mu(out), nc * Cs, np.float64),
            mu_has=_arr(L.cso_mu_has(out), nc * Cs, np.uint8),
            records=_arr(L.cso_records(out), L.cso_n_records(out), abi.RECORD_DTYPE),
            alerts=_arr(L.cso_alerts(out), L.cso_n_alerts(out), abi.ALERT_DTYPE))
    finally:
        L.cso_free(out)
    return res
