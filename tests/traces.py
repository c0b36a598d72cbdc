"""Hand-built traces mirroring the reference's own fixtures
(/root/reference/proj/tests/test_cycles.cpp, test_rca.cpp), expressed as
32-byte records.  `build(spec)` interns names lexicographically, assigns
event ids in listing order and sorts canonically by (start_ts, event_id)
(trace.hpp:110-113), exactly what Trace::sort_events does.
"""
from __future__ import annotations

import numpy as np

from paper_2601_09258_b200 import abi

# A fixed 1-tree model for fixtures too small to fit one (the reference needs
# >= 20 samples): predicts 1e-7 s for W_kv <= 100.5, else 3e-7 s.
TINY_MODEL = {
    "format_version": 1, "kind": "latency_gbdt", "features": ["batch", "w_kv"],
    "residual_stats": {"mu": 0.01, "sigma": 0.01, "calibration_size": 10},
    "gbdt": {"params": {"n_trees": 1, "max_depth": 5, "learning_rate": 0.1,
                        "min_samples_leaf": 5, "prediction_floor": 1e-06},
             "n_features": 2, "base": 5e-07, "degenerate": False, "importance": [0.0, 0.0],
             "trees": [[{"f": 1, "t": 100.5, "l": 1, "r": 2, "v": 0.0},
                        {"f": -1, "t": 0.0, "l": -1, "r": -1, "v": 1e-06},
                        {"f": -1, "t": 0.0, "l": -1, "r": -1, "v": 3e-06}]]},
}

FM = {None: 0, "prefill": abi.FM_PREFILL, "decode": abi.FM_DECODE, "other": abi.FM_OTHER}
KIND = {"span": abi.SPAN, "instant": abi.INSTANT, "counter": abi.COUNTER, "flow": abi.FLOW}


def ev(name, start, dur=0, kind="span", cat="python_call", fm=None, batch=None, input_len=None,
       output_len=None, comm=None, rank=None, value=None):
    return dict(name=name, start=start, dur=dur, kind=kind, cat=cat, fm=fm, batch=batch,
                input_len=input_len, output_len=output_len, comm=comm, rank=rank, value=value)


class Built:
    def __init__(self, events, names, workloads, comm_hash, comm_rank, event_ids):
        self.events = events
        self.names = names
        self.workloads = workloads
        self.comm_hash = comm_hash
        self.comm_rank = comm_rank
        self.event_ids = event_ids

    @property
    def n_comm(self):
        return len(self.comm_hash)


def build(spec) -> Built:
    names = sorted({e["name"] for e in spec})
    nid = {n: i for i, n in enumerate(names)}
    comm_keys = sorted({(e["name"], e["comm"], int(e["rank"])) for e in spec
                        if e["kind"] == "span" and e["cat"] == "collective_comm"
                        and e["comm"] is not None and e["rank"] is not None})
    cslot = {k: i for i, k in enumerate(comm_keys)}
    ids = np.arange(1, len(spec) + 1, dtype=np.uint64)
    starts = np.array([e["start"] for e in spec], dtype=np.int64)
    order = np.lexsort((ids, starts))
    out = np.zeros(len(spec), dtype=abi.EVENT_DTYPE)
    wls = []
    for k, i in enumerate(order):
        e = spec[i]
        r = out[k]
        r["start_ts"] = e["start"]
        kind = KIND[e["kind"]]
        r["kind"] = kind
        r["duration"] = e["dur"] if kind == abi.SPAN else 0
        r["name_id"] = nid[e["name"]]
        r["category"] = abi.CAT[e["cat"]]
        flags = FM[e["fm"]]
        payload = 0
        if e["batch"] is not None:
            flags |= abi.EV_HAS_BATCH
            il = e["input_len"] if e["input_len"] is not None else -(1 << 63)
            ol = e["output_len"] if e["output_len"] is not None else -(1 << 63)
            if (e["input_len"] is not None and e["output_len"] is not None and e["batch"] >= 0
                    and il >= 0 and ol >= 0):
                flags |= abi.EV_WL_OK
            payload |= len(wls)
            wls.append((e["batch"], il, ol))
        key = (e["name"], e["comm"], int(e["rank"]) if e["rank"] is not None else 0)
        if kind == abi.SPAN and e["cat"] == "collective_comm" and key in cslot:
            flags |= abi.EV_HAS_COMM
            payload |= cslot[key] << 32
        if kind == abi.COUNTER and e["value"] is not None:
            flags |= abi.EV_HAS_VALUE
            r["duration"] = np.array([e["value"]], np.float64).view(np.int64)[0]
        r["flags"] = flags
        r["payload"] = payload
    wl = np.array(wls, dtype=abi.WORKLOAD_DTYPE) if wls else np.zeros(0, abi.WORKLOAD_DTYPE)
    return Built(out, names, wl, [k[1] for k in comm_keys], [k[2] for k in comm_keys],
                 ids[order])


def rng_uniform(seed):
    """A tiny deterministic stream for synthetic fixtures (not the reference Rng)."""
    r = np.random.default_rng(seed)
    return lambda lo, hi: float(r.uniform(lo, hi))


# ------------------------------------------------------------------ fixtures
def anchor_prefers_stable(seed=1):
    """test_cycles.cpp:36-53: run_batch tight, helper wild -> run_batch."""
    u = rng_uniform(seed)
    spec, t = [], 0
    for _ in range(500):
        spec.append(ev("run_batch", t, 1000 + int(u(-50, 50))))
        spec.append(ev("helper", t + 10, 500 + int(u(0, 2000))))
        t += 2000
    return spec


def too_few_calls():
    """test_cycles.cpp:55-61: nothing exceeds min calls -> NoAnchorFound."""
    return [ev("f", 0, 10), ev("f", 100, 10)]


def identical_candidates():
    """test_cycles.cpp:63-72: identical stats tie-break by name -> 'a'."""
    spec = []
    for i in range(20):
        spec.append(ev("b", i * 100, 10))
        spec.append(ev("a", i * 100 + 50, 10))
    return spec


def three_anchors():
    """test_cycles.cpp:74-85: anchors at 0/10/20 -> [0,10), [10,20)."""
    return [ev("run_batch", 0, 8), ev("run_batch", 10, 8), ev("run_batch", 20, 8)]


def component_durations():
    """test_cycles.cpp:87-95: run_batch component inside one cycle == 6."""
    return [ev("anchor", 0, 10), ev("anchor", 10, 10), ev("run_batch", 2, 6)]


def forward_mode_priority():
    """test_cycles.cpp:120-133."""
    return [ev("run_batch", i * 100, 80, fm=("decode" if i == 1 else "prefill")) for i in range(3)]


def keyword_stages():
    """test_cycles.cpp:135-147."""
    return [ev("run_batch", 0, 80), ev("forward_prefill", 10, 20), ev("run_batch", 100, 80),
            ev("process_batch_result_decode", 110, 20), ev("run_batch", 200, 80)]


def temporal_heuristic():
    """test_cycles.cpp:149-172: 8 unknown, decodes, then one prefill."""
    spec, t = [], 0
    for _ in range(20):
        spec.append(ev("run_batch", t, 80))
        t += 100
    t += 80
    spec.append(ev("run_batch", t, 1180))
    spec.append(ev("run_batch", t + 1200, 80))
    return spec


def workload_wkv():
    """test_cycles.cpp:184-197: B=4, L_in=100, L_out=28 -> W_kv=512."""
    return [ev("run_batch", 0, 80, batch=4, input_len=100, output_len=28), ev("run_batch", 100, 80)]


def missing_batch():
    """test_cycles.cpp:211-218."""
    return [ev("run_batch", 0, 80), ev("run_batch", 100, 80)]


def frequency_fallback():
    """test_cycles.cpp:220-234: GPU kernels every 5 ms, no python spans."""
    spec = []
    for i in range(200):
        spec.append(ev("kern_a", i * 5_000_000, 400_000, cat="gpu_kernel"))
        spec.append(ev("kern_b", i * 5_000_000 + 500_000, 1_200_000, cat="gpu_kernel"))
    return spec


def beta_029():
    """test_rca.cpp:100-119: oncpu 0.9 ms + 2.0 ms in a 10 ms cycle -> 0.29."""
    return [ev("run_batch", 0, 9_800_000), ev("run_batch", 10_000_000, 9_800_000),
            ev("oncpu", 1_000_000, 900_000, cat="os_sched"),
            ev("oncpu", 5_000_000, 2_000_000, cat="os_sched")]


def edge_cases():
    """Equal timestamps, zero-length cycles, spans crossing the cycle end,
    negative idle gaps, an 'other' forward_mode, collective duplicates,
    counters, missing lens and negative workload args."""
    spec = []
    t = 0
    for i in range(40):
        fm = "decode" if i % 7 else None
        if i == 11:
            fm = "other"
        spec.append(ev("run_batch", t, 900 if i != 5 else 1300, fm=fm,
                       batch=(None if i == 13 else (-1 if i == 17 else 4 + i)),
                       input_len=(None if i == 15 else 10 * i), output_len=i))
        spec.append(ev("oncpu", t, 200, cat="os_sched"))           # same start as anchor
        spec.append(ev("oncpu", t + 50, 2000, cat="os_sched"))     # crosses the cycle end
        spec.append(ev("reduce", t + 100, 300, cat="collective_comm", comm="c0", rank=0))
        spec.append(ev("reduce", t + 150, 300, cat="collective_comm", comm="c0", rank=1))
        if i % 5 == 0:
            spec.append(ev("reduce", t + 400, 100, cat="collective_comm", comm="c0", rank=0))
        spec.append(ev("gpu_usage", t + 300, kind="counter", cat="counter_telemetry", value=50.0 + i))
        spec.append(ev("process_batch_result", t + 600, 150))
        if i == 20:
            spec.append(ev("run_batch", t, 700, fm="decode", batch=1, input_len=1, output_len=1))
        t += 1000 + (i % 3) * 37
    spec.append(ev("run_batch", t, 10))
    return spec


ALL = {
    "anchor_prefers_stable": anchor_prefers_stable,
    "too_few_calls": too_few_calls,
    "identical_candidates": identical_candidates,
    "three_anchors": three_anchors,
    "component_durations": component_durations,
    "forward_mode_priority": forward_mode_priority,
    "keyword_stages": keyword_stages,
    "temporal_heuristic": temporal_heuristic,
    "workload_wkv": workload_wkv,
    "missing_batch": missing_batch,
    "frequency_fallback": frequency_fallback,
    "beta_029": beta_029,
    "edge_cases": edge_cases,
}

# CycleConfig variations some fixtures need (the reference tests call
# segment(trace, "anchor") directly with an explicit name)
CONFIG = {
    "component_durations": {"cycle": {"anchor_hint": "anchor"}},
    "three_anchors": {"cycle": {"anchor_hint": "run_batch"}},
    "forward_mode_priority": {"cycle": {"anchor_hint": "run_batch"}},
    "keyword_stages": {"cycle": {"anchor_hint": "run_batch"}},
    "workload_wkv": {"cycle": {"anchor_hint": "run_batch"}},
    "missing_batch": {"cycle": {"anchor_hint": "run_batch"}},
    "beta_029": {"cycle": {"anchor_hint": "run_batch"}},
    "edge_cases": {"cycle": {"anchor_hint": "run_batch"}},
}
