"""Shared test helpers: run the product on a trace and compare with the oracle.

The oracle is the reference implementation compiled unmodified
(oracle/_ref/libcsref.so via oracle/refbridge.py) and, independently, the C
restatement (oracle/cs_oracle.c via oracle/csoracle.py).
"""
from __future__ import annotations

import numpy as np

from paper_2601_09258_b200 import abi
from paper_2601_09258_b200 import runtime as rt


def run_product(events, names, workloads, n_comm=0, run_config=None, model_json=None,
                mask=abi.RUN_ALL, analyzer=None, fused=False, extras=None):
    """One instance through the C ABI; returns InstanceResult.  extras =
    (keys, refs, values) of the record-extras side table (cs_upload_extras)."""
    an = analyzer or rt.Analyzer()
    an.set_fused(fused)
    span = rt.span_names_mask(events, len(names))
    an.configure(names, span, n_comm_slots=n_comm, run_config=run_config)
    an.upload(events, [0, len(events)], workloads)
    if extras is not None:
        an.upload_extras(*extras)
    if model_json and (mask & (abi.RUN_SCORE | abi.RUN_DETECT)):
        an.load_model(rt.LatencyModel.from_json(model_json))
    an.run(mask)
    scored = bool(mask & abi.RUN_DETECT)
    return an.result(0, beta=bool(mask & abi.RUN_BETA), scored=scored), an


CYCLE_FIELDS = ["index", "start_ts", "end_ts", "anchor_pos", "anchor_span_end", "first_event",
                "last_event", "stage", "workload_status"]
RECORD_EXACT = ["cycle_index", "start_ts", "batch", "input_len", "output_len", "stage"]
RECORD_FLOAT = ["latency_s", "predicted_s", "residual", "statistic"]


def assert_cycles_equal(ref_cycles, got_cycles):
    assert len(ref_cycles) == len(got_cycles), (len(ref_cycles), len(got_cycles))
    for f in CYCLE_FIELDS:
        a, b = ref_cycles[f], got_cycles[f]
        if not np.array_equal(a, b):
            bad = np.nonzero(a != b)[0]
            raise AssertionError(f"cycle field {f} differs at {bad[:5]}: ref {a[bad[:5]]} got {b[bad[:5]]}")


def assert_records_equal(ref_recs, got_recs, n=None, bitexact=True, rtol=1e-6):
    n = len(ref_recs) if n is None else n
    assert len(got_recs) >= n, (len(got_recs), n)
    a, b = ref_recs[:n], got_recs[:n]
    for f in RECORD_EXACT + ["armed", "flagged", "alert"]:
        if not np.array_equal(a[f], b[f]):
            bad = np.nonzero(a[f] != b[f])[0]
            raise AssertionError(f"record field {f} differs at {bad[:5]}: {a[f][bad[:5]]} vs {b[f][bad[:5]]}")
    for f in RECORD_FLOAT:
        x, y = a[f], b[f]
        if bitexact:
            ok = x.view(np.uint64) == y.view(np.uint64)
        else:
            ok = np.isclose(x, y, rtol=rtol, atol=0.0)
        if not ok.all():
            bad = np.nonzero(~ok)[0]
            raise AssertionError(f"record field {f} differs at {bad[:5]}: {x[bad[:5]]!r} vs {y[bad[:5]]!r}")
    al = a["alert"].astype(bool)
    assert np.array_equal(a["episode_id"][al], b["episode_id"][al])


def assert_alerts_equal(ref_alerts, got_alerts):
    assert len(ref_alerts) == len(got_alerts), (len(ref_alerts), len(got_alerts))
    for f in ["cycle", "ts", "strategy", "batch", "input_len", "output_len", "episode_id",
              "record_index"]:
        assert np.array_equal(ref_alerts[f], got_alerts[f]), f
    for f in ["smoothed_error", "limit"]:
        assert np.array_equal(ref_alerts[f].view(np.uint64), got_alerts[f].view(np.uint64)), f


def assert_full_parity(ref, got, n_cycles_check=True, beta=True):
    """ref: oracle.refbridge.RefResult; got: runtime.InstanceResult."""
    assert ref.status == 0 or got.summary.status != 0, (ref.err_type, got.status_type)
    assert_cycles_equal(ref.cycles, got.cycles)
    assert np.array_equal(ref.components, got.components)
    if beta:
        assert np.array_equal(ref.beta_totals, got.beta_totals)
        assert np.array_equal(ref.beta.view(np.uint64), got.beta.view(np.uint64))
        assert np.array_equal(ref.coll_present, got.coll_present)
        assert np.array_equal(ref.coll_beta.view(np.uint64), got.coll_beta.view(np.uint64))
    if ref.status == 0:
        assert_records_equal(ref.records, got.records)
        assert_alerts_equal(ref.alerts, got.alerts)
        assert got.summary.ucl == ref.ucl
