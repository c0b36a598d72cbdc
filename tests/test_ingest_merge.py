"""cmd_ingest's clock unification natively (cs_ingest_merge): beacons ->
calibrate -> apply_calibration -> merge_traces (align.cpp:22-206,
main.cpp:80-97) vs the reference's own pipeline on the same documents:
identical merged records, event ids, names, workload table, collective slots
and topology; the reference's errors for domains without beacons and for
inconsistent beacons."""
import json

import numpy as np
import pytest

from paper_2601_09258_b200 import runtime as rt


def _doc(seed, clock=None, beacons=(), n=600, ranks=2, drift=1.0, offset=0.0, eid0=1):
    rng = np.random.default_rng(seed)
    recs = []
    src = {"clock": clock, "node": f"n{seed}"} if clock else None
    t = 1000.0
    for i in range(n):
        t += float(rng.integers(1, 40)) + (0.25 if i % 7 == 0 else 0.0)
        kind = i % 6
        if kind == 0:
            r = {"ph": "X", "name": "run_batch", "ts": t, "dur": float(rng.integers(5, 30)),
                 "args": {"batch_size": int(rng.integers(1, 64)), "input_len": int(rng.integers(1, 900)),
                          "output_len": int(rng.integers(1, 200)), "forward_mode": "decode"}}
        elif kind == 1:
            r = {"ph": "X", "name": "gemm_kernel", "ts": t, "dur": 3.5, "cat": "gpu_kernel"}
        elif kind == 2:
            r = {"ph": "C", "name": "gpu_usage", "ts": t, "args": {"value": float(rng.random() * 100)}}
        elif kind == 3:
            rk = int(rng.integers(0, ranks))
            r = {"ph": "X", "name": "reduce", "ts": t, "dur": 2.0, "cat": "collective_comm",
                 "args": {"commHash": f"c{seed % 2}", "rank": rk, "hostname": f"h{rk}", "device": rk}}
        elif kind == 4:
            r = {"ph": "i", "name": "marker", "ts": t}
        else:
            r = {"ph": "X", "name": "decode_step", "ts": t, "dur": 1.25, "eid": eid0 + i}
        if src:
            r["src"] = src
        recs.append(r)
    for local in beacons:
        ref = int(round(offset + drift * local * 1000))
        r = {"ph": "i", "name": "beacon", "ts": local, "args": {"reference_ts": ref}}
        if src:
            r["src"] = src
        recs.append(r)
    return json.dumps({"traceEvents": recs}).encode()


def _compare_merge(refbridge, docs, **kw):
    ref = refbridge.RefTrace.merge(docs, **kw)
    try:
        got = rt.ingest_merge(docs, **kw)
    except rt.EngineError as e:
        assert isinstance(ref, tuple) and ref == ("error", e.type)
        return None
    assert not isinstance(ref, tuple), ref
    ex = ref.export(None)
    assert got.names == ex.names
    assert got.events.tobytes() == ex.events.tobytes()
    assert np.array_equal(got.event_ids, ex.event_ids)
    assert got.workloads.tobytes() == ex.workloads.tobytes()
    assert got.comm_hash == ex.comm_hash and list(got.comm_rank) == list(ex.comm_rank)
    assert [list(got.locations[i]) if i >= 0 else None for i in got.comm_location] == ref.topology()
    return got


@pytest.mark.parametrize("drift_fit", [False, True])
def test_merge_three_domains(refbridge, drift_fit):
    a = _doc(1)  # reference domain
    b = _doc(2, "gpu0", beacons=[1500.0, 9000.0, 16000.0], drift=1.00002, offset=-3.5e5)
    c = _doc(3, "host1", beacons=[2000.0], offset=7.7e5, eid0=5)
    got = _compare_merge(refbridge, [a, b, c], estimate_drift=drift_fit, tolerance_ns=1e6)
    assert len(got.events) > 1800 and got.event_ids[0] == 1


def test_merge_identity_and_ties(refbridge):
    d = _doc(4)
    _compare_merge(refbridge, [d, d, d])  # identical timestamps and ids across inputs
    t = refbridge.RefTrace.synth(300, 1, 2, n_ranks=4)
    _compare_merge(refbridge, [t.to_json(), _doc(5)])


def test_merge_errors(refbridge):
    assert _compare_merge(refbridge, [_doc(1), _doc(6, "gpu9")]) is None  # no beacons
    b = _doc(2, "gpu0", beacons=[1500.0, 9000.0, 16000.0], drift=1.001, offset=0.0)
    assert _compare_merge(refbridge, [b], tolerance_ns=10.0) is None        # inconsistent
    with pytest.raises(rt.EngineError) as e:
        rt.ingest_merge([_doc(6, "gpu9")])
    assert e.value.type == "no_beacons"
