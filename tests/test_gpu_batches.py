"""GPU: fleet-shaped batches — many instances of uneven size in one upload,
including an empty instance and one shorter than a cycle — through cs_upload
and the wire format (cs_upload_wire), every instance equal to the C oracle run
on that instance alone (status, cycles, components, beta, records, alerts)."""
import numpy as np
import pytest

from helpers import assert_alerts_equal, assert_cycles_equal, assert_records_equal
from oracle import csoracle
from paper_2601_09258_b200 import abi, runtime as rt

pytestmark = pytest.mark.gpu

FAULTS = [None, "cpu_contention", "gpu_clock_lock", "nvlink_saturation"]


@pytest.fixture(scope="module")
def fleet():
    parts = []
    for i in range(24):
        n = [3000, 40, 700, 2600, 1200][i % 5] + 13 * i
        t = rt.synth_trace(n, 300 + i, 400 + i, fault=FAULTS[i % 4], onset=max(1, n - 300), duration=120,
                           n_ranks=1 + i % 3, compact_names=False)
        ev, wl = t.events, t.workloads
        if i == 5:
            ev = ev[:0]  # empty instance
        if i == 11:
            ev = ev[:12]  # shorter than one cycle
        parts.append((ev, wl, t.n_comm))
    names = rt.synth_trace(10, 1, 2, compact_names=False).names
    rc = {"cycle": {"anchor_hint": "run_batch"}}
    ref0 = csoracle.analyze(parts[0][0], names, parts[0][1], parts[0][2], rc, None)
    r = ref0["records"][:2400]
    x = np.stack([r["batch"].astype(float), (r["batch"] * (r["input_len"] + r["output_len"])).astype(float)], 1)
    model = rt.fit_latency_model(x, r["latency_s"]).to_json()
    # the batch: payloads rebased into one workload table
    evs, offs, base = [], [0], 0
    for ev, wl, _ in parts:
        e = ev.copy()
        has = (e["flags"] & abi.EV_HAS_BATCH) != 0
        e["payload"][has] = (e["payload"][has] & np.uint64(0xFFFFFFFF00000000)) | \
            ((e["payload"][has] & np.uint64(0xFFFFFFFF)) + np.uint64(base))
        base += len(wl)
        evs.append(e)
        offs.append(offs[-1] + len(e))
    events = np.concatenate(evs)
    workloads = np.concatenate([p[1] for p in parts])
    span = rt.span_names_mask(events, len(names))
    n_comm = max(p[2] for p in parts)
    refs = [csoracle.analyze(ev, names, wl, n_comm, rc, model, span=span) for ev, wl, _ in parts]
    return names, span, n_comm, rc, model, events, offs, workloads, refs


@pytest.mark.parametrize("path", ["events", "wire"])
def test_fleet_batch_each_instance_equals_oracle(fleet, path):
    names, span, n_comm, rc, model, events, offs, workloads, refs = fleet
    an = rt.Analyzer(0)
    an.configure(names, span, n_comm_slots=n_comm, run_config=rc)
    if path == "wire":
        an.upload_wire(rt.wire_pack(events, offs, workloads))
    else:
        an.upload(events, offs, workloads)
    an.load_model(rt.LatencyModel.from_json(model))
    an.run(abi.RUN_ALL)
    for i, ref in enumerate(refs):
        got = an.result(i)
        assert (got.summary.status == 0) == (ref["status"] == 0), (i, got.status_type, ref["status"])
        if ref["status"] != 0:
            assert abi.STATUS_TYPES[ref["status"]] == got.status_type, i
        assert_cycles_equal(ref["cycles"], got.cycles)
        assert np.array_equal(ref["components"].reshape(-1), got.components.reshape(-1)), i
        assert np.array_equal(ref["beta_totals"].reshape(-1), got.beta_totals.reshape(-1)), i
        assert np.array_equal(ref["beta"].reshape(-1).view(np.uint64), got.beta.reshape(-1).view(np.uint64)), i
        assert_records_equal(ref["records"], got.records)
        assert_alerts_equal(ref["alerts"], got.alerts)
    assert sum(len(r["alerts"]) for r in refs) >= 3
    an.close()
