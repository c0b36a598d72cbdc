"""GPU: streaming micro-batches (BASELINE config 5; monitor_loop, main.cpp:151-177).

A trace fed as time-sliced micro-batches through cs_stream_* gives exactly the
cycles, per-cycle beta, records (residual, statistic, flags, episode ids) and
alerts of one whole-trace cs_run — which the parity suites pin to the
reference.  Batch-local fields (event positions, record_index) are excluded."""
import numpy as np
import pytest

from paper_2601_09258_b200 import abi

pytestmark = pytest.mark.gpu

FM_MASK = 0x3


def _traces(rt, n_inst, strip_fm):
    out = []
    for i in range(n_inst):
        t = rt.synth_trace(1200, 31 + i, 57 + i, fault=["cpu_contention", "memory_thrash",
                                                          "gpu_clock_lock"][i % 3],
                           onset=700, duration=150, compact_names=False)
        if strip_fm:
            t.events["flags"] &= np.uint16(~FM_MASK & 0xFFFF)
        out.append(t)
    return out


def _merge(traces):
    evs, wls, offs, base = [], [], [0], 0
    for t in traces:
        ev = t.events.copy()
        has = (ev["flags"] & abi.EV_HAS_BATCH) != 0
        ev["payload"][has] = (ev["payload"][has] & np.uint64(0xFFFFFFFF00000000)) | \
            ((ev["payload"][has] & np.uint64(0xFFFFFFFF)) + np.uint64(base))
        base += len(t.workloads)
        wls.append(t.workloads)
        evs.append(ev)
        offs.append(offs[-1] + len(ev))
    return evs, np.concatenate(wls), offs


_WINDOWS = {"detector": None, "stage": None}  # set by a test: larger windows everywhere


def _setup(rt, an, traces):
    names = traces[0].names
    evs, wl, offs = _merge(traces)
    allev = np.concatenate(evs)
    an.set_fused(False)
    an.configure(names, rt.span_names_mask(allev, len(names)),
                 n_comm_slots=max(t.n_comm for t in traces))
    if _WINDOWS["detector"] or _WINDOWS["stage"]:
        if _WINDOWS["detector"]:
            an.control.window = _WINDOWS["detector"]
        if _WINDOWS["stage"]:
            an.cycle.stage_window = _WINDOWS["stage"]
        an.set_config(an.cycle, an.control)
    return evs, wl, offs, allev


def _fit(rt, an, n_inst):
    models = []
    for i in range(n_inst):
        recs = an.records(i)
        tr = recs[recs["cycle_index"] < 500]
        x = np.stack([tr["batch"].astype(float),
                      (tr["batch"] * (tr["input_len"] + tr["output_len"])).astype(float)], 1)
        models.append(rt.fit_latency_model(x, tr["latency_s"]))
    return models


def _cat(parts, dtype):
    return np.concatenate(parts) if parts else np.zeros(0, dtype)


def _calibration_anchors(rt, traces, first):
    """The anchor each instance's first micro-batch (events before `first`)
    discovers; the stream keeps it for the rest of the trace."""
    cal = rt.Analyzer(0)
    evs, wl, offs, _ = _setup(rt, cal, traces)
    head = [e[e["start_ts"] < first] for e in evs]
    off = np.zeros(len(head) + 1, np.uint64)
    off[1:] = np.cumsum([len(h) for h in head])
    cal.upload(np.concatenate(head), off, wl)
    cal.run(abi.RUN_SEGMENT)
    out = [cal.summary(i).anchor_name_id for i in range(len(traces))]
    cal.close()
    return out


def _whole_trace_reference(rt, traces, anchors):
    """One whole-trace run per distinct anchor (anchor_hint), models fit on
    its records; returns (results, models) per instance."""
    n_inst = len(traces)
    ref, models = [None] * n_inst, [None] * n_inst
    for a in sorted(set(anchors)):
        whole = rt.Analyzer(0)
        evs, wl, offs, allev = _setup(rt, whole, traces)
        whole.cycle.anchor_hint_name = a
        whole.set_config(whole.cycle, whole.control)
        whole.upload(allev, offs, wl)
        whole.run(abi.RUN_SEGMENT)
        fitted = _fit(rt, whole, n_inst)
        for i, m in enumerate(fitted):
            whole.load_model(m, i)
        whole.run(abi.RUN_ALL)
        for i in range(n_inst):
            if anchors[i] == a:
                ref[i], models[i] = whole.result(i), fitted[i]
        whole.close()
    return ref, models


@pytest.mark.parametrize("n_inst,strip_fm,slice_ms,hint,windows", [(1, False, 37.0, True, None),
                                                                    (3, False, 113.0, False, None),
                                                                    (2, True, 61.0, False, None),
                                                                    (1, False, 10.0, True, None),
                                                                    (2, True, 41.0, False, (100, 48))])
def test_stream_equals_whole_trace(rt, n_inst, strip_fm, slice_ms, hint, windows):
    _WINDOWS["detector"], _WINDOWS["stage"] = windows or (None, None)
    try:
        _stream_equals_whole_trace(rt, n_inst, strip_fm, slice_ms, hint)
    finally:
        _WINDOWS["detector"] = _WINDOWS["stage"] = None


def _stream_equals_whole_trace(rt, n_inst, strip_fm, slice_ms, hint):
    """hint=True: the anchor is given (anchor_hint); False: the first
    micro-batch (a calibration window of 20% of the trace) discovers it and
    the stream keeps it, so the whole-trace reference runs with that anchor
    (the calibration window may rank candidates differently from the whole
    trace: memory_thrash does)."""
    traces = _traces(rt, n_inst, strip_fm)
    evs = [t.events for t in traces]
    t_end = max(int(e["start_ts"].max()) for e in evs) + 1
    t0 = min(int(e["start_ts"].min()) for e in evs)
    first = t0 + (0 if hint else (t_end - t0) // 5)
    if hint:
        whole = rt.Analyzer(0)
        _, wl, offs, allev = _setup(rt, whole, traces)
        whole.upload(allev, offs, wl)
        whole.run(abi.RUN_SEGMENT)
        anchors = [whole.summary(i).anchor_name_id for i in range(n_inst)]
        whole.close()
        assert len(set(anchors)) == 1
    else:
        anchors = _calibration_anchors(rt, traces, max(first, t0 + int(slice_ms * 1e6)))
    ref, models = _whole_trace_reference(rt, traces, anchors)
    assert all(len(r.alerts) >= 1 for r in ref)

    an = rt.Analyzer(0)
    evs, wl, offs, allev = _setup(rt, an, traces)
    if hint:
        an.cycle.anchor_hint_name = anchors[0]
        an.set_config(an.cycle, an.control)
    for i, m in enumerate(models):
        an.load_model(m, i)
    st = an.stream()
    step = int(slice_ms * 1e6)
    got = [dict(cyc=[], beta=[], rec=[], al=[]) for _ in range(n_inst)]
    n_batches = 0
    bounds = [t0] + list(range(max(first, t0 + step), t_end, step)) + [t_end]
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        batch = []
        for e in evs:
            a, b = np.searchsorted(e["start_ts"], [lo, hi], side="left")
            batch.append(e[a:b])
        res = st.push(batch, wl)
        n_batches += 1
        for i, r in enumerate(res):
            if r.summary.status == 0:
                got[i]["cyc"].append(r.cycles)
                got[i]["beta"].append(r.beta)
                got[i]["rec"].append(r.records)
                got[i]["al"].append(r.alerts)
    st.close()
    assert n_batches > 10
    for i in range(n_inst):
        cyc = _cat(got[i]["cyc"], abi.CYCLE_DTYPE)
        for f in ["index", "start_ts", "end_ts", "anchor_span_end", "stage", "workload_status"]:
            assert np.array_equal(cyc[f], ref[i].cycles[f]), (i, f)
        beta = np.concatenate(got[i]["beta"])
        assert np.array_equal(beta.view(np.uint64), ref[i].beta.view(np.uint64))
        rec = _cat(got[i]["rec"], abi.RECORD_DTYPE)
        assert len(rec) == len(ref[i].records)
        for f in ["cycle_index", "start_ts", "batch", "input_len", "output_len", "stage", "armed",
                  "flagged", "alert", "episode_id"]:
            assert np.array_equal(rec[f], ref[i].records[f]), (i, f)
        for f in ["latency_s", "predicted_s", "residual", "statistic"]:
            assert np.array_equal(rec[f].view(np.uint64), ref[i].records[f].view(np.uint64)), (i, f)
        al = _cat(got[i]["al"], abi.ALERT_DTYPE)
        for f in ["cycle", "ts", "batch", "episode_id"]:
            assert np.array_equal(al[f], ref[i].alerts[f]), (i, f)
        assert np.array_equal(al["smoothed_error"].view(np.uint64),
                              ref[i].alerts["smoothed_error"].view(np.uint64))
    an.close()


def test_native_push_equals_python_push(rt):
    """cs_stream_push (tails, upload, run and alert gather in the library)
    gives the alerts of the Python-driven micro-batch loop, and the union of
    its alerts equals the whole-trace run's (with and without per-phase
    device events)."""
    traces = _traces(rt, 3, False)
    evs = [t.events for t in traces]
    t_end = max(int(e["start_ts"].max()) for e in evs) + 1
    t0 = min(int(e["start_ts"].min()) for e in evs)
    first = t0 + (t_end - t0) // 5  # calibration window: the first push discovers the anchors
    anchors = _calibration_anchors(rt, traces, first)
    ref, models = _whole_trace_reference(rt, traces, anchors)
    step = int(23e6)
    bounds = [t0] + list(range(first, t_end, step)) + [t_end]
    got = {}
    for native in (False, True):
        an = rt.Analyzer(0)
        evs, wl2, _, _ = _setup(rt, an, traces)  # payloads remapped into the merged table
        for i, m in enumerate(models):
            an.load_model(m, i)
        st = an.stream()
        alerts = []
        for k, (lo, hi) in enumerate(zip(bounds[:-1], bounds[1:])):  # noqa: B007
            batch = []
            for e in evs:
                a, b = np.searchsorted(e["start_ts"], [lo, hi], side="left")
                batch.append(e[a:b])
            if native:
                alerts.append(st.push_native(batch, wl2 if k == 0 else None))
                # CS_OPT_PHASE_TIMINGS: a push records its total only unless
                # asked (the option moves no data: alerts stay equal)
                if k == 1:
                    assert list(an.timings()) == ["total"]
                    an.set_phase_timings(1)
                elif k == 2:
                    assert "total" in an.timings() and len(an.timings()) > 1
            else:
                res = st.push(batch, wl2)
                alerts += [r.alerts for r in res if r.summary.status == 0]
        st.close()
        an.close()
        got[native] = np.concatenate(alerts)
    key = lambda a: sorted(zip(a["cycle"].tolist(), a["ts"].tolist(), a["episode_id"].tolist()))
    assert key(got[True]) == key(got[False])
    whole_alerts = np.concatenate([r.alerts for r in ref])
    assert key(got[True]) == key(whole_alerts)


def _ref_stream_setup(rt, refbridge, t, cfg):
    ref = t.run(cfg, None, 2400)
    ex = t.export(cfg)
    an = rt.Analyzer(0)
    an.configure(ex.names, rt.span_names_mask(ex.events, len(ex.names)),
                 n_comm_slots=len(ex.comm_hash), run_config=cfg)
    an.load_model(rt.LatencyModel.from_json(ref.model_json))
    return ref, ex, an


@pytest.mark.parametrize("slice_ms,ranks", [(10.0, 1), (37.0, 4)])
def test_stream_equals_reference_directly(rt, refbridge, slice_ms, ranks):
    """Micro-batched monitor (configs[4]) vs the reference's whole-trace
    monitor_loop on the SAME trace (no transitivity through device runs):
    cycles, records, residuals, flags and alerts identical."""
    cfg = {"cycle": {"anchor_hint": "run_batch"}}
    t = refbridge.RefTrace.synth(3000, 71 + ranks, 72, fault="gpu_contention", onset=2600,
                                 duration=150, n_ranks=ranks, target_rank=0)
    ref, ex, an = _ref_stream_setup(rt, refbridge, t, cfg)
    assert ref.status == 0 and len(ref.alerts) >= 1
    ev = ex.events
    st = an.stream()
    step = int(slice_ms * 1e6)
    t0, t_end = int(ev["start_ts"][0]), int(ev["start_ts"][-1]) + 1
    cyc, rec, al, al_native = [], [], [], []
    for lo in range(t0, t_end, step):
        a, b = np.searchsorted(ev["start_ts"], [lo, lo + step], side="left")
        r = st.push([ev[a:b]], ex.workloads)[0]
        if r.summary.status == 0:
            cyc.append(r.cycles)
            rec.append(r.records)
            al.append(r.alerts)
    st.close()
    cyc, rec, al = (_cat(cyc, abi.CYCLE_DTYPE), _cat(rec, abi.RECORD_DTYPE), _cat(al, abi.ALERT_DTYPE))
    for f in ["index", "start_ts", "end_ts", "anchor_span_end", "stage", "workload_status"]:
        assert np.array_equal(cyc[f], ref.cycles[f]), f
    assert len(rec) == len(ref.records)
    for f in ["cycle_index", "start_ts", "batch", "input_len", "output_len", "stage", "armed",
              "flagged", "alert"]:
        assert np.array_equal(rec[f], ref.records[f]), f
    for f in ["latency_s", "predicted_s", "residual", "statistic"]:
        assert np.array_equal(rec[f].view(np.uint64), ref.records[f].view(np.uint64)), f
    for f in ["cycle", "ts", "batch", "input_len", "output_len", "episode_id"]:
        assert np.array_equal(al[f], ref.alerts[f]), f
    assert np.array_equal(al["smoothed_error"].view(np.uint64), ref.alerts["smoothed_error"].view(np.uint64))
    # the native push (cs_stream_push) gives the same alerts
    an2 = rt.Analyzer(0)
    an2.configure(ex.names, rt.span_names_mask(ev, len(ex.names)), n_comm_slots=len(ex.comm_hash),
                  run_config=cfg)
    an2.load_model(rt.LatencyModel.from_json(ref.model_json))
    st2 = an2.stream()
    for k, lo in enumerate(range(t0, t_end, step)):
        a, b = np.searchsorted(ev["start_ts"], [lo, lo + step], side="left")
        al_native.append(st2.push_native([ev[a:b]], ex.workloads if k == 0 else None))
    st2.close()
    aln = np.concatenate(al_native)
    for f in ["cycle", "ts", "episode_id"]:
        assert np.array_equal(aln[f], ref.alerts[f]), f
    an.close()
    an2.close()


def _overflow_trace(refbridge, bad_cycle):
    """A simkit trace whose cycle `bad_cycle` spans more than 2^63 ns: its
    duration wraps negative in int64 exactly as the reference computes it
    (cycles.hpp:75), so with latency_component "" the record's latency is
    <= 0 and ppe throws NonPositiveLatency (detector.cpp:14-19); monitor_loop
    stops there (main.cpp:162)."""
    t = refbridge.RefTrace.synth(3000, 81, 82, fault="gpu_contention", onset=2600, duration=150)
    probe = t.run({"cycle": {"anchor_hint": "run_batch"}}, None, 2400)
    ex = t.export()
    cut = int(probe.cycles["start_ts"][bad_cycle + 1])
    ev = ex.events.copy()
    head = ev["start_ts"] < cut
    ev["start_ts"][head] -= np.int64(4_700_000_000_000_000_000)
    ev["start_ts"][~head] += np.int64(4_600_000_000_000_000_000)
    bt = refbridge.RefTrace.build(ev, ex.names, ex.workloads, ex.comm_hash, ex.comm_rank,
                                  event_ids=ex.event_ids, sort=False)
    return t, bt, ev, ex


def test_stream_stays_stopped_after_non_positive_latency(rt, refbridge):
    cfg = {"cycle": {"anchor_hint": "run_batch"}, "pipeline": {"latency_component": ""}}
    t, bt, ev, ex = _overflow_trace(refbridge, 2450)
    ref_clean = t.run(cfg, None, 2400)
    ref = bt.run(cfg, ref_clean.model_json, 2400)
    assert ref.err_type == "non_positive_latency"
    # the fault after the bad cycle alerts in the clean trace, never after the stop
    assert (ref_clean.alerts["cycle"] > 2450).any()
    assert not (ref.alerts["cycle"] > 2450).any()
    an = rt.Analyzer(0)
    an.configure(ex.names, rt.span_names_mask(ev, len(ex.names)), n_comm_slots=len(ex.comm_hash),
                 run_config=cfg)
    an.load_model(rt.LatencyModel.from_json(ref_clean.model_json))
    # whole trace: status non_positive_latency, alerts cut at the bad record
    an.upload(ev, [0, len(ev)], ex.workloads)
    an.run(abi.RUN_ALL)
    whole = an.result(0)
    assert whole.status_type == "non_positive_latency"
    assert whole.summary.first_bad_record == ref.first_bad_record
    assert np.array_equal(whole.alerts["cycle"], ref.alerts["cycle"])
    # stream in event-count slices (time slices cannot cross a 2^63 ns gap)
    st = an.stream()
    got, statuses = [], []
    for a in range(0, len(ev), 9000):
        got.append(st.push_native([ev[a:a + 9000]], ex.workloads if a == 0 else None))
        statuses.append(an.summary(0).status)
    st.close()
    got = np.concatenate(got)
    assert np.array_equal(got["cycle"], ref.alerts["cycle"]), "alerts after the stream stopped"
    assert np.array_equal(got["episode_id"], ref.alerts["episode_id"])
    bad = {v: k for k, v in abi.STATUS_TYPES.items()}["non_positive_latency"]
    assert bad in statuses
    k = statuses.index(bad)
    assert all(s == bad for s in statuses[k:]), statuses
    an.close()
