"""K0: canonical event order on the device (Trace::sort_events, trace.cpp:103-109).

- cs_upload_unsorted sorts every instance stably by (start_ts, event_id) on the
  device; the analysis of a shuffled trace equals the reference's analysis of
  the trace in canonical order, bit for bit, and cs_get_order maps canonical
  positions back to input positions.
- cs_upload takes canonically ordered events; cs_run detects a decreasing
  start_ts inside its first event pass and fails loudly (no silent wrong cycles).
"""
import numpy as np
import pytest

from helpers import assert_full_parity, run_product
from paper_2601_09258_b200 import abi
from paper_2601_09258_b200 import runtime as rt

pytestmark = pytest.mark.gpu


def _configure(an, ex, run_config=None):
    span = rt.span_names_mask(ex.events, len(ex.names))
    an.configure(ex.names, span, n_comm_slots=len(ex.comm_hash), run_config=run_config)


def _shuffled(ex, rng):
    perm = rng.permutation(len(ex.events))
    return ex.events[perm], ex.event_ids[perm], perm


def test_shuffled_trace_sorted_on_device_matches_reference(refbridge, analyzer):
    t = refbridge.RefTrace.synth(3000, 41, 42, fault="gpu_contention", onset=2500, duration=150,
                                 n_ranks=4, target_rank=1)
    ref = t.run(None, None, 2400)
    ex = t.export()
    rng = np.random.default_rng(7)
    ev_s, ids_s, perm = _shuffled(ex, rng)
    an = analyzer
    _configure(an, ex)
    an.upload_unsorted(ev_s, [0, len(ev_s)], ex.workloads, ids_s)
    order = an.order(0)
    # canonical position k holds input position order[k]
    assert np.array_equal(perm[order], np.arange(len(ev_s)))
    an.load_model(rt.LatencyModel.from_json(ref.model_json))
    an.run(abi.RUN_ALL)
    got = an.result(0, beta=True, scored=True)
    assert_full_parity(ref, got)


def test_equal_timestamps_break_ties_by_event_id(refbridge, analyzer):
    # many events share a start_ts: only the ids decide their canonical order
    t = refbridge.RefTrace.synth(600, 3, 4, n_ranks=8)
    ex = t.export()
    ev = ex.events.copy()
    ev["start_ts"] = (ev["start_ts"] // 2_000_000) * 2_000_000  # coarse clock: ties everywhere
    ids = ex.event_ids
    rng = np.random.default_rng(11)
    perm = rng.permutation(len(ev))
    an = analyzer
    _configure(an, ex)
    an.upload_unsorted(ev[perm], [0, len(ev)], ex.workloads, ids[perm])
    order = an.order(0)
    got_ids = ids[perm][order]
    want = np.lexsort((ids, ev["start_ts"]))  # sort by (start_ts, id)
    assert np.array_equal(got_ids, ids[want])
    # the device analysis of the sorted copy equals the reference on the sorted trace
    srt = ev[want]
    ref_t = refbridge.RefTrace.build(srt, ex.names, ex.workloads, ex.comm_hash, ex.comm_rank,
                                     event_ids=ids[want], sort=False)
    ref = ref_t.run(None, None, 300, beta=True)
    an.run(abi.RUN_SEGMENT | abi.RUN_BETA)
    got = an.result(0, beta=True, scored=False)
    from helpers import assert_cycles_equal
    assert_cycles_equal(ref.cycles, got.cycles)
    assert np.array_equal(ref.components, got.components)


def test_without_ids_input_position_breaks_ties(analyzer):
    tr = rt.synth_trace(400, 1, 2)
    ev = tr.events.copy()
    rng = np.random.default_rng(3)
    perm = rng.permutation(len(ev))
    an = analyzer
    span = rt.span_names_mask(ev, len(tr.names))
    an.configure(tr.names, span, n_comm_slots=tr.n_comm)
    an.upload_unsorted(ev[perm], [0, len(ev)], tr.workloads)
    order = an.order(0)
    # stable by start_ts over the input positions
    want = np.argsort(ev[perm]["start_ts"], kind="stable")
    assert np.array_equal(order, want)


def test_multi_instance_sort_keeps_instances_apart(refbridge, analyzer):
    ts = [refbridge.RefTrace.synth(1500, 50 + k, 60 + k, n_ranks=2) for k in range(3)]
    exs = [t.export() for t in ts]
    # a shared name table: all three exports intern the same simkit names
    assert all(e.names == exs[0].names for e in exs)
    rng = np.random.default_rng(5)
    parts, ids, offs, wls, wl_base = [], [], [0], [], 0
    for e in exs:
        p = rng.permutation(len(e.events))
        ev = e.events[p].copy()
        has = (ev["flags"] & 0x4) != 0
        ev["payload"][has] += wl_base  # workload indices into the concatenated table
        parts.append(ev)
        ids.append(e.event_ids[p])
        offs.append(offs[-1] + len(ev))
        wls.append(e.workloads)
        wl_base += len(e.workloads)
    an = analyzer
    _configure(an, exs[0])
    an.upload_unsorted(np.concatenate(parts), offs, np.concatenate(wls), np.concatenate(ids))
    an.run(abi.RUN_SEGMENT | abi.RUN_BETA)
    for i, (t, e) in enumerate(zip(ts, exs)):
        ref = t.run(None, None, 300, beta=True)
        got = an.result(i, beta=True, scored=False)
        from helpers import assert_cycles_equal
        assert_cycles_equal(ref.cycles, got.cycles)
        assert np.array_equal(ref.components, got.components)
        assert np.array_equal(ref.beta.view(np.uint64), got.beta.view(np.uint64))


def test_checked_upload_rejects_out_of_order_events(refbridge, analyzer):
    t = refbridge.RefTrace.synth(500, 1, 2)
    ex = t.export()
    ev = ex.events.copy()
    k = len(ev) // 2
    ev[[k, k + 40]] = ev[[k + 40, k]]  # one late event
    an = analyzer
    _configure(an, ex)
    an.upload(ev, [0, len(ev)], ex.workloads)
    with pytest.raises(rt.EngineError) as e:
        an.run(abi.RUN_SEGMENT)
    assert e.value.type == "invalid_argument"
    assert "canonical" in str(e.value)
    # the sorted copy runs
    an.upload(ex.events, [0, len(ex.events)], ex.workloads)
    an.run(abi.RUN_SEGMENT)
