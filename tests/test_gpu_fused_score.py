"""GPU: scoring inside record compaction (batches above kSmallBatch cycles,
cell-table models without record extras) against the reference and against
the separate scoring kernel (option 95).

The fused path records first_bad_record / first_missing_record as absolute
record indices and converts them after the run; a two-instance batch whose
SECOND instance hits NonPositiveLatency (detector.cpp:14-19, main.cpp:162)
checks that conversion: the index must be relative to that instance's own
records, as the reference reports it.
"""
import numpy as np
import pytest

from paper_2601_09258_b200 import abi

pytestmark = pytest.mark.gpu

N_CYCLES = 40_000  # two instances: 80 k cycles, above the single-CTA batch path
BAD_CYCLE = 35_050


def _traces(refbridge):
    t = refbridge.RefTrace.synth(N_CYCLES, 91, 92, fault="gpu_contention", onset=N_CYCLES - 400,
                                 duration=150)
    probe = t.run({"cycle": {"anchor_hint": "run_batch"}}, None, 2400)
    ex = t.export()
    # cycle BAD_CYCLE spans more than 2^63 ns: its int64 duration wraps
    # negative exactly as the reference computes it (cycles.hpp:75)
    cut = int(probe.cycles["start_ts"][BAD_CYCLE + 1])
    ev = ex.events.copy()
    head = ev["start_ts"] < cut
    ev["start_ts"][head] -= np.int64(4_700_000_000_000_000_000)
    ev["start_ts"][~head] += np.int64(4_600_000_000_000_000_000)
    bt = refbridge.RefTrace.build(ev, ex.names, ex.workloads, ex.comm_hash, ex.comm_rank,
                                  event_ids=ex.event_ids, sort=False)
    return t, bt, ev, ex


def test_fused_scoring_two_instances_non_positive_latency(rt, refbridge):
    cfg = {"cycle": {"anchor_hint": "run_batch"}, "pipeline": {"latency_component": ""}}
    t, bt, ev_bad, ex = _traces(refbridge)
    ref_clean = t.run(cfg, None, 2400)
    ref_bad = bt.run(cfg, ref_clean.model_json, 2400)
    assert ref_bad.err_type == "non_positive_latency"
    ev_clean = ex.events
    launches = {}
    for separate in (False, True):
        an = rt.Analyzer(0)
        an._ck(an.L.cs_set_option(an.h, 95, 1 if separate else 0))
        an.configure(ex.names, rt.span_names_mask(ev_clean, len(ex.names)),
                     n_comm_slots=len(ex.comm_hash), run_config=cfg)
        an.load_model(rt.LatencyModel.from_json(ref_clean.model_json))
        an.upload(np.concatenate([ev_clean, ev_bad]), [0, len(ev_clean), len(ev_clean) + len(ev_bad)],
                  ex.workloads)
        an.run(abi.RUN_ALL)
        launches[separate] = an.launches()
        got_clean, got_bad = an.result(0), an.result(1)
        # instance 0: the clean trace, scored and alerting like the reference
        assert got_clean.status_type == "ok"
        assert np.array_equal(got_clean.alerts["cycle"], ref_clean.alerts["cycle"])
        n = len(ref_clean.records)
        assert np.array_equal(got_clean.records["residual"][:n].view(np.uint64),
                              ref_clean.records["residual"].view(np.uint64))
        # instance 1: stops at its own first bad record, relative to its records
        assert got_bad.status_type == "non_positive_latency"
        assert got_bad.summary.first_bad_record == ref_bad.first_bad_record
        assert np.array_equal(got_bad.alerts["cycle"], ref_bad.alerts["cycle"])
        an.close()
    # the fused run launched no separate scoring kernel
    assert launches[False] == launches[True] - 1, launches
