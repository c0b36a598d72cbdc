"""Whole-trace parity at scale: the product's one-shot analysis of a large
8-rank instance (the configs[1] shape) against the reference run over the
SAME trace in cycle-aligned chunks with one Detector stepping every record
in order (oracle/refbridge.full_parity -> ref_full_parity).  Every cycle,
component, beta, collective beta, record (latency, prediction, residual,
statistic, flags) and alert is compared bitwise.  bench.py reports the same
comparison on the full benchmarked 99.9 M-event trace (`parity`).
"""
import os

import numpy as np
import pytest

from paper_2601_09258_b200 import abi

pytestmark = pytest.mark.gpu


def _fit(rt, an):
    recs = an.records(0)
    t = recs[recs["cycle_index"] < 2400]
    x = np.stack([t["batch"].astype(float), (t["batch"] * (t["input_len"] + t["output_len"])).astype(float)], 1)
    return rt.fit_latency_model(x, t["latency_s"])


@pytest.mark.parametrize("cycles,chunk", [(200_000, 250_000), (60_000, 7_000)])
def test_whole_trace_parity_8_ranks(rt, refbridge, cycles, chunk):
    tr = rt.synth_trace(cycles, 7, 8, fault="nvlink_saturation", onset=cycles - 20_000, duration=150,
                        target_rank=3, n_ranks=8, n_chunks=8, n_threads=os.cpu_count(),
                        compact_names=False)
    an = rt.Analyzer(0)
    try:
        an.configure(tr.names, rt.span_names_mask(tr.events, len(tr.names)), n_comm_slots=tr.n_comm)
        an.upload(tr.events, [0, len(tr.events)], tr.workloads)
        an.run(abi.RUN_SEGMENT)
        model = _fit(rt, an)
        an.load_model(model)
        an.run(abi.RUN_ALL)
        anchor = tr.names[an.summary(0).anchor_name_id]
        out = refbridge.full_parity(an, tr.events, tr.names, tr.workloads, tr.n_comm, model.to_json(),
                                    anchor, os.cpu_count() or 4, chunk_events=chunk)
    finally:
        an.close()
    assert out["events_compared"] == len(tr.events)
    assert not out["stages_from_heuristic"]
    assert out["alerts_compared"] >= 1, out
    assert out["identical"], out
