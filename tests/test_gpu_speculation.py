"""The single-read pass sizes a run over an unchanged upload and
configuration from the last verified run (no mid-run synchronisation) and
checks the counts at the end.  Results must equal a fresh analyzer's in every
case: repeated runs, a configuration change, a re-upload, and a skewed
speculation that the run has to notice and redo."""
import numpy as np
import pytest

from paper_2601_09258_b200 import abi

pytestmark = pytest.mark.gpu


def _tables(an):
    out = [an.cycles(0).tobytes(), an.records(0).tobytes(), np.asarray(an.components(0)).tobytes()]
    for x in (an.beta(0), an.collective_beta(0)):
        for y in (x if isinstance(x, tuple) else (x,)):
            out.append(np.asarray(y).tobytes())
    return out


def _fresh(rt, tr):
    an = rt.Analyzer(0)
    an.configure(tr.names, rt.span_names_mask(tr.events, len(tr.names)), n_comm_slots=tr.n_comm)
    an.upload(tr.events, [0, len(tr.events)], tr.workloads)
    an.run(abi.RUN_SEGMENT | abi.RUN_BETA)
    r = _tables(an)
    an.close()
    return r


def _same(an, ref):
    assert _tables(an) == ref


def test_speculated_runs_equal_fresh_runs(rt):
    tr = rt.synth_trace(4000, 21, 22, n_ranks=4, fault="nvlink_saturation", onset=3000, duration=150,
                        compact_names=False)
    tr2 = rt.synth_trace(3000, 23, 24, n_ranks=2, compact_names=False)
    an = rt.Analyzer(0)
    an.configure(tr.names, rt.span_names_mask(tr.events, len(tr.names)), n_comm_slots=tr.n_comm)
    an.upload(tr.events, [0, len(tr.events)], tr.workloads)
    ref = _fresh(rt, tr)
    for _ in range(3):  # the second and third run speculate
        an.run(abi.RUN_SEGMENT | abi.RUN_BETA)
        _same(an, ref)
    # a skewed speculation is caught at the final synchronisation and redone
    an._ck(an.L.cs_set_option(an.h, 99, 7))
    an.run(abi.RUN_SEGMENT | abi.RUN_BETA)
    _same(an, ref)
    an.run(abi.RUN_SEGMENT | abi.RUN_BETA)
    _same(an, ref)
    # another upload on the same context: no stale counts
    an.configure(tr2.names, rt.span_names_mask(tr2.events, len(tr2.names)), n_comm_slots=tr2.n_comm)
    an.upload(tr2.events, [0, len(tr2.events)], tr2.workloads)
    ref2 = _fresh(rt, tr2)
    for _ in range(2):
        an.run(abi.RUN_SEGMENT | abi.RUN_BETA)
        _same(an, ref2)
    an.close()


def test_phase_timing_modes_move_no_data(rt):
    """CS_OPT_PHASE_TIMINGS only chooses which device events a run records:
    -1 / 1 every phase, 2 the segmentation pass and the total, 0 the total.
    Tables are identical in every mode; an out-of-range mode is rejected."""
    tr = rt.synth_trace(4000, 31, 32, n_ranks=4, fault="nvlink_saturation", onset=3000, duration=150,
                        compact_names=False)
    an = rt.Analyzer(0)
    an.configure(tr.names, rt.span_names_mask(tr.events, len(tr.names)), n_comm_slots=tr.n_comm)
    an.upload(tr.events, [0, len(tr.events)], tr.workloads)
    an.run(abi.RUN_SEGMENT | abi.RUN_BETA)
    ref = _tables(an)
    full = set(an.timings())
    assert "total" in full and len(full) > 3
    for mode, expect in ((2, None), (0, {"total"}), (1, full), (-1, full)):
        an.set_phase_timings(mode)
        an.run(abi.RUN_SEGMENT | abi.RUN_BETA)
        _same(an, ref)
        got = set(an.timings())
        if expect is None:
            assert "total" in got and got & {"segment_range", "scan_events"} and got < full, got
        else:
            assert got == expect, (mode, got)
        assert all(v >= 0.0 for v in an.timings().values())
    with pytest.raises(Exception):
        an.set_phase_timings(3)
    an.close()
