"""GPU: the drop-in boundary beyond segment_and_classify.

- the reference's OWN unit tests (proj/tests/test_cycles.cpp, test_detector.cpp,
  test_rca.cpp) compiled against the C++ drop-in (dropin/cyclescope_dropin.cpp,
  linked first: rank_anchor_candidates, discover_anchor, segment,
  classify_stages, extract_workload, segment_by_frequency,
  segment_and_classify, build_cycle_records (both overloads), cycle_stats,
  evaluate_strategy(ies) served by the GPU) pass;
- the C-ABI entry points behind them, bitwise against the reference:
  cs_get_candidates_exact (incl. periodicity), cs_set_cycles + CS_RUN_GIVEN
  (records of caller cycles, classify_stages of caller cycles) and
  cs_detect_residuals (Detector::step over a stream + evaluate_strategy).
"""
import os
import subprocess

import numpy as np
import pytest

from helpers import assert_cycles_equal, assert_records_equal
from paper_2601_09258_b200 import abi
from paper_2601_09258_b200 import runtime as rt

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")


@pytest.mark.parametrize("name", ["test_cycles", "test_detector", "test_rca"])
def test_reference_unit_tests_pass_on_the_gpu_dropin(name):
    exe = os.path.join(REF, f"{name}_gpu")
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (make -C oracle dropin_tests needs /root/reference)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    assert "failed: 0" in p.stdout
    # the drop-in really served them: its device session shows up in the symbols
    nm = subprocess.run(["nm", "-C", exe], capture_output=True, text=True).stdout
    assert "cs_run" in nm


def _setup(an, ex, run_config=None):
    an.configure(ex.names, rt.span_names_mask(ex.events, len(ex.names)), n_comm_slots=len(ex.comm_hash),
                 run_config=run_config)
    an.upload(ex.events, [0, len(ex.events)], ex.workloads)


def test_exact_candidates_equal_reference(refbridge, analyzer):
    for fam, ranks in [("cpu_contention", 1), ("nvlink_saturation", 4)]:
        t = refbridge.RefTrace.synth(3000, 5, 6, fault=fam, onset=2500, duration=100, n_ranks=ranks)
        ref = t.run(None, None, 2400)
        ex = t.export()
        _setup(analyzer, ex)
        analyzer.run(abi.RUN_SEGMENT)
        got = analyzer.candidates_exact(0)
        assert len(got) == len(ref.candidates) >= 3
        for f in ["name_id", "call_count"]:
            assert np.array_equal(got[f], ref.candidates[f]), f
        for f in ["mean_duration_ns", "duration_cv", "score", "periodicity"]:
            assert np.array_equal(got[f].view(np.uint64), ref.candidates[f].view(np.uint64)), f


def test_given_cycles_records_and_classification(refbridge, analyzer):
    t = refbridge.RefTrace.synth(3000, 15, 16, fault="gpu_clock_lock", onset=2500, duration=100, n_ranks=2)
    ref = t.run(None, None, 2400)
    ex = t.export()
    an = analyzer
    _setup(an, ex)
    # build_cycle_records(trace, span<const Cycle>): the reference's cycles with
    # their components give the reference's records
    comp = ref.components.reshape(len(ref.cycles), -1)
    an.set_cycles(ref.cycles, comp)
    an.load_model(rt.LatencyModel.from_json(ref.model_json))
    an.run(abi.RUN_GIVEN | abi.RUN_ALL)
    got = an.result(0)
    assert_cycles_equal(ref.cycles, got.cycles)
    assert_records_equal(ref.records, got.records)
    # a subset of cycles keeps its own indices
    sub = ref.cycles[100:400].copy()
    an.set_cycles(sub, comp[100:400])
    an.run(abi.RUN_GIVEN)
    recs = an.records(0)
    want = ref.records[(ref.records["cycle_index"] >= 100) & (ref.records["cycle_index"] < 400)]
    assert np.array_equal(recs["cycle_index"], want["cycle_index"])
    assert np.array_equal(recs["latency_s"].view(np.uint64), want["latency_s"].view(np.uint64))
    # classify_stages over caller cycles whose stages were wiped
    wiped = ref.cycles.copy()
    wiped["stage"] = 2  # Unknown
    an.set_cycles(wiped)
    an.run(abi.RUN_GIVEN | abi.RUN_CLASSIFY)
    assert np.array_equal(an.cycles(0)["stage"], ref.cycles["stage"])


def test_classify_given_cycles_heuristic(refbridge, analyzer):
    """Stage heuristic (no forward_mode, no keywords) on caller cycles."""
    t = refbridge.RefTrace.synth(1500, 25, 26)
    ex = t.export()
    ev = ex.events.copy()
    ev["flags"] &= np.uint16(~0x3 & 0xFFFF)  # strip forward_mode
    ref_t = refbridge.RefTrace.build(ev, ex.names, ex.workloads, ex.comm_hash, ex.comm_rank,
                                     event_ids=ex.event_ids, sort=False)
    cfg = {"cycle": {"prefill_keywords": ["zz_none"], "decode_keywords": ["zz_none"]}}
    ref = ref_t.run(cfg, None, 300, beta=False)
    an = analyzer
    an.configure(ex.names, rt.span_names_mask(ev, len(ex.names)), n_comm_slots=len(ex.comm_hash),
                 run_config=cfg)
    an.upload(ev, [0, len(ev)], ex.workloads)
    wiped = ref.cycles.copy()
    wiped["stage"] = 2
    an.set_cycles(wiped)
    an.run(abi.RUN_GIVEN | abi.RUN_CLASSIFY)
    got = an.cycles(0)["stage"]
    assert (ref.cycles["stage"] == 0).any() and (ref.cycles["stage"] == 1).any()  # heuristic prefills
    assert np.array_equal(got, ref.cycles["stage"])


@pytest.mark.parametrize("strategy", [0, 1, 2])
def test_detect_residuals_equals_reference_monitor(refbridge, analyzer, strategy):
    t = refbridge.RefTrace.synth(3500, 35, 36, fault="cpu_freq_drop", onset=3000, duration=150)
    name = ["fixed_point", "fixed_window", "dynamic_window"][strategy]
    cfg = {"detector": {"strategy": name, "window": 7, "warmup": 60}}
    ref = t.run(cfg, None, 2400)
    ctl = abi.default_control(strategy)
    ctl.window, ctl.warmup = 7, 60
    st, fl, _ = analyzer.detect_residuals(ref.records["residual"], ctl, ref.ucl)
    assert np.array_equal(st.view(np.uint64), ref.records["statistic"].view(np.uint64))
    assert np.array_equal(fl & 1, ref.records["armed"])
    assert np.array_equal((fl >> 1) & 1, ref.records["flagged"])
    assert np.array_equal((fl >> 2) & 1, ref.records["alert"])
    # evaluate_strategy: labels per sample -> the reference arithmetic (counts from the flags)
    labels = np.zeros(len(st), np.uint8)
    labels[(ref.records["cycle_index"] >= 3000) & (ref.records["cycle_index"] < 3150)] = 1
    _, _, m = analyzer.detect_residuals(ref.records["residual"], ctl, ref.ucl, labels)
    armed = (fl & 1).astype(bool)
    flg = ((fl >> 1) & 1).astype(bool)
    lab = labels.astype(bool)
    assert m.tp == int((armed & flg & lab).sum()) and m.fp == int((armed & flg & ~lab).sum())
    assert m.fn == int((armed & ~flg & lab).sum()) and m.tn == int((armed & ~flg & ~lab).sum())
    assert m.alerts == int(((fl >> 2) & 1).sum())
