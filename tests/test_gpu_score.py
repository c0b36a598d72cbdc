"""GPU: every scoring kernel against the reference (gbdt.cpp:22-30, 173-184;
detector.cpp:14-19).

- k_score<NF> (complete-tree traversal): Extended (5-feature) models trained by
  the reference, and 2-feature Physical models with the cell table disabled
  (CS_OPT_TRAVERSAL), i.e. the path 2-feature models take past the table cap;
- k_score_lut_flat (cell table): the default for <= 2 features;
- a batch whose instances use models with different feature counts.
Residuals, predictions and alerts are compared bitwise.
"""
import numpy as np
import pytest

from helpers import assert_full_parity, run_product
from paper_2601_09258_b200 import abi
from paper_2601_09258_b200 import runtime as rt

pytestmark = pytest.mark.gpu


def _ref_and_product(refbridge, analyzer, trace, run_config, traversal):
    ref = trace.run(run_config, None, 2400)
    assert ref.status == 0, (ref.err_type, ref.err_msg)
    ex = trace.export(run_config)
    analyzer.set_traversal(traversal)
    try:
        got, _ = run_product(ex.events, ex.names, ex.workloads, n_comm=len(ex.comm_hash),
                             run_config=run_config, model_json=ref.model_json, analyzer=analyzer)
    finally:
        analyzer.set_traversal(False)
    return ref, got


@pytest.mark.parametrize("cfg,traversal", [
    ({"feature_set": "extended"}, False),
    ({"feature_set": "extended", "gbdt": {"max_depth": 7, "n_trees": 120}}, False),
    ({"feature_set": "extended", "detector": {"strategy": "fixed_window", "window": 5}}, False),
    ({}, True),
    ({"gbdt": {"max_depth": 3}}, True),
], ids=["extended", "extended_d7", "extended_fixed_window", "physical_traversal", "physical_d3_traversal"])
def test_traversal_scorer_matches_reference(refbridge, analyzer, cfg, traversal):
    t = refbridge.RefTrace.synth(3800, 91, 92, fault="memory_thrash", onset=3000, duration=150,
                                 n_ranks=2, target_rank=1)
    ref, got = _ref_and_product(refbridge, analyzer, t, cfg, traversal)
    assert len(ref.alerts) >= 1
    assert_full_parity(ref, got)


def test_mixed_feature_counts_in_one_batch(refbridge, analyzer):
    """Instance 0 monitored with a Physical (2-feature, cell table) model,
    instance 1 with an Extended (5-feature) one, in one cs_run."""
    ts = [refbridge.RefTrace.synth(3000, 101 + k, 102 + k, fault="cpu_freq_drop", onset=2600,
                                   duration=150) for k in range(2)]
    cfgs = [{}, {"feature_set": "extended"}]
    refs = [t.run(c, None, 2400) for t, c in zip(ts, cfgs)]
    exs = [t.export() for t in ts]
    assert exs[0].names == exs[1].names
    evs, wls, offs, base = [], [], [0], 0
    for e in exs:
        ev = e.events.copy()
        has = (ev["flags"] & abi.EV_HAS_BATCH) != 0
        ev["payload"][has] += np.uint64(base)
        base += len(e.workloads)
        evs.append(ev)
        wls.append(e.workloads)
        offs.append(offs[-1] + len(ev))
    an = analyzer
    allev = np.concatenate(evs)
    an.configure(exs[0].names, rt.span_names_mask(allev, len(exs[0].names)),
                 n_comm_slots=len(exs[0].comm_hash))
    an.upload(allev, offs, np.concatenate(wls))
    for i, r in enumerate(refs):
        an.load_model(rt.LatencyModel.from_json(r.model_json), i)
    an.run(abi.RUN_ALL)
    for i, r in enumerate(refs):
        assert_full_parity(r, an.result(i))
