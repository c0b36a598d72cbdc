"""GPU: BASELINE config 4 (SuiteConfig{} trials: workload drift, sparse true
anomalies) — the per-strategy StrategyMetrics of the reference's own
evaluate_trial (simkit.cpp:796-872) reproduced exactly through the C ABI:
segmentation + records on the device, host fit (byte-identical model),
monitoring from cycle train_cycles, three strategies via cs_redetect, metrics
via cs_evaluate_strategy.  Plus monitor_loop's NDJSON alert sink (A20)."""
import numpy as np
import pytest

from helpers import run_product
from paper_2601_09258_b200 import abi

pytestmark = pytest.mark.gpu


def _fit_on_prefix(rt, an, ex, train_cycles=2400):
    span = rt.span_names_mask(ex.events, len(ex.names))
    cyc, ctl, table = rt.configs_from_json({}, ex.names, span, len(ex.comm_hash))
    an.set_config(cyc, ctl)
    an.set_name_table(table)
    an.upload(ex.events, [0, len(ex.events)], ex.workloads)
    an.run(abi.RUN_SEGMENT)
    recs = an.records(0)
    tr = recs[recs["cycle_index"] < train_cycles]
    x = np.stack([tr["batch"].astype(float),
                  (tr["batch"] * (tr["input_len"] + tr["output_len"])).astype(float)], 1)
    return rt.fit_latency_model(x, tr["latency_s"]), cyc, ctl


@pytest.mark.parametrize("trial", range(8))
def test_config4_strategy_metrics_equal_reference(refbridge, analyzer, rt, trial):
    t = refbridge.RefTrace.trial(trial)
    try:
        ref = t.evaluate_trial(trial)
    except RuntimeError as e:  # the reference's own separability gate
        pytest.skip(str(e))
    ex = t.export()
    labels = t.labels().astype(np.uint8)
    an = analyzer
    an.set_fused(False)
    model, cyc, ctl = _fit_on_prefix(rt, an, ex)
    cyc.monitor_from_cycle = 2400  # evaluate_trial's monitor split (simkit.cpp:837-841)
    an.set_config(cyc, ctl)
    an.load_model(model)
    an.run(abi.RUN_ALL)
    for k, strategy in enumerate([abi.FIXED_POINT, abi.FIXED_WINDOW, abi.DYNAMIC_WINDOW]):
        c = abi.default_control(strategy)
        an.redetect(c)
        m = an.evaluate_strategy(labels)
        got = [m.tp, m.fp, m.fn, m.tn, m.alerts]
        assert got == [int(v) for v in ref[k, :5]], (strategy, got, ref[k])
        assert np.float64(m.f1).view(np.uint64) == ref[k, 5].view(np.uint64)
        assert np.float64(m.fpr).view(np.uint64) == ref[k, 6].view(np.uint64)
        assert np.float64(m.mean_lag).view(np.uint64) == ref[k, 7].view(np.uint64)


def test_evaluate_strategy_requires_labels(analyzer, rt):
    tr = rt.synth_trace(500, 3, 4)
    an = analyzer
    model_json = None
    got, an = run_product(tr.events, tr.names, tr.workloads, n_comm=tr.n_comm,
                          mask=abi.RUN_SEGMENT, analyzer=an)
    recs = got.records
    x = np.stack([recs["batch"].astype(float),
                  (recs["batch"] * (recs["input_len"] + recs["output_len"])).astype(float)], 1)
    an.load_model(rt.fit_latency_model(x, recs["latency_s"]))
    an.run(abi.RUN_ALL)
    with pytest.raises(rt.EngineError) as e:
        an.evaluate_strategy(np.zeros(0, np.uint8))
    assert e.value.type == "no_labels"


@pytest.mark.parametrize("family,strategy", [("cpu_contention", "dynamic_window"),
                                             ("memory_thrash", "fixed_window"),
                                             ("gpu_clock_lock", "fixed_point")])
def test_ndjson_alert_sink_matches_monitor_loop(refbridge, analyzer, rt, family, strategy):
    t = refbridge.RefTrace.synth(4000, 9, 10, fault=family, onset=2600, duration=400)
    cfg = {"detector": {"strategy": strategy}}
    ref = t.run(cfg, None, 2400)
    ex = t.export(cfg)
    got, _ = run_product(ex.events, ex.names, ex.workloads, n_comm=len(ex.comm_hash),
                         run_config=cfg, model_json=ref.model_json, analyzer=analyzer)
    text = rt.alerts_to_ndjson(got.alerts, 5, 20)
    assert text == ref.extra["ndjson"]
    assert len(text.splitlines()) == len(ref.alerts) >= 1


def suite_metrics(refbridge, rt, an, n_trials=20, timer=None):
    """BASELINE config 4 end to end: every SuiteConfig{} trial segmented on the
    device, the 20 latency models fitted in one device batch
    (cs_fit_latency_models), monitored from cycle 2400 under the three
    strategies, pooled as evaluate_suite does.  Returns (ours, reference)
    per-trial metric rows and the trials the reference's own gate skipped."""
    import time
    tick = timer if timer is not None else {}
    prepared, ref_rows, skipped = [], [], []
    for trial in range(n_trials):
        t = refbridge.RefTrace.trial(trial)
        t0 = time.perf_counter()
        try:
            ref = t.evaluate_trial(trial)
        except RuntimeError:
            skipped.append(trial)
            continue
        tick["reference_s"] = tick.get("reference_s", 0.0) + time.perf_counter() - t0
        prepared.append((trial, t.export(), t.labels().astype(np.uint8)))
        ref_rows.append(ref)
    t0 = time.perf_counter()
    xs, ys, cfgs = [], [], []
    for _, ex, _ in prepared:
        span = rt.span_names_mask(ex.events, len(ex.names))
        cyc, ctl, table = rt.configs_from_json({}, ex.names, span, len(ex.comm_hash))
        an.set_config(cyc, ctl)
        an.set_name_table(table)
        an.upload(ex.events, [0, len(ex.events)], ex.workloads)
        an.run(abi.RUN_SEGMENT)
        recs = an.records(0)
        tr = recs[recs["cycle_index"] < 2400]
        xs.append(np.stack([tr["batch"].astype(float),
                            (tr["batch"] * (tr["input_len"] + tr["output_len"])).astype(float)], 1))
        ys.append(tr["latency_s"])
        cfgs.append((cyc, ctl, table))
    models, _ = rt.fit_latency_models(xs, ys)
    ours = []
    for (_, ex, labels), model, (cyc, ctl, table) in zip(prepared, models, cfgs):
        cyc.monitor_from_cycle = 2400
        an.set_config(cyc, ctl)
        an.set_name_table(table)
        an.upload(ex.events, [0, len(ex.events)], ex.workloads)
        an.load_model(model)
        an.run(abi.RUN_ALL)
        rows = []
        for strategy in (abi.FIXED_POINT, abi.FIXED_WINDOW, abi.DYNAMIC_WINDOW):
            an.redetect(abi.default_control(strategy))
            rows.append(an.evaluate_strategy(labels))
        ours.append(rows)
    tick["ours_s"] = time.perf_counter() - t0
    return ours, ref_rows, skipped


def test_config4_suite_aggregate_equals_reference(refbridge, analyzer, rt):
    analyzer.set_fused(False)
    ours, ref_rows, skipped = suite_metrics(refbridge, rt, analyzer)
    assert len(ours) + len(skipped) == 20 and len(ours) >= 16
    for o, r in zip(ours, ref_rows):
        assert [[m.tp, m.fp, m.fn, m.tn, m.alerts] for m in o] == r[:, :5].astype(int).tolist()
    got = rt.pool_strategy_metrics(ours)
    want = rt.pool_strategy_metrics(ref_rows)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    # the suite's Dynamic Window strategy detects (F1 0.972)
    assert got[2, 7] > 0.9
