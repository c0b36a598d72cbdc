"""GPU parity: the CUDA path through the C ABI vs the reference compiled
unmodified (oracle/_ref), on identical 32-byte records.

Bar (BASELINE.json north_star): segmentation, stage attribution and alert
decisions bit-exact; float latencies / residuals within 1e-6 relative — we
assert bit equality of every f64 (the kernels reproduce the reference's
operation order without FMA), which implies the 1e-6 bound.
"""
import numpy as np
import pytest

from helpers import assert_full_parity, assert_cycles_equal, run_product
from paper_2601_09258_b200 import abi

pytestmark = pytest.mark.gpu

FAMILIES = ["cpu_contention", "cpu_freq_drop", "gpu_contention", "gpu_clock_lock",
            "memory_thrash", "nvlink_saturation", "pcie_bottleneck", "bus_contention"]


def _ref_and_product(refbridge, analyzer, trace, run_config=None, train_cycles=2400,
                     mask=abi.RUN_ALL, fused=False):
    ref = trace.run(run_config, None, train_cycles)
    ex = trace.export(run_config)
    got, _ = run_product(ex.events, ex.names, ex.workloads, n_comm=len(ex.comm_hash),
                         run_config=run_config, model_json=ref.model_json, mask=mask,
                         analyzer=analyzer, fused=fused)
    return ref, got, ex


@pytest.mark.parametrize("family", FAMILIES)
def test_simkit_family_full_parity(refbridge, analyzer, family):
    ranks = 4 if family == "nvlink_saturation" else 1
    t = refbridge.RefTrace.synth(3800, 11 + FAMILIES.index(family), 99, fault=family,
                                 onset=3000, duration=150, n_ranks=ranks, target_rank=2)
    ref, got, ex = _ref_and_product(refbridge, analyzer, t)
    assert ref.status == 0, ref.err_msg
    assert got.summary.status == 0
    # the reference may legitimately pick process_batch_result (close scores)
    assert ex.names[got.summary.anchor_name_id] == ref.anchor
    assert_full_parity(ref, got)


@pytest.mark.parametrize("strategy", ["fixed_point", "fixed_window", "dynamic_window"])
def test_strategies_parity(refbridge, analyzer, strategy):
    t = refbridge.RefTrace.synth(4000, 5, 6, fault="gpu_contention", onset=3100, duration=150)
    cfg = {"detector": {"strategy": strategy, "window": 7, "warmup": 50}}
    ref, got, _ = _ref_and_product(refbridge, analyzer, t, run_config=cfg)
    assert_full_parity(ref, got)


def test_eight_rank_collective_beta(refbridge, analyzer):
    t = refbridge.RefTrace.synth(3000, 21, 22, fault="nvlink_saturation", onset=2500,
                                 duration=150, n_ranks=8, target_rank=3)
    ref, got, ex = _ref_and_product(refbridge, analyzer, t)
    assert len(ex.comm_hash) == 8
    assert_full_parity(ref, got)
    nc = len(ex.comm_hash)
    cb = got.coll_beta.reshape(-1, nc)
    # straggler rank 3 dominates inside the fault window
    assert cb[2600:2650, 3].mean() > cb[2600:2650, 0].mean()


@pytest.mark.parametrize("fused", [True, False], ids=["fused", "multikernel"])
def test_c1_scale_parity(refbridge, analyzer, fused):
    """BASELINE config 1: 50k cycles, ~1M events, fault at 40000 for 150."""
    t = refbridge.RefTrace.synth(50000, 1, 2, fault="cpu_contention", onset=40000, duration=150)
    assert t.n_events() == 1000001
    ref, got, _ = _ref_and_product(refbridge, analyzer, t, fused=fused)
    assert_full_parity(ref, got)


def test_run_config_variants(refbridge, analyzer):
    t = refbridge.RefTrace.synth(3000, 31, 32, fault="pcie_bottleneck", onset=2600, duration=150)
    for cfg in [{"pipeline": {"latency_component": ""}},
                {"pipeline": {"include_prefill": True}},
                {"pipeline": {"latency_component": "process_batch_result"}},
                {"cycle": {"anchor_hint": "run_batch"}},
                {"cycle": {"phase_functions": ["run_batch", "oncpu", "run_batch"]}},
                {"cycle": {"min_anchor_calls": 2000000}}]:
        ref, got, _ = _ref_and_product(refbridge, analyzer, t, run_config=cfg)
        assert_full_parity(ref, got)


def test_multi_instance_batch(refbridge, analyzer, rt):
    """Several instances in one upload, each with its own model."""
    traces = [refbridge.RefTrace.synth(2600 + 100 * i, 40 + i, 50 + i, fault=FAMILIES[i],
                                       onset=2450, duration=100, n_ranks=1 + (i % 2) * 3)
              for i in range(4)]
    refs = [t.run(None, None, 2400) for t in traces]
    exps = [t.export() for t in traces]
    # common name table: all simkit names; remap each instance
    names = sorted(set(n for e in exps for n in e.names))
    evs, wls, offs = [], [], [0]
    for e in exps:
        remap = np.array([names.index(n) for n in e.names], dtype=np.uint32)
        ev = e.events.copy()
        ev["name_id"] = remap[ev["name_id"]]
        base = sum(len(w) for w in wls)
        has = (ev["flags"] & abi.EV_HAS_BATCH) != 0
        ev["payload"][has] = (ev["payload"][has] & np.uint64(0xFFFFFFFF00000000)) | \
            ((ev["payload"][has] & np.uint64(0xFFFFFFFF)) + np.uint64(base))
        evs.append(ev)
        wls.append(e.workloads)
        offs.append(offs[-1] + len(ev))
    events = np.concatenate(evs)
    workloads = np.concatenate(wls)
    span = rt.span_names_mask(events, len(names))
    analyzer.configure(names, span, n_comm_slots=4)
    analyzer.upload(events, offs, workloads)
    for i, r in enumerate(refs):
        analyzer.load_model(rt.LatencyModel.from_json(r.model_json), inst=i)
    analyzer.run(abi.RUN_ALL)
    for i, r in enumerate(refs):
        got = analyzer.result(i, beta=False)
        assert_cycles_equal(r.cycles, got.cycles)
        from helpers import assert_records_equal, assert_alerts_equal
        assert_records_equal(r.records, got.records)
        assert_alerts_equal(r.alerts, got.alerts)


def test_product_fit_drives_same_alerts(refbridge, analyzer, rt):
    """Host fit (cs_fit_latency_model) == reference fit -> identical alerts."""
    t = refbridge.RefTrace.synth(3800, 61, 62, fault="bus_contention", onset=3000, duration=150)
    ref = t.run(None, None, 2400)
    ex = t.export()
    got, an = run_product(ex.events, ex.names, ex.workloads, n_comm=1, mask=abi.RUN_SEGMENT,
                          analyzer=analyzer)
    recs = got.records[got.records["cycle_index"] < 2400]
    x = np.stack([recs["batch"].astype(float),
                  (recs["batch"] * (recs["input_len"] + recs["output_len"])).astype(float)], 1)
    model = rt.fit_latency_model(x, recs["latency_s"])
    assert model.to_json() == ref.model_json
    an.load_model(model)
    an.run(abi.RUN_ALL)
    from helpers import assert_alerts_equal
    assert_alerts_equal(ref.alerts, an.alerts(0))


@pytest.mark.parametrize("family,ranks,fused", [("cpu_contention", 1, False),
                                                ("memory_thrash", 1, True),
                                                ("nvlink_saturation", 4, False),
                                                ("gpu_clock_lock", 8, False)])
def test_counter_weighted_mu_parity(refbridge, analyzer, family, ranks, fused):
    """cycle_stats' mu with the trace's CounterTable and the
    default MetricMap (rca.cpp:17-53, 97-126) — bit-equal to the reference."""
    t = refbridge.RefTrace.synth(900, 3 + ranks, 4, fault=family, onset=600, duration=150,
                                 n_ranks=ranks, target_rank=ranks - 1)
    ref = t.run(None, None, 400, beta=True, mu=True)
    ex = t.export(None)
    got, an = run_product(ex.events, ex.names, ex.workloads, n_comm=len(ex.comm_hash),
                          mask=abi.RUN_SEGMENT | abi.RUN_MU, analyzer=analyzer, fused=fused)
    mu, has = an.mu(0)
    assert ref.status == 0
    assert has.sum() > len(got.cycles)  # several mapped classes per cycle
    assert np.array_equal(has, ref.extra["mu_has"])
    assert np.array_equal(mu.view(np.uint64), ref.extra["mu"].view(np.uint64))


def test_counter_weighted_mu_custom_metric_map(refbridge, analyzer):
    cfg = {"metric_map": {"attn_kernel": "frequency", "oncpu": "page_activity",
                          "reduce": "bus_util", "run_batch": "no_such_counter"}}
    t = refbridge.RefTrace.synth(700, 31, 32, fault="bus_contention", onset=500, duration=100,
                                 n_ranks=2, target_rank=1)
    ref = t.run(cfg, None, 300, beta=True, mu=True)
    ex = t.export(cfg)
    got, an = run_product(ex.events, ex.names, ex.workloads, n_comm=len(ex.comm_hash),
                          run_config=cfg, mask=abi.RUN_SEGMENT | abi.RUN_MU, analyzer=analyzer)
    mu, has = an.mu(0)
    assert np.array_equal(has, ref.extra["mu_has"])
    assert np.array_equal(mu.view(np.uint64), ref.extra["mu"].view(np.uint64))
