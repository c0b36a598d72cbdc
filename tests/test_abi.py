"""CPU: the C-ABI library loads and exports what include/*.h declares; host
services (simkit restatement, deterministic fit, model JSON, RunConfig
interning) are bit-identical to the reference; no silent CPU fallback."""
import glob
import json
import os
import re

import numpy as np
import pytest

import traces
from oracle import csoracle
from paper_2601_09258_b200 import abi
from paper_2601_09258_b200 import runtime as rt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def declared_functions(header="cyclescope_b200.h"):
    names = []
    for h in glob.glob(os.path.join(ROOT, "include", header)):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names += re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\**\s*(cs_[a-z_0-9]+)\s*\(", text, re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    L = rt.lib()
    decl = declared_functions()
    assert len(decl) >= 35
    for name in decl:
        assert hasattr(L, name), name
    assert set(rt.EXPORTED_SYMBOLS) <= set(decl)
    assert L.cs_abi_version() == abi.CS_ABI_VERSION
    # benchmark support lives in its own library, never in the product one
    B = rt.bench_lib()
    bench = declared_functions("cs_bench.h")
    assert bench and all(hasattr(B, n) for n in bench)
    assert not any(hasattr(L, n) for n in bench)


def test_status_strings_match_reference_error_types():
    L = rt.lib()
    # errors.hpp:41-82 type() strings
    for code, t in abi.STATUS_TYPES.items():
        assert L.cs_status_type(code).decode() == t


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(rt.EngineError) as e:
        rt.Analyzer(0)
    assert e.value.type == "no_device"


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("name,params", [
    ("simkit_nvlink_r2", (700, 5, "nvlink_saturation", 2)),
    ("simkit_cpu_r1", (700, 9, "cpu_contention", 1)),
    ("simkit_thrash_r1", (700, 13, "memory_thrash", 1)),
])
def test_synth_restatement_matches_reference_simkit_golden(name, params):
    n, seed, fam, ranks = params
    d = load(name)
    s = rt.synth_trace(n, seed, seed + 1, fault=fam, onset=520, duration=60, n_ranks=ranks,
                       target_rank=1)
    assert s.names == json.loads(str(d["names"]))
    assert np.array_equal(s.events, d["events"])
    assert np.array_equal(s.event_ids, d["event_ids"])
    assert np.array_equal(s.workloads, d["workloads"])
    assert np.array_equal(s.labels, d["labels"])


def test_synth_matches_live_reference(refbridge):
    for fam, ranks in [("gpu_contention", 1), ("bus_contention", 3), (None, 8)]:
        t = refbridge.RefTrace.synth(1500, 3, 4, fault=fam, onset=1200, duration=100,
                                     n_ranks=ranks, target_rank=2)
        ex = t.export()
        s = rt.synth_trace(1500, 3, 4, fault=fam, onset=1200, duration=100, n_ranks=ranks,
                           target_rank=2)
        assert np.array_equal(ex.events, s.events)
        assert np.array_equal(ex.workloads, s.workloads)


def test_synth_chunked_is_sorted_and_consistent():
    s = rt.synth_trace(20000, 1, 2, n_ranks=8, n_chunks=7, n_threads=4)
    st = s.events["start_ts"]
    assert np.all(np.diff(st) >= 0)
    assert len(s.labels) == 20000
    anchors = (s.events["name_id"] == s.names.index("run_batch")) & (s.events["kind"] == 0)
    assert anchors.sum() == 20001  # one per cycle + the closing anchor
    assert len(s.workloads) == 20000


def golden_training_set(d, train=300):
    recs = d["records"]
    tr = recs[recs["cycle_index"] < train]
    x = np.stack([tr["batch"].astype(float),
                  (tr["batch"] * (tr["input_len"] + tr["output_len"])).astype(float)], 1)
    return x, tr["latency_s"]


@pytest.mark.parametrize("name", ["simkit_nvlink_r2", "simkit_cpu_r1", "simkit_thrash_r1"])
def test_fit_is_byte_identical_to_reference_golden(name):
    d = load(name)
    x, y = golden_training_set(d)
    m = rt.fit_latency_model(x, y)
    assert m.to_json() == str(d["model_json"])


def test_fit_matches_live_reference(refbridge):
    rng = np.random.default_rng(3)
    for n in [20, 57, 400]:
        b = rng.integers(1, 512, n).astype(float)
        w = b * rng.integers(2, 3000, n)
        y = 2e-8 * w + 1e-5 * b + 1e-3 + rng.lognormal(0, 0.05, n) * 1e-4
        x = np.stack([b, w], 1)
        assert rt.fit_latency_model(x, y).to_json() == refbridge.ref_fit(x, y, ["batch", "w_kv"])
    # ties in feature values exercise std::sort tie order in the split search
    x = np.stack([np.repeat([1.0, 2.0, 3.0, 4.0], 25), np.repeat([5.0, 5.0, 6.0, 7.0], 25)], 1)
    y = 1e-3 + rng.random(100) * 1e-4
    assert rt.fit_latency_model(x, y).to_json() == refbridge.ref_fit(x, y, ["batch", "w_kv"])


def test_fit_errors():
    with pytest.raises(rt.EngineError) as e:
        rt.fit_latency_model(np.ones((5, 2)), np.ones(5))
    assert e.value.type == "insufficient_data"
    with pytest.raises(rt.EngineError) as e:
        rt.fit_latency_model(np.ones((40, 2)), -np.ones(40))
    assert e.value.type == "insufficient_data"


def test_model_json_round_trip_and_version_refusal():
    d = load("simkit_cpu_r1")
    text = str(d["model_json"])
    m = rt.LatencyModel.from_json(text)
    assert m.to_json() == text
    bad = json.loads(text)
    bad["format_version"] = 999
    with pytest.raises(rt.EngineError) as e:
        rt.LatencyModel.from_json(json.dumps(bad))
    assert e.value.type == "model_format_error"
    with pytest.raises(rt.EngineError) as e:
        rt.LatencyModel.from_json("{not json")
    assert e.value.type == "model_format_error"


def test_run_config_interning_matches_oracle_derivation():
    names = ["a_forward_prefill_x", "get_next_batch_to_run", "oncpu", "process_batch_result",
             "process_batch_result_decode", "run_batch", "zz"]
    span = np.array([1, 1, 1, 1, 0, 1, 0], np.uint8)
    for cfg in [{}, {"cycle": {"anchor_hint": "oncpu", "phase_functions": ["oncpu", "zz", "oncpu"]},
                     "pipeline": {"latency_component": "zz", "include_prefill": True},
                     "detector": {"strategy": "fixed_window", "window": 4, "warmup": 7}},
                {"cycle": {"anchor_hint": "missing", "prefill_keywords": ["prefill"],
                           "decode_keywords": []}}]:
        cyc, ctl, table = rt.configs_from_json(cfg, names, span, 3)
        ocyc, octl, otable = csoracle.derive_config(cfg, names, span, 3)
        assert np.array_equal(table, otable)
        for f, _ in abi.CycleConfig._fields_:
            assert getattr(cyc, f) == getattr(ocyc, f), f
        for f, _ in abi.ControlConfig._fields_:
            assert getattr(ctl, f) == getattr(octl, f), f


def test_run_config_rejects_unknown_keys():
    with pytest.raises(rt.EngineError) as e:
        rt.configs_from_json({"cycle": {"bogus": 1}}, ["a"], [1])
    assert e.value.type == "config_error"
    with pytest.raises(rt.EngineError) as e:
        rt.configs_from_json({"detector": {"strategy": "nope"}}, ["a"], [1])
    assert e.value.type == "config_error"


def test_ucl_from_stats():
    c = abi.default_control()
    assert rt.ucl_from_stats(0.02, 0.01, c) == pytest.approx(0.05)  # test_detector.cpp:37
    c.theta_max = 0.4
    assert rt.ucl_from_stats(0.2, 0.2, c) == pytest.approx(0.4)
    c.theta_max = 0.18
    assert rt.ucl_from_stats(0.2, 0.2, c) == pytest.approx(0.18)
    assert rt.ucl_from_stats(0.0, 0.0, c) == pytest.approx(0.02)


def test_metric_map_interned_into_name_table():
    """RunConfig metric_map (rca.cpp:55-69 defaults) -> cs_name_info.metric =
    1 + name id of the counter series, 0 when unmapped or absent."""
    names = ["cpu_usage", "gemm_kernel", "oncpu", "run_batch", "x"]
    span = [0, 1, 1, 1, 1]
    _, _, table = rt.configs_from_json(None, names, span)
    assert table["metric"][names.index("oncpu")] == names.index("cpu_usage") + 1
    assert table["metric"][names.index("gemm_kernel")] == 0  # gpu_usage not in the trace
    assert table["metric"][names.index("x")] == 0
    _, _, table = rt.configs_from_json({"metric_map": {"x": "cpu_usage"}}, names, span)
    assert table["metric"][names.index("x")] == names.index("cpu_usage") + 1
    assert table["metric"][names.index("oncpu")] == 0  # a given map replaces the defaults
