"""GPU: the CUDA path reproduces every committed golden vector (generated
from the reference itself by tests/golden/make_golden.py) bit for bit, and
the hand-built fixtures mirroring the reference's unit tests."""
import glob
import json
import os

import numpy as np
import pytest

import traces
from helpers import run_product
from oracle import csoracle
from paper_2601_09258_b200 import abi

pytestmark = pytest.mark.gpu

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def load_golden(path):
    z = np.load(path, allow_pickle=False)
    d = {k: z[k] for k in z.files}
    d["names"] = json.loads(str(d["names"]))
    d["comm_hash"] = json.loads(str(d["comm_hash"]))
    d["run_config"] = json.loads(str(d["run_config"]))
    d["model_json"] = str(d["model_json"])
    return d


@pytest.mark.parametrize("fused", [True, False], ids=["fused", "multikernel"])
@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_gpu_matches_golden(path, fused, analyzer):
    d = load_golden(path)
    got, _ = run_product(d["events"], d["names"], d["workloads"], n_comm=len(d["comm_hash"]),
                         run_config=d["run_config"], model_json=d["model_json"] or None,
                         analyzer=analyzer, fused=fused)
    status = int(d["status"])
    if status:
        assert got.status_type == str(d["err_type"])
    assert np.array_equal(got.cycles, d["cycles"])
    assert np.array_equal(got.components, d["components"])
    assert np.array_equal(got.beta_totals, d["beta_totals"])
    assert np.array_equal(got.beta.view(np.uint64), d["beta"].view(np.uint64))
    assert np.array_equal(got.coll_beta.view(np.uint64), d["coll_beta"].view(np.uint64))
    assert np.array_equal(got.coll_present, d["coll_present"])
    n = len(d["records"])
    if status == 0:
        assert np.array_equal(got.records, d["records"])
        assert np.array_equal(got.alerts, d["alerts"])
        assert got.summary.ucl == float(d["ucl"])
    if len(d["candidates"]):
        c = got.candidates
        assert np.array_equal(c["name_id"], d["candidates"]["name_id"])
        assert np.array_equal(c["call_count"], d["candidates"]["call_count"])
        # exact-moment scores: within 1e-9 relative of the ordered sums
        np.testing.assert_allclose(c["score"], d["candidates"]["score"], rtol=1e-9)
    assert n == len(got.records) or status != 0


@pytest.mark.parametrize("fused", [True, False], ids=["fused", "multikernel"])
def test_gpu_matches_c_oracle_on_random_edge_traces(analyzer, fused):
    """Seeded random traces with equal timestamps, overlapping anchors,
    missing args, duplicates — GPU vs the C restatement."""
    rng = np.random.default_rng(11)
    for trial in range(16):
        spec, t = [], 0
        n = int(rng.integers(5, 400))
        for i in range(n):
            fm = [None, "decode", "prefill", "other"][int(rng.integers(0, 4))] if trial % 3 else None
            batch = None if rng.random() < 0.1 else int(rng.integers(-1, 64))
            spec.append(traces.ev("run_batch", t, int(rng.integers(1, 3000)), fm=fm, batch=batch,
                                  input_len=int(rng.integers(0, 500)),
                                  output_len=None if rng.random() < 0.05 else int(rng.integers(0, 50))))
            for k in range(int(rng.integers(0, 40))):
                if rng.random() < 0.2:  # counter samples feeding mu (equal timestamps included)
                    spec.append(traces.ev(["cpu_usage", "gpu_usage", "tx_bytes"][int(rng.integers(0, 3))],
                                          t + int(rng.integers(0, 2500)) // 100 * 100, kind="counter",
                                          cat="counter_telemetry", value=float(rng.normal(50, 20))))
                    continue
                nm = ["oncpu", "gemm_kernel", "reduce", "process_batch_result", "forward_prefill",
                      "get_next_batch_to_run"][int(rng.integers(0, 6))]
                cat = {"oncpu": "os_sched", "gemm_kernel": "gpu_kernel",
                       "reduce": "collective_comm"}.get(nm, "python_call")
                spec.append(traces.ev(nm, t + int(rng.integers(0, 2500)), int(rng.integers(-5, 2000)),
                                      cat=cat, comm="c0" if nm == "reduce" else None,
                                      rank=int(rng.integers(0, 4)) if nm == "reduce" else None))
            t += int(rng.integers(0, 3000)) if rng.random() > 0.02 else 0
        b = traces.build(spec)
        cfg = {"detector": {"warmup": int(rng.integers(0, 20)), "window": int(rng.integers(1, 12))}}
        model = json.dumps(traces.TINY_MODEL)
        o = csoracle.analyze(b.events, b.names, b.workloads, b.n_comm, cfg, model)
        got, an = run_product(b.events, b.names, b.workloads, n_comm=b.n_comm, run_config=cfg,
                              model_json=model, analyzer=analyzer, fused=fused,
                              mask=abi.RUN_ALL | abi.RUN_MU)
        mu, has = an.mu(0)
        assert np.array_equal(has, o["mu_has"]), trial
        assert np.array_equal(mu.view(np.uint64), o["mu"].view(np.uint64)), trial
        assert np.array_equal(got.cycles, o["cycles"]), trial
        assert np.array_equal(got.components, o["components"]), trial
        assert np.array_equal(got.beta_totals, o["beta_totals"]), trial
        assert np.array_equal(got.coll_beta.view(np.uint64), o["coll_beta"].view(np.uint64)), trial
        if o["status"] == 0:
            assert np.array_equal(got.records, o["records"]), trial
            assert np.array_equal(got.alerts, o["alerts"]), trial
        else:
            k = int(o["first_bad_record"])
            assert got.summary.first_bad_record == k
            assert np.array_equal(got.records[:k], o["records"][:k]), trial


def test_mu_known_answer(analyzer):
    """test_rca.cpp:121-155: oncpu 1 ms where cpu_usage reads 10, 3 ms where
    it reads 30 -> mu = (1*10 + 3*30) / 4 = 25 (exact here)."""
    import traces
    from traces import ev
    spec = [ev("run_batch", 0, 9_800_000), ev("run_batch", 10_000_000, 9_800_000),
            ev("oncpu", 1_000_000, 1_000_000, cat="os_sched"),
            ev("oncpu", 5_000_000, 3_000_000, cat="os_sched"),
            ev("cpu_usage", 0, kind="counter", cat="counter_telemetry", value=10.0),
            ev("cpu_usage", 3_000_000, kind="counter", cat="counter_telemetry", value=10.0),
            ev("cpu_usage", 4_000_000, kind="counter", cat="counter_telemetry", value=30.0)]
    b = traces.build(spec)
    got, an = run_product(b.events, b.names, b.workloads, mask=abi.RUN_SEGMENT | abi.RUN_MU,
                          run_config={"cycle": {"anchor_hint": "run_batch"}}, analyzer=analyzer)
    mu, has = an.mu(0)
    C = an.cycle.n_beta_slots
    slots = {n: i for i, n in enumerate(n for n, s in zip(b.names, rt_span(b)) if s)}
    assert len(got.cycles) == 1
    assert has[slots["oncpu"]] == 1 and mu[slots["oncpu"]] == 25.0
    assert has[slots["run_batch"]] == 0  # gpu_usage has no series: beta-only entry
    assert len(mu) == C


def rt_span(b):
    from paper_2601_09258_b200 import runtime as rt
    return rt.span_names_mask(b.events, len(b.names))


@pytest.mark.parametrize("scale", [1 << 28, 1 << 41], ids=["u64-rows", "two-pass-fallback"])
def test_gpu_long_cycles_match_c_oracle(analyzer, scale):
    """Long cycles and spans: at 2^28 ns cycles the single-read pass needs its
    u64 rows (duration x events >= 2^32); at 2^41 ns it hands the run to the
    two-pass path (duration >= 2^32, a packed collective row could
    overflow).  Both equal the C oracle."""
    rng = np.random.default_rng(5)
    spec, t = [], 0
    for i in range(60):
        spec.append(traces.ev("run_batch", t, int(rng.integers(1, scale)), batch=int(rng.integers(1, 64)),
                              input_len=int(rng.integers(0, 500)), output_len=int(rng.integers(0, 50)),
                              fm="decode"))
        for k in range(int(rng.integers(1, 120))):
            nm = ["oncpu", "gemm_kernel", "reduce", "process_batch_result"][int(rng.integers(0, 4))]
            cat = {"oncpu": "os_sched", "gemm_kernel": "gpu_kernel", "reduce": "collective_comm"}.get(nm, "python_call")
            spec.append(traces.ev(nm, t + int(rng.integers(0, scale)), int(rng.integers(-5, 2 * scale)),
                                  cat=cat, comm="c0" if nm == "reduce" else None,
                                  rank=int(rng.integers(0, 4)) if nm == "reduce" else None))
        t += int(rng.integers(scale // 2, 2 * scale))
    b = traces.build(spec)
    cfg = {"detector": {"warmup": 5, "window": 4}}
    model = json.dumps(traces.TINY_MODEL)
    o = csoracle.analyze(b.events, b.names, b.workloads, b.n_comm, cfg, model)
    got, an = run_product(b.events, b.names, b.workloads, n_comm=b.n_comm, run_config=cfg,
                          model_json=model, analyzer=analyzer, fused=True)
    assert np.array_equal(got.cycles, o["cycles"])
    assert np.array_equal(got.components, o["components"])
    assert np.array_equal(got.beta_totals, o["beta_totals"])
    assert np.array_equal(got.coll_beta.view(np.uint64), o["coll_beta"].view(np.uint64))
    if o["status"] == 0:
        assert np.array_equal(got.records, o["records"])
        assert np.array_equal(got.alerts, o["alerts"])
