"""GPU: the control chart for every strategy and window sizes on both sides
of k_detect_flags' shared-memory tile (windows <= 64 records read a staged
tile, larger ones read global memory) — records and alerts bit-identical to
the C oracle (detector.cpp:85-130)."""
import numpy as np
import pytest

from helpers import assert_alerts_equal, assert_records_equal, run_product
from oracle import csoracle
from paper_2601_09258_b200 import runtime as rt

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def trace():
    tr = rt.synth_trace(6000, 31, 32, fault="gpu_contention", onset=4000, duration=300, n_ranks=2,
                        compact_names=False)
    rc = {"cycle": {"anchor_hint": "run_batch"}}
    base = csoracle.analyze(tr.events, tr.names, tr.workloads, tr.n_comm, rc, None)
    r = base["records"]
    r = r[r["cycle_index"] < 2400]
    x = np.stack([r["batch"].astype(float), (r["batch"] * (r["input_len"] + r["output_len"])).astype(float)], 1)
    return tr, rt.fit_latency_model(x, r["latency_s"]).to_json()


@pytest.mark.parametrize("strategy", ["fixed_point", "fixed_window", "dynamic_window"])
@pytest.mark.parametrize("window", [1, 10, 63, 64, 65, 200])
def test_detector_windows_match_oracle(trace, strategy, window):
    tr, model = trace
    rc = {"cycle": {"anchor_hint": "run_batch"},
          "detector": {"strategy": strategy, "window": window, "warmup": 100}}
    want = csoracle.analyze(tr.events, tr.names, tr.workloads, tr.n_comm, rc, model)
    got, an = run_product(tr.events, tr.names, tr.workloads, tr.n_comm, run_config=rc, model_json=model)
    assert_records_equal(want["records"], got.records)
    assert_alerts_equal(want["alerts"], got.alerts)
    if strategy != "fixed_point":
        assert (got.records["flagged"] == 1).any()
    an.close()
