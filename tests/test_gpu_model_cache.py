"""GPU: the per-instance model table is cached across cs_run calls; every
change it depends on must rebuild it — a model rebound to the instance, a
control-config change without a model load, cs_redetect, a different instance
count — with results equal to the C oracle after each change."""
import numpy as np
import pytest

from helpers import assert_alerts_equal, assert_records_equal
from oracle import csoracle
from paper_2601_09258_b200 import abi, runtime as rt

pytestmark = pytest.mark.gpu


def _fit(recs, upto):
    r = recs[recs["cycle_index"] < upto]
    x = np.stack([r["batch"].astype(float), (r["batch"] * (r["input_len"] + r["output_len"])).astype(float)], 1)
    return rt.fit_latency_model(x, r["latency_s"]).to_json()


def test_model_table_follows_every_change():
    tr = rt.synth_trace(5000, 71, 72, fault="cpu_freq_drop", onset=3800, duration=300, n_ranks=2,
                        compact_names=False)
    span = rt.span_names_mask(tr.events, len(tr.names))
    rc_a = {"cycle": {"anchor_hint": "run_batch"}}
    rc_b = {"cycle": {"anchor_hint": "run_batch"}, "detector": {"sigma_k": 1.0, "window": 5}}
    base = csoracle.analyze(tr.events, tr.names, tr.workloads, tr.n_comm, rc_a, None, span=span)
    m1, m2 = _fit(base["records"], 2400), _fit(base["records"], 900)
    assert m1 != m2

    def oracle(rc, m):
        return csoracle.analyze(tr.events, tr.names, tr.workloads, tr.n_comm, rc, m, span=span)

    def check(an, want):
        got = an.result(0)
        assert_records_equal(want["records"], got.records)
        assert_alerts_equal(want["alerts"], got.alerts)

    an = rt.Analyzer(0)
    an.configure(tr.names, span, n_comm_slots=tr.n_comm, run_config=rc_a)
    an.upload(tr.events, [0, len(tr.events)], tr.workloads)
    an.load_model(rt.LatencyModel.from_json(m1))
    an.run(abi.RUN_ALL)
    check(an, oracle(rc_a, m1))
    an.run(abi.RUN_ALL)  # cached table
    check(an, oracle(rc_a, m1))
    an.load_model(rt.LatencyModel.from_json(m2), inst=0)  # rebinding
    an.run(abi.RUN_ALL)
    check(an, oracle(rc_a, m2))
    cyc, ctl, table = rt.configs_from_json(rc_b, tr.names, span, tr.n_comm)  # control config only
    an.set_config(cyc, ctl)
    an.run(abi.RUN_ALL)
    check(an, oracle(rc_b, m2))
    an.redetect(abi.default_control(abi.FIXED_WINDOW))  # redetect, then a plain run again
    cyc, ctl, table = rt.configs_from_json(rc_a, tr.names, span, tr.n_comm)
    an.set_config(cyc, ctl)
    an.run(abi.RUN_ALL)
    check(an, oracle(rc_a, m2))
    # two instances, then one again
    half = len(tr.events) // 2
    k = int(np.searchsorted(tr.events["start_ts"], tr.events["start_ts"][half]))
    an.upload(tr.events, [0, k, len(tr.events)], tr.workloads)
    an.run(abi.RUN_ALL)
    an.upload(tr.events, [0, len(tr.events)], tr.workloads)
    an.run(abi.RUN_ALL)
    check(an, oracle(rc_a, m2))
    an.close()
