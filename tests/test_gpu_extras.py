"""GPU: record extras and the Full feature set (A9; cycles.cpp:392-405,
baseline.cpp:43-78, main.cpp:59-78) and deep trees.

- the post_* args of every cycle (last event carrying a key wins) equal the
  reference's CycleRecord::extra, column for column;
- a model the reference trains with feature_set "full" (batch, w_kv, lens,
  stage + post_fwd_mode, post_max_in_len, post_run_latency) monitors bit-
  identically on the device (k_score<8>, double compares on the extras);
- the host fit with named extras columns reproduces that model's JSON byte
  for byte;
- a model feature the trace does not carry stops monitoring at the first
  record with FeatureMismatch, as features_by_name does;
- trees deeper than 8 (complete-tree layout of depth 10)."""
import numpy as np
import pytest

from helpers import assert_full_parity, run_product
from paper_2601_09258_b200 import abi
from paper_2601_09258_b200 import runtime as rt

pytestmark = pytest.mark.gpu


def _trace(refbridge, seed=111, ranks=2):
    return refbridge.RefTrace.synth(3600, seed, seed + 1, fault="pcie_bottleneck", onset=3000, duration=150,
                                    n_ranks=ranks, target_rank=1)


def _extras(ex):
    return (ex.extra_keys, ex.extra_refs, ex.extra_values)


@pytest.mark.parametrize("cfg", [{"feature_set": "full"},
                                 {"feature_set": "full", "gbdt": {"max_depth": 10, "n_trees": 60}},
                                 {"gbdt": {"max_depth": 9}}],
                         ids=["full", "full_depth10", "physical_depth9"])
def test_full_feature_set_and_deep_trees_match_reference(refbridge, analyzer, cfg):
    t = _trace(refbridge)
    ref = t.run(cfg, None, 2400)
    assert ref.status == 0, (ref.err_type, ref.err_msg)
    ex = t.export(cfg)
    got, an = run_product(ex.events, ex.names, ex.workloads, n_comm=len(ex.comm_hash), run_config=cfg,
                          model_json=ref.model_json, analyzer=analyzer, extras=_extras(ex))
    assert_full_parity(ref, got)
    if cfg.get("feature_set") == "full":
        vals, has = an.record_extras(0)
        rk = ref.extra["rec_extra_keys"]
        assert rk == ex.extra_keys
        assert np.array_equal(has[:len(ref.records)], ref.extra["rec_extra_has"])
        assert np.array_equal(vals[:len(ref.records)].view(np.uint64), ref.extra["rec_extra"].view(np.uint64))


def test_named_host_fit_reproduces_full_model_json(refbridge, analyzer):
    t = _trace(refbridge, seed=121, ranks=1)
    cfg = {"feature_set": "full"}
    ref = t.run(cfg, None, 2400)
    ex = t.export(cfg)
    got, an = run_product(ex.events, ex.names, ex.workloads, n_comm=len(ex.comm_hash),
                          run_config=cfg, mask=abi.RUN_SEGMENT, analyzer=analyzer, extras=_extras(ex))
    recs = an.records(0)
    vals, has = an.record_extras(0)
    tr = recs["cycle_index"] < 2400
    r = recs[tr]
    x = np.concatenate([np.stack([r["batch"].astype(float),
                                  (r["batch"] * (r["input_len"] + r["output_len"])).astype(float),
                                  r["input_len"].astype(float), r["output_len"].astype(float),
                                  (r["stage"] == 0).astype(float)], 1),
                        np.where(has[tr] != 0, vals[tr], 0.0)], 1)
    names = ["batch", "w_kv", "input_len", "output_len", "stage"] + ex.extra_keys
    model = rt.fit_latency_model(x, r["latency_s"], names)
    assert model.to_json() == ref.model_json


def test_missing_extra_feature_stops_at_first_record(refbridge, analyzer):
    t = _trace(refbridge, seed=131, ranks=1)
    cfg = {"feature_set": "full"}
    ref_full = t.run(cfg, None, 2400)
    # the same events without their post_* args: the reference stops at record 0
    ex = t.export(cfg)
    bare = refbridge.RefTrace.build(ex.events, ex.names, ex.workloads, ex.comm_hash, ex.comm_rank,
                                    event_ids=ex.event_ids, sort=False)
    ref = bare.run(cfg, ref_full.model_json, 2400)
    assert ref.err_type == "feature_mismatch" and ref.first_bad_record == 0
    got, _ = run_product(ex.events, ex.names, ex.workloads, n_comm=len(ex.comm_hash), run_config=cfg,
                         model_json=ref_full.model_json, analyzer=analyzer)
    assert got.status_type == "feature_mismatch"
    assert got.summary.first_bad_record == 0
    assert len(got.alerts) == 0
