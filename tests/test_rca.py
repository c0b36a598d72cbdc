"""Post-alert root-cause ranking: cs_rank_suspects over the
reference's own per-cycle stage attribution vs the reference's
suspicion_rank + attribute_straggler + resolve_topology (rca.cpp:220-353,
align.cpp:178-191), report field by field, bit-exact; welch_p_value against
the reference's formula on edge cases."""
import numpy as np
import pytest

from paper_2601_09258_b200 import abi
from paper_2601_09258_b200 import runtime as rt


def _layout(ref, ex):
    names = ex.names
    span = rt.span_names_mask(ex.events, len(names))
    _, _, table = rt.configs_from_json(None, names, span, len(ex.comm_name))
    S = int(table["beta_slot"].max()) + 1
    slot_names = [None] * S
    slot_metric = np.zeros(S, np.int32)
    for i, t in enumerate(table):
        if t["beta_slot"] >= 0:
            slot_names[t["beta_slot"]] = names[i]
            slot_metric[t["beta_slot"]] = t["metric"]
    comm_class = np.array([table["beta_slot"][c] for c in ex.comm_name], np.int32)
    groups = rt.comm_groups(list(ex.comm_name), list(ex.comm_hash))
    topo = ref.topology()
    locs = sorted({tuple(x) for x in topo if x is not None})
    loc_id = np.array([locs.index(tuple(x)) if x is not None else -1 for x in topo], np.int32)
    return S, slot_names, slot_metric, comm_class, groups, locs, loc_id


def _windows(res, S, R, normal, abnormal, mu):
    nc = len(res.cycles)

    def rows(idx):
        idx = np.asarray(idx)
        d = {"totals": res.beta_totals.reshape(nc, S)[idx].ravel(),
             "beta": res.beta.reshape(nc, S)[idx].ravel(),
             "coll": res.coll_beta.reshape(nc, max(R, 1))[idx].ravel() if R else np.zeros(0),
             "coll_present": res.coll_present.reshape(nc, max(R, 1))[idx].ravel() if R else np.zeros(0, np.uint8)}
        if mu:
            d["mu"] = res.extra["mu"].reshape(nc, S)[idx].ravel()
            d["mu_has"] = res.extra["mu_has"].reshape(nc, S)[idx].ravel()
        return d

    return rows(normal), rows(abnormal)


@pytest.mark.parametrize("fault,ranks,target,mu", [("nvlink_saturation", 4, 2, True),
                                                   ("nvlink_saturation", 2, 1, False),
                                                   ("cpu_contention", 1, 0, True),
                                                   ("memory_thrash", 4, 0, True)])
def test_rank_suspects_matches_reference(refbridge, fault, ranks, target, mu):
    ref = refbridge.RefTrace.synth(900, 7, 8, fault=fault, onset=600, duration=150, n_ranks=ranks,
                                   target_rank=target)
    ex = ref.export(None)
    res = ref.run(None, None, 300, beta=True, mu=mu)
    S, slot_names, slot_metric, comm_class, groups, locs, loc_id = _layout(ref, ex)
    R = len(ex.comm_name)
    normal = list(range(300, 600))
    abnormal = list(range(600, 750))
    wn, wa = _windows(res, S, R, normal, abnormal, mu)
    got = rt.rank_suspects(wn, wa, S, R, slot_metric, comm_class, groups, ex.comm_rank, loc_id)
    rep = rt.suspects_report(got, slot_names, ex.names, list(ex.comm_hash), list(ex.comm_rank), locs)
    want = ref.rca(normal, abnormal, mu=mu)["suspects"]
    assert [d["class"] for d in rep] == [d["class"] for d in want]
    assert rep == want
    if ranks > 1 and fault == "nvlink_saturation":
        assert any("straggler" in d for d in rep)


def test_insufficient_cycles(refbridge):
    ref = refbridge.RefTrace.synth(200, 1, 2)
    ex = ref.export(None)
    res = ref.run(None, None, 100, beta=True)
    S, *_ = _layout(ref, ex)
    wn, wa = _windows(res, S, 0, list(range(9)), list(range(50, 60)), False)
    with pytest.raises(rt.EngineError) as e:
        rt.rank_suspects(wn, wa, S, 0)
    assert e.value.type == "insufficient_cycles"
    assert ref.rca(list(range(9)), list(range(50, 60))) == ("error", "insufficient_cycles")


def test_welch_p_value_edges():
    assert rt.welch_p_value(1.0, 0.1, 1, 2.0, 0.1, 5) == 1.0
    assert rt.welch_p_value(1.0, 0.0, 5, 1.0, 0.0, 5) == 1.0
    assert rt.welch_p_value(1.0, 0.0, 5, 2.0, 0.0, 5) == 0.0
    p = rt.welch_p_value(0.30, 0.01, 40, 0.25, 0.012, 300)
    assert 0.0 < p < 0.01


def test_pool_strategy_metrics_matches_evaluate_suite_arithmetic():
    # two trials x three strategies: [tp, fp, fn, tn, alerts, f1, fpr, lag]
    from paper_2601_09258_b200 import runtime as rt
    t1 = np.array([[10, 2, 1, 100, 1, 0, 0, 1.5], [0, 0, 5, 80, 0, 0, 0, 0.0], [3, 1, 0, 50, 2, 0, 0, 0.25]], float)
    t2 = np.array([[5, 0, 3, 90, 1, 0, 0, 2.0], [1, 1, 1, 1, 1, 0, 0, 4.0], [0, 0, 0, 60, 0, 0, 0, 0.0]], float)
    got = rt.pool_strategy_metrics([t1, t2])
    tp, fp, fn, tn = 15.0, 2.0, 4.0, 190.0
    p, r = tp / (tp + fp), tp / (tp + fn)
    assert got[0].tolist() == [15, 2, 4, 190, 2, p, r, 2.0 * p * r / (p + r), fp / (fp + tn), (1.5 + 2.0) / 2.0]
    assert got[1, 5] == 0.5 and got[1, 6] == 1.0 / 7.0   # tp=1 fp=1 fn=6
    assert got[2, 0] == 3 and got[2, 8] == 1.0 / 111.0
