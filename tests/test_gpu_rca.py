"""Post-alert root-cause ranking on the device path (cs_suspicion_rank, SURVEY
§8f #4): stage attribution computed by cs_run (beta, counter mu, collective
beta), windows from the device detector's records as cmd_diagnose builds them
(main.cpp:262-298), ranked and attributed — the report equals the
reference's suspicion_rank + attribute_straggler on the same windows."""
import numpy as np
import pytest

from helpers import run_product
from paper_2601_09258_b200 import abi
from paper_2601_09258_b200 import runtime as rt
from test_rca import _layout

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fault,ranks,target", [("nvlink_saturation", 4, 3),
                                                ("cpu_contention", 2, 0),
                                                ("pcie_bottleneck", 8, 5)])
def test_suspicion_rank_device_matches_reference(refbridge, analyzer, fault, ranks, target):
    t = refbridge.RefTrace.synth(2800, 61 + ranks, 62, fault=fault, onset=2500, duration=200,
                                 n_ranks=ranks, target_rank=target)
    ref = t.run(None, None, 2400, beta=True, mu=True)
    assert ref.status == 0
    ex = t.export(None)
    got, an = run_product(ex.events, ex.names, ex.workloads, n_comm=len(ex.comm_hash),
                          model_json=ref.model_json, mask=abi.RUN_ALL | abi.RUN_MU, analyzer=analyzer)
    recs = an.records(0)
    assert np.array_equal(recs["flagged"], ref.records["flagged"][:len(recs)])
    normal, abnormal = rt.diagnose_windows(recs, 0)
    assert (normal, abnormal) == rt.diagnose_windows(ref.records, 0)
    S, slot_names, _, _, groups, locs, loc_id = _layout(t, ex)
    sus = an.suspicion_rank(normal, abnormal, ex.comm_name, groups, ex.comm_rank, loc_id)
    rep = rt.suspects_report(sus, slot_names, ex.names, list(ex.comm_hash), list(ex.comm_rank), locs)
    assert rep == t.rca(normal, abnormal, mu=True)["suspects"]
    if fault == "nvlink_saturation":
        top = next(d for d in rep if d["class"] == "reduce")
        assert top["straggler"]["rank"] == target
