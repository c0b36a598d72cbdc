"""GPU: classify_stages' temporal heuristic (cycles.cpp:190-254) at scale and
for any window, computed in parallel (k_stage_jacobi: chunked sequential
windows + Jacobi refinement) and bit-exact against the reference.

Traces have forward_mode stripped and the keyword lists emptied, so every
cycle's stage comes from the trailing-median heuristic — the path a
non-SGLang producer takes."""
import numpy as np
import pytest

from helpers import assert_full_parity, run_product
from paper_2601_09258_b200 import abi

pytestmark = pytest.mark.gpu
NO_KW = {"prefill_keywords": ["zz_none"], "decode_keywords": ["zz_none"]}


def _stripped(refbridge, n_cycles, seed, n_ranks=1, fault="memory_thrash"):
    t = refbridge.RefTrace.synth(n_cycles, seed, seed + 1, fault=fault, onset=n_cycles - 400,
                                 duration=150, n_ranks=n_ranks)
    ex = t.export()
    ev = ex.events.copy()
    ev["flags"] &= np.uint16(0xFFFC)  # CS_EV_FM_MASK: no forward_mode arg anywhere
    rt_ = refbridge.RefTrace.build(ev, ex.names, ex.workloads, ex.comm_hash, ex.comm_rank,
                                   event_ids=ex.event_ids, sort=False)
    return rt_, ev, ex


@pytest.mark.parametrize("window,factor", [(32, 3.0), (100, 2.5), (8, 3.0), (1, 3.0)])
def test_heuristic_windows_match_reference(refbridge, analyzer, window, factor):
    t, ev, ex = _stripped(refbridge, 6000, 61)
    cfg = {"cycle": dict(NO_KW, stage_window=window, prefill_duration_factor=factor)}
    ref = t.run(cfg, None, 2400)
    assert ref.status == 0, ref.err_msg
    st = ref.cycles["stage"]
    if window >= 8:  # stage_min_history = 8 (cycles.hpp:34): below it every cycle stays Unknown
        assert (st == 0).sum() > 10 and (st == 1).sum() > 1000  # the heuristic decided both ways
    else:
        assert (st == 2).all()
    got, _ = run_product(ev, ex.names, ex.workloads, n_comm=len(ex.comm_hash), run_config=cfg,
                         model_json=ref.model_json, analyzer=analyzer)
    assert_full_parity(ref, got)


@pytest.mark.parametrize("fused", [False, True], ids=["two-pass", "single-read"])
def test_heuristic_100k_cycles_match_reference(refbridge, analyzer, fused):
    t, ev, ex = _stripped(refbridge, 100_000, 71, n_ranks=2, fault="gpu_contention")
    cfg = {"cycle": NO_KW}
    ref = t.run(cfg, None, 2400)
    assert ref.status == 0, ref.err_msg
    assert (ref.cycles["stage"] == 0).sum() > 500
    got, _ = run_product(ev, ex.names, ex.workloads, n_comm=len(ex.comm_hash), run_config=cfg,
                         model_json=ref.model_json, analyzer=analyzer, fused=fused)
    assert_full_parity(ref, got)
