"""GPU: no bound on the number of span classes, collective slots or phase
functions (the reference keys them in std::maps: cycles.cpp:157-166,
rca.cpp:85-115).  A trace with 500+ distinct span names and 128 collective
(name, commHash, rank) slots, and a configuration with 20 phase functions,
run bit-exact against the reference compiled unmodified."""
import numpy as np
import pytest

from helpers import assert_full_parity, run_product
from paper_2601_09258_b200 import abi

pytestmark = pytest.mark.gpu


def _renamed(refbridge, n_cycles, n_ranks, n_kernel_names, seed):
    """A simkit trace whose GpuKernel spans are spread over many names."""
    t = refbridge.RefTrace.synth(n_cycles, seed, seed + 1, fault="nvlink_saturation",
                                 onset=n_cycles - 120, duration=60, n_ranks=n_ranks, target_rank=5)
    ex = t.export()
    ev = ex.events.copy()
    names = list(ex.names)
    extra = [f"kern_{k:04d}" for k in range(n_kernel_names)]
    allnames = sorted(set(names) | set(extra))  # name id == lexicographic rank
    remap = np.array([allnames.index(n) for n in names], np.uint32)
    ev["name_id"] = remap[ev["name_id"]]
    gk = (ev["kind"] == 0) & (ev["category"] == abi.CAT_GPU_KERNEL) if hasattr(abi, "CAT_GPU_KERNEL") \
        else (ev["kind"] == 0) & (ev["category"] == 2)
    idx = np.nonzero(gk)[0]
    ev["name_id"][idx] = np.array([allnames.index(extra[i % n_kernel_names]) for i in range(len(idx))],
                                  np.uint32)
    rt_ = refbridge.RefTrace.build(ev, allnames, ex.workloads, ex.comm_hash, ex.comm_rank,
                                   event_ids=ex.event_ids, sort=False)
    return rt_, ev, allnames, ex


def test_500_span_classes_and_128_collective_slots(refbridge, analyzer):
    t, ev, names, ex = _renamed(refbridge, 2800, 128, 520, 17)
    assert len(ex.comm_hash) == 128
    ref = t.run(None, None, 2400)
    assert ref.status == 0, ref.err_msg
    got, _ = run_product(ev, names, ex.workloads, n_comm=len(ex.comm_hash), model_json=ref.model_json,
                         analyzer=analyzer)
    assert analyzer.cycle.n_beta_slots > 500
    assert_full_parity(ref, got)


def test_many_phase_functions(refbridge, analyzer):
    t, ev, names, ex = _renamed(refbridge, 2600, 2, 40, 23)
    phases = ["run_batch", "process_batch_result", "get_next_batch_to_run"] + \
             [f"kern_{k:04d}" for k in range(0, 40, 2)]
    cfg = {"cycle": {"phase_functions": phases}, "pipeline": {"latency_component": "kern_0004"}}
    ref = t.run(cfg, None, 2400)
    assert ref.status == 0, ref.err_msg
    got, _ = run_product(ev, names, ex.workloads, n_comm=len(ex.comm_hash), run_config=cfg,
                         model_json=ref.model_json, analyzer=analyzer)
    assert analyzer.cycle.n_phases == 23
    assert_full_parity(ref, got)
