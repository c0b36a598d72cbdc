"""The benchmark input producer (benchlib/cs_synth.cpp, a restatement of the
reference's simkit generator, simkit.cpp:34-86, 195-246, 276-506) against the
reference generator itself: the same seeds give the same trace, event for
event and byte for byte (records, names, workload table).  CPU only."""
import numpy as np
import pytest

from paper_2601_09258_b200 import runtime as rt

CASES = [
    (1500, 3, 4, "cpu_contention", 1200, 150, 1),
    (2000, 5, 6, "nvlink_saturation", 1500, 150, 8),
    (800, 7, 8, None, 0, 0, 4),
    (1200, 9, 10, "gpu_clock_lock", 900, 100, 2),
]


@pytest.mark.parametrize("cycles,wseed,sseed,fault,onset,duration,ranks", CASES)
def test_synth_matches_reference_generator(refbridge, cycles, wseed, sseed, fault, onset, duration, ranks):
    ref = refbridge.RefTrace.synth(cycles, wseed, sseed, fault=fault, onset=onset, duration=duration,
                                   n_ranks=ranks).export()
    ours = rt.synth_trace(cycles, wseed, sseed, fault=fault, onset=onset, duration=duration, n_ranks=ranks,
                          target_rank=0, compact_names=False)
    assert list(ref.names) == list(ours.names)
    assert len(ref.events) == len(ours.events)
    assert ref.events.tobytes() == ours.events.tobytes()
    assert np.array_equal(np.asarray(ref.workloads).view(np.uint8), np.asarray(ours.workloads).view(np.uint8))
