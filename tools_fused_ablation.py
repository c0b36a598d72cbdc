"""Profiling helper: times the fused kernel with pieces disabled (outputs invalid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
from paper_2601_09258_b200 import abi, runtime as rt
tr = rt.synth_trace(1_000_000, 7, 8, n_ranks=8, n_chunks=32, n_threads=os.cpu_count(), compact_names=False)
an = rt.Analyzer(0)
an.configure(tr.names, rt.span_names_mask(tr.events, len(tr.names)), n_comm_slots=8)
an.upload(tr.events, [0, len(tr.events)], tr.workloads)
print("events", len(tr.events))
for dbg in [0, 1, 2, 3]:
    an.L.cs_set_option(an.h, 99, dbg)
    ts = []
    for i in range(6):
        an.run(abi.RUN_SEGMENT | abi.RUN_BETA)
        ts.append(an.timings().get("fused_segment", -1))
    print("debug", dbg, "fused_segment ms", [round(x, 3) for x in ts[2:]])
an.L.cs_set_option(an.h, 99, 0)
an.set_fused(False)
for i in range(4):
    an.run(abi.RUN_SEGMENT | abi.RUN_BETA)
tm = an.timings(); print("legacy", {k: round(v, 3) for k, v in tm.items()})
an.L.cs_set_option(an.h, 98, 1)
for i in range(4):
    an.run(abi.RUN_SEGMENT | abi.RUN_BETA)
tm = an.timings(); print("legacy warp-per-cycle", {k: round(v, 3) for k, v in tm.items()})
