"""Profiling helper: times the fused kernel with pieces disabled (outputs
invalid): debug bit0 no look-back, bit1 no event accumulation, bit2 no
cycle-output writes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2601_09258_b200 import abi, runtime as rt

cyc = int(sys.argv[1]) if len(sys.argv) > 1 else 3_700_000
tr = rt.synth_trace(cyc, 7, 8, n_ranks=8, n_chunks=64, n_threads=os.cpu_count(), compact_names=False)
an = rt.Analyzer(0)
an.configure(tr.names, rt.span_names_mask(tr.events, len(tr.names)), n_comm_slots=8)
an.upload(tr.events, [0, len(tr.events)], tr.workloads)
print("events", len(tr.events))
an.set_fused(True)
for dbg in [0, 1, 2, 4, 6, 7]:
    an.L.cs_set_option(an.h, 99, dbg)
    ts = []
    for i in range(6):
        an.run(abi.RUN_SEGMENT | abi.RUN_BETA)
        ts.append(an.timings().get("fused_segment", -1))
    print("debug", dbg, "fused_segment ms", [round(x, 3) for x in ts[2:]], flush=True)
an.L.cs_set_option(an.h, 99, 0)
