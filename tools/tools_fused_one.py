"""Profiling driver: a few fused-pass runs on a ~27M-event trace (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_09258_b200 import abi, runtime as rt

cyc = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
tr = rt.synth_trace(cyc, 7, 8, n_ranks=8, n_chunks=32, n_threads=os.cpu_count(), compact_names=False)
an = rt.Analyzer(0)
an.configure(tr.names, rt.span_names_mask(tr.events, len(tr.names)), n_comm_slots=8)
an.upload(tr.events, [0, len(tr.events)], tr.workloads)
an.set_fused(os.environ.get("CS_FUSED", "1") == "1")
for i in range(3):
    an.run(abi.RUN_SEGMENT | abi.RUN_BETA)
print(an.timings())
