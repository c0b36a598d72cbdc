"""Times cs_set_option(98, v) reduce variants on a configs[1]-sized trace (GPU helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2601_09258_b200 import abi, runtime as rt

cyc = int(sys.argv[1]) if len(sys.argv) > 1 else 3_700_000
variants = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 2, 3, 4]
tr = rt.synth_trace(cyc, 7, 8, n_ranks=8, n_chunks=64, n_threads=os.cpu_count(), compact_names=False)
an = rt.Analyzer(0)
an.configure(tr.names, rt.span_names_mask(tr.events, len(tr.names)), n_comm_slots=8)
an.upload(tr.events, [0, len(tr.events)], tr.workloads)
ref = None
for v in variants:
    an.L.cs_set_option(an.h, 98, v)
    ts = []
    for i in range(6):
        an.run(abi.RUN_SEGMENT | abi.RUN_BETA)
        ts.append(an.timings())
    med = {k: round(float(np.median([d[k] for d in ts[2:]])), 3) for k in ts[-1]}
    b = an.beta(0)[1]
    same = ref is None or np.array_equal(b.view(np.uint64), ref.view(np.uint64))
    ref = b if ref is None else ref
    print("variant", v, med, "equal" if same else "MISMATCH", flush=True)
