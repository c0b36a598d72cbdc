"""Counter-weighted mu on the device vs the reference at configs[0] scale
(GPU helper): device time of the mu stage on C1 (1M events) and C2 (100M),
reference cycle_stats with a CounterTable on C1 (quadratic in the reference)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2601_09258_b200 import abi, runtime as rt

for cyc, ranks in ((50_000, 1), (3_700_000, 8)):
    tr = rt.synth_trace(cyc, 1, 2, n_ranks=ranks, n_chunks=64 if cyc > 100_000 else 1,
                        n_threads=os.cpu_count(), compact_names=False)
    an = rt.Analyzer(0)
    an.configure(tr.names, rt.span_names_mask(tr.events, len(tr.names)), n_comm_slots=tr.n_comm)
    an.upload(tr.events, [0, len(tr.events)], tr.workloads)
    ts = []
    for i in range(5):
        an.run(abi.RUN_SEGMENT | abi.RUN_MU)
        ts.append(an.timings())
    med = {k: round(float(np.median([d[k] for d in ts[1:]])), 4) for k in ts[-1]}
    print(f"events {len(tr.events)} mu stage ms {med.get('mu')} total ms {med['total']}", flush=True)
    an.close()
try:
    from oracle import refbridge as rb
    if rb.available():
        t = rb.RefTrace.synth(50_000, 1, 2)
        t0 = time.time()
        t.run(None, None, 2400, beta=True, mu=False)
        tb = time.time() - t0
        t0 = time.time()
        t.run(None, None, 2400, beta=True, mu=True)
        print(f"reference C1: run with beta {tb:.2f} s, with beta+mu {time.time() - t0:.2f} s (1 core)")
except Exception as e:  # noqa: BLE001
    print("reference timing skipped:", e)
