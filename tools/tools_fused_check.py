"""Fused single pass vs the multi-kernel path at configs[1] scale: identical
outputs (bitwise) and per-stage device timings.  GPU helper, not a test."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2601_09258_b200 import abi, runtime as rt

cyc = int(sys.argv[1]) if len(sys.argv) > 1 else 3_700_000
t0 = time.time()
tr = rt.synth_trace(cyc, 7, 8, fault="nvlink_saturation", onset=cyc - 700_000, duration=150,
                    target_rank=3, n_ranks=8, n_chunks=64, n_threads=os.cpu_count(),
                    compact_names=False)
print("events", len(tr.events), "gen s", round(time.time() - t0, 1), flush=True)
an = rt.Analyzer(0)
an.configure(tr.names, rt.span_names_mask(tr.events, len(tr.names)), n_comm_slots=tr.n_comm)
an.upload(tr.events, [0, len(tr.events)], tr.workloads)
an.run(abi.RUN_SEGMENT)
recs = an.records(0)
t = recs[recs["cycle_index"] < 2400]
x = np.stack([t["batch"].astype(float), (t["batch"] * (t["input_len"] + t["output_len"])).astype(float)], 1)
an.load_model(rt.fit_latency_model(x, t["latency_s"]))
out = {}
for fused in [False, True]:
    an.set_fused(fused)
    ts = []
    for i in range(6):
        an.run(abi.RUN_ALL)
        ts.append(an.timings())
    print("fused" if fused else "legacy",
          {k: round(float(np.median([d[k] for d in ts[2:]])), 3) for k in ts[-1]}, flush=True)
    r = an.result(0)
    out[fused] = r
a, b = out[False], out[True]
for f in a.cycles.dtype.names:
    ok = np.array_equal(a.cycles[f], b.cycles[f])
    if not ok:
        bad = np.nonzero(a.cycles[f] != b.cycles[f])[0]
        print("CYCLES MISMATCH", f, len(bad), bad[:5], a.cycles[f][bad[:3]], b.cycles[f][bad[:3]])
for nm in ["components", "beta_totals", "beta", "coll_beta", "coll_present"]:
    if hasattr(a, nm):
        x1, x2 = getattr(a, nm), getattr(b, nm)
        print(nm, "equal" if np.array_equal(np.asarray(x1).view(np.uint8), np.asarray(x2).view(np.uint8)) else "MISMATCH")
print("records", "equal" if a.records.tobytes() == b.records.tobytes() else "MISMATCH")
print("alerts", len(a.alerts), len(b.alerts), a.alerts.tobytes() == b.alerts.tobytes())
