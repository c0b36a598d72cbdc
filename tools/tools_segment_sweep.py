"""Single-read segmentation (k_segment_range) tuning sweep at configs[1]:
range size (events) x L2 prefetch bytes, against the two-pass path; outputs
checked bitwise once.  GPU helper, not a test."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2601_09258_b200 import abi, runtime as rt

tr = rt.synth_trace(3_700_000, 7, 8, fault="nvlink_saturation", onset=3_000_000, duration=150,
                    target_rank=3, n_ranks=8, n_chunks=64, compact_names=False)
an = rt.Analyzer(0)
an.configure(tr.names, rt.span_names_mask(tr.events, len(tr.names)), n_comm_slots=tr.n_comm)
an.upload(tr.events, [0, len(tr.events)], tr.workloads)
an.run(abi.RUN_SEGMENT)
recs = an.records(0)
t = recs[recs["cycle_index"] < 2400]
x = np.stack([t["batch"].astype(float), (t["batch"] * (t["input_len"] + t["output_len"])).astype(float)], 1)
an.load_model(rt.fit_latency_model(x, t["latency_s"]))


def timed(n=6):
    ts = []
    for _ in range(n):
        an.run(abi.RUN_ALL)
        ts.append(an.timings())
    return {k: round(float(np.median([d[k] for d in ts[2:]])), 4) for k in ts[-1]}


an.set_fused(False)
print("two-pass", timed(), flush=True)
ref = an.result(0)
an.set_fused(True)
first = True
for rev in [int(a) for a in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["0", "4096", "6144", "8192", "12288"])]:
    for pf in [int(a) for a in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["-1", "0", "65536"])]:
        lib = rt.lib()
        lib.cs_set_option(an.h, 96, rev)
        lib.cs_set_option(an.h, 97, pf)
        tm = timed()
        print(f"range {rev} prefetch {pf}", tm, flush=True)
        if first:
            got = an.result(0)
            for f in ["cycles", "components", "beta", "records", "alerts"]:
                a, b = getattr(ref, f), getattr(got, f)
                ok = a.tobytes() == b.tobytes()
                print(f, "equal" if ok else "DIFFER", flush=True)
            first = False
