"""Single-read segmentation tuning sweep on the configs[1] trace: per range
size (option 96, events per warp range), the median segment_range / total
device ms of the fused run.  GPU helper, not a test.
python tools/tools_seg_sweep.py [range_events ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2601_09258_b200 import abi, runtime as rt

sizes = [int(x) for x in sys.argv[1:] if not x.startswith("p")] or [0]
aheads = [int(x[1:]) for x in sys.argv[1:] if x.startswith("p")] or [-1]
cyc = 3_700_000
tr = rt.synth_trace(cyc, 7, 8, fault="nvlink_saturation", onset=cyc - 700_000, duration=150,
                    target_rank=3, n_ranks=8, n_chunks=64, n_threads=os.cpu_count(), compact_names=False)
an = rt.Analyzer(0)
an.configure(tr.names, rt.span_names_mask(tr.events, len(tr.names)), n_comm_slots=tr.n_comm)
an.upload(tr.events, [0, len(tr.events)], tr.workloads)
an.run(abi.RUN_SEGMENT)
recs = an.records(0)
t = recs[recs["cycle_index"] < 2400]
x = np.stack([t["batch"].astype(float), (t["batch"] * (t["input_len"] + t["output_len"])).astype(float)], 1)
an.load_model(rt.fit_latency_model(x, t["latency_s"]))
an.set_fused(False)
an.run(abi.RUN_ALL)
ref = an.result(0)
an.set_fused(True)
for n, pa in [(n, pa) for n in sizes for pa in aheads]:
    an._ck(an.L.cs_set_option(an.h, 96, n))
    an._ck(an.L.cs_set_option(an.h, 97, pa))
    ts = []
    for i in range(7):
        an.run(abi.RUN_ALL)
        ts.append(an.timings())
    seg = float(np.median([d.get("segment_range", float("nan")) for d in ts[2:]]))
    tot = float(np.median([d["total"] for d in ts[2:]]))
    r = an.result(0)
    same = (r.cycles.tobytes() == ref.cycles.tobytes() and r.records.tobytes() == ref.records.tobytes()
            and r.alerts.tobytes() == ref.alerts.tobytes())
    print(f"range_events={n} ahead={pa} segment_range={seg:.3f} total={tot:.3f} identical={same}", flush=True)
