"""configs[1] with forward_mode stripped and the keyword lists emptied: every
stage comes from the trailing-median heuristic (k_stage_jacobi).  Device step
time next to the forward_mode step, and the stages of a 100k-cycle prefix
checked against the reference.  GPU helper, not a test."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2601_09258_b200 import abi, runtime as rt

tr = rt.synth_trace(3_700_000, 7, 8, fault="nvlink_saturation", onset=3_000_000, duration=150,
                    target_rank=3, n_ranks=8, n_chunks=64, compact_names=False)
NO_KW = {"cycle": {"prefill_keywords": ["zz_none"], "decode_keywords": ["zz_none"]}}
out = {}
for label, strip in [("forward_mode", False), ("heuristic", True)]:
    ev = tr.events.copy()
    if strip:
        ev["flags"] &= np.uint16(0xFFFC)
    an = rt.Analyzer(0)
    an.configure(tr.names, rt.span_names_mask(ev, len(tr.names)), n_comm_slots=tr.n_comm,
                 run_config=NO_KW if strip else None)
    an.upload(ev, [0, len(ev)], tr.workloads)
    an.run(abi.RUN_SEGMENT)
    recs = an.records(0)
    t = recs[recs["cycle_index"] < 2400]
    x = np.stack([t["batch"].astype(float), (t["batch"] * (t["input_len"] + t["output_len"])).astype(float)], 1)
    an.load_model(rt.fit_latency_model(x, t["latency_s"]))
    ts = []
    for _ in range(8):
        an.run(abi.RUN_ALL)
        ts.append(an.timings())
    med = {k: round(float(np.median([d[k] for d in ts[3:]])), 4) for k in ts[-1]}
    st = an.cycles(0)["stage"]
    out[label] = {"phase_ms": med, "prefill_cycles": int((st == 0).sum()), "decode_cycles": int((st == 1).sum()),
                  "unknown_cycles": int((st == 2).sum())}
    if strip:
        from oracle import refbridge as rb
        if rb.available():
            n = int(an.cycles(0)["first_event"][100_000])
            t_ref = rb.RefTrace.build(ev[:n], tr.names, tr.workloads, ["comm0"] * tr.n_comm,
                                      list(range(tr.n_comm)), sort=False)
            ref = t_ref.run(NO_KW, None, 2400, beta=False)
            out[label]["stages_first_100k_identical"] = bool(
                np.array_equal(ref.cycles["stage"], st[:len(ref.cycles)]))
            out[label]["cycles_compared"] = int(len(ref.cycles))
    an.close()
out["ratio_total"] = out["heuristic"]["phase_ms"]["total"] / out["forward_mode"]["phase_ms"]["total"]
print(json.dumps(out))
