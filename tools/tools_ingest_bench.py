"""Chrome-trace JSON -> alerts on one B200 vs the reference's parse_trace_json
(GPU helper). configs[0]-shaped trace (simkit, 50 k cycles,
~1 M events, CpuContention at 40 k), serialised by the reference's own
serialize_trace_json. Times, on the box's host cores:
  - native cs_ingest_chrome_json (all threads, and 1 thread);
  - the whole JSON -> alerts path: ingest + cs_wire_pack + cs_upload_wire +
    cs_run(RUN_ALL) + alert read-back (model fit once beforehand, excluded);
  - the reference's parse_trace_json + export (oracle/_ref, 1 thread: the
    reference parser is single-threaded).
Writes gpurun_out/ingest_bench.json."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import refbridge as rb
from paper_2601_09258_b200 import abi, runtime as rt


def main():
    t = rb.RefTrace.synth(50_000, 1, 2, fault="cpu_contention", onset=40_000, duration=150)
    text = t.to_json()
    nt = os.cpu_count() or 1
    out = {"json_bytes": len(text), "host_threads": nt}

    def best(f, k=3):
        ts = []
        for _ in range(k):
            t0 = time.perf_counter()
            r = f()
            ts.append(time.perf_counter() - t0)
        return min(ts), r

    s_all, got = best(lambda: rt.ingest_chrome_json(text, n_threads=nt))
    s_one, _ = best(lambda: rt.ingest_chrome_json(text, n_threads=1), k=1)
    n = len(got.events)
    out.update(events=n, ingest_s=round(s_all, 4), ingest_1thread_s=round(s_one, 4),
               ingest_events_per_s=round(n / s_all), ingest_GB_per_s=round(len(text) / s_all / 1e9, 3))

    # reference parser (and the exporter that interns the same records)
    t0 = time.perf_counter()
    ref, n_issues = rb.RefTrace.from_json(text)
    out["reference_parse_s"] = round(time.perf_counter() - t0, 3)
    ex = ref.export(None)
    assert ex.events.tobytes() == got.events.tobytes() and n_issues == got.n_issues
    out["records_identical"] = True

    # JSON -> alerts on the GPU
    an = rt.Analyzer(0)
    an.configure(got.names, rt.span_names_mask(got.events, len(got.names)), n_comm_slots=got.n_comm)
    offs = [0, n]
    an.upload(got.events, offs, got.workloads)
    an.run(abi.RUN_SEGMENT)
    recs = an.records(0)
    tr = recs[recs["cycle_index"] < 2400]
    x = np.stack([tr["batch"].astype(float),
                  (tr["batch"] * (tr["input_len"] + tr["output_len"])).astype(float)], 1)
    model = rt.fit_latency_model(x, tr["latency_s"])
    an.load_model(model)

    def pipeline():
        g = rt.ingest_chrome_json(text, n_threads=nt)
        w = rt.wire_pack(g.events, offs, g.workloads, n_threads=nt)
        an.upload_wire(w)
        an.run(abi.RUN_ALL)
        return an.alerts(0)

    pipeline()
    s_pipe, alerts = best(pipeline)
    out.update(json_to_alerts_s=round(s_pipe, 4), json_to_alerts_events_per_s=round(n / s_pipe),
               alerts=len(alerts))
    an.close()
    print(json.dumps(out))
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/ingest_bench.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
