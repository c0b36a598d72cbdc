"""configs[1] (one 8-rank instance, ~100 M events) split into N cycle-range
shards with a verified halo (paper_2601_09258_b200/halo.py), run
on ONE B200 shard after shard (GPU helper).

For N in (2, 4, 8): every shard is uploaded (resident) and analysed with
cs_run; its device time is measured with the ctx's CUDA events (median of
`steps` runs), then split_device reads its halo / tail rows and alerts.  The
N-GPU step would cost max(shard device time) + the exchange (one all-gather of
the tails, a few KB, and the alert gather), so the line reports the max and
the sum of the per-shard times, the halo overhead (halo events / owned
events) and the host readback time of the split, and checks that every halo
was accepted and that the merged tables (cycles, components, beta,
collective beta, records, alerts) equal the whole-trace run's bit for bit.
Writes gpurun_out/halo_bench.json."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2601_09258_b200 import abi, halo as hl, runtime as rt


def main(steps=5, halo=1024):
    threads = os.cpu_count() or 1
    tr = rt.synth_trace(3_700_000, 7, 8, fault="nvlink_saturation", onset=3_000_000, duration=150,
                        target_rank=3, n_ranks=8, n_chunks=64, n_threads=threads, compact_names=False)
    ev, wl, names = tr.events, tr.workloads, list(tr.names)
    span = rt.span_names_mask(ev, len(names))
    anchor = names.index("run_batch")
    an = rt.Analyzer(0)
    an.configure(names, span, n_comm_slots=tr.n_comm, run_config={"cycle": {"anchor_hint": "run_batch"}})
    an.upload(ev, [0, len(ev)], wl)
    an.run(abi.RUN_SEGMENT)
    r = an.records(0)
    r = r[r["cycle_index"] < 2400]
    x = np.stack([r["batch"].astype(float), (r["batch"] * (r["input_len"] + r["output_len"])).astype(float)], 1)
    an.load_model(rt.fit_latency_model(x, r["latency_s"]))

    def timed():
        ts = []
        for _ in range(steps):
            an.run(abi.RUN_ALL)
            ts.append(an.timings()["total"])
        return statistics.median(ts)

    def full():
        r = an.result(0)
        return dict(cycles=r.cycles, records=r.records, alerts=r.alerts, components=r.components,
                    beta_totals=r.beta_totals, beta=r.beta, coll_beta=r.coll_beta,
                    coll_present=r.coll_present, status=r.summary.status,
                    first_bad_record=r.summary.first_bad_record)

    def same_tables(a, b):
        ok = np.array_equal(a["cycles"], b["cycles"])
        for k in ("components", "beta_totals", "beta", "coll_beta", "coll_present"):
            ok &= np.array_equal(np.asarray(a[k]).reshape(-1).view(np.uint8),
                                 np.asarray(b[k]).reshape(-1).view(np.uint8))
        for k in ("records", "alerts"):
            ok &= np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8))
        return bool(ok)

    an.run(abi.RUN_ALL)
    whole_ms = timed()
    whole_alerts = an.alerts(0)
    whole = full()
    out = {"events": len(ev), "cycles": int(an.summary(0).n_cycles), "halo_cycles": halo,
           "whole_ms": round(whole_ms, 4), "whole_alerts": len(whole_alerts), "shards": {}}
    cfg = hl.CheckConfig(stage_window=an.cycle.stage_window, window=an.control.window,
                         warmup=an.control.warmup)
    for world in (2, 4, 8):
        _, specs = hl.plan(ev, anchor, world, halo)
        parts, ms, split_ms, owned_full = [], [], [], []
        for s in specs:
            an.upload(np.ascontiguousarray(ev[s.lo:s.hi]), [0, s.hi - s.lo], wl)
            an.run(abi.RUN_ALL)
            ms.append(timed())
            t0 = time.perf_counter()
            parts.append(hl.split_device(s, an, halo))
            split_ms.append((time.perf_counter() - t0) * 1e3)
            owned_full.append(hl.split_local(s, full(), halo)[0])  # the whole tables, for parity
        tables_same = same_tables(whole, hl.merge(owned_full))
        del owned_full
        ok = [hl.halo_ok(specs[r], parts[r][1], [p[2] for p in parts[:r]], cfg) for r in range(world)]
        alerts, status, _ = hl.merge_alerts([p[0] for p in parts])
        same = np.array_equal(alerts.view(np.uint8), whole_alerts.view(np.uint8))
        halo_ev = sum(specs[r].hi - specs[r].lo for r in range(world)) - len(ev)
        out["shards"][world] = {
            "shard_ms": [round(v, 4) for v in ms], "max_shard_ms": round(max(ms), 4),
            "sum_shard_ms": round(sum(ms), 4), "split_readback_ms_max": round(max(split_ms), 3),
            "halo_events_frac": round(halo_ev / len(ev), 5), "halos_accepted": all(ok),
            "alerts_identical": bool(same), "all_tables_identical": tables_same, "status": status,
            "projected_events_per_s_device": round(len(ev) / (max(ms) * 1e-3)),
            "speedup_device_vs_whole": round(whole_ms / max(ms), 3)}
        assert all(ok) and same and tables_same, out["shards"][world]
    an.close()
    print(json.dumps(out))
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/halo_bench.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
