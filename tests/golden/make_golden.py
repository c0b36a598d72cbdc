#!/usr/bin/env python
"""Regenerates tests/golden/*.npz from the REFERENCE implementation itself
(oracle/_ref/libcsref.so = /root/reference/proj/src compiled unmodified).

Each fixture holds the input records (our 32-byte format, converted by the
reference-side exporter) and every output of the reference's hot path
(cycles, components, beta, collective beta, records with predictions /
residuals / control-chart state, alerts, anchor candidates).

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle import refbridge as rb  # noqa: E402
import traces  # noqa: E402

TINY_MODEL = traces.TINY_MODEL


def save(name, ex, ref, run_config, model_json, extra=None):
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"),
        events=ex.events, event_ids=ex.event_ids, workloads=ex.workloads,
        names=np.array(json.dumps(ex.names)), comm_hash=np.array(json.dumps(list(ex.comm_hash))),
        comm_rank=np.asarray(ex.comm_rank, np.int32),
        run_config=np.array(json.dumps(run_config or {})), model_json=np.array(model_json or ""),
        status=np.int32(ref.status), err_type=np.array(ref.err_type), anchor=np.array(ref.anchor),
        fallback=np.bool_(ref.fallback), cycles=ref.cycles, components=ref.components,
        beta_totals=ref.beta_totals, beta=ref.beta, coll_beta=ref.coll_beta,
        coll_present=ref.coll_present, records=ref.records, alerts=ref.alerts,
        candidates=ref.candidates, ucl=np.float64(ref.ucl),
        first_bad_record=np.uint64(ref.first_bad_record), **(extra or {}))
    print(f"{name}: {len(ex.events)} events, {len(ref.cycles)} cycles, "
          f"{len(ref.records)} records, {len(ref.alerts)} alerts, status={ref.err_type or 'ok'}")


def main():
    assert rb.available(), "build oracle/_ref first (make -C oracle)"
    small_det = {"detector": {"warmup": 0, "window": 3}}
    for name, fn in traces.ALL.items():
        b = traces.build(fn())
        cfg = json.loads(json.dumps(traces.CONFIG.get(name, {})))
        cfg.update(small_det)
        t = rb.RefTrace.build(b.events, b.names, b.workloads, b.comm_hash, b.comm_rank,
                              event_ids=b.event_ids, sort=True)
        model = json.dumps(TINY_MODEL)
        ref = t.run(cfg, model, 0)
        ex = t.export(cfg)
        assert np.array_equal(ex.events, b.events), name  # both ingests agree
        save(name, ex, ref, cfg, model)
    for name, (n, fam, ranks, seed) in {
            "simkit_nvlink_r2": (700, "nvlink_saturation", 2, 5),
            "simkit_cpu_r1": (700, "cpu_contention", 1, 9),
            "simkit_thrash_r1": (700, "memory_thrash", 1, 13)}.items():
        t = rb.RefTrace.synth(n, seed, seed + 1, fault=fam, onset=520, duration=60,
                              n_ranks=ranks, target_rank=1)
        cfg = {"detector": {"warmup": 50}}
        ref = t.run(cfg, None, 300)
        ex = t.export(cfg)
        save(name, ex, ref, cfg, ref.model_json, extra={"labels": t.labels()})


if __name__ == "__main__":
    main()
