#!/usr/bin/env python
"""Benchmark: trace events/sec analysed on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c2|c1|c3|c5] [--c2-split replicas|halo]

Workload (default c2 = BASELINE configs[1]): one 8-rank tensor-parallel serving
instance, ~100 M events (3.70 M cycles x 27 events), mixed prefill/decode,
NvlinkSaturation x18 straggler on rank 3 — synthetic, produced by the simkit
restatement (cs_synth.cpp, byte-identical to the reference generator per
chunk; 64 chunks with substream seeds, generated on all host cores).  The
latency model is fit once in setup (one device batch over every instance,
cs_fit_latency_models, byte-identical to the reference's fit) on the first
2400 cycles.

A step = one cs_run over the whole instance: anchor discovery, segmentation,
stage classification, beta stage attribution, records, GBDT predict + ppe,
control chart + alerts.  `value` = events / device time per step with inputs
resident in HBM (CUDA events on the ctx stream, max over ranks).  `e2e` = the
same through the public C ABI with host buffers: H2D of the step's events
from pinned memory + cs_run + D2H of alerts and summary.
N > 1: one process per GPU, each analysing its own instance (instances shard
with no data-path collective: "weak" scaling); the per-shard alert lists and
summaries are gathered to rank 0 over NCCL.  `--c2-split halo` instead splits
configs[1]'s one instance into N cycle-range shards with a verified halo
(halo.py; "strong" scaling; one all-gather of shard tails per step).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "trace events/sec analysed (1/2/4/8 B200, % HBM roofline); alert parity vs CPU"
UNIT = "events/s"

WORKLOADS = {
    # name: (cycles, n_ranks, fault family, onset, duration, chunks, description)
    "c2": (3_700_000, 8, "nvlink_saturation", 3_000_000, 150, 64,
           "configs[1]: one 8-rank TP serving instance, ~100M events, mixed prefill/decode"),
    "c1": (50_000, 1, "cpu_contention", 40_000, 150, 1,
           "configs[0]: single decode instance, 1M events, injected stalls"),
    "c3": (97_700, 1, None, 0, 0, 1, "configs[2] shard: 128 instances x ~1.95M events per GPU"),
    "c5": (3_000, 1, None, 0, 0, 1, "configs[4]: streaming 10 ms micro-batches of a 1024-instance "
           "fleet per GPU, per-batch alert latency"),
}


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                p = [x.strip() for x in line.split(",")]
                if len(p) >= 9:
                    rows.append(p)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for k, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(k)
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(rows)}


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def dist_setup(dist, local_rank):
    """One process per GPU over NCCL: returns (device index, collective device).
    CS_BENCH_DIST_BACKEND=gloo with CS_BENCH_FORCE_DEVICE=0 runs every rank on
    one GPU with CPU collectives: a functional check of the N > 1 path on a
    single-GPU box (not a measurement)."""
    import torch
    backend = os.environ.get("CS_BENCH_DIST_BACKEND", "nccl")
    dev = int(os.environ.get("CS_BENCH_FORCE_DEVICE", local_rank))
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        return dev, f"cuda:{dev}"
    dist.init_process_group(backend)
    return dev, None


def run_reference(args, rank, world):
    """--impl reference: the reference CPU analyzer (oracle/_ref, compiled
    unmodified from /root/reference) on this box's host cores, rank 0 only,
    on the SAME trace the GPU arm times (bench.make_instance, rank 0's seed):
    each step analyses cycle-aligned slices of it (~1M events each, one per
    host thread, the fault window included) with the reference's own anchor
    discovery and fit.  Nothing of this repository's analysis path is used:
    the trace bytes come from the simkit restatement (benchlib), the anchor,
    model and every stage from the reference."""
    if rank != 0:
        return
    from oracle import refbridge as rb
    cores = cpu_cores()
    line = {"impl": "reference", "metric": METRIC, "unit": UNIT, "n_gpus": args.gpus,
            "higher_is_better": True}
    if not rb.available():
        line["unavailable"] = "oracle/_ref/libcsref.so not built"
        print(json.dumps(line))
        return
    from paper_2601_09258_b200 import runtime as rt
    if args.workload in ("c2", "c1"):
        tr = make_instance(rt, args.workload, 7, cores)
        onset = WORKLOADS[args.workload][3]
        anchor, model_json = reference_anchor_and_model(rb, tr.events, tr.names, tr.workloads, tr.n_comm)
        aid = tr.names.index(anchor)
        apos = np.flatnonzero((tr.events["kind"] == 0) & (tr.events["name_id"] == aid))
        center = int(apos[min(onset, len(apos) - 1)]) if onset else None
        per_slice = max(1, min(1_000_000, len(tr.events) // cores))
        cb, _, _ = cpu_reference_same_trace(rb, tr.events, tr.names, tr.workloads, tr.n_comm, cores,
                                            per_slice, center, model_json, anchor)
        sample = (f"{cores} cycle-aligned slices (~{per_slice} events each, {cb.events} of the "
                  f"{len(tr.events)} events) of the GPU arm's benchmarked trace, one per std::thread, "
                  f"anchor '{anchor}' and model from the reference itself; segment_and_classify + beta "
                  f"cycle_stats + build_cycle_records + predict + ppe + Detector::step")
        same = True
    else:
        cyc, ranks = 50_000, 1
        cb = rb.CpuBaseline(cores, cores, cyc, ranks, seed=42)
        sample = (f"{cores} simkit instances x {cyc} cycles (R={ranks}, {cb.events} events), one per "
                  f"std::thread; segment_and_classify + build_cycle_records + beta cycle_stats + predict + "
                  f"ppe + Detector::step")
        same = False
    for _ in range(args.warmup):
        cb.run()
    times, alerts = [], 0
    for _ in range(args.steps):
        s, alerts = cb.run()
        times.append(s)
    ms = 1e3 * sum(times) / len(times)
    value = cb.events / (ms / 1e3)
    line.update({
        "value": value, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "scaling": "weak", "vs_baseline": None, "dtype": "int64+f64",
        "data": "synthetic (simkit restatement, byte-identical to the reference generator per chunk)",
        "config": {"workload": WORKLOADS[args.workload][6], "sample": sample, "same_trace": same},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "alerts": alerts,
    })
    cb.close()
    print(json.dumps(line))


def cycle_aligned_slices(ev, anchor_id, n_slices, per_slice, center_event=None):
    """[lo, hi) event ranges that start at an anchor's lower_bound group and end
    at a later anchor's: each holds whole cycles, so the reference run on the
    slice (with the same anchor) reproduces those cycles exactly
    (cycles.cpp:120-170).  Evenly spaced; with center_event, the middle slice
    is centred there (the fault window)."""
    ts = ev["start_ts"]
    apos = np.flatnonzero((ev["kind"] == 0) & (ev["name_id"] == anchor_id))
    n = len(ev)
    per_slice = min(per_slice, max(1, n // max(1, n_slices)))
    starts = np.linspace(0, max(0, n - per_slice), n_slices).astype(np.int64)
    if center_event is not None and n_slices:
        starts[n_slices // 2] = max(0, min(n - per_slice, center_event - per_slice // 2))
    lo, hi = [], []
    for s in starts:
        a = min(np.searchsorted(apos, s), len(apos) - 1)
        b = min(np.searchsorted(apos, s + per_slice), len(apos) - 1)
        lo.append(int(np.searchsorted(ts, ts[apos[a]], "left")))
        hi.append(int(np.searchsorted(ts, ts[apos[b]], "left")))
    return np.array(lo, np.uint64), np.array(hi, np.uint64)


def reference_anchor_and_model(rb, events, names, workloads, n_comm, head_events=3_000_000):
    """The reference's own anchor discovery and fit (fit_latency_model on the
    first 2400 cycles) on the head of the trace."""
    head = events[:min(len(events), head_events)]
    t = rb.RefTrace.build(head, names, workloads, ["comm0"] * n_comm, list(range(n_comm)), sort=False)
    r = t.run(None, None, 2400)
    if r.status != 0:
        raise RuntimeError(f"reference could not fit on the head: {r.err_type}")
    return r.anchor, r.model_json


def cpu_reference_same_trace(rb, events, names, workloads, n_comm, cores, per_slice, center_event,
                             model_json=None, anchor=None):
    """The reference analyzer (oracle/_ref) on cycle-aligned slices of THIS
    trace, one slice per host thread, anchor and model from the reference
    itself unless given.  Returns (CpuBaseline, anchor, model_json)."""
    if anchor is None or model_json is None:
        anchor, model_json = reference_anchor_and_model(rb, events, names, workloads, n_comm)
    lo, hi = cycle_aligned_slices(events, names.index(anchor), cores, per_slice, center_event)
    cb = rb.CpuBaseline.slices(events, None, names, workloads, ["comm0"] * n_comm, list(range(n_comm)),
                               lo, hi, model_json, anchor, cores)
    return cb, anchor, model_json


def make_instance(rt, workload, seed, threads):
    cyc, ranks, fault, onset, dur, chunks, _ = WORKLOADS[workload]
    return rt.synth_trace(cyc, seed, seed + 1, fault=fault, onset=onset, duration=dur,
                          target_rank=3 % ranks, n_ranks=ranks, n_chunks=chunks,
                          n_threads=threads, compact_names=False)


def run_ours(args, rank, world, local_rank):
    import ctypes as C

    import torch

    from paper_2601_09258_b200 import abi, dist as cdist, runtime as rt

    dist = None
    if world > 1:
        import torch.distributed as dist
        dev, cdev = dist_setup(dist, local_rank)
    else:
        dev, cdev = local_rank, f"cuda:{local_rank}"
    threads = max(1, cpu_cores() // max(1, env_int("LOCAL_WORLD_SIZE", world)))

    t_setup = time.time()
    if args.workload == "c3":
        # configs[2]: 1024 instances over 8 GPUs = 128 per GPU (SURVEY §8d C3:
        # seeds substream(42, i) in the reference; distinct seeds per instance here)
        import concurrent.futures as cf
        per_gpu = 128
        with cf.ThreadPoolExecutor(max(1, threads)) as ex:
            traces = list(ex.map(lambda i: rt.synth_trace(
                WORKLOADS["c3"][0], 1000 + rank * per_gpu + i, 5000 + rank * per_gpu + i,
                fault=rt.FAULT_FAMILIES[i % 8], onset=80_000, duration=150, compact_names=False,
                n_threads=1), range(per_gpu)))
    else:
        traces = [make_instance(rt, args.workload, 7 + 1000 * rank, threads)]
    names = traces[0].names
    events = np.concatenate([t.events for t in traces]) if len(traces) > 1 else traces[0].events
    wl_parts, offs, base = [], [0], 0
    if len(traces) > 1:
        evs = []
        for t in traces:
            ev = t.events.copy()
            has = (ev["flags"] & abi.EV_HAS_BATCH) != 0
            ev["payload"][has] = (ev["payload"][has] & np.uint64(0xFFFFFFFF00000000)) | \
                ((ev["payload"][has] & np.uint64(0xFFFFFFFF)) + np.uint64(base))
            base += len(t.workloads)
            wl_parts.append(t.workloads)
            evs.append(ev)
            offs.append(offs[-1] + len(ev))
        events = np.concatenate(evs)
        workloads = np.concatenate(wl_parts)
    else:
        workloads = traces[0].workloads
        offs = [0, len(events)]
    n_comm = max(t.n_comm for t in traces)
    n_events = len(events)
    n_inst = len(offs) - 1
    del traces

    # pinned host copy (e2e leg) + resident device copy (value leg)
    ev_bytes = events.nbytes
    wl_bytes = workloads.nbytes
    pin_ptr, pin = rt.host_alloc(ev_bytes + wl_bytes)
    pin[:ev_bytes] = events.view(np.uint8)
    pin[ev_bytes:] = workloads.view(np.uint8)
    pin_ev = pin[:ev_bytes].view(abi.EVENT_DTYPE)
    pin_wl = pin[ev_bytes:].view(abi.WORKLOAD_DTYPE)
    del events

    an = rt.Analyzer(dev)
    an.set_fused(os.environ.get("CS_BENCH_FUSED", "1") != "0")
    span = rt.span_names_mask(pin_ev, len(names))
    an.configure(names, span, n_comm_slots=n_comm)
    an.upload(pin_ev, offs, pin_wl)
    # setup: fit the model on the first 2400 cycles of each instance (A17, host)
    an.run(abi.RUN_SEGMENT)
    # one device batch for every instance's model (cs_fit_latency_models,
    # byte-identical to the reference's per-instance fit)
    xs, ys = [], []
    for i in range(n_inst):
        recs = an.records(i)
        tr = recs[recs["cycle_index"] < 2400]
        xs.append(np.stack([tr["batch"].astype(float),
                            (tr["batch"] * (tr["input_len"] + tr["output_len"])).astype(float)], 1))
        ys.append(tr["latency_s"])
    t0 = time.time()
    models, _ = rt.fit_latency_models(xs, ys, device=dev, n_threads=threads)
    fit_s = time.time() - t0
    for i, model in enumerate(models):
        if isinstance(model, Exception):
            raise model
        an.load_model(model, inst=i)
    setup_s = time.time() - t_setup

    mask = abi.RUN_ALL
    for _ in range(args.warmup):
        an.run(mask)
    # per-phase device times from one untimed run; the timed steps record
    # events only around the segmentation pass (CS_OPT_PHASE_TIMINGS=2: an
    # event between two small kernels ends their launch overlap)
    an.run(mask)
    phase_hist = [an.timings()]
    an.set_phase_timings(2)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(dev)
    clocks.start()
    time.sleep(0.3)
    step_ms, scan_ms, reduce_ms, launches = [], [], [], 0
    for _ in range(args.steps):
        an.run(mask)
        tm = an.timings()
        step_ms.append(tm["total"])
        if "segment_range" in tm:
            scan_ms.append(tm["segment_range"])
            reduce_ms.append(0.0)
        else:
            scan_ms.append(tm["scan_events"])
            reduce_ms.append(tm["cycle_reduce"])
        launches += an.launches()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    clk = clocks.stop()
    dev_ms = sum(step_ms) / len(step_ms)

    # e2e through the public API with host buffers.  Headline: the producer
    # hands the step's cs_event records (the ABI's native input, 32 B/event)
    # in pinned host memory; every step copies them in (cs_upload), runs the
    # path and reads alerts + summaries back.  Variants reported beside it:
    # the columnar wire format with the host encoder (cs_wire_pack) timed
    # inside the step, and the same wire batch pre-packed (producer-side
    # encoding excluded; an upper bound, not the headline).
    t_pack = time.perf_counter()
    wt = rt.wire_pack(pin_ev, offs, pin_wl, n_threads=threads)
    pack_s = time.perf_counter() - t_pack
    cols = [getattr(wt, c) for c in rt.WireTrace.COLUMNS]
    if wt.workloads32 is None:  # a workload value that does not fit u32: the i64 table travels
        cols[-1] = pin_wl
    wire_bytes = sum(a.nbytes for a in cols)
    wptr, wpin = rt.host_alloc(max(1, wire_bytes + 16 * len(cols)))
    views, o = [], 0
    for a in cols:
        o = (o + 15) & ~15
        wpin[o:o + a.nbytes] = a.view(np.uint8).reshape(-1)
        views.append(wpin[o:o + a.nbytes].view(a.dtype).reshape(a.shape))
        o += a.nbytes
    if wt.workloads32 is None:
        wire = rt.WireTrace(*views[:-1], None, wt.inst_offsets)
        wire_wl = views[-1]
    else:
        wire = rt.WireTrace(*views, wt.inst_offsets)
        wire_wl = None
    wire_bytes_per_event = wire_bytes / n_events
    del wt, cols

    def e2e_leg(upload):
        times, d2h_b, n_al = [], 0, 0
        for k in range(args.warmup + args.steps):
            if dist:
                dist.barrier()
            t0 = time.perf_counter()
            upload()
            an.run(mask)
            al = [an.alerts(i) for i in range(n_inst)]
            _ = [an.summary(i) for i in range(n_inst)]
            payload = np.concatenate(al).view(np.uint8) if al else np.zeros(0, np.uint8)
            if dist:
                # final gather of per-shard alerts to rank 0 (NCCL over NVLink)
                cdist.gather_bytes(payload, device=cdev)
                torch.cuda.synchronize(dev)
            el = (time.perf_counter() - t0) * 1e3
            if k >= args.warmup:
                times.append(el)
                d2h_b = payload.nbytes + n_inst * C.sizeof(abi.InstanceSummary)
                n_al = sum(len(a) for a in al)
        return sum(times) / len(times), d2h_b, n_al

    e2e32_seq, d2h, alerts_total = e2e_leg(lambda: an.upload(pin_ev, offs, pin_wl))

    def upload_wire_with_pack(a):
        w = rt.wire_pack(pin_ev, offs, pin_wl, n_threads=threads)  # host encoder inside the step
        a.upload_wire(w, None if w.workloads32 is not None else pin_wl)

    e2e_pack_seq, _, _ = e2e_leg(lambda: upload_wire_with_pack(an))
    e2e_wire_seq, _, _ = e2e_leg(lambda: an.upload_wire(wire, wire_wl))

    # Serving pattern: two contexts on their own non-blocking streams, one
    # host thread each taking alternate steps, uploads issued one at a time
    # (cs_upload / cs_upload_wire return when their copies are done), so one
    # step's upload over PCIe overlaps the other's analysis.  Every step still
    # copies its inputs from pinned memory and reads its alerts and summaries
    # back inside the timed region; ms_per_step = wall time / steps.  With
    # N > 1 the per-step gather of each step's alerts to rank 0 is issued by
    # the main thread, in step order (one communicator, one issuing thread,
    # the same collective sequence on every rank).
    import threading
    an2 = rt.Analyzer(dev)
    an2.set_fused(os.environ.get("CS_BENCH_FUSED", "1") != "0")
    an2.configure(names, span, n_comm_slots=n_comm)
    for i, model in enumerate(models):
        an2.load_model(model, inst=i)
    ctxs = [an, an2]
    link = threading.Lock()  # one upload on the host link at a time

    def pipelined(upload):
        def step(a):
            with link:
                upload(a)  # returns when its copies are done
            a.run(mask)
            al = [a.alerts(i) for i in range(n_inst)]
            _ = [a.summary(i) for i in range(n_inst)]
            return al

        for a in ctxs:
            for _ in range(max(1, args.warmup // 2)):
                step(a)
        done = [threading.Event() for _ in range(args.steps)]
        payloads = [None] * args.steps
        n_alerts_step = [0] * args.steps

        def worker(j):
            for k in range(j, args.steps, 2):
                al = step(ctxs[j])
                n_alerts_step[k] = sum(len(x) for x in al)
                payloads[k] = np.concatenate(al).view(np.uint8) if al else np.zeros(0, np.uint8)
                done[k].set()

        if dist:
            dist.barrier()
        th = [threading.Thread(target=worker, args=(j,)) for j in range(2)]
        t0 = time.perf_counter()
        for x in th:
            x.start()
        for k in range(args.steps):
            done[k].wait()
            if dist:
                cdist.gather_bytes(payloads[k], device=cdev)
        for x in th:
            x.join()
        if dist and cdev is not None:
            torch.cuda.synchronize(dev)
        assert all(n == alerts_total for n in n_alerts_step)
        return (time.perf_counter() - t0) * 1e3 / args.steps

    e2e = pipelined(lambda a: a.upload(pin_ev, offs, pin_wl))
    e2e_wire = pipelined(lambda a: a.upload_wire(wire, wire_wl))
    pipeline = 2
    an2.close()
    rt.host_free(wptr)

    if dist:
        dev_ms = cdist.max_over_ranks(dev_ms, device=cdev)
        e2e = cdist.max_over_ranks(e2e, device=cdev)
        e2e_wire = cdist.max_over_ranks(e2e_wire, device=cdev)
        e2e32_seq = cdist.max_over_ranks(e2e32_seq, device=cdev)
        e2e_pack_seq = cdist.max_over_ranks(e2e_pack_seq, device=cdev)
        e2e_wire_seq = cdist.max_over_ranks(e2e_wire_seq, device=cdev)

    # roofline: dominant kernel measured live (CUDA events on the ctx stream)
    import json as _json
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = _json.load(f)
    except OSError:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    summ = [an.summary(i) for i in range(n_inst)]
    n_cycles = sum(s.n_cycles for s in summ)
    n_records = sum(s.n_records for s in summ)
    P, Cs, R = an.cycle.n_phases, an.cycle.n_beta_slots, an.cycle.n_comm_slots
    # algorithmic bytes per launch
    cyc_out = n_cycles * (48 + 4 + 2 + 4 + 8 * P + 8 * Cs + 9 * R)  # per-cycle outputs (beta quotients formed on read)
    scan_t = sum(scan_ms) / len(scan_ms)
    red_t = sum(reduce_ms) / len(reduce_ms)
    if red_t == 0.0:  # single-read segmentation: events read once, cycle outputs written once
        dom = ("segment_range", 32 * n_events + cyc_out + 24 * n_cycles, scan_t)
    else:
        scan_bytes = 32 * n_events + 24 * (n_cycles + n_inst)
        reduce_bytes = 32 * n_events + 32 * n_cycles + cyc_out
        dom = (("cycle_reduce", reduce_bytes, red_t) if red_t >= scan_t
               else ("scan_events", scan_bytes, scan_t))
    achieved = dom[1] / (dom[2] * 1e-3) / 1e9
    # dram bytes of the dominant kernel from the committed ncu --set full
    # capture of this same command (profiles/r2_ncu_traffic.json, else r1); only for
    # the default workload it was taken on
    traffic = None
    kname = {"cycle_reduce": "k_cycle_reduce_v2", "scan_events": "k_scan_warp",
             "segment_range": "k_segment_range"}[dom[0]]
    step_dram = None  # ncu DRAM bytes of the step's captured kernels (the full capture)
    tpath = os.path.join(ROOT, "profiles", "r2_ncu_traffic.json")
    try:
        if not os.path.exists(tpath):
            tpath = os.path.join(ROOT, "profiles", "r1_ncu_traffic.json")
        with open(tpath) as f:
            allk = json.load(f)
        tr = allk.get(kname)
        if tr and args.workload == "c2":
            traffic = tr["dram_read_bytes"] + tr["dram_write_bytes"]
            step_dram = sum(v["dram_read_bytes"] + v["dram_write_bytes"] for k, v in allk.items()
                            if not k.endswith("_2"))  # one launch per kernel of one step
    except (OSError, ValueError):
        pass
    path_bytes = 44.5 * n_events  # SURVEY §8d per-event figure
    line = {
        "metric": METRIC,
        "value": world * n_events / (dev_ms * 1e-3),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dev_ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int64+f64",
        "data": "synthetic (simkit restatement, byte-identical to the reference generator per chunk)",
        "config": {"workload": WORKLOADS[args.workload][6], "events_per_gpu": n_events,
                   "instances_per_gpu": n_inst, "cycles_per_gpu": n_cycles,
                   "records_per_gpu": n_records, "parallelism": f"instance-sharded x{world}",
                   "l2": f"inputs ({(ev_bytes + wl_bytes) / 1e9:.1f} GB/GPU) larger than L2; no flush needed",
                   "model_fit_s": round(fit_s, 3), "setup_s": round(setup_s, 1)},
        "roofline": {"bound": "hbm", "kernel": dom[0], "achieved": achieved, "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "algorithmic_bytes": dom[1],
                     "traffic_source": os.path.relpath(tpath, ROOT) + " (ncu --set full, dram read+write)",
                     "kernel_ms": dom[2], "event_pass_ms": scan_t, "cycle_reduce_ms": red_t,
                     "path_frac_44p5B_per_event": path_bytes / (dev_ms * 1e-3) / 1e9 / peak,
                     "step_dram_frac_ncu": (step_dram / (dev_ms * 1e-3) / 1e9 / peak) if step_dram else None,
                     "step_dram_note": "ncu DRAM read+write of one launch of each captured kernel "
                                       "(segmentation, records, score, detect, stage) over the measured step time"},
        "e2e": {"value": world * n_events / (e2e * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": ev_bytes + wl_bytes, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e,
                "input": "cs_event records (32 B/event) + workload table from pinned host memory (cs_upload)",
                "timer": "host wall clock around the synchronous API calls",
                "pipeline": pipeline, "ms_per_step_one_context": e2e32_seq,
                "wire_incl_host_pack": {
                    "value": world * n_events / (e2e_pack_seq * 1e-3), "ms_per_step": e2e_pack_seq,
                    "note": "cs_wire_pack of the step's cs_event records on the host threads + "
                            "cs_upload_wire + run + read-back, one context"},
                "wire_prepacked": {
                    "value": world * n_events / (e2e_wire * 1e-3), "ms_per_step": e2e_wire,
                    "ms_per_step_one_context": e2e_wire_seq,
                    "h2d_bytes_per_step": wire_bytes,
                    "note": f"columnar wire format ({wire_bytes_per_event:.1f} B/event) packed once "
                            "outside the timed region: an upper bound for a producer that emits it"},
                "host_pack": {"seconds": pack_s, "events_per_s": n_events / pack_s,
                              "input_gbs": (ev_bytes + wl_bytes) / pack_s / 1e9, "threads": threads}},
        "gpu_launches": launches,
        "phase_ms": {k: round(float(np.median([d[k] for d in phase_hist])), 4)
                     for k in phase_hist[-1]},
        "phase_ms_source": "one untimed run with an event between every phase (timed steps: events around the segmentation pass only)",
        "clocks": clk,
        "alerts_per_step": alerts_total,
    }
    # same-run alert parity and the CPU baseline, both on the benchmarked
    # trace itself (rank 0; the oracle library is the checker / baseline only)
    if rank == 0 and len(offs) == 2 and not args.no_parity:
        try:
            from oracle import refbridge as rb
            if rb.available():
                anchor = names[an.summary(0).anchor_name_id]
                line["parity"] = rb.full_parity(an, pin_ev, names, pin_wl, n_comm, models[0].to_json(),
                                                anchor, cpu_cores())
        except Exception as e:  # report, never hide
            line["parity"] = {"identical": None, "error": repr(e)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import refbridge as rb
            if rb.available() and len(offs) == 2:
                cores = cpu_cores()
                onset = WORKLOADS[args.workload][3]
                cyc_tab = an.cycles(0)
                center = int(cyc_tab["first_event"][min(onset, len(cyc_tab) - 1)]) if onset else None
                cb, anchor_r, _ = cpu_reference_same_trace(rb, pin_ev, names, pin_wl, n_comm, cores,
                                                           1_000_000, center, models[0].to_json(),
                                                           names[an.summary(0).anchor_name_id])
                cb.run()
                secs, _ = cb.run()
                line["cpu_baseline"] = {
                    "value": cb.events / secs, "unit": UNIT, "cores": cores, "kind": "reference",
                    "same_trace": True,
                    "sample": f"{cores} cycle-aligned slices (~1M events each, {cb.events} events) of "
                              f"this benchmarked trace, one per std::thread, the trace's anchor and model: "
                              f"segment_and_classify + beta cycle_stats + build_cycle_records + "
                              f"predict + ppe + Detector::step"}
                cb.close()
        except Exception as e:  # the baseline must not break the bench line
            line["cpu_baseline"] = {"value": None, "error": repr(e)}
    if rank == 0:
        print(json.dumps(line))
    an.close()
    rt.host_free(pin_ptr)
    if dist:
        dist.destroy_process_group()


def run_stream(args, rank, world, local_rank):
    """configs[4]: monitor_loop over 10 ms slices of trace time for a fleet of
    instances, one cs_stream_push per slice (tails, H2D, run, alerts on the
    host).  64 distinct simkit instances tiled x16 (distinct instance ids) =
    1024 instances per GPU; one model (fit on instance 0) for all; anchor from
    instance 0.  Reports events/s over the streamed slices and the per-slice
    latency distribution."""
    import concurrent.futures as cf

    import torch

    from paper_2601_09258_b200 import abi, dist as cdist, runtime as rt

    dist = None
    if world > 1:
        import torch.distributed as dist
        dev, cdev = dist_setup(dist, local_rank)
    else:
        dev, cdev = local_rank, f"cuda:{local_rank}"
    cyc = WORKLOADS["c5"][0]
    n_distinct, tile = 64, 16
    with cf.ThreadPoolExecutor(max(1, cpu_cores())) as ex:
        traces = list(ex.map(lambda i: rt.synth_trace(
            cyc, 2000 + 97 * rank + i, 9000 + 97 * rank + i, fault=rt.FAULT_FAMILIES[i % 8],
            onset=cyc - 600, duration=150, compact_names=False, n_threads=1), range(n_distinct)))
    names = traces[0].names
    # one workload table for the fleet; event payloads remapped into it
    evs, wls, base = [], [], 0
    for t in traces:
        ev = t.events.copy()
        has = (ev["flags"] & abi.EV_HAS_BATCH) != 0
        ev["payload"][has] = (ev["payload"][has] & np.uint64(0xFFFFFFFF00000000)) | \
            ((ev["payload"][has] & np.uint64(0xFFFFFFFF)) + np.uint64(base))
        base += len(t.workloads)
        wls.append(t.workloads)
        evs.append(ev)
    wl = np.concatenate(wls)
    fleet = [evs[i % n_distinct] for i in range(n_distinct * tile)]
    n_inst = len(fleet)
    an = rt.Analyzer(dev)
    an.configure(names, rt.span_names_mask(evs[0], len(names)), n_comm_slots=max(t.n_comm for t in traces))
    an.upload(evs[0], [0, len(evs[0])], wl)
    an.run(abi.RUN_SEGMENT)
    anchor = an.summary(0).anchor_name_id
    recs = an.records(0)
    tr = recs[recs["cycle_index"] < 1500]
    x = np.stack([tr["batch"].astype(float),
                  (tr["batch"] * (tr["input_len"] + tr["output_len"])).astype(float)], 1)
    an.load_model(rt.fit_latency_model(x, tr["latency_s"]))
    an.cycle.anchor_hint_name = anchor
    an.set_config(an.cycle, an.control)
    # 10 ms slices of trace time, prepared before timing.  The timed slices
    # start just before instance 0's fault onset (cycle cyc - 600), so alerts
    # are in flight in the measured micro-batches; everything before is the
    # history pushed untimed (the detector warms up on it).
    t0 = min(int(e["start_ts"][0]) for e in evs)
    slice_ns = 10_000_000
    n_slices = args.warmup + args.steps + 1  # + one untimed slice with per-phase device events
    onset_ts = int(an.cycles(0)["start_ts"][cyc - 600])
    first = max(t0 + 20 * slice_ns, onset_ts - (args.warmup + 1) * slice_ns)
    cuts = [[int(np.searchsorted(e["start_ts"], first + k * slice_ns)) for k in range(n_slices + 1)]
            for e in evs]
    # each slice's events sit in pinned host memory, as a producer writing
    # into a pinned ring would leave them (staged outside the timer)
    batches, pins = [], []
    for k in range(n_slices):
        parts = [fleet[i][cuts[i % n_distinct][k]:cuts[i % n_distinct][k + 1]] for i in range(n_inst)]
        off = np.zeros(n_inst + 1, np.uint64)
        off[1:] = np.cumsum([len(p) for p in parts])
        cat = np.concatenate(parts)
        ptr, buf = rt.host_alloc(max(1, cat.nbytes))
        pins.append(ptr)
        ev_pin = buf[:cat.nbytes].view(abi.EVENT_DTYPE)
        ev_pin[:] = cat
        batches.append((ev_pin, off))
    st = an.stream()
    head = np.concatenate([f[:cuts[i % n_distinct][0]] for i, f in enumerate(fleet)])
    hoff = np.zeros(n_inst + 1, np.uint64)
    hoff[1:] = np.cumsum([cuts[i % n_distinct][0] for i in range(n_inst)])
    st.push_packed(head, hoff, wl)  # history up to the first slice (uploads the workload table)
    lat, n_ev, n_alerts, launches, dev_ms = [], 0, 0, 0, []
    torch.cuda.synchronize(dev)
    for k, (ev, off) in enumerate(batches[:-1]):
        if dist:
            dist.barrier()
        t_s = time.perf_counter()
        al = st.push_packed(ev, off)
        el = time.perf_counter() - t_s
        if k >= args.warmup:
            lat.append(el * 1e3)
            n_ev += len(ev)
            n_alerts += len(al)
            launches += an.launches()
            dev_ms.append(an.timings()["total"])
    # device phases: pushes record only their total (an event between the
    # small kernels costs device time); one more slice, untimed, with phases
    an.set_phase_timings(1)
    st.push_packed(*batches[-1])
    phase_ms = {k: round(v, 4) for k, v in an.timings().items()}
    st.close()
    del batches
    for ptr in pins:
        rt.host_free(ptr)
    total_s = sum(lat) / 1e3
    if dist:
        total_s = cdist.max_over_ranks(total_s, device=cdev)
    value = world * n_ev / total_s
    lat_s = sorted(lat)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sum(lat) / len(lat), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64+f64",
        "data": "synthetic (simkit restatement), 64 distinct instances tiled x16",
        "config": {"workload": WORKLOADS["c5"][6], "instances_per_gpu": n_inst,
                   "slice_ms_trace_time": slice_ns / 1e6,
                   "events_per_slice": n_ev / len(lat), "step": "one cs_stream_push per slice"},
        "latency_ms": {"p50": lat_s[len(lat_s) // 2], "p99": lat_s[min(len(lat_s) - 1, int(0.99 * len(lat_s)))],
                       "max": lat_s[-1],
                       "timer": "host wall clock: events on host -> alerts on host"},
        "alerts": n_alerts,
        "device_phase_ms_extra_slice": phase_ms,
        "device_ms_per_slice_median": statistics.median(dev_ms),
        # the line is already measured host to host through cs_stream_push
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": int(32 * n_ev / len(lat)),
                "d2h_bytes_per_step": int(abi.ALERT_DTYPE.itemsize * n_alerts / len(lat)),
                "ms_per_step": sum(lat) / len(lat),
                "input": "each slice's 32-B events in pinned host memory (cs_stream_push)"},
        "gpu_launches": launches,
    }
    if rank == 0:
        print(json.dumps(line))
    an.close()
    if dist:
        dist.destroy_process_group()


def run_halo(args, rank, world, local_rank):
    """--c2-split halo: configs[1]'s single instance split into N cycle-range
    shards, one per GPU, each with a 1024-cycle halo (halo.py):
    strong scaling of one instance.  A step = cs_run on the resident shard
    (device time, CUDA events), then the exchange: the shard's halo / tail rows
    and alerts read back (split_device), one all-gather of the tails (a few
    KB), the halo acceptance check and the alert gather to rank 0.  `value`
    = the instance's events / max over ranks of the device time; the
    exchange is reported beside it and is inside `e2e` (wire upload of the
    shard + step + exchange, wall clock)."""
    import ctypes as C

    import torch

    from paper_2601_09258_b200 import abi, dist as cdist, halo as hl, runtime as rt

    dist = None
    if world > 1:
        import torch.distributed as dist
        dev, cdev = dist_setup(dist, local_rank)
    else:
        dev, cdev = local_rank, f"cuda:{local_rank}"
    threads = max(1, cpu_cores() // max(1, env_int("LOCAL_WORLD_SIZE", world)))

    def allgather(obj):
        if not dist:
            return [obj]
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    t_setup = time.time()
    tr = make_instance(rt, "c2", 7, threads)  # the same instance on every rank
    ev, wl, names = tr.events, tr.workloads, list(tr.names)
    n_events = len(ev)
    span = rt.span_names_mask(ev, len(names))
    an = rt.Analyzer(dev)
    an.configure(names, span, n_comm_slots=tr.n_comm)
    # setup: the whole-trace anchor discovery and the model fit on the first
    # 2400 cycles, identical on every rank; then the anchor is fixed
    an.upload(ev, [0, n_events], wl)
    an.run(abi.RUN_SEGMENT)
    anchor = int(an.summary(0).anchor_name_id)
    recs = an.records(0)
    recs = recs[recs["cycle_index"] < 2400]
    x = np.stack([recs["batch"].astype(float),
                  (recs["batch"] * (recs["input_len"] + recs["output_len"])).astype(float)], 1)
    model = rt.fit_latency_model(x, recs["latency_s"])
    an.configure(names, span, n_comm_slots=tr.n_comm, run_config={"cycle": {"anchor_hint": names[anchor]}})
    an.load_model(model)
    halo = 1024
    _, specs = hl.plan(ev, anchor, world, halo)
    spec = specs[rank]
    loc = np.ascontiguousarray(ev[spec.lo:spec.hi])
    an.upload(loc, [0, len(loc)], wl)
    cfg = hl.CheckConfig(stage_window=an.cycle.stage_window, window=an.control.window,
                         warmup=an.control.warmup)
    wt = rt.wire_pack(loc, [0, len(loc)], wl, n_threads=threads)
    if wt.workloads32 is None:
        raise RuntimeError("configs[1] workloads fit the u32 wire column")
    cols = [getattr(wt, c) for c in rt.WireTrace.COLUMNS]
    wire_bytes = sum(a.nbytes for a in cols)
    wptr, wpin = rt.host_alloc(wire_bytes + 16 * len(cols))  # pinned, as in run_ours
    views, o = [], 0
    for a in cols:
        o = (o + 15) & ~15
        wpin[o:o + a.nbytes] = a.view(np.uint8).reshape(-1)
        views.append(wpin[o:o + a.nbytes].view(a.dtype).reshape(a.shape))
        o += a.nbytes
    wire = rt.WireTrace(*views, wt.inst_offsets)
    del tr, wt, cols
    setup_s = time.time() - t_setup

    def exchange():
        owned, view, tail = hl.split_device(spec, an, halo)
        info = allgather((view, tail))
        ok = all(hl.halo_ok(specs[r], info[r][0], [i[1] for i in info[:r]], cfg) for r in range(world))
        if not ok:  # the synthetic configs[1] trace has explicit stages: never expected
            raise RuntimeError("halo rejected; run halo.ShardedRun for the full-prefix fallback")
        counts = allgather(owned.n_records)
        payload = owned.alerts.view(np.uint8)
        got = cdist.gather_bytes(payload, device=cdev) if dist else [payload]
        return owned, counts, got

    for _ in range(args.warmup):
        an.run(abi.RUN_ALL)
        exchange()
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(dev)
    clocks.start()
    time.sleep(0.3)
    dev_ms, ex_ms, launches = [], [], 0
    for _ in range(args.steps):
        an.run(abi.RUN_ALL)
        dev_ms.append(an.timings()["total"])
        launches += an.launches()
        t0 = time.perf_counter()
        _, _, got = exchange()
        ex_ms.append((time.perf_counter() - t0) * 1e3)
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    clk = clocks.stop()
    # e2e: the shard's wire columns from host memory each step
    e2e = []
    for k in range(args.warmup + args.steps):
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        an.upload_wire(wire)
        an.run(abi.RUN_ALL)
        _, _, got = exchange()
        if k >= args.warmup:
            e2e.append((time.perf_counter() - t0) * 1e3)
    d_ms, x_ms, e_ms = statistics.median(dev_ms), statistics.median(ex_ms), statistics.median(e2e)
    if dist:
        d_ms = cdist.max_over_ranks(d_ms, device=cdev)
        x_ms = cdist.max_over_ranks(x_ms, device=cdev)
        e_ms = cdist.max_over_ranks(e_ms, device=cdev)
    n_alerts = sum(len(g) // abi.ALERT_DTYPE.itemsize for g in got) if got else 0
    # split_device's reads: halo + tail cycle and record rows, summary, alerts
    d2h = (2 * halo * (abi.CYCLE_DTYPE.itemsize + abi.RECORD_DTYPE.itemsize)
           + C.sizeof(abi.InstanceSummary) + n_alerts * abi.ALERT_DTYPE.itemsize)
    rt.host_free(wptr)
    line = {
        "metric": METRIC, "value": n_events / (d_ms * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": d_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64+f64",
        "data": "synthetic (simkit restatement, byte-identical to the reference generator per chunk)",
        "config": {"workload": WORKLOADS["c2"][6] + "; one instance split into cycle-range shards",
                   "events_total": n_events, "events_this_rank": int(len(loc)), "halo_cycles": halo,
                   "parallelism": f"cycle-range shards x{world} with a verified halo",
                   "l2": "inputs larger than L2; no flush needed", "setup_s": round(setup_s, 1)},
        "exchange_ms": x_ms,
        "e2e": {"value": n_events / (e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": wire_bytes,
                "d2h_bytes_per_step": d2h, "ms_per_step": e_ms,
                "input": "the shard's columnar wire format from host memory (cs_upload_wire)",
                "timer": "host wall clock: upload + cs_run + exchange + alert gather"},
        "gpu_launches": launches, "clocks": clk, "alerts_per_step": n_alerts,
    }
    if rank == 0:
        print(json.dumps(line))
    an.close()
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--c2-split", choices=["replicas", "halo"], default="replicas",
                    help="N > 1 on configs[1]: N independent instances (default) or one "
                         "instance split into cycle-range shards with a verified halo")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.workload == "c5":
        run_stream(args, rank, world, local_rank)
    elif args.workload == "c2" and args.c2_split == "halo":
        run_halo(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
