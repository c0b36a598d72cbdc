"""Small workload touching most kernels, for compute-sanitizer (memcheck /
racecheck / synccheck): analysis with mu and beta, wire upload,
batched device fit, streaming push, root-cause ranking."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2601_09258_b200 import abi, runtime as rt

tr = rt.synth_trace(700, 3, 4, n_ranks=4, fault="nvlink_saturation", onset=560, duration=80, target_rank=1)
an = rt.Analyzer(0)
an.configure(tr.names, rt.span_names_mask(tr.events, len(tr.names)), n_comm_slots=tr.n_comm)
an.upload(tr.events, [0, len(tr.events)], tr.workloads)
an.run(abi.RUN_SEGMENT)
recs = an.records(0)
train = recs[recs["cycle_index"] < 500]
x = np.stack([train["batch"].astype(float),
              (train["batch"] * (train["input_len"] + train["output_len"])).astype(float)], 1)
models, _ = rt.fit_latency_models([x, x[:300]], [train["latency_s"], train["latency_s"][:300]])
an.load_model(models[0])
an.run(abi.RUN_ALL | abi.RUN_MU)
res = an.result(0)
an.upload_wire(rt.wire_pack(tr.events, [0, len(tr.events)], tr.workloads))
an.run(abi.RUN_ALL)
recs = an.records(0)
normal = [int(c) for c in recs["cycle_index"][(recs["armed"] == 1) & (recs["flagged"] == 0)]][-100:]
abnormal = [int(c) for c in recs["cycle_index"][recs["flagged"] == 1]][:50]
if len(normal) >= 10 and len(abnormal) >= 3:
    groups = np.arange(tr.n_comm, dtype=np.int32)
    an.suspicion_rank(normal, abnormal, np.zeros(tr.n_comm, np.int32), groups, np.arange(tr.n_comm), None)
an.close()
# streaming micro-batches
an = rt.Analyzer(0)
an.configure(tr.names, rt.span_names_mask(tr.events, len(tr.names)), n_comm_slots=tr.n_comm)
an.load_model(models[0])
st = an.stream()
cut = np.linspace(0, len(tr.events), 6).astype(np.int64)
for k in range(5):
    ev = np.ascontiguousarray(tr.events[cut[k]:cut[k + 1]])
    st.push_packed(ev, np.array([0, len(ev)], np.uint64), tr.workloads if k == 0 else None)
st.close()
an.close()
# a multi-instance batch (uneven sizes, an empty instance) through the wire format
parts = [rt.synth_trace(n, 20 + i, 30 + i, n_ranks=1 + i % 3, fault="cpu_contention" if i == 1 else None,
                        onset=n - 100, duration=60, compact_names=False) for i, n in enumerate((300, 900, 150))]
names = parts[0].names
evs = [p.events for p in parts]
evs.insert(2, evs[0][:0])  # empty instance
off = np.concatenate([[0], np.cumsum([len(e) for e in evs])]).astype(np.uint64)
ev = np.concatenate(evs)
wl = np.concatenate([p.workloads for p in parts])
base = 0
for k, e in enumerate(evs):
    lo, hi = int(off[k]), int(off[k + 1])
    has = (ev["flags"][lo:hi] & abi.EV_HAS_BATCH) != 0
    ev["payload"][lo:hi][has] += np.uint64(base)
    src = [p for p in parts][k - (1 if k > 2 else 0)] if k != 2 else None
    if src is not None:
        base += len(src.workloads)
an = rt.Analyzer(0)
an.configure(names, rt.span_names_mask(ev, len(names)), n_comm_slots=max(p.n_comm for p in parts))
an.load_model(models[0])
an.upload_wire(rt.wire_pack(ev, off, wl))
an.run(abi.RUN_ALL | abi.RUN_MU)
n_cyc = sum(an.summary(i).n_cycles for i in range(len(evs)))
an.close()
# heuristic stages (forward_mode stripped, keywords off): the block-parallel
# kernel (window 32) and the sequential-window kernel (window 40); and the
# two-pass segmentation path
evh = tr.events.copy()
evh["flags"] &= np.uint16(0xFFFC)
for win in (32, 40):
    cfg = {"cycle": {"prefill_keywords": ["zz_none"], "decode_keywords": ["zz_none"], "stage_window": win}}
    an = rt.Analyzer(0)
    an.configure(tr.names, rt.span_names_mask(evh, len(tr.names)), n_comm_slots=tr.n_comm, run_config=cfg)
    an.upload(evh, [0, len(evh)], tr.workloads)
    an.run(abi.RUN_SEGMENT)
    an.close()
an = rt.Analyzer(0)
an.configure(tr.names, rt.span_names_mask(tr.events, len(tr.names)), n_comm_slots=tr.n_comm)
an.set_fused(False)
an.upload(tr.events, [0, len(tr.events)], tr.workloads)
an.load_model(models[0])
an.run(abi.RUN_ALL)
an.close()
print("sanitize workload ok:", len(tr.events), "events,", len(res.cycles), "cycles,", len(res.alerts),
      "alerts; multi-instance batch", len(ev), "events,", n_cyc, "cycles")
