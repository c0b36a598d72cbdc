"""The 16-byte wire format (cs_wire_event, include/cyclescope_b200.h).

CPU: cs_wire_pack round-trips every cs_event field exactly (decoded here in
numpy, the inverse of the device's k_wire_expand), escapes included.
GPU: a batch uploaded with cs_upload_wire analyses bit-identically to the
same batch uploaded with cs_upload."""
import numpy as np
import pytest

from paper_2601_09258_b200 import abi


def unpack(w):
    """numpy inverse of the wire encoding (mirrors k_wire_expand)."""
    off = w.inst_offsets.astype(np.int64)
    n = int(off[-1])
    block = np.empty(n, np.int64)
    b = 0
    for i in range(len(off) - 1):
        m = int(off[i + 1] - off[i])
        nb = (m + abi.WIRE_BLOCK - 1) // abi.WIRE_BLOCK
        block[off[i]:off[i + 1]] = b + np.arange(m) // abi.WIRE_BLOCK
        b += nb
    assert b == len(w.block_base)
    info = w.events["info"].astype(np.int64)
    esc = (info & abi.WIRE_ESCAPE) != 0
    ok = ~esc
    kind = (info >> 16) & 15
    flags = (info >> 24) & 0x3F
    span = ok & (kind == abi.SPAN)
    val = ok & (kind == abi.COUNTER) & ((flags & 0x20) != 0)
    pay = ok & ((flags & 0x14) != 0)
    # column positions: running counts in event order (block_cols = block starts)
    out = np.zeros(n, abi.EVENT_DTYPE)
    out["start_ts"][ok] = w.block_base[block[ok]] + w.events["t_off"][ok].astype(np.int64)
    assert span.sum() == len(w.durations) and pay.sum() == len(w.payloads) and val.sum() == len(w.values)
    assert np.array_equal(w.block_cols[:, 0], np.concatenate([[0], np.cumsum(np.bincount(block[span], minlength=b))])[:b])
    out["duration"][span] = w.durations.astype(np.int64)
    out["duration"][val] = w.values.view(np.int64)
    out["name_id"][ok] = info[ok] & 0xFFFF
    out["kind"][ok] = kind[ok]
    out["category"][ok] = (info[ok] >> 20) & 15
    out["flags"][ok] = flags[ok]
    p = w.payloads.astype(np.uint64)
    comm = (flags[pay] & 0x10) != 0
    p[comm] <<= np.uint64(32)
    out["payload"][pay] = p
    out[esc] = w.escapes[w.events["t_off"][esc]]
    return out


def _edge_events(rt):
    t = rt.synth_trace(400, 3, 4, n_ranks=4, compact_names=False)
    ev = t.events.copy()
    rng = np.random.default_rng(5)
    k = rng.choice(len(ev), 40, replace=False)
    ev["duration"][k[:10]] = (1 << 33) + np.arange(10)            # > 32-bit duration
    ev["name_id"][k[10:20]] = 70000                               # > 16-bit name
    ev["payload"][k[20:30]] |= np.uint64(1 << 40)                 # high payload bits
    sp = np.nonzero(ev["kind"] == 0)[0]
    ev["duration"][sp[:5]] = -3                                   # negative span duration
    # a gap > 4.29 s inside one block
    ev["start_ts"][2000:] += (1 << 33)
    return t, ev


def test_wire_roundtrip_simkit(rt):
    t = rt.synth_trace(3000, 1, 2, n_ranks=8, fault="nvlink_saturation", onset=2000,
                       duration=150, target_rank=3, compact_names=False)
    w = rt.wire_pack(t.events, [0, len(t.events)])
    assert w.events.nbytes == 8 * len(t.events)
    assert len(w.escapes) == 0
    assert w.nbytes < 16 * len(t.events)
    assert np.array_equal(unpack(w).view(np.uint8), t.events.view(np.uint8))


def test_wire_roundtrip_escapes_and_instances(rt):
    t, ev = _edge_events(rt)
    cut = [0, 1500, 1500, len(ev)]  # includes an empty instance
    w = rt.wire_pack(ev, cut, n_threads=3)
    assert len(w.escapes) > 20
    assert np.array_equal(unpack(w).view(np.uint8), ev.view(np.uint8))


@pytest.mark.gpu
def test_upload_wire_matches_upload(rt):
    traces = [rt.synth_trace(2500, 11 + i, 12 + i, n_ranks=4, fault="gpu_clock_lock", onset=2000,
                             duration=150, compact_names=False) for i in range(2)]
    evs = [t.events for t in traces]
    off = np.concatenate([[0], np.cumsum([len(e) for e in evs])]).astype(np.uint64)
    ev = np.concatenate(evs)
    has = (ev["flags"] & abi.EV_HAS_BATCH) != 0
    second = np.zeros(len(ev), bool)
    second[int(off[1]):] = True
    sel = has & second
    ev["payload"][sel] = ev["payload"][sel] + np.uint64(len(traces[0].workloads))
    wl = np.concatenate([t.workloads for t in traces])
    # a few escapes on span durations inside cycles
    w = rt.wire_pack(ev, off)
    names = traces[0].names
    out = []
    for kind in ("upload", "wire"):
        an = rt.Analyzer(0)
        an.configure(names, rt.span_names_mask(ev, len(names)), n_comm_slots=4)
        if kind == "upload":
            an.upload(ev, off, wl)
        else:
            an.upload_wire(w, wl)
        an.run(abi.RUN_SEGMENT)
        recs = an.records(0)
        tr = recs[recs["cycle_index"] < 1500]
        x = np.stack([tr["batch"].astype(float),
                      (tr["batch"] * (tr["input_len"] + tr["output_len"])).astype(float)], 1)
        an.load_model(rt.fit_latency_model(x, tr["latency_s"]))
        an.run(abi.RUN_ALL)
        out.append([an.result(i) for i in range(2)])
        an.close()
    for a, b in zip(*out):
        assert a.cycles.tobytes() == b.cycles.tobytes()
        assert a.beta.tobytes() == b.beta.tobytes()
        assert a.records.tobytes() == b.records.tobytes()
        assert a.alerts.tobytes() == b.alerts.tobytes()
