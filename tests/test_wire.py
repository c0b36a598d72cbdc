"""The columnar wire format (cs_wire_batch, include/cyclescope_b200.h).

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
    bstart = []
    b = 0
    for i in range(len(off) - 1):
        m = int(off[i + 1] - off[i])
        nb = (m + abi.WIRE_BLOCK - 1) // abi.WIRE_BLOCK
        block[off[i]:off[i + 1]] = b + np.arange(m) // abi.WIRE_BLOCK
        bstart += [int(off[i]) + k * abi.WIRE_BLOCK for k in range(nb)]
        b += nb
    assert b == len(w.blocks) and len(w.dict) <= abi.WIRE_MAX_DICT
    bstart = np.asarray(bstart, np.int64)
    code = (w.codes & 0x7F).astype(np.int64)
    esc = code == abi.WIRE_ESCAPE
    ok = ~esc
    longdt = ok & ((w.codes & abi.WIRE_LONG_DT) != 0)
    info = np.zeros(n, np.int64)
    info[ok] = w.dict[code[ok]].astype(np.int64)
    kind = (info >> 16) & 15
    flags = (info >> 24) & 0x3F
    wide = (info & abi.WIRE_WIDE) != 0
    span = ok & (kind == abi.SPAN)
    val = ok & (kind == abi.COUNTER) & ((flags & 0x20) != 0)
    pay = ok & ((flags & 0x14) != 0)
    assert span.sum() == len(w.dur_lo) and val.sum() == len(w.values)
    assert (pay & ~wide).sum() == len(w.pay8) and (pay & wide).sum() == len(w.pay16)
    assert esc.sum() == len(w.escapes) and longdt.sum() == len(w.dt_hi)
    for col, mask in (("dur", span), ("pay8", pay & ~wide), ("pay16", pay & wide), ("val", val),
                      ("dt_hi", longdt), ("esc", esc)):
        starts = np.concatenate([[0], np.cumsum(np.bincount(block[mask], minlength=b))])[:b]
        assert np.array_equal(w.blocks[col].astype(np.int64), starts), col
    # start_ts: per-block prefix sums of the deltas, restarted at escaped records
    dt = w.dt_lo.astype(np.int64)
    dt[longdt] |= w.dt_hi.astype(np.int64) << 16
    dt[esc] = 0
    cs = np.cumsum(dt)
    cs -= (cs - dt)[bstart][block]                 # inclusive sum within the block
    out = np.zeros(n, abi.EVENT_DTYPE)
    out[esc] = w.escapes
    last = np.maximum.accumulate(np.where(esc, np.arange(n), -1))
    restarted = last >= bstart[block]
    base = w.blocks["base_ts"][block].astype(np.int64)
    base[restarted] = out["start_ts"][last[restarted]] - cs[last[restarted]]
    out["start_ts"][ok] = (base + cs)[ok]
    out["duration"][span] = w.dur_lo.astype(np.int64) | (w.dur_hi.astype(np.int64) << 16)
    out["duration"][val] = w.values.view(np.int64)
    out["name_id"][ok] = info[ok] & 0xFFFF
    out["kind"][ok] = kind[ok]
    out["category"][ok] = (info[ok] >> 20) & 15
    out["flags"][ok] = flags[ok]
    p = np.zeros(n, np.uint64)
    p[pay & ~wide] = w.pay8
    p[pay & wide] = w.pay16
    comm = pay & ((flags & 0x10) != 0)
    batch = pay & ~comm
    p[comm] <<= np.uint64(32)
    p[batch] += w.blocks["batch_base"][block[batch]].astype(np.uint64)
    out["payload"][pay] = p[pay]
    return out


def unpack_workloads(w):
    x = w.workloads32.astype(np.int64)
    x[w.workloads32 == 0xFFFFFFFF] = np.iinfo(np.int64).min
    out = np.zeros(len(x), abi.WORKLOAD_DTYPE)
    out["batch"], out["input_len"], out["output_len"] = x[:, 0], x[:, 1], x[:, 2]
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
    # a gap > 4.29 s inside one block, and one of 2^24 ns exactly (escape)
    ev["start_ts"][2000:] += (1 << 33)
    ev["start_ts"][3001:] += (1 << 24) - int(ev["start_ts"][3001] - ev["start_ts"][3000])
    ev["duration"][sp[5:9]] = [(1 << 24) - 1, 1 << 24, 1 << 24 + 5, 0]  # 24-bit limit
    return t, ev


def test_wire_roundtrip_simkit(rt):
    t = rt.synth_trace(3000, 1, 2, n_ranks=8, fault="nvlink_saturation", onset=2000,
                       duration=150, target_rank=3, compact_names=False)
    w = rt.wire_pack(t.events, [0, len(t.events)], t.workloads)
    assert w.codes.nbytes + w.dt_lo.nbytes == 3 * len(t.events)
    assert unpack_workloads(w).tobytes() == t.workloads.tobytes()
    assert len(w.escapes) < 1e-3 * len(t.events)  # run_batch spans >= 16.8 ms under the fault
    assert w.nbytes < 9 * len(t.events)
    assert np.array_equal(unpack(w).view(np.uint8), t.events.view(np.uint8))


def test_wire_roundtrip_escapes_and_instances(rt):
    t, ev = _edge_events(rt)
    cut = [0, 1500, 1500, len(ev)]  # includes an empty instance
    w = rt.wire_pack(ev, cut, n_threads=3)
    assert len(w.escapes) > 20
    assert np.array_equal(unpack(w).view(np.uint8), ev.view(np.uint8))


def test_wire_dictionary_overflow_and_payload_range(rt):
    """More distinct info words than the dictionary holds (the rarest ones
    escape), batch payloads below the block's base or 2^16 above it."""
    t = rt.synth_trace(600, 5, 6, n_ranks=2, compact_names=False)
    ev = t.events.copy()
    inst = np.nonzero(ev["kind"] == abi.INSTANT)[0]
    ev["name_id"][inst[:400]] = 1000 + np.arange(400) % 300        # 300 extra info words
    bat = np.nonzero((ev["flags"] & abi.EV_HAS_BATCH) != 0)[0]
    ev["payload"][bat[3]] = 0                                       # below the block's base
    ev["payload"][bat[7]] = ev["payload"][bat[6]] + np.uint64(70000)
    w = rt.wire_pack(ev, [0, len(ev)], n_threads=2)
    assert len(w.dict) == abi.WIRE_MAX_DICT
    assert len(w.escapes) >= 300 - abi.WIRE_MAX_DICT  # the rarest words escape
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
    # escapes inside cycles: span durations of 2^24 ns and more, a 2^24 ns gap
    sp = np.nonzero((ev["kind"] == abi.SPAN) & second)[0]
    ev["duration"][sp[100:140]] += np.int64(1 << 24)
    ev["start_ts"][sp[300]:int(off[2])] += np.int64(1 << 24)
    w = rt.wire_pack(ev, off)
    w32 = rt.wire_pack(ev, off, wl)  # the workload table inside the wire batch
    assert w32.workloads32 is not None
    assert len(w.escapes) >= 40
    names = traces[0].names
    out = []
    for kind in ("upload", "wire", "wire32"):
        an = rt.Analyzer(0)
        an.configure(names, rt.span_names_mask(ev, len(names)), n_comm_slots=4)
        if kind == "upload":
            an.upload(ev, off, wl)
        else:
            an.upload_wire(w, wl) if kind == "wire" else an.upload_wire(w32)
        an.run(abi.RUN_SEGMENT)
        recs = an.records(0)
        tr = recs[recs["cycle_index"] < 1500]
        x = np.stack([tr["batch"].astype(float),
                      (tr["batch"] * (tr["input_len"] + tr["output_len"])).astype(float)], 1)
        an.load_model(rt.fit_latency_model(x, tr["latency_s"]))
        an.run(abi.RUN_ALL)
        out.append([an.result(i) for i in range(2)])
        an.close()
    for a, b in list(zip(out[0], out[1])) + list(zip(out[0], out[2])):
        assert a.cycles.tobytes() == b.cycles.tobytes()
        assert a.beta.tobytes() == b.beta.tobytes()
        assert a.records.tobytes() == b.records.tobytes()
        assert a.alerts.tobytes() == b.alerts.tobytes()
