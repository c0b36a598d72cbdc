"""GPU: single-instance sharding with a verified halo on the
device path.  Every shard runs through cs_upload + cs_run on one B200 (the
in-process form of what bench.py runs one shard per GPU); the merged result
must equal the whole-trace device run and the C oracle, bit for bit."""
import numpy as np
import pytest

from oracle import csoracle
from paper_2601_09258_b200 import abi, halo as hl, runtime as rt

pytestmark = pytest.mark.gpu

RUN_CONFIG = {"cycle": {"anchor_hint": "run_batch"}}


def _trace(n_cycles, seed, heuristic=False, n_ranks=4):
    tr = rt.synth_trace(n_cycles, seed, seed + 1, fault="cpu_contention", onset=n_cycles * 2 // 3,
                        duration=200, n_ranks=n_ranks, compact_names=False)
    ev, names = tr.events.copy(), list(tr.names)
    if heuristic:
        ev["flags"] &= np.uint32(0xfffffffc)
        names = [n.replace("prefill", "pf").replace("decode", "dc") for n in names]
    return ev, names, tr.workloads, tr.n_comm, rt.span_names_mask(ev, len(names))


def _setup(ev, names, wl, n_comm, span):
    an = rt.Analyzer(0)
    an.configure(names, span, n_comm_slots=n_comm, run_config=RUN_CONFIG)
    an.upload(ev, [0, len(ev)], wl)
    an.run(abi.RUN_SEGMENT)
    r = an.records(0)
    r = r[r["cycle_index"] < 1500]
    x = np.stack([r["batch"].astype(float), (r["batch"] * (r["input_len"] + r["output_len"])).astype(float)], 1)
    model = rt.fit_latency_model(x, r["latency_s"])
    an.load_model(model)
    return an, model


def _as_dict(an):
    r = an.result(0)
    s = r.summary
    return dict(cycles=r.cycles, records=r.records, alerts=r.alerts, components=r.components,
                beta_totals=r.beta_totals, beta=r.beta, coll_beta=r.coll_beta, coll_present=r.coll_present,
                status=s.status, first_bad_record=s.first_bad_record)


def _device_at(an, ev, wl):
    def at(spec):
        an.upload(np.ascontiguousarray(ev[spec.lo:spec.hi]), [0, spec.hi - spec.lo], wl)
        an.run(abi.RUN_ALL)
        return _as_dict(an)
    return at


def _equal(a, b):
    assert np.array_equal(a["cycles"], b["cycles"])
    for k in ("components", "beta_totals", "beta", "coll_beta", "coll_present"):
        x, y = np.asarray(a[k]).reshape(-1), np.asarray(b[k]).reshape(-1)
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8)), k
    assert np.array_equal(a["records"].view(np.uint8), b["records"].view(np.uint8))
    assert np.array_equal(a["alerts"].view(np.uint8), b["alerts"].view(np.uint8))


CFG = hl.CheckConfig(stage_window=32, window=10, warmup=100)


@pytest.mark.parametrize("world,heuristic", [(2, False), (4, False), (8, False), (4, True)])
def test_device_shards_equal_whole_trace(world, heuristic):
    ev, names, wl, n_comm, span = _trace(12000, 21 + world, heuristic=heuristic)
    an, model = _setup(ev, names, wl, n_comm, span)
    an.upload(ev, [0, len(ev)], wl)
    an.run(abi.RUN_ALL)
    whole = _as_dict(an)
    assert len(whole["alerts"]) >= 1
    got, specs, reruns = hl.run_all_in_process(ev, names.index("run_batch"), world, CFG,
                                               _device_at(an, ev, wl), halo=512)
    assert reruns == []
    _equal(whole, got)
    oracle = csoracle.analyze(ev, names, wl, n_comm, RUN_CONFIG, model.to_json(), span=span)
    _equal(oracle, got)
    an.close()


def test_split_device_reads_only_halo_and_tail():
    ev, names, wl, n_comm, span = _trace(9000, 5)
    an, _ = _setup(ev, names, wl, n_comm, span)
    an.upload(ev, [0, len(ev)], wl)
    an.run(abi.RUN_ALL)
    whole = _as_dict(an)
    # ranged getters equal slices of the whole tables
    assert np.array_equal(an.cycle_range(100, 50), whole["cycles"][100:150])
    nr = len(whole["records"])
    assert np.array_equal(an.record_range(nr - 40, 40).view(np.uint8), whole["records"][-40:].view(np.uint8))
    al = whole["records"]["alert"].astype(bool)
    k = int(np.flatnonzero(al)[0])
    assert np.array_equal(an.record_range(k, 5).view(np.uint8), whole["records"][k:k + 5].view(np.uint8))
    with pytest.raises(rt.EngineError):
        an.record_range(nr - 1, 2)
    # the light split: alerts + counts only, merged = the whole-trace alerts
    _, specs = hl.plan(ev, names.index("run_batch"), 3, 400)
    parts = []
    for s in specs:
        an.upload(np.ascontiguousarray(ev[s.lo:s.hi]), [0, s.hi - s.lo], wl)
        an.run(abi.RUN_ALL)
        parts.append(hl.split_device(s, an, 400))
    for r in range(1, 3):
        assert hl.halo_ok(specs[r], parts[r][1], [p[2] for p in parts[:r]], CFG)
    alerts, status, first_bad = hl.merge_alerts([p[0] for p in parts])
    assert np.array_equal(alerts.view(np.uint8), whole["alerts"].view(np.uint8))
    assert status == 0 and first_bad == (1 << 64) - 1
    an.close()
