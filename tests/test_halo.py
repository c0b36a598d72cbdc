"""CPU: single-instance sharding with a verified halo (SURVEY §8e, configs[1]),
paper_2601_09258_b200/halo.py.  Every shard is analysed by the C oracle on
its event range; the merged result must equal the whole-trace oracle run
exactly (cycles, components, beta, records bit for bit, alerts) — for
explicit-stage traces (halo accepted) and for heuristic-stage traces where a
short halo is rejected and the shard re-runs from the start of the trace."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import csoracle
from paper_2601_09258_b200 import abi, halo as hl, runtime as rt

RUN_CONFIG = {"cycle": {"anchor_hint": "run_batch"}}


def _trace(n_cycles=3000, seed=7, heuristic=False, n_ranks=2):
    tr = rt.synth_trace(n_cycles, seed, seed + 1, fault="cpu_contention", onset=n_cycles * 2 // 3,
                        duration=150, n_ranks=n_ranks, compact_names=False)
    ev, names = tr.events.copy(), list(tr.names)
    if heuristic:
        # no forward-mode flags and no stage keywords: stages from the
        # duration / gap heuristic (cycles.cpp:204-250)
        ev["flags"] &= np.uint32(0xfffffffc)  # forward-mode bits (trace.hpp flags 0..1)
        names = [n.replace("prefill", "pf").replace("decode", "dc") for n in names]
    span = rt.span_names_mask(ev, len(names))
    return ev, names, tr.workloads, tr.n_comm, span


def _model(ev, names, wl, n_comm, span):
    base = csoracle.analyze(ev, names, wl, n_comm, RUN_CONFIG, None, span=span)
    r = base["records"]
    r = r[r["cycle_index"] < 1200]
    x = np.stack([r["batch"].astype(float), (r["batch"] * (r["input_len"] + r["output_len"])).astype(float)], 1)
    return rt.fit_latency_model(x, r["latency_s"]).to_json()


def _check_equal(whole, got):
    assert np.array_equal(whole["cycles"], got["cycles"])
    for k in ("components", "beta_totals", "beta", "coll_beta", "coll_present"):
        a, b = np.asarray(whole[k]).reshape(-1), np.asarray(got[k]).reshape(-1)
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), k
    assert np.array_equal(whole["records"].view(np.uint8), got["records"].view(np.uint8))
    assert np.array_equal(whole["alerts"].view(np.uint8), got["alerts"].view(np.uint8))
    assert whole["status"] == got["status"]


def _cfg(include_prefill=False):
    return hl.CheckConfig(stage_window=32, include_prefill=include_prefill, window=10, warmup=100)


def _oracle_at(ev, names, wl, n_comm, span, model):
    return lambda s: csoracle.analyze(ev[s.lo:s.hi], names, wl, n_comm, RUN_CONFIG, model, span=span)


@pytest.mark.parametrize("world", [2, 3, 5, 8])
def test_explicit_stages_halo_accepted(world):
    ev, names, wl, n_comm, span = _trace()
    model = _model(ev, names, wl, n_comm, span)
    whole = csoracle.analyze(ev, names, wl, n_comm, RUN_CONFIG, model, span=span)
    assert len(whole["alerts"]) >= 1
    anchor = names.index("run_batch")
    got, specs, reruns = hl.run_all_in_process(ev, anchor, world, _cfg(),
                                               _oracle_at(ev, names, wl, n_comm, span, model), halo=256)
    assert reruns == []
    assert all(not s.full_prefix for s in specs[1:])
    _check_equal(whole, got)


def test_alert_episode_straddles_a_boundary():
    # put a shard boundary inside the fault window: the episode opened by the
    # previous shard must not re-alert in the next one
    ev, names, wl, n_comm, span = _trace(n_cycles=2400, seed=11)
    model = _model(ev, names, wl, n_comm, span)
    whole = csoracle.analyze(ev, names, wl, n_comm, RUN_CONFIG, model, span=span)
    rec = whole["records"]
    flagged = np.flatnonzero(rec["flagged"] == 1)
    assert len(flagged) > 3
    anchor = names.index("run_batch")
    pos = hl.anchor_positions(ev, anchor)
    c_mid = int(rec["cycle_index"][flagged[len(flagged) // 2]])
    specs = [hl.shard_spec(ev, pos, 0, 0, c_mid, 256), hl.shard_spec(ev, pos, 1, c_mid, len(pos) - 1, 256)]
    at = _oracle_at(ev, names, wl, n_comm, span, model)
    parts = [hl.split_local(s, at(s), 256) for s in specs]
    assert hl.halo_ok(specs[1], parts[1][1], [parts[0][2]], _cfg())
    _check_equal(whole, hl.merge([p[0] for p in parts]))


def test_heuristic_stages_short_halo_rejected_then_exact():
    ev, names, wl, n_comm, span = _trace(n_cycles=2500, seed=3, heuristic=True)
    model = _model(ev, names, wl, n_comm, span)
    whole = csoracle.analyze(ev, names, wl, n_comm, RUN_CONFIG, model, span=span)
    st = whole["cycles"]["stage"]
    assert (st == abi.STAGE_PREFILL).any() and (st == abi.STAGE_DECODE).any()
    anchor = names.index("run_batch")
    at = _oracle_at(ev, names, wl, n_comm, span, model)
    # 16 cycles cannot rebuild a 32-entry stage ring: every boundary re-runs
    got, specs, reruns = hl.run_all_in_process(ev, anchor, 4, _cfg(), at, halo=16)
    assert reruns == [1, 2, 3]
    _check_equal(whole, got)
    # a long halo rebuilds the rings and is accepted
    got, specs, reruns = hl.run_all_in_process(ev, anchor, 4, _cfg(), at, halo=400)
    assert reruns == []
    _check_equal(whole, got)


def test_no_detector_and_include_prefill():
    ev, names, wl, n_comm, span = _trace(n_cycles=1500, seed=5)
    rc = {"cycle": {"anchor_hint": "run_batch"}, "pipeline": {"include_prefill": True}}
    whole = csoracle.analyze(ev, names, wl, n_comm, rc, None, span=span)
    anchor = names.index("run_batch")
    cfg = hl.CheckConfig(include_prefill=True, detector=False)
    got, _, reruns = hl.run_all_in_process(
        ev, anchor, 3, cfg, lambda s: csoracle.analyze(ev[s.lo:s.hi], names, wl, n_comm, rc, None, span=span),
        halo=128)
    assert reruns == []
    _check_equal(whole, got)


def test_plan_covers_every_cycle_once():
    ev, names, *_ = _trace(n_cycles=800, seed=9)
    anchor = names.index("run_batch")
    pos, specs = hl.plan(ev, anchor, 8, halo=50)
    assert specs[0].c0 == 0 and specs[-1].c1 == len(pos) - 1
    for a, b in zip(specs, specs[1:]):
        assert a.c1 == b.c0
    for s in specs:
        assert s.lo <= (pos[s.c0] if s.c0 < len(pos) else len(ev)) and s.hi <= len(ev)
        assert s.full_prefix or s.halo >= 50


# ---------------------------------------------------------------- gloo, world 2
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, heuristic, halo):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ev, names, wl, n_comm, span = _trace(n_cycles=2000, seed=13, heuristic=heuristic)
        model = _model(ev, names, wl, n_comm, span)

        def allgather(obj):
            out = [None] * world
            dist.all_gather_object(out, obj)
            return out

        run = hl.ShardedRun(ev, names.index("run_batch"), world, rank, _cfg(), halo=halo)
        owned, specs = run.run(_oracle_at(ev, names, wl, n_comm, span, model), allgather)
        parts = allgather(owned)
        if rank == 0:
            whole = csoracle.analyze(ev, names, wl, n_comm, RUN_CONFIG, model, span=span)
            _check_equal(whole, hl.merge(parts))
            q.put(("ok", len(whole["alerts"]), allgather(run.reruns)))
        else:
            allgather(run.reruns)
    except Exception as e:  # surface the failure to the parent
        q.put(("error", repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("heuristic,halo,want_reruns", [(False, 200, [[], []]), (True, 16, [[], [1]])],
                         ids=["accepted", "rerun"])
def test_sharded_run_world2_gloo(heuristic, halo, want_reruns):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, heuristic, halo)) for r in range(2)]
    for p in procs:
        p.start()
    status, n_alerts, reruns = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert status == "ok", n_alerts
    assert reruns == want_reruns
    assert all(p.exitcode == 0 for p in procs)
