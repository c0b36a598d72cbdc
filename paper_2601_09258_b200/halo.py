"""Single-instance sharding with a verified halo (SURVEY §8e, configs[1]).

One monitored instance is split into contiguous cycle ranges, one per rank,
and every rank runs the ordinary whole-batch analysis (cs_run) on its range
prefixed by a halo of H preceding cycles.  Cycles are anchor-to-anchor event
ranges (segment_cycles, cycles.cpp:150-175), so a range that starts at
`lower_index(anchor ts)` and ends at the closing anchor reproduces every
cycle's events, components, beta and workload exactly.  What does not
survive a split is the sequential state the reference threads through the
whole trace:

  - the stage heuristic's rings: the last `stage_window` durations and gaps
    of non-prefill cycles and the previous anchor end (cycles.cpp:204-250);
  - the detector's last W-1 residuals, the warm-up count, `in_episode` and
    the record / episode numbering (detector.cpp:34-92, monitor loop).

The halo run starts from an empty state and rebuilds it over the H halo
cycles.  That state equals the true one at the shard boundary when, over the
halo cycles after the first (whose event range may be cut):
  (1) on a suffix of the halo holding at least stage_window + 1 non-prefill
      cycles, which cycles are prefill and the workload statuses equal the
      previous shard's (true) ones — the rings then hold the same durations
      and gaps (unknown and decode stages both enter them and give the same
      is_prefill feature);
  (2) the last W records of that suffix (cycle, residual bits) equal the
      true ones, the halo holds >= warmup records, and the last record's
      armed / flagged bits equal the true ones (in_episode after a record is
      exactly `armed and flagged`).
Record, cycle and episode numbers are then rebased with exclusive prefix
counts.  A boundary that fails the check is re-run with the halo reaching
back to the start of the trace, which is exact by construction; checks are
made left to right against the predecessor's accepted outputs, so the merged
result is always identical to the whole-trace run.

The exchange is one all-gather of per-rank tails (a few KB) plus the final
alert gather; the analysis itself is unchanged.  Host plumbing only — the
per-shard analysis is a callback (the device Analyzer in bench.py and the
GPU tests, the C oracle in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import abi

PER_CYCLE = ("components", "beta_totals", "beta", "coll_beta", "coll_present", "mu", "mu_has")


def anchor_positions(events: np.ndarray, anchor: int) -> np.ndarray:
    """Event indices of the anchor's span events (segment_cycles' `pos`)."""
    return np.flatnonzero((events["kind"] == abi.SPAN) & (events["name_id"] == anchor)).astype(np.int64)


@dataclass
class ShardSpec:
    rank: int
    c0: int            # first owned global cycle
    c1: int            # one past the last owned global cycle
    lo: int            # local event range [lo, hi) in the global array
    hi: int
    a_lo: int          # global cycle of the first local cycle
    full_prefix: bool  # halo reaches the start of the trace: exact by construction

    @property
    def halo(self) -> int:
        return self.c0 - self.a_lo


def _lower_index(ts: np.ndarray, t: int) -> int:
    return int(np.searchsorted(ts, t, side="left"))


def shard_spec(events: np.ndarray, pos: np.ndarray, rank: int, c0: int, c1: int, halo: int | None) -> ShardSpec:
    """Local event range for owned cycles [c0, c1) with `halo` preceding
    cycles (None: from the start of the trace)."""
    n, na = len(events), len(pos)
    ts = events["start_ts"]
    if halo is None or c0 - halo <= 0:
        lo, a_lo, full = 0, 0, True
    else:
        lo = _lower_index(ts, int(ts[pos[c0 - halo]]))
        a_lo = int(np.searchsorted(pos, lo, side="left"))
        full = False
    hi = n if c1 >= na - 1 else int(pos[c1]) + 1
    return ShardSpec(rank, c0, c1, lo, hi, a_lo, full)


def plan(events: np.ndarray, anchor: int, world: int, halo: int = 1024):
    """Owned cycle ranges balanced by event count, one per rank."""
    pos = anchor_positions(events, anchor)
    na = len(pos)
    n_cyc = max(0, na - 1)
    cuts = [0]
    for r in range(1, world):
        c = int(np.searchsorted(pos, len(events) * r // world, side="left")) if n_cyc else 0
        cuts.append(min(max(c, cuts[-1]), n_cyc))
    cuts.append(n_cyc)
    return pos, [shard_spec(events, pos, r, cuts[r], cuts[r + 1], halo) for r in range(world)]


def _rows(arr, nc):
    if arr is None:
        return None
    a = np.asarray(arr)
    if nc == 0:
        return a.reshape(0, -1) if a.ndim == 2 else a.reshape(0, 0)
    return a.reshape(nc, -1)


@dataclass
class Owned:
    """One shard's owned outputs, rebased to global numbering except for the
    record / episode offsets (applied in merge)."""
    cycles: np.ndarray
    per_cycle: dict
    records: np.ndarray
    alerts: np.ndarray
    status: int = 0
    first_bad_record: int = -1  # local owned record index, -1: none


@dataclass
class Tail:
    """What a neighbour needs to check its halo against: per cycle (global
    index order) stage and workload status; records (global cycle index,
    residual bits, armed, flagged)."""
    c_first: int
    stage: np.ndarray
    wl_status: np.ndarray
    rec_cycle: np.ndarray
    rec_resid: np.ndarray
    rec_armed: np.ndarray
    rec_flagged: np.ndarray
    n_halo_records: int = 0  # halo views only: records in all local halo cycles


def _tail_of(cycles, records, c_first_local, c_end_local, a_lo) -> Tail:
    cyc = cycles[c_first_local:c_end_local]
    sel = (records["cycle_index"] >= c_first_local) & (records["cycle_index"] < c_end_local)
    r = records[sel]
    return Tail(c_first_local + a_lo, cyc["stage"].copy(), cyc["workload_status"].copy(),
                r["cycle_index"].astype(np.int64) + a_lo, r["residual"].view(np.uint64).copy(),
                r["armed"].copy(), r["flagged"].copy())


def split_local(spec: ShardSpec, res: dict, tail_cycles: int):
    """Split one shard's local result into its owned part, the halo view and
    the tail it publishes.  `res`: cycles / records / alerts / per-cycle rows
    / status / first_bad_record of the run on events[lo:hi]."""
    cycles, records, alerts = res["cycles"], res["records"], res["alerts"]
    nc = len(cycles)
    h, m = spec.halo, spec.c1 - spec.c0
    if nc < h + m:
        raise RuntimeError(f"shard {spec.rank}: {nc} local cycles, expected >= {h + m}")
    own_c = cycles[h:h + m].copy()
    own_c["index"] += np.uint64(spec.a_lo)
    for f in ("anchor_pos", "first_event", "last_event"):
        own_c[f] += np.uint64(spec.lo)
    per = {}
    for k in PER_CYCLE:
        rows = _rows(res.get(k), nc)
        per[k] = None if rows is None else rows[h:h + m].copy()
    rc = records["cycle_index"]
    n_halo_rec = int(np.count_nonzero(rc < h))
    own_sel = (rc >= h) & (rc < h + m)
    own_r = records[own_sel].copy()
    own_r["cycle_index"] += np.uint64(spec.a_lo)
    halo_alerts = int(np.count_nonzero(alerts["record_index"] < n_halo_rec)) if len(alerts) else 0
    own_sel_a = (alerts["record_index"] >= n_halo_rec) & (alerts["cycle"] < h + m) if len(alerts) else np.zeros(0, bool)
    own_a = alerts[own_sel_a].copy()
    own_a["cycle"] += np.uint64(spec.a_lo)
    own_a["record_index"] -= np.uint64(n_halo_rec)
    own_a["episode_id"] -= np.uint64(halo_alerts)
    al = own_r["alert"].astype(bool)
    own_r["episode_id"][al] -= np.uint64(halo_alerts)
    fb = int(res.get("first_bad_record", -1))
    status = int(res.get("status", 0))
    if fb >= 0 and fb != (1 << 64) - 1:
        fb = fb - n_halo_rec
    else:
        fb = -1
    owned = Owned(own_c, per, own_r, own_a, status, fb)
    view = _tail_of(cycles, records, 0, h, spec.a_lo)
    view.n_halo_records = n_halo_rec
    t0 = max(h, h + m - tail_cycles)
    tail = _tail_of(cycles, records, t0, h + m, spec.a_lo)
    return owned, view, tail


def _tail(c_first, cyc, rec, a_lo) -> Tail:
    return Tail(c_first, cyc["stage"].copy(), cyc["workload_status"].copy(),
                rec["cycle_index"].astype(np.int64) + a_lo, rec["residual"].view(np.uint64).copy(),
                rec["armed"].copy(), rec["flagged"].copy())


@dataclass
class OwnedAlerts:
    """A shard's owned alerts (cycle rebased; record / episode offsets
    applied by merge_alerts) and record count, without its full tables."""
    alerts: np.ndarray
    n_records: int
    status: int = 0
    first_bad_record: int = -1


def split_device(spec: ShardSpec, an, tail_cycles: int, inst: int = 0, detect: bool = True):
    """split_local for a shard analysed by the device Analyzer `an`, reading
    only the halo rows, the tail rows and the alerts (cs_get_cycle_range /
    cs_get_record_range): returns (OwnedAlerts, halo view, tail)."""
    sm = an.summary(inst)
    nc, nr = int(sm.n_cycles), int(sm.n_records)
    h, m = spec.halo, spec.c1 - spec.c0
    if nc < h + m:
        raise RuntimeError(f"shard {spec.rank}: {nc} local cycles, expected >= {h + m}")
    hc = an.cycle_range(0, h, inst)
    hr = an.record_range(0, min(h, nr), inst)  # at most one record per cycle
    hr = hr[hr["cycle_index"] < h]
    n_halo_rec = len(hr)
    view = _tail(spec.a_lo, hc, hr, spec.a_lo)
    view.n_halo_records = n_halo_rec
    t0 = max(h, h + m - tail_cycles)
    tc = an.cycle_range(t0, h + m - t0, inst)
    k = min(h + m - t0, nr - n_halo_rec)
    tr = an.record_range(nr - k, k, inst)
    tr = tr[tr["cycle_index"] >= t0]
    tail = _tail(t0 + spec.a_lo, tc, tr, spec.a_lo)
    alerts = an.alerts(inst) if detect else np.zeros(0, abi.ALERT_DTYPE)
    halo_alerts = int(np.count_nonzero(alerts["record_index"] < n_halo_rec))
    a = alerts[alerts["record_index"] >= n_halo_rec].copy()
    a["cycle"] += np.uint64(spec.a_lo)
    a["record_index"] -= np.uint64(n_halo_rec)
    a["episode_id"] -= np.uint64(halo_alerts)
    fb = int(sm.first_bad_record)
    fb = fb - n_halo_rec if fb != (1 << 64) - 1 and fb >= n_halo_rec else -1
    return OwnedAlerts(a, nr - n_halo_rec, int(sm.status), fb), view, tail


def merge_alerts(owned: list):
    """merge() for OwnedAlerts: the whole-trace alert list, its status and
    first bad record (UINT64_MAX: none)."""
    out, rec_off = [], 0
    for o in owned:
        a = o.alerts.copy()
        a["record_index"] += np.uint64(rec_off)
        a["episode_id"] = np.arange(len(a), dtype=np.uint64) + np.uint64(sum(len(x) for x in out))
        out.append(a)
        if o.first_bad_record >= 0:
            return np.concatenate(out), o.status, rec_off + o.first_bad_record
        rec_off += o.n_records
    return (np.concatenate(out) if out else np.zeros(0, abi.ALERT_DTYPE)), 0, (1 << 64) - 1


@dataclass
class CheckConfig:
    stage_window: int = 32
    include_prefill: bool = False
    window: int = 10
    warmup: int = 100
    detector: bool = True


def halo_ok(spec: ShardSpec, view: Tail, truth: list, cfg: CheckConfig) -> bool:
    """(1)-(2) of the module docstring for shard `spec` whose halo outputs are
    `view`, against the accepted tails `truth` of earlier shards."""
    if spec.full_prefix or spec.halo == 0:
        return True
    lo_c, hi_c = spec.a_lo + 1, spec.c0  # halo cycles after the first
    st = {f: [] for f in ("stage", "wl", "rc", "rr", "ra", "rf")}
    covered = lo_c
    for t in truth:
        a = max(lo_c, t.c_first)
        b = min(hi_c, t.c_first + len(t.stage))
        if a >= b:
            continue
        if a != covered:
            return False  # gap in the published tails
        st["stage"].append(t.stage[a - t.c_first:b - t.c_first])
        st["wl"].append(t.wl_status[a - t.c_first:b - t.c_first])
        sel = (t.rec_cycle >= a) & (t.rec_cycle < b)
        st["rc"].append(t.rec_cycle[sel])
        st["rr"].append(t.rec_resid[sel])
        st["ra"].append(t.rec_armed[sel])
        st["rf"].append(t.rec_flagged[sel])
        covered = b
    if covered != hi_c:
        return False
    cat = {k: (np.concatenate(v) if v else np.zeros(0)) for k, v in st.items()}
    k0 = lo_c - view.c_first
    # the rings hold the last stage_window non-prefill cycles: what must agree
    # is which cycles are prefill (unknown and decode both enter the rings and
    # give the same is_prefill feature) over a suffix holding at least
    # stage_window + 1 of them, and the workload statuses there
    v_pf = view.stage[k0:] == abi.STAGE_PREFILL
    t_pf = cat["stage"] == abi.STAGE_PREFILL
    same = (v_pf == t_pf) & (view.wl_status[k0:] == cat["wl"])
    bad = np.flatnonzero(~same)
    start = int(bad[-1]) + 1 if len(bad) else 0
    if np.count_nonzero(~v_pf[start:]) < cfg.stage_window + 1:
        return False
    if not cfg.detector:
        return True
    # detector: the last W records (cycle, residual) and the last one's
    # armed / flagged bits; warm-up complete inside the halo
    w = max(cfg.window, 1)
    vs = view.rec_cycle >= lo_c + start
    ts = cat["rc"] >= lo_c + start
    vc, vr = view.rec_cycle[vs], view.rec_resid[vs]
    tc, tr = cat["rc"][ts], cat["rr"][ts]
    if len(vc) < w or len(tc) != len(vc) or view.n_halo_records < cfg.warmup:
        return False
    if not (np.array_equal(vc[-w:], tc[-w:]) and np.array_equal(vr[-w:], tr[-w:])):
        return False
    return bool(view.rec_armed[vs][-1] == cat["ra"][ts][-1] == 1 and
                view.rec_flagged[vs][-1] == cat["rf"][ts][-1])


def merge(owned: list) -> dict:
    """Concatenate the owned parts in rank order with record / episode
    numbering rebased; a non-positive latency stops the detector for the rest
    of the trace, as in the whole-trace loop."""
    cycles = np.concatenate([o.cycles for o in owned])
    per = {}
    for k in PER_CYCLE:
        parts = [o.per_cycle.get(k) for o in owned]
        per[k] = None if any(p is None for p in parts) else np.concatenate(parts).reshape(-1)
    recs, alerts = [], []
    rec_off = ep_off = 0
    status, first_bad, stopped = 0, (1 << 64) - 1, False
    for o in owned:
        r = o.records.copy()
        a = o.alerts.copy()
        if stopped:
            for f in ("predicted_s", "residual", "statistic"):
                r[f] = 0.0
            for f in ("armed", "flagged", "alert"):
                r[f] = 0
            r["episode_id"] = 0
            a = a[:0]
        else:
            al = r["alert"].astype(bool)
            r["episode_id"][al] += np.uint64(ep_off)
            a["episode_id"] += np.uint64(ep_off)
            a["record_index"] += np.uint64(rec_off)
            if o.first_bad_record >= 0:
                stopped = True
                status = o.status
                first_bad = rec_off + o.first_bad_record
            ep_off += len(a)
        recs.append(r)
        alerts.append(a)
        rec_off += len(r)
    out = dict(cycles=cycles, records=np.concatenate(recs), alerts=np.concatenate(alerts),
               status=status, first_bad_record=first_bad)
    out.update(per)
    return out


@dataclass
class ShardedRun:
    """Driver of the protocol for one rank (or, with a local all-gather,
    for all shards in one process).

    analyze(spec) -> local result dict for events[spec.lo:spec.hi];
    allgather(obj) -> list of every rank's obj (rank order)."""
    events: np.ndarray
    anchor: int
    world: int
    rank: int
    cfg: CheckConfig
    halo: int = 1024
    reruns: list = field(default_factory=list)

    def run(self, analyze, allgather, specs=None, split=None):
        """analyze(spec) -> local result; split(spec, local result, tail_n)
        -> (owned, view, tail), default split_local (split_device for a
        device Analyzer: analyze then returns the Analyzer)."""
        split = split or split_local
        if specs is None:
            _, specs = plan(self.events, self.anchor, self.world, self.halo)
        spec = specs[self.rank]
        tail_n = max(self.halo, 1)
        owned, view, tail = split(spec, analyze(spec), tail_n)
        while True:
            info = allgather((spec, view, tail))
            specs = [i[0] for i in info]
            views = [i[1] for i in info]
            tails = [i[2] for i in info]
            # acceptance chain, left to right: the first shard whose halo
            # fails against its accepted predecessors re-runs with the halo
            # reaching the start of the trace (exact), then the chain is
            # re-checked against its new tail (at most `world` rounds)
            first = next((r for r in range(self.world)
                          if not halo_ok(specs[r], views[r], tails[:r], self.cfg)), None)
            if first is None:
                return owned, specs
            if self.rank == first:
                pos = anchor_positions(self.events, self.anchor)
                spec = shard_spec(self.events, pos, self.rank, spec.c0, spec.c1, None)
                self.reruns.append(self.rank)
                owned, view, tail = split(spec, analyze(spec), tail_n)


def run_all_in_process(events, anchor, world, cfg, analyze_at, halo=1024):
    """Every shard in one process (the GPU tests run it on one device):
    returns (merged result, specs, reruns)."""
    _, specs = plan(events, anchor, world, halo)
    parts = [split_local(s, analyze_at(s), max(halo, 1)) for s in specs]
    reruns = []
    while True:
        acc = [False] * world
        for r in range(world):
            acc[r] = halo_ok(specs[r], parts[r][1], [p[2] for p in parts[:r]], cfg) and (r == 0 or acc[r - 1])
            if not acc[r]:
                break
        if all(acc):
            break
        f = acc.index(False)
        pos = anchor_positions(events, anchor)
        specs[f] = shard_spec(events, pos, f, specs[f].c0, specs[f].c1, None)
        parts[f] = split_local(specs[f], analyze_at(specs[f]), max(halo, 1))
        reruns.append(f)
    return merge([p[0] for p in parts]), specs, reruns
