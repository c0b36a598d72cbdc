"""Batched device GBDT fit (cs_fit_latency_models) vs the
reference's fit_latency_model (oracle/_ref) and the host fit: byte-identical
model JSON for every model of a batch: tie-heavy integer features, several
sizes (including one that runs from global scratch instead of shared
memory), a degenerate target, other feature sets and GbdtParams; per-model
errors for too few samples and non-positive targets."""
import numpy as np
import pytest

from paper_2601_09258_b200 import abi
from paper_2601_09258_b200 import runtime as rt

pytestmark = pytest.mark.gpu


def _samples(n, seed, n_features=2, distinct_batch=64):
    rng = np.random.default_rng(seed)
    batch = rng.integers(1, distinct_batch + 1, n).astype(float)
    inp = rng.integers(16, 2048, n).astype(float)
    out = rng.integers(1, 512, n).astype(float)
    w_kv = batch * (inp + out)
    y = 2e-3 + 1e-5 * batch + 3e-9 * w_kv + rng.normal(0, 2e-4, n) ** 2
    cols = [batch, w_kv, inp, out, (rng.random(n) < 0.3).astype(float)][:n_features]
    return np.stack(cols, 1), y


def _check_batch(refbridge, xs, ys, names, params=None):
    models, ms = rt.fit_latency_models(xs, ys, names, params=params)
    assert ms > 0
    for x, y, m in zip(xs, ys, models):
        opts = abi.default_fit_options(len(names))
        opts.stratify_col = list(names).index("w_kv") if "w_kv" in names else 0
        try:
            host = rt.fit_latency_model(x, y, names, params=params, options=opts).to_json()
        except rt.EngineError as e:
            assert isinstance(m, rt.EngineError) and m.status == e.status
            continue
        assert not isinstance(m, rt.EngineError)
        got = m.to_json()
        assert got == host
        assert got == refbridge.ref_fit(x, y, list(names), params=params, options=opts)
    return models


def test_batch_matches_reference(refbridge):
    sizes = [40, 300, 1900, 2400, 700, 6000]
    xs, ys = [], []
    for k, n in enumerate(sizes):
        x, y = _samples(n, 10 + k, distinct_batch=[4, 64, 64, 64, 1000, 64][k])
        xs.append(x)
        ys.append(y)
    # degenerate target, too few samples, a non-positive target
    x, _ = _samples(200, 99)
    xs.append(x)
    ys.append(np.full(200, 0.004))
    x, y = _samples(7, 98)
    xs.append(x)
    ys.append(y)
    x, y = _samples(100, 97)
    y[5] = -1.0
    xs.append(x)
    ys.append(y)
    models = _check_batch(refbridge, xs, ys, ("batch", "w_kv"))
    assert isinstance(models[-1], rt.EngineError) and isinstance(models[-2], rt.EngineError)


def test_batch_feature_sets_and_params(refbridge):
    xs, ys = zip(*[_samples(n, 50 + n, n_features=5) for n in (150, 900, 2000)])
    names = ("batch", "w_kv", "input_len", "output_len", "stage")
    _check_batch(refbridge, list(xs), list(ys), names)
    p = abi.default_gbdt_params()
    p.n_trees, p.max_depth, p.min_samples_leaf, p.learning_rate = 40, 8, 1, 0.3
    xs2, ys2 = zip(*[_samples(n, 70 + n) for n in (64, 500, 1500)])
    _check_batch(refbridge, list(xs2), list(ys2), ("batch", "w_kv"), params=p)
    p.max_depth, p.min_samples_leaf = 3, 20
    _check_batch(refbridge, list(xs2), list(ys2), ("w_kv", "batch"), params=p)


def test_simkit_instances_batch(refbridge):
    """The bench's per-instance fits (first 2400 cycles of each instance)."""
    xs, ys = [], []
    for i in range(6):
        t = rt.synth_trace(2600, 100 + i, 200 + i, n_ranks=1 + (i % 3), compact_names=False)
        an = rt.Analyzer(0)
        an.configure(t.names, rt.span_names_mask(t.events, len(t.names)), n_comm_slots=t.n_comm)
        an.upload(t.events, [0, len(t.events)], t.workloads)
        an.run(abi.RUN_SEGMENT)
        recs = an.records(0)
        an.close()
        tr = recs[recs["cycle_index"] < 2400]
        xs.append(np.stack([tr["batch"].astype(float),
                            (tr["batch"] * (tr["input_len"] + tr["output_len"])).astype(float)], 1))
        ys.append(tr["latency_s"])
    _check_batch(refbridge, xs, ys, ("batch", "w_kv"))
