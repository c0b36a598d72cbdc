"""Native Chrome-trace JSON ingest (cs_ingest_chrome_json)
vs the reference's own parse_trace_json (trace_io.cpp:87-206) followed by
the oracle-side exporter (oracle/ref_bridge.cpp): identical records, event
ids, names, workload table, collective slots and issue counts, on simkit
traces serialized by the reference and on hand-written edge documents."""
import json

import numpy as np
import pytest

from paper_2601_09258_b200 import abi, runtime as rt


def _compare(refbridge, text: bytes):
    ref, n_issues = refbridge.RefTrace.from_json(text)
    ex = ref.export(None)
    got = rt.ingest_chrome_json(text, n_threads=4)
    assert got.n_issues == n_issues
    assert got.names == ex.names
    assert got.events.tobytes() == ex.events.tobytes()
    assert np.array_equal(got.event_ids, ex.event_ids)
    assert got.workloads.tobytes() == ex.workloads.tobytes()
    assert got.comm_hash == ex.comm_hash
    assert list(got.comm_rank) == list(ex.comm_rank)
    # the ValidationReport (validate_trace with the parse issues)
    iss, cats, n_err = ref.validate()
    assert got.issues.tobytes() == iss.tobytes()
    assert np.array_equal(got.category_counts, cats)
    assert got.n_errors == n_err and got.ok == (n_err == 0)
    # resolve_topology per comm slot (align.cpp:178-191)
    if not got.topology_conflict:
        topo = ref.topology()
        assert [list(got.locations[i]) if i >= 0 else None for i in got.comm_location] == topo
    return got


@pytest.mark.parametrize("ranks,fault", [(1, "cpu_contention"), (4, "nvlink_saturation"),
                                         (8, "pcie_bottleneck")])
def test_simkit_round_trip(refbridge, ranks, fault):
    t = refbridge.RefTrace.synth(1500, 3, 4, n_ranks=ranks, fault=fault, onset=1000, duration=100,
                                 target_rank=ranks - 1)
    text = t.to_json()
    got = _compare(refbridge, text)
    assert len(got.events) > 1500 * 19
    wrapped = b'{"displayTimeUnit": "ns", "traceEvents": ' + text + b', "x": [1, {"y": null}]}'
    _compare(refbridge, wrapped)


def _doc(records, wrap=False):
    body = "[" + ",\n".join(r if isinstance(r, str) else json.dumps(r) for r in records) + "]"
    return (('{"traceEvents": ' + body + '}') if wrap else body).encode()


EDGE = [
    # phases, metadata, malformed records
    {"ph": "M", "name": "process_name", "args": {"name": "x"}},
    {"ph": "B", "name": "unsupported", "ts": 1},
    {"name": "no_phase", "ts": 2},
    '5',
    {"ph": "X", "name": "run_batch", "ts": 10, "dur": 4.5, "args": {"forward_mode": "DECODE",
                                                                     "batch_size": 3,
                                                                     "input_len": 7,
                                                                     "output_len": 1}},
    {"ph": "X", "name": "run_batch", "ts": 20.0004, "dur": 3, "eid": 100,
     "args": {"forward_mode": "Extend", "batch_size": 2.9, "input_len": True, "output_len": 0}},
    {"ph": "X", "name": "run_batch", "ts": 20.0004, "dur": 1, "eid": 7},   # equal ts, lower id
    {"ph": "X", "name": "gemm_kernel", "ts": 12, "dur": 1, "cat": "gpu_kernel"},
    {"ph": "X", "name": "oddcat", "ts": 13, "dur": 1, "cat": "not_a_category"},
    {"ph": "X", "name": "badcat", "ts": 13, "dur": 1, "cat": 5},          # type error: dropped
    {"ph": "X", "name": 17, "ts": 14},                                    # type error: dropped
    {"ph": "X", "name": "str_ts", "ts": "15"},                            # type error: dropped
    {"ph": "X", "name": "bool_ts", "ts": True},                           # type error: dropped
    {"ph": "X", "name": "pid_str", "ts": 16, "pid": "a"},                 # type error: dropped
    {"ph": "X", "name": "eid_float", "ts": 17, "eid": 9.7},
    {"ph": "i", "name": "inst", "ts": 18, "dur": 5, "args": {"forward_mode": "prefill"}},
    {"ph": "C", "name": "cpu_usage", "ts": 19, "args": {"value": 3}},
    {"ph": "C", "name": "cpu_usage", "ts": 19.5, "args": {"value": 2.25}},
    {"ph": "C", "name": "gpu_usage", "ts": 19.7, "args": {"other": 1}},
    {"ph": "C", "name": "bool_value", "ts": 19.8, "args": {"value": False}},
    {"ph": "X", "name": "reduce", "ts": 21, "dur": 2, "cat": "collective_comm",
     "args": {"commHash": "abc", "rank": 3}},
    {"ph": "X", "name": "reduce", "ts": 22, "dur": 2, "cat": "collective_comm",
     "args": {"commHash": "abc", "rank": 1.9}},
    {"ph": "X", "name": "reduce", "ts": 23, "dur": 2, "cat": "collective_comm",
     "args": {"commHash": 5, "rank": 1}},
    {"ph": "s", "name": "flow", "ts": 24, "id": 1},
    {"ph": "f", "name": "flow", "ts": 25, "args": {"flow": "zz"}},
    # args: nesting, arrays, nulls, duplicate keys, keys that flatten alike
    '{"ph": "X", "name": "nest", "ts": 26, "dur": 1, "args": {"a": {"forward_mode": "decode"},'
    ' "b": [1, {"c": 2}], "z": null, "batch_size": 4, "batch_size": 5, "input_len": 1,'
    ' "output_len": 2}}',
    '{"ph": "X", "name": "flat", "ts": 27, "dur": 1, "args": {"x": {"batch_size": 9},'
    ' "x.batch_size": 8, "batch_size": {"a": 1}}}',
    '{"ph": "X", "name": "dupkey", "ts": 28, "ph": "i", "dur": 3, "name": "dup2"}',
    # strings, numbers
    {"ph": "X", "name": "café \U0001F600 \"q\" \\ /", "ts": 29, "dur": 1},
    '{"ph": "X", "name": "esc\\u00e9\\ud83d\\ude00\\t", "ts": 30, "dur": 1e0, "tid": -0}',
    '{"ph": "X", "name": "bigint", "ts": 31, "dur": 1, "eid": 18446744073709551615,'
    ' "args": {"batch_size": 9223372036854775808, "input_len": -5, "output_len": 1E2}}',
    '{"ph": "X", "name": "tiny", "ts": 32, "dur": 1, "args": {"batch_size": 1e-400}}',
    {"ph": "X", "name": "neg_dur", "ts": 33, "dur": -2.5},
    {"ph": "X", "name": "round", "ts": 0.0005, "dur": 0.0015},
]


@pytest.mark.parametrize("wrap", [False, True])
def test_edge_records(refbridge, wrap):
    got = _compare(refbridge, _doc(EDGE, wrap))
    assert got.n_issues > 5


@pytest.mark.parametrize("text", [
    b'[{"ph": "X", "ts": 1,}]', b'[{"ph": "X", "ts": 01}]', b'[{"ph": "X", "name": "a\x01"}]',
    b'[{"ph": "X", "name": "\xff"}]', b'[{"ph": "X"}] trailing', b'{"traceEvents": 5}',
    b'"just a string"', b'[{"ph": "X", "ts": 1e}]', b'[{"ph": "X", "name": "\\x"}]',
    b'[{"ph": "X", "name": "\\ud800"}]', b'', b'[{"ph": "X", "ts": -}]', b'{}',
    b'{"traceEvents": [{"ph": "X", "ts": 1}], "traceEvents": [{"ph": "i", "ts": 2}]}'])
def test_invalid_and_odd_documents(refbridge, text):
    _compare(refbridge, text)


def test_float_overflow_rejects_the_document():
    """nlohmann throws out_of_range.406 on 1e400, which the reference's
    parse_trace_json does not catch (the process terminates); the native
    ingest treats it as an invalid document instead."""
    got = rt.ingest_chrome_json(b'[{"ph": "X", "ts": 1, "args": {"v": 1e400}}, {"ph": "X", "ts": 2}]')
    assert got.n_issues == 1 and len(got.events) == 0


def _nasty(seed, n):
    """Records whose strings hold quotes, backslash runs, brackets and commas,
    at random lengths so the splitter's chunk boundaries land inside them."""
    rng = np.random.default_rng(seed)
    alphabet = ['"', '\\', '[', ']', '{', '}', ',', ':', 'a', ' ', '\\\\', '\\"']
    recs = []
    for i in range(n):
        k = int(rng.integers(0, 40))
        name = "".join(alphabet[j] for j in rng.integers(0, len(alphabet), k))
        r = {"ph": "X", "name": name[:6] or "n", "ts": int(rng.integers(0, 10**6)), "dur": 1,
             "args": {"note": name, "deep": [[{"s": name}], {"t": [name, 1]}],
                      "batch_size": int(rng.integers(1, 9))}}
        recs.append(r)
    return recs


@pytest.mark.parametrize("seed", [0, 1])
def test_parallel_split_adversarial_strings(refbridge, seed):
    text = _doc(_nasty(seed, 12000), wrap=bool(seed))
    assert len(text) > 1 << 21
    got = _compare(refbridge, text)
    for nt in (1, 3, 8):
        alt = rt.ingest_chrome_json(text, n_threads=nt)
        assert alt.events.tobytes() == got.events.tobytes() and alt.names == got.names
    # a stray backslash outside any string, deep in the document, rejects it
    cut = len(text) // 2
    pos = text.index(b'"ts"', cut)
    bad = text[:pos] + b'\\' + text[pos:]
    for nt in (1, 8):
        r = rt.ingest_chrome_json(bad, n_threads=nt)
        assert r.n_issues == 1 and len(r.events) == 0


VALIDATION = [
    # duplicate ids (reported once, at the second occurrence), negative spans
    {"ph": "X", "name": "a", "ts": 1, "dur": 1, "eid": 5},
    {"ph": "X", "name": "b", "ts": 2, "dur": 1, "eid": 5},
    {"ph": "i", "name": "c", "ts": 3, "eid": 5},
    {"ph": "X", "name": "neg", "ts": 4, "dur": -1},
    # correlations: matched, unmatched device, duplicate device / host, float ids
    {"ph": "X", "name": "launch", "ts": 5, "dur": 1, "cat": "runtime_api", "args": {"correlation_id": 1}},
    {"ph": "X", "name": "k1", "ts": 6, "dur": 1, "cat": "gpu_kernel", "args": {"correlation_id": 1}},
    {"ph": "X", "name": "k2", "ts": 7, "dur": 1, "cat": "gpu_kernel", "args": {"correlation_id": 2}},
    {"ph": "X", "name": "m1", "ts": 8, "dur": 1, "cat": "mem_copy", "args": {"correlation_id": 3}},
    {"ph": "X", "name": "m2", "ts": 9, "dur": 1, "cat": "mem_copy", "args": {"correlation_id": 3}},
    {"ph": "X", "name": "l2", "ts": 10, "dur": 1, "cat": "runtime_api", "args": {"correlation_id": 4}},
    {"ph": "X", "name": "l3", "ts": 11, "dur": 1, "cat": "runtime_api", "args": {"correlation_id": 4}},
    {"ph": "X", "name": "kf", "ts": 12, "dur": 1, "cat": "gpu_kernel", "args": {"correlation_id": 9.5}},
    {"ph": "X", "name": "py", "ts": 13, "dur": 1, "args": {"correlation_id": 77}},
    # counters: missing / non-numeric value, non-increasing series (flagged once)
    {"ph": "C", "name": "cpu", "ts": 20, "args": {"value": 1}},
    {"ph": "C", "name": "cpu", "ts": 20, "args": {"value": 2}},
    {"ph": "C", "name": "cpu", "ts": 19, "args": {"value": 3}},
    {"ph": "C", "name": "gpu", "ts": 21, "args": {"other": 1}},
    {"ph": "C", "name": "gpu", "ts": 22, "args": {"value": "x"}},
    {"ph": "C", "name": "mem", "ts": 23, "args": {"value": True}},
    # parse-side issues with event ids (unknown category, dropped null args)
    {"ph": "X", "name": "odd", "ts": 24, "dur": 1, "cat": "zzz", "args": {"p": None, "q": None}},
    {"ph": "X", "name": "odd2", "ts": 25, "dur": 1, "cat": "zzz", "eid": 900, "src": {"collector": 3}},
]


@pytest.mark.parametrize("wrap", [False, True])
def test_validation_report(refbridge, wrap):
    got = _compare(refbridge, _doc(VALIDATION, wrap))
    codes = {abi.ISSUE_CODES[c] for c in got.issues["code"]}
    assert {"duplicate_event_id", "negative_duration", "duplicate_correlation",
            "unmatched_correlation", "non_monotone_counter", "malformed_args"} <= codes
    assert not got.ok


def test_validation_many_duplicate_ids(refbridge):
    """Out-of-order, repeating explicit ids (the parallel duplicate search)."""
    rng = np.random.default_rng(3)
    recs = [{"ph": "X", "name": f"n{i % 7}", "ts": int(t), "dur": 1, "eid": int(e)}
            for i, (t, e) in enumerate(zip(rng.integers(0, 5000, 20000), rng.integers(0, 15000, 20000)))]
    got = _compare(refbridge, _doc(recs))
    assert (got.issues["code"] == 2).sum() > 1000


def test_topology_and_conflict(refbridge):
    recs = [{"ph": "X", "name": "reduce", "ts": 1 + r, "dur": 1, "cat": "collective_comm",
             "args": {"commHash": h, "rank": r, "hostname": f"n{r // 2}", "device": r % 2}}
            for h in ("a", "b") for r in range(4)]
    recs.append({"ph": "i", "name": "reduce", "ts": 9, "cat": "collective_comm",  # instants count too
                 "args": {"commHash": "c", "rank": 0, "hostname": "n9", "device": 3}})
    recs.append({"ph": "X", "name": "reduce", "ts": 10, "dur": 1, "cat": "collective_comm",
                 "args": {"commHash": "c", "rank": 0}})                          # unmapped slot? no: mapped
    recs.append({"ph": "X", "name": "reduce", "ts": 11, "dur": 1, "cat": "collective_comm",
                 "args": {"commHash": "d", "rank": 1}})                          # unmapped
    got = _compare(refbridge, _doc(recs))
    assert not got.topology_conflict and -1 in list(got.comm_location)
    recs.append({"ph": "X", "name": "reduce", "ts": 12, "dur": 1, "cat": "collective_comm",
                 "args": {"commHash": "a", "rank": 0, "hostname": "elsewhere", "device": 0}})
    assert rt.ingest_chrome_json(_doc(recs)).topology_conflict
