"""BASELINE config 4 (SuiteConfig{}: 20 trials x 3800 cycles) on one B200 vs
the reference's evaluate_trial (GPU helper).

Ours: every trial segmented on the device, the 20 latency models fitted in
one device batch, monitoring under the three strategies (cs_redetect) and
cs_evaluate_strategy, pooled as evaluate_suite pools them
(simkit.cpp:1038-1068).  Reference: its own evaluate_trial per trial
(oracle/_ref, one thread), pooled the same way.  Checks the per-trial counts
and the pooled metrics bit for bit; reports both wall times (trial
generation excluded on both sides).  Writes gpurun_out/suite_bench.json."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

from oracle import refbridge
from paper_2601_09258_b200 import runtime as rt
from test_gpu_eval import suite_metrics


def main():
    an = rt.Analyzer(0)
    an.set_fused(False)
    suite_metrics(refbridge, rt, an, n_trials=2)  # warm-up (allocations, first fit)
    tick = {}
    ours, ref_rows, skipped = suite_metrics(refbridge, rt, an, timer=tick)
    an.close()
    got = rt.pool_strategy_metrics(ours)
    want = rt.pool_strategy_metrics(ref_rows)
    same = bool(np.array_equal(got.view(np.uint64), want.view(np.uint64)))
    names = ["fixed_point", "fixed_window", "dynamic_window"]
    out = {"trials": len(ours), "skipped_by_reference_gate": skipped, "identical": same,
           "ours_s": round(tick["ours_s"], 3), "reference_s": round(tick["reference_s"], 3),
           "aggregate": {n: dict(zip(["tp", "fp", "fn", "tn", "alerts", "precision", "recall", "f1", "fpr",
                                      "mean_lag"], [float(v) for v in got[k]]))
                         for k, n in enumerate(names)}}
    print(json.dumps(out))
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/suite_bench.json", "w") as f:
        json.dump(out, f, indent=1)
    assert same


if __name__ == "__main__":
    main()
