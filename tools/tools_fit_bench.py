"""Batched device GBDT fit vs host fits (GPU helper).
configs[2]-shaped: 1024 instances, ~2400 training samples each (tie-heavy
integer features: batch in 1..64, w_kv = batch * (in + out)), default
GbdtParams (200 trees, depth 5).  Reports the device batch (wall and kernel
time), the host C++ fit and the reference's fit per model, and checks a
sample of the device models against both byte for byte.
Writes gpurun_out/fit_bench.json."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2601_09258_b200 import runtime as rt


def samples(n, seed):
    rng = np.random.default_rng(seed)
    batch = rng.integers(1, 65, n).astype(float)
    inp = rng.integers(16, 2048, n).astype(float)
    out = rng.integers(1, 512, n).astype(float)
    w_kv = batch * (inp + out)
    y = 2e-3 + 1e-5 * batch + 3e-9 * w_kv + rng.normal(0, 2e-4, n) ** 2
    return np.stack([batch, w_kv], 1), y


def main():
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    sets = [samples(2400, s) for s in range(M)]
    xs, ys = [s[0] for s in sets], [s[1] for s in sets]
    rt.fit_latency_models(xs[:2], ys[:2])  # context warm-up
    t0 = time.perf_counter()
    models, dev_ms = rt.fit_latency_models(xs, ys)
    wall = time.perf_counter() - t0
    out = {"models": M, "rows_per_model": 2400, "device_batch_wall_s": round(wall, 3),
           "device_kernel_ms": round(dev_ms, 1), "host_threads": os.cpu_count()}
    k = 8
    t0 = time.perf_counter()
    host = [rt.fit_latency_model(xs[i], ys[i]).to_json() for i in range(k)]
    per_host = (time.perf_counter() - t0) / k
    out["host_fit_s_per_model"] = round(per_host, 4)
    out["host_fit_all_models_est_s_on_all_threads"] = round(per_host * M / (os.cpu_count() or 1), 2)
    assert all(models[i].to_json() == host[i] for i in range(k))
    try:
        from oracle import refbridge as rb
        if rb.available():
            t0 = time.perf_counter()
            ref = [rb.ref_fit(xs[i], ys[i], ["batch", "w_kv"]) for i in range(4)]
            out["reference_fit_s_per_model"] = round((time.perf_counter() - t0) / 4, 4)
            assert all(models[i].to_json() == ref[i] for i in range(4))
            out["identical_to_reference"] = True
    except Exception as e:  # noqa: BLE001
        out["reference"] = f"skipped: {e}"
    print(json.dumps(out))
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/fit_bench.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
