# Copy one tools_evidence_gpu.sh run (gpurun_out/) into profiles/: bench lines, fit
# and ingest benches, launch list + summary, ncu summary, raw metrics and the
# dominant kernels' DRAM traffic (profiles/r1_ncu_traffic.json, read by bench.py).
set -e
cd "$(dirname "$0")/.."
for f in bench:r1_bench_c2 bench_ref:r1_bench_ref bench_c3:r1_bench_c3 bench_c5:r1_bench_c5 \
         bench_c1:r1_bench_c1 bench_c1_ref:r1_bench_c1_ref bench_c2_halo:r1_bench_c2_halo_n1; do
  tail -1 gpurun_out/${f%%:*}.log > profiles/${f##*:}.json
done
cp gpurun_out/fit_bench.json profiles/r1_fit_bench.json
cp gpurun_out/halo_bench.json profiles/r1_halo_bench.json
cp gpurun_out/suite_bench.json profiles/r1_suite_bench.json
cp gpurun_out/ingest_bench.json profiles/r1_ingest_bench.json
cp gpurun_out/launches.csv profiles/r1_launches.csv
python tools/tools_launches.py gpurun_out/launches.csv > profiles/r1_launches_summary.txt
python tools/tools_ncu_summary.py gpurun_out/full.ncu-rep > profiles/r1_ncu_summary.txt
ncu -i gpurun_out/full.ncu-rep --page raw --csv > profiles/r1_full_raw.csv 2>/dev/null
python - <<'PY'
import csv, json
rows = list(csv.reader(open("profiles/r1_full_raw.csv")))
h, units = rows[0], rows[1]
ki = h.index("Kernel Name")
cols = {m: h.index(m) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1,
         "usecond": 1, "ms": 1e3, "msecond": 1e3}
out = {}
for r in rows[2:]:
    name = r[ki].split("(")[0].strip()
    val = lambda m: float(r[cols[m]].replace(",", "")) * scale.get(units[cols[m]], 1)
    key = name
    if name == "k_scan_warp" and val("gpu__time_duration.sum") < 100:
        key = "k_scan_warp_sample"
    if key in out:
        key += "_2"
    out[key] = {"dram_read_bytes": val("dram__bytes_read.sum"), "dram_write_bytes": val("dram__bytes_write.sum"),
                "duration_us": val("gpu__time_duration.sum"),
                "workload": "bench.py default (configs[1], 99.9M events)"}
json.dump(out, open("profiles/r1_ncu_traffic.json", "w"), indent=1)
for f in ["r1_bench_c2", "r1_bench_ref", "r1_bench_c3", "r1_bench_c5"]:
    d = json.load(open(f"profiles/{f}.json"))
    e2e = d.get("e2e") or {}
    rf = d.get("roofline") or {}
    print(f, d.get("value"), d.get("ms_per_step"), e2e.get("value"), rf.get("frac"), rf.get("kernel_ms"),
          (d.get("latency_ms") or {}).get("p50"))
print({k: round(v["duration_us"], 1) for k, v in out.items()})
PY
