# Copy one tools_evidence_gpu.sh run (gpurun_out/r2_*) into profiles/: bench
# lines, heuristic / suite benches, launch list + summary, ncu summary, raw
# metrics and the captured kernels' DRAM traffic (profiles/r2_ncu_traffic.json,
# read by bench.py).   Usage: bash tools/tools_evidence_collect.sh [tag]
set -e
cd "$(dirname "$0")/.."
T=${1:-r2}
for f in bench:bench_c2 bench_ref:bench_ref bench_twopass:bench_c2_twopass bench_c3:bench_c3 bench_c5:bench_c5 \
         bench_c1:bench_c1 bench_c1_ref:bench_c1_ref bench_c2_halo:bench_c2_halo_n1 heuristic:heuristic_bench; do
  [ -f gpurun_out/${T}_${f%%:*}.log ] && tail -1 gpurun_out/${T}_${f%%:*}.log > profiles/${T}_${f##*:}.json
done
grep -h "cs_run_us\|cs_stream_push_us" gpurun_out/${T}_c5_host.log | tail -6 > profiles/${T}_c5_host_phases.txt || true
[ -f gpurun_out/suite_bench.json ] && cp gpurun_out/suite_bench.json profiles/${T}_suite_bench.json
cp gpurun_out/${T}_launches.csv profiles/${T}_launches.csv
python tools/tools_launches.py gpurun_out/${T}_launches.csv > profiles/${T}_launches_summary.txt
python tools/tools_ncu_summary.py gpurun_out/${T}_full.ncu-rep > profiles/${T}_ncu_summary.txt
ncu -i gpurun_out/${T}_full.ncu-rep --page raw --csv > profiles/${T}_full_raw.csv 2>/dev/null
T=$T python - <<'PY'
import csv, json, os
T = os.environ["T"]
rows = list(csv.reader(open(f"profiles/{T}_full_raw.csv")))
h, units = rows[0], rows[1]
ki = h.index("Kernel Name")
cols = {m: h.index(m) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1,
         "usecond": 1, "ms": 1e3, "msecond": 1e3}
out = {}
for r in rows[2:]:
    name = r[ki].split("(")[0].replace("void ", "").strip()
    val = lambda m: float(r[cols[m]].replace(",", "")) * scale.get(units[cols[m]], 1)
    key = name
    if key in out:
        key += "_2"
    out[key] = {"dram_read_bytes": val("dram__bytes_read.sum"), "dram_write_bytes": val("dram__bytes_write.sum"),
                "duration_us": val("gpu__time_duration.sum"),
                "workload": "bench.py default (configs[1], 99.9M events)"}
json.dump(out, open(f"profiles/{T}_ncu_traffic.json", "w"), indent=1)
for f in ["bench_c2", "bench_ref", "bench_c2_twopass", "bench_c3", "bench_c5", "bench_c1"]:
    p = f"profiles/{T}_{f}.json"
    if not os.path.exists(p):
        continue
    d = json.load(open(p))
    e2e = d.get("e2e") or {}
    rf = d.get("roofline") or {}
    print(f, d.get("value"), d.get("ms_per_step"), e2e.get("value"), rf.get("frac"), rf.get("kernel_ms"),
          (d.get("latency_ms") or {}).get("p50"))
print({k: round(v["duration_us"], 1) for k, v in out.items()})
PY
