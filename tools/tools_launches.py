"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per kernel count / mean / share, over all launches and over the timed-step
kernels only (setup: the device fit, the LUT compile and the record gather;
the e2e leg's wire expand).  python tools_launches.py launches.csv"""
import collections
import csv
import sys

SETUP = {"k_gbdt_fit", "k_lut_build", "k_gather_records"}
E2E = {"k_wire_expand"}
SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = collections.defaultdict(list)
for r in rows[hi + 1:]:
    name = r[ki].split("(")[0].replace("<unnamed>::", "").replace("void ", "").replace("csb::", "").strip()
    tot[name].append(float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0))


def table(title, names):
    allt = sum(sum(tot[k]) for k in names) or 1.0
    print(title)
    for k in sorted(names, key=lambda k: -sum(tot[k])):
        v = tot[k]
        print(f"  {k:28s} n={len(v):3d} mean={sum(v) / len(v):10.1f} us  min={min(v):10.1f}  "
              f"max={max(v):10.1f}  share={100 * sum(v) / allt:5.1f}%")


table("all launches (setup + timed steps + e2e legs)", list(tot))
table("timed-step kernels (device-resident analysis)", [k for k in tot if k not in SETUP | E2E])
