import csv, subprocess, sys
rep, regex = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{regex}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if "Source" in r][-1]
hdr = rows[hi]
si = hdr.index("Source"); wi = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for k, r in enumerate(rows[hi + 1:]):
    try:
        data.append((int(r[wi]), k, r[si]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print("samples", tot, "instructions", len(data))
srcs = [d[2] for d in data]
for w, k, s in sorted(data, reverse=True)[:n]:
    ctx = " | ".join(x.strip() for x in srcs[max(0, k - 3):k])
    print(f"{100 * w / tot:5.1f}%  {s.strip():45s}  <- {ctx[-110:]}")
