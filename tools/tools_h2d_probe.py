"""H2D ceiling probe (GPU helper): one large pinned copy vs the columnar wire
upload (9 copies + expand) of configs[1]-shaped data."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2601_09258_b200 import abi, runtime as rt

n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
print(f"single pinned copy: {5 * n / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
for parts in (2, 9, 32):
    cs = n // parts
    t0 = time.perf_counter()
    for _ in range(5):
        for k in range(parts):
            d[k * cs:(k + 1) * cs].copy_(h[k * cs:(k + 1) * cs], non_blocking=True)
    torch.cuda.synchronize()
    print(f"{parts} pinned copies: {5 * cs * parts / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
del d, h

tr = rt.synth_trace(400_000, 1, 2, n_ranks=8, n_chunks=16, n_threads=os.cpu_count(), compact_names=False)
wt = rt.wire_pack(tr.events, [0, len(tr.events)], tr.workloads)
cols = [getattr(wt, c) for c in rt.WireTrace.COLUMNS]
nb = sum(a.nbytes for a in cols)
ptr, pin = rt.host_alloc(nb + 16 * len(cols))
views, o = [], 0
for a in cols:
    o = (o + 15) & ~15
    pin[o:o + a.nbytes] = a.view(np.uint8).reshape(-1)
    views.append(pin[o:o + a.nbytes].view(a.dtype).reshape(a.shape))
    o += a.nbytes
wire = rt.WireTrace(*views, wt.inst_offsets)
an = rt.Analyzer(0)
an.configure(tr.names, rt.span_names_mask(tr.events, len(tr.names)), n_comm_slots=tr.n_comm)
for _ in range(3):
    an.upload_wire(wire)
    an.sync()
t0 = time.perf_counter()
for _ in range(5):
    an.upload_wire(wire)
    an.sync()
el = (time.perf_counter() - t0) / 5
print(f"wire upload+expand: {len(tr.events)} events, {nb / 1e6:.0f} MB, {el * 1e3:.2f} ms, {nb / el / 1e9:.1f} GB/s")
an.close()
rt.host_free(ptr)
