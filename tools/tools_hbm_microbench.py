"""HBM streaming microbenchmark: LDG vs TMA bulk (profiling helper)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_09258_b200 import runtime as rt
L = rt.lib()
nbytes = 3_200_000_000
buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
buf.fill_(1)
torch.cuda.synchronize()
def run(v, p0, p1, p2):
    ms = C.c_double()
    rc = rt.bench_lib().cs_microbench(v, C.c_void_p(buf.data_ptr()), nbytes, p0, p1, p2, 5, C.byref(ms))
    return rc, ms.value, nbytes / ms.value / 1e6
for cfg in [(0, 4, 256, 8), (0, 8, 256, 8), (0, 2, 512, 8), (0, 8, 256, 1), (0, 16, 256, 1)]:
    print("LDG ctas/sm,threads,unroll", cfg[1:], "-> rc %d %.3f ms %.0f GB/s" % run(*cfg))
for cfg in [(1, 32768, 2, 1), (1, 32768, 4, 1), (1, 32768, 6, 1), (1, 65536, 3, 1), (1, 16384, 8, 1),
            (1, 8192, 16, 1), (1, 32768, 2, 2), (1, 16384, 4, 2), (1, 16384, 6, 2), (1, 8192, 8, 3),
            (1, 4096, 12, 4)]:
    print("TMA chunk,stages,ctas/sm", cfg[1:], "-> rc %d %.3f ms %.0f GB/s" % run(*cfg))
