"""Small device-fit batch for profiling (GPU helper): M models x 1920 rows."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from tools_fit_bench import samples  # noqa: E402

from paper_2601_09258_b200 import abi, runtime as rt  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 8
T = int(sys.argv[2]) if len(sys.argv) > 2 else 200
p = abi.default_gbdt_params()
p.n_trees = T
sets = [samples(2400, s) for s in range(M)]
models, ms = rt.fit_latency_models([s[0] for s in sets], [s[1] for s in sets], params=p)
print(f"models {M} trees {T} kernel_ms {ms:.1f}")
