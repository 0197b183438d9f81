"""Driver for ncu / timing of the greedy kernels on SURVEY C2 (10^5 tasks x 10^3 clouds)."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2012_12419_b200 as V  # noqa: E402
from paper_2012_12419_b200 import _native as N  # noqa: E402

ni = V.generate_instance(N.VCS_GEN_GREEDY, 12345, 0, 1000, 100, 1000, 3, as_objects=False)
tgt = np.empty(100000, np.int32)
paid, unused = C.c_int64(), C.c_int64()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    N.check(N.lib().vcs_greedy(ni.ref, 0, N.ptr(tgt, C.c_int32), None, C.byref(paid), C.byref(unused)))
    ts.append((time.perf_counter() - t0) * 1e3)
print(f"greedy C2: paid={paid.value} unused={unused.value} e2e_ms={[round(t, 2) for t in ts]}")
