"""Throughput of vcs_policy_query on C4: 1M random full states (layers 20..47, free VMs in
[0, 8] per cloud: reachable in C4's saturated layers), device-resident inputs and outputs."""
import ctypes as C
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2012_12419_b200 as V  # noqa: E402
from paper_2012_12419_b200 import _native as N  # noqa: E402

ni = V.generate_instance(N.VCS_GEN_HOMOG, 2012, 0, 6, 8, 48, 3, as_objects=False)
sp = V.StateSpace.build_native(ni, 10**9)
opts = N.vcs_solve_opts(1e-6, 1, 0, 1.0, 0)
rep = N.vcs_solve_report()
N.check(N.lib().vcs_solve(sp.handle, C.byref(opts), None, None, C.byref(rep)))
n = 1 << 20
rng = np.random.default_rng(1)
fv = rng.integers(0, 9, size=(n, 6), dtype=np.int32)
ti = rng.integers(20, 48, size=n, dtype=np.int32)
te = np.zeros(n, dtype=np.uint8)
dev = torch.device("cuda", 0)
dfv, dti, dte = (torch.from_numpy(x).to(dev) for x in (fv, ti, te))
dval = torch.empty(n, dtype=torch.float64, device=dev)
dact = torch.empty(n, dtype=torch.int32, device=dev)
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
s = torch.cuda.Stream(dev)
for _ in range(3):
    N.check(N.lib().vcs_policy_query(sp.handle, n, p(dfv), p(dti), p(dte), p(dval), p(dact), None,
                                     C.c_void_p(s.cuda_stream)))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(10):
    N.check(N.lib().vcs_policy_query(sp.handle, n, p(dfv), p(dti), p(dte), p(dval), p(dact), None,
                                     C.c_void_p(s.cuda_stream)))
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
found = int((~torch.isnan(dval)).sum())
print(f"{n} queries in {ms:.3f} ms = {n / ms / 1e3:.1f} M queries/s; reachable {found}")
# host arrays (staged copies included)
vals = np.empty(n); acts = np.empty(n, np.int32)
t0 = time.perf_counter()
N.check(N.lib().vcs_policy_query(sp.handle, n, C.c_void_p(fv.ctypes.data), C.c_void_p(ti.ctypes.data),
                                 C.c_void_p(te.ctypes.data), C.c_void_p(vals.ctypes.data),
                                 C.c_void_p(acts.ctypes.data), None, None))
print(f"host buffers: {1e3 * (time.perf_counter() - t0):.2f} ms")
