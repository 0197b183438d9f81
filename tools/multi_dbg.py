import sys, ctypes as C, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import paper_2012_12419_b200 as V
from paper_2012_12419_b200 import _native as N
ni = V.generate_instance(N.VCS_GEN_HOMOG, 2012, 0, 5, 8, 40, 3, as_objects=False)
sp = V.StateSpace.build_native(ni, 10**9)
opts = N.vcs_solve_opts(1e-6, 1, 0, 1.0, 3)
dv = np.zeros(2, np.int32)
rep = N.vcs_solve_report()
N.check(N.lib().vcs_solve_multi(sp.handle, C.byref(opts), 2, N.ptr(dv, C.c_int32), 0, None, None, C.byref(rep)))
print("ok", rep.sweeps)
