"""One warm C4 build after one cold build (for ncu launch lists of the builder)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2012_12419_b200 as V  # noqa: E402
from paper_2012_12419_b200 import _native as N  # noqa: E402

ni = V.generate_instance(1, 2012, 0, 6, 8, 48, 3, as_objects=False)
for it in range(2):
    h = C.c_void_p()
    N.check(N.lib().vcs_space_build(ni.ref, 10**9, 0, C.byref(h)))
    N.lib().vcs_space_free(h)
