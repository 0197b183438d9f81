"""Per-layer host timeline of warm C4 builds (VCS_TRACE=1) and pinned D2H bandwidth."""
import ctypes as C
import os
import sys
import time
from pathlib import Path

os.environ["VCS_TRACE"] = "1"
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import paper_2012_12419_b200 as V  # noqa: E402
from paper_2012_12419_b200 import _native as N  # noqa: E402

ni = V.generate_instance(1, 2012, 0, 6, 8, 48, 3, as_objects=False)
for it in range(4):
    print(f"--- build {it}", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    h = C.c_void_p()
    N.check(N.lib().vcs_space_build(ni.ref, 10**9, 0, C.byref(h)))
    print(f"build {it}: {1e3 * (time.perf_counter() - t0):.2f} ms", file=sys.stderr, flush=True)
    N.lib().vcs_space_free(h)

S = 19333781
for nbytes in (S * 8, S * 4, 4 << 20):
    src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    dst = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"D2H pinned {nbytes / 1e6:.1f} MB: {dt * 1e3:.3f} ms = {nbytes / dt / 1e9:.1f} GB/s",
          file=sys.stderr)
