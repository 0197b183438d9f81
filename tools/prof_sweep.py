"""Short driver for ncu: build C4 on the device and run two solves (~100 kernel launches).

    python tools/prof_sweep.py [c4|c3] [auto|jacobi|wavefront]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2012_12419_b200 as V  # noqa: E402
from paper_2012_12419_b200 import _native as N  # noqa: E402

workload = sys.argv[1] if len(sys.argv) > 1 else "c4"
method = {"auto": N.VCS_METHOD_AUTO, "jacobi": N.VCS_METHOD_JACOBI,
          "wavefront": N.VCS_METHOD_WAVEFRONT}[sys.argv[2] if len(sys.argv) > 2 else "auto"]
args = {"c4": (1, 2012, 0, 6, 8, 48, 3), "c3": (1, 2012, 0, 5, 8, 40, 3)}[workload]
ni = V.generate_instance(*args, as_objects=False)
sp = V.StateSpace.build_native(ni, 10**9)
for _ in range(2):
    r = V.run_value_iteration(sp, V.ViOptions(method=method))
rep = r.values.report
print(f"S={sp.size()} E={sp.edges()} sweeps={rep.sweeps} sweep_ms={rep.sweep_ms:.3f} "
      f"extract_ms={rep.extract_ms:.3f} build_ms={sp.info.build_ms:.1f} launches={N.kernel_launches()}")
