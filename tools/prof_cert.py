"""Short driver for ncu: build one bench workload on the device and run two certified solves.

    python tools/prof_cert.py [c4|c3|c7|c1]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench_workloads as W  # noqa: E402
import paper_2012_12419_b200 as V  # noqa: E402
from paper_2012_12419_b200 import _native as N  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
p = V.parse_instance(W.instance_text(name))
inst = V.MdpInstance.from_workload(p.vcc, p.bots)
sp = V.StateSpace.build_native(inst.native(), 10**9, 0, inst)
for _ in range(2):
    r = V.run_value_iteration(sp, V.ViOptions(method=N.VCS_METHOD_CERTIFIED))
rep = r.values.report
print(f"{name}: S={sp.size()} E={sp.edges()} sweeps={rep.sweeps} solve_ms={rep.sweep_ms:.3f} "
      f"build_ms={sp.info.build_ms:.1f} launches={N.kernel_launches()}")
