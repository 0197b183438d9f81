"""Median device time-to-convergence of repeated certified solves of one bench workload (the
bench `value` without the rest of bench.py), for A/B runs of kernel switches.

    python tools/solve_time.py [c4|c3|c1|c7] [solves]"""
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench_workloads as W  # noqa: E402
import paper_2012_12419_b200 as V  # noqa: E402
from paper_2012_12419_b200 import _native as N  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
p = V.parse_instance(W.instance_text(name))
inst = V.MdpInstance.from_workload(p.vcc, p.bots)
sp = V.StateSpace.build_native(inst.native(), 10**9, 0, inst)
ts = []
for i in range(n + 3):
    r = V.run_value_iteration(sp, V.ViOptions(method=N.VCS_METHOD_CERTIFIED))
    if i >= 3:
        ts.append(r.values.report.sweep_ms)
print(f"{name}: S={sp.size()} median {statistics.median(ts):.4f} ms min {min(ts):.4f} "
      f"sweeps={r.values.report.sweeps}")
