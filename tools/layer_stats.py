"""Layer sizes vs key-space sizes of a bench workload (which certified kernel walks each layer)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench_workloads as W  # noqa: E402
import paper_2012_12419_b200 as V  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
p = V.parse_instance(W.instance_text(name))
inst = V.MdpInstance.from_workload(p.vcc, p.bots)
sp = V.StateSpace.build_native(inst.native(), 10**9, 0, inst)
lo = sp.layer_offsets().astype(np.int64)
n = np.diff(lo)
caps = [c.vm_free + 1 for c in p.vcc.clouds]
print(name, "S", sp.size(), "key space", int(np.prod(caps)))
print("layer sizes:", n.tolist())
