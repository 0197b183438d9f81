"""Layer sizes vs key-space sizes of a bench workload (which certified kernel walks each layer);
writes tools/<name>_layers.json for tools/ncu_cert_summary.py.

    python tools/layer_stats.py [c4|c7|c3|c1]"""
import json
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
key_space = int(np.prod([c.vm_free + 1 for c in p.vcc.clouds]))
H = sp.task_count()
doc = {"workload": name, "S": sp.size(), "H": H, "key_space": key_space,
       "layers": [int(x) for x in n],
       # k_cert_dense walks layer t >= 1 when at least half its key space is reached
       "dense_layers_desc": [t for t in range(H - 1, 0, -1) if 2 * int(n[t]) >= key_space]}
(ROOT / "tools" / f"{name}_layers.json").write_text(json.dumps(doc))
print(name, "S", sp.size(), "key space", key_space, "dense layers", len(doc["dense_layers_desc"]))
