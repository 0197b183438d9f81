"""Distinct values per layer of the C4 solution (is a per-layer dictionary worth it on the wire?)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2012_12419_b200 as V  # noqa: E402

ni = V.generate_instance(1, 2012, 0, 6, 8, 48, 3, as_objects=False)
sp = V.StateSpace.build_native(ni, 10**9)
r = V.run_value_iteration(sp, V.ViOptions(epsilon=1e-6))
vals = r.values.raw_values()
off = sp.layer_offsets()
tot_u = 0
for t in range(len(off) - 1):
    v = vals[off[t]:off[t + 1]]
    u = np.unique(v).size
    tot_u += u
    if t % 6 == 0 or t > 44:
        print(f"layer {t}: n={v.size} distinct={u}")
print("total states", vals.size, "distinct per-layer sum", tot_u)
