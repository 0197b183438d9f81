"""Quick check of the persistent streaming certified pass against the golden digests + timing."""
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import paper_2012_12419_b200 as V  # noqa: E402
from paper_2012_12419_b200 import _native as N  # noqa: E402

golden = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())["cases"]
sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
for name in sys.argv[1:] or ["C3", "C4"]:
    p = V.load_instance(str(ROOT / "tests" / "golden" / "instances" / f"{name.lower()}.txt"))
    sp = V.StateSpace.build_native(V.NativeInstance(p.vcc, bots=p.bots), 10**9)
    for rep in range(3):
        t0 = time.time()
        r = V.run_value_iteration(sp, V.ViOptions(method=N.VCS_METHOD_CERTIFIED))
        g = golden[name]["eps=1e-06"] if name in golden else None
        ok = g is None or (sha(r.values.raw_values()) == g["values_sha"] and
                           sha(r.policy.raw_actions()) == g["actions_sha"])
        print(name, "method", r.values.report.method, "sweeps", r.values.sweeps(), "ok", ok,
              "device_ms %.4f" % r.values.report.sweep_ms, "wall %.1f ms" % ((time.time() - t0) * 1e3),
              flush=True)
