"""Generate tests/golden/golden.json from the UNMODIFIED reference (oracle/_ref/libvcsref.so).

Run here (the container that has /root/reference):  python tests/golden/make_golden.py
The JSON holds, per case, the reference's state count, layer offsets digest, sweep count,
sha256 of raw_values (f64 LE) and raw_actions (i32 LE), V(initial), rollout and greedy outcomes,
and testutil::brute_force_optimum where the reference tests use it.  GPU tests on the box (where
/root/reference does not exist) compare against these digests.
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2012_12419_b200 as V  # noqa: E402
from paper_2012_12419_b200 import _native as N  # noqa: E402
from cases import FAMILIES, named_cases  # noqa: E402
from oracle_bind import Reference  # noqa: E402
import ctypes as C  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def brute(ref: Reference, ni) -> float:
    f = ref.L.ref_brute_force
    f.restype = C.c_int
    f.argtypes = [C.POINTER(N.vcs_instance), C.POINTER(C.c_double)]
    out = C.c_double()
    assert f(ni.ref, C.byref(out)) == 0
    return out.value


def record(ref: Reference, ni, eps_list=(1e-6,), cap=10**9, with_brute=False):
    s = ni.struct
    rec = {"n_clouds": s.n_clouds, "n_tasks": s.n_tasks}
    t0 = time.time()
    sp = ref.build(ni.ref, cap)
    rec["S"] = sp.S
    rec["layers_sha"] = sha(sp.layers())
    rec["ref_build_ms"] = sp.build_ms
    for eps in eps_list:
        r = sp.vi(eps=eps, workers=1 if sp.S < 2_000_000 else 8)
        key = f"eps={eps:g}"
        ro = r.rollout(s.n_tasks, s.n_clouds)
        rec[key] = {
            "sweeps": r.sweeps,
            "values_sha": sha(r.values()),
            "actions_sha": sha(r.actions()),
            "v0": r.initial_value(),
            "v0_hex": float(r.initial_value()).hex(),
            "rollout_paid": ro["paid"], "rollout_unused": ro["unused"],
            "rollout_reward": ro["reward"], "rollout_targets_sha": sha(ro["targets"]),
            "ref_vi_ms": r.ms,
        }
    g = ref.greedy(ni.ref, s.n_tasks)
    ids = np.ctypeslib.as_array(s.cloud_id, shape=(s.n_clouds,)) if s.n_clouds else np.zeros(0)
    idx = {int(c): i for i, c in reversed(list(enumerate(ids)))}
    tgt_index = np.array([idx[int(t)] if t >= 0 else -1 for t in g["target_ids"]], np.int32)
    rec["greedy"] = {"paid": g["paid"], "unused": g["unused"], "placed": g["placed"],
                     "reward": g["reward"], "targets_sha": sha(tgt_index)}
    if with_brute:
        rec["brute_force"] = brute(ref, ni)
    rec["gen_s"] = time.time() - t0
    return rec


# C5 points with reference digests (both channel schemes, small to ~0.8 M states)
C5_SAMPLES = ((3, 6, "static1609"), (3, 6, "aaa"), (4, 10, "aaa"), (5, 9, "aaa"),
              (6, 8, "static1609"), (7, 6, "aaa"))


def extra(ref, argv):
    """Add digests to the existing golden.json without regenerating it (--early, --c5)."""
    if "--early" in argv:  # early-stop digests for C3 (eps 3) and C4 (eps 4): the fallback path
        old = json.loads((HERE / "golden.json").read_text())
        for name, eps in (("C3", 3.0), ("C4", 4.0)):
            p = V.load_instance(str(HERE / "instances" / f"{name.lower()}.txt"))
            ni = V.MdpInstance.from_workload(p.vcc, p.bots).native()
            rec = record(ref, ni, eps_list=(eps,))
            old["cases"][name][f"eps={eps:g}"] = rec[f"eps={eps:g}"]
            print(name, eps, rec[f"eps={eps:g}"]["sweeps"], flush=True)
        (HERE / "golden.json").write_text(json.dumps(old, indent=1, sort_keys=True))
        return
    if "--c5" in argv:  # add / refresh only the C5 sample points (bench_workloads.c5_text)
        import bench_workloads as W
        old = json.loads((HERE / "golden.json").read_text())
        table = W.channel_table()
        for K, c, scheme in C5_SAMPLES:
            p = V.parse_instance(W.c5_text(K, c, scheme, table))
            ni = V.MdpInstance.from_workload(p.vcc, p.bots).native()
            old["cases"][f"C5_K{K}_c{c}_{scheme}"] = record(ref, ni)
            print("C5", K, c, scheme, old["cases"][f"C5_K{K}_c{c}_{scheme}"]["S"], flush=True)
        (HERE / "golden.json").write_text(json.dumps(old, indent=1, sort_keys=True))
        print("wrote", HERE / "golden.json")
        return


def main(argv):
    ref = Reference()
    if "--early" in argv or "--c5" in argv:
        return extra(ref, argv)
    out = {"generator": "tests/golden/make_golden.py", "reference": "oracle/_ref/libvcsref.so",
           "cases": {}, "families": {}}
    for name, (ni, eps_list) in named_cases().items():
        out["cases"][name] = record(ref, ni, eps_list)
        print(name, out["cases"][name]["S"], flush=True)
    for fam, (seed, params, n, brute_ok) in FAMILIES.items():
        recs = []
        for trial in range(n):
            ni = V.generate_instance(N.VCS_GEN_RANDOM, seed, trial, *params, as_objects=False)
            recs.append(record(ref, ni, with_brute=brute_ok))
        out["families"][fam] = recs
        print(fam, len(recs), flush=True)
    if "--big" in argv:
        for name, args in (("C3", (2012, 0, 5, 8, 40, 3)), ("C4", (2012, 0, 6, 8, 48, 3))):
            ni = V.generate_instance(N.VCS_GEN_HOMOG, *args, as_objects=False)
            out["cases"][name] = record(ref, ni)
            print(name, out["cases"][name]["S"], flush=True)
        ni = V.generate_instance(N.VCS_GEN_GREEDY, 12345, 0, 1000, 100, 1000, 3, as_objects=False)
        g = ref.greedy(ni.ref, 100000)
        ids = np.ctypeslib.as_array(ni.struct.cloud_id, shape=(1000,))
        tgt = np.where(g["target_ids"] >= 0, g["target_ids"] - 1, -1).astype(np.int32)
        assert np.array_equal(np.where(tgt >= 0, ids[np.maximum(tgt, 0)], -1), g["target_ids"])
        out["cases"]["C2"] = {"greedy": {"paid": g["paid"], "unused": g["unused"],
                                         "placed": g["placed"], "reward": g["reward"],
                                         "targets_sha": sha(tgt)}, "ref_ms": g["ms"]}
    else:
        old = json.loads((HERE / "golden.json").read_text()) if (HERE / "golden.json").exists() else {}
        for name in ("C3", "C4", "C2"):
            if name in old.get("cases", {}):
                out["cases"][name] = old["cases"][name]
    (HERE / "golden.json").write_text(json.dumps(out, indent=1, sort_keys=True))
    print("wrote", HERE / "golden.json")


if __name__ == "__main__":
    main(sys.argv[1:])
