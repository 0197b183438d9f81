"""Developer check on a GPU box: builder/solver/greedy parity vs the C oracle + rough timings.

Usage: python tools/gpu_quick.py [c4]
"""
import sys
import time
import traceback
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2012_12419_b200 as V  # noqa: E402
from paper_2012_12419_b200 import _native as N  # noqa: E402
from oracle_bind import Oracle  # noqa: E402

orc = Oracle()


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64 if a.dtype == np.float64 else a.dtype)


def check_space(name, ni, cap=10**9, eps_list=(1e-6,), workers=8):
    t0 = time.time()
    sp = V.StateSpace.build_native(ni, cap)
    t_build = time.time() - t0
    os_ = orc.build(ni.ref, cap)
    lo, rp, su, rw, ac = os_.csr()
    grp, gsu, grw, gac = sp.csr()
    ok_csr = (np.array_equal(lo, sp.layer_offsets()) and np.array_equal(rp, grp)
              and np.array_equal(su, gsu) and np.array_equal(bits(rw), bits(grw))
              and np.array_equal(ac, gac))
    print(f"[{name}] S={sp.size()} E={sp.edges()} H={sp.task_count()} build {t_build*1e3:.1f} ms "
          f"(dev {sp.info.build_ms:.1f}) csr_equal={ok_csr}")
    if not ok_csr:
        for nm, x, y in (("layers", lo, sp.layer_offsets()), ("row_ptr", rp, grp), ("succ", su, gsu),
                         ("reward", bits(rw), bits(grw)), ("action", ac, gac)):
            if not np.array_equal(x, y):
                bad = np.nonzero(x != y)[0] if len(x) == len(y) else None
                print("   mismatch", nm, len(x), len(y), bad[:10] if bad is not None else "len")
    for eps in eps_list:
        for skip in (True, False):
            opts = V.ViOptions(epsilon=eps, skip_converged=skip)
            r = V.run_value_iteration(sp, opts)
            v, a, sw, tsw, tex = os_.vi(eps=eps, workers=workers)
            rep = r.values.report
            ok = (np.array_equal(bits(v), bits(r.values.raw_values()))
                  and np.array_equal(a, r.policy.raw_actions()) and sw == r.values.sweeps())
            bps = rep.backups_ref / (rep.sweep_ms * 1e-3) if rep.sweep_ms > 0 else 0
            gbs = rep.alg_bytes_done / (rep.sweep_ms * 1e-3) / 1e9 if rep.sweep_ms > 0 else 0
            print(f"   eps={eps:g} skip={skip} sweeps gpu={r.values.sweeps()} orc={sw} parity={ok} "
                  f"sweep_ms={rep.sweep_ms:.3f} extract_ms={rep.extract_ms:.3f} "
                  f"backups/s={bps:.3e} alg_GB/s(done)={gbs:.1f} cpu_ms={tsw:.1f}")
    # warm timing
    r = V.run_value_iteration(sp, V.ViOptions())
    rep = r.values.report
    print(f"   warm: sweep_ms={rep.sweep_ms:.3f} extract_ms={rep.extract_ms:.3f}")
    return sp


def main():
    print("devices:", N.device_count())
    try:
        p = V.load_instance(str(ROOT / "tests" / "golden" / "canonical_instance.txt"))
        inst = V.MdpInstance.from_workload(p.vcc, p.bots)
        ni = inst.native()
        sp = check_space("canonical", ni, eps_list=(1e-6, 5.0), workers=1)
        r = V.value_iteration(inst)
        print("   V0", r.values.initial_value())
        ro = V.rollout(r.policy, inst)
        print("   rollout paid", ro.paid_vms, "unused", ro.unused_vms, "reward",
              V.greedy_reward(ro, p.vcc))
    except Exception:
        traceback.print_exc()
    for trial in range(5):
        try:
            g = V.generate_instance(N.VCS_GEN_RANDOM, 3003, trial, 4, 5, 25, 3, as_objects=False)
            check_space(f"rand3003#{trial}", g, workers=1)
        except Exception:
            traceback.print_exc()
    try:
        c3 = V.generate_instance(N.VCS_GEN_HOMOG, 2012, 0, 5, 8, 40, 3, as_objects=False)
        check_space("C3", c3)
    except Exception:
        traceback.print_exc()
    if "c4" in sys.argv:
        try:
            c4 = V.generate_instance(N.VCS_GEN_HOMOG, 2012, 0, 6, 8, 48, 3, as_objects=False)
            check_space("C4", c4)
        except Exception:
            traceback.print_exc()
    try:
        for nm, ni, T, K in (("canon-greedy", ni, 330, 11),):
            pass
        p = V.load_instance(str(ROOT / "tests" / "golden" / "canonical_instance.txt"))
        nic = V.NativeInstance(p.vcc, bots=p.bots)
        g = V.greedy_schedule(p.vcc, p.bots, native=nic)
        o = orc.greedy(nic.ref, 330, 11)
        print("[greedy canonical] paid", g.paid_vms, "unused", g.unused_vms, "reward",
              V.greedy_reward(g, p.vcc), "targets_equal", np.array_equal(g.target_index, o[0]))
        c2 = V.generate_instance(N.VCS_GEN_GREEDY, 12345, 0, 1000, 100, 1000, 3, as_objects=False)
        for rep in range(3):
            t0 = time.time()
            tgt = np.empty(100000, np.int32)
            import ctypes as C
            paid, unused = C.c_int64(), C.c_int64()
            N.check(N.lib().vcs_greedy(c2.ref, 0, N.ptr(tgt, C.c_int32), None, C.byref(paid),
                                       C.byref(unused)))
            dt = time.time() - t0
        o = orc.greedy(c2.ref, 100000, 1000)
        print(f"[greedy C2] paid={paid.value} unused={unused.value} e2e_ms={dt*1e3:.2f} "
              f"targets_equal={np.array_equal(tgt, o[0])} oracle_ms={o[4]:.1f}")
    except Exception:
        traceback.print_exc()
    print("kernel launches:", N.kernel_launches())


if __name__ == "__main__":
    main()
