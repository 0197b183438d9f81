"""C5 (BASELINE.json configs[4]): the vehicle-count / RSU-coverage density sweep with the two
channel-availability schemes (bench_workloads.c5_text).  Sampled points must reproduce the
reference's golden digests (tests/golden/make_golden.py --c5: the unmodified reference on the
same instance text), and the whole grid must build and solve with the certificate holding."""
from __future__ import annotations

import pytest

import bench_workloads as W
import paper_2012_12419_b200 as V
from conftest import sha

pytestmark = pytest.mark.gpu


def _solve(K, c, scheme, table):
    p = V.parse_instance(W.c5_text(K, c, scheme, table))
    inst = V.MdpInstance.from_workload(p.vcc, p.bots)
    sp = V.StateSpace.build_native(inst.native(), 10**9, 0, inst)
    return sp, inst, V.run_value_iteration(sp, V.ViOptions())


def test_c5_sample_points_match_reference(gpu, golden):
    table = W.channel_table()
    samples = [k for k in golden["cases"] if k.startswith("C5_")]
    assert len(samples) >= 6
    for key in samples:
        _, K, c, scheme = key.split("_", 3)
        K, c = int(K[1:]), int(c[1:])
        sp, inst, r = _solve(K, c, scheme, table)
        g = golden["cases"][key]
        assert sp.size() == g["S"], key
        e = g["eps=1e-06"]
        assert r.values.sweeps() == e["sweeps"], key
        assert sha(r.values.raw_values()) == e["values_sha"], key
        assert sha(r.policy.raw_actions()) == e["actions_sha"], key
        ro = V.rollout(r.policy, inst)
        assert (ro.paid_vms, ro.unused_vms) == (e["rollout_paid"], e["rollout_unused"]), key
        assert sha(ro.target_index) == e["rollout_targets_sha"], key


def test_c5_grid_solves(gpu):
    """Every point of the 5 x 9 x 2 grid: built, solved, V(initial) finite and the sweep count
    within the layered bound (certified or not, the result is the reference's by the parity
    tests above)."""
    table = W.channel_table()
    sizes = {}
    for K, c, scheme in W.c5_points():
        sp, inst, r = _solve(K, c, scheme, table)
        assert 1 <= r.values.sweeps() <= sp.task_count() + 1
        v0 = r.values.initial_value()
        assert v0 == v0 and abs(v0) < 1e9
        sizes[(K, c, scheme)] = sp.size()
    # the channel scheme changes the state space on part of the grid
    assert sum(sizes[(K, c, "aaa")] != sizes[(K, c, "static1609")]
               for K in W.C5_CLOUDS for c in W.C5_VMS) >= 15
