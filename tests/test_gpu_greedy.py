"""GPU parity of the first-fit placement (greedy.cpp:5-36): placements bit-exact vs the C
oracle and the reference's golden digests; the reference's greedy property tests."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import paper_2012_12419_b200 as V
from paper_2012_12419_b200 import _native as N
from cases import FAMILIES, GOLDEN, named_cases
from conftest import sha

pytestmark = pytest.mark.gpu


def test_canonical_published_outcome(gpu, golden):
    """test_greedy.cpp:37-54 / PAPER.md:655-656."""
    p = V.load_instance(str(GOLDEN / "canonical_instance.txt"))
    r = V.greedy_schedule(p.vcc, p.bots)
    assert (r.paid_vms, r.unused_vms, r.vc_placed_vms()) == (85, 27, 245)
    assert V.greedy_reward(r, p.vcc) == pytest.approx(116.0, rel=1e-12)
    leftovers = {2: 1, 4: 2, 5: 4, 7: 4, 8: 1, 9: 1, 10: 7, 11: 7}
    for c in p.vcc.clouds:
        assert c.vm_total - r.per_vc_used[c.id] == leftovers.get(c.id, 0)
    assert sha(r.target_index) == golden["cases"]["canonical"]["greedy"]["targets_sha"]


@pytest.mark.parametrize("name", list(named_cases().keys()))
def test_named_cases(gpu, oracle, golden, name):
    ni, _ = named_cases()[name]
    s = ni.struct
    r = V.greedy_schedule(None, None, native=ni)
    tgt, used, paid, unused, _ = oracle.greedy(ni.ref, s.n_tasks, s.n_clouds)
    assert np.array_equal(r.target_index, tgt)
    g = golden["cases"][name]["greedy"]
    assert (r.paid_vms, r.unused_vms, r.vc_placed_vms()) == (g["paid"], g["unused"], g["placed"])


@pytest.mark.parametrize("family", list(FAMILIES.keys()))
def test_random_families(gpu, oracle, golden, family):
    seed, params, n, _ = FAMILIES[family]
    for trial in range(n):
        ni = V.generate_instance(N.VCS_GEN_RANDOM, seed, trial, *params, as_objects=False)
        r = V.greedy_schedule(None, None, native=ni)
        assert sha(r.target_index) == golden["families"][family][trial]["greedy"]["targets_sha"]
        g = golden["families"][family][trial]["greedy"]
        assert (r.paid_vms, r.unused_vms) == (g["paid"], g["unused"])


def test_c2_full_size(gpu, oracle, golden):
    """10^5 tasks over 1,000 clouds: placements identical to the reference."""
    ni = V.generate_instance(N.VCS_GEN_GREEDY, 12345, 0, 1000, 100, 1000, 3, as_objects=False)
    r = V.greedy_schedule(None, None, native=ni)
    g = golden["cases"]["C2"]["greedy"]
    assert (r.paid_vms, r.unused_vms, r.vc_placed_vms()) == (g["paid"], g["unused"], g["placed"])
    assert sha(r.target_index) == g["targets_sha"]
    tgt, *_ = oracle.greedy(ni.ref, 100000, 1000)
    assert np.array_equal(r.target_index, tgt)


@pytest.mark.parametrize("n_clouds,n_demand_levels", [(1500, 3), (70, 40), (3000, 25)])
def test_wide_and_generic_paths(gpu, oracle, n_clouds, n_demand_levels):
    """More than 1024 clouds (multi-round ballot) and more than 16 distinct demands (generic
    capacity test) against the oracle."""
    rng = np.random.default_rng(n_clouds)
    clouds = [V.VehicularCloud(i + 1, int(c), int(c), float(t), float(d)) for i, (c, t, d) in
              enumerate(zip(rng.integers(1, 60, n_clouds), rng.integers(60, 161, n_clouds),
                            rng.integers(5, 51, n_clouds)))]
    tasks = [V.Task(j + 1, int(rng.integers(1, n_demand_levels + 1)), float(rng.integers(5, 61)),
                    float(rng.integers(50, 171))) for j in range(4000)]
    vcc = V.VccModel(clouds)
    bots = [V.BagOfTasks(1, tasks)]
    ni = V.NativeInstance(vcc, bots=bots)
    r = V.greedy_schedule(vcc, bots, native=ni)
    tgt, used, paid, unused, _ = oracle.greedy(ni.ref, len(tasks), n_clouds)
    assert np.array_equal(r.target_index, tgt)
    assert (r.paid_vms, r.unused_vms) == (paid, unused)


def test_feasibility_and_prefix_consistency(gpu):
    """test_greedy.cpp:73-111."""
    for trial in range(30):
        p = V.generate_instance(N.VCS_GEN_RANDOM, 17, trial, 5, 8, 25, 3)
        r = V.greedy_schedule(p.vcc, p.bots)
        clouds = {c.id: V.VehicularCloud(c.id, c.vm_total, c.vm_free, c.vm_throughput_kbps,
                                         c.v2i_delay_ms) for c in p.vcc.clouds}
        tasks = V.flatten_tasks(p.bots)
        assert len(r.placements) == len(tasks)
        for rec, t in zip(r.placements, tasks):
            assert rec.vms_used == t.vm_demand
            if rec.target == V.kPaidCloud:
                continue
            assert V.feasible(clouds[rec.target], t)
            clouds[rec.target].vm_free -= rec.vms_used
        assert r.paid_vms + r.vc_placed_vms() == V.total_demand(p.bots)
        assert r.unused_vms == V.total_capacity(p.vcc) - r.vc_placed_vms()
    for trial in range(15):
        p = V.generate_instance(N.VCS_GEN_RANDOM, 19, trial, 4, 6, 15, 2)
        full = V.greedy_schedule(p.vcc, p.bots)
        tasks = V.flatten_tasks(p.bots)
        cut = trial % (len(tasks) + 1)
        part = V.greedy_schedule(p.vcc, [V.BagOfTasks(1, tasks[:cut])])
        for i in range(cut):
            assert part.placements[i].target == full.placements[i].target


def test_batch_matches_single(gpu):
    insts = [V.generate_instance(N.VCS_GEN_RANDOM, 29, t, 5, 8, 30, 3, as_objects=False)
             for t in range(24)]
    insts.append(V.generate_instance(N.VCS_GEN_GREEDY, 7, 0, 200, 10, 100, 3, as_objects=False))
    n = len(insts)
    arr = (N.vcs_instance * n)(*[ni.struct for ni in insts])
    outs = [np.full(max(ni.struct.n_tasks, 1), -7, np.int32) for ni in insts]
    ptrs = (C.POINTER(C.c_int32) * n)(*[o.ctypes.data_as(C.POINTER(C.c_int32)) for o in outs])
    paid = np.zeros(n, np.int64)
    unused = np.zeros(n, np.int64)
    N.check(N.lib().vcs_greedy_batch(n, arr, 0, ptrs, paid.ctypes.data_as(C.POINTER(C.c_int64)),
                                     unused.ctypes.data_as(C.POINTER(C.c_int64))))
    for i, ni in enumerate(insts):
        r = V.greedy_schedule(None, None, native=ni)
        assert np.array_equal(outs[i][:ni.struct.n_tasks], r.target_index)
        assert (paid[i], unused[i]) == (r.paid_vms, r.unused_vms)


@pytest.mark.parametrize("n_tasks,n_clouds,n_levels,cap_hi", [
    (1, 1, 1, 2), (31, 7, 2, 3), (33, 33, 3, 4), (127, 64, 5, 6), (129, 1000, 3, 3),
    (545, 1024, 8, 9), (1000, 5, 2, 40), (5000, 300, 3, 5), (5000, 1024, 8, 12), (4096, 96, 1, 2)])
def test_speculative_chunks_against_oracle(gpu, oracle, n_tasks, n_clouds, n_levels, cap_hi):
    """The chunked first-fit (k_first_fit_spec): task counts across the 32-task chunk, 128-row
    block and 512-row ring (+shadow rows) boundaries, 1..1024 clouds, 1..8 demand levels (every
    template width) and tight capacities (many overflowing chunks, many paid tasks)."""
    rng = np.random.default_rng(n_tasks * 7919 + n_clouds)
    vm = rng.integers(1, cap_hi + 1, n_clouds)
    clouds = [V.VehicularCloud(i + 1, int(c), int(c), float(t), float(d)) for i, (c, t, d) in
              enumerate(zip(vm, rng.integers(60, 161, n_clouds), rng.integers(5, 51, n_clouds)))]
    tasks = [V.Task(j + 1, int(rng.integers(1, n_levels + 1)), float(rng.integers(5, 61)),
                    float(rng.integers(50, 171))) for j in range(n_tasks)]
    vcc = V.VccModel(clouds)
    bots = [V.BagOfTasks(1, tasks)]
    ni = V.NativeInstance(vcc, bots=bots)
    r = V.greedy_schedule(vcc, bots, native=ni)
    tgt, used, paid, unused, _ = oracle.greedy(ni.ref, n_tasks, n_clouds)
    assert np.array_equal(r.target_index, tgt)
    assert (r.paid_vms, r.unused_vms) == (paid, unused)
