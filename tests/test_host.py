"""Host logic of the product (no GPU): instance parser and validation (io.cpp:51-101,
workload.cpp:35-57), seeded generators vs the reference's own testutil generator, the shard
plan, BlockPartition / SweepBarrier and greedy_reward."""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import pytest

import paper_2012_12419_b200 as V
from paper_2012_12419_b200 import _native as N
from paper_2012_12419_b200.sharded import halo_transfers, shard_plans, sweep_row_end
from cases import FAMILIES, GOLDEN


# ---- parser ---------------------------------------------------------------------------------

def test_parse_canonical_matches_reference_parser(reference):
    p = V.load_instance(str(GOLDEN / "canonical_instance.txt"))
    assert len(p.vcc.clouds) == 11 and len(p.bots) == 11
    assert sum(len(b.tasks) for b in p.bots) == 330
    n = [C.c_int32() for _ in range(3)]
    assert reference.L.ref_load_counts(str(GOLDEN / "canonical_instance.txt").encode(),
                                       *[C.byref(x) for x in n]) == 0
    assert [x.value for x in n] == [11, 330, 11]
    assert all(c.vm_free == c.vm_total for c in p.vcc.clouds)  # io.cpp:71
    assert (p.vcc.reward_per_vc_vm, p.vcc.cost_per_tcc_vm, p.vcc.penalty_per_idle_vm) == (1, 1.2, 1)


@pytest.mark.parametrize("text,msg", [
    ("frobnicate 1\n", "line 1: unknown directive 'frobnicate' in 'frobnicate 1'"),
    ("cloud 1 5 60 10 99\n", "line 1: unexpected trailing field '99' in 'cloud 1 5 60 10 99'"),
    ("task 1 1 10 60\n", "line 1: task before any bot in 'task 1 1 10 60'"),
    ("# c\ncloud 1 x 60 10\n",
     "line 2: expected: cloud <id> <vm_total> <thr> <delay> in 'cloud 1 x 60 10'"),
    ("beta_vc\n", "line 1: expected a value in 'beta_vc'"),
    ("bot 1\ntask 1 0 10 60\n", "task 1: vm_demand < 1"),
    ("bot 1\ntask 7 1 0 60\n", "task 7: requirements must be positive"),
    ("beta_tc -1\n", "rate parameters must be non-negative"),
    ("cloud 3 -2 60 10\n", "cloud 3: vm_total < 0"),
])
def test_parse_errors_match_reference_messages(text, msg):
    with pytest.raises(V.ConfigError) as e:
        V.parse_instance(text)
    assert str(e.value) == msg


@pytest.mark.parametrize("thr,delay", [
    ("60", "10"), ("+60", "-0"), ("007", "1e1"), ("60.", ".5"), ("6.0e1", "1E-3"),
    ("123456789012345", "0.1"), ("1234567890123456789", "2.5e-310"), ("1e400", "10"),
    ("0x10", "10"), ("inf", "10"), ("60x", "10"), ("--1", "10"), ("1e", "10"), ("6-0", "10"),
])
def test_parser_fast_path_matches_reference(reference, thr, delay):
    """Directive lines go through a strtol/strtod fast path when every field is a plain decimal
    number, else through the stream extraction; either way the instance (or the error message)
    is the reference parser's: same doubles bit for bit, same diagnostics."""
    txt = (f"beta_vc {delay}\ncloud 1 5 {thr} {delay}\ncloud +2 007 {thr} 20\nbot 1\n"
           f"task 1 2 {thr} {delay}\ntask -3 1 30 60\n")
    try:
        ref = reference.parse(txt).text()
    except Exception as e:  # noqa: BLE001
        with pytest.raises(V.ConfigError) as ours:
            V.parse_instance(txt)
        assert str(ours.value) in str(e), (str(ours.value), str(e))
        return
    assert V.instance_text(V.parse_instance(txt)) == ref


def test_load_missing_file_is_io_error():
    with pytest.raises(V.IoError, match="cannot read instance file: /nonexistent/x.txt"):
        V.load_instance("/nonexistent/x.txt")


def test_comments_and_blank_lines_are_skipped():
    p = V.parse_instance("  # leading comment\n\n   \nbeta_vc 2\ncloud 4 3 90 20\nbot 9\n"
                         "task 5 2 30 80\n")
    assert p.vcc.reward_per_vc_vm == 2.0
    assert p.vcc.clouds[0] == V.VehicularCloud(4, 3, 3, 90.0, 20.0)
    assert p.bots[0].id == 9 and p.bots[0].tasks[0] == V.Task(5, 2, 30.0, 80.0)


# ---- generators ----------------------------------------------------------------------------

def _ref_random(reference, seed, trial, a, b, c, d):
    f = reference.L.ref_random_instance
    I32 = C.POINTER(C.c_int32)
    F64 = C.POINTER(C.c_double)
    f.restype = C.c_int
    f.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, I32, I32, F64,
                  F64, I32, I32, I32, F64, F64, I32, I32]
    nc, nt, nb = C.c_int32(), C.c_int32(), C.c_int32()
    cap = np.zeros(a, np.int32)
    cd, ct = np.zeros(a), np.zeros(a)
    tid, td = np.zeros(c, np.int32), np.zeros(c, np.int32)
    tdl, tth = np.zeros(c), np.zeros(c)
    bs = np.zeros(3, np.int32)
    p = lambda x, t: x.ctypes.data_as(C.POINTER(t))  # noqa: E731
    assert f(seed, trial, a, b, c, d, C.byref(nc), p(cap, C.c_int32), p(cd, C.c_double),
             p(ct, C.c_double), C.byref(nt), p(tid, C.c_int32), p(td, C.c_int32),
             p(tdl, C.c_double), p(tth, C.c_double), C.byref(nb), p(bs, C.c_int32)) == 0
    k, t, b_ = nc.value, nt.value, nb.value
    return dict(cloud_vm_total=cap[:k], cloud_delay=cd[:k], cloud_thr=ct[:k], task_id=tid[:t],
                task_demand=td[:t], task_max_delay=tdl[:t], task_min_thr=tth[:t],
                bot_sizes=bs[:b_])


@pytest.mark.parametrize("family", list(FAMILIES.keys()))
def test_random_generator_matches_reference_testutil(reference, family):
    seed, params, n, _ = FAMILIES[family]
    for trial in range(min(n, 60)):
        ni = V.generate_instance(N.VCS_GEN_RANDOM, seed, trial, *params, as_objects=False)
        got = ni.arrays()
        want = _ref_random(reference, seed, trial, *params)
        for key in ("cloud_vm_total", "cloud_delay", "cloud_thr", "task_id", "task_demand",
                    "task_max_delay", "task_min_thr"):
            assert np.array_equal(got[key], want[key]), (trial, key)
        assert np.array_equal(np.diff(got["bot_off"]), want["bot_sizes"])
        assert np.array_equal(got["cloud_vm_free"], got["cloud_vm_total"])


def test_homog_and_greedy_generators_shape():
    c3 = V.generate_instance(N.VCS_GEN_HOMOG, 2012, 0, 5, 8, 40, 3, as_objects=False).arrays()
    assert len(c3["cloud_id"]) == 5 and len(c3["task_id"]) == 40
    assert set(np.unique(c3["task_demand"])) <= {1, 2, 3}
    assert np.all(c3["cloud_vm_total"] == 8)
    # round-robin deal into 5 bags: bag b holds task ids b+1, b+6, ...
    assert list(c3["task_id"][:8]) == [1, 6, 11, 16, 21, 26, 31, 36]
    c2 = V.generate_instance(N.VCS_GEN_GREEDY, 12345, 0, 1000, 100, 1000, 3,
                             as_objects=False).arrays()
    assert len(c2["cloud_id"]) == 1000 and len(c2["task_id"]) == 100000
    assert int(c2["cloud_vm_total"].sum()) == 98991  # = placed + unused of the golden run


# ---- bench workloads: both arms read the same instance ------------------------------------

@pytest.mark.parametrize("name,args", [("c3", (5, 8, 40, 3)), ("c4", (6, 8, 48, 3))])
def test_committed_instance_files_match_generators(reference, name, args):
    """tests/golden/instances/cN.txt = the product generator's instance, and the reference's own
    parser reads it back to the same text the reference's restated generator writes."""
    import bench_workloads as W
    prod = V.generate_instance(N.VCS_GEN_HOMOG, 2012, 0, *args)
    body = W.instance_text(name).split("\n", 2)[2]  # drop the two comment lines
    assert V.instance_text(prod) == body
    via_ref_parser = reference.load(W.FILES[name]).text()
    via_ref_gen = reference.generate(N.VCS_GEN_HOMOG, 2012, *args).text()
    assert via_ref_parser == via_ref_gen == body
    assert V.instance_text(V.load_instance(str(W.FILES[name]))) == body


def test_c2_generator_restatement_matches_product(reference):
    import bench_workloads as W
    kind, seed, a, b, c, d = W.C2_GEN
    prod = V.generate_instance(kind, seed, 0, a, b, c, d)
    assert V.instance_text(prod) == reference.generate(kind, seed, a, b, c, d).text()


def test_c5_points_parse_identically(reference):
    """Every C5 point parses to the same instance in both arms' parsers; the channel variants
    really differ (the scheme changes at least one cloud's throughput on most points)."""
    import bench_workloads as W
    table = W.channel_table()
    differ = 0
    for K, c, scheme in W.c5_points():
        txt = W.c5_text(K, c, scheme, table)
        ours = V.instance_text(V.parse_instance(txt))
        assert ours == reference.parse(txt).text(), (K, c, scheme)
        if scheme == "aaa":
            differ += W.c5_text(K, c, "static1609", table).split("bot", 1)[0] != txt.split("bot", 1)[0]
    assert differ >= 30


def test_c5_channel_table_is_the_reference_simulator(reference):
    import bench_workloads as W
    table = W.channel_table()
    for n in (5, 15, 20, 28, 35, 84):
        for scheme, k in (("static1609", 0), ("aaa", 1)):
            out = C.c_double()
            assert reference.L.ref_per_vehicle_kbps(n, k, 42, 10_000, C.byref(out)) == 0
            assert out.value == table[scheme][n - 1]
    # static 120/96/72/57.6 kbps at 10/15/20/25 vehicles, AAA 120/120/96.6/69.12
    assert [round(table["static1609"][n - 1], 2) for n in (10, 15, 20, 25)] == [120, 96, 72, 57.6]
    assert [round(table["aaa"][n - 1], 2) for n in (10, 15, 20, 25)] == [120, 120, 96.6, 69.12]


def test_generator_rejects_bad_kind():
    with pytest.raises(V.InvalidArgument):
        V.generate_instance(7, 1)


# ---- shard plan ----------------------------------------------------------------------------

@pytest.mark.parametrize("case", ["canonical", "c3"])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_plan_covers_and_halo_contains_successors(oracle, case, world):
    if case == "canonical":
        p = V.load_instance(str(GOLDEN / "canonical_instance.txt"))
        ni = V.NativeInstance(p.vcc, bots=p.bots)
    else:
        ni = V.generate_instance(N.VCS_GEN_HOMOG, 2012, 0, 5, 8, 40, 3, as_objects=False)
    sp = oracle.build(ni.ref, 10**9)
    lo, rp, su, _, _ = sp.csr()
    le = np.array([rp[lo[t + 1]] - rp[lo[t]] for t in range(sp.H + 1)], np.uint64)
    for skip_weighted in (False, True):
        plans = shard_plans(lo, le, world, skip_weighted)
        assert plans[0].row_begin == 0 and plans[-1].row_end == sp.S
        for a, b in zip(plans, plans[1:]):
            assert a.row_end == b.row_begin
        for pl in plans:
            if pl.row_end == pl.row_begin:
                continue
            e0, e1 = int(rp[pl.row_begin]), int(rp[pl.row_end])
            succ = su[e0:e1].astype(np.int64)
            outside = succ[succ >= pl.row_end]
            assert np.all(succ > pl.row_begin)  # successors live in later layers
            if outside.size:
                assert outside.min() >= pl.halo_begin and outside.max() < pl.halo_end
            # the halo never exceeds one layer past the block's last layer
            assert pl.halo_end - pl.halo_begin <= 2 * int(np.max(np.diff(lo)))
    # balance (the plan interpolates inside a layer assuming its mean degree): every block
    # within 3% of an equal share of the sweep bytes
    cost = 24 * sp.S + 12 * sp.E
    plans = shard_plans(lo, le, world, False)
    for pl in plans:
        c = 24 * (pl.row_end - pl.row_begin) + 12 * int(rp[pl.row_end] - rp[pl.row_begin])
        assert c <= cost / world * 1.03 + 24 + 12 * 64


def test_halo_transfers_are_clipped_to_changed_rows():
    lo = np.array([0, 1, 4, 10, 20, 21], np.uint64)
    le = np.array([3, 12, 20, 10, 0], np.uint64)
    plans = shard_plans(lo, le, 3)
    full = halo_transfers(plans, int(lo[-1]))
    for src, dst, b, e in full:
        assert plans[src].row_begin <= b < e <= plans[src].row_end
        assert plans[dst].halo_begin <= b and e <= plans[dst].halo_end
    assert halo_transfers(plans, 0) == []
    assert sweep_row_end(lo, 1, True) == 21 and sweep_row_end(lo, 2, True) == 20
    assert sweep_row_end(lo, 5, True) == 1 and sweep_row_end(lo, 6, True) == 0
    assert sweep_row_end(lo, 3, False) == 21


# ---- parallel_vi.hpp utilities -------------------------------------------------------------

def test_block_partition_even():
    """test_parallel.cpp:18-40 restated."""
    for n in (0, 1, 7, 100, 1001):
        for blocks in (1, 2, 4, 8):
            part = V.BlockPartition.even(n, blocks)
            assert len(part.ranges) == blocks
            begin, lens = 0, []
            for lo, hi in part.ranges:
                assert lo == begin
                begin = hi
                lens.append(hi - lo)
            assert sum(lens) == n and max(lens) - min(lens) <= 1
            if n > 0:
                assert part.block_of(n - 1) == min(blocks, n) - 1
    with pytest.raises(V.InvalidArgument):
        V.BlockPartition.even(10, 0)


def test_sweep_barrier_generations():
    """test_parallel.cpp:42-62 restated."""
    workers, rounds = 4, 50
    barrier = V.SweepBarrier(workers)
    lock = threading.Lock()
    state = {"in": 0, "torn": False}

    def body():
        for _ in range(rounds):
            with lock:
                state["in"] += 1
            barrier.arrive_and_wait()
            with lock:
                if state["in"] % workers:
                    state["torn"] = True
            barrier.arrive_and_wait()

    ts = [threading.Thread(target=body) for _ in range(workers)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not state["torn"] and state["in"] == workers * rounds


def test_greedy_reward_formula():
    """test_greedy.cpp:455-470."""
    r = V.ScheduleResult(paid_vms=10)
    assert V.greedy_reward(r, V.VccModel([], 1.0, 1.2, 1.0)) == pytest.approx(-12.0)
    sizes = [5, 7, 10, 15, 20, 25, 28, 35, 40, 42, 45]
    vcc = V.VccModel([V.VehicularCloud(i + 1, s, s, 100.0, 10.0) for i, s in enumerate(sizes)])
    perfect = V.ScheduleResult(per_vc_used={i + 1: s for i, s in enumerate(sizes)})
    assert V.greedy_reward(perfect, vcc) == pytest.approx(272.0)
    ni = V.NativeInstance(vcc, bots=[])
    assert N.lib().vcs_greedy_reward(ni.ref, 272, 0, 0) == 272.0


def test_full_state_helpers():
    """transition / legal_actions / step_reward, test_mdp.cpp:31-63."""
    from cases import tiny
    vcc, bots = tiny(5, [5])
    inst = V.MdpInstance.from_workload(vcc, bots)
    s0 = V.initial_state(inst)
    drained = V.transition(s0, V.MdpAction(0), inst)
    assert drained.free_vms == [0] and drained.next_task_index == 1 and drained.terminal
    paid = V.transition(s0, V.MdpAction(V.kPaidCloud), inst)
    assert paid.free_vms == [5] and paid.terminal
    with pytest.raises(V.InvalidArgument, match="transition from terminal state"):
        V.transition(drained, V.MdpAction(V.kPaidCloud), inst)
    vcc, bots = tiny(3, [5])
    inst = V.MdpInstance.from_workload(vcc, bots)
    with pytest.raises(V.InvalidArgument):
        V.transition(V.initial_state(inst), V.MdpAction(0), inst)
    acts = V.legal_actions(inst, V.initial_state(inst))
    assert len(acts) == 1 and acts[0].is_paid()
    vcc, bots = tiny(10, [5, 10])
    inst = V.MdpInstance.from_workload(vcc, bots)
    s0 = V.initial_state(inst)
    s1 = V.transition(s0, V.MdpAction(0), inst)
    assert V.step_reward(s0, V.MdpAction(0), s1, inst) == pytest.approx(5.0)
    s2 = V.transition(s1, V.MdpAction(V.kPaidCloud), inst)
    assert V.step_reward(s1, V.MdpAction(V.kPaidCloud), s2, inst) == pytest.approx(-12.0)


def test_speedup_csv_format():
    """io.cpp:351-357: header, then workers,wall_ms,speedup_vs_one with %.17g doubles."""
    rows = [V.SpeedupRow(1, 12.5, 1.0), V.SpeedupRow(8, 0.1, 125.0), V.SpeedupRow(2, 1 / 3, 37.5)]
    assert V.speedup_csv(rows) == ("workers,wall_ms,speedup_vs_one\n1,12.5,1\n8,0.10000000000000001,125\n"
                                   "2,0.33333333333333331,37.5\n")
    assert V.speedup_csv([]) == "workers,wall_ms,speedup_vs_one\n"
