"""GPU parity: the sm_100a builder and Jacobi solver vs the C oracle and the reference's golden
vectors — bit-exact CSR (succ, fp64 reward bits, action, row_ptr), values (memcmp), policies,
sweep counts; plus the reference's property tests (test_mdp.cpp, test_parallel.cpp)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import paper_2012_12419_b200 as V
from paper_2012_12419_b200 import _native as N
from cases import FAMILIES, GOLDEN, named_cases, named_workloads, tiny
from conftest import bits, sha

pytestmark = pytest.mark.gpu


def _csr_equal(sp, osp):
    lo, rp, su, rw, ac = osp.csr()
    grp, gsu, grw, gac = sp.csr()
    assert np.array_equal(lo, sp.layer_offsets())
    assert np.array_equal(rp, grp)
    assert np.array_equal(su, gsu)
    assert np.array_equal(bits(rw), bits(grw))  # fp64 reward BITS (no FMA contraction)
    assert np.array_equal(ac, gac)


# (method, skip): every solver path must give the same bits
METHODS = [(N.VCS_METHOD_JACOBI, True), (N.VCS_METHOD_JACOBI, False),
           (N.VCS_METHOD_WAVEFRONT, True), (N.VCS_METHOD_CERTIFIED, True)]


def _ran(method):
    """Methods a report may name for a requested method (a failed proof runs the wavefront)."""
    if method == N.VCS_METHOD_CERTIFIED:
        return (N.VCS_METHOD_CERTIFIED, N.VCS_METHOD_WAVEFRONT)
    return (method,)


def _solve(sp, eps=1e-6, skip=True, discount=1.0, method=N.VCS_METHOD_AUTO):
    return V.run_value_iteration(sp, V.ViOptions(epsilon=eps, skip_converged=skip,
                                                 discount=discount, method=method))


@pytest.mark.parametrize("name", list(named_cases().keys()))
def test_named_cases_bitwise(gpu, oracle, golden, name):
    ni, eps_list = named_cases()[name]
    sp = V.StateSpace.build_native(ni, 10**9)
    osp = oracle.build(ni.ref, 10**9)
    _csr_equal(sp, osp)
    rec = golden["cases"][name]
    assert sp.size() == rec["S"]
    assert sha(sp.layer_offsets()) == rec["layers_sha"]
    for eps in eps_list:
        g = rec[f"eps={eps:g}"]
        for method, skip in METHODS:
            r = _solve(sp, eps, skip, method=method)
            assert r.values.report.method in _ran(method)
            assert r.values.sweeps() == g["sweeps"]
            assert sha(r.values.raw_values()) == g["values_sha"]
            assert sha(r.policy.raw_actions()) == g["actions_sha"]


@pytest.mark.parametrize("family", list(FAMILIES.keys()))
def test_random_families_bitwise(gpu, oracle, golden, family):
    seed, params, n, brute = FAMILIES[family]
    for trial in range(n):
        ni = V.generate_instance(N.VCS_GEN_RANDOM, seed, trial, *params, as_objects=False)
        sp = V.StateSpace.build_native(ni, 10**9)
        rec = golden["families"][family][trial]
        assert sp.size() == rec["S"] and sha(sp.layer_offsets()) == rec["layers_sha"]
        g = rec["eps=1e-06"]
        for method, skip in METHODS:
            r = _solve(sp, method=method, skip=skip)
            assert r.values.sweeps() == g["sweeps"], (trial, method)
            assert sha(r.values.raw_values()) == g["values_sha"], (trial, method)
            assert sha(r.policy.raw_actions()) == g["actions_sha"], (trial, method)
        if trial % 7 == 0:  # full CSR check on a sample (the value digests cover the rest)
            _csr_equal(sp, oracle.build(ni.ref, 10**9))


def test_canonical_known_answers(gpu, golden):
    p = V.load_instance(str(GOLDEN / "canonical_instance.txt"))
    inst = V.MdpInstance.from_workload(p.vcc, p.bots)
    r = V.value_iteration(inst)
    g = golden["cases"]["canonical"]["eps=1e-06"]
    assert r.values.initial_value().hex() == g["v0_hex"]
    assert abs(r.values.initial_value() - 202.4) <= 1e-9           # acceptance.cpp:87
    assert r.values.sweeps() == 331 and r.values.states_explored() == 68797
    ro = V.rollout(r.policy, inst)
    assert (ro.paid_vms, ro.unused_vms) == (58, 0)                  # test_mdp.cpp:270-281
    assert abs(V.greedy_reward(ro, p.vcc) - 202.4) <= 1e-9
    assert sha(ro.target_index) == g["rollout_targets_sha"]
    for c in p.vcc.clouds:
        assert ro.per_vc_used[c.id] == c.vm_total                   # 100 % utilization


def test_c3_full_size(gpu, oracle, golden):
    ni = V.generate_instance(N.VCS_GEN_HOMOG, 2012, 0, 5, 8, 40, 3, as_objects=False)
    sp = V.StateSpace.build_native(ni, 10**9)
    assert (sp.size(), sp.edges()) == (1788700, 8478149)
    _csr_equal(sp, oracle.build(ni.ref, 10**9))
    g = golden["cases"]["C3"]["eps=1e-06"]
    for method, skip in METHODS:
        r = _solve(sp, skip=skip, method=method)
        assert r.values.sweeps() == g["sweeps"] == 41
        assert sha(r.values.raw_values()) == g["values_sha"]
        assert sha(r.policy.raw_actions()) == g["actions_sha"]
        assert float(r.values.raw_values()[0]).hex() == (-23.599999999999973).hex()


def test_c4_full_size(gpu, golden):
    """~10^7 states: bit-exact against the reference's digests (no CPU run needed)."""
    ni = V.generate_instance(N.VCS_GEN_HOMOG, 2012, 0, 6, 8, 48, 3, as_objects=False)
    sp = V.StateSpace.build_native(ni, 10**9)
    assert (sp.size(), sp.edges()) == (19333781, 106428994)
    g = golden["cases"]["C4"]
    assert sha(sp.layer_offsets()) == g["layers_sha"]
    for method, skip in METHODS:
        r = _solve(sp, skip=skip, method=method)
        assert r.values.sweeps() == g["eps=1e-06"]["sweeps"] == 49
        assert sha(r.values.raw_values()) == g["eps=1e-06"]["values_sha"]
        assert sha(r.policy.raw_actions()) == g["eps=1e-06"]["actions_sha"]


def test_solver_on_uploaded_oracle_csr(gpu, oracle):
    """The solver alone (vcs_space_from_csr), independent of the device builder."""
    for seed, trial in ((3003, 1), (47, 4), (2002, 5)):
        params = {3003: (4, 5, 25, 3), 47: (4, 6, 25, 3), 2002: (6, 5, 50, 3)}[seed]
        ni = V.generate_instance(N.VCS_GEN_RANDOM, seed, trial, *params, as_objects=False)
        osp = oracle.build(ni.ref)
        lo, rp, su, rw, ac = osp.csr()
        sp = V.StateSpace.from_csr(lo, rp, su, rw, ac)
        for eps in (1e-6, 0.4):
            v, a, sw, _, _ = osp.vi(eps=eps)
            for method, skip in METHODS:
                r = _solve(sp, eps, skip=skip, method=method)
                assert r.values.sweeps() == sw
                assert np.array_equal(bits(r.values.raw_values()), bits(v))
                assert np.array_equal(r.policy.raw_actions(), a)


@pytest.mark.parametrize("discount", [0.9, 0.5])
def test_discounted_extension_matches_oracle(gpu, oracle, discount):
    """LABELLED EXTENSION (no reference counterpart): q = r + gamma*V(s'), separate mul/add."""
    p = V.load_instance(str(GOLDEN / "canonical_instance.txt"))
    ni = V.NativeInstance(p.vcc, bots=p.bots)
    sp = V.StateSpace.build_native(ni)
    osp = oracle.build(ni.ref)
    v, a, sw, _, _ = osp.vi(discount=discount)
    for method, skip in METHODS:
        r = _solve(sp, discount=discount, skip=skip, method=method)
        assert r.values.sweeps() == sw
        assert np.array_equal(bits(r.values.raw_values()), bits(v))
        assert np.array_equal(r.policy.raw_actions(), a)


@pytest.mark.parametrize("discount", [1.0, 0.9, 0.5])
def test_keyspace_certified_against_oracle(gpu, oracle, discount):
    """A dense instance (implicit-CSR build, certified pass by key-space index: k_cert_dense on
    the full layers, DISC and non-DISC kernels) against the oracle, bit for bit, every method."""
    ni = V.generate_instance(N.VCS_GEN_HOMOG, 2012, 0, 4, 6, 20, 3, as_objects=False)
    sp = V.StateSpace.build_native(ni, 10**9)
    osp = oracle.build(ni.ref, 10**9)
    v, a, sw, _, _ = osp.vi(discount=discount)
    for method, skip in METHODS:
        r = _solve(sp, discount=discount, skip=skip, method=method)
        if method == N.VCS_METHOD_CERTIFIED:  # the key-space pass itself, not the fallback
            assert r.values.report.method == N.VCS_METHOD_CERTIFIED
        assert r.values.sweeps() == sw
        assert np.array_equal(bits(r.values.raw_values()), bits(v))
        assert np.array_equal(r.policy.raw_actions(), a)
    # retiring clouds (random attributes): the retired-VM reward from the digits
    for trial in range(3):
        ni = V.generate_instance(N.VCS_GEN_RANDOM, 41, trial, 5, 6, 18, 3, as_objects=False)
        sp = V.StateSpace.build_native(ni, 10**9)
        osp = oracle.build(ni.ref, 10**9)
        v, a, sw, _, _ = osp.vi(discount=discount)
        r = _solve(sp, discount=discount, method=N.VCS_METHOD_CERTIFIED)
        assert r.values.sweeps() == sw
        assert np.array_equal(bits(r.values.raw_values()), bits(v))
        assert np.array_equal(r.policy.raw_actions(), a)


def test_capped_sweeps_match_oracle(gpu, oracle):
    """max_sweeps caps (bench sampling): both methods return V_M of the capped Jacobi run."""
    p = V.load_instance(str(GOLDEN / "canonical_instance.txt"))
    ni = V.NativeInstance(p.vcc, bots=p.bots)
    sp = V.StateSpace.build_native(ni)
    osp = oracle.build(ni.ref)
    import ctypes as C
    for cap in (1, 7, 150):
        v, a, sw, _, _ = osp.vi(max_sweeps=cap)
        for method, skip in METHODS:
            opts = N.vcs_solve_opts(1e-6, 1 if skip else 0, cap, 1.0, method)
            vals = np.empty(sp.size())
            acts = np.empty(sp.size(), np.int32)
            rep = N.vcs_solve_report()
            N.check(N.lib().vcs_solve(sp.handle, C.byref(opts), N.ptr(vals, C.c_double),
                                      N.ptr(acts, C.c_int32), C.byref(rep)))
            assert rep.sweeps == sw == cap
            assert np.array_equal(bits(vals), bits(v)), (cap, method, skip)
            assert np.array_equal(acts, a)


@pytest.mark.parametrize("method", ["WAVEFRONT", "AUTO"])
@pytest.mark.parametrize("narrow", [True, False])
@pytest.mark.parametrize("streamed", [True, False])
def test_pinned_outputs_overlapped_download(gpu, golden, monkeypatch, method, narrow, streamed):
    """vcs_solve into PINNED host buffers: streamed (VCS_STREAM_MIN_MB=0 forces the path the
    results >= 32 MB take: pieces behind the layer events, int8 action column widened on the
    host, or int32 with VCS_NO_NARROW) or in one copy after the pass; an early stop (eps = 5,
    0.5) rewrites a prefix afterwards (AUTO: after the certified pass's fallback) — all must be
    exact."""
    import torch
    if not narrow:
        monkeypatch.setenv("VCS_NO_NARROW", "1")
    if streamed:
        monkeypatch.setenv("VCS_STREAM_MIN_MB", "0")
    p = V.load_instance(str(GOLDEN / "canonical_instance.txt"))
    ni = V.NativeInstance(p.vcc, bots=p.bots)
    sp = V.StateSpace.build_native(ni)
    S = sp.size()
    vals = torch.empty(S, dtype=torch.float64, pin_memory=True)
    acts = torch.empty(S, dtype=torch.int32, pin_memory=True)
    vp = C.cast(C.c_void_p(vals.data_ptr()), C.POINTER(C.c_double))
    ap = C.cast(C.c_void_p(acts.data_ptr()), C.POINTER(C.c_int32))
    for eps in (1e-6, 5.0, 0.5):
        g = golden["cases"]["canonical"][f"eps={eps:g}"]
        for _ in range(2):  # first solve captures the graph, the second replays it
            vals.fill_(float("nan"))
            acts.fill_(-7)
            opts = N.vcs_solve_opts(eps, 1, 0, 1.0, getattr(N, f"VCS_METHOD_{method}"))
            rep = N.vcs_solve_report()
            N.check(N.lib().vcs_solve(sp.handle, C.byref(opts), vp, ap, C.byref(rep)))
            assert rep.sweeps == g["sweeps"]
            assert sha(vals.numpy()) == g["values_sha"]
            assert sha(acts.numpy()) == g["actions_sha"]


def test_state_cap_error(gpu):
    """test_mdp.cpp:248-259."""
    vcc, bots = tiny(6, [1] * 6)
    with pytest.raises(V.StateCapacityError) as e:
        V.value_iteration(V.MdpInstance.from_workload(vcc, bots), V.ViOptions(state_cap=3))
    assert e.value.cap() == 3 and "3" in str(e.value)
    assert str(e.value) == "reachable state space exceeds cap of 3 states"


def test_free_count_limit(gpu):
    vcc = V.VccModel([V.VehicularCloud(1, 70000, 70000, 100.0, 10.0)])
    bots = [V.BagOfTasks(1, [V.Task(1, 1, 50.0, 50.0)])]
    with pytest.raises(V.InvalidArgument, match="cloud free counts above 65535 are not supported"):
        V.value_iteration(V.MdpInstance.from_workload(vcc, bots))


def test_epsilon_must_be_positive(gpu):
    vcc, bots = tiny(2, [1])
    with pytest.raises(V.InvalidArgument, match="epsilon must be > 0"):
        V.value_iteration(V.MdpInstance.from_workload(vcc, bots), V.ViOptions(epsilon=0.0))


def test_terminal_values_and_lookups(gpu):
    """test_mdp.cpp:65-72 and :261-268."""
    vcc, bots = tiny(27, [27])
    inst = V.MdpInstance.from_workload(vcc, bots)
    vi = V.value_iteration(inst)
    assert vi.values.value_of(V.MdpState([27], 1, True)) == pytest.approx(-27.0)
    assert vi.values.value_of(V.MdpState([0], 1, True)) == pytest.approx(0.0)
    vcc, bots = tiny(2, [1])
    inst = V.MdpInstance.from_workload(vcc, bots)
    vi = V.value_iteration(inst)
    with pytest.raises(V.OutOfRange):
        vi.policy.action_for(V.MdpState([2], 1, True))
    with pytest.raises(V.OutOfRange):
        vi.policy.action_for(V.MdpState([1], 0, False))


def test_tie_breaks(gpu):
    """test_mdp.cpp:74-106."""
    w = named_workloads()
    vcc, bots, _ = w["tie_single_paid"]
    inst = V.MdpInstance.from_workload(vcc, bots)
    vi = V.value_iteration(inst)
    val, act = V.bellman_backup(V.initial_state(inst), vi.values, inst)
    assert val == pytest.approx(-1.2) and act.is_paid()
    vcc, bots, _ = w["tie_two_branch"]
    inst = V.MdpInstance.from_workload(vcc, bots)
    vi = V.value_iteration(inst)
    val, act = V.bellman_backup(V.initial_state(inst), vi.values, inst)
    assert val == pytest.approx(1.0) and act == V.MdpAction(0)
    vcc, bots, _ = w["tie_symmetric"]
    inst = V.MdpInstance.from_workload(vcc, bots)
    vi = V.value_iteration(inst)
    val, act = V.bellman_backup(V.initial_state(inst), vi.values, inst)
    assert act == V.MdpAction(0)
    assert vi.policy.action_for(V.initial_state(inst)) == V.MdpAction(0)


def test_empty_task_list(gpu):
    """test_mdp.cpp:108-116."""
    vcc = V.VccModel([V.VehicularCloud(1, 4, 4, 100.0, 10.0)])
    inst = V.MdpInstance.from_workload(vcc, [])
    vi = V.value_iteration(inst)
    assert vi.values.sweeps() == 1
    assert vi.values.initial_value() == 0.0
    assert V.rollout(vi.policy, inst).placements == []


def test_full_state_reference_walks(gpu, reference):
    """test_mdp.cpp:126-156: value_of / action_for along random trajectories vs the
    reference's memoised full-state recursion (testutil::FullStateReference)."""
    f = reference.L.ref_full_state
    f.restype = C.c_int
    f.argtypes = [C.POINTER(N.vcs_instance), C.POINTER(C.c_int32), C.c_int32,
                  C.POINTER(C.c_double), C.POINTER(C.c_int32)]
    rng = np.random.default_rng(61)
    for trial in range(12):
        p = V.generate_instance(N.VCS_GEN_RANDOM, 61, trial, 3, 6, 10, 3)
        inst = V.MdpInstance.from_workload(p.vcc, p.bots)
        ni = V.NativeInstance(p.vcc, bots=p.bots)
        vi = V.value_iteration(inst)

        def ref_value(s):
            fv = np.array(s.free_vms, np.int32)
            out, act = C.c_double(), C.c_int32()
            t = s.next_task_index
            assert f(ni.ref, fv.ctypes.data_as(C.POINTER(C.c_int32)), t, C.byref(out),
                     C.byref(act)) == 0
            return out.value

        for walk in range(3):
            s = V.initial_state(inst)
            while True:
                assert vi.values.value_of(s) == pytest.approx(ref_value(s), rel=1e-12, abs=1e-12)
                if s.terminal:
                    break
                chosen = vi.policy.action_for(s)
                after = V.transition(s, chosen, inst)
                q = V.step_reward(s, chosen, after, inst) + ref_value(after)
                assert q == pytest.approx(ref_value(s), rel=1e-12, abs=1e-12)
                acts = V.legal_actions(inst, s)
                step = chosen if walk == 0 or rng.random() < 0.5 else acts[rng.integers(len(acts))]
                s = V.transition(s, step, inst)


def test_one_step_optimality_and_rollout(gpu):
    """test_mdp.cpp:158-180 and :204-214."""
    rng = np.random.default_rng(67)
    for trial in range(10):
        p = V.generate_instance(N.VCS_GEN_RANDOM, 67, trial, 3, 6, 12, 3)
        inst = V.MdpInstance.from_workload(p.vcc, p.bots)
        vi = V.value_iteration(inst)
        s = V.initial_state(inst)
        while not s.terminal:
            value, action = V.bellman_backup(s, vi.values, inst)
            assert value == pytest.approx(vi.values.value_of(s), rel=1e-12, abs=1e-12)
            acts = V.legal_actions(inst, s)
            s = V.transition(s, acts[rng.integers(len(acts))], inst)
        ro = V.rollout(vi.policy, inst)
        assert V.greedy_reward(ro, p.vcc) == pytest.approx(vi.values.initial_value(), rel=1e-12)


def test_scale_covariance_bitwise(gpu):
    """test_mdp.cpp:216-236: doubling every rate doubles V0 exactly, same raw actions."""
    for trial in range(10):
        p = V.generate_instance(N.VCS_GEN_RANDOM, 37, trial, 3, 6, 12, 3)
        inst = V.MdpInstance.from_workload(p.vcc, p.bots)
        vcc2 = V.VccModel(p.vcc.clouds, 2 * p.vcc.reward_per_vc_vm, 2 * p.vcc.cost_per_tcc_vm,
                          2 * p.vcc.penalty_per_idle_vm)
        inst2 = V.MdpInstance.from_workload(vcc2, p.bots)
        a, b = V.value_iteration(inst), V.value_iteration(inst2)
        assert b.values.initial_value() == 2.0 * a.values.initial_value()
        assert np.array_equal(a.policy.raw_actions(), b.policy.raw_actions())


def test_sweeps_bounded_and_dominates_greedy(gpu):
    """test_mdp.cpp:193-202 and :238-246."""
    for trial in range(15):
        p = V.generate_instance(N.VCS_GEN_RANDOM, 41, trial, 4, 6, 25, 3)
        inst = V.MdpInstance.from_workload(p.vcc, p.bots)
        vi = V.value_iteration(inst)
        assert vi.values.sweeps() <= len(inst.tasks) + 1
        g = V.greedy_schedule(p.vcc, p.bots)
        assert vi.values.initial_value() >= V.greedy_reward(g, p.vcc) - 1e-9


def test_parallel_api_bit_identical(gpu):
    """test_parallel.cpp:64-106 through the mirrored API (worker count is partition-free)."""
    p = V.load_instance(str(GOLDEN / "canonical_instance.txt"))
    inst = V.MdpInstance.from_workload(p.vcc, p.bots)
    seq = V.value_iteration(inst)
    for w in (1, 2, 4, 8):
        par = V.parallel_value_iteration(inst, V.ViOptions(), w)
        assert np.array_equal(bits(par.values.raw_values()), bits(seq.values.raw_values()))
        assert np.array_equal(par.policy.raw_actions(), seq.policy.raw_actions())
        assert par.values.sweeps() == seq.values.sweeps()
    with pytest.raises(V.InvalidArgument, match="n_workers must be >= 1"):
        V.parallel_value_iteration(inst, V.ViOptions(), 0)
    rows = V.measure_speedup(inst, [1, 2])
    assert rows[0].workers == 1 and rows[0].speedup_vs_one == pytest.approx(1.0)


def test_shard_kernels_emulated_ranks(gpu, oracle):
    """The device shard API (vcs_shard_begin/sweep/finish) over 1..4 row blocks in ONE
    process: the blocks' sweeps run back to back on one buffer set (their atomicMax into the
    shared residual slot is the all-reduce), which must reproduce the oracle bit for bit."""
    import torch
    from paper_2012_12419_b200.sharded import CudaBackend, shard_plans
    p = V.load_instance(str(GOLDEN / "canonical_instance.txt"))
    ni = V.NativeInstance(p.vcc, bots=p.bots)
    sp = V.StateSpace.build_native(ni)
    v_ref, a_ref, sw_ref, _, _ = oracle.build(ni.ref).vi()
    lo, le = sp.layer_offsets(), sp.layer_edges()
    for world in (1, 2, 4):
        for skip in (0, 1):
            be = CudaBackend(sp, torch.device("cuda", 0))
            opts = N.vcs_solve_opts(1e-6, skip, 0, 1.0)
            be.begin(opts)
            plans = shard_plans(lo, le, world)
            M = sp.task_count() + 1
            for k in range(1, M + 1):
                for pl in plans:
                    be.sweep(k, pl.row_begin, pl.row_end, opts)
            values = np.zeros(sp.size())
            actions = np.zeros(sp.size(), np.int32)
            sweeps = [be.finish(M, pl.row_begin, pl.row_end, opts, values, actions)
                      for pl in plans]
            torch.cuda.synchronize()
            assert set(sweeps) == {sw_ref}
            assert np.array_equal(bits(values), bits(v_ref))
            assert np.array_equal(actions, a_ref)


@pytest.mark.parametrize("form", ["implicit", "explicit"])
def test_certified_proof_and_fallback(gpu, golden, form, monkeypatch):
    """VCS_METHOD_CERTIFIED: the two-version backward pass is the whole solve exactly when its
    residual lower bounds prove K* = H+1; early stops and sweep caps must take the wavefront
    fallback (implicit form: at collect, after materialising the CSR; explicit form: the graph
    IF node).  Bits equal the reference's digests either way."""
    import ctypes as C
    p = V.load_instance(str(GOLDEN / "canonical_instance.txt"))
    ni = V.NativeInstance(p.vcc, bots=p.bots)
    if form == "explicit":
        monkeypatch.setenv("VCS_BUILD_EXPLICIT", "1")
    sp = V.StateSpace.build_native(ni)
    monkeypatch.delenv("VCS_BUILD_EXPLICIT", raising=False)
    H = sp.task_count()

    def run(eps, cap=0):
        opts = N.vcs_solve_opts(eps, 1, cap, 1.0, N.VCS_METHOD_CERTIFIED)
        vals = np.empty(sp.size())
        acts = np.empty(sp.size(), np.int32)
        rep = N.vcs_solve_report()
        N.check(N.lib().vcs_solve(sp.handle, C.byref(opts), N.ptr(vals, C.c_double),
                                  N.ptr(acts, C.c_int32), C.byref(rep)))
        return vals, acts, rep

    for eps in (1e-6, 5.0, 0.5):
        g = golden["cases"]["canonical"][f"eps={eps:g}"]
        vals, acts, rep = run(eps)
        assert rep.sweeps == g["sweeps"]
        assert sha(vals) == g["values_sha"] and sha(acts) == g["actions_sha"]
        if g["sweeps"] == H + 1:
            assert rep.method == N.VCS_METHOD_CERTIFIED, eps  # the proof holds
        else:
            assert rep.method == N.VCS_METHOD_WAVEFRONT, eps  # early stop: the fallback ran
    # a sweep cap below H+1 can never be certified
    vals, acts, rep = run(1e-6, cap=H)
    assert rep.sweeps == H and rep.method == N.VCS_METHOD_WAVEFRONT
    # the same graph alternates between both outcomes when re-run with other options
    vals, acts, rep = run(1e-6)
    assert rep.method == N.VCS_METHOD_CERTIFIED
    assert sha(vals) == golden["cases"]["canonical"]["eps=1e-06"]["values_sha"]


def test_certified_full_size(gpu, golden):
    """C3 and C4: the proof holds and the single pass reproduces the reference digests."""
    for gen, name in (((N.VCS_GEN_HOMOG, 2012, 0, 5, 8, 40, 3), "C3"),
                      ((N.VCS_GEN_HOMOG, 2012, 0, 6, 8, 48, 3), "C4")):
        ni = V.generate_instance(*gen, as_objects=False)
        sp = V.StateSpace.build_native(ni, 10**9)
        r = _solve(sp, method=N.VCS_METHOD_CERTIFIED)
        g = golden["cases"][name]["eps=1e-06"]
        assert r.values.report.method == N.VCS_METHOD_CERTIFIED
        assert r.values.sweeps() == g["sweeps"] == sp.task_count() + 1
        assert sha(r.values.raw_values()) == g["values_sha"]
        assert sha(r.policy.raw_actions()) == g["actions_sha"]


@pytest.mark.parametrize("layout", ["keyspace", "bfs"])
def test_certified_pair_layouts(gpu, golden, monkeypatch, layout):
    """Both pair layouts of the implicit certified pass reproduce the reference digests. The
    default layout stores pairs by key-space index: C4's full layers run k_cert_dense and its
    sparse layers the BFS-order kernel. VCS_CERT_BFS=1 keeps pairs by BFS index with a
    rank-table hop. The canonical instance covers the early stop (eps = 5): the proof fails
    and the fallback runs at collect."""
    if layout == "bfs":
        monkeypatch.setenv("VCS_CERT_BFS", "1")
    for gen, name in (((N.VCS_GEN_HOMOG, 2012, 0, 5, 8, 40, 3), "C3"),
                      ((N.VCS_GEN_HOMOG, 2012, 0, 6, 8, 48, 3), "C4")):
        ni = V.generate_instance(*gen, as_objects=False)
        sp = V.StateSpace.build_native(ni, 10**9)  # a fresh space: a fresh graph
        r = _solve(sp, method=N.VCS_METHOD_CERTIFIED)
        g = golden["cases"][name]["eps=1e-06"]
        assert r.values.report.method == N.VCS_METHOD_CERTIFIED
        assert sha(r.values.raw_values()) == g["values_sha"]
        assert sha(r.policy.raw_actions()) == g["actions_sha"]
    p = V.load_instance(str(GOLDEN / "canonical_instance.txt"))
    sp = V.StateSpace.build_native(V.NativeInstance(p.vcc, bots=p.bots))
    for eps in (1e-6, 5.0):
        r = _solve(sp, eps=eps, method=N.VCS_METHOD_AUTO)
        g = golden["cases"]["canonical"][f"eps={eps:g}"]
        assert r.values.sweeps() == g["sweeps"]
        assert sha(r.values.raw_values()) == g["values_sha"]
        assert sha(r.policy.raw_actions()) == g["actions_sha"]


def test_builder_paths_agree(gpu, oracle, monkeypatch):
    """The persistent one-kernel builder (dense key spaces) and the layered multi-kernel builder
    produce identical CSR; a wide-capacity instance (key space far beyond the dense limit) takes
    the hash path and still matches the oracle bit for bit."""
    from cases import cloud
    ni = V.generate_instance(N.VCS_GEN_HOMOG, 2012, 0, 5, 8, 40, 3, as_objects=False)
    a = V.StateSpace.build_native(ni, 10**9)
    monkeypatch.setenv("VCS_BUILD_LAYERED", "1")
    b = V.StateSpace.build_native(ni, 10**9)
    monkeypatch.delenv("VCS_BUILD_LAYERED")
    assert np.array_equal(a.layer_offsets(), b.layer_offsets())
    for x, y in zip(a.csr(), b.csr()):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
    # 8 clouds x 300 VMs: 301^8 keys -> hash path
    vcc = V.VccModel([cloud(i + 1, 300, 100.0 + i, 5.0 + i) for i in range(8)], 1.0, 1.2, 0.5)
    tasks = [V.Task(j + 1, 1 + (j * 7) % 3, 60.0, 90.0) for j in range(7)]
    wide = V.NativeInstance(vcc, bots=[V.BagOfTasks(1, tasks)])
    sp = V.StateSpace.build_native(wide, 10**9)
    _csr_equal(sp, oracle.build(wide.ref, 10**9))
    # the state cap is enforced with the reference's message on the persistent path too
    with pytest.raises(N.StateCapacityError, match="exceeds cap of 1000 states"):
        V.StateSpace.build_native(ni, 1000)


def test_batched_policy_query(gpu, reference):
    """vcs_policy_query: value_of / action_for for many full states at once on the
    device, bit-identical to the UNMODIFIED reference's ValueTable::value_of and
    Policy::action_for (oracle/_ref ref_res_value_of / ref_res_action_for) on the same states;
    unreachable -> NaN / VCS_NO_ACTION where the reference raises, terminal -> VCS_NO_ACTION;
    host and device buffers both accepted."""
    import torch
    rng = np.random.default_rng(7)
    for trial in range(4):
        p = V.generate_instance(N.VCS_GEN_RANDOM, 61, trial, 3, 6, 10, 3)
        inst = V.MdpInstance.from_workload(p.vcc, p.bots)
        vi = V.value_iteration(inst)
        ni = inst.native()
        ref_vi = reference.build(ni.ref, 10**9).vi(eps=1e-6)
        states = []
        for walk in range(6):
            s = V.initial_state(inst)
            while True:
                states.append(s)
                if s.terminal:
                    break
                acts = V.legal_actions(inst, s)
                s = V.transition(s, acts[rng.integers(len(acts))], inst)
        # unreachable: more free VMs than the cloud has
        s0 = V.initial_state(inst)
        bad = V.MdpState([v + 1 for v in s0.free_vms], s0.next_task_index, False)
        states.append(bad)
        vals = vi.values.value_of_many(states)
        acts = vi.policy.action_for_many(states)
        for s, v, a in zip(states, vals, acts):
            ref_v = ref_vi.value_of(s.free_vms, s.next_task_index, s.terminal)
            ref_a = ref_vi.action_for(s.free_vms, s.next_task_index, s.terminal)
            if ref_v is None:  # the reference throws std::out_of_range
                assert np.isnan(v) and a == N.VCS_NO_ACTION
                continue
            assert np.float64(v).view(np.uint64) == np.float64(ref_v).view(np.uint64)
            assert a == (N.VCS_NO_ACTION if ref_a is None else ref_a)
            # and the per-state device path agrees
            assert np.float64(vi.values.value_of(s)).view(np.uint64) == np.float64(v).view(np.uint64)
        # device-resident inputs and outputs are used in place
        space = vi.values.space()
        fv, ti, te = space._state_arrays(states)
        dev = torch.device("cuda", 0)
        dfv, dti, dte = (torch.from_numpy(x).to(dev) for x in (fv, ti, te))
        dval = torch.empty(len(states), dtype=torch.float64, device=dev)
        dact = torch.empty(len(states), dtype=torch.int32, device=dev)
        torch.cuda.synchronize()
        ptr = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
        N.check(N.lib().vcs_policy_query(space.handle, len(states), ptr(dfv), ptr(dti), ptr(dte),
                                         ptr(dval), ptr(dact), None, None))
        torch.cuda.synchronize()
        assert np.array_equal(dval.cpu().numpy().view(np.uint64), vals.view(np.uint64))
        assert np.array_equal(dact.cpu().numpy(), acts)


@pytest.mark.parametrize("streamed", [True, False])
def test_pinned_download_large(gpu, golden, monkeypatch, streamed):
    """C3 (1.8 M states) into pinned buffers: the chunked download behind the layer events of the
    certified pass (forced: C3's 21 MB is below the 32 MB default) and the single copy are exact,
    on a fresh and on a re-used graph."""
    import torch
    if streamed:
        monkeypatch.setenv("VCS_STREAM_MIN_MB", "1")
    ni = V.generate_instance(N.VCS_GEN_HOMOG, 2012, 0, 5, 8, 40, 3, as_objects=False)
    sp = V.StateSpace.build_native(ni, 10**9)
    S = sp.size()
    vals = torch.full((S,), float("nan"), dtype=torch.float64, pin_memory=True)
    acts = torch.full((S,), 12345, dtype=torch.int32, pin_memory=True)
    g = golden["cases"]["C3"]["eps=1e-06"]
    for _ in range(2):
        opts = N.vcs_solve_opts(1e-6, 1, 0, 1.0, N.VCS_METHOD_AUTO)
        rep = N.vcs_solve_report()
        N.check(N.lib().vcs_solve(sp.handle, C.byref(opts),
                                  C.cast(C.c_void_p(vals.data_ptr()), C.POINTER(C.c_double)),
                                  C.cast(C.c_void_p(acts.data_ptr()), C.POINTER(C.c_int32)),
                                  C.byref(rep)))
        assert rep.sweeps == g["sweeps"]
        assert sha(vals.numpy()) == g["values_sha"]
        assert sha(acts.numpy()) == g["actions_sha"]


def test_concurrent_pinned_solves(gpu, golden):
    """Two host threads, each with its own space, solve into pinned buffers at the same time:
    the narrowed download's host workers serve one job at a time (the other caller widens
    inline), and both results equal the reference digests (C ABI re-entrancy)."""
    import threading
    import torch
    gen = (N.VCS_GEN_HOMOG, 2012, 0, 5, 8, 40, 3)  # C3
    g = golden["cases"]["C3"]["eps=1e-06"]
    out, errs = {}, []

    def run(tag):
        try:
            ni = V.generate_instance(*gen, as_objects=False)
            sp = V.StateSpace.build_native(ni, 10**9)
            S = sp.size()
            vals = torch.empty(S, dtype=torch.float64, pin_memory=True)
            acts = torch.empty(S, dtype=torch.int32, pin_memory=True)
            for _ in range(3):
                opts = N.vcs_solve_opts(1e-6, 1, 0, 1.0, N.VCS_METHOD_AUTO)
                rep = N.vcs_solve_report()
                N.check(N.lib().vcs_solve(sp.handle, C.byref(opts),
                                          C.cast(C.c_void_p(vals.data_ptr()), C.POINTER(C.c_double)),
                                          C.cast(C.c_void_p(acts.data_ptr()), C.POINTER(C.c_int32)),
                                          C.byref(rep)))
                out.setdefault(tag, []).append((sha(vals.numpy()), sha(acts.numpy())))
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    ts = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for tag in range(2):
        for vs, as_ in out[tag]:
            assert (vs, as_) == (g["values_sha"], g["actions_sha"])


@pytest.mark.parametrize("pull", [True, False])
def test_layered_implicit_build_matches_golden(gpu, golden, monkeypatch, pull):
    """The layered builder's implicit form (the path of spaces too large for the persistent
    builder, e.g. C7), in its pull form (k_pull_first / k_pull_rank on non-retiring transitions,
    the default) and its push form (VCS_BUILD_NO_PULL): forced on C3/C4 with
    VCS_BUILD_NO_PERSISTENT, the certified pass on its keys + rank tables reproduces the
    reference digests, and the explicit CSR materialised from it later (Jacobi) gives the same
    bits."""
    monkeypatch.setenv("VCS_BUILD_NO_PERSISTENT", "1")
    if not pull:
        monkeypatch.setenv("VCS_BUILD_NO_PULL", "1")
    for name in ("C3", "C4"):
        p = V.load_instance(str(GOLDEN / "instances" / f"{name.lower()}.txt"))
        sp = V.StateSpace.build_native(V.NativeInstance(p.vcc, bots=p.bots), 10**9)
        g = golden["cases"][name]["eps=1e-06"]
        assert sp.size() == golden["cases"][name]["S"]
        r = _solve(sp, method=N.VCS_METHOD_CERTIFIED)
        assert r.values.report.method == N.VCS_METHOD_CERTIFIED
        assert sha(r.values.raw_values()) == g["values_sha"]
        assert sha(r.policy.raw_actions()) == g["actions_sha"]
        if name == "C3":
            r = _solve(sp, method=N.VCS_METHOD_JACOBI)
            assert sha(r.values.raw_values()) == g["values_sha"]


def test_certified_tma_kernel_matches_golden(gpu, golden, monkeypatch):
    """The TMA-staged key-space walk (k_cert_dense_tma, VCS_CERT_TMA=1) gives the reference's
    bits on C3 and C4 (its non-retiring layers; the retiring ones keep k_cert_dense)."""
    monkeypatch.setenv("VCS_CERT_TMA", "1")
    for name in ("C3", "C4"):
        p = V.load_instance(str(GOLDEN / "instances" / f"{name.lower()}.txt"))
        sp = V.StateSpace.build_native(V.NativeInstance(p.vcc, bots=p.bots), 10**9)
        g = golden["cases"][name]["eps=1e-06"]
        r = _solve(sp, method=N.VCS_METHOD_CERTIFIED)
        assert sha(r.values.raw_values()) == g["values_sha"]
        assert sha(r.policy.raw_actions()) == g["actions_sha"]


def test_small_builder_matches_layered_and_oracle(gpu, oracle, monkeypatch):
    """The single-CTA small-space builder (k_build_small: the canonical instance's 330 hash-path
    layers in one launch) writes the same CSR as the layered builder and the oracle; an instance
    whose layers outgrow its shared-memory tables falls back to the layered path; the state cap
    raises the reference's error from inside it."""
    from cases import cloud
    p = V.load_instance(str(GOLDEN / "canonical_instance.txt"))
    ni = V.NativeInstance(p.vcc, bots=p.bots)
    a = V.StateSpace.build_native(ni, 10**9)
    monkeypatch.setenv("VCS_NO_SMALL_BUILD", "1")
    b = V.StateSpace.build_native(ni, 10**9)
    monkeypatch.delenv("VCS_NO_SMALL_BUILD")
    assert np.array_equal(a.layer_offsets(), b.layer_offsets())
    for x, y in zip(a.csr(), b.csr()):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
    _csr_equal(a, oracle.build(ni.ref, 10**9))
    with pytest.raises(N.StateCapacityError, match="exceeds cap of 50000 states"):
        V.StateSpace.build_native(ni, 50000)
    # 8 clouds x 300 VMs with 7 tasks: layers outgrow the tables -> layered fallback, same bits
    vcc = V.VccModel([cloud(i + 1, 300, 100.0 + i, 5.0 + i) for i in range(8)], 1.0, 1.2, 0.5)
    tasks = [V.Task(j + 1, 1 + (j * 7) % 3, 60.0, 90.0) for j in range(7)]
    wide = V.NativeInstance(vcc, bots=[V.BagOfTasks(1, tasks)])
    _csr_equal(V.StateSpace.build_native(wide, 10**9), oracle.build(wide.ref, 10**9))


@pytest.mark.parametrize("name,eps", [("C3", 3.0), ("C4", 4.0)])
def test_certificate_failure_at_scale(gpu, golden, name, eps):
    """An early stop on a full-size implicit space (C3 at eps 3 stops at 39 of 41 sweeps, C4 at
    eps 4 at 24 of 49): the certificate fails, the fallback runs inside collect (reported as
    deferred), and the result is the reference's."""
    p = V.load_instance(str(GOLDEN / "instances" / f"{name.lower()}.txt"))
    sp = V.StateSpace.build_native(V.NativeInstance(p.vcc, bots=p.bots), 10**9)
    g = golden["cases"][name][f"eps={eps:g}"]
    r = _solve(sp, eps=eps, method=N.VCS_METHOD_AUTO)
    rep = r.values.report
    assert rep.method == N.VCS_METHOD_WAVEFRONT and rep.fallback_deferred == 1
    assert r.values.sweeps() == g["sweeps"] < sp.task_count() + 1
    assert sha(r.values.raw_values()) == g["values_sha"]
    assert sha(r.policy.raw_actions()) == g["actions_sha"]
    # and the certified case on the same space is not deferred
    r = _solve(sp, eps=1e-6, method=N.VCS_METHOD_AUTO)
    assert r.values.report.method == N.VCS_METHOD_CERTIFIED and r.values.report.fallback_deferred == 0


def test_certified_ilp2_kernel_matches_golden(gpu, golden, monkeypatch):
    """k_cert_dense2 (two key-space indices in flight per thread, VCS_CERT_ILP2=1) gives the
    reference's bits on C3 and C4."""
    monkeypatch.setenv("VCS_CERT_ILP2", "1")
    for name in ("C3", "C4"):
        p = V.load_instance(str(GOLDEN / "instances" / f"{name.lower()}.txt"))
        sp = V.StateSpace.build_native(V.NativeInstance(p.vcc, bots=p.bots), 10**9)
        g = golden["cases"][name]["eps=1e-06"]
        r = _solve(sp, method=N.VCS_METHOD_CERTIFIED)
        assert sha(r.values.raw_values()) == g["values_sha"]
        assert sha(r.policy.raw_actions()) == g["actions_sha"]


@pytest.mark.parametrize("kernel", ["generic", "permute", "nr", "win"])
def test_certified_kernel_variants_match_golden(gpu, golden, monkeypatch, kernel):
    """The generic key-space walk (VCS_CERT_GENERIC=1, the retiring-capable kernel on every
    layer), the non-retiring walk with key-space-ordered results + gather pass
    (VCS_CERT_PERMUTE=1, the default only for pair vectors beyond L2), the non-retiring walk
    writing at the BFS rank (VCS_CERT_NR=1) and its shared-memory-window form (VCS_CERT_WIN=1)
    reproduce the reference's digests on C3 and C4."""
    monkeypatch.setenv({"generic": "VCS_CERT_GENERIC", "permute": "VCS_CERT_PERMUTE",
                        "nr": "VCS_CERT_NR", "win": "VCS_CERT_WIN"}[kernel], "1")
    for name in ("C3", "C4"):
        p = V.load_instance(str(GOLDEN / "instances" / f"{name.lower()}.txt"))
        sp = V.StateSpace.build_native(V.NativeInstance(p.vcc, bots=p.bots), 10**9)
        g = golden["cases"][name]["eps=1e-06"]
        r = _solve(sp, method=N.VCS_METHOD_CERTIFIED)
        assert sha(r.values.raw_values()) == g["values_sha"]
        assert sha(r.policy.raw_actions()) == g["actions_sha"]


def test_c7_kernel_variants_agree(gpu, monkeypatch):
    """C7 (190.7 M states, no reference digest: the reference cannot build it in a test's time)
    is solved bit-identically by the default path (non-retiring walk + gather pass), the
    generic walk and the scattered-store variant; the certificate holds (57 sweeps)."""
    p = V.load_instance(str(GOLDEN / "instances" / "c7.txt"))
    sp = V.StateSpace.build_native(V.NativeInstance(p.vcc, bots=p.bots), 10**9)
    assert sp.size() == 190740125
    digests = []
    for env in ({}, {"VCS_CERT_GENERIC": "1"}, {"VCS_CERT_PERMUTE": "0"}):
        for k in ("VCS_CERT_GENERIC", "VCS_CERT_PERMUTE"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        sp2 = V.StateSpace.build_native(V.NativeInstance(p.vcc, bots=p.bots), 10**9)
        r = _solve(sp2, method=N.VCS_METHOD_CERTIFIED)
        assert r.values.sweeps() == 57 and r.values.report.method == N.VCS_METHOD_CERTIFIED
        digests.append((sha(r.values.raw_values()), sha(r.policy.raw_actions())))
        del r, sp2
    assert digests[0] == digests[1] == digests[2]


def test_certified_streaming_kernel_matches_golden(gpu, golden, monkeypatch):
    """k_cert_stream (VCS_CERT_STREAM=1): the whole certified pass as one persistent kernel with
    per-tile dependency flags (window deps on non-retiring transitions, whole-layer deps
    otherwise, four rotating pair buffers) reproduces the reference's digests on C3, C4 and the
    C5 sample points, and terminates (no tile waits on a later one)."""
    import bench_workloads as W
    monkeypatch.setenv("VCS_CERT_STREAM", "1")
    for name in ("C3", "C4"):
        p = V.load_instance(str(GOLDEN / "instances" / f"{name.lower()}.txt"))
        sp = V.StateSpace.build_native(V.NativeInstance(p.vcc, bots=p.bots), 10**9)
        g = golden["cases"][name]["eps=1e-06"]
        for _ in range(2):  # direct first solve, then the captured graph
            r = _solve(sp, method=N.VCS_METHOD_CERTIFIED)
            assert sha(r.values.raw_values()) == g["values_sha"]
            assert sha(r.policy.raw_actions()) == g["actions_sha"]
    table = W.channel_table()
    for key in [k for k in golden["cases"] if k.startswith("C5_")]:
        _, K, c, scheme = key.split("_", 3)
        p = V.parse_instance(W.c5_text(int(K[1:]), int(c[1:]), scheme, table))
        sp = V.StateSpace.build_native(V.NativeInstance(p.vcc, bots=p.bots), 10**9)
        r = _solve(sp, method=N.VCS_METHOD_CERTIFIED)
        e = golden["cases"][key]["eps=1e-06"]
        assert sha(r.values.raw_values()) == e["values_sha"], key
        assert sha(r.policy.raw_actions()) == e["actions_sha"], key


def test_certified_tail_kernel_matches_golden(gpu, golden, monkeypatch):
    """k_cert_tail (VCS_CERT_TAIL=1: the small sparse bottom layers in one block) gives the
    reference's bits on C3 and C4."""
    monkeypatch.setenv("VCS_CERT_TAIL", "1")
    for name in ("C3", "C4"):
        p = V.load_instance(str(GOLDEN / "instances" / f"{name.lower()}.txt"))
        sp = V.StateSpace.build_native(V.NativeInstance(p.vcc, bots=p.bots), 10**9)
        g = golden["cases"][name]["eps=1e-06"]
        for _ in range(2):
            r = _solve(sp, method=N.VCS_METHOD_CERTIFIED)
            assert sha(r.values.raw_values()) == g["values_sha"]
            assert sha(r.policy.raw_actions()) == g["actions_sha"]


@pytest.mark.parametrize("pull", [True, False])
def test_pull_builder_matches_golden_and_oracle(gpu, golden, oracle, monkeypatch, pull):
    """The persistent builder's pull form (first edges pulled from layer t's rank table on
    non-retiring transitions, BFS ranks from a bitmap over the edge keys; the default) and its
    push form (VCS_BUILD_NO_PULL: an atomicMin per edge) number every layer alike: C3 / C4 give
    the reference digests through the certified pass and Jacobi on the materialised CSR, and
    random instances with retiring clouds (pull and push layers interleaved) equal the oracle
    bit for bit, layer sizes and policy queries included."""
    from conftest import bits
    if not pull:
        monkeypatch.setenv("VCS_BUILD_NO_PULL", "1")
    for name in ("C3", "C4"):
        p = V.load_instance(str(GOLDEN / "instances" / f"{name.lower()}.txt"))
        sp = V.StateSpace.build_native(V.NativeInstance(p.vcc, bots=p.bots), 10**9)
        g = golden["cases"][name]["eps=1e-06"]
        assert sp.size() == golden["cases"][name]["S"]
        r = _solve(sp, method=N.VCS_METHOD_CERTIFIED)
        assert sha(r.values.raw_values()) == g["values_sha"]
        assert sha(r.policy.raw_actions()) == g["actions_sha"]
        if name == "C3":
            r = _solve(sp, method=N.VCS_METHOD_JACOBI)
            assert sha(r.values.raw_values()) == g["values_sha"]
    for trial in range(4):
        ni = V.generate_instance(N.VCS_GEN_RANDOM, 43, trial, 5, 6, 18, 3, as_objects=False)
        sp = V.StateSpace.build_native(ni, 10**9)
        osp = oracle.build(ni.ref, 10**9)
        assert sp.size() == osp.S
        assert np.array_equal(sp.layer_offsets().astype(np.uint64), osp.csr()[0])
        v, a, sw, _, _ = osp.vi()
        r = _solve(sp, method=N.VCS_METHOD_CERTIFIED)
        assert r.values.report.sweeps == sw
        assert np.array_equal(bits(r.values.raw_values()), bits(v)), trial
        assert np.array_equal(r.policy.raw_actions(), a), trial


@pytest.mark.parametrize("env", [
    {"VCS_NO_SMALL_SOLVE": "1"},                         # per-layer k_cert_rows + graph IF node
    {"VCS_CERT_SMALL_THREADS": "256"}, {"VCS_CERT_SMALL_THREADS": "1024"},
    {"VCS_SMALL_THREADS": "128"}, {"VCS_SMALL_THREADS": "256"}, {"VCS_SMALL_THREADS": "1024"},
])
def test_small_space_kernel_variants_match_golden(gpu, golden, monkeypatch, env):
    """The single-CTA builder at every block size it is compiled for, the single-CTA certified
    pass at every block size, and the per-layer certified pass on the same small explicit space
    (the canonical instance) give the reference's digests at eps = 1e-6 (certified) and at
    eps = 5 / 0.5 (early stops: the fallback), with the sweep counts."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    p = V.load_instance(str(GOLDEN / "canonical_instance.txt"))
    sp = V.StateSpace.build_native(V.NativeInstance(p.vcc, bots=p.bots))
    assert sha(sp.layer_offsets()) == golden["cases"]["canonical"]["layers_sha"]
    for eps in (1e-6, 5.0, 0.5):
        g = golden["cases"]["canonical"][f"eps={eps:g}"]
        for _ in range(2):  # direct first solve, then the captured graph
            r = _solve(sp, eps=eps, method=N.VCS_METHOD_CERTIFIED)
            assert r.values.report.sweeps == g["sweeps"], (env, eps)
            assert sha(r.values.raw_values()) == g["values_sha"], (env, eps)
            assert sha(r.policy.raw_actions()) == g["actions_sha"], (env, eps)


@pytest.mark.parametrize("form", ["explicit", "implicit"])
def test_layered_builder_growth_path(gpu, golden, monkeypatch, form):
    """The layered builder without its a-priori sizing (VCS_BUILD_NO_PRESIZE: the arrays grow
    geometrically, as for spaces whose bound is unaffordable) builds C3 exactly: the explicit CSR
    (VCS_BUILD_LAYERED) and the implicit form (VCS_BUILD_NO_PERSISTENT) both give the reference's
    digests."""
    monkeypatch.setenv("VCS_BUILD_NO_PRESIZE", "1")
    monkeypatch.setenv("VCS_BUILD_LAYERED" if form == "explicit" else "VCS_BUILD_NO_PERSISTENT", "1")
    p = V.load_instance(str(GOLDEN / "instances" / "c3.txt"))
    sp = V.StateSpace.build_native(V.NativeInstance(p.vcc, bots=p.bots), 10**9)
    g = golden["cases"]["C3"]["eps=1e-06"]
    assert sp.size() == golden["cases"]["C3"]["S"]
    r = _solve(sp, method=N.VCS_METHOD_CERTIFIED)
    assert sha(r.values.raw_values()) == g["values_sha"]
    assert sha(r.policy.raw_actions()) == g["actions_sha"]


@pytest.mark.parametrize("name", ["canonical", "C3"])
def test_enqueue_collect_on_a_caller_stream(gpu, golden, name):
    """vcs_solve_enqueue on a caller's stream right after the build (the solve buffers are
    allocated on the space's stream in the same call and ordered by an event, not a host sync),
    then vcs_solve_collect into host buffers on that stream: the reference's digests, on a fresh
    space and on the replayed graph."""
    import torch
    path = GOLDEN / ("canonical_instance.txt" if name == "canonical" else "instances/c3.txt")
    p = V.load_instance(str(path))
    sp = V.StateSpace.build_native(V.NativeInstance(p.vcc, bots=p.bots), 10**9)
    g = golden["cases"][name]["eps=1e-06"]
    st = torch.cuda.Stream()
    h = C.c_void_p(st.cuda_stream)
    vals = np.empty(sp.size())
    acts = np.empty(sp.size(), np.int32)
    for _ in range(2):
        opts = N.vcs_solve_opts(1e-6, 1, 0, 1.0, N.VCS_METHOD_CERTIFIED)
        N.check(N.lib().vcs_solve_enqueue(sp.handle, C.byref(opts), h))
        rep = N.vcs_solve_report()
        N.check(N.lib().vcs_solve_collect(sp.handle, N.ptr(vals, C.c_double), N.ptr(acts, C.c_int32),
                                          C.byref(rep), h))
        st.synchronize()
        assert rep.sweeps == g["sweeps"]
        assert sha(vals) == g["values_sha"]
        assert sha(acts) == g["actions_sha"]
