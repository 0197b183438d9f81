"""Pin the C oracle (oracle/vcs_oracle.c) against the reference: golden vectors generated from
the unmodified reference (tests/golden/golden.json) and, where the reference library is
present, direct bitwise comparison.  CPU only."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2012_12419_b200 as V
from paper_2012_12419_b200 import _native as N
from cases import FAMILIES, named_cases
from conftest import sha


def _oracle_record(oracle, ni, eps_list):
    sp = oracle.build(ni.ref, 10**9)
    lo = sp.csr()[0]
    out = {"S": sp.S, "layers_sha": sha(lo)}
    for eps in eps_list:
        v, a, sw, _, _ = sp.vi(eps=eps)
        out[f"eps={eps:g}"] = (sw, sha(v), sha(a), v)
    return sp, out


def _check(rec, got, eps_list):
    assert got["S"] == rec["S"]
    assert got["layers_sha"] == rec["layers_sha"]
    for eps in eps_list:
        key = f"eps={eps:g}"
        sw, vs, as_, _ = got[key]
        assert sw == rec[key]["sweeps"], key
        assert vs == rec[key]["values_sha"], key
        assert as_ == rec[key]["actions_sha"], key


@pytest.mark.parametrize("name", list(named_cases().keys()))
def test_named_cases_match_reference_golden(oracle, golden, name):
    ni, eps_list = named_cases()[name]
    _, got = _oracle_record(oracle, ni, eps_list)
    _check(golden["cases"][name], got, eps_list)
    s = ni.struct
    tgt, used, paid, unused, _ = oracle.greedy(ni.ref, s.n_tasks, s.n_clouds)
    g = golden["cases"][name]["greedy"]
    assert (paid, unused, int(used.sum())) == (g["paid"], g["unused"], g["placed"])
    assert sha(tgt) == g["targets_sha"]


def test_known_answers(golden):
    """The reference's published/known answers are in the golden file."""
    c = golden["cases"]
    assert abs(c["canonical"]["eps=1e-06"]["v0"] - 202.4) <= 1e-9        # acceptance.cpp:87
    assert c["canonical"]["eps=1e-06"]["rollout_paid"] == 58             # test_mdp.cpp:276
    assert c["canonical"]["eps=1e-06"]["rollout_unused"] == 0
    assert c["canonical"]["greedy"]["paid"] == 85                       # test_greedy.cpp:39
    assert c["canonical"]["greedy"]["unused"] == 27
    assert c["canonical"]["greedy"]["placed"] == 245
    assert c["canonical"]["greedy"]["reward"] == 116.0
    assert c["canonical"]["S"] == 68797 and c["canonical"]["eps=1e-06"]["sweeps"] == 331
    assert c["canonical"]["eps=5"]["sweeps"] == 229                      # early stop
    assert abs(c["tiny_2vm_3tasks"]["eps=1e-06"]["v0"] - 0.8) <= 1e-12   # test_mdp.cpp:118-124
    assert c["empty_tasks"]["eps=1e-06"]["sweeps"] == 1                  # test_mdp.cpp:108-116
    assert c["C3"]["S"] == 1788700 and c["C3"]["eps=1e-06"]["sweeps"] == 41
    assert c["C3"]["eps=1e-06"]["v0_hex"] == (-23.599999999999973).hex()
    assert c["C4"]["S"] == 19333781 and c["C4"]["eps=1e-06"]["sweeps"] == 49
    assert c["C2"]["greedy"]["paid"] == 101300 and c["C2"]["greedy"]["placed"] == 98991


@pytest.mark.parametrize("family", list(FAMILIES.keys()))
def test_random_families_match_reference_golden(oracle, golden, family):
    seed, params, n, brute = FAMILIES[family]
    recs = golden["families"][family]
    assert len(recs) == n
    for trial in range(n):
        ni = V.generate_instance(N.VCS_GEN_RANDOM, seed, trial, *params, as_objects=False)
        sp, got = _oracle_record(oracle, ni, (1e-6,))
        _check(recs[trial], got, (1e-6,))
        s = ni.struct
        tgt, used, paid, unused, _ = oracle.greedy(ni.ref, s.n_tasks, s.n_clouds)
        assert sha(tgt) == recs[trial]["greedy"]["targets_sha"]
        if brute:  # acceptance criterion 3: V(initial) equals exhaustive search to 1e-9
            v = got["eps=1e-06"][3]
            fv = np.ctypeslib.as_array(s.cloud_vm_free, shape=(s.n_clouds,)).astype(np.int32)
            import ctypes as C
            hp = oracle.L.orc_hidden_penalty(sp.h, fv.ctypes.data_as(C.POINTER(C.c_int32)), 0,
                                             1 if s.n_tasks == 0 else 0)
            assert abs((v[0] - hp) - recs[trial]["brute_force"]) <= 1e-9


def test_c3_matches_reference_golden(oracle, golden):
    ni = V.generate_instance(N.VCS_GEN_HOMOG, 2012, 0, 5, 8, 40, 3, as_objects=False)
    sp = oracle.build(ni.ref, 10**9)
    assert (sp.S, sp.E) == (1788700, 8478149)
    v, a, sw, _, _ = sp.vi(workers=8)
    rec = golden["cases"]["C3"]
    assert sw == rec["eps=1e-06"]["sweeps"]
    assert sha(v) == rec["eps=1e-06"]["values_sha"]
    assert sha(a) == rec["eps=1e-06"]["actions_sha"]


def test_c2_greedy_matches_reference_golden(oracle, golden):
    ni = V.generate_instance(N.VCS_GEN_GREEDY, 12345, 0, 1000, 100, 1000, 3, as_objects=False)
    tgt, used, paid, unused, _ = oracle.greedy(ni.ref, 100000, 1000)
    g = golden["cases"]["C2"]["greedy"]
    assert (paid, unused, int(used.sum())) == (g["paid"], g["unused"], g["placed"])
    assert sha(tgt) == g["targets_sha"]


@pytest.mark.parametrize("workers", [2, 4, 8])
def test_oracle_worker_counts_bit_identical(oracle, workers):
    """test_parallel.cpp:89-106 restated on the oracle."""
    for trial in range(10):
        ni = V.generate_instance(N.VCS_GEN_RANDOM, 47, trial, 4, 6, 25, 3, as_objects=False)
        sp = oracle.build(ni.ref)
        v1, a1, s1, _, _ = sp.vi(workers=1)
        vw, aw, sw, _, _ = sp.vi(workers=workers)
        assert np.array_equal(v1.view(np.uint64), vw.view(np.uint64))
        assert np.array_equal(a1, aw) and s1 == sw


def test_oracle_against_reference_directly(oracle, reference):
    """Fresh seeds not in the golden file, compared bit for bit with the live reference."""
    for trial in range(40):
        ni = V.generate_instance(N.VCS_GEN_RANDOM, 9001, trial, 4, 6, 30, 3, as_objects=False)
        osp = oracle.build(ni.ref)
        rsp = reference.build(ni.ref)
        assert osp.S == rsp.S
        assert np.array_equal(osp.csr()[0], rsp.layers())
        for eps in (1e-6, 0.7):
            v, a, sw, _, _ = osp.vi(eps=eps)
            r = rsp.vi(eps=eps)
            assert sw == r.sweeps
            assert np.array_equal(v.view(np.uint64), r.values().view(np.uint64))
            assert np.array_equal(a, r.actions())


def test_oracle_cap_error(oracle):
    from cases import tiny
    vcc, bots = tiny(6, [1] * 6)
    ni = V.NativeInstance(vcc, bots=bots)
    from oracle_bind import OracleError
    with pytest.raises(OracleError) as e:
        oracle.build(ni.ref, 3)
    assert e.value.code == N.VCS_ECAP and "3" in str(e.value)
