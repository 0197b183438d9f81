"""Multi-GPU certified pass (vcs_solve_multi): ONE state space split across ranks,
emulated on one B200 by giving several ranks the same device (ordering is by stream events
only, no kernel waits on another rank, so the code path is the multi-GPU one).

Parity: raw values / actions / sweeps equal the reference's golden digests for every rank count,
both exchange modes, both space forms (implicit key space: halo on non-retiring transitions;
explicit CSR: row ranges + all-gather), and the certificate-failure fallback (canonical at
eps = 5).  The reference's own contract is bit-identity across worker counts
(tests/test_parallel.cpp:89-106, acceptance.cpp:129-150)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import paper_2012_12419_b200 as V
from paper_2012_12419_b200 import _native as N
from cases import GOLDEN
from conftest import sha

pytestmark = pytest.mark.gpu


def _multi(sp, ranks, eps=1e-6, exchange=N.VCS_EXCHANGE_HALO, method=N.VCS_METHOD_CERTIFIED):
    opts = N.vcs_solve_opts(eps, 1, 0, 1.0, method)
    vals = np.empty(sp.size())
    acts = np.empty(sp.size(), np.int32)
    rep = N.vcs_solve_report()
    dv = np.zeros(ranks, np.int32)  # every rank on cuda:0
    N.check(N.lib().vcs_solve_multi(sp.handle, C.byref(opts), ranks, N.ptr(dv, C.c_int32),
                                    exchange, N.ptr(vals, C.c_double), N.ptr(acts, C.c_int32),
                                    C.byref(rep)))
    info = N.vcs_multi_report()
    if ranks > 1:
        N.check(N.lib().vcs_multi_info(sp.handle, C.byref(info)))
    return vals, acts, rep, info


@pytest.mark.parametrize("name,gen", [("C3", (N.VCS_GEN_HOMOG, 2012, 0, 5, 8, 40, 3)),
                                      ("C4", (N.VCS_GEN_HOMOG, 2012, 0, 6, 8, 48, 3))])
def test_multi_keyspace_matches_golden(gpu, golden, monkeypatch, name, gen):
    monkeypatch.setenv("VCS_MULTI_MIN_SPLIT", "4096")  # split C3's layers too
    ni = V.generate_instance(*gen, as_objects=False)
    sp = V.StateSpace.build_native(ni, 10**9)
    g = golden["cases"][name]["eps=1e-06"]
    for ranks in (2, 3, 8):
        for ex in (N.VCS_EXCHANGE_HALO, N.VCS_EXCHANGE_ALLGATHER):
            for use in range(2):  # direct launches first, then the captured multi-device graph
                vals, acts, rep, info = _multi(sp, ranks, exchange=ex)
                assert rep.method == N.VCS_METHOD_CERTIFIED
                assert rep.sweeps == g["sweeps"]
                assert sha(vals) == g["values_sha"], (ranks, ex, use)
                assert sha(acts) == g["actions_sha"], (ranks, ex, use)
                assert info.n_ranks == ranks and info.split_layers > 0
                assert info.graph == 1
        # the halo moves strictly less than the all-gather
        _, _, _, halo = _multi(sp, ranks, exchange=N.VCS_EXCHANGE_HALO)
        _, _, _, full = _multi(sp, ranks, exchange=N.VCS_EXCHANGE_ALLGATHER)
        assert 0 < halo.halo_bytes < full.halo_bytes


def test_multi_splits_small_layers_too(gpu, golden, monkeypatch):
    """VCS_MULTI_MIN_SPLIT=1 splits every dense layer (ranges of a few indices, empty ranks)."""
    monkeypatch.setenv("VCS_MULTI_MIN_SPLIT", "1")
    ni = V.generate_instance(N.VCS_GEN_HOMOG, 2012, 0, 5, 8, 40, 3, as_objects=False)
    sp = V.StateSpace.build_native(ni, 10**9)
    g = golden["cases"]["C3"]["eps=1e-06"]
    for ranks in (2, 5, 7):
        vals, acts, rep, info = _multi(sp, ranks)
        assert sha(vals) == g["values_sha"] and sha(acts) == g["actions_sha"]
        assert info.split_layers >= 30


@pytest.mark.parametrize("form", ["implicit", "explicit"])
def test_multi_canonical_and_fallback(gpu, golden, monkeypatch, form):
    """The canonical instance (hash-built explicit CSR; with VCS_BUILD_EXPLICIT too): row-range
    split with all-gather.  eps = 5 and 0.5 stop early: the certificate fails and the fallback
    runs at collect; eps = 1e-6 is certified."""
    monkeypatch.setenv("VCS_MULTI_MIN_SPLIT", "64")
    if form == "explicit":
        monkeypatch.setenv("VCS_BUILD_EXPLICIT", "1")
    p = V.load_instance(str(GOLDEN / "canonical_instance.txt"))
    sp = V.StateSpace.build_native(V.NativeInstance(p.vcc, bots=p.bots))
    monkeypatch.delenv("VCS_BUILD_EXPLICIT", raising=False)
    H = sp.task_count()
    for ranks in (2, 3):
        for eps in (1e-6, 5.0, 0.5):
            gd = golden["cases"]["canonical"][f"eps={eps:g}"]
            vals, acts, rep, info = _multi(sp, ranks, eps=eps)
            assert rep.sweeps == gd["sweeps"], (ranks, eps)
            assert sha(vals) == gd["values_sha"] and sha(acts) == gd["actions_sha"], (ranks, eps)
            expect = N.VCS_METHOD_CERTIFIED if gd["sweeps"] == H + 1 else N.VCS_METHOD_WAVEFRONT
            assert rep.method == expect, (ranks, eps)


def test_multi_python_api_and_errors(gpu, golden):
    ni = V.generate_instance(N.VCS_GEN_HOMOG, 2012, 0, 5, 8, 40, 3, as_objects=False)
    sp = V.StateSpace.build_native(ni, 10**9)
    g = golden["cases"]["C3"]["eps=1e-06"]
    r = V.run_value_iteration(sp, V.ViOptions(), devices=[0, 0, 0, 0])
    assert sha(r.values.raw_values()) == g["values_sha"]
    assert sha(r.policy.raw_actions()) == g["actions_sha"]
    # n_workers beyond the visible GPUs uses the GPUs there are (bit-identical)
    r = V.run_value_iteration(sp, V.ViOptions(), n_workers=8)
    assert sha(r.values.raw_values()) == g["values_sha"]
    with pytest.raises(V.InvalidArgument):
        V.run_value_iteration(sp, V.ViOptions(method=N.VCS_METHOD_JACOBI), devices=[0, 0])
    dv = np.zeros(2, np.int32)
    opts = N.vcs_solve_opts(1e-6, 1, 0, 1.0, N.VCS_METHOD_CERTIFIED)
    assert N.lib().vcs_solve_multi_enqueue(sp.handle, C.byref(opts), 2, N.ptr(dv, C.c_int32),
                                           7, None) == N.VCS_EINVAL
    dv[1] = 99
    assert N.lib().vcs_solve_multi_enqueue(sp.handle, C.byref(opts), 2, N.ptr(dv, C.c_int32),
                                           0, None) == N.VCS_EINVAL


@pytest.mark.parametrize("discount", [1.0, 0.9])
def test_multi_random_instances_against_oracle(gpu, oracle, monkeypatch, discount):
    """Random instances with retiring clouds (the transitions the halo cannot bound take the
    whole-layer exchange) and the labelled discounted extension: the multi-GPU pass at 2-5
    emulated ranks, every layer split, equals the oracle bit for bit."""
    from conftest import bits
    monkeypatch.setenv("VCS_MULTI_MIN_SPLIT", "1")
    for trial in range(4):
        ni = V.generate_instance(N.VCS_GEN_RANDOM, 41, trial, 5, 6, 18, 3, as_objects=False)
        sp = V.StateSpace.build_native(ni, 10**9)
        osp = oracle.build(ni.ref, 10**9)
        v, a, sw, _, _ = osp.vi(discount=discount)
        for ranks in (2, 5):
            opts = N.vcs_solve_opts(1e-6, 1, 0, discount, N.VCS_METHOD_CERTIFIED)
            vals = np.empty(sp.size())
            acts = np.empty(sp.size(), np.int32)
            rep = N.vcs_solve_report()
            dv = np.zeros(ranks, np.int32)
            N.check(N.lib().vcs_solve_multi(sp.handle, C.byref(opts), ranks, N.ptr(dv, C.c_int32),
                                            N.VCS_EXCHANGE_HALO, N.ptr(vals, C.c_double),
                                            N.ptr(acts, C.c_int32), C.byref(rep)))
            assert rep.sweeps == sw, (trial, ranks)
            assert np.array_equal(bits(vals), bits(v)), (trial, ranks)
            assert np.array_equal(acts, a), (trial, ranks)
