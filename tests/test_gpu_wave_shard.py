"""GPU: the version-band sharded wavefront (vcs_wave_shard_*) with 1..7 ranks EMULATED in one
process (one space per rank on one stream; the column exchange is a device copy), bit-exact
against the reference's golden digests — including early stops, where the fix-up is split
between the owners of version K* of layers t and t+1."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2012_12419_b200 as V
from paper_2012_12419_b200 import _native as N
from paper_2012_12419_b200.sharded import WaveBandCuda, band, halo_schedule, run_wave_emulated
from cases import FAMILIES, GOLDEN
from conftest import sha

pytestmark = pytest.mark.gpu


def _solve_emulated(ni, world, eps):
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    spaces = [V.StateSpace.build_native(ni, 10**9) for _ in range(world)]
    backends = [WaveBandCuda(sp, dev, stream) for sp in spaces]
    opts = N.vcs_solve_opts(eps, 1, 0, 1.0, N.VCS_METHOD_WAVEFRONT)
    with torch.cuda.stream(stream):
        return run_wave_emulated(backends, spaces[0].layer_offsets(), opts)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 7])
def test_band_sharded_canonical(gpu, golden, world):
    p = V.load_instance(str(GOLDEN / "canonical_instance.txt"))
    ni = V.NativeInstance(p.vcc, bots=p.bots)
    for eps in (1e-6, 5.0, 0.5):
        g = golden["cases"]["canonical"][f"eps={eps:g}"]
        values, actions, K = _solve_emulated(ni, world, eps)
        assert K == g["sweeps"]
        assert sha(values) == g["values_sha"], (world, eps)
        assert sha(actions) == g["actions_sha"], (world, eps)


@pytest.mark.parametrize("world", [2, 5])
def test_band_sharded_families(gpu, golden, world):
    for family in ("acc5_seed3003", "par_seed47"):
        seed, params, n, _ = FAMILIES[family]
        for trial in range(0, n, 5):
            ni = V.generate_instance(N.VCS_GEN_RANDOM, seed, trial, *params, as_objects=False)
            values, actions, K = _solve_emulated(ni, world, 1e-6)
            g = golden["families"][family][trial]["eps=1e-06"]
            assert K == g["sweeps"]
            assert sha(values) == g["values_sha"] and sha(actions) == g["actions_sha"]


def test_band_sharded_c3(gpu, golden):
    ni = V.generate_instance(N.VCS_GEN_HOMOG, 2012, 0, 5, 8, 40, 3, as_objects=False)
    values, actions, K = _solve_emulated(ni, 4, 1e-6)
    g = golden["cases"]["C3"]["eps=1e-06"]
    assert K == 41 and sha(values) == g["values_sha"] and sha(actions) == g["actions_sha"]


def test_band_plan_matches_library(gpu):
    """The Python mirror of the band formula (used for the exchange schedule) agrees with the
    library's plan, and the schedule only ever asks for versions the sender holds."""
    p = V.load_instance(str(GOLDEN / "canonical_instance.txt"))
    ni = V.NativeInstance(p.vcc, bots=p.bots)
    sp = V.StateSpace.build_native(ni)
    H = sp.task_count()
    import ctypes as C
    delta = torch.zeros(H + 3, dtype=torch.float64, device="cuda")
    for world in (2, 3, 8):
        for r in range(world):
            opts = N.vcs_solve_opts(1e-6, 1, 0, 1.0, N.VCS_METHOD_WAVEFRONT)
            N.check(N.lib().vcs_wave_shard_begin(sp.handle, world, r, C.byref(opts),
                                                 C.c_void_p(delta.data_ptr()), None))
            for t in range(H + 1):
                lo, hi = C.c_int32(), C.c_int32()
                N.check(N.lib().vcs_wave_shard_band(sp.handle, t, C.byref(lo), C.byref(hi)))
                assert (lo.value, hi.value) == band(H - t, r, world)
        for t in range(H):
            for src, dst, v in halo_schedule(H, world, t):
                lo, hi = band(H - t, src, world)
                assert lo <= v < hi and v == band(H - t, dst, world)[0] - 1
