"""The reference's OWN solver suites (test_workload.cpp, test_greedy.cpp, test_mdp.cpp,
test_parallel.cpp — compiled unchanged from /root/reference by the Makefile into
oracle/_ref/ref_suite_on_b200) and its acceptance suite (acceptance.cpp ->
oracle/_ref/acceptance_on_b200) run against the B200 drop-in shim libvcsched_b200.so."""
from __future__ import annotations

import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SUITE = ROOT / "oracle" / "_ref" / "ref_suite_on_b200"
ACCEPT = ROOT / "oracle" / "_ref" / "acceptance_on_b200"


def test_reference_suites_pass_on_b200(gpu):
    if not SUITE.exists():
        pytest.fail(f"{SUITE} missing: build it with `make ref` where /root/reference exists")
    r = subprocess.run([str(SUITE)], cwd=ROOT, capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "| 0 failed |" in r.stdout


def test_reference_suites_pass_with_emulated_ranks(gpu):
    """VCS_EMULATE_RANKS=1: parallel_value_iteration(n) runs n ranks of the multi-GPU certified
    pass (round robin over the visible GPUs), so test_parallel.cpp's bit-identity checks for
    1..8 workers exercise the sharded path even on one B200."""
    import os
    if not SUITE.exists():
        pytest.fail(f"{SUITE} missing")
    env = dict(os.environ, VCS_EMULATE_RANKS="1", VCS_MULTI_MIN_SPLIT="16")
    r = subprocess.run([str(SUITE)], cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "| 0 failed |" in r.stdout


@pytest.mark.parametrize("emulate", [False, True])
def test_reference_acceptance_suite_on_b200(gpu, emulate):
    """acceptance.cpp criteria 1-5 (the solver path: canonical 116 / 202.4 / 58 / 0 within 10 s,
    100 % utilisation, brute-force optimality on 200 instances within 30 s, optimal >= greedy,
    bit-identity across 1/2/4/8 workers) — plus 6-9 on the reference's own simulator sources."""
    import os
    if not ACCEPT.exists():
        pytest.fail(f"{ACCEPT} missing: build it with `make ref` where /root/reference exists")
    env = dict(os.environ)
    if emulate:
        env.update(VCS_EMULATE_RANKS="1", VCS_MULTI_MIN_SPLIT="16")
    r = subprocess.run([str(ACCEPT)], cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env=env)
    print(r.stdout[-4000:], r.stderr[-4000:])
    for k in range(1, 6):
        assert f"[PASS] criterion {k}:" in r.stdout, r.stdout
    assert r.returncode == 0, r.stdout
