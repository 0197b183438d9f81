"""The reference's OWN solver suites (test_workload.cpp, test_greedy.cpp, test_mdp.cpp,
test_parallel.cpp — compiled unchanged from /root/reference by the Makefile into
oracle/_ref/ref_suite_on_b200) run against the B200 drop-in shim libvcsched_b200.so."""
from __future__ import annotations

import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SUITE = ROOT / "oracle" / "_ref" / "ref_suite_on_b200"


def test_reference_suites_pass_on_b200(gpu):
    if not SUITE.exists():
        pytest.fail(f"{SUITE} missing: build it with `make ref` where /root/reference exists")
    r = subprocess.run([str(SUITE)], cwd=ROOT, capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "| 0 failed |" in r.stdout
