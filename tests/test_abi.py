"""The C-ABI library loads and exports every symbol include/vcs_gpu.h declares (CPU only: no
compute call needs a GPU here)."""
from __future__ import annotations

import ctypes as C
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2012_12419_b200 import _native as N

HEADER = ROOT / "include" / "vcs_gpu.h"


def header_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vcs_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_bound_symbols():
    assert header_functions() == sorted(N.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    for name in header_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [f for f in header_functions() if f not in exported]
    assert not missing, missing


def test_library_is_built_for_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_host_only_calls_work_without_gpu():
    assert N.kernel_launches() >= 0
    assert N.device_count() >= 0
    assert N.last_error() is not None


def test_reference_and_oracle_libraries_load(oracle, reference):
    assert oracle.L.orc_build
    assert reference.threads() >= 1


@pytest.mark.skipif(N.device_count() > 0, reason="checks the no-GPU failure mode")
def test_device_calls_fail_loudly_without_gpu():
    import paper_2012_12419_b200 as V
    from cases import tiny
    vcc, bots = tiny(2, [1, 1, 1])
    with pytest.raises(N.CudaError, match="no CUDA device"):
        V.value_iteration(V.MdpInstance.from_workload(vcc, bots))
    with pytest.raises(N.CudaError):
        V.greedy_schedule(vcc, bots)
