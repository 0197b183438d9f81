"""The CLI's schedule / speedup subcommands (paper_2012_12419_b200/vcsched-b200, the reference's
tools/cli.cpp run_schedule / run_speedup over the drop-in shim, plus scheduler mdp-gpu).

CPU: argument and exit-code behaviour (tools/cli.hpp:30-33: 2 config, 3 cap, 4 io).
GPU: the schedule files are byte-identical to the reference's own io.cpp writers
(schedule_csv / schedule_json via oracle/_ref) for greedy and mdp; mdp-gpu adds its
SolverDiagnostics fields after the reference's."""
from __future__ import annotations

import ctypes as C
import json
import subprocess

import pytest

from conftest import ROOT

CLI = ROOT / "paper_2012_12419_b200" / "vcsched-b200"
CANON = ROOT / "tests" / "golden" / "canonical_instance.txt"


def run(*args, **kw):
    if not CLI.exists():
        pytest.fail(f"{CLI} missing: build it with `make`")
    return subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True,
                          timeout=600, **kw)


def test_cli_exit_codes():
    assert run().returncode == 2
    assert run("simulate", "--instance", CANON).returncode == 2
    assert run("schedule", "--instance", CANON, "--format", "xml").returncode == 2
    assert run("schedule", "--instance", CANON, "--workers", "x").returncode == 2
    r = run("schedule", "--instance", "/nonexistent/instance.txt")
    assert r.returncode == 4 and "cannot read instance file" in r.stderr
    assert run("schedule", "--instance", CANON, "--scheduler", "nope").returncode == 2


def _ref_text(reference, scheduler, fmt):
    f = reference.L.ref_schedule_text
    f.restype = C.c_uint64
    f.argtypes = [C.c_char_p, C.c_int, C.c_double, C.c_int, C.c_char_p, C.c_uint64]
    n = f(str(CANON).encode(), scheduler, 1e-6, fmt, None, 0)
    buf = C.create_string_buffer(int(n) + 1)
    f(str(CANON).encode(), scheduler, 1e-6, fmt, buf, n)
    return buf.raw[:n].decode()


@pytest.mark.gpu
@pytest.mark.parametrize("scheduler,code", [("greedy", 0), ("mdp", 1), ("mdp-parallel", 1)])
@pytest.mark.parametrize("fmt,fcode", [("csv", 0), ("json", 1)])
def test_cli_schedule_matches_reference_writers(gpu, reference, tmp_path, scheduler, code, fmt,
                                                fcode):
    out = tmp_path / f"s.{fmt}"
    r = run("schedule", "--instance", CANON, "--scheduler", scheduler, "--workers", 4,
            "--out", out, "--format", fmt)
    assert r.returncode == 0, r.stderr
    assert out.read_text() == _ref_text(reference, code, fcode)
    if scheduler != "greedy":
        assert "sweeps=331 states_explored=68797" in r.stdout


@pytest.mark.gpu
def test_cli_mdp_gpu_diagnostics(gpu, reference, tmp_path):
    out = tmp_path / "s.json"
    r = run("schedule", "--instance", CANON, "--scheduler", "mdp-gpu", "--gpus", 1,
            "--out", out, "--format", "json")
    assert r.returncode == 0, r.stderr
    got = json.loads(out.read_text())
    want = json.loads(_ref_text(reference, 1, 1))
    assert got["placements"] == want["placements"]
    for k, v in want["summary"].items():
        assert got["summary"][k] == v
    assert got["summary"]["solver"] == "b200-certified" and got["summary"]["gpus"] == 1
    assert got["summary"]["device_ms"] > 0
    csv_out = tmp_path / "s.csv"
    r = run("schedule", "--instance", CANON, "--scheduler", "mdp-gpu", "--out", csv_out)
    ref_csv = _ref_text(reference, 1, 0)
    assert csv_out.read_text().startswith(ref_csv)  # the B200 rows follow the reference's
    assert "summary,solver,b200-certified" in csv_out.read_text()
    # the state cap exits 3 with the reference's message
    r = run("schedule", "--instance", CANON, "--scheduler", "mdp-gpu", "--state-cap", 1000)
    assert r.returncode == 3 and "exceeds cap of 1000 states" in r.stderr


@pytest.mark.gpu
def test_cli_speedup_rows(gpu):
    r = run("speedup", "--instance", CANON)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0] == "workers,wall_ms,speedup_vs_one"
    assert [int(x.split(",")[0]) for x in lines[1:]] == [1, 2, 4, 8]
