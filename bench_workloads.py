"""The benchmark workloads of BASELINE.json / SURVEY 8(d), as instance TEXT in the reference's
input grammar (io.hpp:33-40), so that both bench arms read the same bytes through their own
parser: the B200 arm through vcs_instance_parse / vcs_instance_load (the product), the reference
arm through io.cpp parse_instance / load_instance (oracle/_ref/libvcsref.so).

Pure Python, no product or oracle import (the reference arm must not load libvcs_gpu.so).

  c1  data/canonical_instance.txt of the reference (tests/golden/canonical_instance.txt):
      11 clouds, 330 unit tasks; S = 68,797, 331 sweeps (configs[0])
  c2  greedy first-fit, 1,000 clouds x 10^5 tasks (seed 12345): generated, not text (configs[1])
  c3  5 clouds x 8 VMs, 40 tasks demand U[1,3], seed 2012: S = 1,788,700 (configs[2])
  c4  6 clouds x 8 VMs, 48 tasks demand U[1,3], seed 2012: S = 19,333,781 (configs[3])
  c5  density / channel-availability sweep (configs[4]), see c5_text()
  c7  7 clouds x 8 VMs, 56 tasks demand U[1,3], seed 2012: the size where the certified pass is
      bound by HBM rather than L2 (no reference timing: its hash-map build would take minutes)
"""
from __future__ import annotations

import json
from pathlib import Path

ROOT = Path(__file__).resolve().parent
INSTANCES = ROOT / "tests" / "golden" / "instances"

FILES = {
    "c1": ROOT / "tests" / "golden" / "canonical_instance.txt",
    "c3": INSTANCES / "c3.txt",
    "c4": INSTANCES / "c4.txt",
    "c7": INSTANCES / "c7.txt",
}
DESCRIPTIONS = {
    "c1": "C1: canonical instance (reference data/canonical_instance.txt), 11 clouds, 330 unit tasks",
    "c2": "C2: greedy first-fit, 1000 clouds x U[50,150] VMs, 10^5 tasks demand U[1,3] (seed 12345)",
    "c3": "C3: 5 clouds x 8 VMs, 40 tasks demand U[1,3] (mt19937_64 seed 2012), 5 bags",
    "c4": "C4: 6 clouds x 8 VMs, 48 tasks demand U[1,3] (mt19937_64 seed 2012), 6 bags",
    "c7": "C7: 7 clouds x 8 VMs, 56 tasks demand U[1,3] (mt19937_64 seed 2012), 7 bags "
          "(HBM-bound: a layer's pair vector is 76 MB, two exceed the 126 MB L2)",
}
# C2 through the seeded generator (kind 2 = VCS_GEN_GREEDY): seed, clouds, bags, tasks/bag, demand
C2_GEN = (2, 12345, 1000, 100, 1000, 3)

# ---- C5: vehicle-count / RSU-coverage density sweep with the two channel schemes -------------
C5_CLOUDS = tuple(range(3, 8))   # K: RSUs (vehicular clouds)
C5_VMS = tuple(range(4, 13))     # c: vehicles (one VM each) per cloud
C5_SCHEMES = ("static1609", "aaa")
C5_MIN_THR = (30.0, 50.0, 90.0)  # task throughput thresholds, cycled over the task sequence


def channel_table() -> dict:
    """Per-vehicle service-channel kbps of the reference's DSRC simulator at n = 1..128 vehicles,
    tabulated once from the unmodified reference by tools/c5_channel_table.py."""
    doc = json.loads((ROOT / "tests" / "golden" / "c5_channel.json").read_text())
    return doc["per_vehicle_kbps"]


def _fmt(v: float) -> str:
    return "%.17g" % float(v)


def c5_text(K: int, c: int, scheme: str, table: dict | None = None) -> str:
    """One C5 point (the coupling is builder-defined, the reference's `benchmark`
    never feeds the channel model into the solver, tools/cli.cpp:132-197).

    * K clouds; cloud k (0-based) has c VMs (one per vehicle), v2i delay 10 + 5k ms and an RSU
      coverage density of n_k = c*(k+1) vehicles sharing the channel; its vm_throughput_kbps is
      the simulator's per-vehicle share at n_k under `scheme` (static1609 or aaa).
    * H = floor(K*c/2) unit-demand tasks (max_delay 100 ms) whose min_thr cycles through
      30 / 50 / 90 kbps, dealt into K bags round-robin.  A cloud is eligible for a task iff its
      share meets the threshold, so the scheme changes eligibility and with it the state space.
    * beta_vc = 1, beta_tc = 1.2, gamma_vc = 1 (the reference defaults, workload.hpp:40-42).
    """
    table = table or channel_table()
    kbps = table[scheme]
    lines = [f"# C5 point K={K} c={c} scheme={scheme}", "beta_vc 1", "beta_tc 1.2", "gamma_vc 1"]
    for k in range(K):
        n = min(c * (k + 1), len(kbps))
        lines.append(f"cloud {k + 1} {c} {_fmt(kbps[n - 1])} {_fmt(10 + 5 * k)}")
    H = (K * c) // 2
    bags = [[] for _ in range(K)]
    for j in range(H):
        bags[j % K].append(f"task {j + 1} 1 100 {_fmt(C5_MIN_THR[j % len(C5_MIN_THR)])}")
    for b in range(K):
        lines.append(f"bot {b + 1}")
        lines.extend(bags[b])
    return "\n".join(lines) + "\n"


def c5_points():
    return [(K, c, s) for K in C5_CLOUDS for c in C5_VMS for s in C5_SCHEMES]


def instance_text(name: str) -> str:
    return FILES[name].read_text()
