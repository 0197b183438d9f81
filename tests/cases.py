"""Instances shared by the golden generator and the parity tests.

Named cases restate the reference's hand-built test instances (tests/test_mdp.cpp:17-27 tiny,
:74-116 tie-break / empty, test_greedy.cpp:13-36 single-cloud cases) and the canonical fixture
(data/canonical_instance.txt, copied to tests/golden/).  FAMILIES are the seeded random
families of the reference suites: (seed, InstanceParams{max_clouds, max_cloud_cap, max_tasks,
max_demand}, trials, brute-force checked).
"""
from __future__ import annotations

from pathlib import Path

import paper_2012_12419_b200 as V

GOLDEN = Path(__file__).resolve().parent / "golden"

FAMILIES = {
    "acc3_seed1001": (1001, (3, 6, 8, 3), 200, True),    # acceptance.cpp:104-115
    "acc4_seed2002": (2002, (6, 5, 50, 3), 100, False),  # acceptance.cpp:117-127
    "acc5_seed3003": (3003, (4, 5, 25, 3), 50, False),   # acceptance.cpp:129-150
    "par_seed47": (47, (4, 6, 25, 3), 25, False),         # test_parallel.cpp:89-106
    "mdp_seed23": (23, (3, 6, 8, 3), 40, True),           # test_mdp.cpp:182-191
    "mdp_seed29": (29, (5, 8, 30, 3), 40, False),         # test_mdp.cpp:193-202
    "mdp_seed31": (31, (4, 7, 20, 3), 30, False),         # test_mdp.cpp:204-214
    "mdp_seed37": (37, (3, 6, 12, 3), 20, False),         # test_mdp.cpp:216-236
    "mdp_seed41": (41, (4, 6, 25, 3), 20, False),         # test_mdp.cpp:238-246
    "par_seed43": (43, (4, 6, 20, 3), 1, False),          # test_parallel.cpp:64-74
    "grd_seed17": (17, (5, 8, 25, 3), 100, False),        # test_greedy.cpp:73-93
}


def cloud(cid, total, thr, delay, free=None):
    return V.VehicularCloud(cid, total, total if free is None else free, thr, delay)


def tiny(cap, demands):
    """test_mdp.cpp:17-27."""
    vcc = V.VccModel([cloud(1, cap, 100.0, 10.0)], 1.0, 1.2, 1.0)
    bots = [V.BagOfTasks(1, [V.Task(i + 1, d, 50.0, 50.0) for i, d in enumerate(demands)])]
    return vcc, bots


def named_workloads():
    """name -> (vcc, bots, eps_list)."""
    w = {}
    p = V.load_instance(str(GOLDEN / "canonical_instance.txt"))
    w["canonical"] = (p.vcc, p.bots, (1e-6, 5.0, 0.5))
    w["tiny_2vm_3tasks"] = (*tiny(2, [1, 1, 1]), (1e-6,))
    w["tiny_drain"] = (*tiny(5, [5]), (1e-6,))
    w["tiny_over_capacity"] = (*tiny(3, [5]), (1e-6,))
    w["tiny_sign"] = (*tiny(10, [5, 10]), (1e-6,))
    w["terminal_penalty"] = (*tiny(27, [27]), (1e-6,))
    w["tie_single_paid"] = (V.VccModel([], 1.0, 1.2, 1.0),
                            [V.BagOfTasks(1, [V.Task(1, 1, 50.0, 50.0)])], (1e-6,))
    w["tie_two_branch"] = (*tiny(1, [1]), (1e-6,))
    w["tie_symmetric"] = (V.VccModel([cloud(1, 2, 100.0, 10.0), cloud(2, 2, 100.0, 10.0)]),
                          [V.BagOfTasks(1, [V.Task(1, 1, 50.0, 50.0)])], (1e-6,))
    w["empty_tasks"] = (V.VccModel([cloud(1, 4, 100.0, 10.0)]), [], (1e-6,))
    w["cap_six_units"] = (*tiny(6, [1] * 6), (1e-6,))
    w["greedy_fill_one"] = (V.VccModel([cloud(1, 5, 100.0, 10.0)]),
                            [V.BagOfTasks(1, [V.Task(t + 1, 1, 50.0, 50.0) for t in range(5)])],
                            (1e-6,))
    w["greedy_all_paid"] = (V.VccModel([cloud(1, 10, 100.0, 500.0)]),
                            [V.BagOfTasks(1, [V.Task(t + 1, 1, 50.0, 50.0) for t in range(4)])],
                            (1e-6,))
    vcc, bots = tiny(2, [1, 1, 1])
    vcc.reward_per_vc_vm, vcc.cost_per_tcc_vm, vcc.penalty_per_idle_vm = 0.0, 0.0, 0.0
    w["zero_rates_signed_zero"] = (vcc, bots, (1e-6,))
    return w


def named_cases():
    """name -> (NativeInstance, eps_list)."""
    return {k: (V.NativeInstance(vcc, bots=bots), eps) for k, (vcc, bots, eps) in
            named_workloads().items()}
