"""The multi-PROCESS form of the certified pass (vcs_cert_shard_*, driven by
sharded.run_cert_sharded under torchrun) on one B200: world-1 through a real NCCL group, and
2-4 ranks emulated in one process — one state space per rank, the windows moved by device
copies exactly as run_cert_sharded moves them with send/recv (no kernel waits on another rank).
Results must equal the reference's golden digests."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

import paper_2012_12419_b200 as V
from paper_2012_12419_b200 import _native as N
from paper_2012_12419_b200.sharded import CertShardCuda
from cases import GOLDEN
from conftest import sha

pytestmark = pytest.mark.gpu


def _space(name):
    path = {"C3": GOLDEN / "instances" / "c3.txt", "C4": GOLDEN / "instances" / "c4.txt",
            "canonical": GOLDEN / "canonical_instance.txt"}[name]
    p = V.load_instance(str(path))
    return V.StateSpace.build_native(V.NativeInstance(p.vcc, bots=p.bots), 10**9)


def _emulated(name, world, eps, exchange):
    """All ranks in one process on cuda:0 (run_cert_sharded's protocol, copies for send/recv)."""
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    spaces = [_space(name) for _ in range(world)]
    bes = [CertShardCuda(sp, dev, stream, exchange) for sp in spaces]
    opts = N.vcs_solve_opts(eps, 1, 0, 1.0, N.VCS_METHOD_CERTIFIED)
    H = bes[0].H
    with torch.cuda.stream(stream):
        for r, be in enumerate(bes):
            be.begin(world, r, opts)
        moved = 0
        for t in range(H - 1, -1, -1):
            for be in bes:
                be.layer(t)
            plans = [bes[0].plan(t, q) for q in range(world)]
            if t == 0 or not plans[0][0]:
                continue
            for q in range(world):  # owner q -> reader h
                for h in range(world):
                    if h == q:
                        continue
                    x, y = max(plans[h][3], plans[q][1]), min(plans[h][4], plans[q][2])
                    if x < y:
                        src = bes[q].pairs(t, plans[q][5])
                        dst = bes[h].pairs(t, plans[h][5])
                        dst[2 * x:2 * y].copy_(src[2 * x:2 * y])
                        moved += 16 * (y - x)
        lbs = [be.buffers()[0] for be in bes]
        lb = torch.stack(lbs).max(dim=0).values
        certified = bes[0].finish(lb.cpu().numpy())
        torch.cuda.synchronize()
        if not certified:
            v, a, K = bes[0].fallback(opts)
            return v, a, K, False, moved
        vals = sum(be.buffers()[1].view(torch.int64) for be in bes)
        acts = sum(be.buffers()[2] for be in bes)
        torch.cuda.synchronize()
    return (vals.view(torch.float64).cpu().numpy(), acts.cpu().numpy(), H + 1, True, moved)


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_cert_shard_emulated_matches_golden(gpu, golden, monkeypatch, name):
    monkeypatch.setenv("VCS_MULTI_MIN_SPLIT", "4096")
    g = golden["cases"][name]["eps=1e-06"]
    for world in (2, 3, 4):
        for ex in (N.VCS_EXCHANGE_HALO, N.VCS_EXCHANGE_ALLGATHER):
            v, a, K, cert, moved = _emulated(name, world, 1e-6, ex)
            assert cert and K == g["sweeps"]
            assert sha(v) == g["values_sha"], (world, ex)
            assert sha(a) == g["actions_sha"], (world, ex)
            assert moved > 0


def test_cert_shard_emulated_canonical_fallback(gpu, golden, monkeypatch):
    monkeypatch.setenv("VCS_MULTI_MIN_SPLIT", "64")
    for eps in (1e-6, 5.0):
        g = golden["cases"]["canonical"][f"eps={eps:g}"]
        v, a, K, cert, _ = _emulated("canonical", 3, eps, N.VCS_EXCHANGE_HALO)
        assert cert == (eps == 1e-6)
        assert K == g["sweeps"]
        assert sha(v) == g["values_sha"] and sha(a) == g["actions_sha"]


def test_run_cert_sharded_nccl_world1(gpu, golden):
    """The torchrun driver itself through a 1-rank NCCL process group."""
    import torch.distributed as dist
    from paper_2012_12419_b200.sharded import run_cert_sharded
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        sp = _space("C4")
        be = CertShardCuda(sp, dev)
        opts = N.vcs_solve_opts(1e-6, 1, 0, 1.0, N.VCS_METHOD_CERTIFIED)
        v, a, K = run_cert_sharded(be, opts)
        g = golden["cases"]["C4"]["eps=1e-06"]
        assert K == g["sweeps"] and sha(v) == g["values_sha"] and sha(a) == g["actions_sha"]
    finally:
        dist.destroy_process_group()
