"""Multi-rank remap on CPU: world_size 2 and 4 processes over torch.distributed
(gloo), one library context per rank (host-only: plan + exchange schedule).

What is checked is the N > 1 data path's host logic -- which blocks each
rank sends, to whom, and where they land (Alg. Execute's Shard, P:L1312,
P:L1367-1371): each rank starts from its shard of the exact state
at the end of stage k-1 (oracle O1, laid out by the plan's sigma/flips),
applies the plan's local pack permutation, performs the library's own
exchange schedule (atlas_remap_schedule -- the transfers atlas_run hands to
NCCL) with gloo isend/irecv, and must end with exactly (bit for bit) its
shard of the same state in stage k's layout.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import remap as R
from oracle import sim as O
from workloads import circuits as C

A = pytest.importorskip("paper_2408_09055_b200.atlas")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _layout(psi, sigma, flips):
    fm = 0
    for q, f in enumerate(flips):
        fm |= int(f) << sigma[q]
    return R.to_physical(psi, sigma, fm)


def _pack(shard, newpos):
    L = len(newpos)
    i = np.arange(1 << L, dtype=np.int64)
    o = np.zeros_like(i)
    for b in range(L):
        o |= ((i >> b) & 1) << newpos[b]
    out = np.empty_like(shard)
    out[o] = shard
    return out


def _circuit(name, n):
    if name.startswith("random"):
        return C.random_circuit(n, 60, int(name[6:]))
    return C.make(name, n)


def _worker(rank, world, port, name, n, res):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = _circuit(name, n)
        with A.Simulator(n, 0, world, rank) as s:  # host-only: no nccl_uid needed
            s.load_circuit(c.gates)
            s.plan()
            pj = s.plan_json()
            sched = {k: s.remap_schedule(k) for k in range(1, pj["staging"]["s"])}
        L = n - int(math.log2(world))
        lo, hi = rank << L, (rank + 1) << L
        gs = pj["staging"]["gate_stage"]
        st = pj["stages"]
        checked = 0
        for k in range(1, len(st)):
            if st[k]["remap_qubits"] == 0:
                continue
            psi = O.simulate(C.Circuit(n, [g for g, sk in zip(c.gates, gs) if sk < k]))
            shard = _layout(psi, st[k - 1]["sigma"], st[k - 1]["flip_end"])[lo:hi].copy()
            if st[k]["pack_newpos"] is not None:
                shard = _pack(shard, st[k]["pack_newpos"])
            src = torch.from_numpy(shard.view(np.uint8).copy())
            dst = torch.zeros_like(src)
            reqs = []
            for kind, peer, so, do, nb in sched[k]:
                if kind == "local":
                    dst[do:do + nb] = src[so:so + nb]
                elif kind == "send":
                    reqs.append(dist.isend(src[so:so + nb].clone(), peer))
                else:
                    buf = torch.empty(nb, dtype=torch.uint8)
                    reqs.append((dist.irecv(buf, peer), buf, do))
            for r in reqs:
                if isinstance(r, tuple):
                    r[0].wait()
                    dst[r[2]:r[2] + len(r[1])] = r[1]
                else:
                    r.wait()
            got = dst.numpy().view(np.complex128)
            want = _layout(psi, st[k]["sigma"], st[k]["flip_begin"])[lo:hi]
            assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), \
                f"rank {rank} stage {k}: remap result differs"
            checked += 1
        res[rank] = checked
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,name,n", [
    (2, "qft", 9), (2, "su2random", 8), (4, "su2random", 9), (4, "random3", 9),
    (4, "random4", 10), (4, "random17", 10), (2, "ising", 9), (4, "wstate", 9)])
def test_remap_exchange_gloo(world, name, n):
    ctx = mp.get_context("spawn")
    res = ctx.Manager().dict()
    mp.start_processes(_worker, args=(world, _free_port(), name, n, res), nprocs=world,
                       join=True, start_method="spawn")
    assert len(res) == world
    assert all(v >= 1 for v in res.values()), dict(res)
