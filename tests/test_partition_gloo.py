"""Host-side logic of the partitioned (multi-GPU) path, on CPU
with torch.distributed over gloo, world_size 2 and 4 (no GPU).

Each rank asks the library (host-only calls, include/mgdtn.h
mg_partition_plan / mg_partition_side_edges -- the same level structure and
halo ordering the CUDA path and the NCCL exchange use) for its decomposition,
then:
  1. the ranks agree on the hierarchy and the gather level, and every
     interface side's global edge list equals the neighbour's matching side,
     in the same order (the message layout of the halo exchange);
  2. a distributed trace apply built ONLY from that plan -- each rank applies
     its own elements' oracle DtN maps in its local numbering, exchanges the
     interface partial sums with its neighbours over gloo in the plan's side
     order, and adds them -- equals the oracle's global assembled apply;
  3. owned-dof dot products (the rank below / left owns an interface edge),
     all-reduced, equal the global dot product.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as W
from oracle import assembly
from oracle import element as el
from oracle import mesh

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_1811_09909_b200", "libmgdtn.so")
pytestmark = pytest.mark.skipif(not os.path.exists(LIB), reason="libmgdtn.so not built")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _local_edges(bx, by, il, jl):
    """{bottom, right, top, left} local edge ids of local element (il, jl) (header numbering)."""
    return [jl * bx + il, bx * (by + 1) + jl * (bx + 1) + il + 1, (jl + 1) * bx + il,
            bx * (by + 1) + jl * (bx + 1) + il]


def _worker(rank, world, port, n, p, px, py, gather_ne, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1811_09909_b200 import Partition, partition_plan, partition_side_edges
        part = Partition(rank, world, px, py, gather_ne=gather_ne)
        plan = partition_plan(n, n, p, part)
        # 1. plans agree; interface sides pair up edge by edge
        plans = [None] * world
        dist.all_gather_object(plans, (plan["nlevels"], plan["gather_level"]))
        assert all(pl == plans[0] for pl in plans), plans
        N, Lg = plan["nlevels"], plan["gather_level"]
        sides = {}
        for lev in range(Lg + 1, N + 1):
            for f in range(4):
                sides[(lev, f)] = partition_side_edges(n, n, p, part, lev, f).tolist()
        allsides = [None] * world
        dist.all_gather_object(allsides, sides)
        rx, ry = rank % px, rank // px
        nbr = [rank - px if ry > 0 else -1, rank + 1 if rx < px - 1 else -1,
               rank + px if ry < py - 1 else -1, rank - 1 if rx > 0 else -1]
        for lev in range(Lg + 1, N + 1):
            L = plan["levels"][lev - 1]
            for f in range(4):
                mine = sides[(lev, f)]
                if nbr[f] < 0:
                    assert not mine and not ((L["imask"] >> f) & 1)
                    assert (L["dmask"] >> f) & 1
                    continue
                assert (L["imask"] >> f) & 1
                theirs = allsides[nbr[f]][(lev, (f + 2) % 4)]
                assert mine == theirs and len(mine) > 0, (lev, f)
        # 2. distributed apply on the finest level from the plan + gloo halo sums
        cfg = W.scaled_config(4, n) if p == 3 else W.scaled_config(2, n)
        pr = W.make_problem(cfg, with_f=False)
        L = plan["levels"][N - 1]
        bx, by, ox, oy = L["nx"], L["ny"], L["ox"], L["oy"]
        k1 = p + 1
        jj, ii = np.divmod(np.arange(bx * by), bx)
        ge = (oy + jj) * n + (ox + ii)
        S = el.element_dtn(p, pr.K[ge], pr.method[ge], pr.tau[ge], 1.0 / n)
        gid = W.dof_ids(W.block_edge_ids_at(n, ox, oy, bx, by), p)
        x = W.random_trace_vector(mesh.n_edges(n) * k1, 77)
        xl = x[gid]
        yl = np.zeros_like(xl)
        for t in range(bx * by):
            d = np.concatenate([np.arange(e * k1, (e + 1) * k1)
                                for e in _local_edges(bx, by, ii[t], jj[t])])
            yl[d] += S[t] @ xl[d]
        # halo: per interface side, the partial sums in side order, one message per neighbour
        loc_side = {0: [jl for jl in range(bx)], 2: [by * bx + i for i in range(bx)],
                    3: [bx * (by + 1) + j * (bx + 1) for j in range(by)],
                    1: [bx * (by + 1) + j * (bx + 1) + bx for j in range(by)]}
        reqs, recvd = [], {}
        for f in range(4):
            if nbr[f] < 0:
                continue
            idx = np.concatenate([np.arange(e * k1, (e + 1) * k1) for e in loc_side[f]])
            send = torch.from_numpy(yl[idx].copy())
            recv = torch.empty_like(send)
            reqs.append(dist.isend(send, nbr[f]))
            reqs.append(dist.irecv(recv, nbr[f]))
            recvd[f] = (idx, recv)
        for r in reqs:
            r.wait()
        for f, (idx, recv) in recvd.items():
            yl[idx] = yl[idx] + recv.numpy()
        A = assembly.assemble_full(n, p, el.element_dtn(p, pr.K, pr.method, pr.tau, 1.0 / n))
        yg = A @ x
        err = np.linalg.norm(yl - yg[gid]) / np.linalg.norm(yg[gid])
        assert err <= 1e-13, err
        # 3. owned dots: skip bottom / left interface sides (the rank below / left owns them)
        own = np.ones(len(xl), bool)
        for f in (0, 3):
            if nbr[f] >= 0:
                own[np.concatenate([np.arange(e * k1, (e + 1) * k1) for e in loc_side[f]])] = False
        t = torch.tensor([float(xl[own] @ yl[own])], dtype=torch.float64)
        dist.all_reduce(t)
        ref = float(x @ yg)
        assert abs(t.item() - ref) <= 1e-12 * abs(ref), (t.item(), ref)
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("world,px,py,n,p,gne", [(2, 2, 1, 16, 4, 16), (2, 1, 2, 16, 3, 0),
                                                   (4, 2, 2, 32, 4, 16)])
def test_partition_plan_and_halo_gloo(world, px, py, n, p, gne):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, p, px, py, gne, q))
             for r in range(world)]
    for pr_ in procs:
        pr_.start()
    res = [q.get(timeout=300) for _ in procs]
    for pr_ in procs:
        pr_.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res
