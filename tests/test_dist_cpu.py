"""world_size-2 host-side tests on CPU (gloo): NCCL-id bootstrap through torch.distributed and
SPMD-identical plans on every rank (the structure NCCL exchanges rely on)."""
from __future__ import annotations

import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import paper_2504_17881_b200 as P
    from paper_2504_17881_b200 import ps
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nid = ps.bootstrap_nccl_id(rank)
        ids = [None] * world
        dist.all_gather_object(ids, nid)
        n = 12
        codes, ang = workloads.random_layer(n, 200, seed=3, kind="R10")
        codes[::5, n - 1] = 1  # X on the global qubit
        x, z = P.pauli_encode_codes(codes)
        ops, rots = P.plan_describe(n, x, z, ang, world=world, rank=rank, fusion=2, tile_bits=8)
        struct = [(o["kind"], o["exch_bit"], o["exch_gx"], o["first_rot"], o["n_rot"]) for o in ops]
        assert any(o["kind"] == 5 for o in ops)
        xs = [(r["x"], r["z"], r["y"]) for r in rots]
        signs = [r["sign"] for r in rots]
        allst = [None] * world
        dist.all_gather_object(allst, (struct, xs, signs))
        q.put((rank, ids, allst))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_bootstrap_and_spmd_plans():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ids, allst in res:
        assert len(set(ids)) == 1 and len(ids[0]) == 128  # every rank holds rank 0's id
        (s0, x0, g0), (s1, x1, g1) = allst
        assert s0 == s1  # identical op sequence (kinds, pivots, partners, rotation ranges)
        assert x0 == x1  # identical physical masks
        assert any(a != b for a, b in zip(g0, g1))  # per-rank signs differ where z touches the top qubit
        assert any(k == 5 for k, *_ in s0)  # the plan contains exchanges
