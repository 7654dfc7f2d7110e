"""Data-parallel plumbing on CPU (gloo, world size 2): every rank measures a
different cost table, agree_cost_table makes them identical, and the DELTA
plans (a pure function of trace + config) come out identical on every rank;
allreduce_mean averages gradients."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2203_15980_b200 import graph as G
        from paper_2203_15980_b200 import planner as P
        from paper_2203_15980_b200.runtime import agree_cost_table, allreduce_mean, apply_anchors
        g = G.build_resnet(50, 64)
        apply_anchors(g, "out+narrow")
        G.estimate_costs(g)
        for i, n in enumerate(g.nodes):  # rank-dependent "measurements"
            n.cost_us += (i * 7 + rank * 13) % 5
        link = agree_cost_table(g, 50.0 + rank, dist.group.WORLD)
        t = G.to_trace(g)
        cm = P.CostModel((int(link * 1e3), 1), (1, 1))
        base = P.run_unconstrained_baseline(t, P.EngineConfig(cost_model=cm))
        prog = P.Program(t, P.EngineConfig(budget=base.peak_bytes // 2, cost_model=cm))
        mine = ([n.cost_us for n in g.nodes], link, prog.decisions, prog.arena_bytes,
                prog.actions.tobytes())
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        grad = torch.full((1000,), float(rank + 1))
        allreduce_mean(grad, dist.group.WORLD)
        q.put((rank, all(v == allv[0] for v in allv), link, float(grad[0]),
               prog.infeasible is None))
    finally:
        dist.destroy_process_group()


def test_ranks_agree_on_costs_and_plans():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert len(res) == world
    for rank, same, link, g0, feasible in res:
        assert same, f"rank {rank} disagrees"
        assert link == 50.0
        assert g0 == 1.5
        assert feasible
