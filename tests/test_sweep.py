"""Multi-process host logic of the budget-sharded sweep (world_size 2, gloo,
CPU).  The per-rank solve is injected (the CPU oracle), so this covers the
sharding + gather path without a GPU; the GPU solve itself is covered by the
gpu-marked parity tests."""

from __future__ import annotations

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1905_11722_b200.sweep import shard, sweep_budgets


def test_shard_is_a_partition():
    items = list(range(64))
    for world in (1, 2, 3, 4, 8):
        parts = [shard(items, world, r) for r in range(world)]
        assert [x for p in parts for x in p] == items
        assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_sweep_budgets_endpoints():
    b = sweep_budgets(55, 385, 64)
    assert len(b) == 64 and b[0] == 55 and b[-1] == 385
    assert b == sorted(b)
    assert sweep_budgets(10, 10, 4) == [10] * 4


def _oracle_solve(g, budgets, family, objective, cap):
    from oracle import oracle as orc

    return [orc.dp_plan(g, b, family, objective, cap, nthreads=1) for b in budgets]


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1905_11722_b200 import named_graph
    from paper_1905_11722_b200.sweep import budget_sweep

    g = named_graph("pspnet")
    budgets = sweep_budgets(55, 385, 10)
    res = budget_sweep(g, budgets, "pruned", "minimize", solve=_oracle_solve)
    if rank == 0:
        q.put([(r["feasible"], r.get("objective_value"), r["stats"]["transitions"]) for r in res])
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_budget_sweep_two_ranks_matches_single_process():
    from paper_1905_11722_b200 import named_graph

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = named_graph("pspnet")
    want = [(r["feasible"], r.get("objective_value"), r["stats"]["transitions"])
            for r in _oracle_solve(g, sweep_budgets(55, 385, 10), "pruned", "minimize", 0)]
    assert got == want


def _search_worker(rank, world, port, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1905_11722_b200 import named_graph
    from paper_1905_11722_b200.sweep import min_feasible_budget_sharded

    out = []
    for name, kw, fam, obj in [("unet", {"skip_len": 2}, "full", "minimize"),
                               ("unet", {"skip_len": 2}, "full", "maximize"),
                               ("pspnet", {}, "pruned", "minimize")]:
        g = named_graph(name, **kw)
        b, plan = min_feasible_budget_sharded(g, fam, obj, probes_per_rank=3, solve=_oracle_solve)
        out.append((b, plan["objective_value"], plan["stats"]["transitions"]))
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_budget_search_two_ranks_matches_reference_search():
    """The sharded k-ary B_min search (host logic, 2 gloo ranks, CPU oracle as
    the per-rank solve) returns the reference binary search's B_min and plan."""
    from oracle import oracle as orc
    from paper_1905_11722_b200 import named_graph

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_search_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = []
    for name, kw, fam, obj in [("unet", {"skip_len": 2}, "full", "minimize"),
                               ("unet", {"skip_len": 2}, "full", "maximize"),
                               ("pspnet", {}, "pruned", "minimize")]:
        b, r = orc.min_feasible_budget(named_graph(name, **kw), fam, obj)
        want.append((b, r["objective_value"], r["stats"]["transitions"]))
    assert got == want


@pytest.mark.gpu
def test_sharded_budget_search_on_gpu_matches_golden():
    from _util import assert_plan_matches, golden, load
    from paper_1905_11722_b200.sweep import min_feasible_budget_sharded

    n = 0
    for rec in golden("mfb_corpus.json")[:20]:
        g = load(rec["graph"])
        for case in rec["cases"]:
            if "b_min" not in case:
                continue
            fam, obj = case["plan"]["family"], case["plan"]["objective"]
            b, plan = min_feasible_budget_sharded(g, fam, obj)
            assert b == case["b_min"]
            assert_plan_matches(plan, case["plan"], (fam, obj))
            n += 1
    assert n > 20
