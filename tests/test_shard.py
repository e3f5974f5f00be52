"""Level sharding.

CPU: the target partition (through the C-ABI host helper) and the 2-rank
gloo exchange of the communicator id.  GPU: the level-sharded solve with 2-4
replicas on one device (loopback exchange — the same pack / all-gather /
unpack path as NCCL, with device copies) must be bit-identical to the
single-GPU solve and to the oracle."""

from __future__ import annotations

import os
import socket

import pytest
import torch.multiprocessing as mp

from _util import assert_plan_matches, stats_of


def test_level_partition_covers_each_target_once():
    from paper_1905_11722_b200._native import level_partition

    for j0, width in [(0, 1), (1, 26), (6700, 171), (100, 7), (5, 0)]:
        for world in (1, 2, 3, 4, 8):
            parts = [level_partition(j0, width, world, r) for r in range(world)]
            assert parts[0][0] == j0 and parts[-1][1] == j0 + width
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_level_partition_rejects_bad_rank():
    from paper_1905_11722_b200._native import level_partition

    with pytest.raises(ValueError):
        level_partition(0, 10, 2, 2)


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1905_11722_b200.shard import exchange_unique_id

    uid = exchange_unique_id(make=lambda: bytes(range(128)))
    q.put((rank, uid))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_unique_id_reaches_every_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0] == got[1] == bytes(range(128))


@pytest.fixture(params=["0", "default"])
def replicate(request, monkeypatch):
    """Shard every level (REMAT_SHARD_REPLICATE=0: every level exchanged), or
    the default split (light levels replicated on every rank, batched)."""
    if request.param == "default":
        monkeypatch.delenv("REMAT_SHARD_REPLICATE", raising=False)
    else:
        monkeypatch.setenv("REMAT_SHARD_REPLICATE", request.param)
    return request.param


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 4])
def test_loopback_level_sharding_matches_single_gpu(world, replicate):
    from paper_1905_11722_b200 import Solver, named_graph
    from paper_1905_11722_b200.shard import loopback_plans

    g = named_graph("unet", skip_len=4)
    budgets = [2 * g.total_memory, g.total_memory // 2, 200]
    s = Solver(g, "full")
    want = s.plans(budgets)
    wmax = s.plans(budgets[:1], "maximize")
    s.close()
    got = loopback_plans(g, budgets, world)
    for a, b in zip(got, want):
        assert a.feasible == b.feasible and a.objective_value == b.objective_value
        assert stats_of(a) == stats_of(b)
        if a.feasible:
            assert a.sequence == b.sequence and a.evaluation == b.evaluation
    gmax = loopback_plans(g, budgets[:1], world, objective="maximize")
    assert gmax[0].objective_value == wmax[0].objective_value
    assert stats_of(gmax[0]) == stats_of(wmax[0])


@pytest.mark.gpu
def test_loopback_level_sharding_random_dag_matches_oracle(replicate):
    from oracle import oracle as orc
    from paper_1905_11722_b200 import named_graph
    from paper_1905_11722_b200.shard import loopback_plans

    g = named_graph("random-dag", depth=516, edge_prob=0.4, seed=0)
    b = 2 * g.total_memory
    ref = orc.dp_plan(g, b, "full", "minimize")
    (plan,) = loopback_plans(g, [b], 4)
    assert_plan_matches(plan, ref)


@pytest.mark.gpu
def test_wide_keys_path_matches_oracle():
    """The 64-bit key / 16-byte entry path (graphs whose M(V) does not fit the
    packed 32-bit key) on a graph that fits both: forced wide == narrow."""
    from oracle import oracle as orc
    from paper_1905_11722_b200 import PlanRequest, dp_plan, named_graph
    from paper_1905_11722_b200.shard import loopback_plans

    g = named_graph("unet", skip_len=3)
    os.environ["REMAT_FORCE_WIDE"] = "1"
    try:
        for b, obj in [(2 * g.total_memory, "minimize"), (300, "minimize"),
                       (2 * g.total_memory, "maximize")]:
            ref = orc.dp_plan(g, b, "full", obj)
            assert_plan_matches(dp_plan(PlanRequest(g, b, "full", obj)), ref, (b, obj))
        (plan,) = loopback_plans(g, [400], 2)
        assert_plan_matches(plan, orc.dp_plan(g, 400, "full", "minimize"))
    finally:
        del os.environ["REMAT_FORCE_WIDE"]


def _nccl_one_rank_worker(port, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["REMAT_SHARD_EXCHANGE"] = "1"  # run the all-gather even on one rank
    dist.init_process_group("gloo", rank=0, world_size=1)
    from paper_1905_11722_b200 import Solver, named_graph
    from paper_1905_11722_b200.shard import LevelShardedSolver

    g = named_graph("unet", skip_len=4)
    budgets = [2 * g.total_memory, 300]
    ls = LevelShardedSolver(g, "full")
    got = ls.plans(budgets)
    ls.close()
    s = Solver(g, "full")
    want = s.plans(budgets)
    s.close()
    q.put([(a.objective_value == b.objective_value, stats_of(a) == stats_of(b),
            a.sequence == b.sequence) for a, b in zip(got, want)])
    dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_level_sharded_path_one_rank():
    """The real NCCL path (dlopen'ed libnccl, ncclCommInitRank, one
    ncclAllGather per level on the solver's stream) on a one-rank communicator."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_one_rank_worker, args=(_free_port(), q))
    p.start()
    res = q.get(timeout=600)
    p.join(timeout=120)
    assert p.exitcode == 0
    assert res == [(True, True, True)] * 2


@pytest.mark.gpu
@pytest.mark.parametrize("replicate", ["0"], indirect=True)
def test_loopback_level_sharding_sparse_cells(replicate):
    """Level sharding over the sparse-cell path (FLOP-valued compute costs):
    every level exchanged between 3 replicas, plans equal to the reference's."""
    from _util import golden, load
    from paper_1905_11722_b200.shard import loopback_plans

    for rec in golden("large_costs.json")[-3:-1]:
        g = load(rec["graph"])
        cases = [c for c in rec["cases"] if c["family"] == "full" and c["objective"] == "minimize"]
        got = loopback_plans(g, [c["budget"] for c in cases], 3)
        for plan, case in zip(got, cases):
            assert_plan_matches(plan, case, case["budget"])
