"""CPU tests of the data-parallel host logic (gloo, world_size 2)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2511_18871_b200.dp import bootstrap_comm, group_cost, lpt_assign, rank_groups


def test_lpt_partition_and_balance():
    import random

    rnd = random.Random(20251118)
    lens = [[rnd.randint(1024, 16384) for _ in range(8)] for _ in range(16)]  # C4-style ragged batch
    costs = [group_cost(2048, l, 1536, 28, 8960, 151936) for l in lens]
    for world in (1, 2, 4, 8):
        a = lpt_assign(costs, world)
        flat = sorted(i for r in a for i in r)
        assert flat == list(range(16))
        loads = [sum(costs[i] for i in r) for r in a]
        assert max(loads) <= sum(costs) / world + max(costs)  # LPT bound
    # C4 seed from SURVEY.md §8d: group 0 lengths
    assert lens[0] == [15781, 14233, 10574, 3139, 3977, 14992, 13452, 9697]


def test_round_robin_when_uniform():
    assert rank_groups(8, None, 4, 1) == [1, 5]
    assert rank_groups(8, [1.0] * 8, 2, 0) == [0, 2, 4, 6]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = bootstrap_comm(None, rank, world, make_id=lambda: b"\x07" * 128)
    # per-rank partial loss scalars, summed like parl_stats_allreduce
    stats = torch.tensor([0.5 * (rank + 1), 0.25, 0.01 * rank, 3.0, 10.0], dtype=torch.float64)
    dist.all_reduce(stats)
    mine = rank_groups(6, [5, 1, 4, 2, 3, 6], world, rank)
    q.put((rank, uid, stats.tolist(), mine))
    dist.destroy_process_group()


def test_gloo_world2_bootstrap_and_reduce():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert res[0][1] == res[1][1] == b"\x07" * 128
    assert res[0][2] == res[1][2] == pytest.approx([1.5, 0.5, 0.01, 6.0, 20.0])
    assert sorted(res[0][3] + res[1][3]) == list(range(6))
