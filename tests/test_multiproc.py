"""Multi-process (world size 2, gloo on CPU) tests of the sweep plumbing in
paper_2510_15152_b200/sweep.py: sharding is a deterministic partition, and the gathered
result table is identical to the single-process one, whatever the world size."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_15152_b200.abi_types import RESULT_DTYPE
from paper_2510_15152_b200.inputs import config5_rows
from paper_2510_15152_b200.sweep import gather_results, shard_instances


def fake_results(rows):
    """Stand-in per-instance results: a deterministic function of the instance row."""
    out = np.zeros(len(rows), RESULT_DTYPE)
    for i, (t, pol, C, xi, qh, slo) in enumerate(rows):
        out[i]["requests"] = 1000 + t
        out[i]["sum_uncached"] = C * 7 + xi
        out[i]["tel_blocks"] = pol * 13 + xi
        out[i]["p90"] = C % 97
        out[i]["max_occupancy"] = C
    return out


def test_shards_partition_deterministically():
    rows = config5_rows(10)
    ev = {t: 2_500_000 + 37 * t for t in range(10)}
    for world in (1, 2, 3, 4, 8):
        sh = shard_instances(rows, world, ev)
        flat = sorted(i for s in sh for i in s)
        assert flat == list(range(len(rows)))
        assert sh == shard_instances(rows, world, ev)
        if world <= 10:  # whole traces stay on one rank
            owner = {}
            for k, s in enumerate(sh):
                for i in s:
                    assert owner.setdefault(rows[i][0], k) == k
        loads = [len(s) for s in sh]
        assert max(loads) - min(loads) <= 1000 * (1 if world <= 10 else 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rows = config5_rows(4)
        shards = shard_instances(rows, world)
        mine = shards[rank]
        local = fake_results([rows[i] for i in mine])
        table = gather_results(local, mine, len(rows))
        if rank == 0:
            q.put(table.tobytes())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2])
def test_gather_identical_for_any_world_size(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expected = fake_results(config5_rows(4)).tobytes()
    assert got == expected


def test_plan_strong_partitions_and_balances():
    """Strong-scaling shards (sweep.plan_strong): a deterministic partition, contiguous in the stack
    engine's (trace, D, C) order, within the modelled optimum for contiguous cuts, and cutting inside
    traces so 10 traces spread over 8 ranks (whole-trace sharding would cap efficiency at 10/16)."""
    from paper_2510_15152_b200.sweep import plan_strong, row_d_key, shard_cost
    rows = config5_rows(10)
    total = shard_cost(rows, range(len(rows)))
    for world in (1, 2, 3, 4, 8, 16):
        sh = plan_strong(rows, world)
        assert len(sh) == world and sh == plan_strong(rows, world)
        assert sorted(i for s in sh for i in s) == list(range(len(rows)))
        order = sorted(range(len(rows)), key=lambda i: (rows[i][0], row_d_key(rows[i]), rows[i][2], i))
        pos = {i: k for k, i in enumerate(order)}
        for s in sh:  # contiguous in the engine's order
            if s:
                ks = sorted(pos[i] for i in s)
                assert ks[-1] - ks[0] + 1 == len(ks)
        costs = [shard_cost(rows, s) for s in sh]
        assert max(costs) <= total / world * 1.25 + 0.61  # one extra trace pass per shard at most
    sh8 = plan_strong(rows, 8)
    assert all(len({rows[i][0] for i in s}) <= 2 for s in sh8)
    assert max(shard_cost(rows, s) for s in sh8) < total / 8 / 0.8  # modelled efficiency > 80%
    assert plan_strong(rows[:3], 5)[3:] == [[], []]  # more ranks than instances: idle ranks
