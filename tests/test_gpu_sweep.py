"""The multi-GPU sweep path (row a10) on the CUDA device: two processes share cuda:0
(gloo, collectives staged through host memory -- NCCL needs one GPU per rank) and each runs its
strong-scaling shard exactly as bench.py does (sweep.Sweep: plan_strong -> generate -> simulate ->
pool -> all_gather + all_reduce -> reassemble -> pooled tail metrics).  Checks: the gathered table
and the pooled metrics are byte-identical to world size 1, sampled b rows of both ranks equal the
oracle, and the pooled metrics equal the oracle's tail metrics over the pool's concatenated b."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N_CONV = 6000
SEEDS = 3


def sweep_rows():
    from paper_2510_15152_b200.inputs import Q_HAT, SLO_BLOCKS
    return [(t, pol, C, xi, Q_HAT, SLO_BLOCKS) for t in range(SEEDS) for pol in (0, 1) for C in (16, 45, 128, 700)
            for xi in (2, 6, 16, 30)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_rank(rank, world, port, q, pipelined=True):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    from paper_2510_15152_b200.inputs import preset
    from paper_2510_15152_b200.sweep import Sweep
    if world > 1:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        sw = Sweep(sweep_rows(), world, rank, lambda s: preset("wildchat", 100 + s, N_CONV), "cuda:0",
                   scaling="strong", backend="gloo")
        st = torch.cuda.current_stream()
        if pipelined:
            sw.step(st, torch.cuda.Stream(), [torch.cuda.Stream(), torch.cuda.Stream()])
        else:
            sw.step(st)
        torch.cuda.synchronize()
        # this rank's b rows for its first and last instance of every local trace
        brows = {}
        for j, ids in enumerate(sw.ids_by_trace):
            for k in sorted({0, len(ids) - 1}):
                brows[ids[k]] = sw.batches[j].b(k).copy()
        out = (sw.table_numpy().tobytes(), sw.pooled_tails_numpy().tobytes(), brows, sw.shards[rank],
               sw.requests_local)
        if q is None:
            return out
        q.put((rank, out))
    finally:
        if world > 1:
            dist.destroy_process_group()


@pytest.fixture(scope="module")
def single():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    return run_rank(0, 1, 0, None, pipelined=False)


def test_two_ranks_on_one_gpu_equal_world_size_one(single):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=run_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    table1, tails1 = single[0], single[1]
    shards = [got[r][3] for r in range(2)]
    assert sorted(shards[0] + shards[1]) == list(range(len(sweep_rows())))  # a partition
    assert shards[0] and shards[1]
    for r in range(2):
        assert got[r][0] == table1, f"rank {r}: gathered table differs from world size 1"
        assert got[r][1] == tails1, f"rank {r}: pooled metrics differ from world size 1"
    assert got[0][4] + got[1][4] == single[4]  # requests: no instance simulated twice or dropped

    import oracle as O
    from paper_2510_15152_b200.abi_types import RESULT_DTYPE, TAIL_DTYPE
    from paper_2510_15152_b200.inputs import ALPHA_MS, preset
    rows = sweep_rows()
    otr = [O.generate(preset("wildchat", 100 + s, N_CONV)) for s in range(SEEDS)]
    table = np.frombuffer(table1, RESULT_DTYPE)
    for r in range(2):
        for gid, b in got[r][2].items():  # sampled b rows of both ranks vs the oracle
            t, pol, C, xi, qh, slo = rows[gid]
            o = O.replay(otr[t].conv, otr[t].q, otr[t].a, pol, C, xi, qh)
            assert np.array_equal(b.astype(np.uint64), o.b), rows[gid]
            tl = O.tail(o.b, xi, ALPHA_MS * xi, slo, ALPHA_MS)
            assert (table[gid]["tel_blocks"], table[gid]["p90"], table[gid]["p95"]) == (tl.tel_blocks, tl.p90, tl.p95)
    # pooled metrics of two pools vs the oracle over the concatenated b of their seeds
    keys = sorted({r[1:] for r in rows})
    tails = np.frombuffer(tails1, TAIL_DTYPE)
    for key in (keys[0], keys[-1]):
        pol, C, xi, qh, slo = key
        bs = np.concatenate([O.replay(otr[t].conv, otr[t].q, otr[t].a, pol, C, xi, qh).b for t in range(SEEDS)])
        tl = O.tail(bs, xi, ALPHA_MS * xi, slo, ALPHA_MS)
        o = tails[keys.index(key)]
        assert (o["n"], o["tel_blocks"], o["slo_violations"], o["p50"], o["p90"], o["p95"], o["p99"]) == (
            tl.n, tl.tel_blocks, tl.slo_violations, tl.p50, tl.p90, tl.p95, tl.p99), key
        assert o["tel_ms"] == pytest.approx(tl.tel_ms, rel=1e-9)
