"""Edge cases of every policy family on the CUDA path, against the oracle: empty and one-event
traces, C = 0, C beyond every history (and beyond u16), xi = 0 and xi beyond every history,
a single conversation, ragged trace lengths that are not a multiple of 32."""
import math

import numpy as np
import pytest
import torch

import oracle as O
from paper_2510_15152_b200.inputs import random_trace
from test_gpu_aware import upload as _upload


def upload(T, conv, q, a):
    """Upload with arrival time = event index (explicit ticks: ET-LRU rejects synthetic ones)."""
    if len(conv) == 0:
        return _upload(T, conv, q, a)
    c = torch.from_numpy(np.asarray(conv, np.uint32).view(np.int32).copy()).cuda()
    qq = torch.from_numpy(np.asarray(q, np.uint16).view(np.int16).copy()).cuda()
    aa = torch.from_numpy(np.asarray(a, np.uint16).view(np.int16).copy()).cuda()
    return T.trace_from_turns(c, qq, aa, ticks=torch.arange(len(conv), dtype=torch.int64, device="cuda"))

pytestmark = pytest.mark.gpu
TAB = [0.0, 0.0, math.log(0.4), math.log(0.2), -math.inf]
MU = 0.1
POLICIES = (0, 1, 2, 3, 4, 5, 6, 7)


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2510_15152_b200.tlru as T
    T.set_etlru_model(MU, TAB)
    yield T
    T.set_sim_options(0, 0)
    T.set_sim_engine(T.ENGINE_STACK)


def oracle_b(pol, conv, q, a, C, xi, qh, thr=0):
    if pol == 6:
        ticks = np.arange(len(conv), dtype=np.uint64)  # uploaded with time = event index
        return O.replay_etlru(conv, q, a, ticks, C, xi, MU, TAB)
    return O.replay(conv, q, a, pol, C, xi, qh, threshold=thr)


def rows_for(C_list, xi_list):
    return [(0, pol, C, xi, 2, 8) + ((3,) if pol == 2 else ()) for pol in POLICIES for C in C_list
            for xi in xi_list]


def run_and_check(T, conv, q, a, rows):
    tr = upload(T, conv, q, a)
    bt = T.simulate_batch([tr], rows)
    res = bt.results_numpy()
    assert T.last_sim_stats()["failed_chains"] == 0
    for i, r in enumerate(rows):
        o = oracle_b(r[1], np.asarray(conv, np.uint32), np.asarray(q, np.uint32), np.asarray(a, np.uint32),
                     r[2], r[3], r[4], r[6] if len(r) > 6 else 0)
        assert np.array_equal(bt.b(i).astype(np.uint64), o.b), r
        assert (res[i]["evicted_trim"], res[i]["evicted_lru"], res[i]["max_occupancy"]) == (
            o.evicted_trim, o.evicted_lru, o.max_occupancy), r
        assert res[i]["requests"] == len(conv)


def test_empty_trace_every_policy(T):
    tr = upload(T, [], [], [])
    rows = rows_for((0, 10), (0, 4))
    bt = T.simulate_batch([tr], rows)
    assert np.all(bt.results_numpy()["requests"] == 0)


def test_one_event_and_single_conversation(T):
    run_and_check(T, [5], [3], [2], rows_for((0, 1, 4, 10), (0, 3, 9)))
    run_and_check(T, [7] * 45, [1, 2, 3] * 15, [2, 0, 1] * 15, rows_for((0, 3, 40, 5000), (0, 2, 7, 60)))


@pytest.mark.parametrize("E", [31, 33, 95, 1000])
def test_ragged_lengths_and_extreme_parameters(T, E):
    conv, q, a = random_trace(6000 + E, E, 12, q_max=5, a_max=5, locality=0.5)
    run_and_check(T, conv, q, a, rows_for((0, 1, 7, 64, 70000, 0x7FFFFFFF), (0, 1, 6, 40000)))


def test_tiny_traces_grid_every_policy(T):
    """BASELINE config 2 (<= 4 conversations, <= 3 turns) for the policy families beyond
    LRU / T-LRU (those have the full grid in test_gpu_parity): every C in [0, 8], xi in [0, 5],
    Q_hat in [0, 3] on 60 traces, GPU against the oracle."""
    from paper_2510_15152_b200.inputs import tiny_trace
    traces, otr, rows = [], [], []
    for seed in range(60):
        conv, q, a = tiny_trace(seed)
        traces.append(upload(T, conv, q, a))
        otr.append((conv, q, a))
        for pol in (2, 3, 4, 5, 6, 7):
            for C in range(9):
                for xi in range(6):
                    for qh in (range(4) if pol in (3, 4, 7) else (0,)):
                        rows.append((seed, pol, C, xi, qh, 2) + ((2,) if pol == 2 else ()))
    bt = T.simulate_batch(traces, rows)
    assert T.last_sim_stats()["failed_chains"] == 0
    res = bt.results_numpy()
    for i, r in enumerate(rows):
        conv, q, a = otr[r[0]]
        o = oracle_b(r[1], conv, q, a, r[2], r[3], r[4], r[6] if len(r) > 6 else 0)
        assert np.array_equal(bt.b(i).astype(np.uint64), o.b), r
        assert (res[i]["evicted_trim"], res[i]["evicted_lru"], res[i]["max_occupancy"]) == (
            o.evicted_trim, o.evicted_lru, o.max_occupancy), r
