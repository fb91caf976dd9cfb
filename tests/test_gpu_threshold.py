"""Threshold-LRU (Reading #23) on the CUDA path, element by element against the
oracle, through the C ABI: both engines, mixed batches (LRU / T-LRU / Threshold-LRU rows in one
stack-engine chunk), edge thresholds."""
import json
import os

import numpy as np
import pytest
import torch

import oracle as O
from paper_2510_15152_b200.inputs import ALPHA_MS, CAPS_CONFIG3, Q_HAT, SLO_BLOCKS, preset, random_trace

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ENGINES = pytest.mark.parametrize("engine", [0, 1], ids=["replay", "stack"])
THR = 2


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2510_15152_b200.tlru as T
    yield T
    T.set_sim_engine(T.ENGINE_STACK)


def upload(T, conv, q, a):
    c = torch.from_numpy(np.asarray(conv, np.uint32).view(np.int32).copy()).cuda()
    qq = torch.from_numpy(np.asarray(q, np.uint16).view(np.int16).copy()).cuda()
    aa = torch.from_numpy(np.asarray(a, np.uint16).view(np.int16).copy()).cuda()
    return T.trace_from_turns(c, qq, aa)


def check(T, bt, rows, otr):
    res = bt.results_numpy()
    for i, r in enumerate(rows):
        t, pol, C, xi, qh, slo = r[:6]
        thr = r[6] if len(r) > 6 else 0
        conv, q, a = otr[t]
        o = O.replay(conv, q, a, pol, C, xi, qh, threshold=thr)
        assert np.array_equal(bt.b(i).astype(np.uint64), o.b), (i, r)
        tl = O.tail(o.b, xi, ALPHA_MS * xi, slo, ALPHA_MS)
        g = res[i]
        assert (g["sum_uncached"], g["tel_blocks"], g["slo_violations"]) == (tl.sum_b, tl.tel_blocks,
                                                                           tl.slo_violations), r
        assert (g["p50"], g["p90"], g["p95"], g["p99"]) == (tl.p50, tl.p90, tl.p95, tl.p99), r
        assert (g["evicted_trim"], g["evicted_lru"], g["max_occupancy"]) == (o.evicted_trim, o.evicted_lru,
                                                                           o.max_occupancy), r


@ENGINES
def test_hand_vector(T, engine):
    T.set_sim_engine(engine)
    g = json.load(open(os.path.join(GOLDEN, "threshold_lru.json")))
    tr = upload(T, g["conv"], g["q"], g["a"])
    rows = [(0, THR, g["C"], 0, 0, 16, g["threshold"]), (0, 0, g["C"], 0, 0, 16)]
    bt = T.simulate_batch([tr], rows)
    assert list(bt.b(0)) == g["threshold_b"] and list(bt.b(1)) == g["lru_b"]
    res = bt.results_numpy()
    assert res[0]["evicted_lru"] == g["threshold_evicted_lru"] and res[1]["evicted_lru"] == g["lru_evicted_lru"]


@ENGINES
def test_random_traces_mixed_batch(T, engine):
    """LRU, T-LRU and Threshold-LRU rows of several thresholds in one batch (one stack chunk
    with masked and unmasked rows side by side)."""
    T.set_sim_engine(engine)
    traces, otr, rows = [], [], []
    for s in range(4):
        conv, q, a = random_trace(300 + s, 3000, 60, q_max=6, a_max=8)
        traces.append(upload(T, conv, q, a))
        otr.append((conv, q, a))
        for C in (0, 1, 9, 40, 150, 600):
            rows += [(s, 0, C, 4, 2, 8), (s, 1, C, 9, 2, 8)]
            rows += [(s, THR, C, 6, 0, 8, thr) for thr in (0, 1, 5, 8, 20, 65535)]
    bt = T.simulate_batch(traces, rows)
    check(T, bt, rows, otr)


@ENGINES
def test_generated_preset_threshold8(T, engine):
    """BASELINE config 3 shape: 10^4-conversation WildChat-shaped traces, Threshold-LRU with the
    paper's 1024 tokens = 8 blocks, beside LRU and T-LRU(xi = 16)."""
    T.set_sim_engine(engine)
    params = [preset("wildchat", s, 10_000) for s in range(3)]
    traces = T.generate_traces(params, exports=False)
    otr = []
    for p in params:
        o = O.generate(p)
        otr.append((o.conv, o.q, o.a))
    rows = [(t, pol, C, 16, Q_HAT, SLO_BLOCKS) + ((8,) if pol == THR else ()) for t in range(3)
            for pol in (0, 1, THR) for C in CAPS_CONFIG3]
    bt = T.simulate_batch(traces, rows)
    check(T, bt, rows, otr)


def test_threshold_range_checked(T):
    tr = upload(T, [0, 1], [1, 1], [0, 0])
    with pytest.raises(T.TlruError):
        T.simulate_batch([tr], [(0, THR, 4, 0, 0, 1, 70000)])
