"""End-Aware / Length-Aware T-LRU (Readings #24-#25) on the CUDA path (replay engine,
whole-trace chains), element by element against the oracle through the C ABI."""
import json
import os

import numpy as np
import pytest
import torch

import oracle as O
from paper_2510_15152_b200.inputs import ALPHA_MS, CAPS_CONFIG3, Q_HAT, SLO_BLOCKS, preset, random_trace

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
END, LEN = 3, 4


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2510_15152_b200.tlru as T
    yield T
    T.set_sim_options(0, 0)
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
        conv, q, a = otr[t]
        o = O.replay(conv, q, a, pol, C, xi, qh, threshold=r[6] if len(r) > 6 else 0)
        assert np.array_equal(bt.b(i).astype(np.uint64), o.b), (i, r, np.flatnonzero(bt.b(i) != o.b)[:5])
        tl = O.tail(o.b, xi, ALPHA_MS * xi, slo, ALPHA_MS)
        g = res[i]
        assert (g["sum_uncached"], g["tel_blocks"], g["slo_violations"]) == (tl.sum_b, tl.tel_blocks,
                                                                           tl.slo_violations), r
        assert (g["p50"], g["p90"], g["p95"], g["p99"]) == (tl.p50, tl.p90, tl.p95, tl.p99), r
        assert (g["evicted_trim"], g["evicted_lru"], g["max_occupancy"]) == (o.evicted_trim, o.evicted_lru,
                                                                           o.max_occupancy), r


def test_hand_vectors(T):
    g = json.load(open(os.path.join(GOLDEN, "aware_tlru.json")))
    for key in ("fig1_terminating", "length_vs_end"):
        v = g[key]
        tr = upload(T, v["conv"], v["q"], v["a"])
        rows = [(0, END, v["C"], v["xi"], v["q_hat"], 16), (0, LEN, v["C"], v["xi"], v["q_hat"], 16)]
        bt = T.simulate_batch([tr], rows)
        assert list(bt.b(0)) == v["end_aware_b"] and list(bt.b(1)) == v["length_aware_b"]
        assert T.last_sim_stats()["engine"] == T.ENGINE_REPLAY


@pytest.mark.parametrize("engine", [0, 1], ids=["replay", "stack-requested"])
def test_random_traces_mixed_batch(T, engine):
    """Aware lanes beside LRU / T-LRU / Threshold-LRU lanes (the whole batch runs on the replay
    engine; the others keep their segmented warm-started chains)."""
    T.set_sim_engine(engine)
    traces, otr, rows = [], [], []
    for s in range(3):
        conv, q, a = random_trace(800 + s, 5000, 80, q_max=6, a_max=8, locality=0.5)
        traces.append(upload(T, conv, q, a))
        otr.append((conv, q, a))
        for C in (0, 3, 20, 90, 400):
            rows += [(s, END, C, xi, 2, 8) for xi in (0, 4, 9, 17)]
            rows += [(s, LEN, C, xi, 2, 8) for xi in (0, 4, 9, 17)]
            rows += [(s, 0, C, 4, 2, 8), (s, 1, C, 9, 2, 8), (s, 2, C, 9, 0, 8, 8)]
    bt = T.simulate_batch(traces, rows)
    check(T, bt, rows, otr)


def test_generated_preset(T):
    """BASELINE config-3 shape (10^4-conversation WildChat-shaped traces): the paper's
    predictability spectrum T-LRU / End-Aware / Length-Aware at xi = 16 blocks (200 ms)."""
    params = [preset("wildchat", s, 10_000) for s in range(2)]
    traces = T.generate_traces(params, exports=False)
    otr = []
    for p in params:
        o = O.generate(p)
        otr.append((o.conv, o.q, o.a))
    rows = [(t, pol, C, 16, Q_HAT, SLO_BLOCKS) for t in range(2) for pol in (1, END, LEN) for C in CAPS_CONFIG3]
    bt = T.simulate_batch(traces, rows)
    check(T, bt, rows, otr)
    res = bt.results_numpy()
    for t in range(2):  # release only frees space: End-Aware never misses more than T-LRU (oracle pin)
        for C in CAPS_CONFIG3:
            i1, ie = rows.index((t, 1, C, 16, Q_HAT, SLO_BLOCKS)), rows.index((t, END, C, 16, Q_HAT, SLO_BLOCKS))
            assert np.all(bt.b(ie) <= bt.b(i1)) and res[ie]["tel_blocks"] <= res[i1]["tel_blocks"]


def test_spill_path(T):
    """Force the smallest on-chip state (32 entries): whole-trace aware chains overflow and are
    re-run by the spill kernel with global-memory state; results must not change."""
    conv, q, a = random_trace(900, 4000, 300, q_max=3, a_max=3, locality=0.2)
    tr = upload(T, conv, q, a)
    rows = [(0, pol, C, 9, 2, 8) for pol in (END, LEN) for C in (200, 600)]
    T.set_sim_options(0, 32)
    try:
        bt = T.simulate_batch([tr], rows)
        st = T.last_sim_stats()
    finally:
        T.set_sim_options(0, 0)
    assert st["spilled_chains"] > 0 and st["failed_chains"] == 0
    check(T, bt, rows, [(conv, q, a)])
