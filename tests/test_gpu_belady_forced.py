"""Tail-Optimized Belady under forced caching (App. C: "Theorem 1 continues to hold" with
constraint (3) as an equality; Reading #29) on the CUDA path (replay engine, burn-in segments
verified by the fix-up), element by element against the oracle (policy 8) through the C ABI."""
import json
import os

import pytest
import torch

import oracle as O
from paper_2510_15152_b200.inputs import CAPS_CONFIG3, Q_HAT, SLO_BLOCKS, preset, random_trace
from test_gpu_aware import check, upload

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
BEL, BELF, TF = 5, 8, 7


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


def test_policy_constant(T):
    assert T.POLICY_BELADY_FORCED == BELF == O.BELADY_FORCED


def test_fig1_forced_hand_vector(T):
    """Fig. 1 under forced caching: B must keep its 100 blocks, so A pays 200
    (tests/golden/tail_belady.json fig1_forced)."""
    v = json.load(open(os.path.join(GOLDEN, "tail_belady.json")))["fig1_forced"]
    bt = T.simulate_batch([upload(T, v["conv"], v["q"], v["a"])], [(0, BELF, v["C"], v["xi"], 0, 16)])
    r = bt.results_numpy()[0]
    assert list(bt.b(0)) == v["b"] and [r["evicted_trim"], r["evicted_lru"]] == v["evicted"]
    assert r["max_occupancy"] == v["max_occupancy"]


@pytest.mark.parametrize("engine", [0, 1], ids=["replay", "stack-requested"])
def test_random_traces_mixed_batch(T, engine):
    """Forced Belady lanes beside optional Belady, forced T-LRU, LRU and T-LRU lanes; capacities
    from 0 (theta alone always exceeds C) to beyond the universe."""
    T.set_sim_engine(engine)
    traces, otr, rows = [], [], []
    for s in range(3):
        conv, q, a = random_trace(2800 + s, 6000, 90, q_max=6, a_max=8, locality=0.5)
        traces.append(upload(T, conv, q, a))
        otr.append((conv, q, a))
        for C in (0, 1, 3, 20, 90, 400, 5000):
            rows += [(s, BELF, C, xi, 0, 8) for xi in (0, 1, 4, 9, 17, 60)]
        rows += [(s, BEL, 40, 9, 0, 8), (s, TF, 40, 9, 2, 8), (s, 0, 40, 4, 2, 8), (s, 1, 40, 9, 2, 8)]
    bt = T.simulate_batch(traces, rows)
    check(T, bt, rows, otr)


def test_generated_preset_forced_spectrum(T):
    """BASELINE config-3 shape (10^4-conversation WildChat-shaped traces, several burn-in segments
    per chain); App. C pathwise: TEL(forced Belady) <= TEL(forced T-LRU) (the forced hindsight
    optimum against a forced online policy) and TEL(Belady) <= TEL(forced Belady) (forcing only
    removes options)."""
    params = [preset("wildchat", s, 10_000) for s in range(2)]
    traces = T.generate_traces(params, exports=False)
    otr = []
    for p in params:
        o = O.generate(p)
        otr.append((o.conv, o.q, o.a))
    rows = [(t, pol, C, xi, Q_HAT, SLO_BLOCKS) for t in range(2) for pol in (TF, BEL, BELF)
            for C in CAPS_CONFIG3 for xi in (4, 16)]
    bt = T.simulate_batch(traces, rows)
    check(T, bt, rows, otr)
    res = bt.results_numpy()
    for t in range(2):
        for C in CAPS_CONFIG3:
            for xi in (4, 16):
                tel = {pol: res[rows.index((t, pol, C, xi, Q_HAT, SLO_BLOCKS))]["tel_blocks"] for pol in (TF, BEL, BELF)}
                assert tel[BEL] <= tel[BELF] <= tel[TF], (t, C, xi, tel)


def test_uncoupled_segments_are_rerun(T):
    """Short segments and few, long-lived conversations: burn-in segments disagree with the exact
    state and are re-run by the fix-up."""
    conv, q, a = random_trace(2900, 40000, 40, q_max=4, a_max=4, locality=0.1)
    tr = upload(T, conv, q, a)
    rows = [(0, BELF, C, xi, 0, 8) for C in (10, 60, 200, 1000) for xi in (0, 5, 12)]
    bt = T.simulate_batch([tr], rows)
    assert T.last_sim_stats()["failed_chains"] == 0
    check(T, bt, rows, [(conv, q, a)])


def test_state_overflow_rerun(T):
    """The smallest on-chip state (32 entries) with more live conversations: segments overflow and
    are re-run from global memory; results must not change."""
    conv, q, a = random_trace(2950, 12000, 300, q_max=3, a_max=3, locality=0.2)
    tr = upload(T, conv, q, a)
    rows = [(0, BELF, C, xi, 0, 8) for C in (200, 600) for xi in (0, 9)]
    T.set_sim_options(0, 32)
    try:
        bt = T.simulate_batch([tr], rows)
        st = T.last_sim_stats()
    finally:
        T.set_sim_options(0, 0)
    assert st["spilled_chains"] > 0 and st["failed_chains"] == 0
    check(T, bt, rows, [(conv, q, a)])


def test_full_size_sampled(T):
    """BASELINE full trace size (10^6 conversations) in the launch configuration of
    `bench.py --config forced_belady` (one trace, its 100 rows in one batch): sampled instances
    against the oracle element by element."""
    from paper_2510_15152_b200.inputs import CAPS_CONFIG5
    p = preset("wildchat", 5, 1_000_000)
    tr = T.generate_traces([p], exports=False)[0]
    rows = [(0, BELF, C, xi, Q_HAT, SLO_BLOCKS) for C in CAPS_CONFIG5 for xi in (4, 8, 16, 24)]
    bt = T.simulate_batch([tr], rows)
    assert T.last_sim_stats()["failed_chains"] == 0
    o = O.generate(p)
    picks = [(16, 4), (256, 24), (4096, 16), (CAPS_CONFIG5[9], 8)]
    sub_rows = [rows.index((0, BELF, C, xi, Q_HAT, SLO_BLOCKS)) for C, xi in picks]

    class Sub:  # the picked instances of the full batch
        def __init__(self, bt, idx):
            self.bt, self.idx = bt, idx

        def b(self, k):
            return self.bt.b(self.idx[k])

        def results_numpy(self):
            return self.bt.results_numpy()[self.idx]

    check(T, Sub(bt, sub_rows), [rows[i] for i in sub_rows], [(o.conv, o.q, o.a)])
