"""ET-LRU under forced caching (App. C: Y_theta = L; Reading #30) on the CUDA path
(one warp per instance, etlru.cuh), element by element against the oracle (replay_etlru(forced=True))
through the C ABI."""
import math

import numpy as np
import pytest
import torch

import oracle as O
from paper_2510_15152_b200.inputs import ALPHA_MS, CAPS_CONFIG3, SLO_BLOCKS, WILDCHAT, preset, prompt_law_ln_surv
from paper_2510_15152_b200.inputs import random_trace
from test_gpu_etlru import TABLES, upload_ticks

pytestmark = pytest.mark.gpu
ET, ETF, TF = 6, 9, 7


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


def check(bt, rows, otr, mu, table):
    res = bt.results_numpy()
    for i, r in enumerate(rows):
        t, pol, C, xi, qh, slo = r[:6]
        conv, q, a, ticks = otr[t]
        if pol in (ET, ETF):
            o = O.replay_etlru(conv, q, a, ticks, C, xi, mu, table, forced=pol == ETF)
        else:
            o = O.replay(conv, q, a, pol, C, xi, qh)
        assert np.array_equal(bt.b(i).astype(np.uint64), o.b), (i, r, np.flatnonzero(bt.b(i) != o.b)[:5])
        tl = O.tail(o.b, xi, ALPHA_MS * xi, slo, ALPHA_MS)
        g = res[i]
        assert (g["sum_uncached"], g["tel_blocks"], g["slo_violations"], g["p90"], g["p95"]) == (
            tl.sum_b, tl.tel_blocks, tl.slo_violations, tl.p90, tl.p95), r
        assert (g["evicted_trim"], g["evicted_lru"], g["max_occupancy"]) == (o.evicted_trim, o.evicted_lru,
                                                                           o.max_occupancy), r


def test_policy_constant(T):
    assert T.POLICY_ETLRU_FORCED == ETF == O.ETLRU_FORCED


@pytest.mark.parametrize("tab", range(len(TABLES)))
def test_random_traces_mixed_batch(T, tab):
    """Forced ET-LRU warps beside optional ET-LRU, forced T-LRU and LRU; capacities from 0 (theta
    alone always exceeds C) to beyond the universe; times with ties."""
    rng = np.random.default_rng(90 + tab)
    mu = 0.05
    T.set_etlru_model(mu, TABLES[tab])
    traces, otr, rows = [], [], []
    for s in range(2):
        conv, q, a = random_trace(9000 + 10 * tab + s, 3000, 60, q_max=5, a_max=6, locality=0.5)
        ticks = np.cumsum(rng.integers(0, 40, conv.size)).astype(np.uint64)
        traces.append(upload_ticks(T, conv, q, a, ticks))
        otr.append((conv, q, a, ticks))
        for C in (0, 1, 4, 25, 120, 900, 20000):
            rows += [(s, ETF, C, xi, 2, 8) for xi in (0, 2, 5, 11)]
        rows += [(s, ET, 25, 5, 2, 8), (s, TF, 25, 5, 2, 8), (s, 0, 25, 5, 2, 8)]
    bt = T.simulate_batch(traces, rows)
    assert T.last_sim_stats()["failed_chains"] == 0
    check(bt, rows, otr, mu, TABLES[tab])


def test_point_mass_equals_forced_tlru_on_gpu(T):
    """P:668 on the GPU: with a fixed prompt length forced ET-LRU's b equals forced T-LRU's."""
    T.set_etlru_model(0.3, TABLES[2])  # point mass at 2
    conv, q, a = random_trace(9100, 4000, 70, q_max=5, a_max=6, locality=0.5)
    ticks = np.cumsum(np.random.default_rng(5).integers(1, 30, conv.size)).astype(np.uint64)
    tr = upload_ticks(T, conv, q, a, ticks)
    rows = [(0, pol, C, xi, 2, 8) for C in (3, 40, 300) for xi in (2, 6, 13) for pol in (ETF, TF)]
    bt = T.simulate_batch([tr], rows)
    for k in range(0, len(rows), 2):
        assert np.array_equal(bt.b(k), bt.b(k + 1)), rows[k]


def test_generated_preset_with_segments(T):
    """BASELINE config-3 shape (10^4-conversation WildChat-shaped trace, the preset's own prompt
    law, real microsecond ticks): several burn-in segments per instance, verified by the fix-up."""
    p = preset("wildchat", 4, 10_000)
    mu = WILDCHAT["death_rate"] * 1e-6
    tab = prompt_law_ln_surv(WILDCHAT)
    T.set_etlru_model(mu, tab)
    tr = T.generate_traces([p], exports=True)[0]
    o = O.generate(p)
    rows = [(0, ETF, C, xi, 2, SLO_BLOCKS) for C in CAPS_CONFIG3 for xi in (4, 16)]
    T.set_sim_options(2048, 0)
    try:
        bt = T.simulate_batch([tr], rows)
        st = T.last_sim_stats()
    finally:
        T.set_sim_options(0, 0)
    assert st["failed_chains"] == 0
    check(bt, rows, [(o.conv, o.q, o.a, o.ticks)], mu, tab)


def test_full_size_sampled(T):
    """BASELINE trace size (10^6 conversations) in the launch configuration of
    `bench.py --config etlru_forced` (one trace, its 100 rows in one batch): sampled instances
    against the oracle, b and eviction counters."""
    from paper_2510_15152_b200.inputs import CAPS_CONFIG5
    p = preset("wildchat", 6, 1_000_000)
    mu = WILDCHAT["death_rate"] * 1e-6
    tab = prompt_law_ln_surv(WILDCHAT)
    T.set_etlru_model(mu, tab)
    tr = T.generate_traces([p], exports=True)[0]
    rows = [(0, ETF, C, xi, 2, SLO_BLOCKS) for C in CAPS_CONFIG5 for xi in (4, 8, 16, 24)]
    bt = T.simulate_batch([tr], rows)
    assert T.last_sim_stats()["failed_chains"] == 0
    o = O.generate(p)
    res = bt.results_numpy()
    for C, xi in ((16, 4), (256, 16), (CAPS_CONFIG5[20], 24)):
        i = rows.index((0, ETF, C, xi, 2, SLO_BLOCKS))
        r = O.replay_etlru(o.conv, o.q, o.a, o.ticks, C, xi, mu, tab, forced=True)
        assert np.array_equal(bt.b(i).astype(np.uint64), r.b), (C, xi)
        assert (res[i]["evicted_trim"], res[i]["evicted_lru"], res[i]["max_occupancy"]) == (
            r.evicted_trim, r.evicted_lru, r.max_occupancy)
