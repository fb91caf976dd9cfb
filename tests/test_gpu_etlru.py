"""Expected-Tail-Optimized LRU (Def. 1 / Alg. 2; Reading #27) on the CUDA
path (one warp per instance, etlru.cuh), element by element against the oracle through the C ABI."""
import math

import numpy as np
import pytest
import torch

import oracle as O
from paper_2510_15152_b200.inputs import (ALPHA_MS, CAPS_CONFIG3, SLO_BLOCKS, WILDCHAT, preset,
                                          prompt_law_ln_surv, random_trace)
from test_gpu_aware import upload

pytestmark = pytest.mark.gpu
ET = 6
TABLES = [
    [0.0, 0.0, math.log(0.3), -math.inf],
    [0.0, 0.0, math.log(0.55), math.log(0.55), math.log(0.3), math.log(0.05)],
    [0.0, 0.0, 0.0, -math.inf],  # point mass at 2: T-LRU with Q_hat = 2
]


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


def upload_ticks(T, conv, q, a, ticks):
    """Upload with the trace's real arrival times (tlru_trace_from_turns' ticks input)."""
    c = torch.from_numpy(np.asarray(conv, np.uint32).view(np.int32).copy()).cuda()
    qq = torch.from_numpy(np.asarray(q, np.uint16).view(np.int16).copy()).cuda()
    aa = torch.from_numpy(np.asarray(a, np.uint16).view(np.int16).copy()).cuda()
    tk = torch.from_numpy(np.asarray(ticks, np.uint64).view(np.int64).copy()).cuda()
    tr = T.trace_from_turns(c, qq, aa, ticks=tk)
    assert tr.flags == 0
    return tr


def test_etlru_rejects_synthetic_ticks(T):
    """An upload without ticks numbers the events (TLRU_TRACE_SYNTHETIC_TICKS): ET-LRU's beliefs
    decay with time, so the batch is TLRU_EINVAL rather than silently per-event decay."""
    tr = upload(T, [0, 1, 0], [1, 1, 1], [0, 0, 0])
    assert tr.flags == 1
    assert np.array_equal(tr.time_ticks[:3].cpu().numpy(), [0, 1, 2])
    T.set_etlru_model(1e-6, prompt_law_ln_surv(WILDCHAT))
    with pytest.raises(T.TlruError, match="EINVAL.*ticks"):
        T.simulate_batch([tr], [(0, ET, 4, 2, 2, 16)])
    with pytest.raises(T.TlruError, match="EINVAL.*non-decreasing"):
        upload_ticks(T, [0, 1, 0], [1, 1, 1], [0, 0, 0], [5, 3, 9])


def check_et(bt, rows, otr, mu, table):
    res = bt.results_numpy()
    for i, r in enumerate(rows):
        t, pol, C, xi, qh, slo = r[:6]
        conv, q, a, ticks = otr[t]
        if pol == ET:
            o = O.replay_etlru(conv, q, a, ticks, C, xi, mu, table)
        else:
            o = O.replay(conv, q, a, pol, C, xi, qh)
        assert np.array_equal(bt.b(i).astype(np.uint64), o.b), (i, r, np.flatnonzero(bt.b(i) != o.b)[:5])
        tl = O.tail(o.b, xi, ALPHA_MS * xi, slo, ALPHA_MS)
        g = res[i]
        assert (g["sum_uncached"], g["tel_blocks"], g["slo_violations"]) == (tl.sum_b, tl.tel_blocks,
                                                                           tl.slo_violations), r
        assert (g["p50"], g["p90"], g["p95"], g["p99"]) == (tl.p50, tl.p90, tl.p95, tl.p99), r
        assert (g["evicted_trim"], g["evicted_lru"], g["max_occupancy"]) == (o.evicted_trim, o.evicted_lru,
                                                                           o.max_occupancy), r


@pytest.mark.parametrize("tab", range(len(TABLES)))
def test_random_traces_mixed_batch(T, tab):
    """ET-LRU warps beside LRU / T-LRU / Belady lanes; times with ties (equal ticks)."""
    mu = [0.7, 0.05, 3.0][tab]
    T.set_etlru_model(mu, TABLES[tab])
    rng = np.random.default_rng(tab)
    traces, otr, rows = [], [], []
    for s in range(2):
        conv, q, a = random_trace(4000 + 10 * tab + s, 5000, 70, q_max=5, a_max=6, locality=0.6)
        ticks = np.cumsum(rng.integers(0, 4, size=conv.size)).astype(np.uint64)
        traces.append(upload_ticks(T, conv, q, a, ticks))
        otr.append((conv, q, a, ticks))
        for C in (0, 1, 3, 20, 90, 400):
            rows += [(s, ET, C, xi, 0, 8) for xi in (0, 2, 5, 12)]
        rows += [(s, 0, 40, 4, 2, 8), (s, 1, 40, 5, 2, 8), (s, 5, 40, 5, 0, 8)]
    bt = T.simulate_batch(traces, rows)
    assert T.last_sim_stats()["failed_chains"] == 0
    check_et(bt, rows, otr, mu, TABLES[tab])
    if tab == 2:  # point mass at Q_hat = 2: ET-LRU == T-LRU, GPU against GPU
        for s in range(2):
            for C in (3, 20, 90, 400):
                for xi in (0, 2, 5, 12):
                    e = rows.index((s, ET, C, xi, 0, 8))
                    tb = T.simulate_batch([traces[s]], [(0, 1, C, xi, 2, 8)])
                    assert np.array_equal(bt.b(e), tb.b(0))


def test_generated_preset(T):
    """BASELINE config-3 shape with the preset's own prompt law and mu = 1/90 s (per microsecond
    tick): ET-LRU against the oracle, and against LRU / T-LRU on the same trace."""
    p = preset("wildchat", 5, 10_000)
    mu = p["death_rate"] * 1e-6
    tab = prompt_law_ln_surv(WILDCHAT)
    T.set_etlru_model(mu, tab)
    tr = T.generate_traces([p], exports=True)[0]
    o = O.generate(p)
    assert np.array_equal(tr.time_ticks[: tr.num_events].cpu().numpy().view(np.uint64), o.ticks)
    rows = [(0, pol, C, xi, 2, SLO_BLOCKS) for pol in (ET, 0, 1) for C in CAPS_CONFIG3 for xi in (4, 16)]
    bt = T.simulate_batch([tr], rows)
    check_et(bt, rows, [(o.conv, o.q, o.a, o.ticks)], mu, tab)


def test_state_overflow_rerun(T):
    """Force 32 shared-memory slots with more live conversations: chains overflow and are re-run
    with global-memory state; results must not change."""
    tab = TABLES[1]
    T.set_etlru_model(0.2, tab)
    conv, q, a = random_trace(4100, 6000, 200, q_max=3, a_max=3, locality=0.2)
    ticks = np.arange(conv.size, dtype=np.uint64) * 3
    tr = upload_ticks(T, conv, q, a, ticks)
    rows = [(0, ET, C, xi, 0, 8) for C in (300, 900) for xi in (0, 6)]
    T.set_sim_options(0, 32)
    try:
        bt = T.simulate_batch([tr], rows)
        st = T.last_sim_stats()
    finally:
        T.set_sim_options(0, 0)
    assert st["spilled_chains"] > 0 and st["failed_chains"] == 0
    check_et(bt, rows, [(conv, q, a, ticks)], 0.2, tab)


def test_model_errors(T):
    with pytest.raises(T.TlruError, match="EINVAL"):
        T.set_etlru_model(0.1, [0.0, -1.0, -0.5])  # increasing
    with pytest.raises(T.TlruError, match="EINVAL"):
        T.set_etlru_model(-1.0, [0.0])
    with pytest.raises(T.TlruError, match="EINVAL"):
        T.set_etlru_model(0.1, [0.0, 0.5])  # not a log-probability


def test_full_size_sampled(T):
    """BASELINE trace size (10^6 conversations) in the launch configuration of
    `bench.py --config etlru` (one trace, its 100 rows in one batch); sampled instances vs the oracle."""
    from paper_2510_15152_b200.inputs import CAPS_CONFIG5
    p = preset("wildchat", 2, 1_000_000)
    mu = p["death_rate"] * 1e-6
    tab = prompt_law_ln_surv(WILDCHAT)
    T.set_etlru_model(mu, tab)
    tr = T.generate_traces([p], exports=True)[0]
    rows = [(0, ET, C, xi, 2, SLO_BLOCKS) for C in CAPS_CONFIG5 for xi in (4, 8, 16, 24)]
    bt = T.simulate_batch([tr], rows)
    assert T.last_sim_stats()["failed_chains"] == 0
    o = O.generate(p)
    res = bt.results_numpy()
    for C, xi in ((16, 4), (256, 16), (CAPS_CONFIG5[20], 24)):
        i = rows.index((0, ET, C, xi, 2, SLO_BLOCKS))
        r = O.replay_etlru(o.conv, o.q, o.a, o.ticks, C, xi, mu, tab)
        assert np.array_equal(bt.b(i).astype(np.uint64), r.b), (C, xi)
        assert (res[i]["evicted_trim"], res[i]["evicted_lru"]) == (r.evicted_trim, r.evicted_lru)


def test_short_segments_verified(T):
    """Short time segments (256 events, burn-in 4096) on a trace with few, long-lived
    conversations: the burn-in segments' start states are checked against the exact end states
    of their predecessors and re-run where they differ; outputs stay exact."""
    tab = TABLES[0]
    T.set_etlru_model(0.02, tab)
    conv, q, a = random_trace(4200, 20000, 30, q_max=4, a_max=4, locality=0.1)
    ticks = np.cumsum(np.random.default_rng(4).integers(0, 5, size=conv.size)).astype(np.uint64)
    tr = upload_ticks(T, conv, q, a, ticks)
    rows = [(0, ET, C, xi, 0, 8) for C in (8, 40, 150, 600) for xi in (0, 3, 9)]
    T.set_sim_options(256, 0)
    try:
        bt = T.simulate_batch([tr], rows)
        st = T.last_sim_stats()
    finally:
        T.set_sim_options(0, 0)
    assert st["failed_chains"] == 0
    check_et(bt, rows, [(conv, q, a, ticks)], 0.02, tab)


def test_long_prompt_law_table(T):
    """A prompt law with K = 700 > the 256 table entries kept in shared memory: the kernel reads
    the tail of ln P(Q >= k) from global memory.  Large xi makes k = X - L + xi reach it."""
    K = 700
    tab = [0.0, 0.0] + [math.log(max(1e-300, (1.0 - k / (K + 1.0)) ** 3)) for k in range(2, K + 1)]
    tab = list(np.minimum.accumulate(np.array(tab)))
    T.set_etlru_model(0.03, tab)
    conv, q, a = random_trace(4300, 4000, 40, q_max=30, a_max=30, locality=0.6)
    ticks = np.cumsum(np.random.default_rng(7).integers(0, 3, size=conv.size)).astype(np.uint64)
    tr = upload_ticks(T, conv, q, a, ticks)
    rows = [(0, ET, C, xi, 0, 8) for C in (50, 300, 1500) for xi in (200, 450, 690)]
    bt = T.simulate_batch([tr], rows)
    check_et(bt, rows, [(conv, q, a, ticks)], 0.03, tab)


@pytest.mark.parametrize("entries", [256, 512, 1024])
def test_incremental_candidates_forced_class(T, entries):
    """ET-LRU / forced ET-LRU in the slot classes that keep incremental eviction candidates
    (et_rescan / et_offer), forced onto small random traces with short segments (the fix-up path
    loads snapshots into them): element by element against the oracle."""
    mu = 0.3
    T.set_etlru_model(mu, TABLES[0])
    rng = np.random.default_rng(entries)
    conv, q, a = random_trace(4300 + entries, 4000, 60, q_max=5, a_max=7, locality=0.5)
    ticks = np.cumsum(rng.integers(0, 3, size=conv.size)).astype(np.uint64)
    tr = upload_ticks(T, conv, q, a, ticks)
    rows = [(0, pol, C, xi, 0, 8) for pol in (ET, 9) for C in (0, 2, 15, 60, 250) for xi in (0, 3, 9)]
    for seg in (0, 256):
        T.set_sim_options(seg, entries)
        try:
            bt = T.simulate_batch([tr], rows)
            assert T.last_sim_stats()["failed_chains"] == 0
        finally:
            T.set_sim_options(0, 0)
        for i, (t, pol, C, xi, qh, slo) in enumerate(rows):
            o = O.replay_etlru(conv, q, a, ticks, C, xi, mu, TABLES[0], forced=pol != ET)
            assert np.array_equal(bt.b(i).astype(np.uint64), o.b), (seg, rows[i])
            r = bt.results_numpy()[i]
            assert (r["evicted_trim"], r["evicted_lru"], r["max_occupancy"]) == (o.evicted_trim, o.evicted_lru,
                                                                               o.max_occupancy), (seg, rows[i])
