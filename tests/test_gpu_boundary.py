"""Boundary behaviour of tlru_simulate_batch(_ex) added in round 2, through the C ABI, vs the oracle:

* a batch that mixes stack-eligible policies (LRU, T-LRU, Threshold-LRU) with replay-only ones
  (End-/Length-Aware, Tail-Optimized Belady, forced caching, ET-LRU) runs BOTH engines, each on
  its own instances (stats.engine = MIXED), with results identical to single-policy batches and
  to the oracle;
* the per-instance histograms of b (tlru_simulate_batch_ex) equal np.bincount of the oracle's b;
* pooled histograms (tlru_pool_histograms + tlru_tail_from_histograms, row a10) equal the oracle's
  tail metrics over the concatenated b of each pool's instances;
* a trace whose universe exceeds the stack engine's 32-bit window sums runs on the replay engine;
* Belady lanes stay exact when tlru_set_sim_options asks for 1024-entry states.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2510_15152_b200.inputs import (ALPHA_MS, WILDCHAT, preset, prompt_law_ln_surv, random_trace)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2510_15152_b200.tlru as T
    T.set_sim_options(0, 0)
    T.set_sim_engine(T.ENGINE_STACK)
    yield T
    T.set_sim_options(0, 0)
    T.set_sim_engine(T.ENGINE_STACK)


def oracle_b(ot, row, mu=None, tab=None):
    t, pol, C, xi, qh = row[:5]
    if pol == O.ET_LRU:
        return O.replay_etlru(ot.conv, ot.q, ot.a, ot.ticks, C, xi, mu, tab)
    return O.replay(ot.conv, ot.q, ot.a, pol, C, xi, qh, threshold=row[6] if len(row) > 6 else 0)


def test_mixed_batch_runs_both_engines(T):
    p = preset("wildchat", 11, 4000)
    ot = O.generate(p)
    g = T.generate_traces([p])[0]
    mu, tab = p["death_rate"] * 1e-6, prompt_law_ln_surv(WILDCHAT)
    T.set_etlru_model(mu, tab)
    rows = []
    for C in (16, 90, 700):
        rows += [(0, 0, C, 8, 2, 16), (0, 1, C, 12, 2, 16), (0, 2, C, 8, 2, 16, 8), (0, 3, C, 12, 2, 16),
                 (0, 4, C, 12, 2, 16), (0, 5, C, 12, 2, 16), (0, 6, C, 12, 2, 16), (0, 7, C, 12, 2, 16)]
    rng = np.random.default_rng(3)
    rows = [rows[k] for k in rng.permutation(len(rows))]  # engines interleaved in instance order
    bins = g.max_history + 5
    bt = T.simulate_batch([g], rows, hist_bins=bins)
    st = T.last_sim_stats()
    assert st["engine"] == T.ENGINE_MIXED and st["failed_chains"] == 0
    res = bt.results_numpy()
    hist = bt.hist.cpu().numpy().view(np.uint32).reshape(len(rows), bins)
    for i, row in enumerate(rows):
        r = oracle_b(ot, row, mu, tab)
        assert np.array_equal(bt.b(i).astype(np.uint64), r.b), row
        assert np.array_equal(hist[i], np.bincount(r.b.astype(np.int64), minlength=bins)), row
        tl = O.tail(r.b, row[3], ALPHA_MS * row[3], row[5], ALPHA_MS)
        assert (res[i]["tel_blocks"], res[i]["p90"], res[i]["p95"], res[i]["slo_violations"]) == (
            tl.tel_blocks, tl.p90, tl.p95, tl.slo_violations), row
        assert res[i]["evicted_trim"] == r.evicted_trim and res[i]["evicted_lru"] == r.evicted_lru, row
    # the same instances one engine at a time give identical bytes
    stack_ids = [i for i, r in enumerate(rows) if r[1] <= 2]
    solo = T.simulate_batch([g], [rows[i] for i in stack_ids])
    assert T.last_sim_stats()["engine"] == T.ENGINE_STACK
    assert solo.results_numpy().tobytes() == res[stack_ids].tobytes()


@pytest.mark.parametrize("engine", [0, 1], ids=["replay", "stack"])
def test_histogram_export_and_pooled_metrics(T, engine):
    """Pools = (C, xi, policy) over 3 seeds, as the config-5 sweep pools over its 10 seeds."""
    T.set_sim_engine(engine)
    ps = [preset("wildchat", s, 3000) for s in (21, 22, 23)]
    ots = [O.generate(p) for p in ps]
    gs = T.generate_traces(ps)
    cfg = [(pol, C, xi) for pol in (0, 1) for C in (32, 256) for xi in (4, 16)]
    rows = [(t, pol, C, xi, 2, 16) for t in range(3) for (pol, C, xi) in cfg]
    bins = 1025
    bt = T.simulate_batch(gs, rows, hist_bins=bins)
    pool = [cfg.index((r[1], r[2], r[3])) for r in rows]
    pool[5] = T.TLRU_NONE  # skipped instance
    pooled = T.pool_histograms(bt.hist, bins, pool, len(cfg))
    out = T.tail_from_histograms(pooled, bins, [c[2] for c in cfg], [ALPHA_MS * c[2] for c in cfg],
                                 [16] * len(cfg), ALPHA_MS).cpu().numpy().view(T.TAIL_DTYPE)
    for k, (pol, C, xi) in enumerate(cfg):
        bs = [O.replay(ots[r[0]].conv, ots[r[0]].q, ots[r[0]].a, pol, C, xi, 2).b
              for i, r in enumerate(rows) if pool[i] == k]
        tl = O.tail(np.concatenate(bs), xi, ALPHA_MS * xi, 16, ALPHA_MS)
        o = out[k]
        assert (o["n"], o["tel_blocks"], o["slo_violations"], o["sum_b"]) == (tl.n, tl.tel_blocks,
                                                                              tl.slo_violations, tl.sum_b)
        assert (o["p50"], o["p90"], o["p95"], o["p99"]) == (tl.p50, tl.p90, tl.p95, tl.p99)
        for f in ("tel_ms", "p50_ms", "p90_ms", "p95_ms", "p99_ms", "mean_ms"):
            assert o[f] == pytest.approx(getattr(tl, f), rel=1e-9, abs=1e-12), f
    with pytest.raises(T.TlruError, match="ERANGE"):  # hist_bins must exceed max_history
        T.simulate_batch(gs, rows[:2], hist_bins=max(g.max_history for g in gs))
    with pytest.raises(T.TlruError, match="EINVAL"):
        T.pool_histograms(bt.hist, bins, [len(cfg)] * len(rows), len(cfg))
    T.set_sim_engine(T.ENGINE_STACK)


def test_universe_beyond_32_bits_runs_on_the_replay_engine(T):
    """65537 conversations of 65535 blocks: a universe of 2^32 + 2^16 - 1 blocks exceeds the stack
    engine's 32-bit window sums, so LRU / T-LRU instances on it run on the replay engine (exact)."""
    n = 65537
    qq = torch.from_numpy(np.full(n, 65535, np.uint16).view(np.int16)).cuda()
    aa = torch.zeros(n, dtype=torch.int16, device="cuda")
    twice = np.arange(n, dtype=np.uint32)
    twice[-1] = 0  # conversation 0 returns: 131070 blocks > 65535
    with pytest.raises(T.TlruError, match="ERANGE"):
        T.trace_from_turns(torch.from_numpy(twice.view(np.int32)).cuda(), qq, aa)
    ids = torch.arange(n, dtype=torch.int32, device="cuda")
    tr = T.trace_from_turns(ids[: n - 1], qq[: n - 1], aa[: n - 1])
    assert tr.universe_blocks == (n - 1) * 65535 == 0xFFFF0000  # the stack engine's limit
    tr2 = T.trace_from_turns(ids, qq, aa)
    assert tr2.universe_blocks == n * 65535 > 0xFFFF0000
    rows = [(0, 0, 100000, 4, 2, 16), (0, 1, 70000, 8, 2, 16)]
    bt = T.simulate_batch([tr2], rows)
    assert T.last_sim_stats()["engine"] == T.ENGINE_REPLAY
    for i in range(2):
        assert np.all(bt.b(i) == 65535)
    bt = T.simulate_batch([tr], rows)
    assert T.last_sim_stats()["engine"] == T.ENGINE_STACK


def test_belady_lanes_with_1024_entry_option(T):
    """state_entries = 1024 must not send Belady lanes to an unlaunched class."""
    conv, q, a = random_trace(5, 6000, 300)
    c = torch.from_numpy(conv.view(np.int32)).cuda()
    qq = torch.from_numpy(q.astype(np.uint16).view(np.int16)).cuda()
    aa = torch.from_numpy(a.astype(np.uint16).view(np.int16)).cuda()
    tr = T.trace_from_turns(c, qq, aa)
    rows = [(0, 5, C, xi, 2, 16) for C in (8, 64, 400, 3000) for xi in (0, 6)] + [(0, 3, 64, 6, 2, 16),
                                                                                    (0, 4, 400, 6, 2, 16)]
    for opt in (0, 1024, 32):
        T.set_sim_options(0, opt)
        bt = T.simulate_batch([tr], rows)
        assert T.last_sim_stats()["failed_chains"] == 0
        for i, r in enumerate(rows):
            o = O.replay(conv, q, a, r[1], r[2], r[3], r[4])
            assert np.array_equal(bt.b(i).astype(np.uint64), o.b), (opt, r)
    T.set_sim_options(0, 0)
