"""Pins of the oracle's ET-LRU under forced caching (App. C; Reading #30): the decision
space X_F(X, theta, L) fixes Y_theta = L, and App. C states that Thm 3 continues to hold -- ET-LRU
stays optimal -- with a known fixed prompt length and homogeneous turn rates, where it "is reduced to
a deterministic version", i.e. T-LRU, here forced T-LRU (Reading #28, itself pinned to the
forced belief-MDP optimum in tests/test_oracle_forced.py).  No GPU."""
import numpy as np
import pytest

import oracle as O
from paper_2510_15152_b200.inputs import random_trace
from test_oracle_etlru import PMFS, ln_table, point_mass_table, times_for


@pytest.mark.parametrize("seed", range(5))
def test_deterministic_q_reduces_to_forced_tlru(seed):
    """with a fixed prompt length Q_hat, forced ET-LRU is forced T-LRU: identical b, P = 0
    (Phase-1) and other (Phase-2 + theta's own overflow) evictions, occupancy."""
    conv, q, a = random_trace(5000 + seed, 900, 35, q_max=5, a_max=5, locality=0.6)
    ticks = times_for(conv.size, np.random.default_rng(50 + seed))
    for C in (0, 3, 16, 60, 250):
        for xi, qh in ((0, 0), (3, 1), (6, 2), (15, 3), (30, 2)):
            for mu in (1e-6, 0.3, 7.0):
                e = O.replay_etlru(conv, q, a, ticks, C, xi, mu, point_mass_table(qh), forced=True)
                t = O.replay(conv, q, a, O.TLRU_FORCED, C, xi, qh)
                assert np.array_equal(e.b, t.b), (C, xi, qh, mu)
                assert (e.evicted_trim, e.evicted_lru, e.max_occupancy) == (t.evicted_trim, t.evicted_lru,
                                                                            t.max_occupancy)


@pytest.mark.parametrize("seed", range(3))
def test_xi0_reduces_to_lru(seed):
    """xi = 0: every block has P = 1, the criterion is recency alone; theta, the most
    recent, is never the greedy's choice before the others are gone, so forcing changes nothing:
    LRU, whatever the prompt law."""
    conv, q, a = random_trace(5100 + seed, 900, 35, q_max=5, a_max=5, locality=0.6)
    ticks = times_for(conv.size, np.random.default_rng(60 + seed), ties=False)
    for C in (0, 4, 20, 90):
        for pmf in PMFS:
            e = O.replay_etlru(conv, q, a, ticks, C, 0, 0.05, ln_table(pmf), forced=True)
            l = O.replay(conv, q, a, O.LRU, C)
            assert np.array_equal(e.b, l.b) and e.evicted_lru == l.evicted_lru and e.evicted_trim == 0


def test_fig1_forced_point_mass():
    """Fig. 1 with Q = 100 under forced caching: B must keep its 100 blocks, so A's budget
    trim (50 above (100 + 100 - 150)^+) is not enough: A pays 200 (forced T-LRU's vector)."""
    e = O.replay_etlru([0, 1, 0], [100, 100, 100], [0, 0, 0], [0, 5, 9], 100, 150, 0.01, point_mass_table(100),
                       forced=True)
    t = O.replay([0, 1, 0], [100, 100, 100], [0, 0, 0], O.TLRU_FORCED, 100, 150, 100)
    assert [int(x) for x in e.b] == [int(x) for x in t.b] == [100, 100, 200]
    assert (e.evicted_trim, e.evicted_lru) == (t.evicted_trim, t.evicted_lru)


@pytest.mark.parametrize("seed", range(3))
def test_forced_invariants(seed):
    """Occupancy <= C; evicted = Sum(a + b) - min(C, Sum(a + b)) (no release); a request whose
    history fits (L_after <= C) leaves theta fully cached, so a next turn that follows immediately
    pays exactly q."""
    conv, q, a = random_trace(5200 + seed, 500, 25)
    ticks = times_for(conv.size, np.random.default_rng(70 + seed))
    d = O.derive(conv, q, a)
    tab = ln_table(PMFS[seed])
    for C in (5, 40, 150):
        r = O.replay_etlru(conv, q, a, ticks, C, 4, 0.1, tab, forced=True)
        ins = int(a.astype(np.int64).sum() + r.b.astype(np.int64).sum())
        assert r.max_occupancy == min(C, ins) and r.evicted_trim + r.evicted_lru == ins - min(C, ins)
        nxt = np.full(conv.size, -1)
        last = {}
        for e in range(conv.size - 1, -1, -1):
            nxt[e] = last.get(int(conv[e]), -1)
            last[int(conv[e])] = e
        for e in range(conv.size):
            n = nxt[e]
            if n >= 0 and n == e + 1 and int(d.L_after[e]) <= C:  # no request in between
                assert int(r.b[n]) == int(q[n]), (C, e)
