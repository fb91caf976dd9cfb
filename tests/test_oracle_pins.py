"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Each test cites the passage or the independent fact it checks.  A plausible
mistake in the oracle (a dropped term, a wrong sign or index, a transposed
operand, the weak-inequality budget, newest-first trimming, literal one-block
Phase 1) fails at least one of these.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
from stackdist import topc_replay
from paper_2510_15152_b200.inputs import random_trace, tiny_trace

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def tel(b, xi):
    return int(sum(max(int(x) - xi, 0) for x in b))


# ----------------------------------------------------------------------------- Figure 1
def test_fig1_worked_example():
    """P:37 / P:62: LRU max uncached 200, T-LRU(xi=150, Q_hat=100) 150, 25% lower."""
    g = json.load(open(os.path.join(GOLDEN, "fig1.json")))
    lru = O.replay(g["conv"], g["q"], g["a"], O.LRU, g["C"])
    tl = O.replay(g["conv"], g["q"], g["a"], O.TLRU, g["C"], g["xi"], g["q_hat"])
    assert list(lru.b) == [100, 100, 200]
    assert list(tl.b) == [100, 100, 150]
    assert int(lru.b.max()) == g["lru_max_uncached"]
    assert int(tl.b.max()) == g["tlru_max_uncached"]
    assert 100.0 * (1 - tl.b.max() / lru.b.max()) == g["improvement_pct"]
    # "66.7th percentile = max" with nearest rank on 3 requests: k = ceil(0.667 * 3) = 3
    k = (int(g["tail_percentile"] * 100) * 3 + 9999) // 10000
    assert k == 3 and sorted(tl.b)[k - 1] == 150
    # TEL at xi = 150 blocks: LRU 50, T-LRU 0; sums 400 vs 350
    assert tel(lru.b, 150) == 50 and tel(tl.b, 150) == 0
    assert lru.b.sum() == 400 and tl.b.sum() == 350
    # evictions: LRU 300 (all Phase 2); T-LRU 150 Phase 1 + 100 Phase 2
    assert (lru.evicted_trim, lru.evicted_lru) == (0, 300)
    assert (tl.evicted_trim, tl.evicted_lru) == (150, 100)
    assert lru.max_occupancy == 100 and tl.max_occupancy == 100


def test_fig1_state_after_step2_is_50_50():
    """'both A and B retain 50 cached' -> third request from A or B: 150."""
    for third in (0, 1):
        tl = O.replay([0, 1, third], [100] * 3, [0] * 3, O.TLRU, 100, 150, 100)
        assert int(tl.b[2]) == 150
    lru_b = O.replay([0, 1, 1], [100] * 3, [0] * 3, O.LRU, 100)
    assert list(lru_b.b) == [100, 100, 100]


def test_fig1_rules_out_literal_and_weak_readings():
    """Readings #1/#2: literal one-block Phase 1 would give 199 and the weak
    budget 151 (SURVEY c.3); the oracle must give the paper's 150."""
    tl = O.replay([0, 1, 0], [100] * 3, [0] * 3, O.TLRU, 100, 150, 100)
    assert int(tl.b[2]) not in (199, 151)


# ----------------------------------------------------------------------------- convention vectors
@pytest.mark.parametrize("conv,q,a,C,xi,qh,lru_b,tlru_b", [
    ([0, 1, 0], [2, 2, 2], [0, 0, 0], 2, 3, 2, [2, 2, 4], [2, 2, 3]),   # Fig. 1 / 50
    ([0, 1, 0], [1, 1, 1], [0, 0, 0], 1, 2, 1, [1, 1, 2], [1, 1, 2]),   # oldest-first free order (Reading #3)
    ([0, 0], [3, 2], [2, 0], 4, 3, 1, [3, 3], [3, 3]),                  # theta alone exceeds C (self-trim)
])
def test_convention_vectors(conv, q, a, C, xi, qh, lru_b, tlru_b):
    assert list(O.replay(conv, q, a, O.LRU, C).b) == lru_b
    assert list(O.replay(conv, q, a, O.TLRU, C, xi, qh).b) == tlru_b


def test_fig2_budget_zero_then_exact_budget():
    """Fig. 2: turn 1 with L1 + Q < xi needs no caching (budget 0); turn 2
    with L2 + Q > xi keeps exactly L2 + Q - xi blocks under pressure."""
    # A: q=1,a=1 (L1=2; 2+1 < 4 -> budget 0); B: q=3 forces overflow 2; A: q=1,a=3; A: q=1
    conv, q, a = [0, 1, 0, 0], [1, 3, 1, 1], [1, 0, 3, 0]
    r = O.replay(conv, q, a, O.TLRU, 3, 4, 1)
    # step 2: Phase 1 evicts all of A (free) -> A's second request is fully uncached: J = 3
    assert int(r.b[2]) == 3
    # after step 3: L2 = 6, budget = 6 + 1 - 4 = 3 -> X_A = 3 -> b = 7 - 3 = 4 = xi
    assert int(r.b[3]) == 4
    assert tel(r.b, 4) == 0


def test_spec_lru_evict_example():
    """S:213-214 lru_evict: tau {A:1, B:2}, X {3, 3}, overflow 4 -> 3 from A, 1 from B."""
    # A(3), B(3), D(4) with C = 6 -> overflow 4; then B and A return with q = 1
    r = O.replay([0, 1, 2, 1, 0], [3, 3, 4, 1, 1], [0] * 5, O.LRU, 6)
    assert list(r.b) == [3, 3, 4, 2, 4]


# ----------------------------------------------------------------------------- metrics
def test_metrics_spec_examples():
    """tel([100,250,300],200)=150; slo(...)=2; slo([200],200)=0;
    percentile([1..10], 90) = 9 (nearest rank, Reading #11)."""
    t = O.tail([100, 250, 300], 200, 200.0, 200, 1.0)
    assert t.tel_blocks == 150 and t.slo_violations == 2 and t.tel_ms == 150.0
    assert O.tail([200], 0, 0.0, 200, 1.0).slo_violations == 0
    t = O.tail(list(range(1, 11)), 0, 0.0, 0, 1.0)
    assert t.p90 == 9 and t.p50 == 5 and t.p95 == 10 and t.p99 == 10
    assert O.tail([], 0, 0.0, 0, 12.5).n == 0


def test_metrics_ms_fields_alpha():
    """Eq. 2: ttft = alpha*b; TEL_ms = alpha*TEL_blocks when xi_s = alpha*xi (Eq. 3)."""
    rng = np.random.default_rng(3)
    b = rng.integers(0, 60, size=1001)
    t = O.tail(b, 16, 200.0, 16, 12.5)
    assert t.tel_ms == 12.5 * t.tel_blocks
    assert t.p90_ms == 12.5 * t.p90 and t.mean_ms == pytest.approx(12.5 * b.mean(), rel=1e-12)
    sb = np.sort(b)
    assert t.p90 == sb[math.ceil(0.9 * b.size) - 1]


# ----------------------------------------------------------------------------- closed form
def _cells():
    for seed in range(120):
        conv, q, a = random_trace(seed, 50, 10, q_max=6, a_max=6)
        for C in (0, 1, 5, 13, 40):
            for xi, qh in ((0, 0), (4, 1), (9, 2), (30, 2)):
                yield seed, conv, q, a, C, xi, qh


def test_replay_equals_topc_closed_form():
    """Independent algorithm (tests/stackdist.py): cache = top-C blocks of the
    universe under the static key (non-free?, tau, -position).  For D = 0 this is
    the Mattson weighted-reuse-distance form of LRU."""
    n = 0
    for seed, conv, q, a, C, xi, qh in _cells():
        for pol in (O.LRU, O.TLRU):
            D = max(xi - qh, 0) if pol == O.TLRU else 0
            r = O.replay(conv, q, a, pol, C, xi, qh)
            assert list(r.b) == topc_replay(conv, q, a, C, D), (seed, C, xi, qh, pol)
            n += 1
    assert n == 120 * 5 * 4 * 2


def test_tiny_traces_closed_form_all_params():
    """BASELINE config 2 grid on the oracle: every C in [0,8], xi in [0,5], Q_hat in [0,3]."""
    for seed in range(60):
        conv, q, a = tiny_trace(seed)
        for C in range(9):
            for xi in range(6):
                for qh in range(4):
                    r = O.replay(conv, q, a, O.TLRU, C, xi, qh)
                    assert list(r.b) == topc_replay(conv, q, a, C, max(xi - qh, 0))


# ----------------------------------------------------------------------------- invariants
def test_invariants_random():
    for seed in range(80):
        conv, q, a = random_trace(seed, 80, 12)
        d = O.derive(conv, q, a)
        first = d.prev == O.NONE
        total = int(q.sum() + a.sum())
        for C in (0, 3, 9, 27, 81, total):
            for pol, xi, qh in ((O.LRU, 0, 0), (O.TLRU, 7, 2), (O.TLRU, 2, 2), (O.TLRU, 20, 0)):
                r = O.replay(conv, q, a, pol, C, xi, qh)
                assert np.all(r.b >= q) and np.all(r.b <= d.J)              # q <= b <= J
                assert np.all(r.b[first] == q[first])                        # first turn b = q
                assert r.max_occupancy <= C                                  # constraint (2)
                if C == 0:
                    assert np.array_equal(r.b, d.J)
                if C >= total:
                    assert np.array_equal(r.b, q.astype(np.uint64))
            # T-LRU with xi <= Q_hat is LRU exactly (D = 0)
            lru = O.replay(conv, q, a, O.LRU, C)
            same = O.replay(conv, q, a, O.TLRU, C, 2, 2)
            assert np.array_equal(lru.b, same.b) and same.evicted_trim == 0
            assert same.evicted_lru == lru.evicted_lru


def test_inclusion_monotone_in_capacity():
    """Stack property: per-request b non-increasing in C for both policies."""
    for seed in range(60):
        conv, q, a = random_trace(seed, 70, 9)
        for pol, xi, qh in ((O.LRU, 0, 0), (O.TLRU, 10, 2), (O.TLRU, 30, 1)):
            prev = None
            for C in range(0, 60, 3):
                b = O.replay(conv, q, a, pol, C, xi, qh).b
                if prev is not None:
                    assert np.all(b <= prev)
                prev = b


def test_tlru_never_worse_than_lru_deterministic_q():
    """SURVEY c.3 #22: pathwise TEL(T-LRU) <= TEL(LRU) when every q equals Q_hat."""
    for seed in range(80):
        conv, _, a = random_trace(seed, 60, 8)
        qv = 3
        q = np.full(conv.shape, qv, np.uint32)
        for C in (5, 15, 40):
            for xi in (4, 8, 15):
                t = O.replay(conv, q, a, O.TLRU, C, xi, qv)
                l = O.replay(conv, q, a, O.LRU, C)
                assert tel(t.b, xi) <= tel(l.b, xi)


# ----------------------------------------------------------------------------- derive
def test_derive_links_and_prefix_sums():
    conv, q, a = random_trace(7, 300, 25)
    d = O.derive(conv, q, a)
    for e in range(conv.size):
        p = int(d.prev[e])
        if p == O.NONE:
            assert d.J[e] == q[e]
            assert not np.any(conv[:e] == conv[e])
        else:
            assert conv[p] == conv[e] and not np.any(conv[p + 1:e] == conv[e])
            assert d.next[p] == e
            assert d.J[e] == d.L_after[p] + q[e]
        assert d.L_after[e] == d.J[e] + a[e]
