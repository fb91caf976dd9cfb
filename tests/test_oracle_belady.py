"""Pins of the oracle's Tail-Optimized Belady (Thm 1; proof App. A, P:468-508;
SPEC S:244-252; Reading #26).  No GPU.

The strongest pin is Theorem 1 itself: on tiny traces the policy's TEL equals the exact
hindsight optimum of Eq. (5) (oracle/brute.py hindsight_opt, a dynamic program over every
feasible cache schedule -- no eviction rule in it), for every xi; with xi = 0 its total
uncached blocks equal the optimum of average latency (classical Belady)."""
import json
import os
import random

import numpy as np
import pytest

import oracle as O
from oracle.brute import hindsight_opt
from paper_2510_15152_b200.inputs import random_trace, tiny_trace

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def tel(b, xi):
    return int(np.maximum(np.asarray(b, dtype=np.int64) - xi, 0).sum())


def test_fig1_known_third_request():
    g = json.load(open(os.path.join(GOLDEN, "tail_belady.json")))["fig1_known_third"]
    for key in ("third_from_A", "third_from_B"):
        v = g[key]
        r = O.replay(v["conv"], v["q"], v["a"], O.TAIL_BELADY, g["C"], g["xi"])
        assert [int(x) for x in r.b] == v["b"], key
        assert [r.evicted_trim, r.evicted_lru] == v["evicted"] and r.max_occupancy == v["max_occupancy"]
        assert tel(r.b, g["xi"]) == v["tel"] == hindsight_opt(np.array(v["conv"]), np.array(v["q"]),
                                                               np.array(v["a"]), g["C"], g["xi"])
        # online T-LRU hedges to 150 and LRU pays 200 on the A-variant
        t = O.replay(v["conv"], v["q"], v["a"], O.TLRU, g["C"], g["xi"], 100)
        assert max(int(x) for x in t.b) == 150


def test_furthest_in_future_order():
    v = json.load(open(os.path.join(GOLDEN, "tail_belady.json")))["furthest_order"]
    r = O.replay(v["conv"], v["q"], v["a"], O.TAIL_BELADY, v["C"], v["xi"])
    assert [int(x) for x in r.b] == v["b"]
    assert [r.evicted_trim, r.evicted_lru] == v["evicted"] and r.max_occupancy == v["max_occupancy"]
    assert [int(x) for x in O.replay(v["conv"], v["q"], v["a"], O.LRU, v["C"]).b] == v["lru_b"]


@pytest.mark.parametrize("chunk", range(6))
def test_thm1_tail_belady_attains_hindsight_optimum(chunk):
    """Thm 1: TEL of Tail-Optimized Belady == min over all cache schedules
    obeying (2)-(4) of Eq. (5).  The test has power: T-LRU and LRU miss the optimum on a
    share of the same instances."""
    rnd = random.Random(100 + chunk)
    n = miss = 0
    for seed in range(60 * chunk, 60 * chunk + 60):
        nc = 4 if chunk >= 4 else 3
        conv, q, a = tiny_trace(seed, max_conv=nc, max_turns=3, qs=(1, 2, 3), as_=(0, 1, 2))
        if conv.size > 8:
            conv, q, a = conv[:8], q[:8], a[:8]
        C = rnd.randint(0, 6)
        xi = rnd.randint(0, 5)
        opt = hindsight_opt(conv, q, a, C, xi)
        r = O.replay(conv, q, a, O.TAIL_BELADY, C, xi)
        assert tel(r.b, xi) == opt, (seed, C, xi)
        t = O.replay(conv, q, a, O.TLRU, C, xi, 2)
        miss += tel(t.b, xi) > opt
        n += 1
    assert miss > 0


def test_thm1_xi0_is_belady_average_latency_optimum():
    """xi = 0: 'we recover the Belady optimal policy' -- the total of uncached blocks
    (TEL at xi = 0) is the hindsight minimum, and never above LRU's."""
    rnd = random.Random(7)
    strict = 0
    for seed in range(160):
        conv, q, a = tiny_trace(1000 + seed, max_conv=3, max_turns=3, qs=(1, 2, 3), as_=(0, 1))
        C = rnd.randint(1, 6)
        r = O.replay(conv, q, a, O.TAIL_BELADY, C, 0)
        lru = O.replay(conv, q, a, O.LRU, C)
        assert int(r.b.sum()) == hindsight_opt(conv, q, a, C, 0)
        assert int(r.b.sum()) <= int(lru.b.sum())
        strict += int(r.b.sum()) < int(lru.b.sum())
    assert strict > 0


@pytest.mark.parametrize("seed", range(6))
def test_hindsight_policy_never_worse_pathwise(seed):
    """Optimality at any size: TEL(T-Belady) <= TEL of every online policy on the same trace
    (LRU, T-LRU, End-/Length-Aware T-LRU, Threshold-LRU), for every C and xi."""
    conv, q, a = random_trace(900 + seed, 600, 30, q_max=6, a_max=6, locality=0.6)
    for C in (0, 4, 17, 60, 150):
        for xi in (0, 3, 8, 14):
            tb = tel(O.replay(conv, q, a, O.TAIL_BELADY, C, xi).b, xi)
            for pol, qh in ((O.LRU, 0), (O.TLRU, 3), (O.END_AWARE, 3), (O.LENGTH_AWARE, 3)):
                assert tb <= tel(O.replay(conv, q, a, pol, C, xi, qh).b, xi), (C, xi, pol)
            assert tb <= tel(O.replay(conv, q, a, O.THRESHOLD, C, xi, 0, 5).b, xi)


@pytest.mark.parametrize("seed", range(4))
def test_special_cases_and_invariants(seed):
    """C = 0 -> b = J; C >= total history -> returning requests find everything (b = q) and
    nothing is evicted; b >= q; occupancy <= C.  Evictions telescope: every request
    inserts L_after - X_old = a + b blocks and nothing is released, so the cache fills to
    min(C, inserted) and stays there: evicted = Sum(a + b) - min(C, Sum(a + b))."""
    conv, q, a = random_trace(950 + seed, 400, 25)
    d = O.derive(conv, q, a)
    r0 = O.replay(conv, q, a, O.TAIL_BELADY, 0, 5)
    assert np.array_equal(r0.b, d.J.astype(np.uint64))
    big = int((q.astype(np.int64) + a).sum())
    rb = O.replay(conv, q, a, O.TAIL_BELADY, big, 5)
    assert np.array_equal(rb.b, q.astype(np.uint64)) and rb.evicted_trim + rb.evicted_lru == 0
    for C in (3, 20, 90, 400):
        for xi in (0, 6, 30):
            r = O.replay(conv, q, a, O.TAIL_BELADY, C, xi)
            assert np.all(r.b >= q) and r.max_occupancy <= C
            ins = int(a.astype(np.int64).sum() + r.b.astype(np.int64).sum())
            assert r.evicted_trim + r.evicted_lru == ins - min(C, ins)
            assert r.max_occupancy == min(C, ins)
            if xi == 0:
                # xi = 0: only never-returning conversations hold free blocks
                pass


# ----------------------------------------------------------------------------- forced caching (App. C)
def test_forced_belady_hand_vector():
    """Fig. 1 under forced caching (Reading #29): B must keep its 100 blocks, so A pays 200."""
    v = json.load(open(os.path.join(GOLDEN, "tail_belady.json")))["fig1_forced"]
    r = O.replay(v["conv"], v["q"], v["a"], O.BELADY_FORCED, v["C"], v["xi"])
    assert [int(x) for x in r.b] == v["b"]
    assert [r.evicted_trim, r.evicted_lru] == v["evicted"] and r.max_occupancy == v["max_occupancy"]
    assert tel(r.b, v["xi"]) == v["tel"] == hindsight_opt(np.array(v["conv"]), np.array(v["q"]),
                                                           np.array(v["a"]), v["C"], v["xi"], forced=True)


def test_forced_belady_attains_the_forced_hindsight_optimum():
    """App. C: Theorem 1 continues to hold under forced caching -- the forced
    Tail-Optimized Belady's TEL equals the exact forced hindsight optimum (Eq. 5 with constraint
    (3) as an equality; a DP over every feasible schedule, no eviction rule in it) on tiny traces,
    for every xi.  Power: it differs from the optional-caching Belady on a quarter of them, and it
    never exceeds forced T-LRU."""
    rnd = random.Random(9)
    n = differs = 0
    for seed in range(690):
        if seed < 400:
            conv, q, a = tiny_trace(seed, max_conv=3, max_turns=2, qs=(1, 2), as_=(0, 1))
        else:
            conv, q, a = tiny_trace(1000 + seed, max_conv=3, max_turns=3, qs=(1, 2, 3), as_=(0, 1, 2))
            if len(conv) > 7:
                continue
        C, xi = rnd.randint(0, 6), rnd.randint(0, 4)
        r = O.replay(conv, q, a, O.BELADY_FORCED, C, xi)
        got = tel(r.b, xi)
        assert got == hindsight_opt(conv, q, a, C, xi, forced=True), (seed, C, xi)
        assert got <= tel(O.replay(conv, q, a, O.TLRU_FORCED, C, xi, 1).b, xi)
        differs += got != tel(O.replay(conv, q, a, O.TAIL_BELADY, C, xi).b, xi)
        n += 1
    assert n >= 600 and differs >= 40


def test_forced_belady_invariants():
    """Occupancy <= C after every request, b >= q, first turns b = q, eviction identity
    (inserted - cached at the end), and theta keeps min(L, C) blocks after its own request."""
    for seed in range(30):
        conv, q, a = random_trace(seed, 400, 20, q_max=6, a_max=4)
        for C in (0, 3, 17, 60, 10 ** 4):
            for xi in (0, 4, 12):
                r = O.replay(conv, q, a, O.BELADY_FORCED, C, xi)
                b = r.b.astype(np.int64)
                assert r.max_occupancy <= C and np.all(b >= q)
                seen = set()
                for t, c in enumerate(conv.tolist()):
                    if c not in seen:
                        assert b[t] == q[t]
                        seen.add(c)
                total_in = int(a.astype(np.int64).sum() + b.sum())
                assert r.evicted_trim + r.evicted_lru == total_in - min(C, total_in)
