"""Pins of the oracle's Threshold-LRU (the paper's baseline; SPEC S:279;
Reading #23: a history is cached only when L_after >= threshold, plain LRU among admitted
conversations).  No GPU."""
import json
import os

import numpy as np
import pytest

import oracle as O
from stackdist import topc_replay, topc_replay_threshold
from paper_2510_15152_b200.inputs import random_trace

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_hand_vector():
    """tests/golden/threshold_lru.json, derived by hand: the long conversation B keeps its
    cache because the short one A is never admitted; LRU evicts B for A."""
    g = json.load(open(os.path.join(GOLDEN, "threshold_lru.json")))
    r = O.replay(g["conv"], g["q"], g["a"], O.THRESHOLD, g["C"], threshold=g["threshold"])
    assert list(r.b) == g["threshold_b"]
    assert (r.evicted_trim, r.evicted_lru, r.max_occupancy) == (0, g["threshold_evicted_lru"],
                                                               g["threshold_max_occupancy"])
    lru = O.replay(g["conv"], g["q"], g["a"], O.LRU, g["C"])
    assert list(lru.b) == g["lru_b"] and lru.evicted_lru == g["lru_evicted_lru"]


@pytest.mark.parametrize("seed", range(6))
def test_threshold_zero_is_lru(seed):
    """T = 0 admits every history: identical to LRU for every request and counter."""
    conv, q, a = random_trace(seed, 400, 12)
    for C in (0, 3, 17, 60, 10**6):
        t = O.replay(conv, q, a, O.THRESHOLD, C, threshold=0)
        l = O.replay(conv, q, a, O.LRU, C)
        assert np.array_equal(t.b, l.b) and (t.evicted_trim, t.evicted_lru, t.max_occupancy) == \
            (l.evicted_trim, l.evicted_lru, l.max_occupancy)


@pytest.mark.parametrize("seed", range(4))
def test_threshold_above_every_history_caches_nothing(seed):
    """T > every L_after: nothing is ever cached, so b = J = L_before + q, no evictions."""
    conv, q, a = random_trace(seed, 300, 10)
    d = O.derive(conv, q, a)
    r = O.replay(conv, q, a, O.THRESHOLD, 5, threshold=10**9)
    assert np.array_equal(r.b, d.J.astype(np.uint64))
    assert (r.evicted_trim, r.evicted_lru, r.max_occupancy) == (0, 0, 0)


@pytest.mark.parametrize("seed", range(8))
def test_closed_form_with_admission(seed):
    """Independent algorithm (tests/stackdist.py): LRU with admission is the top-C of the
    admitted universe by recency, b = J - min(w_theta, (C - s_T)^+) with weights
    w = L [L >= T].  Pinned to the plain LRU closed form at T = 0."""
    conv, q, a = random_trace(100 + seed, 250, 9, q_max=6, a_max=6)
    for C in (0, 1, 7, 25, 80):
        assert topc_replay_threshold(conv, q, a, C, 0) == topc_replay(conv, q, a, C, 0)
        for T in (1, 4, 8, 15, 40):
            r = O.replay(conv, q, a, O.THRESHOLD, C, threshold=T)
            assert [int(x) for x in r.b] == topc_replay_threshold(conv, q, a, C, T), (C, T)


@pytest.mark.parametrize("seed", range(6))
def test_evictions_and_occupancy_identities(seed):
    """Blocks inserted = sum over admitted requests of (L_after - X_before) = a + b; the
    cache holds min(C, admitted universe) after every request (LRU fills to C and the
    admitted universe never shrinks), so evictions = sum_adm (a + b) - min(C, U_adm) and
    max occupancy = min(C, U_adm).  Threshold-LRU never trims (no free blocks)."""
    conv, q, a = random_trace(200 + seed, 300, 11)
    d = O.derive(conv, q, a)
    for C in (0, 4, 30, 100):
        for T in (0, 5, 12):
            r = O.replay(conv, q, a, O.THRESHOLD, C, threshold=T)
            adm = d.L_after >= T
            last = {}
            for e, c in enumerate(conv.tolist()):
                last[c] = int(d.L_after[e])
            U = sum(v for v in last.values() if v >= T)
            ins = int((a.astype(np.int64)[adm] + r.b.astype(np.int64)[adm]).sum())
            assert r.evicted_trim == 0
            assert r.evicted_lru == ins - min(C, U), (C, T)
            assert r.max_occupancy == min(C, U)
