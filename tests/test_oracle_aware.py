"""Pins of the oracle's End-Aware and Length-Aware T-LRU (
Readings #24-#25).  No GPU."""
import json
import os

import numpy as np
import pytest

import oracle as O
from stackdist import block_replay, topc_replay
from paper_2510_15152_b200.inputs import random_trace, tiny_trace

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def tel(b, xi):
    return int(sum(max(int(x) - xi, 0) for x in b))


def test_fig1_with_terminating_turns():
    g = json.load(open(os.path.join(GOLDEN, "aware_tlru.json")))["fig1_terminating"]
    for pol, key in ((O.END_AWARE, "end_aware_b"), (O.LENGTH_AWARE, "length_aware_b")):
        r = O.replay(g["conv"], g["q"], g["a"], pol, g["C"], g["xi"], g["q_hat"])
        assert list(r.b) == g[key]
        assert [r.evicted_trim, r.evicted_lru] == g["evicted"] and r.max_occupancy == g["max_occupancy"]


def test_length_aware_uses_true_next_prompt():
    """SPEC S:259 arithmetic (budget with the true next prompt) in a trace: the hand vector
    where Length-Aware trims the conversation whose next prompt is short instead of evicting
    another one by LRU."""
    g = json.load(open(os.path.join(GOLDEN, "aware_tlru.json")))["length_vs_end"]
    e = O.replay(g["conv"], g["q"], g["a"], O.END_AWARE, g["C"], g["xi"], g["q_hat"])
    l = O.replay(g["conv"], g["q"], g["a"], O.LENGTH_AWARE, g["C"], g["xi"], g["q_hat"])
    assert list(e.b) == g["end_aware_b"] and [e.evicted_trim, e.evicted_lru] == g["end_aware_evicted"]
    assert list(l.b) == g["length_aware_b"] and [l.evicted_trim, l.evicted_lru] == g["length_aware_evicted"]
    assert tel(e.b, g["xi"]) == g["tel_at_xi"]["end_aware"] and tel(l.b, g["xi"]) == g["tel_at_xi"]["length_aware"]


def test_block_brute_force_is_pinned():
    """The brute force itself reproduces the T-LRU / LRU closed form (tests/stackdist.py)."""
    for seed in range(4):
        conv, q, a = random_trace(700 + seed, 120, 8, q_max=4, a_max=4)
        for C in (0, 3, 11, 40):
            for D in (0, 2, 5):
                assert block_replay(conv, q, a, C, D + 2, 2) == topc_replay(conv, q, a, C, D)


@pytest.mark.parametrize("seed", range(8))
def test_block_brute_force(seed):
    """Oracle == the block-priority brute force (tests/stackdist.py block_replay)."""
    conv, q, a = random_trace(400 + seed, 140, 9, q_max=4, a_max=4, locality=0.6)
    for C in (0, 2, 9, 30, 60):
        for xi, qh in ((0, 0), (4, 2), (9, 2), (14, 3)):
            e = O.replay(conv, q, a, O.END_AWARE, C, xi, qh)
            assert [int(x) for x in e.b] == block_replay(conv, q, a, C, xi, qh, "end"), (C, xi, qh)
            l = O.replay(conv, q, a, O.LENGTH_AWARE, C, xi, qh)
            assert [int(x) for x in l.b] == block_replay(conv, q, a, C, xi, qh, "length"), (C, xi, qh)


@pytest.mark.parametrize("seed", range(150))
def test_block_brute_force_tiny(seed):
    conv, q, a = tiny_trace(seed)
    for C in range(0, 9):
        for xi in range(0, 6):
            assert [int(x) for x in O.replay(conv, q, a, O.END_AWARE, C, xi, 1).b] == \
                block_replay(conv, q, a, C, xi, 1, "end")
            assert [int(x) for x in O.replay(conv, q, a, O.LENGTH_AWARE, C, xi, 1).b] == \
                block_replay(conv, q, a, C, xi, 1, "length")


@pytest.mark.parametrize("seed", range(5))
def test_special_cases(seed):
    """q identically Q_hat: Length-Aware's budget equals End-Aware's.  xi <= Q_hat: End-Aware
    has no free blocks (LRU with release), so it never trims.  C >= total history: every
    returning request finds its whole history cached (b = q) and nothing is evicted."""
    conv, q, a = random_trace(500 + seed, 300, 14)
    qc = np.full_like(q, 3)
    for C in (0, 5, 40, 200):
        for xi in (2, 6, 11):
            e = O.replay(conv, qc, a, O.END_AWARE, C, xi, 3)
            l = O.replay(conv, qc, a, O.LENGTH_AWARE, C, xi, 3)
            assert np.array_equal(e.b, l.b) and (e.evicted_trim, e.evicted_lru) == (l.evicted_trim, l.evicted_lru)
        d0 = O.replay(conv, q, a, O.END_AWARE, C, 2, 2)
        assert d0.evicted_trim == 0
    d = O.derive(conv, q, a)
    big = O.replay(conv, q, a, O.END_AWARE, 10**9, 7, 2)
    first = d.prev == O.NONE
    assert np.array_equal(big.b[~first], q[~first].astype(np.uint64))  # every return hits its whole history
    assert big.evicted_trim == 0 and big.evicted_lru == 0


@pytest.mark.parametrize("seed", range(5))
def test_release_never_increases_others_misses(seed):
    """End-Aware vs T-LRU with the same D: releasing blocks of conversations that never return
    only frees space, so on every request b(End-Aware) <= b(T-LRU) (pathwise)."""
    conv, q, a = random_trace(600 + seed, 400, 16)
    for C in (3, 20, 70):
        for xi, qh in ((2, 2), (8, 2)):
            e = O.replay(conv, q, a, O.END_AWARE, C, xi, qh)
            t = O.replay(conv, q, a, O.TLRU, C, xi, qh)
            assert np.all(e.b <= t.b), (C, xi)
