"""Pins of the oracle's T-LRU under forced caching (App. C; Reading #28): the
post-decision state must hold theta's whole history (constraint (3) with equality),
capped by the capacity.  No GPU."""
import random
from fractions import Fraction as F

import numpy as np
import pytest

import oracle as O
from oracle.brute import belief_mdp_value, hindsight_opt, tlru_step
from paper_2510_15152_b200.inputs import random_trace, tiny_trace

FORCED = 7


def tel(b, xi):
    return int(np.maximum(np.asarray(b, dtype=np.int64) - xi, 0).sum())


def test_fig1_forced():
    """Fig. 1 under forced caching: B's history must stay whole, so A loses all 100 blocks
    (50 free, then 50 by LRU) and A2 pays 200 -- hedging needs optional caching.  A2's own 200
    blocks then exceed C = 100: B goes (50 free + 50), then A's tail 100 (capacity first)."""
    r = O.replay([0, 1, 0], [100, 100, 100], [0, 0, 0], FORCED, 100, 150, 100)
    assert [int(x) for x in r.b] == [100, 100, 200]
    assert (r.evicted_trim, r.evicted_lru, r.max_occupancy) == (100, 200, 100)
    # the hindsight optimum under forced caching is the same 50 blocks of TEL
    assert hindsight_opt(np.array([0, 1, 0]), np.array([100, 100, 100]), np.array([0, 0, 0]), 100, 150,
                         forced=True) == tel(r.b, 150) == 50


def test_thm3_forced_tlru_optimal_in_belief_mdp():
    """App. C: with deterministic prompt lengths and homogeneous turn rates,
    (E)T-LRU stays optimal under forced caching -- expected TEL of forced T-LRU equals the
    minimum over every forced decision in the belief MDP.  Power: forced LRU misses it."""
    rnd = random.Random(41)
    n = lru_opt = 0
    for _ in range(150):
        inst = dict(C=rnd.randint(1, 6), xi=rnd.randint(0, 5), Q=rnd.choice([1, 2]),
                    A_set=rnd.choice([(0,), (0, 1), (1, 2)]), rho=rnd.choice([F(1, 2), F(1, 3), F(2, 3)]),
                    w_new=rnd.choice([F(1, 2), F(1), F(2)]), n_max=rnd.choice([2, 3]), M=rnd.choice([4, 5]))
        vo = belief_mdp_value(**inst, forced=True)
        assert belief_mdp_value(**inst, policy="tlru", forced=True) == vo, inst
        lru_opt += belief_mdp_value(**inst, policy="lru", forced=True) == vo
        n += 1
    assert lru_opt < n - 10


def test_c_oracle_equals_python_alg1_forced():
    """brute.tlru_step(forced=True) and the C oracle agree request by request."""
    for seed in range(200):
        conv, q, a = tiny_trace(seed)
        for C in (0, 1, 3, 6, 9):
            for xi, qh in ((0, 0), (3, 1), (5, 2)):
                r = O.replay(conv, q, a, FORCED, C, xi, qh)
                ids = sorted(set(conv.tolist()))
                X = {c: 0 for c in ids}
                L = {c: 0 for c in ids}
                tau = {c: -1 for c in ids}
                for t, (c, qq, aa) in enumerate(zip(conv.tolist(), q.tolist(), a.tolist())):
                    assert L[c] + qq - X[c] == int(r.b[t]), (seed, C, xi, t)
                    L[c] += qq + aa
                    X[c] = L[c]
                    tau[c] = t
                    newX = tlru_step([X[i] for i in ids], [L[i] for i in ids], [t - tau[i] for i in ids],
                                     ids.index(c), C, xi, qh, "tlru", forced=True)
                    X = dict(zip(ids, newX))


def test_thm1_forced_lower_bound():
    """Thm 1 holds under forced caching -- the forced hindsight optimum lower-bounds the
    forced online policy, and optional caching can only do better (a larger feasible set)."""
    rnd = random.Random(9)
    for seed in range(150):
        conv, q, a = tiny_trace(500 + seed, max_conv=3, max_turns=3)
        if conv.size > 7:
            conv, q, a = conv[:7], q[:7], a[:7]
        C, xi = rnd.randint(0, 6), rnd.randint(0, 4)
        opt_f = hindsight_opt(conv, q, a, C, xi, forced=True)
        assert opt_f <= tel(O.replay(conv, q, a, FORCED, C, xi, 1).b, xi)
        assert hindsight_opt(conv, q, a, C, xi) <= opt_f


@pytest.mark.parametrize("seed", range(4))
def test_forced_special_cases(seed):
    """xi <= Q_hat (no free blocks): LRU already evicts theta last and only when it alone
    exceeds C, so forced == optional == LRU.  b >= q, occupancy <= C, and with nothing
    released the eviction identity Sum(a + b) - min(C, Sum(a + b)) holds."""
    conv, q, a = random_trace(5000 + seed, 700, 30, q_max=6, a_max=6)
    for C in (0, 5, 30, 120):
        f = O.replay(conv, q, a, FORCED, C, 2, 2)
        l = O.replay(conv, q, a, O.LRU, C)
        assert np.array_equal(f.b, l.b) and (f.evicted_trim, f.evicted_lru) == (l.evicted_trim, l.evicted_lru)
        for xi in (5, 12):
            r = O.replay(conv, q, a, FORCED, C, xi, 2)
            ins = int(a.astype(np.int64).sum() + r.b.astype(np.int64).sum())
            assert np.all(r.b >= q) and r.max_occupancy == min(C, ins)
            assert r.evicted_trim + r.evicted_lru == ins - min(C, ins)
