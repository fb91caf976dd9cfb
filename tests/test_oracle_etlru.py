"""Pins of the oracle's Expected-Tail-Optimized LRU (Def. 1; Alg. 2, P:603-650;
Thm 3; Reading #27).  No GPU.

Chain of pins: the exact-rational greedy (oracle/brute.py etlru_step) solves Def. 1's program
(the Lemma, by exhaustive minimisation) and attains the optimal expected TEL of the
belief MDP with random prompts (Thm 3, finite-horizon Bellman DP); the C oracle equals that
greedy on traces; and the paper's two reductions hold exactly: deterministic Q -> T-LRU
(P:286), xi = 0 -> LRU."""
import math
import random
from fractions import Fraction as F

import numpy as np
import pytest

import oracle as O
from oracle.brute import belief_mdp_value, etlru_objective, etlru_objective_min, etlru_step, surv
from paper_2510_15152_b200.inputs import random_trace, tiny_trace

PMFS = [{1: F(7, 10), 2: F(3, 10)}, {1: F(9, 20), 3: F(11, 20)}, {1: F(1, 5), 2: F(1, 2), 4: F(3, 10)},
        {2: F(13, 20), 3: F(7, 20)}]


def ln_table(pmf, K=12):
    return [math.log(float(surv(pmf, k))) if surv(pmf, k) > 0 else -math.inf for k in range(K + 1)]


def point_mass_table(q_hat, K=None):
    K = K if K is not None else q_hat + 2
    return [0.0 if k <= q_hat else -math.inf for k in range(K + 1)]


def times_for(n, rng, ties=True):
    gaps = rng.integers(0 if ties else 1, 4, size=n)
    return np.cumsum(gaps).astype(np.uint64)


def test_lemma_alg2_solves_def1():
    """P:648 Lemma: the greedy returns a minimiser of objective (8)."""
    rnd = random.Random(21)
    for _ in range(300):
        n = rnd.randint(1, 3)
        L = [rnd.randint(0, 5) for _ in range(n)]
        X = [rnd.randint(0, l) for l in L]
        X[0] = L[0]  # theta just served: X_theta <- L_theta
        lam = [F(1)] + [F(1, 2) ** rnd.randint(1, 4) for _ in range(n - 1)]
        C, xi, pmf = rnd.randint(0, 8), rnd.randint(0, 4), rnd.choice(PMFS)
        Y = etlru_step(X, L, lam, C, xi, pmf)
        assert sum(Y) <= C and all(0 <= y <= x for y, x in zip(Y, X))
        assert etlru_objective(Y, L, lam, xi, pmf) == etlru_objective_min(X, L, lam, min(C, sum(X)), xi, pmf)


def test_thm3_etlru_attains_optimal_expected_tel():
    """Thm 3: ET-LRU minimises expected TEL in the belief MDP, here with random prompt
    lengths (no deterministic-Q reduction available).  Power: LRU misses the optimum."""
    rnd = random.Random(31)
    n = lru_opt = 0
    for _ in range(60):
        inst = dict(C=rnd.randint(1, 5), xi=rnd.randint(0, 4), Q=1, A_set=rnd.choice([(0,), (0, 1), (1,)]),
                    rho=rnd.choice([F(1, 2), F(1, 3), F(2, 3)]), w_new=rnd.choice([F(1, 2), F(1), F(2)]),
                    n_max=rnd.choice([2, 3]), M=rnd.choice([3, 4]))
        pmf = rnd.choice(PMFS)
        vo = belief_mdp_value(**inst, q_pmf=pmf)
        assert belief_mdp_value(**inst, q_pmf=pmf, policy="etlru") == vo, (inst, pmf)
        lru_opt += belief_mdp_value(**inst, q_pmf=pmf, policy="lru") == vo
        n += 1
    assert lru_opt < n - 5


def _python_etlru(conv, q, a, ticks, C, xi, pmf):
    """Exact-rational replay: belief lam_i = (1/2)^(t - ticks_i) (mu = ln 2 per tick)."""
    ids = sorted(set(conv.tolist()))
    X = {c: 0 for c in ids}
    L = {c: 0 for c in ids}
    tl = {c: 0 for c in ids}
    tau = {c: -1 for c in ids}
    out = []
    for t, (c, qq, aa) in enumerate(zip(conv.tolist(), q.tolist(), a.tolist())):
        out.append(L[c] + qq - X[c])
        L[c] += qq + aa
        X[c] = L[c]
        tl[c] = int(ticks[t])
        tau[c] = t
        now = int(ticks[t])
        lam = [F(1, 2) ** (now - tl[i]) for i in ids]
        Y = etlru_step([X[i] for i in ids], [L[i] for i in ids], lam, C, xi, pmf, [tau[i] for i in ids])
        X = dict(zip(ids, Y))
    return out


@pytest.mark.parametrize("seed", range(6))
def test_c_oracle_equals_exact_alg2(seed):
    rng = np.random.default_rng(seed)
    for k in range(25):
        conv, q, a = tiny_trace(100 * seed + k, max_conv=4, max_turns=4, qs=(1, 2, 3), as_=(0, 1, 2))
        ticks = times_for(conv.size, rng)
        pmf = PMFS[k % len(PMFS)]
        for C in (0, 2, 5, 9):
            for xi in (0, 2, 4):
                r = O.replay_etlru(conv, q, a, ticks, C, xi, math.log(2.0), ln_table(pmf))
                assert [int(x) for x in r.b] == _python_etlru(conv, q, a, ticks, C, xi, pmf), (k, C, xi)


@pytest.mark.parametrize("seed", range(6))
def test_deterministic_q_reduces_to_tlru(seed):
    """with a deterministic prompt length (point-mass law at Q_hat) ET-LRU is T-LRU
    (Alg. 1 with Q_hat): identical b, Phase-1 (P = 0 blocks) and Phase-2 eviction counts."""
    conv, q, a = random_trace(3000 + seed, 900, 35, q_max=5, a_max=5, locality=0.6)
    ticks = times_for(conv.size, np.random.default_rng(seed))
    for C in (0, 3, 16, 60, 250):
        for xi, qh in ((0, 0), (3, 1), (6, 2), (15, 3), (30, 2)):
            for mu in (1e-6, 0.3, 7.0):
                e = O.replay_etlru(conv, q, a, ticks, C, xi, mu, point_mass_table(qh))
                t = O.replay(conv, q, a, O.TLRU, C, xi, qh)
                assert np.array_equal(e.b, t.b), (C, xi, qh, mu)
                assert (e.evicted_trim, e.evicted_lru, e.max_occupancy) == (t.evicted_trim, t.evicted_lru,
                                                                            t.max_occupancy)


@pytest.mark.parametrize("seed", range(4))
def test_xi0_reduces_to_lru(seed):
    """xi = 0 with homogeneous rates -> LRU, whatever the prompt law."""
    conv, q, a = random_trace(3100 + seed, 900, 35, q_max=5, a_max=5, locality=0.6)
    ticks = times_for(conv.size, np.random.default_rng(10 + seed))
    for C in (0, 4, 20, 90):
        for pmf in PMFS:
            e = O.replay_etlru(conv, q, a, ticks, C, 0, 0.05, ln_table(pmf))
            l = O.replay(conv, q, a, O.LRU, C)
            assert np.array_equal(e.b, l.b) and e.evicted_lru == l.evicted_lru and e.evicted_trim == 0


def test_fig1_point_mass():
    """Fig. 1 with the deterministic law Q = 100: ET-LRU = T-LRU = [100, 100, 150]."""
    r = O.replay_etlru([0, 1, 0], [100, 100, 100], [0, 0, 0], [0, 5, 9], 100, 150, 0.01, point_mass_table(100))
    assert [int(x) for x in r.b] == [100, 100, 150] and (r.evicted_trim, r.evicted_lru) == (150, 100)


@pytest.mark.parametrize("seed", range(3))
def test_invariants(seed):
    """b >= q; occupancy <= C; no release, so the cache fills to min(C, inserted) and stays:
    evicted = Sum(a + b) - min(C, Sum(a + b)); C = 0 -> b = J; huge C -> b = q."""
    conv, q, a = random_trace(3200 + seed, 500, 25)
    ticks = times_for(conv.size, np.random.default_rng(seed))
    d = O.derive(conv, q, a)
    tab = ln_table(PMFS[seed])
    assert np.array_equal(O.replay_etlru(conv, q, a, ticks, 0, 3, 0.1, tab).b, d.J.astype(np.uint64))
    big = int((q.astype(np.int64) + a).sum())
    assert np.array_equal(O.replay_etlru(conv, q, a, ticks, big, 3, 0.1, tab).b, q.astype(np.uint64))
    for C in (5, 40, 150):
        r = O.replay_etlru(conv, q, a, ticks, C, 4, 0.1, tab)
        ins = int(a.astype(np.int64).sum() + r.b.astype(np.int64).sum())
        assert np.all(r.b >= q) and r.max_occupancy == min(C, ins)
        assert r.evicted_trim + r.evicted_lru == ins - min(C, ins)
