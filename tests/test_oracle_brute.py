"""Oracle policy checked against exact brute force (Thm 1, Thm 2; no GPU)."""
import random
from fractions import Fraction

import numpy as np

import oracle as O
from oracle.brute import belief_mdp_value, hindsight_opt, tlru_step
from paper_2510_15152_b200.inputs import tiny_trace


def _instances(n, seed):
    rnd = random.Random(seed)
    for _ in range(n):
        yield dict(C=rnd.randint(1, 6), xi=rnd.randint(0, 5), Q=rnd.choice([1, 2]),
                   A_set=rnd.choice([(0,), (0, 1), (1, 2), (0, 2), (0, 1, 2)]),
                   rho=rnd.choice([Fraction(1, 2), Fraction(1, 3), Fraction(2, 3)]),
                   w_new=rnd.choice([Fraction(1, 2), Fraction(1), Fraction(2)]),
                   n_max=rnd.choice([2, 3]), M=rnd.choice([4, 5]))


def test_thm2_tlru_attains_optimal_expected_tel():
    """Thm 2 corollary: with deterministic Q and homogeneous rates T-LRU
    (Alg. 1, Q_hat = Q) minimizes expected TEL in the belief MDP (App. B).
    Also checks the test has power: LRU and the weak-budget reading miss the optimum."""
    n = lru_opt = weak_opt = 0
    for inst in _instances(240, 11):  # >= 200 instances (BASELINE config 2, SURVEY c.5)
        vo = belief_mdp_value(**inst)
        vt = belief_mdp_value(**inst, policy="tlru")
        assert vt == vo, inst
        lru_opt += belief_mdp_value(**inst, policy="lru") == vo
        weak_opt += belief_mdp_value(**inst, policy="tlru", budget="weak") == vo
        n += 1
    assert n >= 200
    assert lru_opt < n - 40 and weak_opt < n - 40


def test_thm2_corollary_lru_optimal_at_xi0():
    """xi = 0 with homogeneous rates -> LRU optimal for average latency."""
    for inst in _instances(60, 12):
        inst["xi"] = 0
        assert belief_mdp_value(**inst, policy="lru") == belief_mdp_value(**inst)


def test_python_alg1_matches_oracle_on_tiny_traces():
    """brute.tlru_step (Python Alg. 1) and the C oracle agree request by request."""
    for seed in range(150):
        conv, q, a = tiny_trace(seed)
        for C in range(0, 9, 2):
            for xi, qh in ((0, 0), (3, 1), (5, 2)):
                r = O.replay(conv, q, a, O.TLRU, C, xi, qh)
                ids = sorted(set(conv.tolist()))
                X = {c: 0 for c in ids}
                L = {c: 0 for c in ids}
                tau = {c: -1 for c in ids}
                for t, (c, qq, aa) in enumerate(zip(conv.tolist(), q.tolist(), a.tolist())):
                    assert L[c] + qq - X[c] == int(r.b[t])
                    L[c] += qq + aa
                    X[c] = L[c]
                    tau[c] = t
                    newX = tlru_step([X[i] for i in ids], [L[i] for i in ids],
                                     [t - tau[i] for i in ids], None, C, xi, qh, "tlru")
                    X = dict(zip(ids, newX))


def test_thm1_hindsight_opt_lower_bounds_online_policies():
    """Thm 1 / Eq. 5: the hindsight optimum lower-bounds LRU and T-LRU;
    with C large enough every policy reaches sum (q - xi)^+ ... and OPT equals it."""
    rnd = random.Random(5)
    strict = 0
    for seed in range(220):
        conv, q, a = tiny_trace(seed, max_conv=3, max_turns=2, qs=(1, 2), as_=(0, 1))
        C = rnd.randint(0, 5)
        xi = rnd.randint(0, 3)
        opt = hindsight_opt(conv, q, a, C, xi)
        t = O.replay(conv, q, a, O.TLRU, C, xi, 1)
        l = O.replay(conv, q, a, O.LRU, C)
        tel_t = int(np.maximum(t.b.astype(np.int64) - xi, 0).sum())
        tel_l = int(np.maximum(l.b.astype(np.int64) - xi, 0).sum())
        assert opt <= tel_t and opt <= tel_l
        strict += opt < min(tel_t, tel_l)
        big = hindsight_opt(conv, q, a, 10 ** 3, xi)
        assert big == int(np.maximum(q.astype(np.int64) - xi, 0).sum())
    assert strict > 0
