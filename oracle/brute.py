"""Exact brute-force oracles on tiny instances — TEST INFRASTRUCTURE ONLY.

Two independent checks of the policy the hot path simulates, both in exact
rational arithmetic (``fractions.Fraction``):

* ``hindsight_opt``: the hindsight-optimal TEL of a known trace, Eq. (5)
  (Sec. 3), by dynamic programming over cache vectors subject to
  constraints (2)-(4).  Theorem 1 makes it a lower
  bound for every online policy.
* ``belief_mdp_value``: the expected TEL of a policy in the paper's belief MDP
  (finite-horizon Bellman recursion of App. B) with
  homogeneous turn rates, deterministic prompt length Q and responses A drawn
  uniformly from a small set.  Conversation j (last turn `age` arrivals ago)
  is the next arrival with weight rho**age (belief pi_j = exp(-mu * elapsed),
  P:255, with unit spacing rho = e^-mu) and a new conversation with weight
  w_new while fewer than n_max exist.  ``policy=None`` minimizes over every
  feasible caching decision (sum Y <= C, Y_theta <= L_theta, Y_i <= X_i).
  Theorem 2's corollary says T-LRU (Alg. 1 with Q_hat = Q) attains the
  minimum; its first corollary says LRU does when xi = 0.

* ``etlru_step`` / ``etlru_objective_min``: Expected-Tail-Optimized LRU (Def. 1)
  in exact rationals -- the greedy of Alg. 2 and, independently, the exhaustive
  minimum of Def. 1's objective (8) over every feasible allocation (the Lemma).
  ``belief_mdp_value(..., q_pmf=...)`` draws the next prompt from a pmf (Thm 3).

``tlru_step`` is a plain Python transcription of Alg. 1 used only
inside these recursions (and by the convention-vector tests); it shares no
code with the C oracle or the CUDA path.
"""
from __future__ import annotations

from fractions import Fraction
from functools import lru_cache
from itertools import product


def tlru_step(X, L, ages, theta, C, xi, q_hat, policy, budget="strict", forced=False):
    """One Alg. 1 decision after serving `theta` (whose X/L are already updated
    per P:206: X_theta = L_theta).  X, L, ages: lists (ages: larger = older).
    policy 'lru' skips Phase 1.  budget 'strict' trims to (L + Q_hat - xi)^+
    (Reading #2); 'weak' is the literal `X_i >= L_i + Q_hat - xi` test that
    trims one block below the budget.  forced (App. C): theta (an index) keeps its
    whole history unless it alone exceeds C.  Returns the new X (list)."""
    X = list(X)
    over = sum(X) - C
    order = sorted(range(len(X)), key=lambda i: -ages[i])  # ascending tau = oldest first
    if over > 0 and policy == "tlru":
        for i in order:  # Phase 1, bulk, oldest first, theta last (Readings #1, #3, #5)
            if forced and i == theta:
                continue
            budget_i = max(L[i] + q_hat - xi, 0)
            if budget == "weak":
                budget_i = max(budget_i - 1, 0) if X[i] >= L[i] + q_hat - xi else X[i]
            k = min(max(X[i] - budget_i, 0), over)
            X[i] -= k
            over -= k
            if over == 0:
                break
    if over > 0:
        for i in order:  # Phase 2
            if forced and i == theta:
                continue
            k = min(X[i], over)
            X[i] -= k
            over -= k
            if over == 0:
                break
    if over > 0 and forced:  # theta alone exceeds C
        X[theta] -= over
    return X


# ----------------------------------------------------------------------------- Def. 1 / Alg. 2
def surv(q_pmf, k):
    """P(Q >= k) for a pmf {q: p} (exact)."""
    return sum((p for qq, p in q_pmf.items() if qq >= k), Fraction(0))


def etlru_step(X, L, lam, C, xi, q_pmf, tau=None):
    """Alg. 2: evict sum(X) - C blocks one at a time from argmin of
    v_i = lam_i * P(L_i + Q_i - xi >= X_i) (X_i >= 1), re-scoring after each block.
    Ties -> smaller tau (older last turn) first.  X, L, lam (Fractions), tau: lists."""
    X = list(X)
    tau = tau if tau is not None else list(range(len(X)))
    while sum(X) > C:
        best = None
        for i in range(len(X)):
            if X[i] < 1:
                continue
            v = lam[i] * surv(q_pmf, X[i] - L[i] + xi)
            if best is None or v < best[0] or (v == best[0] and tau[i] < tau[best[1]]):
                best = (v, i)
        X[best[1]] -= 1
    return X


def etlru_objective(Y, L, lam, xi, q_pmf):
    """Def. 1 objective (8): sum_i lam_i E[(L_i + Q_i - Y_i - xi)^+]."""
    return sum(lam[i] * sum(p * max(L[i] + qq - Y[i] - xi, 0) for qq, p in q_pmf.items())
               for i in range(len(Y)))


def etlru_objective_min(X, L, lam, C, xi, q_pmf):
    """min of (8) over Y with Y_i <= X_i (X_theta = L_theta already) and sum Y <= C."""
    best = None
    for Y in product(*[range(u + 1) for u in X]):
        if sum(Y) > C:
            continue
        v = etlru_objective(Y, L, lam, xi, q_pmf)
        if best is None or v < best:
            best = v
    return best


# ----------------------------------------------------------------------------- Thm 1 / Eq. 5
def hindsight_opt(conv, q, a, C: int, xi: int, forced: bool = False) -> int:
    """min sum_t (J_t - x_{theta,t} - xi)^+ over cache schedules obeying (2)-(4); forced: (3) with
    equality (App. C), capped by the capacity (Reading #28)."""
    ids = sorted(set(int(c) for c in conv))
    idx = {c: i for i, c in enumerate(ids)}
    n = len(ids)
    ev = [(idx[int(c)], int(qq), int(aa)) for c, qq, aa in zip(conv, q, a)]
    T = len(ev)

    @lru_cache(maxsize=None)
    def V(t, X, L):
        if t == T:
            return 0
        th, qq, aa = ev[t]
        cost = max(L[th] + qq - X[th] - xi, 0)
        L2 = list(L)
        L2[th] += qq + aa
        ub = [X[i] if i != th else L2[th] for i in range(n)]  # constraints (3), (4)
        target = min(C, sum(ub))                            # maximal schedules dominate
        best = None
        for Y in product(*[range(u + 1) for u in ub]):
            if sum(Y) != target:
                continue
            if forced and Y[th] != min(L2[th], C):
                continue
            v = V(t + 1, tuple(Y), tuple(L2))
            if best is None or v < best:
                best = v
        return cost + best

    return V(0, tuple([0] * n), tuple([0] * n))


# ----------------------------------------------------------------------------- Thm 2 belief MDP
def belief_mdp_value(C, xi, Q, A_set, rho, w_new, n_max, M, policy=None, budget="strict", q_pmf=None,
                     forced=False):
    """Expected TEL (in blocks) over M arrivals from an empty system.

    policy: None (optimal), 'tlru' (Alg. 1 with Q_hat = Q), 'lru' or 'etlru' (Alg. 2 with the
    belief lam_j = rho**age_j).  q_pmf: {q: p} prompt law (default: deterministic Q)."""
    q_pmf = {Q: Fraction(1)} if q_pmf is None else {int(k): Fraction(v) for k, v in q_pmf.items()}
    rho = Fraction(rho)
    w_new = Fraction(w_new)
    A_set = tuple(A_set)
    pA = Fraction(1, len(A_set))

    def canon(state):
        return tuple(sorted(state))

    @lru_cache(maxsize=None)
    def V(k, state):
        # state: tuple of (L, X, age) per existing conversation
        if k == M:
            return Fraction(0)
        convs = list(state)
        weights = [rho ** age for (_, _, age) in convs]
        if len(convs) < n_max:
            weights.append(w_new)
        total = sum(weights)
        ev = Fraction(0)
        for j, w in enumerate(weights):
            p = w / total
            if j < len(convs):
                L, X, _ = convs[j]
                rest = convs[:j] + convs[j + 1:]
            else:
                L, X = 0, 0
                rest = convs
            for Qd, pQ in q_pmf.items():
                cost = max(L + Qd - X - xi, 0)  # (L_theta + Q - X_theta - xi)^+, App. B
                for A in A_set:
                    L_new = L + Qd + A
                    others = [(Lr, Xr, ager + 1) for (Lr, Xr, ager) in rest]  # Phi: discount all others
                    # decision over theta (first, age 0) and the others
                    Ls = [L_new] + [o[0] for o in others]
                    Xs = [L_new] + [o[1] for o in others]   # X_theta <- L_theta
                    ages = [0] + [o[2] for o in others]
                    if policy is None:
                        ub = Xs
                        target = min(C, sum(ub))
                        best = None
                        for Y in product(*[range(u + 1) for u in ub]):
                            if sum(Y) != target:
                                continue
                            if forced and Y[0] != min(L_new, C):  # App. C: theta kept whole
                                continue
                            nxt = canon(tuple((Ls[i], Y[i], ages[i]) for i in range(len(Y))))
                            v = V(k + 1, nxt)
                            if best is None or v < best:
                                best = v
                        cont = best
                    else:
                        if policy == "etlru":  # belief lam = rho**age, older = larger age
                            Y = etlru_step(Xs, Ls, [rho ** g for g in ages], C, xi, q_pmf, [-g for g in ages])
                        else:
                            Y = tlru_step(Xs, Ls, ages, 0, C, xi, Q, policy, budget, forced)
                        nxt = canon(tuple((Ls[i], Y[i], ages[i]) for i in range(len(Y))))
                        cont = V(k + 1, nxt)
                    ev += p * pQ * pA * (cost + cont)
        return ev

    return V(0, tuple())
