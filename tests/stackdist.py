"""Independent closed-form replay used as a pin for the oracle (tests only).

Claim checked: LRU and T-LRU with the
oldest-first free-block order are priority stack algorithms whose cache content
after every request is the top-C blocks of the *universe* (every block of every
conversation's current history) under the static key
    (non-free?, tau of the conversation's last turn, -block position),
where the free blocks of conversation j are the last min(L_j, D) blocks of its
history, D = max(xi - Q_hat, 0) (P:56, P:62 footnote; D = 0 for LRU).  Hence,
for the request of conversation theta with previous turn at tau_theta:

    X_theta = min(NF_theta, (C - A_nf)^+) + min(F_theta, (C - NF_all - A_f)^+)

with NF_j = max(L_j - D, 0), F_j = min(L_j, D), A_nf / A_f the non-free / free
blocks of conversations whose last turn is after tau_theta, and NF_all the
non-free blocks of every conversation.  For D = 0 this is the Mattson /
weighted-reuse-distance closed form of LRU: b = J - clamp(C - s, 0, L_before).
No eviction loop is involved, so it is an algorithm independent of Alg. 1.
"""
from __future__ import annotations


def topc_replay(conv, q, a, C: int, D: int):
    L: dict[int, int] = {}
    tau: dict[int, int] = {}
    out = []
    for t, (c, qq, aa) in enumerate(zip(conv.tolist(), q.tolist(), a.tolist())):
        X = 0
        if c in L:
            Lc, tc = L[c], tau[c]
            nf_c, f_c = max(Lc - D, 0), min(Lc, D)
            a_nf = sum(max(L[j] - D, 0) for j in L if j != c and tau[j] > tc)
            a_f = sum(min(L[j], D) for j in L if j != c and tau[j] > tc)
            nf_all = sum(max(L[j] - D, 0) for j in L)
            X = min(nf_c, max(C - a_nf, 0)) + min(f_c, max(C - nf_all - a_f, 0))
        out.append(L.get(c, 0) + qq - X)
        L[c] = L.get(c, 0) + qq + aa
        tau[c] = t
    return out


def topc_replay_threshold(conv, q, a, C: int, T: int):
    """Threshold-LRU in the same closed form: LRU over the admitted blocks,
    i.e. conversation weights w_j = L_j if L_j >= T else 0 (Reading #23), so
    X_theta = min(w_theta, (C - sum of w_j over conversations used after theta's
    previous turn)^+).  T = 0 is the LRU closed form above."""
    L: dict[int, int] = {}
    tau: dict[int, int] = {}
    out = []
    w = lambda v: v if v >= T else 0  # noqa: E731
    for t, (c, qq, aa) in enumerate(zip(conv.tolist(), q.tolist(), a.tolist())):
        X = 0
        if c in L:
            s = sum(w(L[j]) for j in L if j != c and tau[j] > tau[c])
            X = min(w(L[c]), max(C - s, 0))
        out.append(L.get(c, 0) + qq - X)
        L[c] = L.get(c, 0) + qq + aa
        tau[c] = t
    return out
