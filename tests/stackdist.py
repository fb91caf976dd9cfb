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



def block_replay(conv, q, a, C: int, xi: int, q_hat: int, kind: str = "tlru"):
    """Definitional brute force of Alg. 1 and its End-/Length-Aware variants (P:206-218,
    P:389-395; Readings #1-#5, #24, #25), written as a priority cache of individual blocks:
    every cached block has the key (class, tau of its conversation, -position) with class 0
    for free blocks (the last min(L, D) of a history, "infinitely old") and 1 for the
    rest; an overflow evicts the minimum-key block, one block at a time, until the cache
    fits.  Within a conversation the cached blocks are then always a prefix of its history,
    so a count X per conversation represents them.  No surplus bookkeeping or eviction lists
    are shared with the oracle.  kind: "tlru", "end" (a terminating turn releases theta's
    blocks) or "length" ("end" + D from the true next prompt)."""
    conv, q, a = list(map(int, conv)), list(map(int, q)), list(map(int, a))
    E = len(conv)
    nxt, seen = [None] * E, {}
    for t in range(E - 1, -1, -1):
        nxt[t] = seen.get(conv[t])
        seen[conv[t]] = t
    X, L, F, tau = {}, {}, {}, {}
    out = []
    for e in range(E):
        c = conv[e]
        Lb = L.get(c, 0)
        out.append(Lb + q[e] - X.get(c, 0))
        La = Lb + q[e] + a[e]
        L[c] = La
        if kind in ("end", "length") and nxt[e] is None:
            X[c] = 0  # released
            continue
        qn = q[nxt[e]] if (kind == "length" and nxt[e] is not None) else q_hat
        X[c], F[c], tau[c] = La, min(La, max(xi - qn, 0)), e
        while sum(X.values()) > C:
            def key(j):
                free_cached = X[j] - (L[j] - F[j])
                return (0 if free_cached > 0 else 1, tau[j])
            j = min((j for j in X if X[j] > 0), key=key)
            X[j] -= 1
    return out
