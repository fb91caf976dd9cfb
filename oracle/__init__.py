"""CPU oracle for the T-LRU hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2510_15152_b200`` never imports it and shares no code with it.

This module is a thin ctypes wrapper over ``oracle/tlru_oracle.c`` (plain,
single-threaded C; see that file's header for the paper passages each function
follows) plus the exact-rational brute-force oracles in ``oracle/brute.py``.

Parity pins (tests/test_oracle_*.py): Fig. 1 worked example,
closed-form/stack replay (independent algorithm), invariants, Thm-2 DP and
Thm-1 hindsight brute force, numpy Philox and libm for the sampler.
Functions without an independent pin say "parity unpinned" here and in
DESIGN.md: only the free-block order convention (Reading #3) for raw b.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tlru_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

NONE = 0xFFFFFFFF


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, plain -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
             "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        u64p = ctypes.POINTER(ctypes.c_uint64)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        L.oracle_philox4x64.argtypes = [u64p, u64p, u64p]
        L.oracle_philox4x64.restype = None
        L.oracle_u01.argtypes = [ctypes.c_uint64]
        L.oracle_u01.restype = ctypes.c_double
        L.oracle_det_ln.argtypes = [ctypes.c_double]
        L.oracle_det_ln.restype = ctypes.c_double
        L.oracle_det_exp.argtypes = [ctypes.c_double]
        L.oracle_det_exp.restype = ctypes.c_double
        L.oracle_generate.argtypes = [ctypes.c_void_p, ctypes.POINTER(u64p)] + [ctypes.POINTER(u32p)] * 4
        L.oracle_generate.restype = ctypes.c_int64
        L.oracle_free.argtypes = [ctypes.c_void_p]
        L.oracle_free.restype = None
        L.oracle_derive.argtypes = [u32p, u32p, u32p, ctypes.c_uint64, u32p, u64p, u64p, u32p]
        L.oracle_derive.restype = ctypes.c_int
        L.oracle_replay.argtypes = [u32p, u32p, u32p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64,
                                    ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, u64p, u64p]
        L.oracle_replay.restype = ctypes.c_int
        L.oracle_replay_etlru.argtypes = [u32p, u32p, u32p, u64p, ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.c_uint64, ctypes.c_double, ctypes.POINTER(ctypes.c_double),
                                          ctypes.c_uint64, ctypes.c_int, u64p, u64p]
        L.oracle_replay_etlru.restype = ctypes.c_int
        L.oracle_tail.argtypes = [u64p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double, ctypes.c_uint64,
                                  ctypes.c_double, u64p, ctypes.POINTER(ctypes.c_double)]
        L.oracle_tail.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(arr, ct):
    return arr.ctypes.data_as(ctypes.POINTER(ct))


# ----------------------------------------------------------------------------- RNG / math
def philox4x64(ctr, key):
    c = np.ascontiguousarray(ctr, dtype=np.uint64)
    k = np.ascontiguousarray(key, dtype=np.uint64)
    o = np.zeros(4, dtype=np.uint64)
    lib().oracle_philox4x64(_p(c, ctypes.c_uint64), _p(k, ctypes.c_uint64), _p(o, ctypes.c_uint64))
    return o


def u01(x: int) -> float:
    return lib().oracle_u01(int(x))


def det_ln(x: float) -> float:
    return lib().oracle_det_ln(float(x))


def det_exp(x: float) -> float:
    return lib().oracle_det_exp(float(x))


# ----------------------------------------------------------------------------- generator
class _GenParams(ctypes.Structure):
    _fields_ = [
        ("seed", ctypes.c_uint64),
        ("num_conversations", ctypes.c_uint32),
        ("block_tokens", ctypes.c_uint32),
        ("birth_rate", ctypes.c_double),
        ("turn_rate", ctypes.c_double),
        ("death_rate", ctypes.c_double),
        ("prompt_mean_tokens", ctypes.c_double),
        ("prompt_sigma_ln", ctypes.c_double),
        ("response_mean_tokens", ctypes.c_double),
        ("response_sigma_ln", ctypes.c_double),
        ("prompt_min_tokens", ctypes.c_uint32),
        ("prompt_max_tokens", ctypes.c_uint32),
        ("response_min_tokens", ctypes.c_uint32),
        ("response_max_tokens", ctypes.c_uint32),
        ("max_history_blocks", ctypes.c_uint32),
        ("max_turns", ctypes.c_uint32),
    ]


@dataclass
class Trace:
    """Event-ordered trace: one request per event."""
    ticks: np.ndarray
    conv: np.ndarray
    q: np.ndarray
    a: np.ndarray
    is_last: np.ndarray

    @property
    def E(self) -> int:
        return int(self.conv.shape[0])


def generate(params: dict) -> Trace:
    """Synthetic trace from the paper's stochastic conversation model.

    ``params`` uses the field names of ``tlru_gen_params`` (include/tlru.h) and
    is filled from ``tests/inputs.py`` presets.
    """
    gp = _GenParams(**params)
    u64p = ctypes.POINTER(ctypes.c_uint64)
    u32p = ctypes.POINTER(ctypes.c_uint32)
    t, c, q, a, l = u64p(), u32p(), u32p(), u32p(), u32p()
    n = lib().oracle_generate(ctypes.byref(gp), ctypes.byref(t), ctypes.byref(c), ctypes.byref(q),
                              ctypes.byref(a), ctypes.byref(l))
    if n < 0:
        raise ValueError("oracle_generate: invalid parameters")

    def take(ptr, dt):
        arr = np.ctypeslib.as_array(ptr, shape=(max(n, 1),))[:n].astype(dt, copy=True)
        lib().oracle_free(ctypes.cast(ptr, ctypes.c_void_p))
        return arr

    return Trace(take(t, np.uint64), take(c, np.uint32), take(q, np.uint32), take(a, np.uint32),
                 take(l, np.uint32))


# ----------------------------------------------------------------------------- derive / replay
@dataclass
class Derived:
    prev: np.ndarray
    J: np.ndarray
    L_after: np.ndarray
    next: np.ndarray


def derive(conv, q, a) -> Derived:
    conv = np.ascontiguousarray(conv, dtype=np.uint32)
    q = np.ascontiguousarray(q, dtype=np.uint32)
    a = np.ascontiguousarray(a, dtype=np.uint32)
    E = conv.shape[0]
    prev = np.zeros(E, np.uint32)
    nxt = np.zeros(E, np.uint32)
    J = np.zeros(E, np.uint64)
    La = np.zeros(E, np.uint64)
    rc = lib().oracle_derive(_p(conv, ctypes.c_uint32), _p(q, ctypes.c_uint32), _p(a, ctypes.c_uint32), E,
                             _p(prev, ctypes.c_uint32), _p(J, ctypes.c_uint64), _p(La, ctypes.c_uint64),
                             _p(nxt, ctypes.c_uint32))
    if rc != 0:
        raise MemoryError("oracle_derive")
    return Derived(prev, J, La, nxt)


LRU = 0
TLRU = 1
THRESHOLD = 2
END_AWARE = 3
LENGTH_AWARE = 4
TAIL_BELADY = 5  # Thm 1 hindsight policy, Reading #26
TLRU_FORCED = 7  # T-LRU under forced caching (App. C), Reading #28
BELADY_FORCED = 8  # Tail-Optimized Belady under forced caching (App. C), Reading #29
ETLRU_FORCED = 9  # ET-LRU under forced caching (App. C), Reading #30 (replay_etlru(forced=True))
ET_LRU = 6  # Def. 1 / Alg. 2, Reading #27 -- see replay_etlru


@dataclass
class Replay:
    b: np.ndarray
    evicted_trim: int
    evicted_lru: int
    max_occupancy: int


def replay(conv, q, a, policy: int, C: int, xi: int = 0, q_hat: int = 0, threshold: int = 0) -> Replay:
    """Alg. 1 replay of one instance; LRU = Phase 2 only; policy 2 =
    Threshold-LRU with admission threshold `threshold` blocks."""
    conv = np.ascontiguousarray(conv, dtype=np.uint32)
    q = np.ascontiguousarray(q, dtype=np.uint32)
    a = np.ascontiguousarray(a, dtype=np.uint32)
    E = conv.shape[0]
    b = np.zeros(E, np.uint64)
    cnt = np.zeros(3, np.uint64)
    rc = lib().oracle_replay(_p(conv, ctypes.c_uint32), _p(q, ctypes.c_uint32), _p(a, ctypes.c_uint32), E,
                             int(policy), int(C), int(xi), int(q_hat), int(threshold), _p(b, ctypes.c_uint64),
                             _p(cnt, ctypes.c_uint64))
    if rc != 0:
        raise MemoryError("oracle_replay")
    return Replay(b, int(cnt[0]), int(cnt[1]), int(cnt[2]))


def replay_etlru(conv, q, a, ticks, C: int, xi: int, mu_tick: float, ln_surv, forced: bool = False) -> Replay:
    """Expected-Tail-Optimized LRU (Def. 1 / Alg. 2; Reading #27):
    greedy block-by-block eviction by the ranking criterion mu * time_i + ln P(Q >= X_i - L_i + xi).
    ticks[E]: event times (u64 microseconds); ln_surv[k] = ln P(Q >= k), k = 0..K.
    evicted_trim = blocks evicted with P = 0, evicted_lru = the others.
    forced: under forced caching (App. C; Reading #30) theta keeps its whole history
    while its turn is served (only if it alone exceeds C does it lose the excess, evicted_lru)."""
    conv = np.ascontiguousarray(conv, dtype=np.uint32)
    q = np.ascontiguousarray(q, dtype=np.uint32)
    a = np.ascontiguousarray(a, dtype=np.uint32)
    ticks = np.ascontiguousarray(ticks, dtype=np.uint64)
    ls = np.ascontiguousarray(ln_surv, dtype=np.float64)
    E = conv.shape[0]
    b = np.zeros(E, np.uint64)
    cnt = np.zeros(3, np.uint64)
    rc = lib().oracle_replay_etlru(_p(conv, ctypes.c_uint32), _p(q, ctypes.c_uint32), _p(a, ctypes.c_uint32),
                                   _p(ticks, ctypes.c_uint64), E, int(C), int(xi), float(mu_tick),
                                   _p(ls, ctypes.c_double), ls.shape[0] - 1, 1 if forced else 0,
                                   _p(b, ctypes.c_uint64), _p(cnt, ctypes.c_uint64))
    if rc != 0:
        raise MemoryError("oracle_replay_etlru")
    return Replay(b, int(cnt[0]), int(cnt[1]), int(cnt[2]))


@dataclass
class Tail:
    n: int
    tel_blocks: int
    slo_violations: int
    sum_b: int
    p50: int
    p90: int
    p95: int
    p99: int
    tel_ms: float
    p50_ms: float
    p90_ms: float
    p95_ms: float
    p99_ms: float
    mean_ms: float


def tail(b, xi: int, xi_ms: float, slo: int, alpha: float) -> Tail:
    """Tail metrics of one request segment (Eq. 1-3)."""
    b = np.ascontiguousarray(b, dtype=np.uint64)
    ints = np.zeros(8, np.uint64)
    dbl = np.zeros(6, np.float64)
    rc = lib().oracle_tail(_p(b, ctypes.c_uint64), b.shape[0], int(xi), float(xi_ms), int(slo), float(alpha),
                           _p(ints, ctypes.c_uint64), _p(dbl, ctypes.c_double))
    if rc != 0:
        raise MemoryError("oracle_tail")
    return Tail(*[int(x) for x in ints], *[float(x) for x in dbl])
