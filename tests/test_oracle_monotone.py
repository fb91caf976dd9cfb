"""Per-request b is non-increasing in the capacity C for every policy family of the build -- the
observable consequence of inclusion (cache at C contained in the cache at C + 1), which is what an
all-capacities (stack) evaluation would need.  LRU / T-LRU have it by the
stack property (Sec. 3); for the NEXT policies it is an empirical pin: a search over 7.7x10^6
tiny-trace cells (End-/Length-Aware, Tail-Optimized Belady, forced T-LRU / Belady,
Threshold-LRU) and 1.5x10^6 ET-LRU cells found no violation.  These tests keep a slice of it."""
import numpy as np

import oracle as O


def _tiny(rng):
    k = int(rng.integers(2, 5))
    E = int(rng.integers(3, 10))
    conv = rng.integers(0, k, E).astype(np.uint32)
    q = rng.integers(1, 4, E).astype(np.uint32)
    a = rng.integers(0, 4, E).astype(np.uint32)
    return conv, q, a


def _monotone(bs):
    return all(np.all(bs[i + 1] <= bs[i]) for i in range(len(bs) - 1))


def test_b_monotone_in_capacity_next_policies():
    rng = np.random.default_rng(20261017)
    pols = (O.THRESHOLD, O.END_AWARE, O.LENGTH_AWARE, O.TAIL_BELADY, O.TLRU_FORCED, O.BELADY_FORCED)
    for _ in range(400):
        conv, q, a = _tiny(rng)
        for pol in pols:
            for xi in (0, 1, 3, 6):
                bs = [O.replay(conv, q, a, pol, C, xi, 2, threshold=3).b for C in range(0, 16)]
                assert _monotone(bs), (pol, xi, conv.tolist(), q.tolist(), a.tolist())


def test_b_monotone_in_capacity_etlru():
    rng = np.random.default_rng(11)
    ln_surv = np.log(np.array([1.0, 1.0, 0.7, 0.4, 0.2, 0.1, 0.05, 0.02]))
    for _ in range(150):
        conv, q, a = _tiny(rng)
        ticks = np.cumsum(rng.integers(1, 50, conv.shape[0])).astype(np.uint64)
        for xi in (0, 3, 6):
            for mu in (0.0, 0.2):
                bs = [O.replay_etlru(conv, q, a, ticks, C, xi, mu, ln_surv).b for C in range(0, 16)]
                assert _monotone(bs), (xi, mu, conv.tolist(), q.tolist(), a.tolist(), ticks.tolist())
