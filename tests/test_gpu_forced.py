"""T-LRU under forced caching (App. C; Reading #28) on the CUDA path (replay engine,
burn-in segments verified by the fix-up), element by element against the oracle via the C ABI."""
import numpy as np
import pytest
import torch

from paper_2510_15152_b200.inputs import CAPS_CONFIG3, Q_HAT, SLO_BLOCKS, preset, random_trace
from test_gpu_aware import check, upload

import oracle as O

pytestmark = pytest.mark.gpu
FORCED = 7


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2510_15152_b200.tlru as T
    yield T
    T.set_sim_options(0, 0)
    T.set_sim_engine(T.ENGINE_STACK)


def test_fig1_forced(T):
    tr = upload(T, [0, 1, 0], [100, 100, 100], [0, 0, 0])
    bt = T.simulate_batch([tr], [(0, FORCED, 100, 150, 100, 16), (0, 1, 100, 150, 100, 16)])
    assert list(bt.b(0)) == [100, 100, 200] and list(bt.b(1)) == [100, 100, 150]
    r = bt.results_numpy()[0]
    assert (r["evicted_trim"], r["evicted_lru"], r["max_occupancy"]) == (100, 200, 100)


def test_random_traces_mixed_batch(T):
    traces, otr, rows = [], [], []
    for s in range(3):
        conv, q, a = random_trace(5100 + s, 6000, 80, q_max=6, a_max=8, locality=0.5)
        traces.append(upload(T, conv, q, a))
        otr.append((conv, q, a))
        for C in (0, 1, 3, 20, 90, 400):
            rows += [(s, FORCED, C, xi, qh, 8) for xi, qh in ((0, 0), (4, 2), (9, 2), (17, 3), (40, 1))]
        rows += [(s, 1, 40, 9, 2, 8), (s, 3, 40, 9, 2, 8), (s, 5, 40, 9, 0, 8)]
    bt = T.simulate_batch(traces, rows)
    assert T.last_sim_stats()["failed_chains"] == 0
    check(T, bt, rows, otr)


def test_generated_preset_and_short_segments(T):
    """Config-3 shape; then the same rows with 512-event segments (burn-in 4096) so most segment
    starts go through the fix-up's verification.  Outputs must not change."""
    p = preset("wildchat", 8, 10_000)
    tr = T.generate_traces([p], exports=False)[0]
    o = O.generate(p)
    rows = [(0, FORCED, C, xi, Q_HAT, SLO_BLOCKS) for C in CAPS_CONFIG3 for xi in (4, 16, 40)]
    bt = T.simulate_batch([tr], rows)
    check(T, bt, rows, [(o.conv, o.q, o.a)])
    T.set_sim_options(512, 0)
    try:
        bt2 = T.simulate_batch([tr], rows)
    finally:
        T.set_sim_options(0, 0)
    assert bt2.results_numpy().tobytes() == bt.results_numpy().tobytes()
    for i in range(len(rows)):
        assert np.array_equal(bt2.b(i), bt.b(i))


def test_full_size_sampled(T):
    """BASELINE trace size (10^6 conversations) in the launch configuration of
    `bench.py --config forced` (one trace, its 100 rows in one batch): sampled instances against
    the oracle element by element, and no failed chains."""
    from paper_2510_15152_b200.inputs import CAPS_CONFIG5
    p = preset("wildchat", 4, 1_000_000)
    tr = T.generate_traces([p], exports=False)[0]
    rows = [(0, FORCED, C, xi, Q_HAT, SLO_BLOCKS) for C in CAPS_CONFIG5 for xi in (4, 8, 16, 24)]
    bt = T.simulate_batch([tr], rows)
    assert T.last_sim_stats()["failed_chains"] == 0
    o = O.generate(p)
    res = bt.results_numpy()
    for C, xi in ((16, 4), (256, 24), (CAPS_CONFIG5[24], 16)):
        i = rows.index((0, FORCED, C, xi, Q_HAT, SLO_BLOCKS))
        r = O.replay(o.conv, o.q, o.a, FORCED, C, xi, Q_HAT)
        assert np.array_equal(bt.b(i).astype(np.uint64), r.b), (C, xi)
        assert (res[i]["evicted_trim"], res[i]["evicted_lru"], res[i]["max_occupancy"]) == (
            r.evicted_trim, r.evicted_lru, r.max_occupancy)


@pytest.mark.parametrize("entries", [256, 512, 1024])
def test_packed_lanes_forced_class(T, entries):
    """Forced-caching T-LRU and End-Aware lanes forced into the 256..1024-entry classes, whose
    no-surplus state is packed ((tau - chain start) << 12 | X, SmemStatePk), with short segments
    (snapshots of packed lanes go through the fix-up): against the oracle."""
    conv, q, a = random_trace(5300 + entries, 5000, 90, q_max=6, a_max=9, locality=0.4)
    tr = upload(T, conv, q, a)
    rows = [(0, pol, C, xi, 2, 8) for pol in (FORCED, 3) for C in (0, 5, 40, 300) for xi in (0, 6, 20)]
    for seg in (0, 512):
        T.set_sim_options(seg, entries)
        try:
            bt = T.simulate_batch([tr], rows)
            assert T.last_sim_stats()["failed_chains"] == 0
        finally:
            T.set_sim_options(0, 0)
        check(T, bt, rows, [(conv, q, a)])
