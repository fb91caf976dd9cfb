"""b-row layouts of the stack engine: rows 16-byte aligned take s2_out's TMA bulk-store writer
path, other alignments the 16-/8-byte and scalar store paths; traces whose length is not a
multiple of 8 exercise every path's tail.  Element by element against the oracle (Alg. 1,
P:195-221) and its tail metrics, through the C ABI."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2510_15152_b200.inputs import ALPHA_MS, preset, random_trace
from test_gpu_aware import upload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2510_15152_b200.tlru as T
    T.set_sim_engine(T.ENGINE_STACK)
    yield T
    T.set_sim_engine(T.ENGINE_STACK)


def _rows(t):
    rows = []
    for C in (0, 5, 16, 37, 128, 700, 4096):
        rows += [(t, 0, C, xi, 2, 8) for xi in (4, 9)]          # LRU: equal-C runs of two rows
        rows += [(t, 1, C, xi, 2, 8) for xi in (2, 3, 9, 17)]  # T-LRU: D = 0, 1, 7, 15
        rows.append((t, 2, C, 0, 0, 8, 6))                     # Threshold-LRU, T = 6
    return rows


@pytest.mark.parametrize("align", [1, 2, 4, 8])
def test_row_alignment_paths(T, align):
    conv, q, a = random_trace(4100 + align, 4999, 70, q_max=6, a_max=8, locality=0.5)  # E odd
    p = preset("wildchat", 11, 6001)
    otr = [(np.asarray(conv), np.asarray(q), np.asarray(a))]
    o = O.generate(p)
    otr.append((o.conv, o.q, o.a))
    traces = [upload(T, conv, q, a), T.generate_traces([p], exports=False)[0]]
    assert traces[0].num_events % 8 != 0
    rows = _rows(0) + _rows(1)
    bt = T.prepare_batch(traces, rows, align=align)
    bt.run()
    torch.cuda.synchronize()
    st = T.last_sim_stats()
    assert st["engine"] == T.ENGINE_STACK and st["failed_chains"] == 0
    res = bt.results_numpy()
    for i, r in enumerate(rows):
        cv, qq, aa = otr[r[0]]
        ob = O.replay(cv, qq, aa, r[1], r[2], r[3], r[4], threshold=r[6] if len(r) > 6 else 0)
        assert np.array_equal(bt.b(i).astype(np.uint64), ob.b), (align, r)
        tl = O.tail(ob.b, r[3], ALPHA_MS * r[3], r[5], ALPHA_MS)
        g = res[i]
        assert (g["sum_uncached"], g["tel_blocks"], g["slo_violations"], g["p50"], g["p90"], g["p95"], g["p99"]) == (
            tl.sum_b, tl.tel_blocks, tl.slo_violations, tl.p50, tl.p90, tl.p95, tl.p99), (align, r)
        assert (g["evicted_trim"], g["evicted_lru"]) == (ob.evicted_trim, ob.evicted_lru), (align, r)
