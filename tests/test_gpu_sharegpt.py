"""App. E's ShareGPT-shaped trace model (lambda_conv = 1, lambda_turn = 3, mu = 1.2 -> 3.5
turns, prompt mean 100 tokens) through the whole CUDA path: the generator bit-exact against the
oracle's, and every policy family element by element against the oracle's replays and tail
metrics, at a config-3-sized trace (several segments and s2_out ranges)."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2510_15152_b200.inputs import ALPHA_MS, CAPS_CONFIG3, SHAREGPT, preset, prompt_law_ln_surv

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2510_15152_b200.tlru as T
    yield T
    T.set_sim_engine(T.ENGINE_STACK)


def test_sharegpt_generator_and_all_policies(T):
    p = preset("sharegpt", 21, 20_000)
    o = O.generate(p)
    g = T.generate_traces([p], exports=True)[0]
    assert g.num_events == o.E
    assert np.array_equal(g.conv[: g.num_events].cpu().numpy().view(np.uint32), o.conv)
    assert np.array_equal(g.prompt[: g.num_events].cpu().numpy().view(np.uint16), o.q)
    assert np.array_equal(g.response[: g.num_events].cpu().numpy().view(np.uint16), o.a)
    mu = SHAREGPT["death_rate"] * 1e-6
    tab = prompt_law_ln_surv(SHAREGPT)
    T.set_etlru_model(mu, tab)
    rows = []
    for C in CAPS_CONFIG3:
        for xi in (4, 16):
            rows += [(0, 0, C, xi, 1, 16), (0, 1, C, xi, 1, 16), (0, 2, C, xi, 0, 16, 8)]
            rows += [(0, pol, C, xi, 1, 16) for pol in (3, 4, 5, 6, 7, 8, 9)]
    bt = T.simulate_batch([g], rows)
    res = bt.results_numpy()
    for i, r in enumerate(rows):
        pol, C, xi, qh, slo = r[1:6]
        if pol in (6, 9):
            ob = O.replay_etlru(o.conv, o.q, o.a, o.ticks, C, xi, mu, tab, forced=pol == 9)
        else:
            ob = O.replay(o.conv, o.q, o.a, pol, C, xi, qh, threshold=r[6] if len(r) > 6 else 0)
        assert np.array_equal(bt.b(i).astype(np.uint64), ob.b), r
        tl = O.tail(ob.b, xi, ALPHA_MS * xi, slo, ALPHA_MS)
        gr = res[i]
        assert (gr["tel_blocks"], gr["slo_violations"], gr["p50"], gr["p90"], gr["p95"], gr["p99"]) == (
            tl.tel_blocks, tl.slo_violations, tl.p50, tl.p90, tl.p95, tl.p99), r
        assert (gr["evicted_trim"], gr["evicted_lru"], gr["max_occupancy"]) == (
            ob.evicted_trim, ob.evicted_lru, ob.max_occupancy), r
