"""Parity of the CUDA path (through the C ABI) with the CPU oracle, element by element.

Bars: every integer output bit-exact (generated trace
arrays, per-request uncached blocks b, evictions, occupancy, TEL in blocks, SLO
counts, percentiles in blocks); millisecond fields within 1e-9 relative (they are
alpha times exact integers, summed in a different order).
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2510_15152_b200.inputs import (CAPS_CONFIG3, CAPS_CONFIG4, CAPS_CONFIG5, FIG1, Q_HAT, SLO_BLOCKS,
                                          XI_BLOCKS, XI_CONFIG5, ALPHA_MS, config5_rows, preset, random_trace,
                                          tiny_trace)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2510_15152_b200.tlru as T
    T.set_sim_options(0, 0)
    yield T
    T.set_sim_options(0, 0)
    T.set_sim_engine(T.ENGINE_STACK)


ENGINES = pytest.mark.parametrize("engine", [0, 1], ids=["replay", "stack"])


def upload(T, conv, q, a):
    c = torch.from_numpy(np.asarray(conv, np.uint32).view(np.int32).copy()).cuda()
    qq = torch.from_numpy(np.asarray(q, np.uint16).view(np.int16).copy()).cuda()
    aa = torch.from_numpy(np.asarray(a, np.uint16).view(np.int16).copy()).cuda()
    return T.trace_from_turns(c, qq, aa)


def check_instances(T, batch, rows, oracle_traces, alpha=ALPHA_MS):
    res = batch.results_numpy()
    for i, (t, pol, C, xi, qh, slo) in enumerate(rows):
        conv, q, a = oracle_traces[t]
        r = O.replay(conv, q, a, pol, C, xi, qh)
        b = batch.b(i).astype(np.uint64)
        assert np.array_equal(b, r.b), f"row {i} {rows[i]}: first diff at {np.flatnonzero(b != r.b)[:5]}"
        tl = O.tail(r.b, xi, alpha * xi, slo, alpha)
        got = res[i]
        assert got["requests"] == tl.n and got["sum_uncached"] == tl.sum_b
        assert got["tel_blocks"] == tl.tel_blocks and got["slo_violations"] == tl.slo_violations
        assert (got["p50"], got["p90"], got["p95"], got["p99"]) == (tl.p50, tl.p90, tl.p95, tl.p99)
        assert got["evicted_trim"] == r.evicted_trim and got["evicted_lru"] == r.evicted_lru, rows[i]
        assert got["max_occupancy"] == r.max_occupancy
        assert got["max_uncached"] == (int(r.b.max()) if r.b.size else 0)


# ----------------------------------------------------------------------------- config 1: Figure 1
@ENGINES
def test_fig1_through_the_abi(T, engine):
    T.set_sim_engine(engine)
    tr = upload(T, FIG1["conv"], FIG1["q"], FIG1["a"])
    rows = [(0, 0, FIG1["C"], FIG1["xi"], FIG1["q_hat"], 0), (0, 1, FIG1["C"], FIG1["xi"], FIG1["q_hat"], 0)]
    bt = T.simulate_batch([tr], rows)
    assert list(bt.b(0)) == [100, 100, 200]  # P:37 LRU tail 200
    assert list(bt.b(1)) == [100, 100, 150]  # P:37 partial eviction 150
    res = bt.results_numpy()
    assert (res[0]["evicted_trim"], res[0]["evicted_lru"]) == (0, 300)
    assert (res[1]["evicted_trim"], res[1]["evicted_lru"]) == (150, 100)
    assert res[0]["tel_blocks"] == 50 and res[1]["tel_blocks"] == 0
    assert res[0]["max_uncached"] == 200 and res[1]["max_uncached"] == 150


# ----------------------------------------------------------------------------- config 2: tiny traces, full grid
@ENGINES
def test_tiny_traces_full_parameter_grid(T, engine):
    T.set_sim_engine(engine)
    traces, otr, rows = [], [], []
    for seed in range(120):
        conv, q, a = tiny_trace(seed)
        traces.append(upload(T, conv, q, a))
        otr.append((conv, q, a))
        t = len(traces) - 1
        for pol in (0, 1):
            for C in range(9):
                for xi in range(6):
                    for qh in range(4):
                        rows.append((t, pol, C, xi, qh, seed % 4))
    bt = T.simulate_batch(traces, rows)
    check_instances(T, bt, rows, otr)


# ----------------------------------------------------------------------------- upload path + segmentation
def test_upload_derivation_matches_oracle(T):
    conv, q, a = random_trace(3, 5000, 300)
    tr = upload(T, conv, q, a)
    prev, J, La = tr.prev_J_La()
    d = O.derive(conv, q, a)
    assert np.array_equal(prev, d.prev) and np.array_equal(J, d.J) and np.array_equal(La, d.L_after)
    nxt = tr.next[: tr.num_events].cpu().numpy().view(np.uint32)
    assert np.array_equal(nxt, d.next)
    assert tr.num_conversations == np.unique(conv).size and tr.max_history == int(d.L_after.max())


@pytest.mark.parametrize("seg", [32, 64, 96, 256])
def test_segment_warm_start_is_exact(T, seg):
    """Segment starts rebuilt from the stack property reproduce the
    sequential replay for every segment length."""
    traces, otr, rows = [], [], []
    for s in range(6):
        conv, q, a = random_trace(100 + s, 1500, 60 + 20 * s, q_max=6, a_max=6)
        traces.append(upload(T, conv, q, a))
        otr.append((conv, q, a))
        for pol, xi, qh in ((0, 0, 0), (1, 6, 2), (1, 20, 2), (1, 40, 1), (1, 2, 2)):
            for C in (0, 1, 7, 30, 120, 500, 100000):
                rows.append((s, pol, C, xi, qh, 16))
    T.set_sim_engine(T.ENGINE_REPLAY)
    T.set_sim_options(seg, 0)
    try:
        bt = T.simulate_batch(traces, rows)
        check_instances(T, bt, rows, otr)
        st = T.last_sim_stats()
        assert st["segment_events"] == seg and st["failed_chains"] == 0
    finally:
        T.set_sim_options(0, 0)


@ENGINES
def test_extreme_parameters(T, engine):
    """Capacities 0 / 1 / huge and free tails D around max L_after and beyond 2^16."""
    T.set_sim_engine(engine)
    conv, q, a = random_trace(21, 3000, 200, q_max=9, a_max=9)
    tr = upload(T, conv, q, a)
    mL = tr.max_history
    rows = []
    for xi, qh in ((0, 0), (1, 0), (mL - 1, 0), (mL, 0), (mL + 1, 0), (70000, 3), (2**31, 0)):
        for C in (0, 1, 17, 400, 2**31 - 1, 2**32 - 1):
            rows.append((0, 1, C, xi, qh, 16))
    rows += [(0, 0, C, 5, 2, 16) for C in (0, 1, 2**32 - 1)]
    bt = T.simulate_batch([tr], rows)
    check_instances(T, bt, rows, [(conv, q, a)])


def test_spill_path_is_exact(T):
    """Force W = 32 entries with capacities that need more: chains spill to
    global memory and are re-run; results stay exact."""
    conv, q, a = random_trace(11, 4000, 400, q_max=3, a_max=3, locality=0.3)
    tr = upload(T, conv, q, a)
    rows = [(0, pol, C, xi, 1, 16) for pol in (0, 1) for C in (50, 200, 800) for xi in (0, 9)]
    T.set_sim_engine(T.ENGINE_REPLAY)
    T.set_sim_options(256, 32)
    try:
        bt = T.simulate_batch([tr], rows)
        st = T.last_sim_stats()
        check_instances(T, bt, rows, [(conv, q, a)])
        assert st["spilled_chains"] > 0 and st["failed_chains"] == 0
    finally:
        T.set_sim_options(0, 0)


def test_determinism_across_launch_configs(T):
    conv, q, a = random_trace(5, 6000, 500)
    tr = upload(T, conv, q, a)
    rows = [(0, pol, C, 12, 2, 16) for pol in (0, 1) for C in (10, 60, 300)]
    outs = []
    for engine, seg, w in ((0, 0, 0), (0, 64, 0), (0, 2048, 1024), (0, 128, 64), (1, 0, 0)):
        T.set_sim_engine(engine)
        T.set_sim_options(seg, w)
        bt = T.simulate_batch([tr], rows)
        outs.append((b"".join(bt.b(i).tobytes() for i in range(len(rows))), bt.results.cpu().numpy().tobytes()))
    T.set_sim_options(0, 0)
    assert all(o == outs[0] for o in outs)


# ----------------------------------------------------------------------------- generator parity
@pytest.mark.parametrize("name,seed,n", [("wildchat", 0, 10_000), ("wildchat", 9, 10_000), ("sharegpt", 2, 5_000)])
def test_generator_bit_exact(T, name, seed, n):
    p = preset(name, seed, n)
    g = T.generate_traces([p])[0]
    o = O.generate(p)
    E = g.num_events
    assert E == o.E
    assert np.array_equal(g.time_ticks[:E].cpu().numpy().view(np.uint64), o.ticks)
    assert np.array_equal(g.conv[:E].cpu().numpy().view(np.uint32), o.conv)
    assert np.array_equal(g.prompt[:E].view(torch.int16).cpu().numpy().view(np.uint16), o.q)
    assert np.array_equal(g.response[:E].view(torch.int16).cpu().numpy().view(np.uint16), o.a)
    assert np.array_equal(g.is_last[:E].cpu().numpy(), o.is_last.astype(np.uint8))
    prev, J, La = g.prev_J_La()
    d = O.derive(o.conv, o.q, o.a)
    assert np.array_equal(prev, d.prev) and np.array_equal(J, d.J) and np.array_equal(La, d.L_after)
    assert np.array_equal(g.next[:E].cpu().numpy().view(np.uint32), d.next)
    assert g.max_history == int(d.L_after.max()) and g.num_conversations == np.unique(o.conv).size


@pytest.mark.parametrize("capacity", ["exact", "slots", "bound"])
def test_generator_context_cap_bit_exact(T, capacity):
    """L_max small enough that the context window ends conversations: with exact
    capacity the exact count path runs, with the N * max_turns bound the capped
    slots are dropped through the sentinel sort."""
    p = preset("wildchat", 4, 4000)
    p["max_history_blocks"] = 30
    g = T.generate_traces([p], capacity=capacity)[0]
    o = O.generate(p)
    E = g.num_events
    assert E == o.E
    assert np.array_equal(g.time_ticks[:E].cpu().numpy().view(np.uint64), o.ticks)
    assert np.array_equal(g.conv[:E].cpu().numpy().view(np.uint32), o.conv)
    assert np.array_equal(g.is_last[:E].cpu().numpy(), o.is_last.astype(np.uint8))
    prev, J, La = g.prev_J_La()
    d = O.derive(o.conv, o.q, o.a)
    assert np.array_equal(prev, d.prev) and np.array_equal(La, d.L_after) and La.max() <= 30
    assert np.array_equal(g.next[:E].cpu().numpy().view(np.uint32), d.next)
    if capacity == "slots":  # the clock-only slot count bounds E; this cap drops some turns
        assert g.sim.numel() > E


def test_event_slots_bound_events(T):
    """tlru_count_event_slots >= tlru_count_events (= the oracle's E); equal without the cap."""
    import ctypes
    from paper_2510_15152_b200 import _abi as A
    for cap in (30, 65535):
        p = preset("wildchat", 5, 3000)
        p["max_history_blocks"] = cap
        g = T._gen_struct(p)
        sz = ctypes.c_size_t()
        A.check(A.lib.tlru_gen_workspace_size(ctypes.byref(g), 0, ctypes.byref(sz)))
        ws = torch.empty(sz.value, dtype=torch.uint8, device="cuda")
        E, S = ctypes.c_uint64(), ctypes.c_uint64()
        A.check(A.lib.tlru_count_events(ctypes.byref(g), ctypes.byref(E), T._ptr(ws), sz.value, None))
        A.check(A.lib.tlru_count_event_slots(ctypes.byref(g), ctypes.byref(S), T._ptr(ws), sz.value, None))
        assert E.value == O.generate(p).E
        assert (S.value > E.value) if cap == 30 else (S.value >= E.value)


# ----------------------------------------------------------------------------- config 3: 10^4 conversations
@ENGINES
def test_config3_full_parity(T, engine):
    """BASELINE config 3: 10^4-conversation WildChat-shaped traces, seeds 0..9,
    C in {32..1024}, xi in {4..40} (50..500 ms), Q_hat = 2, LRU and T-LRU."""
    T.set_sim_engine(engine)
    params = [preset("wildchat", s, 10_000) for s in range(10)]
    traces = T.generate_traces(params, exports=False)
    otr = []
    for p in params:
        o = O.generate(p)
        otr.append((o.conv, o.q, o.a))
    rows = [(t, pol, C, xi, Q_HAT, SLO_BLOCKS) for t in range(10) for pol in (0, 1) for C in CAPS_CONFIG3
            for xi in XI_BLOCKS]
    bt = T.simulate_batch(traces, rows)
    check_instances(T, bt, rows, otr)


# ----------------------------------------------------------------------------- config 4 (bench launch), sampled
@ENGINES
def test_config4_bench_launch_sampled(T, engine):
    """The bench's launch configuration (10^6 conversations, 96 instances of one
    seed in one batch); every capacity checked against the oracle for one xi per
    policy, and every instance checked for properties that hold at any size."""
    T.set_sim_engine(engine)
    p = preset("wildchat", 0, 1_000_000)
    g = T.generate_traces([p], exports=False)[0]
    o = O.generate(p)
    assert g.num_events == o.E
    rows = [(0, pol, C, xi, Q_HAT, SLO_BLOCKS) for pol in (0, 1) for C in CAPS_CONFIG4 for xi in XI_BLOCKS]
    bt = T.simulate_batch([g], rows)
    res = bt.results_numpy()
    _, J, _ = g.prev_J_La()
    sample = [i for i, r in enumerate(rows) if (r[1] == 0 and r[3] == 4) or (r[1] == 1 and r[3] == 16)]
    for i in sample:
        _, pol, C, xi, qh, slo = rows[i]
        r = O.replay(o.conv, o.q, o.a, pol, C, xi, qh)
        assert np.array_equal(bt.b(i).astype(np.uint64), r.b), rows[i]
        assert res[i]["evicted_trim"] == r.evicted_trim and res[i]["evicted_lru"] == r.evicted_lru
    for i, (_, pol, C, xi, qh, slo) in enumerate(rows):
        b = bt.b(i)
        assert res[i]["requests"] == g.num_events and np.all(b <= J) and res[i]["max_occupancy"] <= C
        if pol == 0:  # LRU b is independent of xi
            j = rows.index((0, 0, C, 4, Q_HAT, SLO_BLOCKS))
            assert np.array_equal(b, bt.b(j))
    # per-request b non-increasing in C (stack property) for LRU and T-LRU(xi=16)
    for pol, xi in ((0, 4), (1, 16)):
        prevb = None
        for C in CAPS_CONFIG4:
            b = bt.b(rows.index((0, pol, C, xi, Q_HAT, SLO_BLOCKS)))
            if prevb is not None:
                assert np.all(b <= prevb)
            prevb = b


# ----------------------------------------------------------------------------- config 5 (the bench workload)
def test_config5_bench_launch_sampled(T):
    """bench.py's launch: the 10^4-instance config-5 sweep (10 seeds x 25 C x 20 xi x
    {LRU, T-LRU}) in ONE tlru_simulate_batch on 10^6-conversation traces, default engine.
    Sampled instances of three seeds against the oracle element by element; every
    instance against properties that hold at any size."""
    T.set_sim_engine(T.ENGINE_STACK)
    params = [preset("wildchat", s, 1_000_000) for s in range(10)]
    traces = T.generate_traces(params, exports=False)
    rows = config5_rows(10)
    bt = T.simulate_batch(traces, rows)
    res = bt.results_numpy()
    rng = np.random.default_rng(5)
    for t in (0, 4, 9):
        o = O.generate(params[t])
        assert traces[t].num_events == o.E
        idx = [i for i, r in enumerate(rows) if r[0] == t]
        for i in rng.choice(idx, size=3, replace=False):
            _, pol, C, xi, qh, slo = rows[i]
            r = O.replay(o.conv, o.q, o.a, pol, C, xi, qh)
            assert np.array_equal(bt.b(i).astype(np.uint64), r.b), rows[i]
            tl = O.tail(r.b, xi, ALPHA_MS * xi, slo, ALPHA_MS)
            assert (res[i]["tel_blocks"], res[i]["slo_violations"], res[i]["p90"], res[i]["p95"]) == \
                (tl.tel_blocks, tl.slo_violations, tl.p90, tl.p95)
            assert (res[i]["evicted_trim"], res[i]["evicted_lru"], res[i]["max_occupancy"]) == \
                (r.evicted_trim, r.evicted_lru, r.max_occupancy)
    key = {r: i for i, r in enumerate(rows)}
    for i, (t, pol, C, xi, qh, slo) in enumerate(rows):
        assert res[i]["requests"] == traces[t].num_events and res[i]["max_occupancy"] <= C
        if pol == 0:  # LRU ignores xi except in TEL: identical b statistics across xi
            j = key[(t, 0, C, XI_CONFIG5[0], qh, slo)]
            assert res[i]["sum_uncached"] == res[j]["sum_uncached"] and res[i]["p99"] == res[j]["p99"]
        if pol == 1 and xi <= qh:  # T-LRU with xi <= Q_hat is LRU
            j = key[(t, 0, C, xi, qh, slo)]
            assert res[i].tobytes() == res[j].tobytes()
    for t in range(10):  # inclusion: sum b non-increasing in C, per policy and xi
        for pol in (0, 1):
            for xi in XI_CONFIG5:
                sums = [res[key[(t, pol, C, xi, Q_HAT, SLO_BLOCKS)]]["sum_uncached"] for C in CAPS_CONFIG5]
                assert all(a >= b for a, b in zip(sums, sums[1:]))


def test_config5_full_grid_one_seed(T):
    """SURVEY 8(d) full-sweep parity, one seed: EVERY (C, xi, policy) cell of the config-5 grid --
    all 1000 instances of seed 0 in the bench's one-trace launch (default engine) -- against the
    oracle element by element (1000 oracle replays on host threads; the ctypes calls release the
    GIL, and each worker compares its own row so host memory stays bounded).  Then the replay
    engine (Alg. 1 request by request) on the same 1000 instances: identical b BYTES, histograms
    and results."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    T.set_sim_engine(T.ENGINE_STACK)
    p = preset("wildchat", 0, 1_000_000)
    g = T.generate_traces([p], exports=False)[0]
    o = O.generate(p)
    assert g.num_events == o.E
    rows = [(0,) + tuple(r[1:]) for r in config5_rows(1)]
    assert len({r[1:4] for r in rows}) == 1000
    bins = g.max_history + 1
    bt = T.simulate_batch([g], rows, hist_bins=bins)
    torch.cuda.synchronize()
    res = bt.results_numpy()

    def one(i):
        _, pol, C, xi, qh, slo = rows[i]
        r = O.replay(o.conv, o.q, o.a, pol, C, xi, qh)
        if not np.array_equal(bt.b(i).astype(np.uint64), r.b):
            return i, "b"
        tl = O.tail(r.b, xi, ALPHA_MS * xi, slo, ALPHA_MS)
        got = res[i]
        if (got["sum_uncached"], got["tel_blocks"], got["slo_violations"]) != (tl.sum_b, tl.tel_blocks,
                                                                                tl.slo_violations):
            return i, "tel/slo"
        if (got["p50"], got["p90"], got["p95"], got["p99"]) != (tl.p50, tl.p90, tl.p95, tl.p99):
            return i, "percentiles"
        if (got["evicted_trim"], got["evicted_lru"], got["max_occupancy"]) != (r.evicted_trim, r.evicted_lru,
                                                                                r.max_occupancy):
            return i, "evictions"
        return i, None

    with ThreadPoolExecutor(max_workers=max(1, os.cpu_count() or 1)) as ex:
        bad = [(rows[i], what) for i, what in ex.map(one, range(len(rows))) if what]
    assert not bad, bad[:5]
    # the replay engine on the same launch: byte-identical b rows, histograms and results
    bt.uncached.zero_()
    bt.run(check_state=True)
    T.set_sim_engine(T.ENGINE_REPLAY)
    rb = T.prepare_batch([g], rows, hist_bins=bins)
    rb.uncached.zero_()
    rb.run(check_state=True)
    assert T.last_sim_stats()["engine"] == T.ENGINE_REPLAY
    T.set_sim_engine(T.ENGINE_STACK)
    assert torch.equal(rb.uncached, bt.uncached)
    assert torch.equal(rb.hist, bt.hist)
    assert rb.results_numpy().tobytes() == bt.results_numpy().tobytes()


# ----------------------------------------------------------------------------- tail metrics
def test_tail_metrics_against_oracle(T):
    rng = np.random.default_rng(4)
    lens = [0, 1, 3, 10, 1001, 4096, 50_000, 7]
    b = rng.integers(0, 300, size=sum(lens)).astype(np.uint16)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    xi = rng.integers(0, 40, size=len(lens)).astype(np.uint32)
    slo = rng.integers(0, 60, size=len(lens)).astype(np.uint32)
    alpha = 0.37
    xi_ms = xi * 0.41
    dev = torch.from_numpy(b.view(np.int16).copy()).cuda()
    out = T.tail_metrics(dev, off, xi, xi_ms, slo, alpha, 299)
    for s in range(len(lens)):
        seg = b[off[s]:off[s + 1]]
        t = O.tail(seg, int(xi[s]), float(xi_ms[s]), int(slo[s]), alpha)
        o = out[s]
        assert (o["n"], o["tel_blocks"], o["slo_violations"], o["sum_b"]) == (t.n, t.tel_blocks, t.slo_violations,
                                                                              t.sum_b)
        assert (o["p50"], o["p90"], o["p95"], o["p99"]) == (t.p50, t.p90, t.p95, t.p99)
        for k in ("tel_ms", "p50_ms", "p90_ms", "p95_ms", "p99_ms", "mean_ms"):
            assert o[k] == pytest.approx(getattr(t, k), rel=1e-9, abs=1e-12), k
        assert o["n_clamped"] == 0


def test_tail_metrics_never_truncates(T):
    """b above max_b is TLRU_ERANGE, not a clamped percentile (never silent truncation)."""
    b = np.array([1, 5, 9, 70, 80], np.uint16)
    dev = torch.from_numpy(b.view(np.int16).copy()).cuda()
    with pytest.raises(T.TlruError, match="ERANGE.*2 values"):
        T.tail_metrics(dev, [0, 5], [0], [0.0], [0], 1.0, 50)
    out = T.tail_metrics(dev, [0, 5], [0], [0.0], [0], 1.0, 80)
    assert out[0]["n_clamped"] == 0 and out[0]["max_b"] == 80 and out[0]["p99"] == 80


# ----------------------------------------------------------------------------- errors through the ABI
def test_upload_errors(T):
    with pytest.raises(T.TlruError, match="EINVAL"):
        upload(T, [0, 1], [1, 0], [0, 0])
    with pytest.raises(T.TlruError, match="ERANGE"):
        upload(T, [0, 0], [40000, 30000], [0, 0])
    tr = upload(T, [0], [1], [0])
    with pytest.raises(T.TlruError, match="EINVAL"):
        T.set_sim_engine(7)
    with pytest.raises(T.TlruError, match="EUNSUPPORTED"):  # > ETLRU_FORCED: not built
        T.simulate_batch([tr], [(0, 10, 10, 0, 0, 0)])


@ENGINES
def test_empty_trace(T, engine):
    T.set_sim_engine(engine)
    tr = upload(T, [], [], [])
    assert tr.num_events == 0
    bt = T.simulate_batch([tr], [(0, 1, 10, 4, 2, 16)])
    assert bt.results_numpy()[0]["requests"] == 0
