"""Pins of the oracle's synthetic-trace generator (paper Sec. 5 model, App. E)."""
import math

import numpy as np
import pytest

import oracle as O
from paper_2510_15152_b200.inputs import preset


def test_philox4x64_matches_numpy():
    """Philox4x64-10 against numpy.random.Philox (which increments the counter
    before each block, so numpy counter c-1 yields our block c)."""
    rng = np.random.default_rng(0)
    for _ in range(50):
        key = [int(x) for x in rng.integers(0, 2 ** 63, size=2)]
        ctr = [int(x) for x in rng.integers(1, 2 ** 63, size=4)]
        bg = np.random.Philox(key=np.array(key, np.uint64),
                              counter=np.array([ctr[0] - 1] + ctr[1:], np.uint64))
        assert list(bg.random_raw(4)) == [int(x) for x in O.philox4x64(ctr, key)]


def test_u01_range():
    assert O.u01(0) == 2.0 ** -53
    assert O.u01(2 ** 64 - 1) == 1.0


def _ulps(a, b):
    return abs(a - b) / math.ulp(b) if b != 0 else abs(a)


def test_det_ln_exp_against_libm():
    rng = np.random.default_rng(1)
    xs = np.concatenate([rng.random(4000), rng.random(1000) * 1e6, [2.0 ** -53, 1.0, 0.5, 2.0, 200.0]])
    for x in xs:
        if x <= 0:
            continue
        assert _ulps(O.det_ln(float(x)), math.log(x)) <= 4, x
    for y in np.concatenate([rng.normal(0, 3, 4000), [0.0, 1.0, -1.0, 10.0, -30.0]]):
        assert _ulps(O.det_exp(float(y)), math.exp(y)) <= 4, y


@pytest.fixture(scope="module")
def trace100k():
    return O.generate(preset("wildchat", 0, 100_000))


def test_generator_order_and_flags(trace100k):
    t = trace100k
    assert np.all(np.diff(t.ticks.astype(np.int64)) >= 0)
    key = t.ticks.astype(object) * (1 << 32) + t.conv.astype(object)
    # ties in time broken by conversation id, then turn (Reading #9)
    same = np.diff(t.ticks.astype(np.int64)) == 0
    assert np.all(np.diff(t.conv.astype(np.int64))[same] >= 0)
    assert t.q.min() >= 1
    # exactly one last turn per conversation, and it is its final event
    assert t.is_last.sum() == np.unique(t.conv).size
    last_pos = {}
    for i, c in enumerate(t.conv.tolist()):
        last_pos[c] = i
    assert all(t.is_last[i] == 1 for i in last_pos.values())
    del key


def test_generator_turn_process_statistics(trace100k):
    """with Exp(mu) life and Poisson(lambda_turn) turns, turns per
    conversation are geometric with continuation lambda_turn/(lambda_turn+mu) = 0.6,
    mean 1 + lambda_turn/mu = 2.5; births are Poisson(lambda_conv = 1/s)."""
    t = trace100k
    n = 100_000
    counts = np.bincount(t.conv, minlength=n)
    assert counts.min() >= 1
    assert abs(counts.mean() - 2.5) / 2.5 < 0.015
    for k in (2, 3, 4):
        assert abs((counts >= k).mean() - 0.6 ** (k - 1)) < 0.01
    first = np.full(n, np.iinfo(np.int64).max)
    np.minimum.at(first, t.conv, t.ticks.astype(np.int64))
    gaps = np.diff(np.sort(first)) / 1e6
    assert abs(gaps.mean() - 1.0) < 0.015
    d = O.derive(t.conv, t.q, t.a)
    assert d.L_after.max() <= preset()["max_history_blocks"]


def test_generator_length_laws_match_numpy_lognormal(trace100k):
    """P:242 / P:307: prompt tokens lognormal with mean 200 (WildChat average);
    block quantization q = max(1, ceil(tok/128)), a = ceil(tok/128).  The block
    distribution must match numpy's lognormal pushed through the same quantizer."""
    p = preset()
    rng = np.random.default_rng(99)
    for field, mean, sig, lo, hi, vals, qmin in (
            ("prompt", p["prompt_mean_tokens"], p["prompt_sigma_ln"], p["prompt_min_tokens"],
             p["prompt_max_tokens"], trace100k.q, 1),
            ("response", p["response_mean_tokens"], p["response_sigma_ln"], p["response_min_tokens"],
             p["response_max_tokens"], trace100k.a, 0)):
        x = rng.lognormal(math.log(mean) - sig * sig / 2, sig, size=2_000_000)
        tok = np.clip(np.floor(x + 0.5), lo, hi)
        blk = np.maximum(np.ceil(tok / p["block_tokens"]), qmin)
        ref = np.bincount(blk.astype(np.int64), minlength=200)[:200] / blk.size
        got = np.bincount(vals.astype(np.int64), minlength=200)[:200] / vals.size
        assert np.abs(ref - got).max() < 0.006, field
        assert abs(vals.mean() - blk.mean()) / blk.mean() < 0.01, field


def test_generator_appendix_e_preset_mean_turns():
    """App. E: lambda_conv = 1, lambda_turn = 3, ~3.5 turns per conversation."""
    t = O.generate(preset("sharegpt", 3, 40_000))
    counts = np.bincount(t.conv, minlength=40_000)
    assert abs(counts.mean() - 3.5) / 3.5 < 0.03


def test_generator_deterministic_and_seeded():
    a = O.generate(preset("wildchat", 5, 3000))
    b = O.generate(preset("wildchat", 5, 3000))
    c = O.generate(preset("wildchat", 6, 3000))
    assert np.array_equal(a.ticks, b.ticks) and np.array_equal(a.q, b.q) and np.array_equal(a.a, b.a)
    assert not np.array_equal(a.ticks[:100], c.ticks[:100])


def test_generator_context_cap():
    p = preset("wildchat", 1, 20_000)
    p["max_history_blocks"] = 40
    t = O.generate(p)
    d = O.derive(t.conv, t.q, t.a)
    assert d.L_after.max() <= 40
    counts = np.bincount(t.conv)
    assert counts.mean() < 2.5  # the cap ends some conversations early
