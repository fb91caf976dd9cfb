"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle's tests.

This module holds NO arithmetic of the method: only parameter presets (the
paper's stochastic-model rates and WildChat/ShareGPT-shaped length laws) and
seeded numpy generators of small (conv, q, a) request sequences used as test
inputs.  Both the oracle (oracle/) and the CUDA path (paper_2510_15152_b200)
consume these; neither computes anything here.

Input recipe:
  * WILDCHAT preset (BASELINE configs 3-5): lambda_conv = 1/s, lambda_turn = 1/60 s,
    mu = 1/90 s (mean 1 + lambda_turn/mu = 2.5 turns), prompt tokens
    lognormal mean 200 (WildChat average) sigma_ln 1.2 clipped [1, 16384],
    response tokens lognormal mean 400 sigma_ln 0.8 clipped [0, 8192],
    128-token blocks, L_max = 1024 blocks, <= 64 turns.
  * SHAREGPT preset (App. E): lambda_conv = 1, lambda_turn = 3,
    mu = 1.2 (3.5 turns), prompt mean 100 tokens.
  * tiny traces (BASELINE config 2): <= 4 conversations, <= 3 turns each,
    q in {1,2,3}, a in {0,1,2}, random interleaving.
"""
from __future__ import annotations

import numpy as np

WILDCHAT = dict(
    num_conversations=1_000_000,
    block_tokens=128,
    birth_rate=1.0,
    turn_rate=1.0 / 60.0,
    death_rate=1.0 / 90.0,
    prompt_mean_tokens=200.0,
    prompt_sigma_ln=1.2,
    response_mean_tokens=400.0,
    response_sigma_ln=0.8,
    prompt_min_tokens=1,
    prompt_max_tokens=16384,
    response_min_tokens=0,
    response_max_tokens=8192,
    max_history_blocks=1024,
    max_turns=64,
)

SHAREGPT = dict(WILDCHAT, turn_rate=3.0, death_rate=1.2, prompt_mean_tokens=100.0,
                response_mean_tokens=250.0, response_sigma_ln=1.0)

# Fixed model conventions (SURVEY 8 / DESIGN.md): alpha = 12.5 ms per 128-token block,
# Q_hat = 2 blocks, SLO 200 ms -> b > 16 blocks, xi_s in {50..500} ms -> xi blocks.
ALPHA_MS = 12.5
Q_HAT = 2
SLO_BLOCKS = 16
XI_BLOCKS = (4, 8, 12, 16, 24, 40)
CAPS_CONFIG3 = (32, 64, 128, 256, 512, 1024)
CAPS_CONFIG4 = (64, 128, 256, 512, 1024, 2048, 3072, 4096)
# BASELINE config 5 (the sweep): 25 capacities geometric 16..4096, 20 xi values 2..40
CAPS_CONFIG5 = tuple(int(round(16 * 256 ** (k / 24))) for k in range(25))
XI_CONFIG5 = tuple(range(2, 41, 2))
SEEDS_CONFIG5 = 10


def prompt_law_ln_surv(preset_params: dict, K: int = 160) -> np.ndarray:
    """ET-LRU's model of the next prompt length (Def. 1; Reading #27): ln P(q >= k)
    for k = 0..K under the preset's own prompt law, q = max(1, ceil(tok / block_tokens)) with
    tok = lognormal(mean, sigma_ln) rounded and clipped.  A model parameter handed to both the
    oracle and the CUDA path (like the preset rates); -inf where the probability is 0.
    Computed with the lognormal CDF (math.erf) at the rounding boundaries."""
    import math
    m, sg = float(preset_params["prompt_mean_tokens"]), float(preset_params["prompt_sigma_ln"])
    lo, hi = int(preset_params["prompt_min_tokens"]), int(preset_params["prompt_max_tokens"])
    B = int(preset_params["block_tokens"])
    mu_ln = math.log(m) - 0.5 * sg * sg

    def cdf_tok_below(x):  # P(rounded, clipped tok < x) for integer x
        if x <= lo:
            return 0.0
        if x > hi:
            return 1.0
        return 0.5 * (1.0 + math.erf((math.log(x - 0.5) - mu_ln) / (sg * math.sqrt(2.0))))

    out = np.empty(K + 1, np.float64)
    for k in range(K + 1):
        if k <= 1:
            out[k] = 0.0  # q >= 1 always
            continue
        p = 1.0 - cdf_tok_below((k - 1) * B + 1)  # q >= k  <=>  tok > (k - 1) B
        out[k] = math.log(p) if p > 0.0 else -math.inf
    return np.minimum.accumulate(out)


# Threshold-LRU admission threshold: 1024 tokens (the OpenAI rule the paper follows) = 8 blocks
THRESHOLD_BLOCKS = 8


def config5_rows(n_traces: int = SEEDS_CONFIG5, threshold_lru: bool = False):
    """(trace, policy, C, xi, Q_hat, slo[, threshold]) for the config-5 sweep over n_traces seeds;
    with threshold_lru the paper's third policy (Threshold-LRU, T = 8 blocks) joins LRU and T-LRU."""
    rows = []
    for t in range(n_traces):
        for pol in ((0, 1, 2) if threshold_lru else (0, 1)):
            for C in CAPS_CONFIG5:
                for xi in XI_CONFIG5:
                    rows.append((t, pol, C, xi, Q_HAT, SLO_BLOCKS) + ((THRESHOLD_BLOCKS,) if pol == 2 else ()))
    return rows

# Figure 1: events A, B, A with 100-block prompts, no responses, C = 100.
FIG1 = dict(conv=[0, 1, 0], q=[100, 100, 100], a=[0, 0, 0], C=100, xi=150, q_hat=100)


def preset(name: str = "wildchat", seed: int = 0, num_conversations: int | None = None) -> dict:
    p = dict(WILDCHAT if name == "wildchat" else SHAREGPT)
    p["seed"] = int(seed)
    if num_conversations is not None:
        p["num_conversations"] = int(num_conversations)
    return p


def tiny_trace(seed: int, max_conv: int = 4, max_turns: int = 3, qs=(1, 2, 3), as_=(0, 1, 2)):
    """Random interleaving of <= max_conv conversations with <= max_turns turns each."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, max_conv + 1))
    turns = rng.integers(1, max_turns + 1, size=n)
    order = np.repeat(np.arange(n), turns)
    rng.shuffle(order)
    q = rng.choice(np.asarray(qs), size=order.size)
    a = rng.choice(np.asarray(as_), size=order.size)
    return order.astype(np.uint32), q.astype(np.uint32), a.astype(np.uint32)


def random_trace(seed: int, n_events: int, n_conv: int, q_max: int = 8, a_max: int = 8,
                 locality: float = 0.7):
    """Random (conv, q, a) request sequence with temporal locality: with probability
    `locality` the next request comes from one of the 8 most recent conversations."""
    rng = np.random.default_rng(seed)
    conv = np.empty(n_events, np.uint32)
    recent: list[int] = []
    for i in range(n_events):
        if recent and rng.random() < locality:
            c = recent[int(rng.integers(0, min(8, len(recent))))]
        else:
            c = int(rng.integers(0, n_conv))
        conv[i] = c
        if c in recent:
            recent.remove(c)
        recent.insert(0, c)
    q = rng.integers(1, q_max + 1, size=n_events).astype(np.uint32)
    a = rng.integers(0, a_max + 1, size=n_events).astype(np.uint32)
    return conv, q, a
