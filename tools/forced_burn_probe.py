"""Forced-caching T-LRU (policy 7) per seed: device ms and fix-up re-runs of one 100-instance batch
(25 capacities x xi in {4, 8, 16, 24}) -- for choosing the forced lanes' burn-in (TLRU_FORCED_BURN)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_15152_b200.tlru as T  # noqa: E402
from paper_2510_15152_b200.inputs import CAPS_CONFIG5, Q_HAT, SLO_BLOCKS, preset  # noqa: E402

for name, seeds in (("wildchat", range(10)), ("sharegpt", range(3))):
    for seed in seeds:
        tr = T.generate_traces([preset(name, seed, 1_000_000)], exports=False)[0]
        rows = [(0, 7, C, xi, Q_HAT, SLO_BLOCKS) for C in CAPS_CONFIG5 for xi in (4, 8, 16, 24)]
        bt = T.prepare_batch([tr], rows)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        bt.run()
        t1.record()
        torch.cuda.synchronize()
        print(f"{name} seed {seed}: {t0.elapsed_time(t1):.1f} ms re-runs {T.last_sim_stats()['spilled_chains']}",
              flush=True)
        del bt, tr
