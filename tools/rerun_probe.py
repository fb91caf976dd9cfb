"""Fix-up re-runs of the aware / Belady lanes on several preset seeds (python tools/rerun_probe.py)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_15152_b200.tlru as T  # noqa: E402
from paper_2510_15152_b200.inputs import CAPS_CONFIG5, Q_HAT, SLO_BLOCKS, preset  # noqa: E402

for seed in range(10):
    tr = T.generate_traces([preset("wildchat", seed, 1_000_000)], exports=False)[0]
    rows = [(0, pol, C, xi, Q_HAT, SLO_BLOCKS) for pol in (3, 4, 5, 8) for C in CAPS_CONFIG5 for xi in (4, 24)]
    bt = T.prepare_batch([tr], rows)
    bt.run()
    torch.cuda.synchronize()
    st = T.last_sim_stats()
    print(f"seed {seed}: re-run {st['spilled_chains']} failed {st['failed_chains']} k2 {st['k2_ms']:.1f} ms", flush=True)
