"""One config-5 trace (10^6 conversations, 1000 instances) through the stack engine, run twice:
the launch pattern of one bench trace, for ncu captures of the stack kernels
(ncu -k regex:'s2_(hist|out|win)' -s <first run's launches> ...)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_15152_b200.tlru as T  # noqa: E402
from paper_2510_15152_b200.inputs import config5_rows, preset  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
g = T.generate_traces([preset("wildchat", 0, n)], exports=False)[0]
rows = [(0,) + tuple(r[1:]) for r in config5_rows(1)]
bt = T.prepare_batch([g], rows, hist_bins=g.max_history + 1)
for _ in range(2):
    bt.run()
    torch.cuda.synchronize()
print("events", g.num_events, "stats", T.last_sim_stats())
