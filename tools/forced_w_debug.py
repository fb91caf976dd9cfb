"""Forced-caching T-LRU with every lane forced to W entries vs the oracle (python tools/forced_w_debug.py W)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2510_15152_b200.tlru as T  # noqa: E402
from paper_2510_15152_b200.inputs import Q_HAT, SLO_BLOCKS, preset  # noqa: E402

W = int(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
p = preset("wildchat", 0, n)
tr = T.generate_traces([p], exports=False)[0]
o = O.generate(p)
rows = [(0, 7, C, xi, Q_HAT, SLO_BLOCKS) for C in (16, 64, 256, 1024, 4096) for xi in (4, 16)]
T.set_sim_options(0, W)
bt = T.simulate_batch([tr], rows)
st = T.last_sim_stats()
T.set_sim_options(0, 0)
print("stats", st)
for i, r in enumerate(rows):
    ob = O.replay(o.conv, o.q, o.a, 7, r[2], r[3], r[4]).b
    g = bt.b(i).astype(np.uint64)
    d = np.flatnonzero(g != ob)
    print(r, "OK" if len(d) == 0 else f"DIFF at {d[:5]} (of {len(d)}), gpu {g[d[:5]]} oracle {ob[d[:5]]}")
