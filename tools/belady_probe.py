"""Timing / ncu probe: Tail-Optimized Belady lanes (one warp of 32 xi lanes per C) on one trace."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2510_15152_b200.tlru as T  # noqa: E402
from paper_2510_15152_b200.inputs import Q_HAT, SLO_BLOCKS, preset  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
tr = T.generate_traces([preset("wildchat", 0, n)], exports=False)[0]
for C in (16, 256, 4096):
    rows = [(0, 5, C, xi, Q_HAT, SLO_BLOCKS) for xi in range(2, 34)]
    bt = T.prepare_batch([tr], rows)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    bt.run()
    torch.cuda.synchronize()
    st = T.last_sim_stats()
    print(f"Belady C {C}: {1e3 * (time.perf_counter() - t0):.1f} ms re-run {st['spilled_chains']} "
          f"W {st['state_entries']}", flush=True)
