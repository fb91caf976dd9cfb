"""Timing probe: forced-caching T-LRU vs End-Aware on one trace (one warp of 32 xi lanes per row)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2510_15152_b200.tlru as T  # noqa: E402
from paper_2510_15152_b200.inputs import Q_HAT, SLO_BLOCKS, preset  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
tr = T.generate_traces([preset("wildchat", 0, n)], exports=False)[0]
for pol, C in ((3, 256), (7, 256), (3, 4096), (7, 4096), (7, 16)):
    rows = [(0, pol, C, xi, Q_HAT, SLO_BLOCKS) for xi in range(2, 34)]
    bt = T.prepare_batch([tr], rows)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    bt.run()
    torch.cuda.synchronize()
    st = T.last_sim_stats()
    print(f"policy {pol} C {C}: {1e3 * (time.perf_counter() - t0):.1f} ms k2 {st['k2_ms']:.1f} chains {st['chains']} "
          f"re-run/spilled {st['spilled_chains']} failed {st['failed_chains']} W {st['state_entries']}", flush=True)
