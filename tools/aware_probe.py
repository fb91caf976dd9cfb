"""Timing probe for whole-trace End-/Length-Aware chains (one 10^6-conversation trace)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2510_15152_b200.tlru as T  # noqa: E402
from paper_2510_15152_b200.inputs import Q_HAT, SLO_BLOCKS, preset  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
tr = T.generate_traces([preset("wildchat", 0, n)], exports=False)[0]
for pol, C in ((1, 256), (3, 16), (3, 256), (3, 4096), (4, 4096)):
    rows = [(0, pol, C, xi, Q_HAT, SLO_BLOCKS) for xi in range(2, 34)]  # one full warp of lanes
    T.set_sim_engine(T.ENGINE_REPLAY)
    bt = T.prepare_batch([tr], rows)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    bt.run()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st = T.last_sim_stats()
    print(f"policy {pol} C {C}: {dt*1e3:.1f} ms  k2 {st['k2_ms']:.1f} ms  chains {st['chains']} spilled {st['spilled_chains']} "
          f"W {st['state_entries']} seg {st['segment_events']}", flush=True)
