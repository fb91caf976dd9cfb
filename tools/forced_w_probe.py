"""Forced-caching T-LRU: device ms and re-runs per capacity at forced state classes (tlru_set_sim_options
state_entries = 128 / 256 / 384? / 512 entries), one 10^6-conversation trace."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_15152_b200.tlru as T  # noqa: E402
from paper_2510_15152_b200.inputs import CAPS_CONFIG5, Q_HAT, SLO_BLOCKS, preset  # noqa: E402

tr = T.generate_traces([preset("wildchat", int(sys.argv[1]) if len(sys.argv) > 1 else 0, 1_000_000)],
                       exports=False)[0]
for C in CAPS_CONFIG5[8::2]:
    line = f"C={C}:"
    for w in (128, 256, 512):
        T.set_sim_options(0, w)
        rows = [(0, 7, C, xi, Q_HAT, SLO_BLOCKS) for xi in (4, 8, 16, 24)] * 8
        bt = T.prepare_batch([tr], rows)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        bt.run()
        t1.record()
        torch.cuda.synchronize()
        line += f"  W{w} {t0.elapsed_time(t1):.1f} ms re-runs {T.last_sim_stats()['spilled_chains']}"
        del bt
    print(line, flush=True)
T.set_sim_options(0, 0)
