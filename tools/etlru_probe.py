"""Timing probe of the ET-LRU kernel (one 10^6-conversation trace): device ms per capacity."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2510_15152_b200.tlru as T  # noqa: E402
from paper_2510_15152_b200.inputs import CAPS_CONFIG5, WILDCHAT, preset, prompt_law_ln_surv  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
p = preset("wildchat", 0, n)
T.set_etlru_model(p["death_rate"] * 1e-6, prompt_law_ln_surv(WILDCHAT))
tr = T.generate_traces([p], exports=True)[0]
print("events", tr.num_events, flush=True)
for C in (CAPS_CONFIG5[0], CAPS_CONFIG5[8], CAPS_CONFIG5[12], CAPS_CONFIG5[16], CAPS_CONFIG5[20], CAPS_CONFIG5[24]):
    rows = [(0, 6, C, xi, 2, 16) for xi in (4, 8, 16, 24)]
    bt = T.prepare_batch([tr], rows)
    torch.cuda.synchronize()
    t0 = time.time()
    bt.run()
    torch.cuda.synchronize()
    st = T.last_sim_stats()
    print(f"C={C} wall {1000 * (time.time() - t0):.1f} ms k2 {st['k2_ms']:.1f} ms state {st['state_entries']} "
          f"spilled {st['spilled_chains']}", flush=True)
