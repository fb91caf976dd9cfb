"""ET-LRU burn-in verification per capacity at a fixed segment length (one 10^6-conversation trace):
which capacities' segments fail the fix-up's start-state check (re-runs = spilled_chains)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2510_15152_b200.tlru as T  # noqa: E402
from paper_2510_15152_b200.inputs import CAPS_CONFIG5, WILDCHAT, preset, prompt_law_ln_surv  # noqa: E402

seg = int(sys.argv[1]) if len(sys.argv) > 1 else 69632
pols = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [6]
p = preset("wildchat", 0, 1_000_000)
T.set_etlru_model(p["death_rate"] * 1e-6, prompt_law_ln_surv(WILDCHAT))
tr = T.generate_traces([p], exports=True)[0]
T.set_sim_options(seg, 0)
for pol in pols:
    for C in CAPS_CONFIG5[::3]:
        rows = [(0, pol, C, xi, 2, 16) for xi in (4, 8, 16, 24)]
        bt = T.prepare_batch([tr], rows)
        torch.cuda.synchronize()
        t0 = time.time()
        bt.run()
        torch.cuda.synchronize()
        st = T.last_sim_stats()
        print(f"pol {pol} C={C} wall {1000 * (time.time() - t0):.1f} ms k2 {st['k2_ms']:.1f} ms state {st['state_entries']} "
              f"segs {st['segment_events']} spilled {st['spilled_chains']}", flush=True)
T.set_sim_options(0, 0)
