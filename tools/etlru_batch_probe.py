"""ET-LRU / forced ET-LRU: one batch of 25 capacities x xi in {4, 8, 16, 24} on one 10^6-conversation
trace, at the automatic segment length and at given ones: device ms and fix-up re-runs."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2510_15152_b200.tlru as T  # noqa: E402
from paper_2510_15152_b200.inputs import CAPS_CONFIG5, WILDCHAT, preset, prompt_law_ln_surv  # noqa: E402

segs = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 32768]
pols = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [6]
p = preset("wildchat", 0, 1_000_000)
T.set_etlru_model(p["death_rate"] * 1e-6, prompt_law_ln_surv(WILDCHAT))
tr = T.generate_traces([p], exports=True)[0]
for pol in pols:
    rows = [(0, pol, C, xi, 2, 16) for C in CAPS_CONFIG5 for xi in (4, 8, 16, 24)]
    for seg in segs:
        T.set_sim_options(seg, 0)
        bt = T.prepare_batch([tr], rows)
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.time()
            bt.run()
            torch.cuda.synchronize()
            st = T.last_sim_stats()
            print(f"pol {pol} seg {seg} rep {rep}: wall {1000 * (time.time() - t0):.1f} ms k2 {st['k2_ms']:.1f} ms "
                  f"segs {st['segment_events']} spilled {st['spilled_chains']} "
                  f"req/s {tr.num_events * len(rows) / (st['k2_ms'] / 1000):.3g}", flush=True)
T.set_sim_options(0, 0)
