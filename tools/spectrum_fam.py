"""Device ms per NEXT family on one 10^6-conversation trace (25 capacities x xi in {4, 8, 16, 24})."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_15152_b200.tlru as T  # noqa: E402
from paper_2510_15152_b200.inputs import CAPS_CONFIG5, Q_HAT, SLO_BLOCKS, WILDCHAT, preset, prompt_law_ln_surv  # noqa: E402

tr = T.generate_traces([preset("wildchat", 0, 1_000_000)], exports=True)[0]
T.set_etlru_model(WILDCHAT["death_rate"] * 1e-6, prompt_law_ln_surv(WILDCHAT))
for pol in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "3,4,5,7,8").split(",")]:
    rows = [(0, pol, C, xi, Q_HAT, SLO_BLOCKS) for C in CAPS_CONFIG5 for xi in (4, 8, 16, 24)]
    bt = T.prepare_batch([tr], rows)
    bt.run()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    bt.run()
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    print(f"policy {pol}: {ms:.1f} ms  {tr.num_events * len(rows) / ms * 1e3:.3g} req/s  re-runs "
          f"{T.last_sim_stats()['spilled_chains']}", flush=True)
