"""One replay-engine launch per (policy, C): 32 xi lanes on one 10^6-conversation trace, for ncu
captures of sim_kernel / aware_fix_kernel / etlru_seg_kernel (python tools/replay_probe.py POL C)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_15152_b200.tlru as T  # noqa: E402
from paper_2510_15152_b200.inputs import Q_HAT, SLO_BLOCKS, WILDCHAT, preset, prompt_law_ln_surv  # noqa: E402

pol, C = int(sys.argv[1]), int(sys.argv[2])
p = preset("wildchat", 0, 1_000_000)
tr = T.generate_traces([p], exports=pol == 6)[0]
if pol == 6:
    T.set_etlru_model(WILDCHAT["death_rate"] * 1e-6, prompt_law_ln_surv(WILDCHAT))
rows = [(0, pol, C, xi, Q_HAT, SLO_BLOCKS) for xi in range(2, 34)]
bt = T.prepare_batch([tr], rows)
torch.cuda.synchronize()
t0 = time.perf_counter()
bt.run()
torch.cuda.synchronize()
st = T.last_sim_stats()
print(f"policy {pol} C {C}: {1e3 * (time.perf_counter() - t0):.1f} ms, k2 {st['k2_ms']:.1f} ms, "
      f"{32 * tr.num_events / (st['k2_ms'] / 1e3):.3g} req/s, chains {st['chains']} re-run {st['spilled_chains']} "
      f"W {st['state_entries']} seg {st['segment_events']}")
