"""The spectrum workload of one trace (End-/Length-Aware, Tail-Optimized Belady; 25 C x 4 xi) timed
with the automatic per-capacity state classes and with every lane forced to W entries
(tlru_set_sim_options(0, W)); results must not change (python tools/spectrum_w.py)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_15152_b200.tlru as T  # noqa: E402
from paper_2510_15152_b200.inputs import CAPS_CONFIG5, Q_HAT, SLO_BLOCKS, preset  # noqa: E402

tr = T.generate_traces([preset("wildchat", 0, 1_000_000)], exports=False)[0]
pols = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else "3,4,5")]
rows = [(0, pol, C, xi, Q_HAT, SLO_BLOCKS) for pol in pols for C in CAPS_CONFIG5 for xi in (4, 8, 16, 24)]
ref = None
for W in (0, 96, 128):
    T.set_sim_options(0, W)
    bt = T.prepare_batch([tr], rows)
    bt.run()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    bt.run()
    ev1.record()
    torch.cuda.synchronize()
    st = T.last_sim_stats()
    b = bt.uncached.clone()
    same = ref is None or torch.equal(b, ref)
    ref = b if ref is None else ref
    print(f"W {W or 'auto'}: {ev0.elapsed_time(ev1):.1f} ms, {len(rows) * tr.num_events / ev0.elapsed_time(ev1) * 1e3:.3g} "
          f"req/s, re-run {st['spilled_chains']}, failed {st['failed_chains']}, identical {same}", flush=True)
T.set_sim_options(0, 0)
