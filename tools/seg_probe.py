"""Replay-engine workloads of one trace (spectrum rows, forced rows) timed for several segment
lengths (tlru_set_sim_options(segment_events, 0)); b must not change (python tools/seg_probe.py)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_15152_b200.tlru as T  # noqa: E402
from paper_2510_15152_b200.inputs import CAPS_CONFIG5, Q_HAT, SLO_BLOCKS, preset  # noqa: E402

tr = T.generate_traces([preset("wildchat", 0, 1_000_000)], exports=False)[0]
for name, pols in (("spectrum", (3, 4, 5)), ("forced", (7,)), ("forced_belady", (8,))):
    rows = [(0, pol, C, xi, Q_HAT, SLO_BLOCKS) for pol in pols for C in CAPS_CONFIG5 for xi in (4, 8, 16, 24)]
    ref = None
    for seg in (0, 4096, 16384, 32768, 65536):
        T.set_sim_options(seg, 0)
        bt = T.prepare_batch([tr], rows)
        bt.run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        bt.run()
        e1.record()
        torch.cuda.synchronize()
        st = T.last_sim_stats()
        rs = [bt.b(i).copy() for i in range(0, len(rows), 7)]
        same = ref is None or all((a == b).all() for a, b in zip(rs, ref))
        ref = rs if ref is None else ref
        ms = e0.elapsed_time(e1)
        print(f"{name} seg {seg or 'auto'} ({st['segment_events']}): {ms:.1f} ms, "
              f"{len(rows) * tr.num_events / ms * 1e3:.3g} req/s, chains {st['chains']}, re-run {st['spilled_chains']}, "
              f"identical {same}", flush=True)
T.set_sim_options(0, 0)
