"""One spectrum batch (End-Aware, Length-Aware, Belady x 25 C x xi in {4, 8, 16, 24} on one 10^6-conversation
trace), run twice -- for ncu captures of the lockstep replay kernels."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_15152_b200.tlru as T  # noqa: E402
from paper_2510_15152_b200.inputs import CAPS_CONFIG5, Q_HAT, SLO_BLOCKS, preset  # noqa: E402

pols = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [3, 4, 5]
tr = T.generate_traces([preset("wildchat", 0, 1_000_000)], exports=True)[0]
rows = [(0, pol, C, xi, Q_HAT, SLO_BLOCKS) for pol in pols for C in CAPS_CONFIG5 for xi in (4, 8, 16, 24)]
bt = T.prepare_batch([tr], rows)
for _ in range(2):
    bt.run()
    torch.cuda.synchronize()
    print(T.last_sim_stats(), flush=True)
