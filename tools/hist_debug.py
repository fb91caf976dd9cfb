"""Debug: per-instance histograms of the stack engine vs bincount of the oracle's b."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
import paper_2510_15152_b200.tlru as T
from paper_2510_15152_b200.inputs import random_trace, preset

def upload(conv, q, a):
    c = torch.from_numpy(np.asarray(conv, np.uint32).view(np.int32).copy()).cuda()
    qq = torch.from_numpy(np.asarray(q, np.uint16).view(np.int16).copy()).cuda()
    aa = torch.from_numpy(np.asarray(a, np.uint16).view(np.int16).copy()).cuda()
    return T.trace_from_turns(c, qq, aa)

def run(name, conv, q, a, rows, HB=2048):
    tr = upload(conv, q, a)
    bt = T.simulate_batch([tr], rows, hist_bins=HB)
    torch.cuda.synchronize()
    h = bt.hist.view(len(rows), HB).cpu().numpy().view(np.uint32)
    bad = 0
    for i, r in enumerate(rows):
        o = O.replay(conv, q, a, r[1], r[2], r[3], r[4])
        assert np.array_equal(bt.b(i).astype(np.uint64), o.b)
        ref = np.bincount(o.b.astype(np.int64), minlength=HB)[:HB]
        if not np.array_equal(ref, h[i]):
            bad += 1
            d = np.flatnonzero(ref != h[i])
            print(name, "row", r, "bins differ", d[:10], "ref", ref[d[:10]], "got", h[i][d[:10]].astype(np.int64))
    print(name, "bad", bad, "of", len(rows), "maxhist", tr.max_history, "E", tr.num_events, flush=True)

T.set_sim_engine(T.ENGINE_STACK)
conv, q, a = random_trace(800, 5000, 80, q_max=6, a_max=8, locality=0.5)
rows = [(0, 0, C, 4, 2, 8) for C in (0, 3, 20, 90, 400)] + [(0, 1, C, 9, 2, 8) for C in (0, 3, 20, 90, 400)]
run("rand", conv, q, a, rows)
run("rand-lru0", conv, q, a, [(0, 0, 0, 4, 2, 8)])
run("rand-lru", conv, q, a, [(0, 0, 400, 4, 2, 8)])
p = preset("wildchat", 3, 3000)
ot = O.generate(p)
run("wild", ot.conv, ot.q, ot.a, [(0, pol, C, 16, 2, 16) for pol in (0, 1) for C in (0, 16, 64, 1024)])
