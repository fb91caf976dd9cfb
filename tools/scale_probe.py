"""Strong-scaling prediction measured on ONE B200: time every rank's share of the config-5 sweep
(sweep.plan_strong at world size N) alone on the GPU, with bench.py's pipelined step minus the
collectives (row a10's all_gather of 10^4 x 72 B and all_reduce of 1000 x 1025 x 8 B, tens of
microseconds over NVLink).  The max over ranks is the predicted N-GPU step time; every GPU of a
B200 box is identical and the shards share nothing.

    python tools/scale_probe.py [--worlds 1 2 4 8] [--steps 5] [--warmup 2]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--conversations", type=int, default=1_000_000)
    args = ap.parse_args()
    import bench
    from paper_2510_15152_b200.inputs import preset
    from paper_2510_15152_b200.sweep import Sweep, shard_cost
    rows, _, _ = bench.workload_global("config5")
    st = torch.cuda.current_stream()
    sA = torch.cuda.Stream(priority=-1)
    sBs = [torch.cuda.Stream() for _ in range(4)]  # as bench.py
    out = {}
    for world in args.worlds:
        per_rank = []
        for rank in range(world):
            sw = Sweep(rows, world, rank, lambda s: preset("wildchat", s, args.conversations), "cuda:0", comm=False)
            for _ in range(args.warmup):
                sw.step(st, sA, sBs, combine=False)
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(st)
            for _ in range(args.steps):
                sw.step(st, sA, sBs, combine=False)
            t1.record(st)
            torch.cuda.synchronize()
            ms = t0.elapsed_time(t1) / args.steps
            per_rank.append({"rank": rank, "ms": ms, "instances": len(sw.shards[rank]),
                             "traces": len(sw.my_traces), "requests": sw.requests_local,
                             "modelled_ms": shard_cost(rows, sw.shards[rank], owners=sw.owners, rank=rank)})
            del sw
            torch.cuda.empty_cache()
        step = max(r["ms"] for r in per_rank)
        req = sum(r["requests"] for r in per_rank)
        out[world] = {"predicted_step_ms": step, "requests_per_s": req / (step / 1000.0), "ranks": per_rank}
        print(json.dumps({"world": world, **out[world]}), flush=True)
    base = out[min(out)]["requests_per_s"] / min(out)
    print(json.dumps({"efficiency": {w: v["requests_per_s"] / (w * base) for w, v in out.items()}}), flush=True)


if __name__ == "__main__":
    main()
