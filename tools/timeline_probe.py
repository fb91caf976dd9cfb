"""GPU busy fraction of the pipelined config-5 step: torch.profiler (CUPTI activity) records every
kernel's [start, end) over a few steps; the union of the intervals against the step span shows
whether the GPU ever idles between the host-orchestrated launches (python tools/timeline_probe.py)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    from paper_2510_15152_b200.inputs import preset
    from paper_2510_15152_b200.sweep import Sweep
    rows, _, _ = bench.workload_global("config5")
    st = torch.cuda.current_stream()
    sA = torch.cuda.Stream(priority=-1)
    sBs = [torch.cuda.Stream() for _ in range(4)]
    sw = Sweep(rows, 1, 0, lambda s: preset("wildchat", s, 1_000_000), "cuda:0")
    for _ in range(3):
        sw.step(st, sA, sBs)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            sw.step(st, sA, sBs)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.end > e.time_range.start]
    iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
    t0, t1 = iv[0][0], max(e[1] for e in iv)
    busy, cur_s, cur_e = 0.0, None, None
    gaps = []
    for s, e, n in iv:
        if cur_s is None:
            cur_s, cur_e = s, e
        elif s > cur_e:
            busy += cur_e - cur_s
            gaps.append((s - cur_e, n))
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    busy += cur_e - cur_s
    gaps.sort(reverse=True)
    print(json.dumps({"span_us": t1 - t0, "busy_us": busy, "busy_frac": busy / (t1 - t0), "kernels": len(iv),
                      "largest_gaps_us": [(round(g, 1), n[:40]) for g, n in gaps[:8]],
                      "gap_total_us": sum(g for g, _ in gaps)}))


if __name__ == "__main__":
    main()
