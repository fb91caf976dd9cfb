#!/usr/bin/env python
"""Benchmark of the T-LRU hot path (BASELINE.json metric: simulated requests/s + HBM roofline %).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--scaling strong|weak]

One step = the whole hot path of SURVEY 8(a) over the BASELINE config-5 sweep (configs[4]):
generate 10 WildChat-shaped traces of 10^6 conversations (a1-a3, K1), simulate 10^4 instances =
10 seeds x 25 capacities x 20 xi x {LRU, T-LRU} (a4-a8), per-instance tail metrics (a9, fused
into the engine), and (a10) the NCCL all_gather of the per-instance results plus the all_reduce
of the pooled (policy, C, xi) histograms over seeds, with pooled P50/P90/P95/P99, TEL and SLO.
Strong scaling (default): the same 10^4 instances are sharded over the N ranks at sub-trace
granularity (sweep.plan_strong); each rank regenerates only the traces its instances use.

`value` = requests simulated by all ranks / max-over-ranks device time per step.
`e2e` = the same metric through the public API from pinned host buffers: H2D of each trace's
(conv, q, a) turns, tlru_trace_from_turns, tlru_simulate_batch_ex, pooling, the collectives and
a D2H read of the result table and pooled metrics, all inside the timed region.
`--impl reference` times the CPU oracle (oracle/, test infrastructure) on a bounded sample of
the same workload on the host cores; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Algorithmic HBM bytes:
#  * replay engine (SURVEY 8(d) model): 8-byte event record read per request + 2-byte b written = 10 B/request;
ALGO_BYTES_PER_REQUEST = 10
#  * s2_out (the dominant kernel): 2-byte b written per request; 4-byte (L_before | J) read per event and
#    one 2-byte A_nf per (event, distinct D) read, shared by the instances of a group.
OUT_B_BYTES = 2
OUT_EVENT_BYTES = 4
OUT_ROW_BYTES = 2


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _clock_sampler_proc(index, go, stop, out, count):
    """Child process (no CUDA): polls NVML every 5 ms between `go` and `stop` (at least once);
    `count` tells the parent how many samples it has taken."""
    res = {"sm": [], "mx": 0, "reasons": 0, "error": None}
    try:
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(index)
        res["mx"] = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        go.wait()
        while True:
            res["sm"].append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            res["reasons"] |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
            count.value += 1
            if stop.is_set():
                break
            time.sleep(0.005)
    except Exception as ex:  # noqa: BLE001 -- report, never fail the bench
        res["error"] = repr(ex)
        count.value += 1
    out.put(res)


class ClockSampler:
    """SM clocks and throttle reasons sampled through NVML (the library nvidia-smi reads)
    every 5 ms while the timed region runs.  The sampler is a forked child process, so it
    keeps sampling while this process blocks in CUDA calls holding the GIL."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        import multiprocessing as mp
        ctx = mp.get_context("fork")
        self.go, self.stop, self.q = ctx.Event(), ctx.Event(), ctx.Queue()
        self.count = ctx.Value("i", 0)
        self.p = ctx.Process(target=_clock_sampler_proc, args=(index, self.go, self.stop, self.q, self.count),
                             daemon=True)
        self.p.start()  # NVML init happens before the timed region
        self.res = None

    def __enter__(self):
        self.go.set()
        t_end = time.time() + 10.0  # the sampler is polling before the timed region starts
        while self.count.value == 0 and time.time() < t_end and self.p.is_alive():
            time.sleep(0.001)
        return self

    def __exit__(self, *a):
        self.stop.set()
        try:
            self.res = self.q.get(timeout=10)
        except Exception as ex:  # noqa: BLE001
            self.res = {"sm": [], "mx": 0, "reasons": 0, "error": repr(ex)}
        self.p.join(timeout=5)

    def summary(self):
        r = self.res or {"sm": [], "mx": 0, "reasons": 0}
        out = {"sm_mhz": statistics.median(r["sm"]) if r["sm"] else None, "sm_max_mhz": r["mx"] or None,
               "reasons": sorted(n for n, bit in self.REASONS.items() if r["reasons"] & bit),
               "samples": len(r["sm"])}
        if r.get("error"):
            out["error"] = r["error"]
        return out


# ----------------------------------------------------------------------------- CPU oracle baseline
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_trace(seed: int, n_conv: int):
    """The oracle's own generation of one config-5 trace (untimed: the baseline times the replay loop)."""
    import oracle as O
    from paper_2510_15152_b200.inputs import preset
    return O.generate(preset("wildchat", seed, n_conv))


def cpu_replay_sample(tr, insts, threads: int, pin_core: int | None = None):
    """Replays `insts` = [(policy, C, xi)] of the config-5 grid on trace `tr` with the plain oracle
    (Alg. 1, oracle/tlru_oracle.c) plus its tail metrics, one instance per host thread; returns
    (requests, seconds).  pin_core: run on that one core (sched_setaffinity of this thread)."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle as O
    from paper_2510_15152_b200.inputs import ALPHA_MS, Q_HAT, SLO_BLOCKS

    def one(x):
        pol, C, xi = x
        r = O.replay(tr.conv, tr.q, tr.a, pol, C, xi, Q_HAT)
        O.tail(r.b, xi, ALPHA_MS * xi, SLO_BLOCKS, ALPHA_MS)
        return tr.E

    old = os.sched_getaffinity(0)
    try:
        if pin_core is not None:
            os.sched_setaffinity(0, {pin_core})
        t0 = time.perf_counter()
        if threads == 1:
            n = sum(one(x) for x in insts)
        else:
            with ThreadPoolExecutor(max_workers=threads) as ex:
                n = sum(ex.map(one, insts))
        dt = time.perf_counter() - t0
    finally:
        os.sched_setaffinity(0, old)
    return n, dt


def cpu_sample_instances(k: int):
    """k instances spread over the config-5 grid: capacities 16..4096, alternating LRU / T-LRU(xi)."""
    from paper_2510_15152_b200.inputs import CAPS_CONFIG5, XI_CONFIG5
    out = []
    for j in range(k):
        C = CAPS_CONFIG5[(j * 7) % len(CAPS_CONFIG5)]
        xi = XI_CONFIG5[(j * 3) % len(XI_CONFIG5)]
        out.append((j % 2, C, xi))
    return out


def cpu_oracle_baseline(n_conv: int, seed: int = 0):
    """the oracle as it stands on the GPU box's host cores -- one pinned core, then all
    cores (one instance per thread) -- timing the replay loop only (generation outside the timer)."""
    tr = oracle_trace(seed, n_conv)
    ncores = len(os.sched_getaffinity(0))
    core0 = min(os.sched_getaffinity(0))
    n1, dt1 = cpu_replay_sample(tr, [(0, 256, 16), (1, 1024, 16)], 1, pin_core=core0)
    insts = cpu_sample_instances(ncores)
    na, dta = cpu_replay_sample(tr, insts, ncores)
    return {
        "value": na / dta, "unit": "requests/s", "cores": ncores, "kind": "oracle",
        "sample": (f"config-5 seed {seed} trace ({n_conv} conversations, {tr.E} requests, oracle-generated outside "
                   f"the timer); replay loop + tail metrics of {len(insts)} instances spread over C = 16..4096, "
                   f"LRU / T-LRU, one per host thread on all {ncores} cores"),
        "single_core": {"value": n1 / dt1, "unit": "requests/s", "cores": 1, "pinned_core": core0,
                        "sample": "LRU C=256 and T-LRU C=1024 xi=16 on the same trace, one pinned core"},
        "cpu_model": cpu_model(), "nproc": os.cpu_count(),
    }


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle (test infrastructure) timed on the host cores, rank 0 only.
    Each step replays one instance per core of the config-5 grid on one oracle-generated trace."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    tr = oracle_trace(0, args.conversations)  # untimed
    ncores = len(os.sched_getaffinity(0))
    insts = cpu_sample_instances(ncores)
    times, n_req = [], 0
    for i in range(args.warmup + args.steps):
        n, dt = cpu_replay_sample(tr, insts, ncores)
        if i >= args.warmup:
            times.append(dt)
            n_req = n
    ms = 1000.0 * statistics.mean(times)
    value = n_req / (ms / 1000.0)
    sample = (f"config-5 seed 0 trace ({args.conversations} conversations, {tr.E} requests): replay loop + tail "
              f"metrics of {len(insts)} instances (C = 16..4096, LRU / T-LRU), one per thread on {ncores} cores")
    line = {"impl": "reference", "metric": "simulated requests/sec", "value": value, "unit": "requests/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u32",
            "data": "synthetic",
            "config": {"workload": "config5 sample (CPU oracle, see cpu_baseline.sample)", "requests_per_step": n_req},
            "cpu_baseline": {"value": value, "unit": "requests/s", "cores": ncores, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "requests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- ours
def workload_global(name: str):
    """(rows, n_traces, description) of the whole job: rows = (trace, policy, C, xi, Q_hat, slo[, T])
    with trace = seed index.  Strong scaling shards these rows over the ranks (sweep.plan_strong);
    weak scaling gives every rank all of them on its own seeds."""
    from paper_2510_15152_b200.inputs import CAPS_CONFIG4, CAPS_CONFIG5, Q_HAT, SEEDS_CONFIG5, SLO_BLOCKS, XI_BLOCKS
    from paper_2510_15152_b200.inputs import config5_rows
    n = SEEDS_CONFIG5
    if name == "spectrum":
        rows = [(t, pol, C, xi, Q_HAT, SLO_BLOCKS) for t in range(n) for pol in (3, 4, 5) for C in CAPS_CONFIG5
                for xi in (4, 8, 16, 24)]
        return rows, n, ("predictability spectrum (P:389-395, Thm 1): 10 seeds x 10^6-conversation traces x 25 "
                         "capacities x xi in {4, 8, 16, 24} x {End-Aware, Length-Aware T-LRU, Tail-Optimized Belady} "
                         "= 3000 instances (replay engine, burn-in segments verified by the fix-up)")
    if name == "etlru":
        rows = [(t, 6, C, xi, Q_HAT, SLO_BLOCKS) for t in range(n) for C in CAPS_CONFIG5 for xi in (4, 8, 16, 24)]
        return rows, n, ("ET-LRU (Def. 1 / Alg. 2, P:261-275): 10 seeds x 10^6-conversation traces x 25 capacities "
                         "x xi in {4, 8, 16, 24} = 1000 instances, belief mu = 1/90 s, the preset's prompt law")
    if name == "forced":
        rows = [(t, 7, C, xi, Q_HAT, SLO_BLOCKS) for t in range(n) for C in CAPS_CONFIG5 for xi in (4, 8, 16, 24)]
        return rows, n, ("T-LRU under forced caching (App. C): 10 seeds x 10^6-conversation traces x 25 capacities "
                         "x xi in {4, 8, 16, 24} = 1000 instances (replay engine)")
    if name == "etlru_forced":
        rows = [(t, 9, C, xi, Q_HAT, SLO_BLOCKS) for t in range(n) for C in CAPS_CONFIG5 for xi in (4, 8, 16, 24)]
        return rows, n, ("ET-LRU under forced caching (App. C, P:664-672): 10 seeds x 10^6-conversation traces x "
                         "25 capacities x xi in {4, 8, 16, 24} = 1000 instances, belief mu = 1/90 s, the preset's "
                         "prompt law")
    if name == "forced_belady":
        rows = [(t, 8, C, xi, Q_HAT, SLO_BLOCKS) for t in range(n) for C in CAPS_CONFIG5 for xi in (4, 8, 16, 24)]
        return rows, n, ("Tail-Optimized Belady under forced caching (App. C, P:657-662): 10 seeds x "
                         "10^6-conversation traces x 25 capacities x xi in {4, 8, 16, 24} = 1000 instances "
                         "(replay engine)")
    if name == "config5x3":
        return config5_rows(n, threshold_lru=True), n, (
            "config5 sweep with the paper's three policies: 10 seeds x 10^6-conversation traces x 25 capacities x "
            "20 xi x {LRU, T-LRU, Threshold-LRU (1024 tokens = 8 blocks)} = 1.5x10^4 instances")
    if name == "config4":
        rows = [(t, pol, C, xi, Q_HAT, SLO_BLOCKS) for t in range(4) for pol in (0, 1) for C in CAPS_CONFIG4
                for xi in XI_BLOCKS]
        return rows, 4, ("config4: 4 seeds x 10^6-conversation traces, C in {64..4096} x xi in {4..40} x "
                         "{LRU, T-LRU} = 384 instances")
    return config5_rows(n), n, (
        "config5 sweep (BASELINE configs[4]): 10 seeds x 10^6-conversation WildChat-shaped traces (generated each "
        "step) x 25 capacities (16..4096 blocks, geometric) x 20 xi (2..40 blocks) x {LRU, T-LRU} = 10^4 instances")


NEXT_FAMILIES = (  # (name, policies, xi values, what) -- DESIGN.md 6, bench --config <name> for the full workloads
    ("spectrum", (3, 4, 5), (4, 8, 16, 24), "End-Aware, Length-Aware T-LRU, Tail-Optimized Belady (P:389-395, Thm 1)"),
    ("threshold_lru", (2,), None, "Threshold-LRU, 1024 tokens = 8 blocks (P:307, P:322), stack engine"),
    ("forced", (7,), (4, 8, 16, 24), "T-LRU under forced caching (App. C)"),
    ("forced_belady", (8,), (4, 8, 16, 24), "Tail-Optimized Belady under forced caching (App. C, P:657-662)"),
    ("etlru", (6,), (4, 8, 16, 24), "ET-LRU (Def. 1 / Alg. 2), belief mu = 1/90 s, the preset's prompt law"),
    ("etlru_forced", (9,), (4, 8, 16, 24), "ET-LRU under forced caching (App. C, P:664-672)"),
)


def measure_next_rows(T, traces, HB, stream):
    """One batch per NEXT family over the resident config-5 traces (at N = 1 all ten: the same
    workloads as `bench.py --config <name>`): per trace 25 capacities x its xi values x its
    policies; one warm-up call, then one call timed with CUDA events on `stream`."""
    import torch

    from paper_2510_15152_b200.inputs import (CAPS_CONFIG5, Q_HAT, SLO_BLOCKS, THRESHOLD_BLOCKS, WILDCHAT,
                                              XI_CONFIG5, prompt_law_ln_surv)
    T.set_etlru_model(WILDCHAT["death_rate"] * 1e-6, prompt_law_ln_surv(WILDCHAT))
    out = {}
    for name, pols, xis, what in NEXT_FAMILIES:
        rows = [(t, pol, C, xi, Q_HAT, SLO_BLOCKS) + ((THRESHOLD_BLOCKS,) if pol == 2 else ())
                for t in range(len(traces)) for pol in pols for C in CAPS_CONFIG5 for xi in (xis or XI_CONFIG5)]
        bt = T.prepare_batch(list(traces), rows, hist_bins=HB)
        bt.run()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        bt.run()
        t1.record(stream)
        torch.cuda.synchronize()
        st = T.last_sim_stats()
        assert st["failed_chains"] == 0
        ms = t0.elapsed_time(t1)
        req = sum(traces[r[0]].num_events for r in rows)
        out[name] = {"value": req / (ms / 1000.0), "unit": "requests/s", "ms": ms, "instances": len(rows),
                     "requests": req, "what": what,
                     "engine": {0: "replay", 1: "stack", 2: "mixed"}.get(st["engine"], str(st["engine"])),
                     "spilled_chains": st["spilled_chains"],
                     "sample": f"rank 0's {len(traces)} config-5 traces (10^6 conversations each), resident in "
                               "HBM; one call of tlru_simulate_batch incl. tail metrics (no generation)"}
        del bt
        torch.cuda.empty_cache()
    return out


def run_ours(args, rank, world, local_rank):
    import ctypes

    import torch
    import torch.distributed as dist

    import paper_2510_15152_b200.tlru as T
    from paper_2510_15152_b200 import _abi
    from paper_2510_15152_b200.inputs import preset
    from paper_2510_15152_b200.sweep import Sweep, gather_results, shard_cost

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    rows_all, n_traces, wl_desc = workload_global(args.config)
    if args.segment_events:
        T.set_sim_options(args.segment_events, 0)
    n_total = len(rows_all)
    strong = args.scaling == "strong"
    if any(r[1] in (T.POLICY_ET_LRU, T.POLICY_ETLRU_FORCED) for r in rows_all):  # ET-LRU model: belief decay per µs tick, prompt law
        from paper_2510_15152_b200.inputs import WILDCHAT, prompt_law_ln_surv
        T.set_etlru_model(WILDCHAT["death_rate"] * 1e-6, prompt_law_ln_surv(WILDCHAT))

    # ---- setup (untimed): this rank's traces at their exact size, one batch per trace, pools
    sw = Sweep(rows_all, world, rank, lambda seed: preset(args.preset, seed, args.conversations), dev,
               scaling=args.scaling, backend="nccl")
    shards, traces, batches, ids_by_trace = sw.shards, sw.sim_traces, sw.batches, sw.ids_by_trace
    E_loc, RS, HB, npool = sw.requests_local, sw.RS, sw.HB, sw.npool
    # generation (compute-bound) on a higher-priority stream: its CTAs take SM slots as the
    # memory-bound simulation kernels' CTAs retire
    prio = int(os.environ.get("BENCH_GEN_PRIO", "-1"))
    sA = torch.cuda.Stream(device=dev, priority=prio)
    nsim = int(os.environ.get("BENCH_SIM_STREAMS", "4"))  # measured: 2 / 3 / 4 streams 18.5 / 18.39 / 18.34 ms
    sBs = [torch.cuda.Stream(device=dev) for _ in range(nsim)]

    def step():
        sw.step(stream, sA, sBs)

    def step_seq():
        """One stream, no overlap; returns the summed engine / K3 / s2_out device times of the step."""
        with torch.cuda.stream(stream):
            sw.pooled.zero_()
        for j in range(len(sw.held)):
            sw.produce(j, stream)  # generated here (owner) and / or broadcast (shared generation)
        k2 = k3 = out_ms = 0.0
        out_n = 0
        for j in range(len(batches)):
            sw.simulate(j, stream)  # a4-a9: simulation engine + K3, results, pooling
            st = T.last_sim_stats()
            k2 += st["k2_ms"]
            k3 += st["k3_ms"]
            out_ms += st["out_ms"]
            out_n += st["out_launches"]
        sw.combine(stream)
        return k2, k3, out_ms, out_n

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps: int, warmup: int):
        clk = ClockSampler(local_rank)  # sampler process + NVML init before the timed region
        for _ in range(warmup):
            fn()
        barrier()
        l0 = _abi.lib.tlru_launch_count()
        out = []
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with clk:
            barrier()
            t0.record(stream)
            for _ in range(steps):
                out.append(fn())
            t1.record(stream)
            barrier()
        return dict(ms=t0.elapsed_time(t1) / steps, out=out, launches=(_abi.lib.tlru_launch_count() - l0),
                    clocks=clk.summary())

    # ---- main arm: default (stack) engine, pipelined step; then the sequential step for engine times
    T.set_sim_engine(T.ENGINE_STACK)
    main = timed(step, args.steps, args.warmup)
    seq = timed(step_seq, max(2, args.steps // 2), 1)
    main["k2"] = statistics.mean(o[0] for o in seq["out"])
    main["k3"] = statistics.mean(o[1] for o in seq["out"])
    main["out_ms"] = statistics.mean(o[2] for o in seq["out"])
    main["out_n"] = seq["out"][-1][3]
    stats = T.last_sim_stats()
    assert stats["failed_chains"] == 0
    tab = sw.table.cpu().numpy().tobytes()
    ptails = sw.pooled_tails_numpy()
    step()
    torch.cuda.synchronize()
    assert sw.table.cpu().numpy().tobytes() == tab  # pipelined == sequential, byte for byte
    res = np.frombuffer(tab, dtype=_abi.RESULT_DTYPE)
    if strong or world == 1:
        assert np.all(res["requests"] > 0)
        # the pooled histograms hold every request of their pool's instances (all ranks reduced)
        preq = np.zeros(npool, np.uint64)
        np.add.at(preq, [sw.pidx[tuple(r[1:])] for r in sw.rows], res["requests"])
        assert np.array_equal(ptails["n"], preq)
    if world > 1 and strong:  # the host-side gather (duplicate / missing detection) agrees with the device one
        loc = sw.results_local.view(-1, RS)[: len(sw.local_ids)].cpu().numpy().copy().view(_abi.RESULT_DTYPE)
        host_table = gather_results(loc, sw.local_ids, n_total, device=dev)
        if rank == 0:
            assert host_table.tobytes() == tab

    # ---- replay engine (Alg. 1 request by request) on the first local trace: identical b bytes
    rep = None
    if not args.no_replay and stats["engine"] == T.ENGINE_STACK and batches:
        sub = [(0,) + tuple(rows_all[i][1:]) for i in ids_by_trace[0]]
        if args.replay_instances:
            sub = sub[:args.replay_instances]
        rbatch = T.prepare_batch(traces[:1], sub, hist_bins=HB)
        rbatch.uncached.zero_()
        T.set_sim_engine(T.ENGINE_REPLAY)
        r = timed(lambda: (rbatch.run(), T.last_sim_stats()["k2_ms"])[1], 1, 1)
        rst = T.last_sim_stats()
        T.set_sim_engine(T.ENGINE_STACK)
        nb = int(rbatch.offsets[len(sub) - 1]) + traces[0].num_events
        assert rbatch.results_numpy()[: len(sub)].tobytes() == \
            batches[0].results_numpy()[: len(sub)].tobytes(), "engines disagree (results)"
        assert torch.equal(rbatch.uncached[:nb], batches[0].uncached[:nb]), "engines disagree (b bytes)"
        assert torch.equal(rbatch.hist[: len(sub) * HB], batches[0].hist[: len(sub) * HB]), "engines disagree (hist)"
        rep = dict(r, k2=statistics.mean(r["out"]), requests=traces[0].num_events * len(sub), instances=len(sub),
                   stats=rst)
        del rbatch

    # ---- the paper's other policies on rank 0's traces, one call each,
    # timed on the device (the trace is already resident; generation is not in these figures).  Before the e2e
    # arm, whose upload without ticks rewrites the trace's time_ticks with event indices
    next_rows = None
    if args.config == "config5" and rank == 0 and not args.no_next and traces:
        next_rows = measure_next_rows(T, traces, HB, stream)

    # ---- e2e: the same step through the public API from pinned host buffers (H2D of each trace's
    # turns on stream A, upload + simulation + pooling on the simulation streams, the collectives),
    # the result table and the pooled metrics read back to the host
    need_ticks = any(r[1] in (T.POLICY_ET_LRU, T.POLICY_ETLRU_FORCED) for r in rows_all)  # ET-LRU beliefs read the event times
    host_turns, host_ticks = [], []
    for tr in traces:
        E = tr.num_events
        host_turns.append((tr.conv[:E].cpu().pin_memory(), tr.prompt[:E].view(torch.int16).cpu().pin_memory(),
                           tr.response[:E].view(torch.int16).cpu().pin_memory()))
        host_ticks.append(tr.time_ticks[:E].cpu().pin_memory() if need_ticks else None)
    dev_turns = [(torch.empty_like(c, device=dev), torch.empty_like(q, device=dev), torch.empty_like(a, device=dev))
                 for c, q, a in host_turns]
    dev_ticks = [torch.empty_like(h, device=dev) if h is not None else None for h in host_ticks]
    # the upload's outputs a user of this workload asks for: the simulation view and next links (and
    # the arrival times when ET-LRU rows read them; is_last when End-/Length-Aware rows do) -- not the
    # conv / prompt / response copies
    need_last = any(r[1] in (T.POLICY_END_AWARE, T.POLICY_LENGTH_AWARE) for r in rows_all)
    up_structs = []
    for ts in sw.sim_tstructs:
        u = _abi.Trace()
        ctypes.pointer(u)[0] = ts
        u.conv = u.prompt = u.response = None
        if not need_ticks:
            u.time_ticks = None
        if not need_last:
            u.is_last = None
        up_structs.append(u)
    up_ws = []
    for tr in traces:
        sz = ctypes.c_size_t()
        _abi.check(_abi.lib.tlru_upload_workspace_size(tr.num_events, ctypes.byref(sz)))
        up_ws.append(torch.empty(max(sz.value, 1), dtype=torch.uint8, device=dev))
    host_table = torch.empty(sw.table.numel(), dtype=torch.uint8).pin_memory()
    host_ptails = torch.empty(sw.pooled_tails.numel(), dtype=torch.uint8).pin_memory()
    h2d_bytes = sum(c.numel() * 4 + q.numel() * 2 + a.numel() * 2 for c, q, a in host_turns)
    h2d_bytes += sum(h.numel() * 8 for h in host_ticks if h is not None)
    d2h_bytes = host_table.numel() + host_ptails.numel()

    sU = torch.cuda.Stream(device=dev)  # uploads (each step ends with a host sync, so no cross-step hazard)

    simdone = [torch.cuda.Event() for _ in traces]  # trace j's simulation of the previous step
    d2h_done = [None]  # the previous step's result read-back (host waits on it one step later)

    def e2e_step():
        """One step from pinned host buffers.  Steps are pipelined one deep: step i+1's H2D copies
        and uploads start while step i's last simulations, collectives and D2H still run, and the
        host waits for step i's result read-back during step i+1 (the last one before the timer
        stops).  Hazards: trace j's upload waits for trace j's previous simulation (its arrays are
        rewritten); the simulations wait for this step's pool reset, which follows the previous
        step's collectives and D2H on `stream`."""
        with torch.cuda.stream(stream):
            sw.pooled.zero_()
        ev0 = torch.cuda.Event()
        ev0.record(stream)
        for sB in sBs:
            sB.wait_event(ev0)
        # every trace's H2D copies queued first on stream A (the previous step's uploads of these
        # buffers have returned: each upload synchronizes its stream); each upload (which reads
        # its validation flags back) runs on stream U, so the host waits only for that trace's
        # copy + upload while the simulation streams keep the GPU busy
        evh = []
        for j, ((hc, hq, ha), (dc, dq, da)) in enumerate(zip(host_turns, dev_turns)):
            with torch.cuda.stream(sA):
                dc.copy_(hc, non_blocking=True)
                dq.copy_(hq, non_blocking=True)
                da.copy_(ha, non_blocking=True)
                if dev_ticks[j] is not None:
                    dev_ticks[j].copy_(host_ticks[j], non_blocking=True)
            evh.append(torch.cuda.Event())
            evh[-1].record(sA)
        for j, ((dc, dq, da), tr, ts, w) in enumerate(zip(dev_turns, traces, up_structs, up_ws)):
            sB = sBs[j % len(sBs)]
            sU.wait_event(evh[j])
            sU.wait_event(simdone[j])
            _abi.check(_abi.lib.tlru_trace_from_turns(T._ptr(dc), T._ptr(dq), T._ptr(da), T._ptr(dev_ticks[j]),
                                                      tr.num_events, ctypes.byref(ts), T._ptr(w), w.numel(),
                                                      T._stream(sU)))
            ev = torch.cuda.Event()
            ev.record(sU)
            sB.wait_event(ev)
            sw.simulate(j, sB)
            simdone[j].record(sB)
        if d2h_done[0] is not None:
            d2h_done[0].synchronize()  # the previous step's results are on the host
        stream.wait_stream(sA)
        stream.wait_stream(sU)
        for sB in sBs:
            stream.wait_stream(sB)
        sw.combine(stream)
        host_table.copy_(sw.table, non_blocking=True)
        host_ptails.copy_(sw.pooled_tails, non_blocking=True)
        d2h_done[0] = torch.cuda.Event()
        d2h_done[0].record(stream)

    e2e = timed(e2e_step, args.steps, max(1, min(args.warmup, 2)))
    assert host_table.numpy().tobytes() == tab

    # ---- max over ranks; exact request totals over ranks
    loc = torch.tensor([main["ms"], e2e["ms"], main["k2"], main["k3"], rep["ms"] if rep else 0.0,
                        rep["k2"] if rep else 0.0, seq["ms"], main["out_ms"]], dtype=torch.float64, device=dev)
    req = torch.tensor([float(E_loc)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(loc, op=dist.ReduceOp.MAX)
        dist.all_reduce(req)
    ms, e2e_ms, k2, k3, rep_ms, rep_k2, seq_ms, out_ms = [float(x) for x in loc.tolist()]
    req_all = int(req.item())
    if rank != 0:
        return
    value = req_all / (ms / 1000.0)
    peak, peak_src = peaks()
    # dominant kernel s2_out (rank 0's launches): the irreducible HBM traffic is the 2-byte b it
    # writes per request; its per-event inputs (4 B L_before|J + 2 B A_nf per D) are listed beside
    out_n = max(int(main["out_n"]), 1)
    nd_per_trace = {}
    for j, ids in enumerate(ids_by_trace):
        for i in ids:
            r = rows_all[i]
            D = (r[3] - r[4]) if (r[1] == 1 and r[3] > r[4]) else 0
            Tk = r[6] if (r[1] == 2 and len(r) > 6) else 0  # Threshold-LRU rows: (D = 0, T)
            nd_per_trace.setdefault(j, set()).add((D, Tk))
    ev_tot = sum(traces[j].num_events for j in nd_per_trace)
    ev_rows = sum(traces[j].num_events * len(v) for j, v in nd_per_trace.items())
    b_bytes = OUT_B_BYTES * E_loc
    in_bytes = OUT_EVENT_BYTES * ev_tot + OUT_ROW_BYTES * ev_rows
    achieved = (b_bytes / out_n) / (out_ms / out_n / 1000.0) / 1e9 if out_ms > 0 else None
    achieved_in = ((b_bytes + in_bytes) / out_n) / (out_ms / out_n / 1000.0) / 1e9 if out_ms > 0 else None
    step_achieved = b_bytes / (ms / 1000.0) / 1e9  # rank 0's b bytes over the (max-over-ranks) step
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        t = json.load(open(tpath))
        if "s2_out_dram_bytes_per_request" in t:
            traffic = float(t["s2_out_dram_bytes_per_request"]) * E_loc / out_n
    shard_info = None
    if strong:
        shard_info = {"instances": [len(s_) for s_ in shards],
                      "traces": [len({int(rows_all[i][0]) for i in s_}) for s_ in shards],
                      "modelled_ms": [round(shard_cost(rows_all, s_, owners=sw.owners, rank=r_), 3)
                                      for r_, s_ in enumerate(shards)],
                      "generation": ("shared: each trace generated by the first rank using it and NCCL-broadcast "
                                     "(12 B/event) to the other ranks using it" if sw.owners else
                                     "each rank generates its traces")}
    line = {
        "metric": "simulated requests/sec", "value": value, "unit": "requests/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {
            "workload": wl_desc + ("" if args.preset == "wildchat" else
                                   f" -- traces from the {args.preset} preset (App. E, P:724) instead"),
            "instances": n_total if strong else n_total * world,
            "requests_per_step": req_all, "conversations": args.conversations,
            "parallelism": (f"dp{world}: the sweep's instances sharded over {world} GPU(s) at sub-trace granularity "
                            "(sweep.plan_strong; each trace generated once by its owner rank and broadcast to the "
                            "other ranks using it), NCCL all_gather of the results + all_reduce of the pooled "
                            "histograms" if strong else
                            f"dp{world}: every rank runs the whole sweep on its own seeds; NCCL all_gather / "
                            "all_reduce as in strong mode"),
            "shards": shard_info,
            "l2": f"inputs larger than L2: {2 * E_loc / 1e9:.1f} GB of b written per GPU-step (rank 0)",
            "engine": ("stack (closed form of Alg. 1 from the stack property, all capacities of a trace per pass; "
                       "bit-identical to the replay engine and the oracle); no dedup of identical instances")
            if stats["engine"] == T.ENGINE_STACK else
            "replay (Alg. 1 / Thm 1 request by request; aware / Belady / forced / ET-LRU: burn-in segments verified "
            "by the fix-up)" if stats["engine"] == T.ENGINE_REPLAY else "mixed (stack + replay engines)",
            "engine_ms": k2, "k3_ms": k3, "sequential_ms_per_step": seq_ms,
            "pooled": {"pools": npool, "bins": HB, "what": "per (policy, C, xi) over seeds: u64 b-histograms "
                       "summed per GPU (tlru_pool_histograms), all_reduce over GPUs, tlru_tail_from_histograms"},
            "pipelining": "traces generated on a high-priority stream A while earlier traces are simulated on "
                          "BENCH_SIM_STREAMS (4) alternating streams; engine_ms / k3_ms / roofline.launch_ms from the sequential "
                          "(single-stream) step",
        },
        "e2e": {"value": req_all / (e2e_ms / 1000.0), "unit": "requests/s", "h2d_bytes_per_step": h2d_bytes,
                "d2h_bytes_per_step": d2h_bytes, "ms_per_step": e2e_ms},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if achieved else None, "traffic": traffic,
                     "kernel": "s2_out_kernel (writer groups: b by TMA bulk stores; histogram groups: per-cell "
                               "histograms), per launch",
                     "launch_ms": out_ms / out_n, "launches_per_step": out_n,
                     "algorithmic_bytes_per_launch": b_bytes / out_n,
                     "algorithmic_bytes": f"{OUT_B_BYTES} B/request: the b row written (irreducible output)",
                     "with_inputs": {"achieved": achieved_in, "frac": achieved_in / peak if achieved_in else None,
                                     "bytes": f"+ {OUT_EVENT_BYTES} B/event + {OUT_ROW_BYTES} B/(event, D) read"},
                     "step_frac": step_achieved / peak, "step_achieved": step_achieved,
                     "step_note": "the 2 B/request b write over the whole pipelined step (generation, window "
                                  "sums, s2_out, pooling, collectives)",
                     "peak_source": peak_src,
                     "survey_model_10B": {"frac": ALGO_BYTES_PER_REQUEST * E_loc / (k2 / 1000.0) / 1e9 / peak,
                                          "note": "SURVEY 8(d)'s 8 B event read + 2 B write per request is the "
                                                  "replay engine's model; the stack engine reads per-event inputs "
                                                  "once per instance group, never per request, so this figure "
                                                  "exceeds 1 and does not apply"}},
        "gpu_launches": int(main["launches"] // max(args.steps, 1)),
        "clocks": main["clocks"],
    }
    if stats["engine"] != T.ENGINE_STACK:
        # replay-engine workload: the dominant kernels are K2's (sim_kernel + fix-up), SURVEY 8(d)'s model
        ach = ALGO_BYTES_PER_REQUEST * E_loc / (k2 / 1000.0) / 1e9
        line["roofline"] = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                            "traffic": None, "kernel": "sim_kernel<W, AWARE> + fix-up / etlru_seg_kernel (K2 replay), "
                                                       "per step (sequential stream)",
                            "launch_ms": k2, "algorithmic_bytes_per_launch": ALGO_BYTES_PER_REQUEST * E_loc,
                            "algorithmic_bytes": f"{ALGO_BYTES_PER_REQUEST} B/request (8 B event read + 2 B b "
                                                 "written)", "peak_source": peak_src,
                            "note": "issue/shared-memory-latency bound state machine, not HBM (DESIGN.md 6)"}
    if rep is not None:
        rep_achieved = ALGO_BYTES_PER_REQUEST * rep["requests"] / (rep_k2 / 1000.0) / 1e9
        line["replay_engine"] = {
            "value": rep["requests"] / (rep_k2 / 1000.0), "unit": "requests/s (K2 kernels only)",
            "instances": rep["instances"], "k2_ms": rep_k2, "ms_per_call": rep_ms,
            "segment_events": rep["stats"]["segment_events"], "spilled_chains": rep["stats"]["spilled_chains"],
            "roofline": {"bound": "hbm", "achieved": rep_achieved, "peak": peak, "unit": "GB/s",
                         "frac": rep_achieved / peak, "kernel": "sim_kernel<W> (K2 replay)"},
            "note": "Alg. 1 replayed request by request (one lane per instance) on the first trace's instances; "
                    "b bytes, histograms and results identical to the stack engine"}
    if next_rows is not None:
        for v in next_rows.values():
            v["roofline_10B"] = {"achieved": ALGO_BYTES_PER_REQUEST * v["value"] / 1e9, "peak": peak, "unit": "GB/s",
                                 "frac": ALGO_BYTES_PER_REQUEST * v["value"] / 1e9 / peak}
        line["next_rows"] = next_rows
    if not args.no_cpu_baseline and world == 1:  # the CPU oracle baseline: rank 0 at N = 1 only
        line["cpu_baseline"] = cpu_oracle_baseline(args.conversations)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--conversations", type=int, default=1_000_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-replay", action="store_true", help="skip timing the replay engine")
    ap.add_argument("--no-next", action="store_true", help="skip the NEXT-row policy measurements")
    ap.add_argument("--replay-instances", type=int, default=0, help="limit the replay-engine sample (0 = all of seed 0)")
    ap.add_argument("--config", choices=("config5", "config5x3", "spectrum", "etlru", "forced", "forced_belady",
                                         "etlru_forced", "config4"),
                    default="config5")
    ap.add_argument("--preset", choices=("wildchat", "sharegpt"), default="wildchat",
                    help="synthetic trace model: WildChat-shaped (BASELINE) or App. E's ShareGPT-shaped")
    ap.add_argument("--segment-events", type=int, default=0,
                    help="replay-engine segment length (tlru_set_sim_options; 0 = automatic)")
    ap.add_argument("--scaling", choices=("strong", "weak"), default="strong",
                    help="strong: the one sweep sharded over the ranks (default); weak: every rank its own seeds")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch.distributed as dist
    if world > 1:
        import torch
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
