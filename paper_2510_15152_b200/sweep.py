"""Multi-GPU sweep: instances are independent, so they are sharded
across ranks with no data-path collective; the exchange is one all_gather of the 72-byte
per-instance results and one all_reduce of the pooled b-histograms.  One process per GPU,
torch.distributed (NCCL on GPUs; gloo -- staged through host memory -- in the tests, where two
processes share one GPU or have none).

The instance -> rank assignment (plan_strong) is a pure function of (instance list, world size),
and the gathered table is re-ordered by global instance id, so the bytes every rank ends up with
are the same for any world size.  `Sweep` is the per-rank driver bench.py times and the tests run.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .abi_types import RESULT_DTYPE, TAIL_DTYPE


def instance_cost(rows, trace_events) -> np.ndarray:
    """Relative cost of each instance: its trace's length (the stack engine's per-instance
    work is one pass over the trace's events)."""
    return np.array([float(trace_events[r[0]]) for r in rows], dtype=np.float64)


def shard_instances(rows, world: int, trace_events=None) -> list[list[int]]:
    """Deterministic LPT partition of instance indices into `world` shards.

    Instances of the same trace are kept together where possible (each rank generates
    the traces its instances use): whole traces are assigned largest-first to the least
    loaded rank; ties break by trace index, then rank."""
    if world < 1:
        raise ValueError("world must be >= 1")
    rows = list(rows)
    by_trace: dict[int, list[int]] = {}
    for i, r in enumerate(rows):
        by_trace.setdefault(int(r[0]), []).append(i)
    ev = trace_events or {}
    work = sorted(by_trace.items(), key=lambda kv: (-(len(kv[1]) * float(ev.get(kv[0], 1))), kv[0]))
    load = [0.0] * world
    shards: list[list[int]] = [[] for _ in range(world)]
    for t, ids in work:
        k = min(range(world), key=lambda j: (load[j], j))
        shards[k].extend(ids)
        load[k] += len(ids) * float(ev.get(t, 1))
    for s in shards:
        s.sort()
    return shards


# ----------------------------------------------------------------------------- strong scaling
# Cost model of the stack engine per trace pass, in ms for a trace of E_REF events (measured on one
# B200 at config 5, profiles/r01_launches_head.csv): generating the trace (K1),
# the per-trace stack kernels (s1, totals, count tables, finalize, s3), the per-distinct-D window
# sums (s2_win + s2_warm) and the per-instance output kernel (s2_out: b rows + histograms).
E_REF = 2.5e6
COST_TRACE_GEN_MS = 0.50
COST_TRACE_PASS_MS = 0.10
COST_PER_D_MS = 0.022
COST_PER_INSTANCE_MS = 0.00088  # round 2: s2_out 0.88 ms per 1000 instances (TMA writer groups)
# replay-engine policies (End-/Length-Aware, Belady, ET-LRU, forced): per-instance replay cost
COST_REPLAY_INSTANCE_MS = 0.40


def row_d_key(r) -> int:
    """The stack engine's row key of an instance (stack.cu make_stack_plan): D = max(xi - Q_hat, 0) for
    T-LRU, 0 for LRU, T << 32 for Threshold-LRU; replay-only policies sort after every stack key."""
    t, pol, C, xi, qh = (int(x) for x in r[:5])
    if pol == 2:
        return int(r[6]) << 32 if len(r) > 6 else 0
    if pol == 1:
        return max(xi - qh, 0)
    if pol == 0:
        return 0
    return (1 << 48) + pol


def plan_strong(rows, world: int, trace_events=None) -> list[list[int]]:
    """Strong-scaling shards of one sweep: a pure function of (rows, world, trace_events).

    Instances are ordered by (trace, D key, C, index) -- the order the stack engine groups them in --
    and cut into `world` contiguous shards minimising the largest modelled shard time (bisection on
    the bottleneck with a greedy left-to-right fill, exact for this monotone cost).  A shard pays
    COST_TRACE_* once for every trace it touches (each rank regenerates its traces locally from the
    seed: no broadcast), COST_PER_D_MS for every (trace, D) it touches and the
    per-instance cost of each instance, all scaled by the trace's events.  Cutting inside a trace
    (sub-trace granularity) is what lets 10 traces spread over 8 GPUs without the 62.5% cap of
    whole-trace sharding."""
    if world < 1:
        raise ValueError("world must be >= 1")
    rows = list(rows)
    ev = trace_events or {}
    order = sorted(range(len(rows)), key=lambda i: (int(rows[i][0]), row_d_key(rows[i]), int(rows[i][2]), i))
    keys = [(int(rows[i][0]), row_d_key(rows[i])) for i in order]
    scale = [float(ev.get(int(rows[i][0]), E_REF)) / E_REF for i in order]
    inst_c = [scale[k] * (COST_PER_INSTANCE_MS if rows[i][1] <= 2 else COST_REPLAY_INSTANCE_MS)
              for k, i in enumerate(order)]

    def fill(B):
        """Greedy left-to-right: shard boundaries with every shard's cost <= B (None if an item alone exceeds B)."""
        cuts, cost, seen_t, seen_d = [0], 0.0, set(), set()
        for k in range(len(order)):
            t, d = keys[k]
            add = inst_c[k]
            if t not in seen_t:
                add += scale[k] * (COST_TRACE_GEN_MS + COST_TRACE_PASS_MS)
            if (t, d) not in seen_d and d < (1 << 48):
                add += scale[k] * COST_PER_D_MS
            if cost + add > B and k > cuts[-1]:
                cuts.append(k)
                cost, seen_t, seen_d = 0.0, set(), set()
                add = inst_c[k] + scale[k] * (COST_TRACE_GEN_MS + COST_TRACE_PASS_MS)
                add += scale[k] * COST_PER_D_MS if d < (1 << 48) else 0.0
            if add > B:
                return None
            cost += add
            seen_t.add(t)
            seen_d.add((t, d))
        return cuts

    lo, hi = 0.0, sum(inst_c) + sum(scale) * (COST_TRACE_GEN_MS + COST_TRACE_PASS_MS + COST_PER_D_MS) + 1.0
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        c = fill(mid)
        if c is not None and len(c) <= world:
            hi = mid
        else:
            lo = mid
    cuts = fill(hi) + [len(order)]
    shards = [sorted(order[cuts[k]:cuts[k + 1]]) for k in range(len(cuts) - 1)]
    return shards + [[] for _ in range(world - len(shards))]


def shard_cost(rows, ids, trace_events=None) -> float:
    """Modelled time (ms) of one shard under plan_strong's cost model."""
    ev = trace_events or {}
    tr, ds, c = set(), set(), 0.0
    for i in ids:
        r = rows[i]
        sc = float(ev.get(int(r[0]), E_REF)) / E_REF
        c += sc * (COST_PER_INSTANCE_MS if r[1] <= 2 else COST_REPLAY_INSTANCE_MS)
        if int(r[0]) not in tr:
            tr.add(int(r[0]))
            c += sc * (COST_TRACE_GEN_MS + COST_TRACE_PASS_MS)
        k = (int(r[0]), row_d_key(r))
        if k not in ds and k[1] < (1 << 48):
            ds.add(k)
            c += sc * COST_PER_D_MS
    return c


def gather_results(local: np.ndarray, local_ids, n_total: int, device=None) -> np.ndarray | None:
    """all_gather the RESULT_DTYPE rows of every rank; rank 0 returns the full table ordered
    by global instance id, other ranks return None."""
    world = dist.get_world_size()
    rank = dist.get_rank()
    ids = np.asarray(local_ids, dtype=np.int64)
    n_local = torch.tensor([ids.size], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(sizes, n_local)
    nmax = int(max(int(s.item()) for s in sizes))
    rec = RESULT_DTYPE.itemsize
    buf = np.zeros((nmax, rec), np.uint8)
    buf[: ids.size] = np.ascontiguousarray(local).view(np.uint8).reshape(ids.size, rec)
    idbuf = np.full(nmax, -1, np.int64)
    idbuf[: ids.size] = ids
    t_res = torch.from_numpy(buf.reshape(-1)).to(device) if device is not None else torch.from_numpy(buf.reshape(-1))
    t_ids = torch.from_numpy(idbuf).to(device) if device is not None else torch.from_numpy(idbuf)
    out_res = torch.empty(world * t_res.numel(), dtype=torch.uint8, device=t_res.device)
    out_ids = torch.empty(world * nmax, dtype=torch.int64, device=t_ids.device)
    dist.all_gather_into_tensor(out_res, t_res)
    dist.all_gather_into_tensor(out_ids, t_ids)
    if rank != 0:
        return None
    all_ids = out_ids.cpu().numpy()
    all_res = out_res.cpu().numpy().reshape(world * nmax, rec)
    table = np.zeros((n_total, rec), np.uint8)
    seen = np.zeros(n_total, bool)
    for k in np.flatnonzero(all_ids >= 0):
        g = int(all_ids[k])
        if seen[g]:
            raise RuntimeError(f"instance {g} reported by two ranks")
        table[g] = all_res[k]
        seen[g] = True
    if not seen.all():
        raise RuntimeError(f"{int((~seen).sum())} instances missing from the gather")
    return table.reshape(-1).view(RESULT_DTYPE)


# ----------------------------------------------------------------------------- the per-rank driver
class Sweep:
    """One rank's share of a sweep (rows = (trace, policy, C, xi, Q_hat, slo[, T]) with trace = seed
    index): its traces generated on `device`, one simulation batch per trace (b rows, results and
    per-instance histograms), the pools (one per (policy, C, xi, ...) configuration over seeds) and
    the combination with the other ranks.

    scaling="strong": the rows are sharded over the ranks by plan_strong; "weak": every rank runs
    all rows on its own seeds (trace t of rank r = seed n_traces * r + t).  `params_of(seed)` gives
    the tlru_gen_params dict of a seed.  Every step of the method runs in libtlru's kernels; this
    class only sequences calls, streams and collectives."""

    def __init__(self, rows, world: int, rank: int, params_of, device, scaling: str = "strong",
                 backend: str = "nccl", hist_bins: int | None = None):
        import ctypes

        from . import _abi
        from . import tlru as T
        self.T, self._abi, self._ct = T, _abi, ctypes
        self.rows = [tuple(int(x) for x in r) for r in rows]
        self.world, self.rank, self.device = world, rank, torch.device(device)
        self.strong = scaling == "strong"
        self.host_staged = backend != "nccl"
        n_total = len(self.rows)
        self.n_total = n_total
        self.n_traces = max((r[0] for r in self.rows), default=-1) + 1
        self.shards = plan_strong(self.rows, world) if self.strong else [list(range(n_total))] * world
        mine = self.shards[rank]
        seed_base = 0 if self.strong else self.n_traces * rank
        self.my_traces = sorted({self.rows[i][0] for i in mine})
        self.params = [params_of(seed_base + t) for t in self.my_traces]
        self.HB = hist_bins or (int(self.params[0]["max_history_blocks"]) + 1 if self.params else 1025)
        self.traces = T.generate_traces(self.params, device=self.device, exports=True)
        self.ids_by_trace = [[i for i in mine if self.rows[i][0] == t] for t in self.my_traces]
        self.local_ids = [i for ids in self.ids_by_trace for i in ids]
        self.batches = [T.prepare_batch([self.traces[j]], [(0,) + self.rows[i][1:] for i in ids], hist_bins=self.HB)
                        for j, ids in enumerate(self.ids_by_trace)]
        for bt in self.batches:
            bt.uncached.zero_()  # row padding stays 0, so b buffers compare byte for byte
        self.requests_local = sum(self.traces[j].num_events * len(ids) for j, ids in enumerate(self.ids_by_trace))
        RS = RESULT_DTYPE.itemsize
        self.RS = RS
        self.nmax = max(max(len(s_) for s_ in self.shards), 1)
        self.results_local = torch.zeros(self.nmax * RS, dtype=torch.uint8, device=self.device)
        self.slices, o = [], 0
        for ids in self.ids_by_trace:
            self.slices.append(slice(o * RS, (o + len(ids)) * RS))
            o += len(ids)
        # pools: one per configuration over the seeds
        self.pool_keys = sorted({r[1:] for r in self.rows})
        self.pidx = {k: n for n, k in enumerate(self.pool_keys)}
        self.npool = len(self.pool_keys)
        self.pool_maps = [np.array([self.pidx[self.rows[i][1:]] for i in ids], np.uint32) for ids in self.ids_by_trace]
        self.pool_ws = []
        for pm in self.pool_maps:
            sz = ctypes.c_size_t()
            _abi.check(_abi.lib.tlru_pool_workspace_size(pm.size, ctypes.byref(sz)))
            self.pool_ws.append(torch.empty(max(sz.value, 1), dtype=torch.uint8, device=self.device))
        self.pooled = torch.zeros(self.npool * self.HB, dtype=torch.int64, device=self.device)
        self.pxi = torch.tensor([k[2] for k in self.pool_keys], dtype=torch.int32, device=self.device)
        self.pslo = torch.tensor([k[4] for k in self.pool_keys], dtype=torch.int32, device=self.device)
        from .inputs import ALPHA_MS
        self.alpha = ALPHA_MS  # ms per block (DESIGN.md Reading #14)
        self.pxim = self.pxi.to(torch.float64) * self.alpha
        self.pooled_tails = torch.empty(self.npool * TAIL_DTYPE.itemsize, dtype=torch.uint8, device=self.device)
        # gather: every rank's padded result rows -> the table ordered by global instance id
        self.table = torch.zeros(n_total * RS, dtype=torch.uint8, device=self.device)
        nranks = world if self.strong else 1
        all_ids = np.full(nranks * self.nmax, -1, np.int64)
        for r_ in range(nranks):
            s_ = self.shards[r_]
            ids_r = [i for t in sorted({self.rows[i][0] for i in s_}) for i in s_ if self.rows[i][0] == t]
            all_ids[r_ * self.nmax: r_ * self.nmax + len(ids_r)] = ids_r
        self.gpos = torch.from_numpy(np.flatnonzero(all_ids >= 0)).to(self.device)
        self.gdst = torch.from_numpy(all_ids[all_ids >= 0]).to(self.device)
        self.gathered = (torch.empty(world * self.nmax * RS, dtype=torch.uint8, device=self.device)
                         if (world > 1 and self.strong) else None)
        self.gstructs = [T._gen_struct(p) for p in self.params]
        self.gws = []
        for g, tr in zip(self.gstructs, self.traces):
            sz = ctypes.c_size_t()
            _abi.check(_abi.lib.tlru_gen_workspace_size(ctypes.byref(g), tr.sim.numel(), ctypes.byref(sz)))
            self.gws.append(torch.empty(max(sz.value, 1), dtype=torch.uint8, device=self.device))
        self.tstructs = [tr.struct() for tr in self.traces]

    # -- the steps of one sweep pass
    def gen(self, j: int, stream) -> None:
        """a1-a3: K1 regenerates local trace j in place (deterministic from the seed)."""
        T, A = self.T, self._abi
        A.check(A.lib.tlru_generate_traces(self._ct.byref(self.gstructs[j]), 1, self._ct.byref(self.tstructs[j]),
                                           T._ptr(self.gws[j]), self.gws[j].numel(), T._stream(stream)))

    def simulate(self, j: int, stream) -> None:
        """a4-a9 on batch j, its results into the local table, its histograms into the pools."""
        T, A, bt, pm = self.T, self._abi, self.batches[j], self.pool_maps[j]
        bt.run(stream)
        with torch.cuda.stream(stream):
            self.results_local[self.slices[j]].copy_(bt.results[: bt.ni * self.RS])
        A.check(A.lib.tlru_pool_histograms(T._ptr(bt.hist), bt.ni, self.HB,
                                           pm.ctypes.data_as(self._ct.POINTER(self._ct.c_uint32)), self.npool,
                                           T._ptr(self.pooled), T._ptr(self.pool_ws[j]), self.pool_ws[j].numel(),
                                           T._stream(stream)))

    def combine(self, stream) -> None:
        """a10: all_gather of the per-instance results, all_reduce (sum) of the pooled histograms, the
        table reassembled by global instance id, pooled tail metrics -- on `stream`."""
        import torch.distributed as dist
        T, A, RS = self.T, self._abi, self.RS
        with torch.cuda.stream(stream):
            rs = self.results_local.view(-1, RS)
            if self.world > 1:
                if self.host_staged:  # gloo: collectives on host copies
                    g = torch.empty(self.world * self.nmax * RS, dtype=torch.uint8)
                    pooled = self.pooled.cpu()
                    if self.gathered is not None:
                        dist.all_gather_into_tensor(g, self.results_local.cpu())
                        self.gathered.copy_(g)
                    dist.all_reduce(pooled)
                    self.pooled.copy_(pooled)
                else:
                    if self.gathered is not None:
                        dist.all_gather_into_tensor(self.gathered, self.results_local)
                    dist.all_reduce(self.pooled)
                if self.gathered is not None:
                    rs = self.gathered.view(-1, RS)
            self.table.view(-1, RS).index_copy_(0, self.gdst, rs.index_select(0, self.gpos))
        A.check(A.lib.tlru_tail_from_histograms(T._ptr(self.pooled), self.npool, self.HB, T._ptr(self.pxi),
                                                T._ptr(self.pxim), T._ptr(self.pslo), self.alpha,
                                                T._ptr(self.pooled_tails), T._stream(stream)))

    def step(self, stream, gen_stream=None, sim_streams=None, combine: bool = True) -> None:
        """One pass: pipelined when gen_stream / sim_streams are given (trace j+1 generated on the
        generation stream while traces are simulated on alternating simulation streams), else
        sequential on `stream`.  combine=False skips row a10 (tools/scale_probe.py times one rank's
        share alone on one GPU)."""
        with torch.cuda.stream(stream):
            self.pooled.zero_()
        if gen_stream is None:
            for j in range(len(self.batches)):
                self.gen(j, stream)
            for j in range(len(self.batches)):
                self.simulate(j, stream)
            if combine:
                self.combine(stream)
            return
        ev0 = torch.cuda.Event()
        ev0.record(stream)
        gen_stream.wait_event(ev0)
        for sB in sim_streams:
            sB.wait_event(ev0)
        for j in range(len(self.batches)):
            sB = sim_streams[j % len(sim_streams)]
            self.gen(j, gen_stream)
            ev = torch.cuda.Event()
            ev.record(gen_stream)
            sB.wait_event(ev)
            self.simulate(j, sB)
        stream.wait_stream(gen_stream)
        for sB in sim_streams:
            stream.wait_stream(sB)
        if combine:
            self.combine(stream)

    # -- host views (tests / reports; synchronize)
    def table_numpy(self) -> np.ndarray:
        return self.table.cpu().numpy().view(RESULT_DTYPE).copy()

    def pooled_tails_numpy(self) -> np.ndarray:
        return self.pooled_tails.cpu().numpy().view(TAIL_DTYPE).copy()
