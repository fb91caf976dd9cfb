"""Python binding of libtlru (include/tlru.h) over torch device memory and streams.

Marshalling only: every step of the hot path (trace generation, simulation,
tail metrics) runs in the CUDA kernels of ``libtlru.so``; torch provides device
allocations and the current CUDA stream.  Names follow the C ABI.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _abi
from ._abi import (ENGINE_MIXED, ENGINE_REPLAY, ENGINE_STACK, POLICY_END_AWARE, POLICY_ET_LRU, POLICY_LENGTH_AWARE, POLICY_TLRU_FORCED, POLICY_BELADY_FORCED, POLICY_ETLRU_FORCED, POLICY_LRU, POLICY_TAIL_BELADY, POLICY_THRESHOLD, POLICY_TLRU, RESULT_DTYPE, TAIL_DTYPE, TLRU_NONE, GenParams, Instance, SimStats,
                   Trace, TlruError, check, lib)

__all__ = ["DeviceTrace", "generate_traces", "trace_from_turns", "simulate_batch", "tail_metrics", "last_sim_stats",
           "set_sim_options", "set_sim_engine", "set_etlru_model", "pool_histograms", "tail_from_histograms",
           "ENGINE_REPLAY", "ENGINE_STACK", "ENGINE_MIXED",
           "POLICY_LRU", "POLICY_TLRU", "POLICY_THRESHOLD", "POLICY_END_AWARE", "POLICY_LENGTH_AWARE", "POLICY_TAIL_BELADY", "POLICY_ET_LRU", "POLICY_TLRU_FORCED", "POLICY_BELADY_FORCED", "POLICY_ETLRU_FORCED", "TLRU_NONE", "TlruError", "RESULT_DTYPE", "TAIL_DTYPE", "version"]


def version() -> str:
    return lib.tlru_version().decode()


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


@dataclass
class DeviceTrace:
    """A trace resident in HBM: the 8-byte sim view, next links and the exports."""
    sim: torch.Tensor          # int64 [E]  (prev | J << 32 | L_after << 48)
    next: torch.Tensor         # int32 [E]  (uint32 bit pattern)
    conv: torch.Tensor | None = None
    prompt: torch.Tensor | None = None
    response: torch.Tensor | None = None
    time_ticks: torch.Tensor | None = None
    is_last: torch.Tensor | None = None
    num_events: int = 0
    max_history: int = 0
    num_conversations: int = 0
    universe_blocks: int = 0
    flags: int = 0

    def struct(self) -> Trace:
        t = Trace()
        t.capacity = self.sim.numel()
        t.num_events = self.num_events
        t.max_history = self.max_history
        t.num_conversations = self.num_conversations
        t.universe_blocks = self.universe_blocks
        t.flags = self.flags
        t.sim = self.sim.data_ptr()
        t.next = self.next.data_ptr()
        for name in ("conv", "prompt", "response", "time_ticks", "is_last"):
            v = getattr(self, name)
            setattr(t, name, v.data_ptr() if v is not None else None)
        return t

    # host-side decoded views (tests / reports)
    def prev_J_La(self):
        s = self.sim[: self.num_events].cpu().numpy().view(np.uint64)
        return ((s & 0xFFFFFFFF).astype(np.uint32), ((s >> 32) & 0xFFFF).astype(np.uint32),
                (s >> 48).astype(np.uint32))


def _gen_struct(p: dict) -> GenParams:
    g = GenParams()
    for k, _ in GenParams._fields_:
        setattr(g, k, p[k])
    return g


def _alloc_trace(E: int, device, exports: bool) -> DeviceTrace:
    n = max(E, 1)
    tr = DeviceTrace(sim=torch.empty(n, dtype=torch.int64, device=device),
                     next=torch.empty(n, dtype=torch.int32, device=device))
    if exports:
        tr.conv = torch.empty(n, dtype=torch.int32, device=device)
        tr.prompt = torch.empty(n, dtype=torch.uint16, device=device)
        tr.response = torch.empty(n, dtype=torch.uint16, device=device)
        tr.time_ticks = torch.empty(n, dtype=torch.int64, device=device)
        tr.is_last = torch.empty(n, dtype=torch.uint8, device=device)
    return tr


def generate_traces(params: list[dict], device="cuda", exports: bool = True, stream=None,
                    capacity: str = "slots") -> list[DeviceTrace]:
    """tlru_generate_traces for each params dict (fields of tlru_gen_params).

    capacity: "slots" (default) sizes the trace with tlru_count_event_slots, so every later
    regeneration into it takes one counting pass; "exact" with tlru_count_events (E entries:
    regenerations count twice); "bound" with tlru_trace_max_events (N * max_turns)."""
    out = []
    st = _stream(stream)
    for p in params:
        g = _gen_struct(p)
        sz = ctypes.c_size_t()
        E = ctypes.c_uint64()
        if capacity == "bound":
            check(lib.tlru_trace_max_events(ctypes.byref(g), ctypes.byref(E)))
        else:
            check(lib.tlru_gen_workspace_size(ctypes.byref(g), 0, ctypes.byref(sz)))
            ws = _workspace(sz.value, device)
            count = lib.tlru_count_event_slots if capacity == "slots" else lib.tlru_count_events
            check(count(ctypes.byref(g), ctypes.byref(E), _ptr(ws), sz.value, st))
        tr = _alloc_trace(E.value, device, exports)
        check(lib.tlru_gen_workspace_size(ctypes.byref(g), tr.sim.numel(), ctypes.byref(sz)))
        ws = _workspace(sz.value, device)
        ts = tr.struct()
        check(lib.tlru_generate_traces(ctypes.byref(g), 1, ctypes.byref(ts), _ptr(ws), sz.value, st))
        _read_back(tr, ts)
        out.append(tr)
    return out


def _read_back(tr: DeviceTrace, ts: Trace) -> None:
    tr.num_events, tr.max_history, tr.num_conversations = ts.num_events, ts.max_history, ts.num_conversations
    tr.universe_blocks, tr.flags = ts.universe_blocks, ts.flags


def trace_from_turns(conv: torch.Tensor, q: torch.Tensor, a: torch.Tensor, exports: bool = True,
                     stream=None, ticks: torch.Tensor | None = None) -> DeviceTrace:
    """tlru_trace_from_turns: conv (int32 holding uint32 ids), q, a (16-bit) device tensors in event order;
    ticks (int64 holding uint64 arrival times, non-decreasing) optional -- without them the trace's
    time_ticks are event indices and ET-LRU rejects it (TLRU_TRACE_SYNTHETIC_TICKS)."""
    assert conv.is_cuda and q.is_cuda and a.is_cuda
    if ticks is not None:
        assert ticks.is_cuda and ticks.dtype in (torch.int64, torch.uint64) and ticks.numel() == conv.numel()
        ticks = ticks.contiguous()
    E = conv.numel()
    conv = conv.contiguous()
    assert q.dtype in (torch.uint16, torch.int16) and a.dtype in (torch.uint16, torch.int16)
    q = q.contiguous()
    a = a.contiguous()
    tr = _alloc_trace(E, conv.device, exports)
    sz = ctypes.c_size_t()
    check(lib.tlru_upload_workspace_size(E, ctypes.byref(sz)))
    ws = _workspace(sz.value, conv.device)
    ts = tr.struct()
    check(lib.tlru_trace_from_turns(_ptr(conv), _ptr(q), _ptr(a), _ptr(ticks), E, ctypes.byref(ts), _ptr(ws),
                                    sz.value, _stream(stream)))
    _read_back(tr, ts)
    return tr


def instances_array(rows) -> "ctypes.Array":
    """rows: iterable of (trace, policy, capacity, xi, q_hat, slo[, threshold])."""
    rows = list(rows)
    arr = (Instance * max(len(rows), 1))()
    for i, r in enumerate(rows):
        for k, v in zip(("trace", "policy", "capacity", "xi", "q_hat", "slo", "threshold"), r):
            setattr(arr[i], k, int(v))
    return arr


@dataclass
class SimBatch:
    """Reusable launch state for one (traces, instances) batch: the workspace, b and results."""
    traces: list
    inst: "ctypes.Array"
    ni: int
    uncached: torch.Tensor
    offsets: np.ndarray
    results: torch.Tensor
    ws: torch.Tensor
    tstructs: "ctypes.Array" = field(default=None)
    hist: torch.Tensor | None = None   # [ni][hist_bins] int32 (uint32 counts) when requested
    hist_bins: int = 0

    def run(self, stream=None, check_state: bool = False) -> None:
        """Enqueue tlru_simulate_batch(_ex) on `stream` (asynchronous).  check_state=True
        synchronizes and raises if a replay chain overflowed even its global-memory state
        (failed_chains > 0: its b rows would be invalid; tlru.h)."""
        off = self.offsets.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
        check(lib.tlru_simulate_batch_ex(self.tstructs, len(self.traces), self.inst, self.ni, _ptr(self.uncached),
                                         off, _ptr(self.results), _ptr(self.hist), self.hist_bins, _ptr(self.ws),
                                         self.ws.numel(), _stream(stream)))
        if check_state:
            st = last_sim_stats()
            if st["failed_chains"]:
                raise TlruError(5, f"{st['failed_chains']} chains overflowed their state (TLRU_ESTATE)")

    def results_numpy(self) -> np.ndarray:
        return self.results.cpu().numpy().view(RESULT_DTYPE).copy()

    def b(self, i: int) -> np.ndarray:
        E = self.traces[int(self.inst[i].trace)].num_events
        o = int(self.offsets[i])
        return self.uncached[o:o + E].view(torch.int16).cpu().numpy().view(np.uint16)


def prepare_batch(traces: list[DeviceTrace], rows, align: int = 8, hist_bins: int = 0) -> SimBatch:
    """Allocate b (each instance's row starts at a multiple of `align` requests), results and workspace;
    with hist_bins > 0 also the per-instance histograms of b (tlru_simulate_batch_ex)."""
    rows = list(rows)
    ni = len(rows)
    inst = instances_array(rows)
    device = traces[0].sim.device if traces else "cuda"
    offsets = np.zeros(max(ni, 1), np.uint64)
    tot = 0
    for i, r in enumerate(rows):
        offsets[i] = tot
        E = traces[int(r[0])].num_events
        tot += (E + align - 1) // align * align
    tstructs = (Trace * max(len(traces), 1))(*[t.struct() for t in traces])
    sz = ctypes.c_size_t()
    check(lib.tlru_sim_workspace_size(tstructs, len(traces), inst, ni, ctypes.byref(sz)))
    return SimBatch(traces=traces, inst=inst, ni=ni,
                    uncached=torch.empty(max(tot, 8), dtype=torch.uint16, device=device),
                    offsets=offsets,
                    results=torch.empty(max(ni, 1) * RESULT_DTYPE.itemsize, dtype=torch.uint8, device=device),
                    ws=_workspace(sz.value, device), tstructs=tstructs,
                    hist=torch.empty(max(ni, 1) * hist_bins, dtype=torch.int32, device=device) if hist_bins else None,
                    hist_bins=int(hist_bins))


def simulate_batch(traces: list[DeviceTrace], rows, stream=None, hist_bins: int = 0) -> SimBatch:
    """tlru_simulate_batch: rows = [(trace, policy, capacity, xi, q_hat, slo[, threshold]), ...].
    Synchronizes and raises if a chain overflowed its state (failed_chains, tlru.h)."""
    batch = prepare_batch(traces, rows, hist_bins=hist_bins)
    batch.run(stream, check_state=True)
    return batch


def pool_histograms(hist: torch.Tensor, bins: int, pool, npool: int, pooled: torch.Tensor | None = None,
                    stream=None) -> torch.Tensor:
    """tlru_pool_histograms: pooled[pool[i]] += hist[i] (hist: [ni * bins] int32 of uint32 counts; pooled:
    [npool * bins] int64 of uint64 counts, allocated zeroed when None).  pool[i] = TLRU_NONE skips i."""
    pool = np.ascontiguousarray(np.asarray(pool, np.uint32))
    ni = pool.size
    if pooled is None:
        pooled = torch.zeros(max(npool, 1) * bins, dtype=torch.int64, device=hist.device)
    sz = ctypes.c_size_t()
    check(lib.tlru_pool_workspace_size(ni, ctypes.byref(sz)))
    ws = _workspace(sz.value, hist.device)
    check(lib.tlru_pool_histograms(_ptr(hist), ni, bins, pool.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), npool,
                                   _ptr(pooled), _ptr(ws), sz.value, _stream(stream)))
    return pooled


def tail_from_histograms(hist: torch.Tensor, bins: int, xi, xi_ms, slo, alpha: float, stream=None) -> torch.Tensor:
    """tlru_tail_from_histograms over [ns * bins] int64 (uint64) counts; returns a device uint8 tensor of
    ns TAIL_DTYPE records (asynchronous; `.cpu().numpy().view(TAIL_DTYPE)` to read)."""
    dev = hist.device
    ns = hist.numel() // bins
    xi_t = torch.as_tensor(np.asarray(xi, np.uint32).view(np.int32), device=dev)
    slo_t = torch.as_tensor(np.asarray(slo, np.uint32).view(np.int32), device=dev)
    xim = torch.as_tensor(np.asarray(xi_ms, np.float64), device=dev)
    out = torch.empty(max(ns, 1) * TAIL_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    check(lib.tlru_tail_from_histograms(_ptr(hist), ns, bins, _ptr(xi_t), _ptr(xim), _ptr(slo_t), float(alpha),
                                        _ptr(out), _stream(stream)))
    out.keepalive = (xi_t, slo_t, xim)  # the kernel reads them asynchronously
    return out


def set_sim_options(segment_events: int = 0, state_entries: int = 0) -> None:
    """tlru_set_sim_options (0 = automatic); results never depend on these."""
    check(lib.tlru_set_sim_options(segment_events, state_entries))


def set_etlru_model(mu_tick: float, ln_surv) -> None:
    """tlru_set_etlru_model: ET-LRU's belief decay mu per time tick (ticks are the trace's
    microsecond times) and ln P(Q >= k) for k = 0..K (Def. 1; Reading #27)."""
    import numpy as np
    tab = np.ascontiguousarray(ln_surv, dtype=np.float64)
    check(lib.tlru_set_etlru_model(float(mu_tick), tab.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                   tab.shape[0] - 1))


def set_sim_engine(engine: int) -> None:
    """tlru_set_sim_engine: ENGINE_REPLAY (Alg. 1 replay, K2) or ENGINE_STACK (closed form, default)."""
    check(lib.tlru_set_sim_engine(engine))


def last_sim_stats() -> dict:
    s = SimStats()
    check(lib.tlru_last_sim_stats(ctypes.byref(s)))
    return {k: getattr(s, k) for k, _ in SimStats._fields_}


def tail_metrics(b: torch.Tensor, seg_offsets, xi, xi_ms, slo, alpha: float, max_b: int, stream=None) -> np.ndarray:
    """tlru_tail_metrics over segments of a device uint16 tensor b; returns a TAIL_DTYPE array."""
    dev = b.device
    ns = len(seg_offsets) - 1
    off = torch.as_tensor(np.asarray(seg_offsets, np.uint64).view(np.int64), device=dev)
    xi_t = torch.as_tensor(np.asarray(xi, np.uint32).view(np.int32), device=dev)
    slo_t = torch.as_tensor(np.asarray(slo, np.uint32).view(np.int32), device=dev)
    xim = torch.as_tensor(np.asarray(xi_ms, np.float64), device=dev)
    out = torch.empty(max(ns, 1) * TAIL_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    sz = ctypes.c_size_t()
    check(lib.tlru_tail_workspace_size(ns, max_b, ctypes.byref(sz)))
    ws = _workspace(sz.value, dev)
    check(lib.tlru_tail_metrics(_ptr(b), _ptr(off), ns, _ptr(xi_t), _ptr(xim), _ptr(slo_t), float(alpha), max_b,
                                _ptr(out), _ptr(ws), sz.value, _stream(stream)))
    return out.cpu().numpy().view(TAIL_DTYPE)[:ns].copy()
