"""Multi-GPU sweep plumbing: instances are independent, so they are sharded
across ranks with no data-path collective; the only exchange is one all_gather of the
72-byte per-instance results (row a10).  One process per GPU, torch.distributed (NCCL on
GPUs, gloo in the CPU tests).

The instance -> rank assignment is a pure function of (instance list, world size), and the
gathered table is re-ordered by global instance id, so the bytes rank 0 ends up with are the
same for any world size.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .abi_types import RESULT_DTYPE


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
