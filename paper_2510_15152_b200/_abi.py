"""ctypes view of include/tlru.h (argument marshalling only; every step runs in libtlru).

The product path has no CPU fallback: if ``libtlru.so`` is missing or fails to
load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtlru.so")
# measurement builds of the same sources with other compile-time tunables (tools/build_variant.py)
if os.environ.get("TLRU_LIB_VARIANT"):
    LIB_PATH = os.path.join(HERE, "variants", f"libtlru_{os.environ['TLRU_LIB_VARIANT']}.so")

TLRU_NONE = 0xFFFFFFFF
POLICY_LRU = 0
POLICY_TLRU = 1
POLICY_THRESHOLD = 2
POLICY_END_AWARE = 3
POLICY_LENGTH_AWARE = 4
POLICY_TAIL_BELADY = 5
POLICY_ET_LRU = 6
POLICY_TLRU_FORCED = 7
POLICY_BELADY_FORCED = 8
POLICY_ETLRU_FORCED = 9
ENGINE_REPLAY = 0
ENGINE_STACK = 1
ENGINE_MIXED = 2
TRACE_SYNTHETIC_TICKS = 1

STATUS = {0: "TLRU_OK", 1: "TLRU_EINVAL", 2: "TLRU_ERANGE", 3: "TLRU_ECUDA", 4: "TLRU_EUNSUPPORTED",
          5: "TLRU_ESTATE"}


class TlruError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status


class GenParams(ctypes.Structure):
    _fields_ = [
        ("seed", ctypes.c_uint64),
        ("num_conversations", ctypes.c_uint32),
        ("block_tokens", ctypes.c_uint32),
        ("birth_rate", ctypes.c_double),
        ("turn_rate", ctypes.c_double),
        ("death_rate", ctypes.c_double),
        ("prompt_mean_tokens", ctypes.c_double),
        ("prompt_sigma_ln", ctypes.c_double),
        ("response_mean_tokens", ctypes.c_double),
        ("response_sigma_ln", ctypes.c_double),
        ("prompt_min_tokens", ctypes.c_uint32),
        ("prompt_max_tokens", ctypes.c_uint32),
        ("response_min_tokens", ctypes.c_uint32),
        ("response_max_tokens", ctypes.c_uint32),
        ("max_history_blocks", ctypes.c_uint32),
        ("max_turns", ctypes.c_uint32),
    ]


class Trace(ctypes.Structure):
    _fields_ = [
        ("capacity", ctypes.c_uint64),
        ("num_events", ctypes.c_uint64),
        ("max_history", ctypes.c_uint32),
        ("num_conversations", ctypes.c_uint32),
        ("universe_blocks", ctypes.c_uint64),
        ("flags", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
        ("sim", ctypes.c_void_p),
        ("next", ctypes.c_void_p),
        ("conv", ctypes.c_void_p),
        ("prompt", ctypes.c_void_p),
        ("response", ctypes.c_void_p),
        ("time_ticks", ctypes.c_void_p),
        ("is_last", ctypes.c_void_p),
    ]


class Instance(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint32) for n in ("trace", "policy", "capacity", "xi", "q_hat", "slo", "threshold")]


from .abi_types import RESULT_DTYPE, TAIL_DTYPE  # noqa: E402  (pure-python mirrors of the header)


class SimStats(ctypes.Structure):
    _fields_ = [("chains", ctypes.c_uint64), ("segment_events", ctypes.c_uint64), ("spilled_chains", ctypes.c_uint64),
                ("failed_chains", ctypes.c_uint64), ("kernels", ctypes.c_uint32), ("state_entries", ctypes.c_uint32),
                ("engine", ctypes.c_uint32), ("reserved", ctypes.c_uint32), ("k2_ms", ctypes.c_float),
                ("k3_ms", ctypes.c_float), ("out_ms", ctypes.c_float), ("out_launches", ctypes.c_uint32)]


EXPORTS = (
    "tlru_last_error", "tlru_version", "tlru_launch_count", "tlru_trace_max_events", "tlru_gen_workspace_size", "tlru_count_events", "tlru_count_event_slots",
    "tlru_generate_traces", "tlru_upload_workspace_size", "tlru_trace_from_turns", "tlru_sim_workspace_size",
    "tlru_simulate_batch", "tlru_simulate_batch_ex", "tlru_set_sim_options", "tlru_set_sim_engine",
    "tlru_set_etlru_model", "tlru_last_sim_stats", "tlru_tail_workspace_size", "tlru_tail_metrics",
    "tlru_pool_workspace_size", "tlru_pool_histograms", "tlru_tail_from_histograms",
)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, u32, u64, sz = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_size_t
    P = ctypes.POINTER
    st = ctypes.c_int
    sigs = {
        "tlru_last_error": ([], ctypes.c_char_p),
        "tlru_version": ([], ctypes.c_char_p),
        "tlru_launch_count": ([], ctypes.c_uint64),
        "tlru_trace_max_events": ([P(GenParams), P(u64)], st),
        "tlru_gen_workspace_size": ([P(GenParams), u64, P(sz)], st),
        "tlru_count_events": ([P(GenParams), P(u64), vp, sz, vp], st),
        "tlru_count_event_slots": ([P(GenParams), P(u64), vp, sz, vp], st),
        "tlru_generate_traces": ([P(GenParams), u32, P(Trace), vp, sz, vp], st),
        "tlru_upload_workspace_size": ([u64, P(sz)], st),
        "tlru_trace_from_turns": ([vp, vp, vp, vp, u64, P(Trace), vp, sz, vp], st),
        "tlru_sim_workspace_size": ([P(Trace), u32, P(Instance), u32, P(sz)], st),
        "tlru_simulate_batch": ([P(Trace), u32, P(Instance), u32, vp, P(u64), vp, vp, sz, vp], st),
        "tlru_simulate_batch_ex": ([P(Trace), u32, P(Instance), u32, vp, P(u64), vp, vp, u32, vp, sz, vp], st),
        "tlru_set_sim_options": ([u32, u32], st),
        "tlru_set_sim_engine": ([u32], st),
        "tlru_set_etlru_model": ([ctypes.c_double, P(ctypes.c_double), u32], st),
        "tlru_last_sim_stats": ([P(SimStats)], st),
        "tlru_tail_workspace_size": ([u32, u32, P(sz)], st),
        "tlru_tail_metrics": ([vp, vp, u32, vp, vp, vp, ctypes.c_double, u32, vp, vp, sz, vp], st),
        "tlru_pool_workspace_size": ([u32, P(sz)], st),
        "tlru_pool_histograms": ([vp, u32, u32, P(u32), u32, vp, vp, sz, vp], st),
        "tlru_tail_from_histograms": ([vp, u32, u32, vp, vp, vp, ctypes.c_double, vp, vp], st),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    return L


lib = _load()


def check(status: int) -> None:
    if status != 0:
        raise TlruError(status, lib.tlru_last_error().decode())
