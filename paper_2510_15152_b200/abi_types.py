"""numpy mirrors of the result structs of include/tlru.h (no library loading here)."""
import numpy as np

RESULT_DTYPE = np.dtype([
    ("requests", "<u8"), ("sum_uncached", "<u8"), ("tel_blocks", "<u8"), ("slo_violations", "<u8"),
    ("evicted_trim", "<u8"), ("evicted_lru", "<u8"),
    ("p50", "<u4"), ("p90", "<u4"), ("p95", "<u4"), ("p99", "<u4"),
    ("max_uncached", "<u4"), ("max_occupancy", "<u4"),
])
assert RESULT_DTYPE.itemsize == 72

TAIL_DTYPE = np.dtype([
    ("n", "<u8"), ("tel_blocks", "<u8"), ("slo_violations", "<u8"), ("sum_b", "<u8"),
    ("p50", "<u4"), ("p90", "<u4"), ("p95", "<u4"), ("p99", "<u4"),
    ("max_b", "<u4"), ("n_clamped", "<u4"),
    ("tel_ms", "<f8"), ("p50_ms", "<f8"), ("p90_ms", "<f8"), ("p95_ms", "<f8"), ("p99_ms", "<f8"),
    ("mean_ms", "<f8"),
])
assert TAIL_DTYPE.itemsize == 104
