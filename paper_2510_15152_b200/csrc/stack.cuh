// stack.cuh -- the closed-form "stack" engine (stack.cu).
#pragma once

#include "common.cuh"
#include "metrics.cuh"

namespace tlru {

// Workspace bytes of the stack engine for this batch (excluding the K3 tables).
tlru_status stack_workspace(const tlru_trace* traces, uint32_t nt, const tlru_instance* inst, uint32_t ni,
                            size_t* bytes);

// Interval of the s2_out launches of one call (first / last recorded on the call's stream).
struct OutTiming {
  cudaEvent_t first = nullptr, last = nullptr;
  uint32_t launches = 0;
};

// Runs the stack engine + K3 into `bout` / `results`.  `cv` continues carving the
// caller's workspace (checked against ws_bytes before any launch).
tlru_status stack_simulate(const tlru_trace* traces, uint32_t nt, const tlru_instance* inst, uint32_t ni,
                           const uint64_t* boffs, uint16_t* bout, tlru_result* results, Carver& cv,
                           const SegDev* segs_dev, uint32_t bins, uint32_t* hist, unsigned long long* clamped,
                           size_t ws_bytes, cudaStream_t st, unsigned* nkernels, cudaEvent_t ev_mid,
                           OutTiming* out_timing);

}  // namespace tlru
