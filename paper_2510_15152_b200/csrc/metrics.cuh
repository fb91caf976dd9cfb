// metrics.cuh -- K3: segmented histogram of per-request uncached blocks b and the
// tail metrics derived from it (Eq. 1-3; percentiles P:297; SLO P:361).
#pragma once

#include <stdint.h>

#include "common.cuh"

namespace tlru {

// One request segment [begin, end) of a b array, with its thresholds.
struct SegDev {
  uint64_t begin, end;
  uint32_t xi, slo;
  double xi_ms;
};

// Histogram every segment into hist[s * bins + v] (v clamped to bins - 1).
// Counts above the clamp are added to clamped[s].
tlru_status launch_hist(const uint16_t* b, const SegDev* segs, uint32_t ns, uint32_t bins, uint32_t* hist,
                        unsigned long long* clamped, cudaStream_t st);

// Final metrics from the histograms: writes tlru_tail (if tails != NULL) and/or
// the histogram-derived fields of tlru_result (if results != NULL).
tlru_status launch_finalize(const SegDev* segs, uint32_t ns, uint32_t bins, const uint32_t* hist,
                            const unsigned long long* clamped, double alpha, tlru_tail* tails,
                            tlru_result* results, cudaStream_t st);

// Copy per-instance histogram rows [ni][bins] to out[row][out_bins] (row = map[i], or i if map is
// NULL), zero-filling bins >= bins.
tlru_status launch_hist_export(const uint32_t* hist, uint32_t ni, uint32_t bins, const uint32_t* map, uint32_t* out,
                               uint32_t out_bins, cudaStream_t st);

}  // namespace tlru
