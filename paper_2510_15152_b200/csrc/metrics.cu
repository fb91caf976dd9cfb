// metrics.cu -- K3 and the tlru_tail_metrics entry point.
//
// hist:     one grid row per segment; 16-byte vector loads of b (8 requests per
//           load, HBM-bound), per-warp shared-memory sub-histograms merged into a
//           global [segment][bin] histogram.
// finalize: one CTA per segment; each thread owns a contiguous bin range, a block
//           scan of the counts gives the exact integer nearest ranks (Reading #11);
//           TEL in blocks (Eq. 3), SLO count, sums and max are exact
//           integers; TEL_ms (Eq. 1) is summed per bin in ascending b and the
//           per-thread partials are added in thread order (deterministic).
#include <cub/cub.cuh>

#include <algorithm>

#include "metrics.cuh"

namespace tlru {

constexpr int HIST_THREADS = 256;
constexpr int HIST_WARPS = HIST_THREADS / 32;
constexpr uint32_t SMEM_HIST_BYTES = 96 * 1024;

template <int NSUB>
__global__ void __launch_bounds__(HIST_THREADS) hist_kernel(const uint16_t* __restrict__ b, const SegDev* segs,
                                                            uint32_t bins, uint32_t* hist,
                                                            unsigned long long* clamped) {
  extern __shared__ uint32_t sh[];
  const uint32_t s = blockIdx.y;
  const SegDev sg = segs[s];
  const uint32_t tid = threadIdx.x;
  for (uint32_t k = tid; k < bins * NSUB; k += HIST_THREADS) sh[k] = 0;
  __syncthreads();
  uint32_t* H = sh + (NSUB > 1 ? (tid / 32) % NSUB : 0) * bins;
  const uint32_t top = bins - 1;
  uint32_t nclamp = 0;
  auto add = [&](uint32_t v) {
    if (v > top) {
      v = top;
      ++nclamp;
    }
    atomicAdd(&H[v], 1u);
  };
  const uint64_t stride = uint64_t(gridDim.x) * HIST_THREADS;
  const uint64_t gt = uint64_t(blockIdx.x) * HIST_THREADS + tid;
  uint64_t a0 = (sg.begin + 7) & ~7ull;
  if (a0 > sg.end) a0 = sg.end;
  const uint64_t a1 = a0 + ((sg.end - a0) & ~7ull);
  for (uint64_t i = sg.begin + gt; i < a0; i += stride) add(b[i]);
  for (uint64_t i = a1 + gt; i < sg.end; i += stride) add(b[i]);
  const uint4* bv = reinterpret_cast<const uint4*>(b);
  for (uint64_t j = a0 / 8 + gt; j < a1 / 8; j += stride) {
    uint4 v = __ldcs(bv + j);  // streamed once: evict-first
    add(v.x & 0xFFFFu);
    add(v.x >> 16);
    add(v.y & 0xFFFFu);
    add(v.y >> 16);
    add(v.z & 0xFFFFu);
    add(v.z >> 16);
    add(v.w & 0xFFFFu);
    add(v.w >> 16);
  }
  __syncthreads();
  for (uint32_t k = tid; k < bins; k += HIST_THREADS) {
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < NSUB; ++w) c += sh[w * bins + k];
    if (c) atomicAdd(&hist[uint64_t(s) * bins + k], c);
  }
  typedef cub::WarpReduce<uint32_t> WR;
  __shared__ typename WR::TempStorage wr[HIST_WARPS];
  uint32_t tot = WR(wr[tid / 32]).Sum(nclamp);
  if ((tid & 31) == 0 && tot) atomicAdd(&clamped[s], static_cast<unsigned long long>(tot));
}

// Global-memory histogram for very wide bin ranges.
__global__ void hist_global_kernel(const uint16_t* __restrict__ b, const SegDev* segs, uint32_t bins, uint32_t* hist,
                                   unsigned long long* clamped) {
  const uint32_t s = blockIdx.y;
  const SegDev sg = segs[s];
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = sg.begin + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < sg.end; i += stride) {
    uint32_t v = b[i];
    if (v > bins - 1) {
      v = bins - 1;
      atomicAdd(&clamped[s], 1ull);
    }
    atomicAdd(&hist[uint64_t(s) * bins + v], 1u);
  }
}

constexpr int FIN_THREADS = 256;

// Thresholds of one segment: the SegDev of a b segment, or (xi, xi_ms, slo) arrays for
// tlru_tail_from_histograms (NULL -> 0, 0.0, no SLO).
struct FinParams {
  const SegDev* segs;
  const uint32_t* xi;
  const double* xi_ms;
  const uint32_t* slo;
  __device__ void get(uint32_t s, uint32_t& x, double& xm, uint32_t& sl) const {
    if (segs) {
      x = segs[s].xi;
      xm = segs[s].xi_ms;
      sl = segs[s].slo;
    } else {
      x = xi ? xi[s] : 0u;
      xm = xi_ms ? xi_ms[s] : 0.0;
      sl = slo ? slo[s] : 0xFFFFFFFFu;
    }
  }
};

// One CTA per histogram row: exact integer ranks / TEL / SLO / sums from the counts (CountT =
// u32 for per-instance rows, u64 for pooled rows).
template <typename CountT>
__global__ void __launch_bounds__(FIN_THREADS) finalize_kernel(FinParams prm, uint32_t bins, const CountT* hist,
                                                                const unsigned long long* clamped, double alpha,
                                                                tlru_tail* tails, tlru_result* results) {
  const uint32_t s = blockIdx.x;
  uint32_t sg_xi, sg_slo;
  double sg_xi_ms;
  prm.get(s, sg_xi, sg_xi_ms, sg_slo);
  const uint32_t tid = threadIdx.x;
  const CountT* H = hist + uint64_t(s) * bins;
  const uint32_t per = (bins + FIN_THREADS - 1) / FIN_THREADS;
  const uint32_t lo = min(bins, tid * per), hi = min(bins, lo + per);
  unsigned long long cnt = 0, sum = 0, tel = 0, slo = 0;
  uint32_t vmax = 0;
  double tel_ms = 0.0;
  for (uint32_t v = lo; v < hi; ++v) {
    const unsigned long long c = H[v];
    if (!c) continue;
    cnt += c;
    sum += c * v;
    if (v > sg_xi) tel += c * (v - sg_xi);  // (b - xi)^+  (Eq. 3)
    if (v > sg_slo) slo += c;               // b > slo, strict
    vmax = v;
    const double term = alpha * static_cast<double>(v) - sg_xi_ms;
    if (term > 0.0) tel_ms += static_cast<double>(c) * term;  // (alpha b - xi_s)^+  (Eq. 1)
  }
  typedef cub::BlockScan<unsigned long long, FIN_THREADS> BS;
  typedef cub::BlockReduce<unsigned long long, FIN_THREADS> BR;
  typedef cub::BlockReduce<uint32_t, FIN_THREADS> BRu;
  __shared__ union {
    typename BS::TempStorage scan;
    typename BR::TempStorage red;
    typename BRu::TempStorage redu;
  } tmp;
  __shared__ double part[FIN_THREADS];
  __shared__ uint32_t pv[4];
  __shared__ unsigned long long n_all;
  unsigned long long before, total;
  BS(tmp.scan).ExclusiveSum(cnt, before, total);
  if (tid == 0) n_all = total;
  if (tid < 4) pv[tid] = 0;
  __syncthreads();
  const unsigned long long n = n_all;
  const unsigned long long pbp[4] = {5000, 9000, 9500, 9900};
  if (n > 0 && cnt > 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      unsigned long long k = (pbp[j] * n + 9999ull) / 10000ull;  // nearest rank, integer
      if (k < 1) k = 1;
      if (k > before && k <= before + cnt) {
        unsigned long long acc = before;
        for (uint32_t v = lo; v < hi; ++v) {
          acc += H[v];
          if (acc >= k) {
            pv[j] = v;
            break;
          }
        }
      }
    }
  }
  part[tid] = tel_ms;
  __syncthreads();
  unsigned long long sum_all = BR(tmp.red).Sum(sum);
  __syncthreads();
  unsigned long long tel_all = BR(tmp.red).Sum(tel);
  __syncthreads();
  unsigned long long slo_all = BR(tmp.red).Sum(slo);
  __syncthreads();
  uint32_t max_all = BRu(tmp.redu).Reduce(vmax, cub::Max());
  if (tid == 0) {
    double tms = 0.0;
    for (int t = 0; t < FIN_THREADS; ++t) tms += part[t];
    if (tails) {
      tlru_tail o;
      o.n = n;
      o.tel_blocks = tel_all;
      o.slo_violations = slo_all;
      o.sum_b = sum_all;
      o.p50 = pv[0];
      o.p90 = pv[1];
      o.p95 = pv[2];
      o.p99 = pv[3];
      o.max_b = n ? max_all : 0;
      o.n_clamped = clamped ? static_cast<uint32_t>(clamped[s]) : 0u;
      o.tel_ms = tms;
      o.p50_ms = alpha * static_cast<double>(pv[0]);
      o.p90_ms = alpha * static_cast<double>(pv[1]);
      o.p95_ms = alpha * static_cast<double>(pv[2]);
      o.p99_ms = alpha * static_cast<double>(pv[3]);
      o.mean_ms = n ? (alpha * static_cast<double>(sum_all)) / static_cast<double>(n) : 0.0;
      tails[s] = o;
    }
    if (results) {
      tlru_result& r = results[s];
      r.requests = n;
      r.sum_uncached = sum_all;
      r.tel_blocks = tel_all;
      r.slo_violations = slo_all;
      r.p50 = pv[0];
      r.p90 = pv[1];
      r.p95 = pv[2];
      r.p99 = pv[3];
      r.max_uncached = n ? max_all : 0;
    }
  }
}

// hist_out[row(i)][v] = hist[i][v] for v < bins, 0 for bins <= v < out_bins (row(i) = map[i] or i)
__global__ void hist_export_kernel(const uint32_t* __restrict__ hist, uint32_t ni, uint32_t bins,
                                   const uint32_t* __restrict__ map, uint32_t* __restrict__ out, uint32_t out_bins) {
  const uint32_t i = blockIdx.y;
  const uint32_t row = map ? map[i] : i;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < out_bins; v += gridDim.x * blockDim.x)
    out[uint64_t(row) * out_bins + v] = v < bins ? hist[uint64_t(i) * bins + v] : 0u;
}

// pooled[pool[i]][v] += hist[i][v]
__global__ void pool_kernel(const uint32_t* __restrict__ hist, uint32_t bins, const uint32_t* __restrict__ pool,
                            unsigned long long* __restrict__ pooled) {
  const uint32_t i = blockIdx.y;
  const uint32_t p = pool[i];
  if (p == TLRU_NONE) return;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < bins; v += gridDim.x * blockDim.x) {
    const uint32_t c = hist[uint64_t(i) * bins + v];
    if (c) atomicAdd(pooled + uint64_t(p) * bins + v, static_cast<unsigned long long>(c));
  }
}

tlru_status launch_hist_export(const uint32_t* hist, uint32_t ni, uint32_t bins, const uint32_t* map, uint32_t* out,
                               uint32_t out_bins, cudaStream_t st) {
  if (ni == 0 || !out) return TLRU_OK;
  for (uint32_t i0 = 0; i0 < ni; i0 += 65535u) {
    const uint32_t n = std::min(65535u, ni - i0);
    hist_export_kernel<<<dim3((out_bins + 255) / 256, n), 256, 0, st>>>(hist + uint64_t(i0) * bins, n, bins,
                                                                        map ? map + i0 : nullptr,
                                                                        map ? out : out + uint64_t(i0) * out_bins,
                                                                        out_bins);
    TLRU_CHECK_LAUNCH();
  }
  return TLRU_OK;
}

tlru_status launch_hist(const uint16_t* b, const SegDev* segs, uint32_t ns, uint32_t bins, uint32_t* hist,
                        unsigned long long* clamped, cudaStream_t st) {
  if (ns == 0) return TLRU_OK;
  // at least ~2 waves of 8 resident CTAs per SM over all segments
  const unsigned target = 148u * 8u * 2u;
  const unsigned gx = (target + ns - 1) / ns;
  dim3 grid(gx < 1 ? 1 : gx, ns);
  const bool aligned = (reinterpret_cast<uintptr_t>(b) % 16) == 0;
  if (aligned && size_t(bins) * HIST_WARPS * 4 <= SMEM_HIST_BYTES) {
    size_t sm = size_t(bins) * HIST_WARPS * 4;
    TLRU_CUDA(cudaFuncSetAttribute(hist_kernel<HIST_WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(SMEM_HIST_BYTES)));
    hist_kernel<HIST_WARPS><<<grid, HIST_THREADS, sm, st>>>(b, segs, bins, hist, clamped);
  } else if (aligned && size_t(bins) * 4 <= SMEM_HIST_BYTES) {
    size_t sm = size_t(bins) * 4;
    TLRU_CUDA(cudaFuncSetAttribute(hist_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(SMEM_HIST_BYTES)));
    hist_kernel<1><<<grid, HIST_THREADS, sm, st>>>(b, segs, bins, hist, clamped);
  } else {
    hist_global_kernel<<<grid, 256, 0, st>>>(b, segs, bins, hist, clamped);
  }
  TLRU_CHECK_LAUNCH();
  return TLRU_OK;
}

tlru_status launch_finalize(const SegDev* segs, uint32_t ns, uint32_t bins, const uint32_t* hist,
                            const unsigned long long* clamped, double alpha, tlru_tail* tails,
                            tlru_result* results, cudaStream_t st) {
  if (ns == 0) return TLRU_OK;
  finalize_kernel<uint32_t><<<ns, FIN_THREADS, 0, st>>>(FinParams{segs, nullptr, nullptr, nullptr}, bins, hist, clamped,
                                                        alpha, tails, results);
  TLRU_CHECK_LAUNCH();
  return TLRU_OK;
}

// ----------------------------------------------------------------------------- tlru_tail_metrics
__global__ void tail_segs_kernel(const uint64_t* off, uint32_t ns, const uint32_t* xi, const double* xi_ms,
                                 const uint32_t* slo, SegDev* segs) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += gridDim.x * blockDim.x) {
    SegDev d;
    d.begin = off[s];
    d.end = off[s + 1] < off[s] ? off[s] : off[s + 1];
    d.xi = xi ? xi[s] : 0u;
    d.slo = slo ? slo[s] : 0xFFFFFFFFu;
    d.xi_ms = xi_ms ? xi_ms[s] : 0.0;
    segs[s] = d;
  }
}

struct TailWs {
  SegDev* segs;
  uint32_t* hist;
  unsigned long long* clamped;
};

static void carve_tail(Carver& cv, uint32_t ns, uint32_t bins, TailWs* w) {
  w->segs = cv.take<SegDev>(ns ? ns : 1);
  w->hist = cv.take<uint32_t>(uint64_t(ns ? ns : 1) * bins);
  w->clamped = cv.take<unsigned long long>(ns + 1);  // + the total over segments
}

__global__ void sum_u64_kernel(const unsigned long long* v, uint32_t n, unsigned long long* out) {
  unsigned long long s = 0;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
  warp_atomic_add_u64(out, s);
}

}  // namespace tlru

using namespace tlru;

extern "C" tlru_status tlru_tail_workspace_size(uint32_t ns, uint32_t max_b, size_t* bytes) {
  clear_error();
  if (!bytes) TLRU_FAIL(TLRU_EINVAL, "bytes is NULL");
  if (max_b > 65535) TLRU_FAIL(TLRU_ERANGE, "max_b must be <= 65535");
  Carver cv(nullptr);
  TailWs w;
  carve_tail(cv, ns, max_b + 1, &w);
  *bytes = cv.used;
  return TLRU_OK;
}

extern "C" tlru_status tlru_tail_metrics(const uint16_t* b, const uint64_t* seg_offsets, uint32_t ns,
                                         const uint32_t* xi, const double* xi_ms, const uint32_t* slo,
                                         double alpha, uint32_t max_b, tlru_tail* out, void* ws, size_t ws_bytes,
                                         cudaStream_t st) {
  clear_error();
  if (ns == 0) return TLRU_OK;
  if (!b || !seg_offsets || !out) TLRU_FAIL(TLRU_EINVAL, "b/seg_offsets/out is NULL");
  if (max_b > 65535) TLRU_FAIL(TLRU_ERANGE, "max_b must be <= 65535");
  if (!(alpha >= 0.0)) TLRU_FAIL(TLRU_EINVAL, "alpha must be >= 0");
  const uint32_t bins = max_b + 1;
  Carver cv(ws);
  TailWs w;
  carve_tail(cv, ns, bins, &w);
  TLRU_TRY(check_ws(cv, ws, ws_bytes));
  TLRU_CUDA(cudaMemsetAsync(w.hist, 0, size_t(ns) * bins * sizeof(uint32_t), st));
  TLRU_CUDA(cudaMemsetAsync(w.clamped, 0, size_t(ns) * sizeof(unsigned long long), st));
  tail_segs_kernel<<<grid_for(ns, 128), 128, 0, st>>>(seg_offsets, ns, xi, xi_ms, slo, w.segs);
  TLRU_CHECK_LAUNCH();
  TLRU_TRY(launch_hist(b, w.segs, ns, bins, w.hist, w.clamped, st));
  TLRU_TRY(launch_finalize(w.segs, ns, bins, w.hist, w.clamped, alpha, out, nullptr, st));
  // never report percentiles of truncated data: any b > max_b is an error
  unsigned long long* nbad = w.clamped + ns;
  TLRU_CUDA(cudaMemsetAsync(nbad, 0, sizeof(unsigned long long), st));
  sum_u64_kernel<<<1, 256, 0, st>>>(w.clamped, ns, nbad);
  TLRU_CHECK_LAUNCH();
  unsigned long long bad = 0;
  TLRU_CUDA(cudaMemcpyAsync(&bad, nbad, sizeof(bad), cudaMemcpyDeviceToHost, st));
  TLRU_CUDA(cudaStreamSynchronize(st));
  if (bad) TLRU_FAIL(TLRU_ERANGE, "%llu values of b exceed max_b = %u (see tlru_tail.n_clamped)", bad, max_b);
  return TLRU_OK;
}

extern "C" tlru_status tlru_pool_workspace_size(uint32_t ni, size_t* bytes) {
  clear_error();
  if (!bytes) TLRU_FAIL(TLRU_EINVAL, "bytes is NULL");
  Carver cv(nullptr);
  cv.take<uint32_t>(ni ? ni : 1);
  *bytes = cv.used;
  return TLRU_OK;
}

extern "C" tlru_status tlru_pool_histograms(const uint32_t* hist, uint32_t ni, uint32_t bins, const uint32_t* pool,
                                            uint32_t npool, uint64_t* pooled, void* ws, size_t ws_bytes,
                                            cudaStream_t st) {
  clear_error();
  if (ni == 0) return TLRU_OK;
  if (!hist || !pool || !pooled) TLRU_FAIL(TLRU_EINVAL, "hist/pool/pooled is NULL");
  if (bins == 0 || bins > 65536) TLRU_FAIL(TLRU_EINVAL, "bins must be in 1..65536");
  for (uint32_t i = 0; i < ni; ++i)
    if (pool[i] != TLRU_NONE && pool[i] >= npool) TLRU_FAIL(TLRU_EINVAL, "pool[%u] = %u >= npool = %u", i, pool[i], npool);
  Carver cv(ws);
  uint32_t* dpool = cv.take<uint32_t>(ni);
  TLRU_TRY(check_ws(cv, ws, ws_bytes));
  TLRU_CUDA(cudaMemcpyAsync(dpool, pool, size_t(ni) * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
  for (uint32_t i0 = 0; i0 < ni; i0 += 65535u) {
    const uint32_t n = std::min(65535u, ni - i0);
    pool_kernel<<<dim3((bins + 255) / 256, n), 256, 0, st>>>(hist + uint64_t(i0) * bins, bins, dpool + i0,
                                                             reinterpret_cast<unsigned long long*>(pooled));
    TLRU_CHECK_LAUNCH();
  }
  // the pool map is copied from pageable host memory: it is staged before the call returns
  return TLRU_OK;
}

extern "C" tlru_status tlru_tail_from_histograms(const uint64_t* hist, uint32_t ns, uint32_t bins, const uint32_t* xi,
                                                 const double* xi_ms, const uint32_t* slo, double alpha,
                                                 tlru_tail* out, cudaStream_t st) {
  clear_error();
  if (ns == 0) return TLRU_OK;
  if (!hist || !out) TLRU_FAIL(TLRU_EINVAL, "hist/out is NULL");
  if (bins == 0 || bins > 65536) TLRU_FAIL(TLRU_EINVAL, "bins must be in 1..65536");
  if (!(alpha >= 0.0)) TLRU_FAIL(TLRU_EINVAL, "alpha must be >= 0");
  finalize_kernel<unsigned long long><<<ns, FIN_THREADS, 0, st>>>(
      FinParams{nullptr, xi, xi_ms, slo}, bins, reinterpret_cast<const unsigned long long*>(hist), nullptr, alpha, out,
      nullptr);
  TLRU_CHECK_LAUNCH();
  return TLRU_OK;
}
