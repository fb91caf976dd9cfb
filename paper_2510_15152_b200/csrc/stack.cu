// stack.cu -- "stack" engine of tlru_simulate_batch: exact closed-form evaluation of
// Alg. 1 for every capacity at once.
//
// By the stack property the cache after each request is the top-C
// blocks of the universe under the key (non-free?, tau, -position), D = max(xi - Q_hat, 0)
// (free tail, P:56 / P:62), NF(L) = max(L - D, 0), F(L) = min(L, D).  For the request e
// of conversation theta with previous turn p (history Lb = L_after[p]):
//   A_nf(e) = sum NF(L_x), A_f(e) = sum F(L_x) over x in (p, e) with next[x] > e
//             (the conversations used after theta's previous turn, each at its latest L),
//   NF_all(e), F_all(e) = the same sums over every conversation's last turn before e,
//   X_theta = min(NF(Lb), (C - A_nf)^+) + min(F(Lb), (C - NF_all - A_f)^+),
//   b = J - X_theta
// and, telescoping Alg. 1's per-request evictions over the trace (used and the cached
// free blocks are functions of the universe: used = min(C, U), Fc = min(F_all, (C-NF_all)^+)):
//   evicted_total = sum a + sum b - min(C, U_final)
//   evicted_trim  = sum_e F(L_after_e) - sum_e X_f(e) - Fc_final       (Phase 1)
//   evicted_lru   = evicted_total - evicted_trim                        (Phase 2)
//   max_occupancy = min(C, U_final)
// Pinned against the oracle by tests/test_gpu_parity.py (both engines, every config)
// and, on CPU, tests/stackdist.py.
//
// Kernels per (trace, chunk of <= 8 distinct D):
//   s1_block : block aggregates (saturating) of the per-event universe deltas
//              (NF(L_after) - NF(L_before), F(...) - F(...)) for each D, plus sum F(L_after), sum a
//   s1_scan  : one CTA: exclusive scan of the block aggregates
//   s2_main  : one thread per request event: block scan of the deltas + the block prefix
//              = NF_all(e), F_all(e); backward window scan for A_nf / A_f of every D (early
//              exit once every D's non-free sum reaches its largest C); then b for every
//              instance of the chunk, coalesced 2-byte stores
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "metrics.cuh"
#include "stack.cuh"

namespace tlru {

constexpr int SND = 8;  // D values per chunk

struct Prefix8 {  // saturating per-D prefix sums of non-free / free blocks
  uint32_t nf[SND];
  uint32_t f[SND];
};

struct SatAdd {
  __host__ __device__ __forceinline__ Prefix8 operator()(const Prefix8& a, const Prefix8& b) const {
    Prefix8 r;
#pragma unroll
    for (int d = 0; d < SND; ++d) {
      uint32_t x = a.nf[d] + b.nf[d];
      r.nf[d] = x < a.nf[d] ? 0xFFFFFFFFu : x;
      uint32_t y = a.f[d] + b.f[d];
      r.f[d] = y < a.f[d] ? 0xFFFFFFFFu : y;
    }
    return r;
  }
};

struct ChunkDev {
  uint32_t D[SND];
  uint32_t Cmax[SND];  // largest capacity among the chunk's instances with this D
  uint32_t nd;
  uint32_t inst0, ninst;  // instances [inst0, inst0 + ninst) of the StackInstDev table
  uint32_t pad;
};

struct StackInstDev {
  uint32_t C, d, inst, pad;
  uint64_t boff;
};

struct ChunkTotals {  // per (chunk, d)
  unsigned long long sumF[SND];
  unsigned long long suma;
};

__device__ __forceinline__ uint32_t nf_of(uint32_t L, uint32_t D) { return L > D ? L - D : 0u; }
__device__ __forceinline__ uint32_t f_of(uint32_t L, uint32_t D) { return L < D ? L : D; }
__device__ __forceinline__ uint32_t sat_sub(uint32_t a, uint32_t b) { return a > b ? a - b : 0u; }

constexpr int S_THREADS = 256;  // events per block in s1 / s2 (one thread per event)

// Per-event deltas of the universe sums (non-free, free) for each D: at event e the
// conversation's history goes from L_before to L_after.
__device__ __forceinline__ void universe_delta(const ChunkDev& ch, uint32_t Lb, uint32_t La, Prefix8& v) {
#pragma unroll
  for (int d = 0; d < SND; ++d) {
    const uint32_t D = ch.D[d];
    v.nf[d] = nf_of(La, D) - nf_of(Lb, D);
    v.f[d] = f_of(La, D) - f_of(Lb, D);
  }
}

__device__ __forceinline__ uint32_t L_before(const uint64_t* sim, uint64_t s) {
  const uint32_t p = sim_prev(s);
  return p == TLRU_NONE ? 0u : sim_La(__ldg(sim + p));
}

// s1: block aggregates of the deltas (saturating) + trace totals sum F(L_after), sum a.
__global__ void __launch_bounds__(S_THREADS) s1_block_kernel(const uint64_t* __restrict__ sim, uint32_t E,
                                                             const ChunkDev* __restrict__ chunk,
                                                             Prefix8* __restrict__ blockagg, ChunkTotals* totals) {
  __shared__ ChunkDev ch;
  if (threadIdx.x == 0) ch = *chunk;
  __syncthreads();
  const uint32_t e = blockIdx.x * S_THREADS + threadIdx.x;
  Prefix8 v{};
  unsigned long long sa = 0;
  unsigned long long sf[SND];
#pragma unroll
  for (int d = 0; d < SND; ++d) sf[d] = 0;
  if (e < E) {
    const uint64_t s = __ldg(sim + e);
    const uint32_t La = sim_La(s);
    universe_delta(ch, L_before(sim, s), La, v);
    sa = La - sim_J(s);
#pragma unroll
    for (int d = 0; d < SND; ++d) sf[d] = f_of(La, ch.D[d]);
  }
  typedef cub::BlockReduce<Prefix8, S_THREADS> BRp;
  typedef cub::BlockReduce<unsigned long long, S_THREADS> BR;
  __shared__ union {
    typename BRp::TempStorage p;
    typename BR::TempStorage u;
  } tmp;
  const Prefix8 agg = BRp(tmp.p).Reduce(v, SatAdd());
  if (threadIdx.x == 0) blockagg[blockIdx.x] = agg;
#pragma unroll
  for (int d = 0; d < SND; ++d) {
    __syncthreads();
    const unsigned long long t = BR(tmp.u).Sum(sf[d]);
    if (threadIdx.x == 0 && t) atomicAdd(&totals->sumF[d], t);
  }
  __syncthreads();
  const unsigned long long t = BR(tmp.u).Sum(sa);
  if (threadIdx.x == 0 && t) atomicAdd(&totals->suma, t);
}

// s1b: one CTA scans the block aggregates in place (exclusive) and stores the total.
__global__ void __launch_bounds__(S_THREADS) s1_scan_kernel(Prefix8* blockagg, uint32_t nblocks, Prefix8* total) {
  typedef cub::BlockScan<Prefix8, S_THREADS> BS;
  __shared__ typename BS::TempStorage tmp;
  __shared__ Prefix8 carry;
  if (threadIdx.x == 0) carry = Prefix8{};
  __syncthreads();
  for (uint32_t base = 0; base < nblocks; base += S_THREADS) {
    const uint32_t i = base + threadIdx.x;
    Prefix8 v{};
    if (i < nblocks) v = blockagg[i];
    Prefix8 ex, agg;
    BS(tmp).ExclusiveScan(v, ex, Prefix8{}, SatAdd(), agg);
    const Prefix8 c = carry;
    if (i < nblocks) blockagg[i] = SatAdd()(c, ex);
    __syncthreads();
    if (threadIdx.x == 0) carry = SatAdd()(c, agg);
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

template <int ND>
__global__ void __launch_bounds__(S_THREADS) s2_main_kernel(const uint64_t* __restrict__ sim,
                                                            const uint32_t* __restrict__ next, uint32_t E,
                                                            const ChunkDev* __restrict__ chunk,
                                                            const StackInstDev* __restrict__ insts,
                                                            const Prefix8* __restrict__ blockpre,
                                                            uint16_t* __restrict__ bout, unsigned long long* sumXf) {
  __shared__ ChunkDev ch;
  typedef cub::BlockScan<Prefix8, S_THREADS> BS;
  __shared__ typename BS::TempStorage tmp;
  if (threadIdx.x == 0) ch = *chunk;
  __syncthreads();
  const uint32_t e = blockIdx.x * S_THREADS + threadIdx.x;
  uint64_t s = 0;
  uint32_t Lb = 0;
  Prefix8 v{};
  if (e < E) {
    s = __ldg(sim + e);
    Lb = L_before(sim, s);
    universe_delta(ch, Lb, sim_La(s), v);
  }
  // NF_all(e), F_all(e): universe sums over every conversation's last turn before e
  Prefix8 ex;
  BS(tmp).ExclusiveScan(v, ex, Prefix8{}, SatAdd());
  if (e >= E) return;
  const Prefix8 P = SatAdd()(blockpre[blockIdx.x], ex);
  const uint32_t p = sim_prev(s), J = sim_J(s);
  uint32_t anf[ND], af[ND], nfb[ND], fb[ND], nfall[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    anf[d] = af[d] = nfb[d] = fb[d] = 0;
    nfall[d] = P.nf[d];
  }
  if (p != TLRU_NONE) {
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      nfb[d] = nf_of(Lb, ch.D[d]);
      fb[d] = f_of(Lb, ch.D[d]);
    }
    // backward window scan over x in (p, e): conversations used after theta's last turn
    for (uint32_t x = e - 1; x > p; --x) {
      if (__ldg(next + x) <= e) continue;  // x's conversation returns before e: not its last turn
      const uint32_t L = sim_La(__ldg(sim + x));
      bool done = true;
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        anf[d] += nf_of(L, ch.D[d]);
        af[d] += f_of(L, ch.D[d]);
        done &= anf[d] >= ch.Cmax[d];
      }
      // every capacity already excludes theta's non-free blocks; then NF_all >= A_nf >= C too,
      // so no free block of theta is cached either
      if (done) break;
    }
  }
  for (uint32_t k = 0; k < ch.ninst; ++k) {
    const StackInstDev in = insts[ch.inst0 + k];
    uint32_t nfb_d = 0, fb_d = 0, anf_d = 0, af_d = 0, nfall_d = 0;
#pragma unroll
    for (int d = 0; d < ND; ++d)
      if (static_cast<uint32_t>(d) == in.d) {
        nfb_d = nfb[d];
        fb_d = fb[d];
        anf_d = anf[d];
        af_d = af[d];
        nfall_d = nfall[d];
      }
    uint32_t X = min(nfb_d, sat_sub(in.C, anf_d));
    if (nfall_d < in.C && fb_d > 0) {  // warm-up: free blocks can still be cached
      const uint32_t xf = min(fb_d, sat_sub(sat_sub(in.C, nfall_d), af_d));
      X += xf;
      if (xf) atomicAdd(&sumXf[in.inst], static_cast<unsigned long long>(xf));
    }
    bout[in.boff + e] = static_cast<uint16_t>(J - X);
  }
}

__global__ void s3_results_kernel(const StackInstDev* __restrict__ insts, uint32_t ninst,
                                  const uint32_t* __restrict__ inst_chunk, const ChunkTotals* __restrict__ totals,
                                  const Prefix8* const* __restrict__ finals, const unsigned long long* sumXf,
                                  tlru_result* results) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < ninst; k += gridDim.x * blockDim.x) {
    const StackInstDev in = insts[k];
    const uint32_t c = inst_chunk[k];
    const Prefix8 fin = *finals[c];
    const uint32_t nfE = fin.nf[in.d], fE = fin.f[in.d];
    const uint64_t U = uint64_t(nfE) + fE;
    const uint64_t used_final = U < in.C ? U : in.C;
    const uint64_t fc_final = min(fE, sat_sub(in.C, nfE));
    tlru_result& r = results[in.inst];
    const unsigned long long total = totals[c].suma + r.sum_uncached - used_final;
    const unsigned long long trim = totals[c].sumF[in.d] - sumXf[in.inst] - fc_final;
    r.evicted_trim = trim;
    r.evicted_lru = total - trim;
    r.max_occupancy = static_cast<uint32_t>(used_final);
  }
}

// ----------------------------------------------------------------------------- host
struct StackPlan {
  struct Chunk {
    uint32_t trace;
    ChunkDev dev;
  };
  std::vector<Chunk> chunks;
  std::vector<StackInstDev> insts;
  std::vector<uint32_t> inst_chunk;
  uint64_t Emax = 0;
};

static void make_stack_plan(const tlru_trace* traces, uint32_t nt, const tlru_instance* inst, uint32_t ni,
                            const uint64_t* boffs, StackPlan* P) {
  for (uint32_t t = 0; t < nt; ++t) P->Emax = std::max<uint64_t>(P->Emax, traces[t].num_events);
  for (uint32_t t = 0; t < nt; ++t) {
    std::vector<uint32_t> ids;
    for (uint32_t i = 0; i < ni; ++i)
      if (inst[i].trace == t) ids.push_back(i);
    if (ids.empty() || traces[t].num_events == 0) continue;
    auto Dof = [&](uint32_t i) {
      return (inst[i].policy == TLRU_POLICY_TLRU && inst[i].xi > inst[i].q_hat) ? inst[i].xi - inst[i].q_hat : 0u;
    };
    std::vector<uint32_t> Ds;
    for (uint32_t i : ids) Ds.push_back(Dof(i));
    std::sort(Ds.begin(), Ds.end());
    Ds.erase(std::unique(Ds.begin(), Ds.end()), Ds.end());
    for (size_t c0 = 0; c0 < Ds.size(); c0 += SND) {
      StackPlan::Chunk ch;
      ch.trace = t;
      memset(&ch.dev, 0, sizeof(ch.dev));
      ch.dev.nd = static_cast<uint32_t>(std::min<size_t>(SND, Ds.size() - c0));
      for (uint32_t d = 0; d < SND; ++d) ch.dev.D[d] = d < ch.dev.nd ? Ds[c0 + d] : Ds[c0];
      ch.dev.inst0 = static_cast<uint32_t>(P->insts.size());
      for (uint32_t i : ids) {
        uint32_t D = Dof(i);
        for (uint32_t d = 0; d < ch.dev.nd; ++d)
          if (ch.dev.D[d] == D) {
            StackInstDev s;
            s.C = std::min<uint32_t>(inst[i].capacity, 0x7FFF0000u);
            s.d = d;
            s.inst = i;
            s.pad = 0;
            s.boff = boffs[i];
            ch.dev.Cmax[d] = std::max(ch.dev.Cmax[d], s.C);
            P->insts.push_back(s);
            P->inst_chunk.push_back(static_cast<uint32_t>(P->chunks.size()));
          }
      }
      for (uint32_t d = ch.dev.nd; d < SND; ++d) ch.dev.Cmax[d] = 0;
      ch.dev.ninst = static_cast<uint32_t>(P->insts.size()) - ch.dev.inst0;
      P->chunks.push_back(ch);
    }
  }
}

struct StackWs {
  ChunkDev* chunks;
  StackInstDev* insts;
  uint32_t* inst_chunk;
  ChunkTotals* totals;
  Prefix8** finals;
  Prefix8* fin;
  unsigned long long* sumXf;
  Prefix8* blockpre;  // [chunk][block] exclusive block prefixes
  uint64_t nblocks_max;
};

static void carve_stack(Carver& cv, const StackPlan& P, uint32_t ni, StackWs* w) {
  const size_t nc = P.chunks.size() + 1;
  w->chunks = cv.take<ChunkDev>(nc);
  w->insts = cv.take<StackInstDev>(P.insts.size() + 1);
  w->inst_chunk = cv.take<uint32_t>(P.insts.size() + 1);
  w->totals = cv.take<ChunkTotals>(nc);
  w->finals = cv.take<Prefix8*>(nc);
  w->fin = cv.take<Prefix8>(nc);
  w->sumXf = cv.take<unsigned long long>(ni + 1);
  w->nblocks_max = (P.Emax + S_THREADS - 1) / S_THREADS + 1;
  w->blockpre = cv.take<Prefix8>(nc * w->nblocks_max);
}

tlru_status stack_workspace(const tlru_trace* traces, uint32_t nt, const tlru_instance* inst, uint32_t ni,
                            size_t* bytes) {
  std::vector<uint64_t> boffs(ni, 0);
  StackPlan P;
  make_stack_plan(traces, nt, inst, ni, boffs.data(), &P);
  Carver cv(nullptr);
  StackWs w;
  carve_stack(cv, P, ni, &w);
  *bytes = cv.used;
  return TLRU_OK;
}

template <int ND>
static void launch_s2(const tlru_trace& tr, const ChunkDev* ch, const Prefix8* blockpre, const StackWs& w,
                      uint16_t* bout, cudaStream_t st) {
  const uint32_t E = static_cast<uint32_t>(tr.num_events);
  s2_main_kernel<ND><<<(E + S_THREADS - 1) / S_THREADS, S_THREADS, 0, st>>>(tr.sim, tr.next, E, ch, w.insts, blockpre,
                                                                            bout, w.sumXf);
}

tlru_status stack_simulate(const tlru_trace* traces, uint32_t nt, const tlru_instance* inst, uint32_t ni,
                           const uint64_t* boffs, uint16_t* bout, tlru_result* results, Carver& cv,
                           const SegDev* segs_dev, uint32_t bins, uint32_t* hist, unsigned long long* clamped,
                           size_t ws_bytes, cudaStream_t st, unsigned* nkernels, cudaEvent_t ev_mid) {
  StackPlan P;
  make_stack_plan(traces, nt, inst, ni, boffs, &P);
  StackWs w;
  carve_stack(cv, P, ni, &w);
  TLRU_TRY(check_ws(cv, cv.base, ws_bytes));
  const size_t nc = P.chunks.size();
  TLRU_CUDA(cudaMemsetAsync(results, 0, size_t(ni) * sizeof(tlru_result), st));
  std::vector<ChunkDev> chd(nc);
  std::vector<Prefix8*> finp(nc);
  for (size_t c = 0; c < nc; ++c) {
    chd[c] = P.chunks[c].dev;
    finp[c] = w.fin + c;
  }
  if (nc) {
    TLRU_CUDA(cudaMemcpyAsync(w.chunks, chd.data(), nc * sizeof(ChunkDev), cudaMemcpyHostToDevice, st));
    TLRU_CUDA(cudaMemcpyAsync(w.finals, finp.data(), nc * sizeof(Prefix8*), cudaMemcpyHostToDevice, st));
    TLRU_CUDA(cudaMemcpyAsync(w.insts, P.insts.data(), P.insts.size() * sizeof(StackInstDev),
                              cudaMemcpyHostToDevice, st));
    TLRU_CUDA(cudaMemcpyAsync(w.inst_chunk, P.inst_chunk.data(), P.inst_chunk.size() * sizeof(uint32_t),
                              cudaMemcpyHostToDevice, st));
  }
  TLRU_CUDA(cudaMemsetAsync(w.totals, 0, (nc + 1) * sizeof(ChunkTotals), st));
  TLRU_CUDA(cudaMemsetAsync(w.sumXf, 0, (ni + 1) * sizeof(unsigned long long), st));
  for (size_t c = 0; c < nc; ++c) {
    const tlru_trace& tr = traces[P.chunks[c].trace];
    const uint32_t E = static_cast<uint32_t>(tr.num_events);
    const uint32_t nb = (E + S_THREADS - 1) / S_THREADS;
    Prefix8* bp = w.blockpre + c * w.nblocks_max;
    s1_block_kernel<<<nb, S_THREADS, 0, st>>>(tr.sim, E, w.chunks + c, bp, w.totals + c);
    TLRU_CHECK_LAUNCH();
    s1_scan_kernel<<<1, S_THREADS, 0, st>>>(bp, nb, w.fin + c);
    TLRU_CHECK_LAUNCH();
    switch (P.chunks[c].dev.nd) {
      case 1: launch_s2<1>(tr, w.chunks + c, bp, w, bout, st); break;
      case 2: launch_s2<2>(tr, w.chunks + c, bp, w, bout, st); break;
      case 3: launch_s2<3>(tr, w.chunks + c, bp, w, bout, st); break;
      case 4: launch_s2<4>(tr, w.chunks + c, bp, w, bout, st); break;
      case 5: launch_s2<5>(tr, w.chunks + c, bp, w, bout, st); break;
      case 6: launch_s2<6>(tr, w.chunks + c, bp, w, bout, st); break;
      case 7: launch_s2<7>(tr, w.chunks + c, bp, w, bout, st); break;
      default: launch_s2<8>(tr, w.chunks + c, bp, w, bout, st); break;
    }
    TLRU_CHECK_LAUNCH();
    *nkernels += 3;
  }
  // K3 over b, then the eviction counters from the telescoped identities
  if (ev_mid) TLRU_CUDA(cudaEventRecord(ev_mid, st));
  TLRU_TRY(launch_hist(bout, segs_dev, ni, bins, hist, clamped, st));
  TLRU_TRY(launch_finalize(segs_dev, ni, bins, hist, clamped, 1.0, nullptr, results, st));
  if (!P.insts.empty()) {
    s3_results_kernel<<<grid_for(P.insts.size(), 128), 128, 0, st>>>(w.insts, static_cast<uint32_t>(P.insts.size()),
                                                                     w.inst_chunk, w.totals, w.finals, w.sumXf,
                                                                     results);
    TLRU_CHECK_LAUNCH();
  }
  *nkernels += 3;
  return TLRU_OK;
}

}  // namespace tlru
