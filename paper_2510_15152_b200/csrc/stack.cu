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
  uint32_t Cmax[SND];     // largest capacity among the chunk's instances with this D
  uint32_t dbeg[SND + 1]; // instances of D[d]: [inst0 + dbeg[d], inst0 + dbeg[d+1])
  uint32_t nd;
  uint32_t inst0, ninst;  // instances [inst0, inst0 + ninst) of the StackInstDev table
};

struct StackInstDev {
  uint32_t C, d, inst, pad;
  uint64_t boff;
};

struct ChunkTotals {  // per chunk: exact trace totals
  unsigned long long sumF[SND];  // sum_e F(L_after_e)
  unsigned long long nfE[SND];   // NF_all(E): non-free blocks of the final universe
  unsigned long long fE[SND];    // F_all(E)
  unsigned long long suma;       // sum_e a_e
  uint32_t nsat;                 // first block whose prefix saturates every D (NF_all >= Cmax)
  uint32_t pad;
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

// s1: per-event scan record (next | L_after << 32) for the window scans, block aggregates of
// the universe deltas (saturating, one per 256 events), and the exact trace totals.  A
// persistent grid walks the 256-event blocks so the totals are reduced once per CTA.
constexpr int NTOT = 3 * SND + 1;

__global__ void __launch_bounds__(S_THREADS) s1_block_kernel(const uint64_t* __restrict__ sim,
                                                             const uint32_t* __restrict__ next, uint32_t E,
                                                             const ChunkDev* __restrict__ chunk,
                                                             uint64_t* __restrict__ scanrec,
                                                             Prefix8* __restrict__ blockagg, ChunkTotals* totals) {
  typedef cub::BlockReduce<Prefix8, S_THREADS> BRp;
  __shared__ typename BRp::TempStorage tmp;
  __shared__ ChunkDev ch;
  __shared__ unsigned long long part[S_THREADS / 32][NTOT];
  if (threadIdx.x == 0) ch = *chunk;
  __syncthreads();
  unsigned long long tv[NTOT];
#pragma unroll
  for (int k = 0; k < NTOT; ++k) tv[k] = 0;
  const uint32_t nblocks = (E + S_THREADS - 1) / S_THREADS;
  for (uint32_t blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
    const uint32_t e = blk * S_THREADS + threadIdx.x;
    Prefix8 v{};
    if (e < E) {
      const uint64_t s = __ldg(sim + e);
      const uint32_t La = sim_La(s);
      scanrec[e] = uint64_t(__ldg(next + e)) | (uint64_t(La) << 32);
      universe_delta(ch, L_before(sim, s), La, v);
#pragma unroll
      for (int d = 0; d < SND; ++d) {
        tv[d] += f_of(La, ch.D[d]);
        tv[SND + d] += v.nf[d];
        tv[2 * SND + d] += v.f[d];
      }
      tv[3 * SND] += La - sim_J(s);
    }
    const Prefix8 agg = BRp(tmp).Reduce(v, SatAdd());
    if (threadIdx.x == 0) blockagg[blk] = agg;
    __syncthreads();
  }
  // totals: warp shuffles, then one atomic per value per CTA
#pragma unroll
  for (int k = 0; k < NTOT; ++k) {
    unsigned long long x = tv[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x / 32][k] = x;
  }
  __syncthreads();
  if (threadIdx.x < NTOT) {
    unsigned long long x = 0;
#pragma unroll
    for (int w = 0; w < S_THREADS / 32; ++w) x += part[w][threadIdx.x];
    const int k = threadIdx.x;
    unsigned long long* dst = k < SND ? &totals->sumF[k] : k < 2 * SND ? &totals->nfE[k - SND]
                              : k < 3 * SND ? &totals->fE[k - 2 * SND] : &totals->suma;
    if (x) atomicAdd(dst, x);
  }
}

// s1b: one CTA turns block aggregates into exclusive block prefixes, 256 blocks at a time,
// and stops at the first block whose prefix already reaches every D's largest capacity
// (NF_all is non-decreasing, so from there on no free block is ever cached: s2 treats
// those blocks as saturated).
__global__ void __launch_bounds__(S_THREADS) s1_scan_kernel(Prefix8* blockagg, uint32_t nblocks,
                                                            const ChunkDev* __restrict__ chunk, ChunkTotals* totals) {
  typedef cub::BlockScan<Prefix8, S_THREADS> BS;
  __shared__ typename BS::TempStorage tmp;
  __shared__ Prefix8 carry;
  __shared__ int stop;
  const SatAdd add;
  if (threadIdx.x == 0) {
    carry = Prefix8{};
    stop = 0;
  }
  __syncthreads();
  uint32_t base = 0;
  for (; base < nblocks; base += S_THREADS) {
    const uint32_t i = base + threadIdx.x;
    Prefix8 v{};
    if (i < nblocks) v = blockagg[i];
    Prefix8 ex, agg;
    BS(tmp).ExclusiveScan(v, ex, Prefix8{}, add, agg);
    const Prefix8 c = carry;
    if (i < nblocks) blockagg[i] = add(c, ex);
    __syncthreads();
    if (threadIdx.x == 0) {
      carry = add(c, agg);
      bool sat = true;
      for (int d = 0; d < SND; ++d) sat &= carry.nf[d] >= chunk->Cmax[d];
      stop = sat;
    }
    __syncthreads();
    if (stop) {
      base += S_THREADS;
      break;
    }
  }
  if (threadIdx.x == 0) totals->nsat = min(base, nblocks);
}

// s2: one CTA = 256 consecutive request events.
//   A. natural order: event record, L_before, universe deltas -> block scan + block prefix
//      = NF_all(e), F_all(e) (saturated past nsat); window (p, e) split into chunks of
//      WCH events, numbered by a block scan;
//   B. the CTA's chunks are spread over all 256 threads (balanced): each chunk is scanned
//      backwards, branch-free, summing L and max(L, D) for D pairs in packed 16x2 registers
//      (exact: wch * max(L_after, D) < 2^16), then merged into per-event shared-memory
//      totals A_nf, A_f;
//   C. natural order again: b for every instance, instances grouped by D, coalesced stores.

constexpr uint32_t IT = 512;  // instance-table tile staged in shared memory by s2

template <int ND>
__global__ void __launch_bounds__(S_THREADS, 4) s2_main_kernel(const uint64_t* __restrict__ sim,
                                                            const uint64_t* __restrict__ scanrec, uint32_t E,
                                                            const ChunkDev* __restrict__ chunk,
                                                            const StackInstDev* __restrict__ insts,
                                                            const Prefix8* __restrict__ blockpre,
                                                            const ChunkTotals* __restrict__ totals, uint32_t wch,
                                                            uint32_t maxL, uint16_t* __restrict__ bout,
                                                            unsigned long long* sumXf) {
  constexpr int NP = (ND + 1) / 2;  // D pairs
  typedef cub::BlockScan<Prefix8, S_THREADS> BS;
  typedef cub::BlockScan<uint32_t, S_THREADS> BSu;
  __shared__ ChunkDev ch;
  struct InstTile {  // phase C instance-table tile (reuses the scan storage)
    uint64_t off[IT];
    uint32_t C[IT], inst[IT];
  };
  __shared__ union {
    typename BS::TempStorage scan;
    typename BSu::TempStorage scanu;
    InstTile it;
  } tmp;
  __shared__ uint32_t anf_s[ND][S_THREADS], af_s[ND][S_THREADS];
  __shared__ uint32_t p_s[S_THREADS], cbeg_s[S_THREADS + 1];
  __shared__ uint32_t J_s[S_THREADS], Lb_s[S_THREADS];
  __shared__ uint32_t nfall_s[ND][S_THREADS];
  if (threadIdx.x == 0) ch = *chunk;
  const uint32_t t = threadIdx.x;
#pragma unroll
  for (int d = 0; d < ND; ++d) anf_s[d][t] = af_s[d][t] = 0;
  __syncthreads();
  const uint32_t e0 = blockIdx.x * S_THREADS;
  const uint32_t e = e0 + t;
  uint64_t s = 0;
  uint32_t Lb = 0;
  Prefix8 v{};
  if (e < E) {
    s = __ldg(sim + e);
    Lb = L_before(sim, s);
    universe_delta(ch, Lb, sim_La(s), v);
  }
  // ---- A
  Prefix8 P;
  if (blockIdx.x < totals->nsat) {
    Prefix8 ex;
    BS(tmp.scan).ExclusiveScan(v, ex, Prefix8{}, SatAdd());
    P = SatAdd()(blockpre[blockIdx.x], ex);
  } else {
#pragma unroll
    for (int d = 0; d < SND; ++d) P.nf[d] = P.f[d] = 0xFFFFFFFFu;
  }
  const uint32_t p = (e < E) ? sim_prev(s) : TLRU_NONE;
  p_s[t] = p;
  J_s[t] = sim_J(s);
  Lb_s[t] = (p == TLRU_NONE) ? 0u : Lb;
#pragma unroll
  for (int d = 0; d < ND; ++d) nfall_s[d][t] = P.nf[d];
  const uint32_t wl = (p == TLRU_NONE) ? 0u : e - p - 1;
  uint32_t cb, ntot;
  __syncthreads();
  BSu(tmp.scanu).ExclusiveSum((wl + wch - 1) / wch, cb, ntot);
  cbeg_s[t] = cb;
  if (t == 0) cbeg_s[S_THREADS] = ntot;
  __syncthreads();
  // ---- B
  // window sums only see L <= maxL, so D can be clamped to maxL (<= 65535): max(L - D, 0) and
  // min(L, D) are unchanged for every L in the trace
  uint32_t Deff[ND], Dpk[NP];
#pragma unroll
  for (int d = 0; d < ND; ++d) Deff[d] = min(ch.D[d], maxL);
#pragma unroll
  for (int q = 0; q < NP; ++q) Dpk[q] = Deff[2 * q] | (Deff[min(2 * q + 1, ND - 1)] << 16);
  for (uint32_t it = t; it < ntot; it += S_THREADS) {
    uint32_t lo = 0, hi = S_THREADS;  // owner event: last j with cbeg_s[j] <= it
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (cbeg_s[mid] <= it) lo = mid; else hi = mid;
    }
    const uint32_t j = lo, ej = e0 + j, pj = p_s[j];
    const uint32_t top = ej - 1 - (it - cbeg_s[j]) * wch;          // chunk covers [bot, top]
    const uint32_t bot = max(pj + 1, top >= wch - 1 ? top - (wch - 1) : 0u);
    // Branch-free: a dead element (its conversation returns before ej) counts as L = 0.
    // Per D pair accumulate sum max(L, D) (16x2); with n = elements in the chunk:
    //   A_nf = sum max(L, D) - n D,   A_f = sum L + n D - sum max(L, D)   (max + min = L + D)
    uint32_t mx2[NP], sumL = 0;
#pragma unroll
    for (int q = 0; q < NP; ++q) mx2[q] = 0;
    for (uint32_t x = top + 1; x-- > bot;) {
      const uint64_t r = __ldg(scanrec + x);
      const uint32_t L = static_cast<uint32_t>(r) > ej ? static_cast<uint32_t>(r >> 32) : 0u;
      sumL += L;
      const uint32_t L2 = L * 0x10001u;  // L in both 16-bit halves
#pragma unroll
      for (int q = 0; q < NP; ++q) mx2[q] = __vadd2(mx2[q], __vmaxu2(L2, Dpk[q]));
    }
    const uint32_t n = top + 1 - bot;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int d = 2 * q + h;
        if (d < ND) {
          const uint32_t smax = h ? (mx2[q] >> 16) : (mx2[q] & 0xFFFFu);
          const uint32_t nD = n * Deff[d];
          atomicAdd(&anf_s[d][j], smax - nD);
          atomicAdd(&af_s[d][j], sumL + nD - smax);
        }
      }
    }
  }
  __syncthreads();
  // ---- C: per-instance b (P:154-156 with the closed form of X_theta).  Thread t writes 4
  // consecutive events (one 8-byte store when the instance row is 8-byte aligned) for every
  // fourth instance of each D.
  const uint32_t quad = t & 63, lane4 = t >> 6;
  const uint32_t j0 = quad * 4;
  const bool full = e0 + j0 + 3 < E;
  const bool saturated = blockIdx.x >= totals->nsat;  // NF_all >= every C here: no free blocks cached
  uint32_t Jv[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) Jv[u] = J_s[j0 + u];
  const uint32_t J01 = Jv[0] | (Jv[1] << 16), J23 = Jv[2] | (Jv[3] << 16);
  // The chunk's instance table goes through shared memory in tiles of IT entries.
  for (uint32_t tb = 0; tb < ch.ninst; tb += IT) {
    const uint32_t te = min(ch.ninst, tb + IT);
    __syncthreads();
    for (uint32_t k = tb + t; k < te; k += S_THREADS) {
      const StackInstDev in = insts[ch.inst0 + k];
      tmp.it.C[k - tb] = in.C;
      tmp.it.inst[k - tb] = in.inst;
      tmp.it.off[k - tb] = in.boff;
    }
    __syncthreads();
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      const uint32_t kb = max(ch.dbeg[d], tb), ke = min(ch.dbeg[d + 1], te);
      if (kb >= ke) continue;
      uint32_t nfb[4], fb[4], anf[4], af[4], nfa[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool hit = p_s[j0 + u] != TLRU_NONE;
        const uint32_t Lbu = Lb_s[j0 + u];
        nfb[u] = hit ? nf_of(Lbu, ch.D[d]) : 0u;
        fb[u] = hit ? f_of(Lbu, ch.D[d]) : 0u;
        anf[u] = anf_s[d][j0 + u];
        af[u] = af_s[d][j0 + u];
        nfa[u] = nfall_s[d][j0 + u];
      }
      // packed 16x2 operands for capacities <= 65535: X = min(nfb, max(C, A) - A) with A = A_nf
      // clamped to 65535 (exact: if A > 65535 >= C then both sides give 0)
      const uint32_t A01 = min(anf[0], 65535u) | (min(anf[1], 65535u) << 16);
      const uint32_t A23 = min(anf[2], 65535u) | (min(anf[3], 65535u) << 16);
      const uint32_t N01 = nfb[0] | (nfb[1] << 16), N23 = nfb[2] | (nfb[3] << 16);
#pragma unroll 4
      for (uint32_t k = kb + lane4; k < ke; k += 4) {
        const uint32_t C = tmp.it.C[k - tb];
        uint32_t w01, w23;
        if (saturated && C <= 65535u) {
          const uint32_t C2 = C * 0x10001u;
          w01 = __vsub2(J01, __vminu2(N01, __vsub2(__vmaxu2(C2, A01), A01)));
          w23 = __vsub2(J23, __vminu2(N23, __vsub2(__vmaxu2(C2, A23), A23)));
        } else {
          uint32_t b[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint32_t X = min(nfb[u], sat_sub(C, anf[u]));
            if (!saturated && nfa[u] < C && fb[u] > 0) {  // warm-up: free blocks can still be cached
              const uint32_t xf = min(fb[u], sat_sub(sat_sub(C, nfa[u]), af[u]));
              X += xf;
              if (xf && e0 + j0 + u < E)
                atomicAdd(&sumXf[tmp.it.inst[k - tb]], static_cast<unsigned long long>(xf));
            }
            b[u] = Jv[u] - X;
          }
          w01 = b[0] | (b[1] << 16);
          w23 = b[2] | (b[3] << 16);
        }
        uint16_t* row = bout + tmp.it.off[k - tb] + e0 + j0;
        if (full && ((reinterpret_cast<uintptr_t>(row) & 7u) == 0)) {
          *reinterpret_cast<uint2*>(row) = make_uint2(w01, w23);
        } else {
          const uint32_t bb[4] = {w01 & 0xFFFFu, w01 >> 16, w23 & 0xFFFFu, w23 >> 16};
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (e0 + j0 + u < E) row[u] = static_cast<uint16_t>(bb[u]);
        }
      }
    }
  }
}

__global__ void s3_results_kernel(const StackInstDev* __restrict__ insts, uint32_t ninst,
                                  const uint32_t* __restrict__ inst_chunk, const ChunkTotals* __restrict__ totals,
                                  const unsigned long long* sumXf, tlru_result* results) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < ninst; k += gridDim.x * blockDim.x) {
    const StackInstDev in = insts[k];
    const ChunkTotals& T = totals[inst_chunk[k]];
    const unsigned long long nfE = T.nfE[in.d], fE = T.fE[in.d], C = in.C;
    const unsigned long long U = nfE + fE;
    const unsigned long long used_final = U < C ? U : C;
    const unsigned long long room = C > nfE ? C - nfE : 0ull;
    const unsigned long long fc_final = fE < room ? fE : room;
    tlru_result& r = results[in.inst];
    const unsigned long long total = T.suma + r.sum_uncached - used_final;  // telescoped evictions
    const unsigned long long trim = T.sumF[in.d] - sumXf[in.inst] - fc_final;
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
      for (uint32_t d = 0; d < ch.dev.nd; ++d) {
        ch.dev.dbeg[d] = static_cast<uint32_t>(P->insts.size()) - ch.dev.inst0;
        for (uint32_t i : ids) {
          if (Dof(i) != ch.dev.D[d]) continue;
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
      for (uint32_t d = ch.dev.nd; d <= SND; ++d) ch.dev.dbeg[d] = static_cast<uint32_t>(P->insts.size()) - ch.dev.inst0;
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
  unsigned long long* sumXf;
  Prefix8* blockpre;  // [chunk][block] exclusive block prefixes
  uint64_t* scanrec;  // [event] next | L_after << 32 of the trace being processed
  uint64_t nblocks_max;
};

static void carve_stack(Carver& cv, const StackPlan& P, uint32_t ni, StackWs* w) {
  const size_t nc = P.chunks.size() + 1;
  w->chunks = cv.take<ChunkDev>(nc);
  w->insts = cv.take<StackInstDev>(P.insts.size() + 1);
  w->inst_chunk = cv.take<uint32_t>(P.insts.size() + 1);
  w->totals = cv.take<ChunkTotals>(nc);
  w->sumXf = cv.take<unsigned long long>(ni + 1);
  w->nblocks_max = (P.Emax + S_THREADS - 1) / S_THREADS + 1;
  w->blockpre = cv.take<Prefix8>(nc * w->nblocks_max);
  w->scanrec = cv.take<uint64_t>(P.Emax + 1);
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
static void launch_s2(const tlru_trace& tr, const ChunkDev* ch, const ChunkDev& ch_host, const Prefix8* blockpre,
                      const ChunkTotals* tot, const StackWs& w, uint16_t* bout, cudaStream_t st) {
  const uint32_t E = static_cast<uint32_t>(tr.num_events);
  // 16x2 partial sums of max(L, min(D, maxL)) stay exact while wch * maxL < 2^16
  const uint32_t maxL = std::max<uint32_t>(tr.max_history, 1u);
  const uint32_t wch = std::max<uint32_t>(1u, std::min<uint32_t>(64u, 65535u / maxL));
  (void)ch_host;
  s2_main_kernel<ND><<<(E + S_THREADS - 1) / S_THREADS, S_THREADS, 0, st>>>(tr.sim, w.scanrec, E, ch, w.insts,
                                                                            blockpre, tot, wch, maxL, bout, w.sumXf);
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
  for (size_t c = 0; c < nc; ++c) chd[c] = P.chunks[c].dev;
  if (nc) {
    TLRU_CUDA(cudaMemcpyAsync(w.chunks, chd.data(), nc * sizeof(ChunkDev), cudaMemcpyHostToDevice, st));
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
    s1_block_kernel<<<std::min<uint32_t>(nb ? nb : 1, 148u * 4u), S_THREADS, 0, st>>>(tr.sim, tr.next, E, w.chunks + c,
                                                                                     w.scanrec, bp, w.totals + c);
    TLRU_CHECK_LAUNCH();
    s1_scan_kernel<<<1, S_THREADS, 0, st>>>(bp, nb, w.chunks + c, w.totals + c);
    TLRU_CHECK_LAUNCH();
    switch (P.chunks[c].dev.nd) {
      case 1: launch_s2<1>(tr, w.chunks + c, P.chunks[c].dev, bp, w.totals + c, w, bout, st); break;
      case 2: launch_s2<2>(tr, w.chunks + c, P.chunks[c].dev, bp, w.totals + c, w, bout, st); break;
      case 3: launch_s2<3>(tr, w.chunks + c, P.chunks[c].dev, bp, w.totals + c, w, bout, st); break;
      case 4: launch_s2<4>(tr, w.chunks + c, P.chunks[c].dev, bp, w.totals + c, w, bout, st); break;
      case 5: launch_s2<5>(tr, w.chunks + c, P.chunks[c].dev, bp, w.totals + c, w, bout, st); break;
      case 6: launch_s2<6>(tr, w.chunks + c, P.chunks[c].dev, bp, w.totals + c, w, bout, st); break;
      case 7: launch_s2<7>(tr, w.chunks + c, P.chunks[c].dev, bp, w.totals + c, w, bout, st); break;
      default: launch_s2<8>(tr, w.chunks + c, P.chunks[c].dev, bp, w.totals + c, w, bout, st); break;
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
                                                                     w.inst_chunk, w.totals, w.sumXf, results);
    TLRU_CHECK_LAUNCH();
  }
  *nkernels += 3;
  return TLRU_OK;
}

}  // namespace tlru
