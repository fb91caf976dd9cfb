// stack.cu -- "stack" engine of tlru_simulate_batch: exact closed-form evaluation of
// Alg. 1 for every capacity at once.
//
// By the stack property the cache after each request is the top-C
// blocks of the universe under the key (non-free?, tau, -position), D = max(xi - Q_hat, 0)
// (free tail, P:56 / P:62), NF(L) = max(L - D, 0), F(L) = min(L, D).  For the request e
// of conversation theta with previous turn p (history Lb = L_after[p]):
//   A_nf(e) = sum NF(L_x), A_f(e) = sum F(L_x) over x in (p, e) with next[x] > e
//             (the conversations used after theta's previous turn, each at its latest L),
//   NF_all(e) = the same non-free sum over every conversation's last turn before e,
//   X_theta = min(NF(Lb), (C - A_nf)^+) + min(F(Lb), (C - NF_all - A_f)^+),
//   b = J - X_theta
// and, telescoping Alg. 1's per-request evictions over the trace (used and the cached
// free blocks are functions of the universe: used = min(C, U), Fc = min(F_all, (C-NF_all)^+)):
//   evicted_total = sum a + sum b - min(C, U_final)
//   evicted_trim  = sum_e F(L_after_e) - sum_e X_f(e) - Fc_final       (Phase 1)
//   evicted_lru   = evicted_total - evicted_trim                        (Phase 2)
//   max_occupancy = min(C, U_final)
// Pinned against the oracle by tests/test_gpu_parity.py (both engines, every config).
//
// Kernels per (trace, chunk of <= 24 distinct D):
//   s1_block  : per event the scan record (next | L_after << 32); per 256-event block the
//               growth of NF_all for every D; histograms of L_after over all events and over
//               final turns (for the exact totals); sum a
//   s1_totals : one CTA: exact totals per D from the histograms, and per D the block prefixes
//               of NF_all up to nsat[d] = the first block from which NF_all >= the largest
//               capacity of that D (NF_all is non-decreasing): no free block is cached after it
//   s2_warm   : (block, D) pairs before nsat[d]: the general closed form (exact NF_all, free blocks)
//   s2_sat    : (block, D) pairs from nsat[d]: one CTA = 256 events: (A) window lengths; (B) every
//               window (p, e) cut into <= 64-event chunks spread over all 256 threads,
//               scanned branch-free with sum max(L, D) for D pairs in packed 16x2 registers;
//               (C) b for every instance, 4 events per thread, packed 16x2 arithmetic,
//               8-byte stores, instance table staged in shared memory
//   s3_results: eviction counters and occupancy from the telescoped identities
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "metrics.cuh"
#include "stack.cuh"

namespace tlru {

constexpr int SND = 24;         // D values per chunk
constexpr int S_THREADS = 256;  // events per s2 block
constexpr uint32_t IT = 512;    // instance-table tile staged in shared memory by s2
constexpr uint32_t WCH_MAX = 64;
#ifndef TLRU_WIN_G
#define TLRU_WIN_G 1
#endif
constexpr int WIN_G = TLRU_WIN_G;  // threads per window chunk in s2_win (window_phase)
constexpr uint32_t GI_MAX = 64;                     // instances per s2_out group (hard limit)
// Measured on B200 (config-5 sweep): groups of 13..24 instances are fastest.  Each CTA writes
// one 16-byte store per instance row per 8 events, and the write stream loses DRAM efficiency
// as the number of rows a CTA interleaves grows (tools/write_bw.cu: 7.4 TB/s with one row per
// CTA, 5.9-6.9 with 8, 4.9 with 35); smaller groups re-read the per-event inputs more often.
#ifndef TLRU_GI_CAP
#define TLRU_GI_CAP 16u
#endif
constexpr uint32_t GI_CAP = TLRU_GI_CAP;
constexpr uint32_t OUT_SMEM = 54u * 1024u;          // s2_out dynamic smem budget: 4 CTAs per SM
#ifndef TLRU_OUT_RANGE
#define TLRU_OUT_RANGE (31u * 1024u)
#endif
constexpr uint32_t OUT_RANGE_MAX = TLRU_OUT_RANGE;  // events per s2_out CTA (<= 31744: 16-bit counters)
static_assert(OUT_RANGE_MAX <= 31u * 1024u && OUT_RANGE_MAX % 1024u == 0, "s2_out range");
#ifndef TLRU_OUT_WRANGE
#define TLRU_OUT_WRANGE 32768u  // measured: 2048 / 4096 / 8192 -> s2_out 1.21 / 1.02 / 0.92 ms vs 0.87 (no split)
#endif
constexpr uint32_t OUT_WRANGE = TLRU_OUT_WRANGE;  // s2_out writer groups: events per CTA (a multiple of 2048)
#ifndef TLRU_WIN_EVICT_LAST
#define TLRU_WIN_EVICT_LAST 1  // measured: s2_win 0.331 -> 0.308 ms per trace, step -0.2 ms
#endif
#ifndef TLRU_B_EVICT_FIRST
#define TLRU_B_EVICT_FIRST 1  // measured: s2_out 0.884 -> 0.875 ms per trace
#endif
constexpr uint32_t TAB_MAX = 8192;                  // s2_out count table covers capacities < TAB_MAX

struct ChunkDev {
  uint32_t D[SND];
  uint32_t Cmax[SND];      // largest capacity among the chunk's instances with this D
  uint32_t dbeg[SND + 1];  // instances of D[d]: [inst0 + dbeg[d], inst0 + dbeg[d+1]), sorted by C
  uint32_t dbig[SND];      // first instance of D[d] with C > 65535 (packed 16x2 path before it)
  uint32_t T[SND];         // Threshold-LRU admission threshold of the row (0: LRU / T-LRU row)
  uint32_t nd;             // real rows (the rest pad with row 0 and own no instances)
  uint32_t anyT;           // some row has T > 0
  uint32_t inst0, ninst;   // instances [inst0, inst0 + ninst) of the StackInstDev table
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
  unsigned long long suma_adm[SND];  // T rows: sum of a over admitted events (L_after >= T)
  unsigned long long sumJ_na[SND];   // T rows: sum of J over the other events (b = J there)
  uint32_t nsat[SND];            // first 256-event block where NF_all(D[d]) >= Cmax[d]
  uint32_t nsat_min, nsat_max;   // over the real D values
};

__device__ __forceinline__ uint32_t nf_of(uint32_t L, uint32_t D) { return L > D ? L - D : 0u; }
__device__ __forceinline__ uint32_t f_of(uint32_t L, uint32_t D) { return L < D ? L : D; }
// Cached-by-recency weight of a history of length L in a row (D, T): NF(L) = max(L - D, 0), and
// for Threshold-LRU rows (D = 0, T > 0) only admitted histories count: L [L >= T] (Reading #23).
__device__ __forceinline__ uint32_t nft(uint32_t L, uint32_t D, uint32_t T) { return L >= T ? nf_of(L, D) : 0u; }
__device__ __forceinline__ uint32_t sat_sub(uint32_t a, uint32_t b) { return a > b ? a - b : 0u; }

__device__ __forceinline__ uint32_t L_before(const uint64_t* sim, uint64_t s) {
  const uint32_t p = sim_prev(s);
  return p == TLRU_NONE ? 0u : sim_La(__ldg(sim + p));
}

// ----------------------------------------------------------------------------- s1
// Persistent grid over 256-event blocks: scan records, per-block growth of NF_all for every D
// (blockagg[blk * SND + d]), L_after histograms (all events / final turns) and sum a.
__global__ void __launch_bounds__(S_THREADS) s1_block_kernel(const uint64_t* __restrict__ sim,
                                                             const uint32_t* __restrict__ next, uint32_t E,
                                                             const ChunkDev* __restrict__ chunk,
                                                             uint64_t* __restrict__ scanrec,
                                                             uint32_t* __restrict__ blockagg, uint32_t bins,
                                                             uint32_t* hist_all, uint32_t* hist_last,
                                                             ChunkTotals* totals) {
  extern __shared__ uint32_t sh[];  // [2 * bins] when bins fit, else unused
  __shared__ uint32_t wsum[S_THREADS / 32][SND];
  __shared__ uint32_t Ds[SND], Ts[SND];
  __shared__ unsigned long long acc_a[SND], acc_j[SND];  // T rows: admitted a, non-admitted J
  const bool smem_hist = bins <= 8192;
  uint32_t* ha = smem_hist ? sh : hist_all;
  uint32_t* hl = smem_hist ? sh + bins : hist_last;
  if (smem_hist)
    for (uint32_t k = threadIdx.x; k < 2 * bins; k += S_THREADS) sh[k] = 0;
  if (threadIdx.x < SND) {
    Ds[threadIdx.x] = chunk->D[threadIdx.x];
    Ts[threadIdx.x] = chunk->T[threadIdx.x];
    acc_a[threadIdx.x] = acc_j[threadIdx.x] = 0ull;
  }
  const uint32_t nd = chunk->nd;
  const bool anyT = chunk->anyT != 0;
  __syncthreads();
  unsigned long long sa = 0;
  const uint32_t nblocks = (E + S_THREADS - 1) / S_THREADS;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (uint32_t blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
    const uint32_t e = blk * S_THREADS + threadIdx.x;
    uint32_t La = 0, Lb = 0, Jv = 0;
    if (e < E) {
      const uint64_t s = __ldg(sim + e);
      Jv = sim_J(s);
      const uint32_t nx = __ldg(next + e);
      La = sim_La(s);
      Lb = L_before(sim, s);
      scanrec[e] = uint64_t(nx) | (uint64_t(La) << 32);
      sa += La - sim_J(s);
      atomicAdd(&ha[La], 1u);
      if (nx == TLRU_NONE) atomicAdd(&hl[La], 1u);
    }
    for (uint32_t d = 0; d < nd; ++d) {  // growth of NF_all for row d; <= 256 * 65535: no overflow
      const uint32_t v = __reduce_add_sync(0xFFFFFFFFu, nft(La, Ds[d], Ts[d]) - nft(Lb, Ds[d], Ts[d]));
      if (lane == 0) wsum[warp][d] = v;
    }
    if (anyT)
      for (uint32_t d = 0; d < nd; ++d) {  // Threshold-LRU rows: inputs of the eviction identity
        if (Ts[d] == 0) continue;
        const bool adm = La >= Ts[d];
        const uint32_t va = __reduce_add_sync(0xFFFFFFFFu, (e < E && adm) ? La - Jv : 0u);
        const uint32_t vj = __reduce_add_sync(0xFFFFFFFFu, (e < E && !adm) ? Jv : 0u);
        if (lane == 0) {
          if (va) atomicAdd(&acc_a[d], static_cast<unsigned long long>(va));
          if (vj) atomicAdd(&acc_j[d], static_cast<unsigned long long>(vj));
        }
      }
    __syncthreads();
    if (threadIdx.x < nd) {
      uint32_t v = 0;
#pragma unroll
      for (int w = 0; w < S_THREADS / 32; ++w) v += wsum[w][threadIdx.x];
      blockagg[uint64_t(blk) * SND + threadIdx.x] = v;
    }
    __syncthreads();
  }
  if (smem_hist) {
    for (uint32_t k = threadIdx.x; k < bins; k += S_THREADS) {
      if (sh[k]) atomicAdd(&hist_all[k], sh[k]);
      if (sh[bins + k]) atomicAdd(&hist_last[k], sh[bins + k]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sa += __shfl_xor_sync(0xFFFFFFFFu, sa, o);
  if (lane == 0 && sa) atomicAdd(&totals->suma, sa);
  if (anyT) {
    __syncthreads();
    if (threadIdx.x < nd && Ts[threadIdx.x]) {
      if (acc_a[threadIdx.x]) atomicAdd(&totals->suma_adm[threadIdx.x], acc_a[threadIdx.x]);
      if (acc_j[threadIdx.x]) atomicAdd(&totals->sumJ_na[threadIdx.x], acc_j[threadIdx.x]);
    }
  }
}

// One CTA: exact totals per D from the L_after histograms; then, one warp per D, the block
// prefixes of NF_all(D) (in place, exclusive) up to nsat[d] = the first block whose prefix
// reaches Cmax[d] (NF_all is non-decreasing, so no free block of that D is cached after it).
constexpr int T_THREADS = 32 * SND;

__global__ void __launch_bounds__(T_THREADS) s1_totals_kernel(const ChunkDev* __restrict__ chunk, uint32_t bins,
                                                              const uint32_t* __restrict__ hist_all,
                                                              const uint32_t* __restrict__ hist_last,
                                                              uint32_t* __restrict__ blockagg, uint32_t nblocks,
                                                              ChunkTotals* totals) {
  typedef cub::BlockReduce<unsigned long long, T_THREADS> BR;
  __shared__ typename BR::TempStorage red;
  __shared__ uint32_t ns_s[SND];
  const ChunkDev& ch = *chunk;
  for (int d = 0; d < SND; ++d) {
    const uint32_t D = ch.D[d], Tt = ch.T[d];
    unsigned long long sF = 0, nE = 0, fE = 0;
    for (uint32_t L = threadIdx.x; L < bins; L += T_THREADS) {
      const unsigned long long a = hist_all[L], l = hist_last[L];
      sF += a * f_of(L, D);
      nE += l * nft(L, D, Tt);
      fE += l * f_of(L, D);
    }
    sF = BR(red).Sum(sF);
    __syncthreads();
    nE = BR(red).Sum(nE);
    __syncthreads();
    fE = BR(red).Sum(fE);
    __syncthreads();
    if (threadIdx.x == 0) {
      totals->sumF[d] = sF;
      totals->nfE[d] = nE;
      totals->fE[d] = fE;
    }
  }
  const uint32_t d = threadIdx.x / 32, lane = threadIdx.x & 31;
  uint32_t nsat = 0;
  if (d < ch.nd) {
    const unsigned long long cmax = ch.Cmax[d];
    unsigned long long carry = 0;
    nsat = nblocks;
    for (uint32_t base = 0; base < nblocks; base += 32) {
      const uint32_t i = base + lane;
      const unsigned long long v = i < nblocks ? blockagg[uint64_t(i) * SND + d] : 0ull;
      unsigned long long inc = v;  // warp inclusive scan
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= o) inc += y;
      }
      const unsigned long long start = carry + inc - v;  // NF_all(D[d]) at the first event of block i
      const unsigned hit = __ballot_sync(0xFFFFFFFFu, i < nblocks && start >= cmax);
      if (i < nblocks) blockagg[uint64_t(i) * SND + d] = static_cast<uint32_t>(start < 0xFFFFFFFFull ? start
                                                                                                    : 0xFFFFFFFFull);
      if (hit) {
        nsat = base + __ffs(hit) - 1;
        break;
      }
      carry += __shfl_sync(0xFFFFFFFFu, inc, 31);
    }
  }
  if (lane == 0 && d < SND) ns_s[d] = d < ch.nd ? nsat : 0u;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t lo = nblocks, hi = 0;
    for (uint32_t k = 0; k < ch.nd; ++k) {
      totals->nsat[k] = ns_s[k];
      lo = min(lo, ns_s[k]);
      hi = max(hi, ns_s[k]);
    }
    for (uint32_t k = ch.nd; k < SND; ++k) totals->nsat[k] = 0;
    totals->nsat_min = ch.nd ? lo : 0u;
    totals->nsat_max = hi;
  }
}

// ----------------------------------------------------------------------------- s2 common
// Phase B of the s2 kernels: groups of G adjacent threads take window chunks `it` of the block
// and accumulate, branch-free, sum L and sum max(L, Deff) per D pair over the chunk.  Lane l of a
// group reads the chunk's elements top - l, top - l - G, ..., so a group's loads are G
// consecutive 8-byte records (G = 1: one thread per chunk, each lane of a warp on its own line --
// the L1/TEX-bound form); the group's partial sums are then added by G - 1 xor-shuffles and its
// lanes share the chunk's shared-memory atomics.
// HT: the chunk has Threshold-LRU rows; element L then counts only where L >= T (T = 0 on the
// other rows), and those rows (D = 0) have no free blocks.
template <int ND, bool WITH_F, bool HT, int G = 1>
__device__ __forceinline__ void window_phase(const uint64_t* __restrict__ scanrec, uint32_t e0, uint32_t wch,
                                             const uint32_t* p_s, const uint32_t* cbeg_s, uint32_t ntot,
                                             const uint32_t* Deff, const uint32_t* Tr,
                                             uint32_t (*anf_s)[S_THREADS], uint32_t (*af_s)[S_THREADS]) {
  static_assert(G >= 1 && G <= 32 && (G & (G - 1)) == 0, "G: a power of two <= 32");
  constexpr int NP = (ND + 1) / 2;
  constexpr uint32_t NG = S_THREADS / G;  // groups per CTA
  uint32_t Dpk[NP], Tpk[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    Dpk[q] = Deff[2 * q] | (Deff[min(2 * q + 1, ND - 1)] << 16);
    Tpk[q] = HT ? (Tr[2 * q] | (Tr[min(2 * q + 1, ND - 1)] << 16)) : 0u;  // T <= 65535 (validated)
  }
  const uint32_t lane = threadIdx.x % G, grp = threadIdx.x / G;
  // G > 1: every thread runs the same number of rounds (the shuffles need whole warps)
  const uint32_t rounds = G > 1 ? (ntot + NG - 1) / NG : 0u;
  for (uint32_t r = 0, it = grp; G > 1 ? r < rounds : it < ntot; ++r, it += NG) {
    uint32_t j = 0, ej = 0, top = 0, n = 0;
    if (it < ntot) {
      uint32_t lo = 0, hi = S_THREADS;  // owner event: last j with cbeg_s[j] <= it
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (cbeg_s[mid] <= it) lo = mid; else hi = mid;
      }
      j = lo;
      ej = e0 + j;
      const uint32_t pj = p_s[j];
      top = ej - 1 - (it - cbeg_s[j]) * wch;  // chunk covers [bot, top]
      const uint32_t bot = max(pj + 1, top >= wch - 1 ? top - (wch - 1) : 0u);
      n = top + 1 - bot;
    }
    // a dead element (its conversation returns before ej) counts as L = 0; with n elements:
    //   A_nf = sum max(L, D) - n D,   A_f = sum L + n D - sum max(L, D)   (max + min = L + D)
    uint32_t mx2[NP], sumL = 0;
#pragma unroll
    for (int q = 0; q < NP; ++q) mx2[q] = 0;
    for (uint32_t k = lane; k < n; k += G) {
      const uint64_t r_ = __ldg(scanrec + (top - k));
      const uint32_t L = static_cast<uint32_t>(r_) > ej ? static_cast<uint32_t>(r_ >> 32) : 0u;
      if (WITH_F) sumL += L;
      const uint32_t L2 = L * 0x10001u;  // L in both 16-bit halves
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        if (HT) mx2[q] = __vadd2(mx2[q], __vmaxu2(L2, Dpk[q]) & __vcmpgeu2(L2, Tpk[q]));
        else mx2[q] = __vadd2(mx2[q], __vmaxu2(L2, Dpk[q]));
      }
    }
    if (G > 1) {  // the chunk's sums (< 2^16 per half: wch * maxL < 2^16)
#pragma unroll
      for (int o = 1; o < G; o <<= 1) {
#pragma unroll
        for (int q = 0; q < NP; ++q) mx2[q] = __vadd2(mx2[q], __shfl_xor_sync(0xFFFFFFFFu, mx2[q], o));
        if (WITH_F) sumL += __shfl_xor_sync(0xFFFFFFFFu, sumL, o);
      }
    }
    if (n == 0) continue;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int d = 2 * q + h;
        if (d < ND && (G == 1 || d % G == static_cast<int>(lane))) {
          const uint32_t smax = h ? (mx2[q] >> 16) : (mx2[q] & 0xFFFFu);
          const uint32_t nD = n * Deff[d];
          atomicAdd(&anf_s[d][j], smax - nD);
          if (WITH_F && !(HT && Tr[d] > 0)) atomicAdd(&af_s[d][j], sumL + nD - smax);
        }
      }
    }
  }
}

// Phase A shared by both s2 kernels: event record, L_before, window length -> chunk numbering.
__device__ __forceinline__ uint32_t block_setup(const uint64_t* __restrict__ sim, uint32_t E, uint32_t e0,
                                                uint32_t wch, uint32_t* p_s, uint32_t* J_s, uint32_t* Lb_s,
                                                uint32_t* cbeg_s, uint32_t& Lb_out, uint64_t& s_out,
                                                typename cub::BlockScan<uint32_t, S_THREADS>::TempStorage& tmp) {
  const uint32_t t = threadIdx.x, e = e0 + t;
  uint64_t s = 0;
  uint32_t Lb = 0;
  if (e < E) {
    s = __ldg(sim + e);
    Lb = L_before(sim, s);
  }
  const uint32_t p = (e < E) ? sim_prev(s) : TLRU_NONE;
  p_s[t] = p;
  J_s[t] = sim_J(s);
  Lb_s[t] = Lb;
  const uint32_t wl = (p == TLRU_NONE) ? 0u : e - p - 1;
  uint32_t cb, ntot;
  cub::BlockScan<uint32_t, S_THREADS>(tmp).ExclusiveSum((wl + wch - 1) / wch, cb, ntot);
  cbeg_s[t] = cb;
  if (t == 0) cbeg_s[S_THREADS] = ntot;
  Lb_out = Lb;
  s_out = s;
  return ntot;
}

__device__ __forceinline__ void store4(uint16_t* row, bool full, uint32_t w01, uint32_t w23, uint32_t e_first,
                                       uint32_t E) {
  if (full && ((reinterpret_cast<uintptr_t>(row) & 7u) == 0)) {
    *reinterpret_cast<uint2*>(row) = make_uint2(w01, w23);
  } else {
    const uint32_t bb[4] = {w01 & 0xFFFFu, w01 >> 16, w23 & 0xFFFFu, w23 >> 16};
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (e_first + u < E) row[u] = static_cast<uint16_t>(bb[u]);
  }
}

struct InstTile {
  uint64_t off[IT];
  uint32_t C[IT];  // C * 0x10001 (both 16-bit halves) on the packed path, C on the big-C path
};

struct InstTileW {
  uint64_t off[IT];
  uint32_t C[IT], inst[IT];
};

// ----------------------------------------------------------------------------- s2_sat
template <int ND, bool HT>
__global__ void __launch_bounds__(S_THREADS, 4) s2_sat_kernel(const uint64_t* __restrict__ sim,
                                                              const uint64_t* __restrict__ scanrec, uint32_t E,
                                                              const ChunkDev* __restrict__ chunk,
                                                              const StackInstDev* __restrict__ insts,
                                                              const ChunkTotals* __restrict__ totals, uint32_t wch,
                                                              uint32_t maxL, bool aligned,
                                                              uint16_t* __restrict__ bout) {
  typedef cub::BlockScan<uint32_t, S_THREADS> BSu;
  __shared__ ChunkDev ch;
  __shared__ union {
    typename BSu::TempStorage scan;
    InstTile it;
  } tmp;
  __shared__ uint32_t anf_s[ND][S_THREADS];
  __shared__ uint32_t p_s[S_THREADS], cbeg_s[S_THREADS + 1], J_s[S_THREADS], Lb_s[S_THREADS];
  if (blockIdx.x < totals->nsat_min) return;  // no D is saturated yet: s2_warm owns the block
  __shared__ uint32_t nsat_s[SND];
  if (threadIdx.x < SND) nsat_s[threadIdx.x] = totals->nsat[threadIdx.x];
  const uint32_t t = threadIdx.x;
  if (t == 0) ch = *chunk;
#pragma unroll
  for (int d = 0; d < ND; ++d) anf_s[d][t] = 0;
  const uint32_t e0 = blockIdx.x * S_THREADS;
  uint32_t Lb;
  uint64_t s;
  const uint32_t ntot = block_setup(sim, E, e0, wch, p_s, J_s, Lb_s, cbeg_s, Lb, s, tmp.scan);
  __syncthreads();
  // window sums only see L <= maxL, so D can be clamped to maxL (<= 65535): max(L - D, 0) and
  // min(L, D) are unchanged for every L in the trace
  uint32_t Deff[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) Deff[d] = min(ch.D[d], maxL);
  window_phase<ND, false, HT>(scanrec, e0, wch, p_s, cbeg_s, ntot, Deff, ch.T, anf_s, nullptr);
  // ---- C: per-instance b; X = min(NF(Lb), (C - A_nf)^+) (no free block is cached here)
  const uint32_t quad = t & 63, lane4 = t >> 6;
  const uint32_t j0 = quad * 4;
  const bool full = e0 + j0 + 3 < E;
  uint32_t Jv[4];
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 4; ++u) Jv[u] = J_s[j0 + u];
  const uint32_t J01 = Jv[0] | (Jv[1] << 16), J23 = Jv[2] | (Jv[3] << 16);
  constexpr uint32_t j0_base = 0;  // tile offsets already include e0; each thread adds its j0
  const uint32_t joff = j0;
  const bool vec = full && aligned;  // every instance row offset is a multiple of 4 requests
  for (uint32_t tb = 0; tb < ch.ninst; tb += IT) {
    const uint32_t te = min(ch.ninst, tb + IT);
    __syncthreads();
    for (uint32_t k = tb + t; k < te; k += S_THREADS) {
      const StackInstDev in = insts[ch.inst0 + k];
      tmp.it.C[k - tb] = in.C <= 65535u ? in.C * 0x10001u : in.C;
      tmp.it.off[k - tb] = in.boff + e0 + j0_base;
    }
    __syncthreads();
#pragma unroll 1
    for (int d = 0; d < ND; ++d) {  // runtime loop: a fully unrolled one overflows the instruction cache
      const uint32_t kb = max(ch.dbeg[d], tb), ke = min(ch.dbeg[d + 1], te);
      if (kb >= ke || blockIdx.x < nsat_s[d]) continue;  // D[d] still in warm-up here: s2_warm
      uint32_t nfb[4], anf[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        nfb[u] = p_s[j0 + u] != TLRU_NONE ? nft(Lb_s[j0 + u], ch.D[d], ch.T[d]) : 0u;
        anf[u] = anf_s[d][j0 + u];
      }
      // packed 16x2: X = min(nfb, max(C, A) - A), A clamped to 65535 (exact for C <= 65535)
      const uint32_t A01 = min(anf[0], 65535u) | (min(anf[1], 65535u) << 16);
      const uint32_t A23 = min(anf[2], 65535u) | (min(anf[3], 65535u) << 16);
      const uint32_t N01 = nfb[0] | (nfb[1] << 16), N23 = nfb[2] | (nfb[3] << 16);
      const uint32_t kmid = min(max(ch.dbig[d], kb), ke);
      if (vec) {
#pragma unroll 4
        for (uint32_t k = kb + lane4; k < kmid; k += 4) {
          const uint32_t C2 = tmp.it.C[k - tb];
          const uint32_t w01 = __vsub2(J01, __vminu2(N01, __vsub2(__vmaxu2(C2, A01), A01)));
          const uint32_t w23 = __vsub2(J23, __vminu2(N23, __vsub2(__vmaxu2(C2, A23), A23)));
          *reinterpret_cast<uint2*>(bout + tmp.it.off[k - tb] + joff) = make_uint2(w01, w23);
        }
      } else {
        for (uint32_t k = kb + lane4; k < kmid; k += 4) {
          const uint32_t C2 = tmp.it.C[k - tb];
          const uint32_t w01 = __vsub2(J01, __vminu2(N01, __vsub2(__vmaxu2(C2, A01), A01)));
          const uint32_t w23 = __vsub2(J23, __vminu2(N23, __vsub2(__vmaxu2(C2, A23), A23)));
          store4(bout + tmp.it.off[k - tb] + joff, false, w01, w23, e0 + j0, E);
        }
      }
      for (uint32_t k = max(kmid, kb) + ((lane4 + 4 - (max(kmid, kb) - kb) % 4) % 4); k < ke; k += 4) {
        const uint32_t C = tmp.it.C[k - tb];  // capacities above 65535: 32-bit arithmetic
        uint32_t b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) b[u] = Jv[u] - min(nfb[u], sat_sub(C, anf[u]));
        store4(bout + tmp.it.off[k - tb] + joff, full && aligned, b[0] | (b[1] << 16), b[2] | (b[3] << 16),
               e0 + j0, E);
      }
    }
  }
}

// ----------------------------------------------------------------------------- s2_warm
// Blocks before nsat: exact NF_all(e) per D (sum of the universe deltas of every earlier event)
// and the free-block term.  Few blocks, so this kernel favours simplicity; dynamic shared memory.
template <int ND, bool HT>
__global__ void __launch_bounds__(S_THREADS) s2_warm_kernel(const uint64_t* __restrict__ sim,
                                                            const uint64_t* __restrict__ scanrec, uint32_t E,
                                                            const ChunkDev* __restrict__ chunk,
                                                            const StackInstDev* __restrict__ insts,
                                                            const ChunkTotals* __restrict__ totals,
                                                            const uint32_t* __restrict__ blockpre, uint32_t wch,
                                                            uint32_t maxL, uint16_t* __restrict__ bout,
                                                            unsigned long long* sumXf) {
  typedef cub::BlockScan<uint32_t, S_THREADS> BSu;
  extern __shared__ uint32_t dyn[];
  uint32_t(*anf_s)[S_THREADS] = reinterpret_cast<uint32_t(*)[S_THREADS]>(dyn);
  uint32_t(*af_s)[S_THREADS] = reinterpret_cast<uint32_t(*)[S_THREADS]>(dyn + ND * S_THREADS);
  uint32_t(*nfall_s)[S_THREADS] = reinterpret_cast<uint32_t(*)[S_THREADS]>(dyn + 2 * ND * S_THREADS);
  __shared__ ChunkDev ch;
  __shared__ typename BSu::TempStorage scan;
  __shared__ uint32_t p_s[S_THREADS], cbeg_s[S_THREADS + 1], J_s[S_THREADS], Lb_s[S_THREADS];
  __shared__ uint32_t nsat_s[SND];
  __shared__ InstTileW itile;
  const uint32_t t = threadIdx.x;
  if (t == 0) ch = *chunk;
  if (t < SND) nsat_s[t] = totals->nsat[t];
  const uint32_t nwarm = totals->nsat_max;  // blocks from nsat_max on are saturated for every D: s2_sat
  __syncthreads();
  for (uint32_t blk = blockIdx.x; blk < nwarm; blk += gridDim.x) {  // small persistent grid
    for (int d = 0; d < ND; ++d) anf_s[d][t] = af_s[d][t] = 0;
    const uint32_t e0 = blk * S_THREADS;
    uint32_t Lb;
    uint64_t s;
    const uint32_t ntot = block_setup(sim, E, e0, wch, p_s, J_s, Lb_s, cbeg_s, Lb, s, scan);
    __syncthreads();
    // NF_all(D[d]) at e: the block prefix from s1_totals plus the block's own exclusive scan
    const uint32_t La_t = sim_La(s);
#pragma unroll 1
    for (int d = 0; d < ND; ++d) {
      if (blk >= nsat_s[d] || d >= static_cast<int>(ch.nd)) continue;  // uniform across the block
      const uint32_t delta = (e0 + t < E) ? nft(La_t, ch.D[d], ch.T[d]) - nft(Lb, ch.D[d], ch.T[d]) : 0u;
      uint32_t ex;
      BSu(scan).ExclusiveSum(delta, ex);
      nfall_s[d][t] = blockpre[uint64_t(blk) * SND + d] + ex;  // < Cmax[d] + 256 * 65535
      __syncthreads();
    }
    uint32_t Deff[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) Deff[d] = min(ch.D[d], maxL);
    window_phase<ND, true, HT>(scanrec, e0, wch, p_s, cbeg_s, ntot, Deff, ch.T, anf_s, af_s);
    __syncthreads();
    // phase C for the D values still in warm-up: 4 events per thread, instance stride 4, the
    // instance table staged in shared memory (as in s2_sat), general formula with free blocks
    const uint32_t quad = t & 63, lane4 = t >> 6, j0 = quad * 4;
    const bool full = e0 + j0 + 3 < E;
    for (uint32_t tb = 0; tb < ch.ninst; tb += IT) {
      const uint32_t te = min(ch.ninst, tb + IT);
      __syncthreads();
      for (uint32_t k = tb + t; k < te; k += S_THREADS) {
        const StackInstDev in = insts[ch.inst0 + k];
        itile.C[k - tb] = in.C;
        itile.off[k - tb] = in.boff;
        itile.inst[k - tb] = in.inst;
      }
      __syncthreads();
#pragma unroll 1
      for (int d = 0; d < ND; ++d) {
        const uint32_t kb = max(ch.dbeg[d], tb), ke = min(ch.dbeg[d + 1], te);
        if (kb >= ke || blk >= nsat_s[d]) continue;  // saturated: s2_sat writes these instances
        uint32_t nfb[4], fb[4], anf[4], af[4], nfa[4], Jv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool hit = p_s[j0 + u] != TLRU_NONE;
          nfb[u] = hit ? nft(Lb_s[j0 + u], ch.D[d], ch.T[d]) : 0u;
          fb[u] = hit ? f_of(Lb_s[j0 + u], ch.D[d]) : 0u;
          anf[u] = anf_s[d][j0 + u];
          af[u] = af_s[d][j0 + u];
          nfa[u] = nfall_s[d][j0 + u];
          Jv[u] = J_s[j0 + u];
        }
        for (uint32_t k = kb + lane4; k < ke; k += 4) {
          const uint32_t C = itile.C[k - tb];
          uint32_t b[4];
          unsigned long long xfs = 0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint32_t X = min(nfb[u], sat_sub(C, anf[u]));
            if (nfa[u] < C && fb[u] > 0 && e0 + j0 + u < E) {  // free blocks can still be cached
              const uint32_t xf = min(fb[u], sat_sub(sat_sub(C, nfa[u]), af[u]));
              X += xf;
              xfs += xf;
            }
            b[u] = Jv[u] - X;
          }
          if (xfs) atomicAdd(&sumXf[itile.inst[k - tb]], xfs);
          store4(bout + itile.off[k - tb] + e0 + j0, full, b[0] | (b[1] << 16), b[2] | (b[3] << 16), e0 + j0, E);
        }
      }
    }
    __syncthreads();
  }
}

// ----------------------------------------------------------------------------- s2_win / s2_out (fused K3)
// s2_win: phases A and B of s2_sat for every block from nsat_min on, writing the window sums
// A_nf (clamped to AT's range; AT = u16 when every capacity of the chunk is <= 65535) and
// (L_before | J << 16) per event, so the per-instance work can run instance-group-major.
template <int ND, typename AT, bool HT>
__global__ void __launch_bounds__(S_THREADS, 4) s2_win_kernel(const uint64_t* __restrict__ sim,
                                                              const uint64_t* __restrict__ scanrec, uint32_t E,
                                                              const ChunkDev* __restrict__ chunk,
                                                              const ChunkTotals* __restrict__ totals, uint32_t wch,
                                                              uint32_t maxL, AT* __restrict__ A, uint32_t Astride,
                                                              uint32_t* __restrict__ LbJ) {
  typedef cub::BlockScan<uint32_t, S_THREADS> BSu;
  __shared__ ChunkDev ch;
  __shared__ typename BSu::TempStorage scan;
  __shared__ uint32_t anf_s[ND][S_THREADS];
  __shared__ uint32_t p_s[S_THREADS], cbeg_s[S_THREADS + 1], J_s[S_THREADS], Lb_s[S_THREADS];
  if (blockIdx.x < totals->nsat_min) return;  // every D warm here: s2_out reads s2_warm's b
  const uint32_t t = threadIdx.x;
  if (t == 0) ch = *chunk;
#pragma unroll
  for (int d = 0; d < ND; ++d) anf_s[d][t] = 0;
  const uint32_t e0 = blockIdx.x * S_THREADS;
  uint32_t Lb;
  uint64_t s;
  const uint32_t ntot = block_setup(sim, E, e0, wch, p_s, J_s, Lb_s, cbeg_s, Lb, s, scan);
  __syncthreads();
  uint32_t Deff[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) Deff[d] = min(ch.D[d], maxL);
  window_phase<ND, false, HT, WIN_G>(scanrec, e0, wch, p_s, cbeg_s, ntot, Deff, ch.T, anf_s, nullptr);
  __syncthreads();
  const uint32_t e = e0 + t;
  if (e >= E) return;
  const uint32_t amax = static_cast<uint32_t>(static_cast<AT>(~AT(0)));
#if TLRU_WIN_EVICT_LAST
  // s2_out re-reads these (once per instance group) right after: keep them in L2
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(LbJ + e), "r"(Lb_s[t] | (J_s[t] << 16)), "l"(pol)
               : "memory");
  for (uint32_t d = 0; d < ch.nd; ++d) {
    AT* p = A + uint64_t(d) * Astride + e;
    const uint32_t v = min(anf_s[d][t], amax);
    if constexpr (sizeof(AT) == 2)
      asm volatile("st.global.L2::cache_hint.b16 [%0], %1, %2;" ::"l"(p), "h"(static_cast<unsigned short>(v)), "l"(pol)
                   : "memory");
    else
      asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
  }
#else
  LbJ[e] = Lb_s[t] | (J_s[t] << 16);
  for (uint32_t d = 0; d < ch.nd; ++d) A[uint64_t(d) * Astride + e] = static_cast<AT>(min(anf_s[d][t], amax));
#endif
}

// An s2_out group of one chunk row d.  kind 0 (writer): instance rows [inst0 + k0, inst0 + k0 + n)
// (sorted by C), whose b rows it writes.  kind 1 (histograms): the row's distinct capacities
// ("cells" -- instances with equal (D, C) have equal b on every event) [k0, k0 + n) of the chunk's
// cell table, whose histograms of b it builds: once per cell instead of once per instance.
struct GroupDev {
  uint32_t d, k0, n, kind;
};

struct CellDev {  // instances [k0, k0 + m) of the StackInstDev table (batch-global) share (d, C)
  uint32_t C, k0, m, d;
};

// s2_out: one CTA = (instance group, event range).  Per 4 events per thread: b for every
// instance of the group (X = min(NF(Lb), (C - A_nf)^+) on saturated blocks; the
// warm-up blocks' b come back from s2_warm's output), one 8-byte store per instance, and the
// group's histograms of b in shared memory (K3 without re-reading b).  The group's instances
// share D and are sorted by C, so for one event b_i = J - clamp(C_i - A, 0, N) is J on a prefix
// of instances (C_i <= A), J - N on a suffix (C_i >= A + N) and individual only in between: the
// histograms are kept as a difference array along the instance axis (row i holds
// hist[i] - hist[i-1]), a few shared-memory atomics per event instead of one per instance.
// cnt[g][v] = #{i in group g : C_i <= v} for v < tcap (rows padded to 16 bytes), for the
// groups whose capacities are all < tcap.  One CTA per group.
__global__ void __launch_bounds__(256) s2_cnt_kernel(const ChunkDev* __restrict__ chunk,
                                                     const StackInstDev* __restrict__ insts,
                                                     const GroupDev* __restrict__ groups, uint32_t tcap,
                                                     uint8_t* __restrict__ cnt_g, const CellDev* __restrict__ cells) {
  __shared__ uint32_t C_s[GI_MAX];
  const GroupDev g = groups[blockIdx.x];
  const uint32_t t = threadIdx.x;
  if (t < GI_MAX)
    C_s[t] = t < g.n ? (g.kind ? cells[g.k0 + t].C : insts[chunk->inst0 + g.k0 + t].C) : 0xFFFFFFFFu;
  __syncthreads();
  if (C_s[g.n - 1] >= tcap) return;
  uint8_t* row = cnt_g + uint64_t(blockIdx.x) * ((tcap + 15u) & ~15u);
  for (uint32_t v = t; v < tcap; v += blockDim.x) {
    uint32_t k = 0;
#pragma unroll
    for (uint32_t step = GI_MAX / 2; step > 0; step >>= 1)
      if (C_s[k + step - 1] <= v) k += step;
    row[v] = static_cast<uint8_t>(k + (C_s[k] <= v));
  }
}

template <typename AT, bool HT>
__global__ void __launch_bounds__(256, 4) s2_out_kernel(const ChunkDev* __restrict__ chunk,
                                                     const StackInstDev* __restrict__ insts,
                                                     const GroupDev* __restrict__ groups,
                                                     const ChunkTotals* __restrict__ totals,
                                                     const AT* __restrict__ A, uint32_t Astride,
                                                     const uint32_t* __restrict__ LbJ, uint32_t E, uint32_t range_len,
                                                     uint32_t bins, uint32_t rows, uint32_t tcap, bool aligned16,
                                                     uint16_t* __restrict__ bout, uint32_t* __restrict__ hist,
                                                     const uint4* __restrict__ cnt_g, uint32_t n_w, uint32_t n_h,
                                                     uint32_t sub,
                                                     const CellDev* __restrict__ cells, uint32_t* __restrict__ gcell) {
  // [rows >= group size][hb2] difference rows, two 16-bit counters per word (bins 2v, 2v+1).  The
  // counters wrap into each other, but a word's final value is lo + 65536 * hi (mod 2^32) and
  // decodes exactly while |lo|, |hi| <= 32767, which range_len <= OUT_RANGE_MAX guarantees.
  extern __shared__ __align__(128) uint32_t hw[];
  const uint32_t hb2 = (bins + 1) >> 1;
  __shared__ uint32_t C2_s[GI_MAX], C_s[GI_MAX], inst_s[GI_MAX], run_s[GI_MAX];
  __shared__ uint64_t off_s[GI_MAX];
  // cnt[v] = #{i : C_i <= v} for v < tcap, after the histogram rows (used when C_{n-1} < tcap)
  uint8_t* cnt = reinterpret_cast<uint8_t*>(hw + ((rows * hb2 + 3u) & ~3u));  // 16-byte aligned
  // 1-D grid, per event range of range_len events: its histogram groups (the chunk's groups
  // [n_w, ng)), then its writer groups [0, n_w) over `sub` sub-ranges of range_len / sub events,
  // groups fastest -- CTAs resident at one time share event ranges (the per-event inputs LbJ / A_nf
  // are read once from DRAM and then hit in L2), and writers run short ranges (their bulk-store
  // pattern is faster with fewer tiles per CTA) while the histogram groups keep long ones (their
  // per-CTA flush of the difference rows).
  const uint32_t per = n_h + n_w * sub;
  const uint32_t kr = blockIdx.x / per, rr = blockIdx.x % per;
  uint32_t gi, e_begin, e_end;
  if (rr < n_h) {
    gi = n_w + rr;
    e_begin = kr * range_len;
    e_end = min(E, e_begin + range_len);
  } else {
    const uint32_t wsub = range_len / sub, w = rr - n_h;
    gi = w % n_w;
    e_begin = kr * range_len + (w / n_w) * wsub;
    e_end = min(E, e_begin + wsub);
  }
  if (e_begin >= E) return;
  const GroupDev g = groups[gi];
  const uint32_t t = threadIdx.x, n = g.n;
  const bool hist_group = g.kind != 0;  // else a writer group: b rows only
  const uint32_t D = chunk->D[g.d], nsat = totals->nsat[g.d], inst0 = chunk->inst0;
  if (t < GI_MAX) {
    if (t < n) {
      if (hist_group) {  // a cell: its capacity, its first instance's row (warm-up b), its gcell row
        const CellDev cl = cells[g.k0 + t];
        C_s[t] = cl.C;
        C2_s[t] = cl.C * 0x10001u;
        inst_s[t] = g.k0 + t;
        off_s[t] = insts[cl.k0].boff;
      } else {
        const StackInstDev in = insts[inst0 + g.k0 + t];
        C_s[t] = in.C;
        C2_s[t] = in.C * 0x10001u;  // used only when C <= 65535
        inst_s[t] = in.inst;
        off_s[t] = in.boff;
      }
    } else {
      C_s[t] = 0xFFFFFFFFu;  // sentinel: the branch-free searches below never count it
    }
  }
  if (hist_group)
    for (uint32_t k = t; k < n * hb2; k += blockDim.x) hw[k] = 0;  // row n (never read) is not kept
  __syncthreads();
  const bool packed_all = C_s[n - 1] <= 65535u;  // capacities are sorted
  const bool use_cnt = C_s[n - 1] < tcap;
  auto count_le = [&](uint32_t v) {  // #{C_i <= v}: branch-free search over the sentinel-padded C_s
    uint32_t k = 0;
#pragma unroll
    for (uint32_t step = GI_MAX / 2; step > 0; step >>= 1)
      if (C_s[k + step - 1] <= v) k += step;
    return k + (C_s[k] <= v);  // the steps sum to GI_MAX - 1: one last compare reaches GI_MAX
  };
  if (t < n) {  // run_s[i]: end of the run of instances with capacity C_i (equal b on every event)
    uint32_t j = t + 1;
    while (j < n && C_s[j] == C_s[t]) ++j;
    run_s[t] = j;
  }
  if (hist_group && use_cnt) {  // the group's table, built once by s2_cnt_kernel
    const uint4* src = cnt_g + uint64_t(gi) * ((tcap + 15u) >> 4);
    for (uint32_t k = t; k < (tcap + 15u) >> 4; k += blockDim.x) reinterpret_cast<uint4*>(cnt)[k] = src[k];
  }
  __syncthreads();
  auto hadd = [&](uint32_t i, uint32_t v, int delta) {  // row i, bin v += delta
    atomicAdd(&hw[i * hb2 + (v >> 1)], static_cast<uint32_t>(delta) << ((v & 1u) << 4));
  };
  auto hsub = [&](uint32_t j, uint32_t v) {  // -1 at row j: row n is never read
    if (j < n) hadd(j, v, -1);
  };
  const AT* Ad = A + uint64_t(g.d) * Astride;
  constexpr uint32_t EV = 8;  // events per thread per tile: one 16-byte store per instance
  const uint32_t stride = EV * blockDim.x;
  const uint32_t D2 = min(D, 65535u) * 0x10001u;  // NF(L) = max(L, D) - D per 16-bit half (L <= 65535)
  const uint32_t T2 = HT ? chunk->T[g.d] * 0x10001u : 0u;  // Threshold-LRU rows: NF(L) = L [L >= T]
  auto pk = [](uint32_t x, uint32_t y) { return min(x, 65535u) | (min(y, 65535u) << 16); };
  // software pipeline: the next tile's (L_before | J) words and packed A_nf pairs (clamped to
  // 65535, exact for C <= 65535) are loaded one iteration ahead
  uint4 l0n = make_uint4(0, 0, 0, 0), l1n = l0n, an = l0n;
  auto load = [&](uint32_t e, uint4& l0, uint4& l1, uint4& ap) {
    if (e + EV <= e_end) {
      l0 = *reinterpret_cast<const uint4*>(LbJ + e);
      l1 = *reinterpret_cast<const uint4*>(LbJ + e + 4);
      if constexpr (sizeof(AT) == 2) {
        ap = *reinterpret_cast<const uint4*>(Ad + e);
      } else {
        const uint4 x = *reinterpret_cast<const uint4*>(Ad + e), y = *reinterpret_cast<const uint4*>(Ad + e + 4);
        ap = make_uint4(pk(x.x, x.y), pk(x.z, x.w), pk(y.x, y.y), pk(y.z, y.w));
      }
    } else if (e < e_end) {
      uint32_t l[EV], a[EV];
#pragma unroll
      for (uint32_t u = 0; u < EV; ++u) {
        l[u] = e + u < e_end ? LbJ[e + u] : 0u;
        a[u] = e + u < e_end ? static_cast<uint32_t>(Ad[e + u]) : 0u;
      }
      l0 = make_uint4(l[0], l[1], l[2], l[3]);
      l1 = make_uint4(l[4], l[5], l[6], l[7]);
      ap = make_uint4(pk(a[0], a[1]), pk(a[2], a[3]), pk(a[4], a[5]), pk(a[6], a[7]));
    }
  };
  load(e_begin + EV * t, l0n, l1n, an);
  if (!hist_group && packed_all && aligned16) {
    // ---- writer group, TMA path: per tile of stride = 2048 events, b of each run (distinct C)
    // is computed once into a shared-memory stage (one 16-byte vector per thread) and written to
    // every row of the run by cp.async.bulk (4 KB contiguous per row); runs go WB at a time
    // through a WS-slot ring (wait_group.read before a slot is reused).  No histogram work here,
    // so the barriers do not wait on uneven per-thread work.
    constexpr uint32_t WB = 6, WS = 2;  // runs per batch, stage slots: 2 x 6 x 4 KB = 48 KB
    uint4* stg = reinterpret_cast<uint4*>(hw);
    __shared__ uint32_t rstart_s[GI_MAX], ri_s[GI_MAX], nr_s;
    if (t == 0) {  // runs of equal C: their first instance; each instance's run index
      uint32_t nr = 0;
      for (uint32_t i = 0; i < n;) {
        rstart_s[nr] = i;
        for (uint32_t k = i; k < run_s[i]; ++k) ri_s[k] = nr;
        ++nr;
        i = run_s[i];
      }
      nr_s = nr;
    }
    __syncthreads();
    const uint32_t nr = nr_s;
    const uint32_t e_lo = max(e_begin, nsat * S_THREADS);  // warm-up blocks: s2_warm wrote b
    uint32_t it = 0;
    for (uint32_t base = e_begin; base < e_end; base += stride) {
      const uint32_t e = base + EV * t;
      const uint4 l0 = l0n, l1 = l1n, ap = an;
      if (base + stride < e_end) load(e + stride, l0n, l1n, an);
      const uint32_t tlo = max(base, e_lo), thi = min(base + stride, e_end);
      if (tlo >= thi) continue;  // uniform: the whole tile is warm
      const uint32_t lw[EV] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
      const uint32_t A2[4] = {ap.x, ap.y, ap.z, ap.w};
      uint32_t J2[4], N2[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        J2[k] = __byte_perm(lw[2 * k], lw[2 * k + 1], 0x7632);
        const uint32_t L2 = __byte_perm(lw[2 * k], lw[2 * k + 1], 0x5410);
        N2[k] = __vsub2(__vmaxu2(L2, D2), D2);
        if (HT) N2[k] &= __vcmpgeu2(L2, T2);
      }
      const uint32_t v0 = (tlo - base) / EV, nv16 = (thi - tlo) / EV;  // full 8-event vectors
      for (uint32_t rb = 0; rb < nr; rb += WB, ++it) {
        const uint32_t sl = it % WS;
        if (it >= WS && t < GI_MAX) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(WS - 1) : "memory");
        __syncthreads();  // slot sl is free again
        for (uint32_t q = 0; q < WB && rb + q < nr; ++q) {
          const uint32_t C2 = C2_s[rstart_s[rb + q]];
          uint32_t w[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) w[k] = __vsub2(J2[k], __vminu2(N2[k], __vsub2(__vmaxu2(C2, A2[k]), A2[k])));
          stg[(sl * WB + q) * 256 + t] = make_uint4(w[0], w[1], w[2], w[3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (t < n && ri_s[t] >= rb && ri_s[t] < rb + WB) {
          const uint4* src = stg + (sl * WB + (ri_s[t] - rb)) * 256;
          uint16_t* dst = bout + off_s[t] + tlo;
          if (nv16) {
            const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(src + v0));
#if TLRU_B_EVICT_FIRST
            uint64_t pol;  // b is written once and never re-read here: evict it from L2 first
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                         "r"(sa), "r"(nv16 * 16u), "l"(pol)
                         : "memory");
#else
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(sa),
                         "r"(nv16 * 16u)
                         : "memory");
#endif
          }
          const uint16_t* s16 = reinterpret_cast<const uint16_t*>(src);
          for (uint32_t u = tlo + nv16 * EV; u < thi; ++u) bout[off_s[t] + u] = s16[u - base];  // trace end
        }
        if (t < GI_MAX) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (t < GI_MAX) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    return;
  }
  for (uint32_t base = e_begin; base < e_end; base += stride) {
    const uint32_t e = base + EV * t;
    const uint4 l0 = l0n, l1 = l1n, ap = an;
    if (base + stride < e_end) load(e + stride, l0n, l1n, an);
    if (e >= e_end) continue;
    const uint32_t nv = min(EV, e_end - e);
    const bool warm = (e / S_THREADS) < nsat;  // the 8 events share a 256-event block
    if (warm && !hist_group) continue;  // b written by s2_warm
    if (warm) {  // b written by s2_warm: histogram only, one range update per run of equal C
      for (uint32_t i = 0; i < n;) {
        const uint16_t* row = bout + off_s[i] + e;
        const uint32_t j = run_s[i];
        for (uint32_t u = 0; u < nv; ++u) {
          hadd(i, row[u], 1);
          hsub(j, row[u]);
        }
        i = j;
      }
      continue;
    }
    // packed pairs of events (2k, 2k + 1): J, N = NF(L_before) (first turns: L_before = 0), A_nf
    const uint32_t lw[EV] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
    const uint32_t A2[4] = {ap.x, ap.y, ap.z, ap.w};
    uint32_t J2[4], N2[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      J2[k] = __byte_perm(lw[2 * k], lw[2 * k + 1], 0x7632);
      const uint32_t L2 = __byte_perm(lw[2 * k], lw[2 * k + 1], 0x5410);
      N2[k] = __vsub2(__vmaxu2(L2, D2), D2);
      if (HT) N2[k] &= __vcmpgeu2(L2, T2);
    }
    auto half = [](const uint32_t* v2, int u) { return (v2[u >> 1] >> ((u & 1) * 16)) & 0xFFFFu; };
    auto a_of = [&](int u) -> uint32_t {  // exact A_nf of event e + u
      if constexpr (sizeof(AT) == 2) return half(A2, u);
      else return static_cast<uint32_t>(Ad[e + u]);
    };
    if (hist_group) {
    // ---- histograms: per event, prefix (b = J), middle (individual), suffix (b = J - N).
    // k1 = #{C_i <= a}, k2 = #{C_i < a + N} = #{C_i <= a + N - 1}: table lookups (all 8 events
    // before the first atomic), else branch-free searches
    uint32_t kk[EV];  // k1 | k2 << 8
#pragma unroll
    for (int u = 0; u < static_cast<int>(EV); ++u) {
      const uint32_t a = u < static_cast<int>(nv) ? a_of(u) : 0u, top = a + half(N2, u);
      if (use_cnt)
        kk[u] = cnt[min(a, tcap - 1)] | (top ? uint32_t(cnt[min(top - 1, tcap - 1)]) << 8 : 0u);
      else
        kk[u] = count_le(a) | (top ? count_le(top - 1) << 8 : 0u);
    }
#pragma unroll
    for (int u = 0; u < static_cast<int>(EV); ++u) {
      if (u >= static_cast<int>(nv)) break;
      const uint32_t a = a_of(u), b0 = half(J2, u), b1 = b0 - half(N2, u);
      const uint32_t lo = kk[u] & 0xFFu, hi = max(kk[u] >> 8, lo);
      if (lo > 0) {
        hadd(0, b0, 1);
        hsub(lo, b0);
      }
      for (uint32_t i = lo; i < hi;) {  // runs of equal C lie entirely inside [lo, hi)
        const uint32_t j = run_s[i], v = b0 - (C_s[i] - a);
        hadd(i, v, 1);
        hsub(j, v);
        i = j;
      }
      if (hi < n) hadd(hi, b1, 1);
    }
    continue;
    }
    // ---- b for every instance of the group: b = J - min(N, (C - A)^+), once per run of equal C
    if (packed_all && aligned16 && nv == EV) {
      for (uint32_t i = 0; i < n;) {
        const uint32_t C2 = C2_s[i], j = run_s[i];
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = __vsub2(J2[k], __vminu2(N2[k], __vsub2(__vmaxu2(C2, A2[k]), A2[k])));
        const uint4 wv = make_uint4(w[0], w[1], w[2], w[3]);
        for (; i < j; ++i) *reinterpret_cast<uint4*>(bout + off_s[i] + e) = wv;
      }
    } else {
      for (uint32_t i = 0; i < n; ++i) {
        uint32_t b[EV];
#pragma unroll
        for (int u = 0; u < static_cast<int>(EV); ++u)
          b[u] = u < static_cast<int>(nv) ? half(J2, u) - min(half(N2, u), sat_sub(C_s[i], a_of(u))) : 0u;
        uint16_t* row = bout + off_s[i] + e;
        store4(row, e + 4 <= e_end, b[0] | (b[1] << 16), b[2] | (b[3] << 16), e, e_end);
        if (e + 4 < e_end) store4(row + 4, nv == EV, b[4] | (b[5] << 16), b[6] | (b[7] << 16), e + 4, e_end);
      }
    }
  }
  if (!hist_group) return;
  __syncthreads();
  for (uint32_t v2 = t; v2 < hb2; v2 += blockDim.x) {  // prefix over the cell axis -> cell histograms
    int run0 = 0, run1 = 0;
    const uint32_t v = 2 * v2;
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t w = hw[i * hb2 + v2];
      const int lo = static_cast<int16_t>(w & 0xFFFFu);
      run0 += lo;
      run1 += static_cast<int>(w - static_cast<uint32_t>(lo)) >> 16;
      uint32_t* h = gcell + uint64_t(inst_s[i]) * bins + v;
      if (run0) atomicAdd(h, static_cast<uint32_t>(run0));
      if (run1) atomicAdd(h + 1, static_cast<uint32_t>(run1));  // run1 != 0 implies v + 1 < bins
    }
  }
}

// Per (instance of the chunk, bin): the instance's histogram row = its cell's (s2_out's histogram
// groups build one per distinct (D, C)).
__global__ void s2_instcopy_kernel(const StackInstDev* __restrict__ insts, const uint32_t* __restrict__ inst_cell,
                                   uint32_t ninst, uint32_t bins, const uint32_t* __restrict__ gcell,
                                   uint32_t* __restrict__ hist) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x, k = blockIdx.y;
  if (v >= bins || k >= ninst) return;
  hist[uint64_t(insts[k].inst) * bins + v] = gcell[uint64_t(inst_cell[k]) * bins + v];
}

// ----------------------------------------------------------------------------- s3
__global__ void s3_results_kernel(const StackInstDev* __restrict__ insts, uint32_t ninst,
                                  const uint32_t* __restrict__ inst_chunk, const ChunkDev* __restrict__ chunks,
                                  const ChunkTotals* __restrict__ totals, const unsigned long long* sumXf,
                                  tlru_result* results) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < ninst; k += gridDim.x * blockDim.x) {
    const StackInstDev in = insts[k];
    const ChunkTotals& T = totals[inst_chunk[k]];
    const unsigned long long nfE = T.nfE[in.d], fE = T.fE[in.d], C = in.C;
    const unsigned long long U = nfE + fE;
    const unsigned long long used_final = U < C ? U : C;
    const unsigned long long room = C > nfE ? C - nfE : 0ull;
    const unsigned long long fc_final = fE < room ? fE : room;
    tlru_result& r = results[in.inst];
    // telescoped evictions: blocks inserted (a + b per cached request) - blocks still cached.
    // Threshold-LRU rows insert only on admitted requests; the others have b = J.
    const bool thr = chunks[inst_chunk[k]].T[in.d] > 0;
    const unsigned long long total = thr ? T.suma_adm[in.d] + (r.sum_uncached - T.sumJ_na[in.d]) - used_final
                                         : T.suma + r.sum_uncached - used_final;
    const unsigned long long trim = T.sumF[in.d] - sumXf[in.inst] - fc_final;
    r.evicted_trim = trim;
    r.evicted_lru = total - trim;
    r.max_occupancy = static_cast<uint32_t>(used_final);
  }
}

// ----------------------------------------------------------------------------- host
static const int kNDs[] = {2, 4, 8, 12, 16, 20, 24};

struct StackPlan {
  struct Chunk {
    uint32_t trace;
    uint32_t ndk;  // template width
    ChunkDev dev;
  };
  std::vector<Chunk> chunks;
  std::vector<StackInstDev> insts;
  std::vector<uint32_t> inst_chunk;
  std::vector<GroupDev> groups;        // s2_out groups (writers, then histogram groups), chunk-major
  std::vector<uint32_t> group0;        // first group of each chunk (+ end)
  std::vector<CellDev> cells;          // distinct (row, C) of each chunk, chunk-major, (row, C) order
  std::vector<uint32_t> cell0;         // first cell of each chunk (+ end)
  std::vector<uint32_t> inst_cell;     // per StackInstDev: its chunk-local cell
  uint32_t max_cells = 1;              // cells of the largest chunk (gcell rows)
  uint64_t Emax = 0;
  uint32_t maxbins = 1;
  uint32_t gi = 0;                     // instances per s2_out group (0 = unfused path)
  uint32_t tcap = 1;                   // s2_out count table entries (capacities < tcap)
  bool any_big = false;                // some capacity > 65535 -> u32 window sums
};

static void make_stack_plan(const tlru_trace* traces, uint32_t nt, const tlru_instance* inst, uint32_t ni,
                            const uint64_t* boffs, StackPlan* P) {
  for (uint32_t t = 0; t < nt; ++t) {
    P->Emax = std::max<uint64_t>(P->Emax, traces[t].num_events);
    P->maxbins = std::max<uint32_t>(P->maxbins, traces[t].max_history + 1);
  }
  std::vector<std::vector<uint32_t>> by_trace(nt);
  for (uint32_t i = 0; i < ni; ++i) by_trace[inst[i].trace].push_back(i);
  // row key (T << 32 | D): T-LRU rows D = max(xi - Q_hat, 0), T = 0; LRU rows D = T = 0;
  // Threshold-LRU rows D = 0, T = the admission threshold (T = 0 is plain LRU)
  auto Dof = [&](uint32_t i) -> uint64_t {
    if (inst[i].policy == TLRU_POLICY_THRESHOLD) return uint64_t(inst[i].threshold) << 32;
    return (inst[i].policy == TLRU_POLICY_TLRU && inst[i].xi > inst[i].q_hat) ? inst[i].xi - inst[i].q_hat : 0u;
  };
  for (uint32_t t = 0; t < nt; ++t) {
    const std::vector<uint32_t>& ids = by_trace[t];
    if (ids.empty() || traces[t].num_events == 0) continue;
    std::vector<uint64_t> Ds;
    for (uint32_t i : ids) Ds.push_back(Dof(i));
    std::sort(Ds.begin(), Ds.end());
    Ds.erase(std::unique(Ds.begin(), Ds.end()), Ds.end());
    // Threshold-LRU rows (keys with T > 0, sorted last) get chunks of their own, so the D rows
    // keep the unmasked window sums
    const size_t nD = std::lower_bound(Ds.begin(), Ds.end(), uint64_t(1) << 32) - Ds.begin();
    for (size_t c0 = 0; c0 < Ds.size();) {
      const size_t cend = std::min(c0 + SND, c0 < nD ? nD : Ds.size());
      StackPlan::Chunk ch;
      ch.trace = t;
      memset(&ch.dev, 0, sizeof(ch.dev));
      ch.dev.nd = static_cast<uint32_t>(cend - c0);
      ch.ndk = SND;
      for (int k : kNDs)
        if (static_cast<uint32_t>(k) >= ch.dev.nd) {
          ch.ndk = k;
          break;
        }
      for (uint32_t d = 0; d < SND; ++d) {
        const uint64_t key = d < ch.dev.nd ? Ds[c0 + d] : Ds[c0];
        ch.dev.D[d] = static_cast<uint32_t>(key);
        ch.dev.T[d] = static_cast<uint32_t>(key >> 32);
        ch.dev.anyT |= ch.dev.T[d] > 0 ? 1u : 0u;
      }
      ch.dev.inst0 = static_cast<uint32_t>(P->insts.size());
      for (uint32_t d = 0; d < ch.dev.nd; ++d) {
        ch.dev.dbeg[d] = static_cast<uint32_t>(P->insts.size()) - ch.dev.inst0;
        std::vector<uint32_t> mine;
        for (uint32_t i : ids)
          if (Dof(i) == Ds[c0 + d]) mine.push_back(i);
        std::stable_sort(mine.begin(), mine.end(), [&](uint32_t a, uint32_t b) {
          return std::min<uint32_t>(inst[a].capacity, 0x7FFF0000u) < std::min<uint32_t>(inst[b].capacity, 0x7FFF0000u);
        });
        ch.dev.dbig[d] = ch.dev.dbeg[d];
        for (uint32_t i : mine) {
          if (std::min<uint32_t>(inst[i].capacity, 0x7FFF0000u) <= 65535u) ++ch.dev.dbig[d];
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
      for (uint32_t d = 0; d < ch.dev.nd; ++d) P->any_big |= ch.dev.Cmax[d] > 65535u;
      P->chunks.push_back(ch);
      c0 = cend;
    }
  }
  // s2_out groups: the shared-memory histograms of a group hold (gi + 1) x ceil(bins / 2) words
  uint32_t cmax = 0;
  for (const StackInstDev& in : P->insts) cmax = std::max(cmax, in.C);
  P->tcap = std::min(cmax, TAB_MAX - 1u) + 1u;
  const uint32_t hb2 = (P->maxbins + 1) / 2;  // maxbins == the batch's histogram bins
  const uint32_t gfit = (OUT_SMEM - 16u - ((P->tcap + 15u) & ~15u)) / (4u * hb2);
  P->gi = gfit >= 8u ? std::min(GI_CAP, gfit) : 0u;
  P->inst_cell.assign(P->insts.size(), 0u);
  const uint32_t wcap = P->gi;  // measured: 12 / 16 / 24 / 32 rows per writer -> 0.91 / 0.88 / 0.89 / 0.95 ms
  for (const StackPlan::Chunk& ch : P->chunks) {
    P->group0.push_back(static_cast<uint32_t>(P->groups.size()));
    const uint32_t cbase = static_cast<uint32_t>(P->cells.size());
    P->cell0.push_back(cbase);
    for (uint32_t d = 0; d < ch.dev.nd; ++d) {  // cells: runs of equal C within the row
      for (uint32_t k = ch.dev.dbeg[d]; k < ch.dev.dbeg[d + 1];) {
        const uint32_t C = P->insts[ch.dev.inst0 + k].C;
        uint32_t k2 = k + 1;
        while (k2 < ch.dev.dbeg[d + 1] && P->insts[ch.dev.inst0 + k2].C == C) ++k2;
        for (uint32_t x = k; x < k2; ++x) P->inst_cell[ch.dev.inst0 + x] = static_cast<uint32_t>(P->cells.size()) - cbase;
        P->cells.push_back(CellDev{C, ch.dev.inst0 + k, k2 - k, d});
        k = k2;
      }
    }
    P->max_cells = std::max<uint32_t>(P->max_cells, static_cast<uint32_t>(P->cells.size()) - cbase);
    if (!P->gi) continue;
    for (uint32_t d = 0; d < ch.dev.nd; ++d) {  // writers: near-equal groups of <= wcap instances
      const uint32_t m = ch.dev.dbeg[d + 1] - ch.dev.dbeg[d], ngd = (m + wcap - 1) / wcap;
      for (uint32_t q = 0, k = ch.dev.dbeg[d]; q < ngd; ++q) {
        const uint32_t sz = m / ngd + (q < m % ngd ? 1u : 0u);
        P->groups.push_back(GroupDev{d, k, sz, 0u});
        k += sz;
      }
    }
    for (uint32_t d = 0; d < ch.dev.nd; ++d) {  // histograms: near-equal groups of <= gi cells per row
      uint32_t c0 = 0, c1 = 0;
      for (uint32_t c = cbase; c < P->cells.size(); ++c)
        if (P->cells[c].d == d) {
          if (c1 == 0) c0 = c - cbase;
          c1 = c - cbase + 1;
        }
      const uint32_t m = c1 - c0, ngd = (m + P->gi - 1) / P->gi;
      for (uint32_t q = 0, k = c0; q < ngd; ++q) {
        const uint32_t sz = m / ngd + (q < m % ngd ? 1u : 0u);
        P->groups.push_back(GroupDev{d, k, sz, 1u});
        k += sz;
      }
    }
  }
  P->group0.push_back(static_cast<uint32_t>(P->groups.size()));
  P->cell0.push_back(static_cast<uint32_t>(P->cells.size()));
}

struct StackWs {
  ChunkDev* chunks;
  StackInstDev* insts;
  uint32_t* inst_chunk;
  ChunkTotals* totals;
  unsigned long long* sumXf;
  uint32_t* blockagg;  // [block][SND] growth of NF_all per D, then block prefixes; reused per chunk
  uint32_t* hist;      // [2][maxbins] L_after histograms, reused per chunk
  uint64_t* scanrec;   // [event] next | L_after << 32 of the trace being processed
  GroupDev* groups;    // s2_out groups of every chunk
  uint32_t* A;         // [SND][Astride] window sums A_nf (u16 or u32), reused per chunk
  uint32_t* LbJ;       // [event] L_before | J << 16
  uint8_t* cnt;        // [group][tcap rounded to 16] s2_out count tables
  uint32_t Astride;
  CellDev* cells;      // the plan's cells
  uint32_t* inst_cell; // per StackInstDev: chunk-local cell
  uint32_t* gcell;     // [cell][bins] the cells' histograms, reused per chunk
};

static void carve_stack(Carver& cv, const StackPlan& P, uint32_t ni, StackWs* w) {
  const size_t nc = P.chunks.size() + 1;
  w->chunks = cv.take<ChunkDev>(nc);
  w->insts = cv.take<StackInstDev>(P.insts.size() + 1);
  w->inst_chunk = cv.take<uint32_t>(P.insts.size() + 1);
  w->totals = cv.take<ChunkTotals>(nc);
  w->sumXf = cv.take<unsigned long long>(ni + 1);
  w->blockagg = cv.take<uint32_t>(((P.Emax + S_THREADS - 1) / S_THREADS + 1) * SND);
  w->hist = cv.take<uint32_t>(2 * uint64_t(P.maxbins));
  w->scanrec = cv.take<uint64_t>(P.Emax + 1);
  w->groups = cv.take<GroupDev>(P.groups.size() + 1);
  w->Astride = static_cast<uint32_t>((P.Emax + 7) & ~7ull);
  const size_t abytes = P.gi ? size_t(SND) * w->Astride * (P.any_big ? 4 : 2) : 4;
  w->A = cv.take<uint32_t>((abytes + 3) / 4);
  w->LbJ = cv.take<uint32_t>(P.gi ? P.Emax + 8 : 1);
  w->cnt = cv.take<uint8_t>(P.gi ? P.groups.size() * ((P.tcap + 15u) & ~size_t(15)) : 16);
  w->cells = cv.take<CellDev>(P.cells.size() + 1);
  w->inst_cell = cv.take<uint32_t>(P.inst_cell.size() + 1);
  w->gcell = cv.take<uint32_t>(P.gi ? uint64_t(P.max_cells) * P.maxbins : 1);
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

template <int ND, bool HT>
static tlru_status launch_s2(const tlru_trace& tr, const ChunkDev* ch, const ChunkTotals* tot, const StackWs& w,
                             const StackPlan& P, uint32_t c, uint32_t bins, bool aligned, bool aligned16, uint16_t* bout,
                             uint32_t* hist, cudaStream_t st, OutTiming* ot) {
  const uint32_t E = static_cast<uint32_t>(tr.num_events);
  const uint32_t nb = (E + S_THREADS - 1) / S_THREADS;
  // 16x2 partial sums of max(L, min(D, maxL)) stay exact while wch * maxL < 2^16
  const uint32_t maxL = std::max<uint32_t>(tr.max_history, 1u);
  const uint32_t wch = std::max<uint32_t>(1u, std::min<uint32_t>(WCH_MAX, 65535u / maxL));
  const size_t warm_smem = size_t(3) * ND * S_THREADS * sizeof(uint32_t);
  TLRU_CUDA(cudaFuncSetAttribute(s2_warm_kernel<ND, HT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(warm_smem)));
  s2_warm_kernel<ND, HT><<<std::min<uint32_t>(nb ? nb : 1, 2u * 148u), S_THREADS, warm_smem, st>>>(
      tr.sim, w.scanrec, E, ch, w.insts, tot, w.blockagg, wch, maxL, bout, w.sumXf);
  TLRU_CHECK_LAUNCH();
  if (!P.gi) {  // unfused: b written by s2_sat, histograms by the generic K3 afterwards
    s2_sat_kernel<ND, HT><<<nb, S_THREADS, 0, st>>>(tr.sim, w.scanrec, E, ch, w.insts, tot, wch, maxL, aligned, bout);
    TLRU_CHECK_LAUNCH();
    return TLRU_OK;
  }
  const uint32_t g0 = P.group0[c], ng = P.group0[c + 1] - g0;
  const uint32_t target = 148u * 8u;  // CTAs for s2_out
  const uint32_t nr = std::max<uint32_t>(1u, (target + ng - 1) / std::max<uint32_t>(ng, 1u));
  uint32_t rl = (E + nr - 1) / nr;
  rl = std::min(OUT_RANGE_MAX, (rl + 1023u) & ~1023u);
  // writer sub-ranges of OUT_WRANGE events inside the histogram groups' ranges
  uint32_t sub = 1;
  if (rl > OUT_WRANGE) {
    sub = std::min(OUT_RANGE_MAX / OUT_WRANGE, (rl + OUT_WRANGE - 1) / OUT_WRANGE);
    rl = sub * OUT_WRANGE;
  }
  const uint32_t nranges = (E + rl - 1) / rl;
  // histogram groups: rows + count table; writer groups (TMA path): 3 stage slots x 4 runs x 4 KB
  const size_t out_smem = std::max<size_t>(((size_t(P.gi) * ((bins + 1) / 2) + 3) & ~size_t(3)) * sizeof(uint32_t) +
                                               ((P.tcap + 15) & ~15u),
                                           size_t(48) * 1024);
  uint8_t* cnt_g = w.cnt + size_t(g0) * ((P.tcap + 15u) & ~15u);
  auto out = [&](auto* Aptr) -> tlru_status {
    using AT = std::remove_const_t<std::remove_pointer_t<decltype(Aptr)>>;
    s2_win_kernel<ND, AT, HT><<<nb, S_THREADS, 0, st>>>(tr.sim, w.scanrec, E, ch, tot, wch, maxL, Aptr, w.Astride, w.LbJ);
    TLRU_CHECK_LAUNCH();
    TLRU_CUDA(cudaFuncSetAttribute(s2_out_kernel<AT, HT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(out_smem)));
    const CellDev* cells = w.cells + P.cell0[c];
    const uint32_t ncell = P.cell0[c + 1] - P.cell0[c];
    if (ng) {
      s2_cnt_kernel<<<ng, 256, 0, st>>>(ch, w.insts, w.groups + g0, P.tcap, cnt_g, cells);
      TLRU_CHECK_LAUNCH();
      TLRU_CUDA(cudaMemsetAsync(w.gcell, 0, size_t(ncell) * bins * sizeof(uint32_t), st));
    }
    uint32_t n_w = 0;  // the chunk's writer groups come first (make_stack_plan)
    while (n_w < ng && P.groups[g0 + n_w].kind == 0) ++n_w;
    const uint32_t n_h = ng - n_w;
    if (ng) {
      if (ot && ot->first && ot->launches == 0) TLRU_CUDA(cudaEventRecord(ot->first, st));
      const uint64_t nblk = uint64_t(nranges) * (n_h + uint64_t(n_w) * sub);
      s2_out_kernel<AT, HT><<<static_cast<unsigned>(nblk), 256, out_smem, st>>>(
          ch, w.insts, w.groups + g0, tot, Aptr, w.Astride, w.LbJ, E, rl, bins, P.gi, P.tcap, aligned16, bout, hist,
          reinterpret_cast<const uint4*>(cnt_g), n_w, n_h, sub, cells, w.gcell);
      TLRU_CHECK_LAUNCH();
      if (ot && ot->last) {
        TLRU_CUDA(cudaEventRecord(ot->last, st));
        ++ot->launches;
      }
    }
    if (ng) {  // instance histograms = their cells'
      const uint32_t k0 = P.chunks[c].dev.inst0, nik = P.chunks[c].dev.ninst;
      s2_instcopy_kernel<<<dim3((bins + 127) / 128, nik), 128, 0, st>>>(w.insts + k0, w.inst_cell + k0, nik, bins,
                                                                         w.gcell, hist);
      TLRU_CHECK_LAUNCH();
    }
    return TLRU_OK;
  };
  if (P.any_big) return out(w.A);
  return out(reinterpret_cast<uint16_t*>(w.A));
}

tlru_status stack_simulate(const tlru_trace* traces, uint32_t nt, const tlru_instance* inst, uint32_t ni,
                           const uint64_t* boffs, uint16_t* bout, tlru_result* results, Carver& cv,
                           const SegDev* segs_dev, uint32_t bins, uint32_t* hist, unsigned long long* clamped,
                           size_t ws_bytes, cudaStream_t st, unsigned* nkernels, cudaEvent_t ev_mid,
                           OutTiming* out_timing) {
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
    if (!P.groups.empty())
      TLRU_CUDA(cudaMemcpyAsync(w.groups, P.groups.data(), P.groups.size() * sizeof(GroupDev),
                                cudaMemcpyHostToDevice, st));
    if (!P.cells.empty())
      TLRU_CUDA(cudaMemcpyAsync(w.cells, P.cells.data(), P.cells.size() * sizeof(CellDev), cudaMemcpyHostToDevice,
                                st));
    if (!P.inst_cell.empty())
      TLRU_CUDA(cudaMemcpyAsync(w.inst_cell, P.inst_cell.data(), P.inst_cell.size() * sizeof(uint32_t),
                                cudaMemcpyHostToDevice, st));
  }
  TLRU_CUDA(cudaMemsetAsync(w.totals, 0, (nc + 1) * sizeof(ChunkTotals), st));
  TLRU_CUDA(cudaMemsetAsync(w.sumXf, 0, (ni + 1) * sizeof(unsigned long long), st));
  // 8-byte b stores need every instance row to start at a multiple of 4 requests (16-byte base)
  bool aligned = (reinterpret_cast<uintptr_t>(bout) & 7u) == 0;
  for (const StackInstDev& in : P.insts) aligned &= (in.boff & 3u) == 0;
  bool aligned16 = (reinterpret_cast<uintptr_t>(bout) & 15u) == 0;  // s2_out: 16-byte stores of 8 requests
  for (const StackInstDev& in : P.insts) aligned16 &= (in.boff & 7u) == 0;
  for (size_t c = 0; c < nc; ++c) {
    const tlru_trace& tr = traces[P.chunks[c].trace];
    const uint32_t E = static_cast<uint32_t>(tr.num_events);
    const uint32_t nb = (E + S_THREADS - 1) / S_THREADS;
    const uint32_t hb = tr.max_history + 1;
    TLRU_CUDA(cudaMemsetAsync(w.hist, 0, 2 * size_t(hb) * sizeof(uint32_t), st));
    const size_t s1_smem = hb <= 8192 ? 2 * size_t(hb) * sizeof(uint32_t) : 0;
    s1_block_kernel<<<std::min<uint32_t>(nb ? nb : 1, 148u * 4u), S_THREADS, s1_smem, st>>>(
        tr.sim, tr.next, E, w.chunks + c, w.scanrec, w.blockagg, hb, w.hist, w.hist + hb, w.totals + c);
    TLRU_CHECK_LAUNCH();
    s1_totals_kernel<<<1, T_THREADS, 0, st>>>(w.chunks + c, hb, w.hist, w.hist + hb, w.blockagg, nb, w.totals + c);
    TLRU_CHECK_LAUNCH();
    if (P.chunks[c].dev.anyT) {  // Threshold-LRU chunks: masked window sums (three widths)
      if (P.chunks[c].ndk <= 2) TLRU_TRY((launch_s2<2, true>(tr, w.chunks + c, w.totals + c, w, P, c, bins, aligned, aligned16, bout, hist, st, out_timing)));
      else if (P.chunks[c].ndk <= 8) TLRU_TRY((launch_s2<8, true>(tr, w.chunks + c, w.totals + c, w, P, c, bins, aligned, aligned16, bout, hist, st, out_timing)));
      else TLRU_TRY((launch_s2<24, true>(tr, w.chunks + c, w.totals + c, w, P, c, bins, aligned, aligned16, bout, hist, st, out_timing)));
    } else switch (P.chunks[c].ndk) {
      case 2: TLRU_TRY((launch_s2<2, false>(tr, w.chunks + c, w.totals + c, w, P, c, bins, aligned, aligned16, bout, hist, st, out_timing))); break;
      case 4: TLRU_TRY((launch_s2<4, false>(tr, w.chunks + c, w.totals + c, w, P, c, bins, aligned, aligned16, bout, hist, st, out_timing))); break;
      case 8: TLRU_TRY((launch_s2<8, false>(tr, w.chunks + c, w.totals + c, w, P, c, bins, aligned, aligned16, bout, hist, st, out_timing))); break;
      case 12: TLRU_TRY((launch_s2<12, false>(tr, w.chunks + c, w.totals + c, w, P, c, bins, aligned, aligned16, bout, hist, st, out_timing))); break;
      case 16: TLRU_TRY((launch_s2<16, false>(tr, w.chunks + c, w.totals + c, w, P, c, bins, aligned, aligned16, bout, hist, st, out_timing))); break;
      case 20: TLRU_TRY((launch_s2<20, false>(tr, w.chunks + c, w.totals + c, w, P, c, bins, aligned, aligned16, bout, hist, st, out_timing))); break;
      default: TLRU_TRY((launch_s2<24, false>(tr, w.chunks + c, w.totals + c, w, P, c, bins, aligned, aligned16, bout, hist, st, out_timing))); break;
    }
    *nkernels += 4;
  }
  // K3 (fused into s2_out unless the histograms are too wide), then the eviction counters from
  // the telescoped identities
  if (!P.gi) TLRU_TRY(launch_hist(bout, segs_dev, ni, bins, hist, clamped, st));
  if (ev_mid) TLRU_CUDA(cudaEventRecord(ev_mid, st));
  TLRU_TRY(launch_finalize(segs_dev, ni, bins, hist, clamped, 1.0, nullptr, results, st));
  if (!P.insts.empty()) {
    s3_results_kernel<<<grid_for(P.insts.size(), 128), 128, 0, st>>>(w.insts, static_cast<uint32_t>(P.insts.size()),
                                                                     w.inst_chunk, w.chunks, w.totals, w.sumXf,
                                                                     results);
    TLRU_CHECK_LAUNCH();
  }
  *nkernels += 3;
  return TLRU_OK;
}

}  // namespace tlru
