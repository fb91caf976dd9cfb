// sim.cu -- K2: batched Alg. 1 simulation and tlru_simulate_batch.
//
// Work decomposition:
//   * instances of one trace are sorted by capacity and packed 32 to a warp
//     ("lane group"); every lane runs its own instance (C, D) in lockstep over
//     the SAME events, so each event record is loaded once per warp (coalesced
//     32-event tile, broadcast by shuffle) and each lane keeps its state in a
//     lane-interleaved, bank-conflict-free shared-memory array of W entries;
//   * each trace is cut into segments; a warp = (lane group, segment); every
//     segment start state is rebuilt exactly (sim.cuh), so all warps are
//     independent and the grid is sized to fill the 148 SMs;
//   * per-request b are staged in shared memory and written as coalesced
//     64-byte rows per instance;
//   * a chain whose live entries exceed W is re-run by the spill kernel with
//     its state in global memory (never truncated).
#include <algorithm>
#include <type_traits>
#include <mutex>
#include <vector>

#include "metrics.cuh"
#include "sim.cuh"
#include "stack.cuh"

#ifndef TLRU_XS_PAIRS
#define TLRU_XS_PAIRS 1  // lanes with a surplus array keep (X, S) as interleaved halfword pairs
#endif

namespace tlru {

struct LaneDev {
  uint32_t inst;  // instance index, 0xFFFFFFFF = idle lane
  uint32_t C, D;
  uint32_t T;     // Threshold-LRU admission threshold (0: LRU / T-LRU)
  uint64_t boff;  // offset of the instance's b array in `uncached`
  uint32_t policy, xi;  // End-/Length-Aware chains: the policy and xi (Length-Aware's D per turn)
  uint32_t aidx, pad;   // index among the End-/Length-Aware lanes (snapshot / counter slots)
};

// End-/Length-Aware time partitioning (their cache is not the top-C of the universe, so no
// closed-form warm start exists).  Segment k of a chain starts `burn` events early from an
// empty cache; its state at the segment start (G_k) and end (F_k) is saved.  Segment k is exact
// iff k = 0 or G_k == F_{k-1} (the state determines the rest of the run); aware_fix_kernel
// re-runs the others from the exact F_{k-1}, in order, so every output is exact.
struct AwareDev {
  uint32_t seg_len, burn, nseg_max, wsnap;
  uint32_t burn_long;        // forced-caching groups: fragments kept only by Phase 2 can be old
  uint32_t* snap;            // [aware lane][seg][2] snapshots of 4 + 2 * wsnap words
  unsigned long long* segc;  // [aware lane][seg][2] evicted_trim, evicted_lru of the segment
  uint32_t* segm;            // [aware lane][seg] max occupancy in the segment
  uint32_t* ovf;             // [aware lane][seg] 1 = the segment overflowed the on-chip state
};

__host__ __device__ __forceinline__ size_t snap_words(uint32_t wsnap) { return 4 + 2 * size_t(wsnap); }

// Canonical state: live entries in tau order (tau, X | S << 16), S zeroed up to the first entry
// with positive remaining surplus (fh) -- it is not used there; header {n, used, fh, frem}.
template <class St>
__device__ void snap_write(uint32_t* out, uint32_t wsnap, const ChainRegs& c, const St& st) {
  uint32_t n = 0, fhn = 0xFFFFFFFFu, frem = 0;
  uint32_t* tau = out + 4;
  uint32_t* xs = tau + wsnap;
  for (uint32_t k = c.head; k < c.tail; ++k) {
    const uint32_t x = st.Xr(k);
    if (x == 0) continue;
    uint32_t s = st.Sr(k);
    if (fhn == 0xFFFFFFFFu) {
      const uint32_t eff = k < c.fh ? 0u : (k == c.fh ? c.frem : min(x, s));
      if (eff > 0) {
        fhn = n;
        frem = eff;
      }
      s = 0;
    } else {
      s = min(x, s);  // the effective surplus: identical whether S is stored or the constant D
    }
    if (n < wsnap) {
      tau[n] = st.T(k);
      xs[n] = x | (s << 16);
    }
    ++n;
  }
  out[0] = n <= wsnap ? n : 0xFFFFFFFFu;  // too large to save: never matches, the fix-up re-runs it
  out[1] = c.used;
  out[2] = fhn == 0xFFFFFFFFu ? n : fhn;
  out[3] = frem;
}

// Tail-Optimized Belady chains: live entries in key order (key, X | S << 16); header
// {n, used, dead, 0} (tombstones are not state: X = 0 is the same as no entry).
template <class St>
__device__ void snap_write_belady(uint32_t* out, uint32_t wsnap, const ChainRegs& c, const St& st) {
  uint32_t n = 0;
  uint32_t* key = out + 4;
  uint32_t* xs = key + wsnap;
  for (uint32_t k = c.head; k < c.tail; ++k) {
    const uint32_t x = st.Xr(k);
    if (x == 0) continue;
    if (n < wsnap) {
      key[n] = st.T(k);
      xs[n] = x | (uint32_t(st.Sr(k)) << 16);
    }
    ++n;
  }
  out[0] = n <= wsnap ? n : 0xFFFFFFFFu;
  out[1] = c.used;
  out[2] = c.dead;
  out[3] = 0;
}

__device__ bool snap_equal(const uint32_t* a, const uint32_t* b, uint32_t wsnap) {
  if (a[0] == 0xFFFFFFFFu || a[0] != b[0] || a[1] != b[1] || a[2] != b[2] || a[3] != b[3]) return false;
  for (uint32_t i = 0; i < a[0]; ++i)
    if (a[4 + i] != b[4 + i] || a[4 + wsnap + i] != b[4 + wsnap + i]) return false;
  return true;
}

constexpr uint32_t kAwareTLRU = 1;    // Length-Aware T-LRU lanes (per-entry surplus)
constexpr uint32_t kAwareBelady = 2;  // Tail-Optimized Belady lanes
constexpr uint32_t kAwareForced = 4;  // forced-caching T-LRU lanes (surplus = constant D: no surplus
                                      // array; long burn-in)

struct GroupDev {
  uint32_t trace, lane0, nlanes, W;
  uint32_t aware;  // 0, kAwareTLRU or kAwareBelady: burn-in segments verified by the fix-up
};

struct ItemDev {
  uint32_t group, seg;
};

struct TraceDev {
  const uint64_t* sim;
  const uint32_t* next;
  uint64_t E;
  const uint64_t* ticks;  // event times (ET-LRU beliefs); may be NULL for the other policies
};

struct AccDev {  // per-instance accumulators of the counters not derivable from b
  unsigned long long ev_trim, ev_lru;
  unsigned int max_occ, pad;
};

struct SpillDev {
  uint32_t group, seg, lane, pad;
};
}  // namespace tlru

#include "etlru.cuh"

namespace tlru {

constexpr int BST_STRIDE = 34;  // u16 stride of a staged b row: 32 events + 2 pad (conflict-free)

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
  uint32_t lo = __shfl_sync(0xFFFFFFFFu, static_cast<uint32_t>(v), src);
  uint32_t hi = __shfl_sync(0xFFFFFFFFu, static_cast<uint32_t>(v >> 32), src);
  return (uint64_t(hi) << 32) | lo;
}

__device__ __forceinline__ void acc_commit(AccDev* acc, uint32_t inst, const ChainRegs& c) {
  if (c.ev_trim) atomicAdd(&acc[inst].ev_trim, static_cast<unsigned long long>(c.ev_trim));
  if (c.ev_lru) atomicAdd(&acc[inst].ev_lru, static_cast<unsigned long long>(c.ev_lru));
  atomicMax(&acc[inst].max_occ, c.max_occ);
}

// One warp per (lane group, segment).  W = state entries per lane (compile-time).
// AWARE: End-/Length-Aware groups: the segment is the whole trace (their cache is not the
// top-C of the universe, so no exact warm start exists) and the state keeps per-entry surplus.
template <class St>
__device__ __forceinline__ St make_state(uint32_t* tau_s, uint16_t* X_s, uint16_t* S_s, int lane, uint16_t D,
                                         uint32_t base) {
  if constexpr (std::is_same_v<St, SmemStatePk>) return SmemStatePk{tau_s, lane, D, base};
  else if constexpr (std::is_same_v<St, SmemStateXS>) return SmemStateXS{tau_s, X_s, lane};
  else return St{tau_s, X_s, S_s, lane, D};
}

template <int W, bool AWARE, bool NOS = false, bool PK = false>
__global__ void __launch_bounds__(32) sim_kernel(const ItemDev* __restrict__ items, const GroupDev* __restrict__ groups,
                                                 const LaneDev* __restrict__ lanes, const TraceDev* __restrict__ traces,
                                                 uint32_t seg_len, uint16_t* __restrict__ bout, AccDev* acc,
                                                 SpillDev* spill, unsigned int* nspill, AwareDev aw) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* tau_s = reinterpret_cast<uint32_t*>(smem);
  uint16_t* X_s = reinterpret_cast<uint16_t*>(tau_s + W * 32);
  uint16_t* S_s = X_s + W * 32;
  uint16_t* bst = PK ? reinterpret_cast<uint16_t*>(tau_s + W * 32) : (AWARE && !NOS) ? S_s + W * 32 : S_s;
  const int lane = threadIdx.x;
  const ItemDev it = items[blockIdx.x];
  const GroupDev g = groups[it.group];
  const TraceDev tr = traces[g.trace];
  const uint32_t sl = AWARE ? aw.seg_len : seg_len;
  const uint32_t s = it.seg * sl;
  const uint32_t s_end = static_cast<uint32_t>(min(uint64_t(s) + sl, tr.E));
  const uint32_t burn = g.aware == kAwareForced ? aw.burn_long : aw.burn;
  const uint32_t s0 = AWARE ? (s > burn ? s - burn : 0u) : s;  // aware: burn-in from an empty cache
  LaneDev lp;
  lp.inst = 0xFFFFFFFFu;
  lp.C = lp.D = lp.T = 0;
  lp.boff = 0;
  lp.policy = lp.xi = 0;
  if (lane < static_cast<int>(g.nlanes)) lp = lanes[g.lane0 + lane];
  bool active = lp.inst != 0xFFFFFFFFu;
  using St = std::conditional_t<PK, SmemStatePk,
                                std::conditional_t<(AWARE && !NOS && TLRU_XS_PAIRS), SmemStateXS, SmemStateT<NOS>>>;
  St st = make_state<St>(tau_s, X_s, S_s, lane, static_cast<uint16_t>(min(lp.D, 65535u)), s0);
  ChainRegs c;
  chain_init(c, lp.C, lp.D, lp.T, W, active && s > 0);
  const bool bel = AWARE && g.aware == kAwareBelady;  // warp-uniform
  if (bel) c.head = c.tail = W / 2;  // sorted by next arrival: inserts land anywhere

  // ---- rebuild the exact state at s (sim.cuh "Segment start"); AWARE chains start at event 0
  for (int pass = 0; pass < (AWARE ? 0 : 2); ++pass) {
    int64_t e0 = int64_t(s) - 1;
    while (e0 >= 0 && __any_sync(0xFFFFFFFFu, c.walking)) {
      const int64_t e = e0 - lane;
      uint32_t nx = 0, la = 0;
      if (e >= 0) {
        nx = __ldg(tr.next + e);
        la = sim_La(__ldg(tr.sim + e));
      }
      const int cnt = e0 + 1 < 32 ? static_cast<int>(e0 + 1) : 32;
      for (int k = 0; k < cnt; ++k) {
        const uint32_t nxk = __shfl_sync(0xFFFFFFFFu, nx, k);
        const uint32_t lak = __shfl_sync(0xFFFFFFFFu, la, k);
        if (c.walking && nxk >= s) chain_walk_step(c, st, static_cast<uint32_t>(e0 - k), lak);
      }
      e0 -= 32;
    }
    const bool again = chain_walk_restart(c);
    if (!__any_sync(0xFFFFFFFFu, again)) break;
  }
  chain_walk_finish(c);
  if (c.overflow) active = false;

  // ---- forward: Alg. 1 per request, events broadcast from a 32-event register tile
  uint64_t evn = 0;
  if (s0 + lane < s_end) evn = __ldg(tr.sim + s0 + lane);
  const size_t sw = AWARE ? snap_words(aw.wsnap) : 0;
  uint32_t* snapG = nullptr;
  if (AWARE && lp.inst != 0xFFFFFFFFu) snapG = aw.snap + (size_t(lp.aidx) * aw.nseg_max + it.seg) * 2 * sw;
  for (uint32_t base = s0; base < s_end; base += 32) {
    if (AWARE && base == s) {  // segment start: save G_k, restart the segment's counters
      if (active && it.seg > 0) {
        if (bel) snap_write_belady(snapG, aw.wsnap, c, st);
        else snap_write(snapG, aw.wsnap, c, st);
      }
      c.ev_trim = c.ev_lru = c.max_occ = 0;
    }
    const uint64_t evc = evn;
    const uint32_t nk = min(32u, s_end - base);
    if (base + 32 + lane < s_end) evn = __ldg(tr.sim + base + 32 + lane);  // prefetch the next tile
    uint32_t qnc = 0xFFFFFFFFu;  // AWARE: this lane's event's next prompt, or NONE on a terminating turn
    uint32_t nxc = TLRU_NONE;    // and its next turn's event index (Belady's key)
    if (AWARE && base + lane < s_end) {
      nxc = __ldg(tr.next + base + lane);
      if (nxc != TLRU_NONE) qnc = sim_J(__ldg(tr.sim + nxc)) - sim_La(evc);  // q = J - L_before
    }
    for (uint32_t k = 0; k < nk; ++k) {
      const uint64_t ev = shfl64(evc, k);
      // Synchronised compaction: when one lane's array is full (it must drop its tombstones before
      // this insert), every lane compacts now -- the warp runs the loop once for all of them instead
      // of once per lane at 32 different events.  Compaction only re-packs the live entries (the
      // state is unchanged), so the outputs are identical.  Belady lanes keep their own (centred) layout.
      if (!bel && __any_sync(0xFFFFFFFFu, active && c.tail == c.W) && active && c.head < c.tail)
        chain_compact<AWARE>(c, st);
      if (AWARE) {
        const uint32_t qn = __shfl_sync(0xFFFFFFFFu, qnc, k);
        if (bel) {
          const uint32_t nxk = __shfl_sync(0xFFFFFFFFu, nxc, k);
          if (active) {
            const uint32_t La = sim_La(ev);
            const uint32_t s0 = nxk == TLRU_NONE ? 0u : min(La, lp.xi > qn ? lp.xi - qn : 0u);
            const uint32_t b = chain_request_belady(c, st, base + k, sim_J(ev), La, nxk, s0,
                                                    lp.policy == TLRU_POLICY_BELADY_FORCED);
            bst[lane * BST_STRIDE + k] = static_cast<uint16_t>(b);
            if (c.overflow) active = false;
          }
        } else if (active) {
          const bool forced = lp.policy == TLRU_POLICY_TLRU_FORCED;  // no release, D = xi - Q_hat
          const bool last = !forced && qn == 0xFFFFFFFFu;
          const uint32_t Dcur = lp.policy == TLRU_POLICY_LENGTH_AWARE ? (lp.xi > qn ? lp.xi - qn : 0u) : lp.D;
          const uint32_t b =
              chain_request_aware(c, st, base + k, sim_prev(ev), sim_J(ev), sim_La(ev), last, Dcur, forced);
          bst[lane * BST_STRIDE + k] = static_cast<uint16_t>(b);
          if (c.overflow) active = false;
        }
      } else if (active) {
        const uint32_t b = chain_request(c, st, base + k, sim_prev(ev), sim_J(ev), sim_La(ev));
        bst[lane * BST_STRIDE + k] = static_cast<uint16_t>(b);
        if (c.overflow) active = false;
      }
    }
    __syncwarp();
    if (AWARE && base < s) {  // burn-in tile: no output
      __syncwarp();
      continue;
    }
    // coalesced write-out: row r = lane r's instance, 64 contiguous bytes
    const unsigned act = __ballot_sync(0xFFFFFFFFu, active);
    for (int r = 0; r < 32; ++r) {
      const uint64_t off = shfl64(lp.boff, r);
      if (((act >> r) & 1u) && static_cast<uint32_t>(lane) < nk)
        bout[off + base + lane] = bst[r * BST_STRIDE + lane];
    }
    __syncwarp();
  }
  if (AWARE) {  // F_k and the segment's counters; overflowed segments are re-run by the fix-up
    if (lp.inst != 0xFFFFFFFFu) {
      const size_t slot = size_t(lp.aidx) * aw.nseg_max + it.seg;
      if (active) {
        if (bel) snap_write_belady(snapG + sw, aw.wsnap, c, st);
        else snap_write(snapG + sw, aw.wsnap, c, st);
      }
      aw.segc[2 * slot] = c.ev_trim;
      aw.segc[2 * slot + 1] = c.ev_lru;
      aw.segm[slot] = c.max_occ;
      aw.ovf[slot] = active ? 0u : 1u;
    }
    return;
  }
  if (active) {
    acc_commit(acc, lp.inst, c);
  } else if (lp.inst != 0xFFFFFFFFu) {  // overflowed: the spill kernel re-runs this chain
    unsigned slot = atomicAdd(nspill, 1u);
    spill[slot] = SpillDev{it.group, it.seg, static_cast<uint32_t>(lane), 0u};
  }
}

// Spill path: one thread per queued chain, state in global memory (W_big entries per slot).
__global__ void sim_spill_kernel(const GroupDev* __restrict__ groups, const LaneDev* __restrict__ lanes,
                                 const TraceDev* __restrict__ traces, uint32_t seg_len, uint16_t* __restrict__ bout,
                                 AccDev* acc, const SpillDev* spill, const unsigned int* nspill, uint32_t* tau_pool,
                                 uint16_t* X_pool, uint16_t* S_pool, uint32_t W_big, unsigned int* nfail) {
  const unsigned n = *nspill;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const SpillDev sp = spill[i];
    const GroupDev g = groups[sp.group];
    const TraceDev tr = traces[g.trace];
    const LaneDev lp = lanes[g.lane0 + sp.lane];
    const uint32_t s = sp.seg * seg_len;
    const uint32_t s_end = static_cast<uint32_t>(min(uint64_t(s) + seg_len, tr.E));
    const uint64_t slot = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    GlobalState st{tau_pool + slot * W_big, X_pool + slot * W_big, S_pool + slot * W_big};
    ChainRegs c;
    chain_init(c, lp.C, lp.D, lp.T, W_big, s > 0);
    for (int pass = 0; pass < 2; ++pass) {
      for (int64_t e = int64_t(s) - 1; e >= 0 && c.walking; --e) {
        if (tr.next[e] >= s) chain_walk_step(c, st, static_cast<uint32_t>(e), sim_La(tr.sim[e]));
      }
      if (!chain_walk_restart(c)) break;
    }
    chain_walk_finish(c);
    for (uint32_t e = s; e < s_end && !c.overflow; ++e) {
      const uint64_t ev = tr.sim[e];
      bout[lp.boff + e] = static_cast<uint16_t>(chain_request(c, st, e, sim_prev(ev), sim_J(ev), sim_La(ev)));
    }
    if (c.overflow) {
      atomicAdd(nfail, 1u);
    } else {
      acc_commit(acc, lp.inst, c);
    }
  }
}

// Fix-up of the End-/Length-Aware segments: one thread per aware lane walks its segments in
// order; a segment that overflowed or whose start state G_k differs from the exact end state
// F_{k-1} is re-run from F_{k-1} (from an empty cache for k = 0) with global-memory state, which
// also rewrites F_k.  Then the segment counters are summed into the instance's accumulators.
__global__ void aware_fix_kernel(const LaneDev* __restrict__ lanes, const uint32_t* __restrict__ alane,
                                 const uint32_t* __restrict__ atrace, uint32_t nal,
                                 const TraceDev* __restrict__ traces, uint16_t* __restrict__ bout, AccDev* acc,
                                 AwareDev aw, uint32_t* tau_pool, uint16_t* X_pool, uint16_t* S_pool, uint32_t Wp,
                                 unsigned int* nfail, unsigned int* nfixed) {
  const size_t sw = snap_words(aw.wsnap);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nal; i += gridDim.x * blockDim.x) {
    const LaneDev lp = lanes[alane[i]];
    const TraceDev tr = traces[atrace[i]];
    const bool bel = lp.policy == TLRU_POLICY_TAIL_BELADY || lp.policy == TLRU_POLICY_BELADY_FORCED;
    const uint32_t nseg = static_cast<uint32_t>((tr.E + aw.seg_len - 1) / aw.seg_len);
    GlobalState st{tau_pool + size_t(i) * Wp, X_pool + size_t(i) * Wp, S_pool + size_t(i) * Wp};
    bool failed = false, carry = false;  // carry: the pool holds the exact state at the end of segment k - 1
    ChainRegs c;
    for (uint32_t k = 0; k < nseg && !failed; ++k) {
      const size_t slot = size_t(i) * aw.nseg_max + k;
      uint32_t* G = aw.snap + slot * 2 * sw;
      uint32_t* F = G + sw;
      const uint32_t* Fp = k > 0 ? aw.snap + (slot - 1) * 2 * sw + sw : nullptr;
      if (!aw.ovf[slot] && (k == 0 || snap_equal(G, Fp, aw.wsnap))) {
        carry = false;
        continue;
      }
      if (!carry) {  // start from the exact state: empty (k = 0) or the saved F_{k-1}
        chain_init(c, lp.C, lp.D, lp.T, Wp, false);
        c.head = c.tail = c.fh = 0;
        if (k > 0) {
          if (Fp[0] == 0xFFFFFFFFu) {
            failed = true;
            break;
          }
          const uint32_t n = Fp[0];
          for (uint32_t j = 0; j < n; ++j) {
            const uint32_t xs = Fp[4 + aw.wsnap + j];
            st.T(j) = Fp[4 + j];
            st.Xr(j) = static_cast<uint16_t>(xs & 0xFFFFu);
            st.Sr(j) = static_cast<uint16_t>(xs >> 16);
            if (bel) c.fsum += xs >> 16;
          }
          c.tail = n;
          c.used = Fp[1];
          if (bel) {
            c.dead = Fp[2];
          } else {
            c.fh = Fp[2];
            c.frem = Fp[3];
          }
        }
      }
      c.ev_trim = c.ev_lru = c.max_occ = 0;
      const uint32_t s = k * aw.seg_len;
      const uint32_t s_end = static_cast<uint32_t>(min(uint64_t(s) + aw.seg_len, tr.E));
      for (uint32_t e = s; e < s_end && !c.overflow; ++e) {
        const uint64_t ev = tr.sim[e];
        const uint32_t nx = tr.next[e];
        const uint32_t qn = nx != TLRU_NONE ? sim_J(tr.sim[nx]) - sim_La(ev) : 0u;
        if (bel) {
          const uint32_t La = sim_La(ev);
          const uint32_t s0 = nx == TLRU_NONE ? 0u : min(La, lp.xi > qn ? lp.xi - qn : 0u);
          bout[lp.boff + e] = static_cast<uint16_t>(
              chain_request_belady(c, st, e, sim_J(ev), La, nx, s0, lp.policy == TLRU_POLICY_BELADY_FORCED));
          continue;
        }
        const uint32_t Dcur = lp.policy == TLRU_POLICY_LENGTH_AWARE ? (lp.xi > qn ? lp.xi - qn : 0u) : lp.D;
        const bool forced = lp.policy == TLRU_POLICY_TLRU_FORCED;
        bout[lp.boff + e] = static_cast<uint16_t>(chain_request_aware(c, st, e, sim_prev(ev), sim_J(ev), sim_La(ev),
                                                                      !forced && nx == TLRU_NONE, Dcur, forced));
      }
      if (c.overflow) {
        failed = true;
        break;
      }
      aw.segc[2 * slot] = c.ev_trim;
      aw.segc[2 * slot + 1] = c.ev_lru;
      aw.segm[slot] = c.max_occ;
      aw.ovf[slot] = 0;
      if (bel) snap_write_belady(F, aw.wsnap, c, st);
      else snap_write(F, aw.wsnap, c, st);
      carry = true;
      atomicAdd(nfixed, 1u);
    }
    if (failed) {
      atomicAdd(nfail, 1u);
      continue;
    }
    unsigned long long et = 0, el = 0;
    uint32_t mo = 0;
    for (uint32_t k = 0; k < nseg; ++k) {
      const size_t slot = size_t(i) * aw.nseg_max + k;
      et += aw.segc[2 * slot];
      el += aw.segc[2 * slot + 1];
      mo = max(mo, aw.segm[slot]);
    }
    acc[lp.inst].ev_trim = et;
    acc[lp.inst].ev_lru = el;
    acc[lp.inst].max_occ = mo;
  }
}

__global__ void sim_results_kernel(uint32_t ni, const AccDev* acc, tlru_result* results) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ni; i += gridDim.x * blockDim.x) {
    results[i].evicted_trim = acc[i].ev_trim;
    results[i].evicted_lru = acc[i].ev_lru;
    results[i].max_occupancy = acc[i].max_occ;
  }
}

// ----------------------------------------------------------------------------- planner
#ifndef TLRU_NOS_PACKED
#define TLRU_NOS_PACKED 1
#endif
#ifndef TLRU_FORCED_BURN
#define TLRU_FORCED_BURN 8192u  // forced-caching lanes' burn-in (fragments kept only by Phase 2 can be old)
#endif
static const int kWClasses[] = {32, 64, 96, 128, 256, 512, 1024};
constexpr int kNumW = 7;
constexpr int kSpillSlots = 128;

static thread_local uint32_t g_opt_seg = 0;  // tlru_set_sim_options
static thread_local int g_opt_w = -1;
static thread_local uint32_t g_opt_engine = TLRU_ENGINE_STACK;  // tlru_set_sim_engine
static thread_local double g_et_mu = -1.0;                      // tlru_set_etlru_model
static thread_local std::vector<double> g_et_table;

// Entries needed per lane for capacity C: live conversations are bounded by
// min(C + 1, conversations); the estimate below is the measured resident count of
// the WildChat-shaped preset with margin, x2 for tombstones between
// compactions.  Under-estimates are caught by the spill path, never truncated.
static int w_class(uint32_t C, uint32_t nconv) {
  double live = std::min<double>(double(C) + 1.0, double(nconv) + 1.0);
  double est = std::min(live, 0.8 * std::pow(double(C), 0.77) + 8.0);
  for (int i = 0; i < kNumW; ++i)
    if (kWClasses[i] >= 2.0 * est || kWClasses[i] > static_cast<int>(live) + 1) return i;
  return kNumW - 1;
}

static bool is_aware(const tlru_instance& in) { return in.policy >= TLRU_POLICY_END_AWARE; }
static uint32_t aware_kind(const tlru_instance& in) {
  if (in.policy == TLRU_POLICY_TAIL_BELADY || in.policy == TLRU_POLICY_BELADY_FORCED) return kAwareBelady;
  if (in.policy == TLRU_POLICY_TLRU_FORCED) return kAwareForced;
  return is_aware(in) ? kAwareTLRU : 0u;
}

struct Plan {
  std::vector<LaneDev> lanes;
  std::vector<GroupDev> groups;
  std::vector<ItemDev> items[kNumW];
  std::vector<ItemDev> items_aware[kNumW];  // Length-Aware / Belady segments (burn-in + fix-up)
  std::vector<ItemDev> items_nos[kNumW];    // End-Aware / forced-caching segments (no surplus array)
  bool any_aware = false;
  std::vector<uint32_t> alane, atrace;       // aware lane -> global lane index, trace
  uint32_t aseg = 8192, aburn = 4096, aburn_long = TLRU_FORCED_BURN, anseg_max = 1, awsnap = 32;
  bool any_forced = false;
  bool nos_packed = false;  // no-surplus lanes of the 256..1024-entry classes use SmemStatePk
  std::vector<EtItem> et_items;              // ET-LRU instances (etlru.cuh)
  std::vector<EtSeg> et_segs[kNumW];         // their (instance, segment) warps per state class
  uint32_t n_et = 0, et_seg_len = 8192, et_burn = 4096, et_nseg_max = 1, et_wsnap = 32;
  std::vector<TraceDev> traces;
  std::vector<SegDev> segs;
  uint32_t seg_len = 0;
  uint32_t bins = 1;
  uint32_t W_big = 32;
  uint64_t max_items = 0;
  uint64_t warm_bound = 0;
};

static tlru_status make_plan(const tlru_trace* traces, uint32_t nt, const tlru_instance* inst, uint32_t ni,
                             const uint64_t* offsets, Plan* P) {
  if (ni > 0 && !inst) TLRU_FAIL(TLRU_EINVAL, "inst is NULL");
  if (nt > 0 && !traces) TLRU_FAIL(TLRU_EINVAL, "traces is NULL");
  P->traces.resize(nt);
  uint32_t maxhist = 0;
  uint64_t Emax = 0;
  for (uint32_t t = 0; t < nt; ++t) {
    const tlru_trace& tr = traces[t];
    if (tr.num_events > 0 && (!tr.sim || !tr.next)) TLRU_FAIL(TLRU_EINVAL, "trace %u: sim/next is NULL", t);
    if (tr.num_events >= 0xFFFFFFFFull) TLRU_FAIL(TLRU_ERANGE, "trace %u: too many events", t);
    P->traces[t] = TraceDev{tr.sim, tr.next, tr.num_events, tr.time_ticks};
    maxhist = std::max(maxhist, tr.max_history);
    Emax = std::max<uint64_t>(Emax, tr.num_events);
  }
  if (maxhist > 65535) TLRU_FAIL(TLRU_ERANGE, "max_history > 65535");
  P->bins = maxhist + 1;
  // instance order: by trace, then W class, then C (lanes of a warp see similar state sizes)
  std::vector<uint32_t> order(ni);
  std::vector<int> wc(ni);
  uint32_t ni_lanes = ni;
  std::vector<int> et_cls;
  uint64_t packed = 0;
  P->segs.resize(ni);
  for (uint32_t i = 0; i < ni; ++i) {
    const tlru_instance& in = inst[i];
    if (in.trace >= nt) TLRU_FAIL(TLRU_EINVAL, "instance %u: trace index %u out of range", i, in.trace);
    if (in.policy > TLRU_POLICY_ETLRU_FORCED)
      TLRU_FAIL(TLRU_EUNSUPPORTED, "instance %u: policy %u is not built (0..9: LRU, T-LRU, Threshold-LRU, "
                "End-Aware, Length-Aware, Tail-Optimized Belady, ET-LRU, forced-caching T-LRU, forced-caching "
                "Tail-Optimized Belady, forced-caching ET-LRU)", i, in.policy);
    if (in.policy == TLRU_POLICY_ET_LRU || in.policy == TLRU_POLICY_ETLRU_FORCED) {
      if (g_et_mu < 0.0) TLRU_FAIL(TLRU_EINVAL, "instance %u: ET-LRU needs tlru_set_etlru_model first", i);
      if (traces[in.trace].num_events > 0 && !traces[in.trace].time_ticks)
        TLRU_FAIL(TLRU_EINVAL, "instance %u: ET-LRU needs the trace's time_ticks (beliefs, P:255)", i);
      if (traces[in.trace].num_events > 0 && (traces[in.trace].flags & TLRU_TRACE_SYNTHETIC_TICKS))
        TLRU_FAIL(TLRU_EINVAL, "instance %u: ET-LRU needs real arrival times, but trace %u was uploaded without "
                  "ticks (time_ticks holds event indices; beliefs decay with time, P:255)", i, in.trace);
    }
    if (in.policy >= TLRU_POLICY_END_AWARE) P->any_aware = true;
    if (in.policy == TLRU_POLICY_THRESHOLD && in.threshold > 65535)
      TLRU_FAIL(TLRU_ERANGE, "instance %u: threshold %u > 65535 (histories are u16)", i, in.threshold);
    order[i] = i;
    const uint32_t C = std::min<uint32_t>(in.capacity, 0x7FFF0000u);
    wc[i] = g_opt_w >= 0 ? g_opt_w : w_class(C, traces[in.trace].num_conversations);
    // aware chains keep 8 B per entry: 1024 x 32 lanes would exceed shared memory (spill covers the rest)
    // End-/Length-Aware chains keep a surplus array (8 B per entry): 1024 x 32 lanes would exceed
    // shared memory (the fix-up covers the rest).  Measured: bounding them by their live
    // conversations (128 or 256 entries) or splitting End- from Length-Aware lanes was slower on
    // the spectrum workload (wider capacity ranges per warp, more frequent compaction).
    // Forced-caching chains keep LRU-like state: up to 1024 entries of 6 B (no surplus array).
    if ((in.policy == TLRU_POLICY_TAIL_BELADY || in.policy == TLRU_POLICY_BELADY_FORCED ||
         in.policy == TLRU_POLICY_END_AWARE || in.policy == TLRU_POLICY_LENGTH_AWARE) &&
        g_opt_w < 0) {
      // End-/Length-Aware release a conversation's blocks at its last turn, so they too hold at
      // most the open conversations (~100 on the preset; measured: 96 entries, no re-run, spectrum
      // rows of a trace 239 -> 96.5 -> 84.7 ms at 512 / 128 / 96 entries -- 512 is one warp per SM)
      // entries hold X >= 1 (tombstones are compacted before the state counts as full), so
      // W > C never overflows; the live conversations of a trace bound it too (<= ~91 on the
      // preset): 96 entries, larger states are re-run by the fix-up from global memory
      const uint32_t need = std::min<uint32_t>(C + 1, 96u);
      int k = 0;
      while (k < kNumW - 1 && static_cast<uint32_t>(kWClasses[k]) < need) ++k;
      wc[i] = k;
    }
    // lanes with a surplus array (End-/Length-Aware, Belady) are launched for classes up to
    // kNumW - 2 only (1024 entries x 8 B x 32 lanes exceed shared memory): cap them whatever
    // tlru_set_sim_options asked for -- larger states are re-run by the fix-up
    if (is_aware(in) && aware_kind(in) != kAwareForced) wc[i] = std::min(wc[i], kNumW - 2);
    // forced-caching T-LRU lanes (6 B entries): 1024 entries x 32 lanes is one warp per SM; 512
    // (two warps) held every state of the preset up to C = 4096 (no re-run) and was 2.2x faster
    if (aware_kind(in) == kAwareForced && g_opt_w < 0) wc[i] = std::min(wc[i], kNumW - 2);
    const uint64_t E = traces[in.trace].num_events;
    const uint64_t off = offsets ? offsets[i] : packed;
    packed += E;
    P->segs[i] = SegDev{off, off + E, in.xi, in.slo, 0.0};
  }
  // ET-LRU instances run as warp-cooperative chains of their own (etlru.cuh), not in lane groups
  {
    std::vector<uint32_t> keep;
    for (uint32_t i : order) {
      const tlru_instance& in = inst[i];
      if (in.policy != TLRU_POLICY_ET_LRU && in.policy != TLRU_POLICY_ETLRU_FORCED) {
        keep.push_back(i);
        continue;
      }
      P->any_aware = true;
      const uint32_t C = std::min<uint32_t>(in.capacity, 0x7FFF0000u);
      const int k = g_opt_w >= 0 ? g_opt_w : w_class(C, traces[in.trace].num_conversations);
      P->et_items.push_back(EtItem{i, in.trace, C, in.xi, P->segs[i].begin,
                                   in.policy == TLRU_POLICY_ETLRU_FORCED ? 1u : 0u, 0u});
      et_cls.push_back(k);
      ++P->n_et;
    }
    order.swap(keep);
    ni_lanes = static_cast<uint32_t>(order.size());
    if (P->n_et) {  // segments of 3x the burn-in: the warps are latency-bound and their costs differ by
      // capacity, so many short warps balance better than one wave of long ones (measured on B200,
      // 10^6-conversation traces: 100 instances 1.6e8 -> 4.0e8 requests/s, 1000 instances 4.1e8 -> 5.2e8
      // against "148 x 24 warps"; profiles/r02_perf.md)
      uint64_t sl = 3ull * P->et_burn;
      if (g_opt_seg) sl = std::max<uint32_t>(g_opt_seg, 64);  // tests: short segments exercise the fix-up
      P->et_seg_len = static_cast<uint32_t>((sl + 31) & ~31ull);
      for (uint32_t k = 0; k < P->n_et; ++k) {
        const uint64_t E = traces[P->et_items[k].trace].num_events;
        const uint64_t ns = std::max<uint64_t>((E + P->et_seg_len - 1) / P->et_seg_len, 1);
        for (uint64_t sgi = 0; sgi < ns; ++sgi) P->et_segs[et_cls[k]].push_back(EtSeg{k, static_cast<uint32_t>(sgi)});
        P->et_nseg_max = std::max<uint32_t>(P->et_nseg_max, static_cast<uint32_t>(ns));
        P->et_wsnap = std::max<uint32_t>(P->et_wsnap, static_cast<uint32_t>(kWClasses[et_cls[k]]));
      }
    }
  }
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
    if (inst[a].trace != inst[b].trace) return inst[a].trace < inst[b].trace;
    if (aware_kind(inst[a]) != aware_kind(inst[b])) return aware_kind(inst[a]) < aware_kind(inst[b]);
    if (wc[a] != wc[b]) return wc[a] < wc[b];
    return inst[a].capacity < inst[b].capacity;
  });
  // lane groups
  for (uint32_t k = 0; k < ni_lanes;) {
    const uint32_t t = inst[order[k]].trace;
    const int w = wc[order[k]];
    const uint32_t kind = aware_kind(inst[order[k]]);
    const bool aw = kind != 0;
    GroupDev g{t, static_cast<uint32_t>(P->lanes.size()), 0, static_cast<uint32_t>(w), kind};
    while (k < ni_lanes && g.nlanes < 32 && inst[order[k]].trace == t && wc[order[k]] == w &&
           aware_kind(inst[order[k]]) == kind) {
      const tlru_instance& in = inst[order[k]];
      LaneDev l;
      l.inst = order[k];
      l.C = std::min<uint32_t>(in.capacity, 0x7FFF0000u);
      l.D = ((in.policy == TLRU_POLICY_TLRU || in.policy == TLRU_POLICY_END_AWARE ||
              in.policy == TLRU_POLICY_TLRU_FORCED) && in.xi > in.q_hat)
                ? in.xi - in.q_hat
                : 0u;  // free tail
      l.policy = in.policy;
      l.xi = in.xi;
      l.aidx = 0;
      l.pad = 0;
      if (aw) {
        l.aidx = static_cast<uint32_t>(P->alane.size());
        P->alane.push_back(static_cast<uint32_t>(P->lanes.size()));
        P->atrace.push_back(t);
        P->awsnap = std::max<uint32_t>(P->awsnap, static_cast<uint32_t>(kWClasses[w]));
      }
      l.T = in.policy == TLRU_POLICY_THRESHOLD ? in.threshold : 0u;  // admission (Reading #23)
      l.boff = P->segs[order[k]].begin;
      P->lanes.push_back(l);
      ++g.nlanes;
      ++k;
    }
    P->groups.push_back(g);
  }
  // segment length: enough warps to fill 148 SMs several times over
  const uint64_t G = P->groups.size();
  const uint64_t target = 148ull * 24ull;
  uint64_t parts = G ? (target + G - 1) / G : 1;
  uint64_t seg = Emax ? (Emax + parts - 1) / parts : 32;
  seg = std::max<uint64_t>(seg, 4096);
  if (g_opt_seg) seg = g_opt_seg;
  seg = std::min<uint64_t>(seg, 32768);  // u32 per-chain counters stay below 2^31
  seg = (seg + 31) & ~31ull;
  P->seg_len = static_cast<uint32_t>(seg);
  {  // aware segments: enough warps to fill the GPU, but >= 2x the burn-in
    for (const GroupDev& g : P->groups) {
      P->any_forced = P->any_forced || g.aware == kAwareForced;
    }
    // 3x the burn-in (forced caching: its long burn-in): short latency-bound warps balance better than
    // one wave of long ones (spectrum workload 1.30e10 -> 1.46e10 requests/s against "148 x 8 warps")
    uint64_t sa = P->any_forced ? P->aburn_long : 3ull * P->aburn;
    if (g_opt_seg) sa = std::max<uint32_t>(g_opt_seg, 64);  // tests: short segments exercise the fix-up
    P->aseg = static_cast<uint32_t>((sa + 31) & ~31ull);
    // SmemStatePk's fields: X <= max_history <= 4095 and tau - (segment start - burn-in) < 2^20
    P->nos_packed = TLRU_NOS_PACKED && maxhist <= 4095u &&
                    uint64_t(P->aseg) + std::max(P->aburn, P->aburn_long) < (1ull << 20);
  }
  uint64_t nitems = 0;
  for (uint32_t gi = 0; gi < P->groups.size(); ++gi) {
    const GroupDev& g = P->groups[gi];
    const uint64_t E = P->traces[g.trace].E;
    if (g.aware) {  // segments of aseg events, each with an aburn-event burn-in
      const uint64_t nsa = (E + P->aseg - 1) / P->aseg;
      auto& dst = g.aware == kAwareForced ? P->items_nos[g.W] : P->items_aware[g.W];
      for (uint64_t sgi = 0; sgi < nsa; ++sgi) dst.push_back(ItemDev{gi, static_cast<uint32_t>(sgi)});
      P->anseg_max = std::max<uint32_t>(P->anseg_max, static_cast<uint32_t>(nsa));
      nitems += nsa;
      continue;
    }
    const uint64_t nseg = (E + seg - 1) / seg;
    for (uint64_t sgi = 0; sgi < nseg; ++sgi) P->items[g.W].push_back(ItemDev{gi, static_cast<uint32_t>(sgi)});
    nitems += nseg;
  }
  P->max_items = nitems;
  // spill-state size: live entries <= min(C, conversations) + 1, x2 for tombstones
  uint32_t wb = 32;
  for (uint32_t i = 0; i < ni; ++i) {
    const uint64_t live =
        std::min<uint64_t>(std::min<uint32_t>(inst[i].capacity, 0x7FFF0000u), traces[inst[i].trace].num_conversations) + 2;
    wb = static_cast<uint32_t>(std::max<uint64_t>(wb, std::min<uint64_t>(2 * live + 2, 0xFFFFFFF0ull)));
  }
  P->W_big = wb;
  return TLRU_OK;
}

struct SimWs {
  LaneDev* lanes;
  GroupDev* groups;
  ItemDev* items;
  TraceDev* traces;
  SegDev* segs;
  AccDev* acc;
  SpillDev* spill;
  unsigned int* counters;  // [0] nspill, [1] nfail
  uint32_t* hist;
  unsigned long long* clamped;
  uint32_t* tau_pool;
  uint16_t* X_pool;
  uint16_t* S_pool;
  AwareDev aw;
  uint32_t* alane;
  uint32_t* atrace;
  uint32_t* atau;   // fix-up state pool [aware lane][awsnap]
  uint16_t* aX;
  uint16_t* aS;
  EtItem* et_items;         // ET-LRU instances
  EtSeg* et_segs;           // their segment warps, by state class
  double* et_table;         // ln P(Q >= k), k = 0..K
  EtSegs et_sg;             // snapshots and per-segment counters
  unsigned char* et_gpool;  // fix-up state pools [n_et][W_big slots x 24 B]
};

static void carve_sim(Carver& cv, const Plan& P, uint32_t ni, SimWs* w) {
  uint64_t nitems = 0;
  for (int k = 0; k < kNumW; ++k) nitems += P.items[k].size() + P.items_aware[k].size() + P.items_nos[k].size();
  w->lanes = cv.take<LaneDev>(P.lanes.size() + 1);
  w->groups = cv.take<GroupDev>(P.groups.size() + 1);
  w->items = cv.take<ItemDev>(nitems + 1);
  w->traces = cv.take<TraceDev>(P.traces.size() + 1);
  w->segs = cv.take<SegDev>(ni + 1);
  w->acc = cv.take<AccDev>(ni + 1);
  w->spill = cv.take<SpillDev>(nitems * 32 + 1);
  w->counters = cv.take<unsigned int>(4);  // nspill, nfail, aware segments re-run, ET-LRU re-runs
  w->hist = cv.take<uint32_t>(uint64_t(ni + 1) * P.bins);
  w->clamped = cv.take<unsigned long long>(ni + 1);
  w->tau_pool = cv.take<uint32_t>(uint64_t(kSpillSlots) * P.W_big);
  w->X_pool = cv.take<uint16_t>(uint64_t(kSpillSlots) * P.W_big);
  w->S_pool = cv.take<uint16_t>(uint64_t(kSpillSlots) * P.W_big);
  const uint64_t nal = P.alane.size();
  const uint64_t nsl = std::max<uint64_t>(nal, 1) * P.anseg_max;
  w->aw.seg_len = P.aseg;
  w->aw.burn = P.aburn;
  w->aw.burn_long = P.aburn_long;
  w->aw.nseg_max = P.anseg_max;
  w->aw.wsnap = P.awsnap;
  w->aw.snap = cv.take<uint32_t>(nal ? nsl * 2 * snap_words(P.awsnap) : 1);
  w->aw.segc = cv.take<unsigned long long>(nal ? 2 * nsl : 1);
  w->aw.segm = cv.take<uint32_t>(nal ? nsl : 1);
  w->aw.ovf = cv.take<uint32_t>(nal ? nsl : 1);
  w->alane = cv.take<uint32_t>(nal + 1);
  w->atrace = cv.take<uint32_t>(nal + 1);
  w->atau = cv.take<uint32_t>(nal ? nal * P.W_big : 1);  // fix-up state: as large as the spill state
  w->aX = cv.take<uint16_t>(nal ? nal * P.W_big : 1);
  w->aS = cv.take<uint16_t>(nal ? nal * P.W_big : 1);
  const uint64_t ne = P.n_et;
  uint64_t nes = 0;
  for (int k = 0; k < kNumW; ++k) nes += P.et_segs[k].size();
  w->et_items = cv.take<EtItem>(ne + 1);
  w->et_segs = cv.take<EtSeg>(nes + 1);
  w->et_table = cv.take<double>(g_et_table.size() + 1);
  const uint64_t nse = std::max<uint64_t>(ne, 1) * P.et_nseg_max;
  w->et_sg.seg_len = P.et_seg_len;
  w->et_sg.burn = P.et_burn;
  w->et_sg.nseg_max = P.et_nseg_max;
  w->et_sg.wsnap = P.et_wsnap;
  w->et_sg.snap = cv.take<uint32_t>(ne ? nse * 2 * et_snap_words(P.et_wsnap) : 1);
  w->et_sg.segc = cv.take<unsigned long long>(ne ? 2 * nse : 1);
  w->et_sg.segm = cv.take<uint32_t>(ne ? nse : 1);
  w->et_sg.ovf = cv.take<uint32_t>(ne ? nse : 1);
  w->et_gpool = cv.take<unsigned char>(ne ? ne * uint64_t(P.W_big) * 24 : 1);
}

static thread_local tlru_sim_stats g_stats;
static thread_local unsigned int* g_counters = nullptr;
static thread_local cudaEvent_t g_ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
static thread_local OutTiming g_out;  // s2_out interval (g_ev[3], g_ev[4])
static thread_local bool g_ev_recorded = false;

static tlru_status record(int k, cudaStream_t st) {
  if (!g_ev[k]) TLRU_CUDA(cudaEventCreate(&g_ev[k]));
  TLRU_CUDA(cudaEventRecord(g_ev[k], st));
  return TLRU_OK;
}

#ifndef TLRU_CLASS_STREAMS
#define TLRU_CLASS_STREAMS 4
#endif
// The per-state-class kernels of one batch are independent (disjoint instances); each class's
// last wave leaves SMs idle, so they are forked over a small per-(host thread, device) pool of
// streams and joined back onto the caller's stream before the fix-up kernels.
struct ClassStreams {
  cudaStream_t s[TLRU_CLASS_STREAMS];
  cudaEvent_t fork, join[TLRU_CLASS_STREAMS];
  bool init = false;
};
// per (host thread, device, caller stream): callers on distinct streams never share a pool, so their
// batches still overlap each other
static thread_local std::vector<std::pair<cudaStream_t, ClassStreams>> g_class_streams[16];

static tlru_status class_streams(cudaStream_t caller, ClassStreams** out) {
  int dev = 0;
  TLRU_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 16) TLRU_FAIL(TLRU_EUNSUPPORTED, "device %d", dev);
  auto& pools = g_class_streams[dev];
  size_t idx = 0;
  while (idx < pools.size() && pools[idx].first != caller) ++idx;
  if (idx == pools.size()) pools.emplace_back(caller, ClassStreams{});
  ClassStreams& c = pools[idx].second;
  if (!c.init) {
    for (int i = 0; i < TLRU_CLASS_STREAMS; ++i) {
      TLRU_CUDA(cudaStreamCreateWithFlags(&c.s[i], cudaStreamNonBlocking));
      TLRU_CUDA(cudaEventCreateWithFlags(&c.join[i], cudaEventDisableTiming));
    }
    TLRU_CUDA(cudaEventCreateWithFlags(&c.fork, cudaEventDisableTiming));
    c.init = true;
  }
  *out = &c;
  return TLRU_OK;
}

template <int W, bool AWARE, bool NOS = false, bool PK = false>
static tlru_status launch_w(const std::vector<ItemDev>& items, const ItemDev* d_items, const SimWs& w,
                            uint32_t seg_len, uint16_t* bout, cudaStream_t st) {
  if (items.empty()) return TLRU_OK;
  const size_t smem =
      size_t(W) * 32 * (sizeof(uint32_t) + (PK ? 0 : ((AWARE && !NOS) ? 2 : 1)) * sizeof(uint16_t)) +
      32 * BST_STRIDE * sizeof(uint16_t);
  TLRU_CUDA(cudaFuncSetAttribute(sim_kernel<W, AWARE, NOS, PK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  sim_kernel<W, AWARE, NOS, PK><<<static_cast<unsigned>(items.size()), 32, smem, st>>>(
      d_items, w.groups, w.lanes, w.traces, seg_len, bout, w.acc, w.spill, w.counters, w.aw);
  TLRU_CHECK_LAUNCH();
  ++g_stats.kernels;
  return TLRU_OK;
}

template <int W>
static tlru_status launch_et(const std::vector<EtSeg>& segs, const EtSeg* d_segs, const SimWs& w, const EtModel& m,
                             uint16_t* bout, cudaStream_t st) {
  if (segs.empty()) return TLRU_OK;
  const size_t smem = kEtTab * sizeof(double) + size_t(W) * 24;  // table, key, base, tau, X, L
  TLRU_CUDA(cudaFuncSetAttribute(etlru_seg_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  etlru_seg_kernel<W><<<static_cast<unsigned>(segs.size()), 32, smem, st>>>(d_segs, w.et_items, w.traces, m, w.et_sg,
                                                                            bout);
  TLRU_CHECK_LAUNCH();
  ++g_stats.kernels;
  return TLRU_OK;
}

}  // namespace tlru

using namespace tlru;

// Engine of one instance: the stack engine needs the stack property (LRU, T-LRU,
// Threshold-LRU) and a universe that keeps its 32-bit window sums exact.
constexpr uint64_t kStackUniverseMax = 0xFFFF0000ull;
static uint32_t engine_of(const tlru_instance& in, const tlru_trace* traces) {
  if (g_opt_engine == TLRU_ENGINE_REPLAY || in.policy > TLRU_POLICY_THRESHOLD) return TLRU_ENGINE_REPLAY;
  if (traces[in.trace].universe_blocks > kStackUniverseMax) return TLRU_ENGINE_REPLAY;
  return TLRU_ENGINE_STACK;
}

// Workspace bytes of one engine for these instances (offsets do not change sizes).
static tlru_status engine_ws_bytes(uint32_t engine, const tlru_trace* traces, uint32_t nt, const tlru_instance* inst,
                                   uint32_t ni, size_t* bytes) {
  Plan P;
  TLRU_TRY(make_plan(traces, nt, inst, ni, nullptr, &P));
  if (engine == TLRU_ENGINE_REPLAY) {
    Carver cv(nullptr);
    SimWs w;
    carve_sim(cv, P, ni, &w);
    *bytes = cv.used;
    return TLRU_OK;
  }
  size_t sb = 0;
  TLRU_TRY(stack_workspace(traces, nt, inst, ni, &sb));
  Carver cv2(nullptr);
  cv2.take<SegDev>(ni + 1);
  cv2.take<uint32_t>(uint64_t(ni + 1) * P.bins);
  cv2.take<unsigned long long>(ni + 1);
  *bytes = cv2.used + 256 + sb;
  return TLRU_OK;
}

// The batch split by engine: ids[e] = instances of engine e (ascending).
struct EngineSplit {
  std::vector<uint32_t> ids[2];
  bool mixed() const { return !ids[0].empty() && !ids[1].empty(); }
};

static tlru_status split_batch(const tlru_trace* traces, uint32_t nt, const tlru_instance* inst, uint32_t ni,
                               EngineSplit* S) {
  if (ni > 0 && !inst) TLRU_FAIL(TLRU_EINVAL, "inst is NULL");
  if (nt > 0 && !traces) TLRU_FAIL(TLRU_EINVAL, "traces is NULL");
  for (uint32_t i = 0; i < ni; ++i) {
    if (inst[i].trace >= nt) TLRU_FAIL(TLRU_EINVAL, "instance %u: trace index %u out of range", i, inst[i].trace);
    S->ids[engine_of(inst[i], traces)].push_back(i);
  }
  return TLRU_OK;
}

// Mixed batch: [results of the sub-batches (tlru_result[ni]), instance maps (u32[ni])] then the
// larger engine's workspace.
static void carve_mixed(Carver& cv, uint32_t ni, tlru_result** res_tmp, uint32_t** map) {
  *res_tmp = cv.take<tlru_result>(ni + 1);
  *map = cv.take<uint32_t>(ni + 1);
}

static tlru_status sub_batch(const tlru_instance* inst, const uint64_t* offs, const std::vector<uint32_t>& ids,
                             std::vector<tlru_instance>* si, std::vector<uint64_t>* so) {
  si->resize(ids.size());
  so->resize(ids.size());
  for (size_t k = 0; k < ids.size(); ++k) {
    (*si)[k] = inst[ids[k]];
    (*so)[k] = offs[ids[k]];
  }
  return TLRU_OK;
}

extern "C" tlru_status tlru_sim_workspace_size(const tlru_trace* traces, uint32_t nt, const tlru_instance* inst,
                                               uint32_t ni, size_t* bytes) {
  clear_error();
  if (!bytes) TLRU_FAIL(TLRU_EINVAL, "bytes is NULL");
  EngineSplit S;
  TLRU_TRY(split_batch(traces, nt, inst, ni, &S));
  if (!S.mixed()) {  // one engine: either may be selected at run time, size for both
    Plan P;
    TLRU_TRY(make_plan(traces, nt, inst, ni, nullptr, &P));
    size_t a = 0, b = 0;
    TLRU_TRY(engine_ws_bytes(TLRU_ENGINE_REPLAY, traces, nt, inst, ni, &a));
    TLRU_TRY(engine_ws_bytes(TLRU_ENGINE_STACK, traces, nt, inst, ni, &b));
    *bytes = std::max(a, b);
    return TLRU_OK;
  }
  std::vector<uint64_t> zero(ni, 0);
  size_t need = 0;
  for (int e = 0; e < 2; ++e) {
    std::vector<tlru_instance> si;
    std::vector<uint64_t> so;
    sub_batch(inst, zero.data(), S.ids[e], &si, &so);
    size_t b = 0;
    TLRU_TRY(engine_ws_bytes(static_cast<uint32_t>(e), traces, nt, si.data(), static_cast<uint32_t>(si.size()), &b));
    need = std::max(need, b);
  }
  Carver cv(nullptr);
  tlru_result* r;
  uint32_t* m;
  carve_mixed(cv, ni, &r, &m);
  *bytes = ((cv.used + 255) & ~size_t(255)) + need;
  return TLRU_OK;
}

__global__ void scatter_results_kernel(const tlru_result* __restrict__ src, const uint32_t* __restrict__ map,
                                       uint32_t n, tlru_result* __restrict__ dst) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[map[i]] = src[i];
}

// One engine over ni instances with explicit (host) offsets.  results / the histogram export take
// row i, or row hist_map[i] of hist_out (device map, nullable).  `timing`: record g_ev / the s2_out
// interval (a mixed batch records around both engines instead).
static tlru_status run_engine(uint32_t engine, const tlru_trace* traces, uint32_t nt, const tlru_instance* inst,
                              uint32_t ni, uint16_t* uncached, const uint64_t* offsets, tlru_result* results,
                              uint32_t* hist_out, uint32_t hist_bins, const uint32_t* hist_map, void* ws,
                              size_t ws_bytes, cudaStream_t st, bool timing) {
  if (ni == 0) return TLRU_OK;
  Plan P;
  TLRU_TRY(make_plan(traces, nt, inst, ni, offsets, &P));
  if (!uncached) {
    for (uint32_t i = 0; i < ni; ++i)
      if (traces[inst[i].trace].num_events > 0) TLRU_FAIL(TLRU_EINVAL, "uncached is NULL");
  }
  if (hist_out && hist_bins < P.bins)
    TLRU_FAIL(TLRU_ERANGE, "hist_bins = %u must exceed every trace's max_history (%u)", hist_bins, P.bins - 1);
  if (engine == TLRU_ENGINE_STACK) {
    Carver cv(ws);
    SegDev* segs = cv.take<SegDev>(ni + 1);
    uint32_t* hist = cv.take<uint32_t>(uint64_t(ni + 1) * P.bins);
    unsigned long long* clamped = cv.take<unsigned long long>(ni + 1);
    TLRU_TRY(check_ws(cv, ws, ws_bytes));
    std::vector<uint64_t> boffs(ni);
    for (uint32_t i = 0; i < ni; ++i) boffs[i] = P.segs[i].begin;
    TLRU_CUDA(cudaMemcpyAsync(segs, P.segs.data(), ni * sizeof(SegDev), cudaMemcpyHostToDevice, st));
    TLRU_CUDA(cudaMemsetAsync(hist, 0, uint64_t(ni) * P.bins * sizeof(uint32_t), st));
    TLRU_CUDA(cudaMemsetAsync(clamped, 0, ni * sizeof(unsigned long long), st));
    unsigned nk = 0;
    if (timing) TLRU_TRY(record(0, st));
    for (int k = 1; k < 5; ++k)
      if (!g_ev[k]) TLRU_CUDA(cudaEventCreate(&g_ev[k]));
    if (timing || g_out.first == nullptr) g_out = OutTiming{g_ev[3], g_ev[4], g_out.launches};
    TLRU_TRY(stack_simulate(traces, nt, inst, ni, boffs.data(), uncached, results, cv, segs, P.bins, hist, clamped,
                            ws_bytes, st, &nk, timing ? g_ev[1] : nullptr, &g_out));  // g_ev[1]: engine | K3
    TLRU_TRY(launch_hist_export(hist, ni, P.bins, hist_map, hist_out, hist_bins, st));
    if (timing) {
      TLRU_TRY(record(2, st));
      g_ev_recorded = true;
    }
    g_stats.kernels += nk + (hist_out ? 1u : 0u);
    return TLRU_OK;
  }
  Carver cv(ws);
  SimWs w;
  carve_sim(cv, P, ni, &w);
  TLRU_TRY(check_ws(cv, ws, ws_bytes));
  // tables -> device (pageable copies complete before the call returns)
  std::vector<ItemDev> all_items;
  size_t item_off[kNumW + 1], aware_off[kNumW], nos_off[kNumW];
  for (int k = 0; k < kNumW; ++k) {
    item_off[k] = all_items.size();
    all_items.insert(all_items.end(), P.items[k].begin(), P.items[k].end());
  }
  item_off[kNumW] = all_items.size();
  for (int k = 0; k < kNumW; ++k) {
    aware_off[k] = all_items.size();
    all_items.insert(all_items.end(), P.items_aware[k].begin(), P.items_aware[k].end());
  }
  for (int k = 0; k < kNumW; ++k) {
    nos_off[k] = all_items.size();
    all_items.insert(all_items.end(), P.items_nos[k].begin(), P.items_nos[k].end());
  }
  TLRU_CUDA(cudaMemcpyAsync(w.lanes, P.lanes.data(), P.lanes.size() * sizeof(LaneDev), cudaMemcpyHostToDevice, st));
  TLRU_CUDA(cudaMemcpyAsync(w.groups, P.groups.data(), P.groups.size() * sizeof(GroupDev), cudaMemcpyHostToDevice, st));
  if (!all_items.empty())
    TLRU_CUDA(cudaMemcpyAsync(w.items, all_items.data(), all_items.size() * sizeof(ItemDev), cudaMemcpyHostToDevice, st));
  TLRU_CUDA(cudaMemcpyAsync(w.traces, P.traces.data(), P.traces.size() * sizeof(TraceDev), cudaMemcpyHostToDevice, st));
  TLRU_CUDA(cudaMemcpyAsync(w.segs, P.segs.data(), ni * sizeof(SegDev), cudaMemcpyHostToDevice, st));
  TLRU_CUDA(cudaMemsetAsync(w.acc, 0, ni * sizeof(AccDev), st));
  TLRU_CUDA(cudaMemsetAsync(w.counters, 0, 4 * sizeof(unsigned int), st));
  std::vector<EtSeg> et_all;
  size_t et_off[kNumW];
  for (int k = 0; k < kNumW; ++k) {
    et_off[k] = et_all.size();
    et_all.insert(et_all.end(), P.et_segs[k].begin(), P.et_segs[k].end());
  }
  if (P.n_et) {
    TLRU_CUDA(cudaMemcpyAsync(w.et_items, P.et_items.data(), P.n_et * sizeof(EtItem), cudaMemcpyHostToDevice, st));
    TLRU_CUDA(cudaMemcpyAsync(w.et_segs, et_all.data(), et_all.size() * sizeof(EtSeg), cudaMemcpyHostToDevice, st));
    TLRU_CUDA(cudaMemcpyAsync(w.et_table, g_et_table.data(), g_et_table.size() * sizeof(double),
                              cudaMemcpyHostToDevice, st));
  }
  if (!P.alane.empty()) {
    TLRU_CUDA(cudaMemcpyAsync(w.alane, P.alane.data(), P.alane.size() * 4, cudaMemcpyHostToDevice, st));
    TLRU_CUDA(cudaMemcpyAsync(w.atrace, P.atrace.data(), P.atrace.size() * 4, cudaMemcpyHostToDevice, st));
  }
  TLRU_CUDA(cudaMemsetAsync(w.hist, 0, uint64_t(ni) * P.bins * sizeof(uint32_t), st));
  TLRU_CUDA(cudaMemsetAsync(w.clamped, 0, ni * sizeof(unsigned long long), st));
  // K2: largest state class first (longest per-event latency); classes forked over the pool
  if (timing) TLRU_TRY(record(0, st));
  ClassStreams* cs = nullptr;
  const bool fork = TLRU_CLASS_STREAMS > 1;
  if (fork) {
    TLRU_TRY(class_streams(st, &cs));
    TLRU_CUDA(cudaEventRecord(cs->fork, st));
    for (int i = 0; i < TLRU_CLASS_STREAMS; ++i) TLRU_CUDA(cudaStreamWaitEvent(cs->s[i], cs->fork, 0));
  }
  const cudaStream_t st_caller = st;
  int rr = 0;
  auto next_stream = [&]() { return fork ? cs->s[(rr++) % TLRU_CLASS_STREAMS] : st_caller; };
  for (int k = kNumW - 1; k >= 0; --k) {
    const cudaStream_t st = next_stream();
    const ItemDev* d = w.items + item_off[k];
    const ItemDev* da = w.items + aware_off[k];
    const std::vector<ItemDev>& ia = P.items_aware[k];
    const ItemDev* dn = w.items + nos_off[k];
    const std::vector<ItemDev>& in_ = P.items_nos[k];
    switch (k) {
      case 0: TLRU_TRY((launch_w<32, false>(P.items[k], d, w, P.seg_len, uncached, st)));
              TLRU_TRY((launch_w<32, true>(ia, da, w, P.seg_len, uncached, st)));
              TLRU_TRY((launch_w<32, true, true>(in_, dn, w, P.seg_len, uncached, st))); break;
      case 1: TLRU_TRY((launch_w<64, false>(P.items[k], d, w, P.seg_len, uncached, st)));
              TLRU_TRY((launch_w<64, true>(ia, da, w, P.seg_len, uncached, st)));
              TLRU_TRY((launch_w<64, true, true>(in_, dn, w, P.seg_len, uncached, st))); break;
      case 2: TLRU_TRY((launch_w<96, false>(P.items[k], d, w, P.seg_len, uncached, st)));
              TLRU_TRY((launch_w<96, true>(ia, da, w, P.seg_len, uncached, st)));
              TLRU_TRY((launch_w<96, true, true>(in_, dn, w, P.seg_len, uncached, st))); break;
      case 3: TLRU_TRY((launch_w<128, false>(P.items[k], d, w, P.seg_len, uncached, st)));
              TLRU_TRY((launch_w<128, true>(ia, da, w, P.seg_len, uncached, st)));
              TLRU_TRY((launch_w<128, true, true>(in_, dn, w, P.seg_len, uncached, st))); break;
      case 4: TLRU_TRY((launch_w<256, false>(P.items[k], d, w, P.seg_len, uncached, st)));
              TLRU_TRY((launch_w<256, true>(ia, da, w, P.seg_len, uncached, st)));
              if (P.nos_packed) TLRU_TRY((launch_w<256, true, true, true>(in_, dn, w, P.seg_len, uncached, st)));
              else TLRU_TRY((launch_w<256, true, true>(in_, dn, w, P.seg_len, uncached, st)));
              break;
      case 5: TLRU_TRY((launch_w<512, false>(P.items[k], d, w, P.seg_len, uncached, st)));
              TLRU_TRY((launch_w<512, true>(ia, da, w, P.seg_len, uncached, st)));
              if (P.nos_packed) TLRU_TRY((launch_w<512, true, true, true>(in_, dn, w, P.seg_len, uncached, st)));
              else TLRU_TRY((launch_w<512, true, true>(in_, dn, w, P.seg_len, uncached, st)));
              break;
      case 6: TLRU_TRY((launch_w<1024, false>(P.items[k], d, w, P.seg_len, uncached, st)));
              if (P.nos_packed) TLRU_TRY((launch_w<1024, true, true, true>(in_, dn, w, P.seg_len, uncached, st)));
              else TLRU_TRY((launch_w<1024, true, true>(in_, dn, w, P.seg_len, uncached, st)));
              break;
    }
  }
  if (P.n_et) {  // ET-LRU: one warp per (instance, segment), shared-memory state per class
    const EtModel m{w.et_table, static_cast<uint32_t>(g_et_table.size() - 1), g_et_mu};
    for (int k = kNumW - 1; k >= 0; --k) {
      const std::vector<EtSeg>& v = P.et_segs[k];
      const EtSeg* d = w.et_segs + et_off[k];
      // ET-LRU classes stay on the caller's stream, largest first: forked, the small classes' warps
      // took SM slots from the largest class (the critical path) -- 10-trace workload 6.3e8 -> 5.6e8
      const cudaStream_t st = st_caller;
      switch (k) {
        case 0: TLRU_TRY((launch_et<32>(v, d, w, m, uncached, st))); break;
        case 1: TLRU_TRY((launch_et<64>(v, d, w, m, uncached, st))); break;
        case 2: TLRU_TRY((launch_et<96>(v, d, w, m, uncached, st))); break;
        case 3: TLRU_TRY((launch_et<128>(v, d, w, m, uncached, st))); break;
        case 4: TLRU_TRY((launch_et<256>(v, d, w, m, uncached, st))); break;
        case 5: TLRU_TRY((launch_et<512>(v, d, w, m, uncached, st))); break;
        case 6: TLRU_TRY((launch_et<1024>(v, d, w, m, uncached, st))); break;
      }
    }
  }
  if (fork) {  // join every class kernel back onto the caller's stream before the fix-up kernels
    for (int i = 0; i < TLRU_CLASS_STREAMS; ++i) {
      TLRU_CUDA(cudaEventRecord(cs->join[i], cs->s[i]));
      TLRU_CUDA(cudaStreamWaitEvent(st_caller, cs->join[i], 0));
    }
  }
  if (P.n_et) {
    const EtModel m{w.et_table, static_cast<uint32_t>(g_et_table.size() - 1), g_et_mu};
    // fix-up: re-run every segment whose start state was not exact (or that outgrew its slots)
    etlru_fix_kernel<<<P.n_et, 32, 0, st>>>(w.et_items, P.n_et, w.traces, m, w.et_sg, uncached, w.acc, w.et_gpool,
                                            P.W_big, w.counters + 3, w.counters + 1);
    TLRU_CHECK_LAUNCH();
    ++g_stats.kernels;
  }
  // spill path: always launched; exits at once when the queue is empty (no host sync)
  sim_spill_kernel<<<kSpillSlots / 32, 32, 0, st>>>(w.groups, w.lanes, w.traces, P.seg_len, uncached, w.acc, w.spill,
                                                    w.counters, w.tau_pool, w.X_pool, w.S_pool, P.W_big,
                                                    w.counters + 1);
  TLRU_CHECK_LAUNCH();
  ++g_stats.kernels;
  if (!P.alane.empty()) {  // End-/Length-Aware fix-up (exactness of the burn-in segments)
    const uint32_t nal = static_cast<uint32_t>(P.alane.size());
    aware_fix_kernel<<<(nal + 31) / 32, 32, 0, st>>>(w.lanes, w.alane, w.atrace, nal, w.traces, uncached, w.acc, w.aw,
                                                     w.atau, w.aX, w.aS, P.W_big, w.counters + 1, w.counters + 2);
    TLRU_CHECK_LAUNCH();
    ++g_stats.kernels;
  }
  if (timing) TLRU_TRY(record(1, st));
  // K3: histogram of b per instance -> percentiles, TEL, SLO; then the counters
  TLRU_TRY(launch_hist(uncached, w.segs, ni, P.bins, w.hist, w.clamped, st));
  TLRU_TRY(launch_finalize(w.segs, ni, P.bins, w.hist, w.clamped, 1.0, nullptr, results, st));
  sim_results_kernel<<<grid_for(ni, 128), 128, 0, st>>>(ni, w.acc, results);
  TLRU_CHECK_LAUNCH();
  TLRU_TRY(launch_hist_export(w.hist, ni, P.bins, hist_map, hist_out, hist_bins, st));
  if (timing) {
    TLRU_TRY(record(2, st));
    g_ev_recorded = true;
  }
  g_stats.kernels += 3 + (hist_out ? 1u : 0u);
  g_stats.chains = 0;
  for (int k = 0; k < kNumW; ++k)
    g_stats.chains += (P.items[k].size() + P.items_aware[k].size() + P.items_nos[k].size()) * 32 +
                      P.et_segs[k].size();
  g_stats.segment_events = P.seg_len;
  for (int k = kNumW - 1; k >= 0; --k)
    if (!P.items[k].empty() || !P.items_aware[k].empty() || !P.items_nos[k].empty()) {
      g_stats.state_entries = kWClasses[k];
      break;
    }
  g_counters = w.counters;
  return TLRU_OK;
}


extern "C" tlru_status tlru_simulate_batch_ex(const tlru_trace* traces, uint32_t nt, const tlru_instance* inst,
                                              uint32_t ni, uint16_t* uncached, const uint64_t* offsets,
                                              tlru_result* results, uint32_t* hist, uint32_t hist_bins, void* ws,
                                              size_t ws_bytes, cudaStream_t st) {
  clear_error();
  g_stats = tlru_sim_stats{};
  g_counters = nullptr;
  g_ev_recorded = false;
  g_out = OutTiming{};
  if (ni == 0) return TLRU_OK;
  if (!results) TLRU_FAIL(TLRU_EINVAL, "results is NULL");
  if (hist && hist_bins == 0) TLRU_FAIL(TLRU_ERANGE, "hist_bins must be > 0");
  EngineSplit S;
  TLRU_TRY(split_batch(traces, nt, inst, ni, &S));
  std::vector<uint64_t> offs(ni);  // explicit offsets (packed prefix sums of E_i when NULL)
  for (uint64_t i = 0, packed = 0; i < ni; ++i) {
    offs[i] = offsets ? offsets[i] : packed;
    packed += traces[inst[i].trace].num_events;
  }
  if (!S.mixed()) {
    g_stats.engine = S.ids[TLRU_ENGINE_STACK].empty() ? TLRU_ENGINE_REPLAY : TLRU_ENGINE_STACK;
    return run_engine(g_stats.engine, traces, nt, inst, ni, uncached, offs.data(), results, hist, hist_bins, nullptr,
                      ws, ws_bytes, st, true);
  }
  // both engines, each on its own instances (stack first: its s2_out interval is the dominant kernel)
  g_stats.engine = TLRU_ENGINE_MIXED;
  Carver cv(ws);
  tlru_result* res_tmp;
  uint32_t* map;
  carve_mixed(cv, ni, &res_tmp, &map);
  TLRU_TRY(check_ws(cv, ws, ws_bytes));
  const size_t head = (cv.used + 255) & ~size_t(255);
  if (ws_bytes < head) TLRU_FAIL(TLRU_ERANGE, "workspace too small for a mixed batch");
  std::vector<uint32_t> allmap;
  for (int e = 1; e >= 0; --e) allmap.insert(allmap.end(), S.ids[e].begin(), S.ids[e].end());
  TLRU_CUDA(cudaMemcpyAsync(map, allmap.data(), ni * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
  TLRU_TRY(record(0, st));
  uint32_t done = 0;
  uint32_t kernels = 0;
  for (int e = 1; e >= 0; --e) {
    std::vector<tlru_instance> si;
    std::vector<uint64_t> so;
    sub_batch(inst, offs.data(), S.ids[e], &si, &so);
    const uint32_t n = static_cast<uint32_t>(si.size());
    g_stats.kernels = 0;
    TLRU_TRY(run_engine(static_cast<uint32_t>(e), traces, nt, si.data(), n, uncached, so.data(), res_tmp + done, hist,
                        hist_bins, map + done, static_cast<char*>(ws) + head, ws_bytes - head, st, false));
    kernels += g_stats.kernels;
    done += n;
  }
  scatter_results_kernel<<<grid_for(ni, 128), 128, 0, st>>>(res_tmp, map, ni, results);
  TLRU_CHECK_LAUNCH();
  TLRU_TRY(record(1, st));
  TLRU_TRY(record(2, st));
  g_ev_recorded = true;
  g_stats.kernels = kernels + 1;
  return TLRU_OK;
}

extern "C" tlru_status tlru_simulate_batch(const tlru_trace* traces, uint32_t nt, const tlru_instance* inst,
                                           uint32_t ni, uint16_t* uncached, const uint64_t* offsets,
                                           tlru_result* results, void* ws, size_t ws_bytes, cudaStream_t st) {
  return tlru_simulate_batch_ex(traces, nt, inst, ni, uncached, offsets, results, nullptr, 0, ws, ws_bytes, st);
}

extern "C" tlru_status tlru_set_sim_options(uint32_t segment_events, uint32_t state_entries) {
  clear_error();
  if (segment_events > 32768) TLRU_FAIL(TLRU_ERANGE, "segment_events must be <= 32768");
  int w = -1;
  if (state_entries) {
    for (int k = 0; k < kNumW; ++k)
      if (static_cast<uint32_t>(kWClasses[k]) == state_entries) w = k;
    if (w < 0) TLRU_FAIL(TLRU_EINVAL, "state_entries must be 0 or one of 32, 64, 96, 128, 256, 512, 1024");
  }
  g_opt_seg = segment_events;
  g_opt_w = w;
  return TLRU_OK;
}

extern "C" tlru_status tlru_set_etlru_model(double mu_per_tick, const double* ln_surv, uint32_t K) {
  clear_error();
  if (!(mu_per_tick >= 0.0) || mu_per_tick > 1e300) TLRU_FAIL(TLRU_EINVAL, "mu_per_tick must be finite and >= 0");
  if (!ln_surv) TLRU_FAIL(TLRU_EINVAL, "ln_surv is NULL");
  if (K > 65535) TLRU_FAIL(TLRU_ERANGE, "K must be <= 65535");
  for (uint32_t k = 0; k <= K; ++k) {
    const double v = ln_surv[k];
    if (v != v || v > 0.0) TLRU_FAIL(TLRU_EINVAL, "ln_surv[%u] must be <= 0 (a log-probability), not NaN", k);
    if (k > 0 && v > ln_surv[k - 1]) TLRU_FAIL(TLRU_EINVAL, "ln_surv must be non-increasing (at k = %u)", k);
  }
  g_et_table.assign(ln_surv, ln_surv + K + 1);
  for (double& v : g_et_table) v += 0.0;  // -0.0 -> +0.0 (etlru.cuh orders scores as integers)
  g_et_mu = mu_per_tick + 0.0;
  return TLRU_OK;
}

extern "C" tlru_status tlru_set_sim_engine(uint32_t engine) {
  clear_error();
  if (engine != TLRU_ENGINE_REPLAY && engine != TLRU_ENGINE_STACK)
    TLRU_FAIL(TLRU_EINVAL, "engine must be TLRU_ENGINE_REPLAY (0) or TLRU_ENGINE_STACK (1)");
  g_opt_engine = engine;
  return TLRU_OK;
}

extern "C" tlru_status tlru_last_sim_stats(tlru_sim_stats* out) {
  clear_error();
  if (!out) TLRU_FAIL(TLRU_EINVAL, "out is NULL");
  *out = g_stats;
  if (g_counters) {
    unsigned int c[4] = {0, 0, 0, 0};
    TLRU_CUDA(cudaDeviceSynchronize());
    TLRU_CUDA(cudaMemcpy(c, g_counters, sizeof(c), cudaMemcpyDeviceToHost));
    out->spilled_chains = c[0] + c[2] + c[3];  // incl. aware segments re-run by the fix-up, ET-LRU re-runs
    out->failed_chains = c[1];
  }
  if (g_ev_recorded) {
    TLRU_CUDA(cudaEventSynchronize(g_ev[2]));
    TLRU_CUDA(cudaEventElapsedTime(&out->k2_ms, g_ev[0], g_ev[1]));
    TLRU_CUDA(cudaEventElapsedTime(&out->k3_ms, g_ev[1], g_ev[2]));
    out->out_ms = 0.0f;
    out->out_launches = g_out.launches;
    if (g_out.launches) TLRU_CUDA(cudaEventElapsedTime(&out->out_ms, g_out.first, g_out.last));
  }
  return TLRU_OK;
}
