// sim.cuh -- per-chain state machine of Alg. 1 used by the K2 kernels.
//
// A chain = one instance (C, D) over one segment [s, s_end) of one trace.
//
// State: one tau-ordered array of entries
//   tau[k]  event index of the conversation's last turn ("Timestamp of Last Turn")
//   X[k]    cached blocks of that conversation (P:117 x_{i,t})
// live in [head, tail).  A request of conversation theta finds its entry by
// binary search on tau == prev (the event index of theta's previous turn),
// tombstones it (X = 0) and appends a fresh entry at `tail` (theta gets the
// newest tau).  Free ("infinitely old") blocks are implied, not
// stored: with D = max(xi - Q_hat, 0), the entries with surplus > 0 always form a
// tau-suffix starting at `fh`; every entry after fh is untouched since its
// insertion, so its surplus is min(X, D); fh's own (possibly partial) surplus is
// the register `frem`.  Phase 1 walks fh forward, Phase 2 walks head forward.
// When tail reaches W the live entries are compacted to the front.
//
// Segment start (exact, no fix-up): the cache content after any request equals
// the top-C blocks of the universe under the static key (non-free?, tau, -pos)
// (pinned by tests/stackdist.py against the oracle).
// So the state at s is rebuilt by walking backwards from s-1 over each
// conversation's last turn before s (next[e'] >= s), granting non-free blocks
// max(L - D, 0) most-recent-first until C is reached; only if the whole prefix
// holds fewer than C non-free blocks are free blocks min(L, D) granted too
// (second walk, most-recent-first).
// Threshold-LRU (D = 0): only admitted histories (L >= T) hold blocks, so the walk grants
// L [L >= T] per conversation (the same top-C argument over the admitted universe).
#pragma once

#include <stdint.h>

#include "common.cuh"

namespace tlru {

// A per-entry surplus that is the chain's constant D (End-Aware and forced-caching T-LRU: the
// surplus at insertion is min(L_after, D) and every read takes min(X, S) with X <= L_after, so
// S = D reads the same): reads give D, writes are dropped -- no shared-memory array.
struct SConstD {
  uint16_t d;
  __device__ __forceinline__ operator uint16_t() const { return d; }
  __device__ __forceinline__ SConstD& operator=(uint16_t) { return *this; }
};

// Lane-interleaved shared-memory state: entry k of lane l at [k * 32 + l]
// (4-byte tau and 2-byte X arrays: conflict-free for any per-lane k).
// NOS: no surplus array (S reads as the constant D, see SConstD).
template <bool NOS>
struct SmemStateT {
  uint32_t* tau;
  uint16_t* X;
  uint16_t* S;  // End-/Length-Aware / Belady chains only: surplus of the entry
  int lane;
  uint16_t D;   // NOS: the constant surplus bound
  __device__ __forceinline__ uint32_t& T(uint32_t k) const { return tau[k * 32u + lane]; }
  __device__ __forceinline__ uint16_t& Xr(uint32_t k) const { return X[k * 32u + lane]; }
  __device__ __forceinline__ decltype(auto) Sr(uint32_t k) const {
    if constexpr (NOS) return SConstD{D};
    else return (S[k * 32u + lane]);
  }
  template <bool WITH_S>
  __device__ __forceinline__ void move(uint32_t d, uint32_t s) const {  // entry s -> entry d
    T(d) = T(s);
    Xr(d) = Xr(s);
    if constexpr (WITH_S && !NOS) Sr(d) = Sr(s);
  }
};
using SmemState = SmemStateT<false>;

// Lanes with a surplus array (End-/Length-Aware, Belady): tau array + interleaved (X, S) halfword
// pairs, entry k of lane l at tau[k * 32 + l] and xs[2 (k * 32 + l)] (X), [... + 1] (S), so moving an
// entry (compaction, Belady's sorted-insert shifts) is two 4-byte copies instead of three.
struct SmemStateXS {
  uint32_t* tau;
  uint16_t* xs;
  int lane;
  __device__ __forceinline__ uint32_t& T(uint32_t k) const { return tau[k * 32u + lane]; }
  __device__ __forceinline__ uint16_t& Xr(uint32_t k) const { return xs[2u * (k * 32u + lane)]; }
  __device__ __forceinline__ uint16_t& Sr(uint32_t k) const { return xs[2u * (k * 32u + lane) + 1u]; }
  template <bool WITH_S>
  __device__ __forceinline__ void move(uint32_t d, uint32_t s) const {
    T(d) = T(s);
    uint32_t* w = reinterpret_cast<uint32_t*>(xs);
    if constexpr (WITH_S) w[d * 32u + lane] = w[s * 32u + lane];
    else Xr(d) = Xr(s);
  }
};

// Packed lane-interleaved state for the no-surplus (NOS) lanes with many entries: one 32-bit word
// per entry, (tau - base) << 12 | X, so a 512-entry lane array takes 64 KB per warp instead of 96
// (three warps per SM instead of two).  Valid while X <= 4095 (X <= L_after <= the trace's
// max_history) and tau - base < 2^20 (base = the chain's first event; the host checks both).
// T(k) / Xr(k) return proxies that read and write their field of the word.
struct PkT {
  uint32_t* w;
  uint32_t base;
  __device__ __forceinline__ operator uint32_t() const { return (*w >> 12) + base; }
  __device__ __forceinline__ const PkT& operator=(uint32_t v) const {
    *w = ((v - base) << 12) | (*w & 0xFFFu);
    return *this;
  }
  __device__ __forceinline__ const PkT& operator=(const PkT& o) const { return *this = static_cast<uint32_t>(o); }
};
struct PkX {
  uint32_t* w;
  __device__ __forceinline__ operator uint16_t() const { return static_cast<uint16_t>(*w & 0xFFFu); }
  __device__ __forceinline__ const PkX& operator=(uint32_t v) const {
    *w = (*w & ~0xFFFu) | (v & 0xFFFu);
    return *this;
  }
  __device__ __forceinline__ const PkX& operator=(const PkX& o) const {
    return *this = static_cast<uint32_t>(static_cast<uint16_t>(o));
  }
};
struct SmemStatePk {
  uint32_t* word;
  int lane;
  uint16_t D;     // the constant surplus bound (NOS)
  uint32_t base;  // tau offset
  __device__ __forceinline__ PkT T(uint32_t k) const { return PkT{word + k * 32u + lane, base}; }
  __device__ __forceinline__ PkX Xr(uint32_t k) const { return PkX{word + k * 32u + lane}; }
  __device__ __forceinline__ SConstD Sr(uint32_t) const { return SConstD{D}; }
  template <bool WITH_S>
  __device__ __forceinline__ void move(uint32_t d, uint32_t s) const {  // tau and X share the word; same base
    word[d * 32u + lane] = word[s * 32u + lane];
  }
};

// Chain-contiguous global-memory state (spill path).
struct GlobalState {
  uint32_t* tau;
  uint16_t* X;
  uint16_t* S;
  __device__ __forceinline__ uint32_t& T(uint32_t k) const { return tau[k]; }
  __device__ __forceinline__ uint16_t& Xr(uint32_t k) const { return X[k]; }
  __device__ __forceinline__ uint16_t& Sr(uint32_t k) const { return S[k]; }
  template <bool WITH_S>
  __device__ __forceinline__ void move(uint32_t d, uint32_t s) const {
    tau[d] = tau[s];
    X[d] = X[s];
    if constexpr (WITH_S) S[d] = S[s];
  }
};

struct ChainRegs {
  uint32_t head, tail, fh, frem;
  uint32_t used, C, D, T, W;  // T: Threshold-LRU admission threshold (0 for LRU / T-LRU)
  uint32_t ev_trim, ev_lru, max_occ;
  // warm-start bookkeeping
  uint32_t r, cum_nf, cum_f, nf_target, free_budget, fh_pos, fh_rem;
  bool walking, overflow;
  // Tail-Optimized Belady chains: blocks still cached by conversations that never return
  // (all free), and the sum of the entries' remaining surplus
  uint32_t dead, fsum;
  // Belady chains: every entry at an index >= p1 has S == 0 (an upper bound on the highest entry
  // with surplus; ~0u = none known), so Phase 1 starts its walk from min(tail, p1)
  uint32_t p1;
};

__device__ __forceinline__ void chain_init(ChainRegs& c, uint32_t C, uint32_t D, uint32_t T, uint32_t W,
                                           bool has_prefix) {
  c.C = C;
  c.D = D;
  c.T = T;
  c.W = W;
  c.head = c.tail = W;
  c.fh = W;
  c.frem = 0;
  c.used = 0;
  c.ev_trim = c.ev_lru = c.max_occ = 0;
  c.r = c.cum_nf = c.cum_f = 0;
  c.nf_target = C;
  c.free_budget = 0;
  c.fh_pos = 0xFFFFFFFFu;
  c.fh_rem = 0;
  c.walking = has_prefix && C > 0;
  c.overflow = false;
  c.dead = c.fsum = 0;
  c.p1 = 0xFFFFFFFFu;
}

// One step of the backward walk: e' is an event before the segment start with
// next[e'] >= s (the last turn of its conversation before s) and L_after = la.
template <class St>
__device__ __forceinline__ void chain_walk_step(ChainRegs& c, const St& st, uint32_t e_prime, uint32_t la) {
  uint32_t nf = (la >= c.T && la > c.D) ? la - c.D : 0u;  // non-free blocks max(L - D, 0), admitted only
  uint32_t f = la < c.D ? la : c.D;        // free blocks min(L, D)
  uint32_t x = min(nf, c.nf_target - c.cum_nf);
  uint32_t y = min(f, c.free_budget - c.cum_f);
  if (x + y > 0) {
    if (c.r == c.W) {
      c.overflow = true;
      c.walking = false;
      return;
    }
    uint32_t k = c.W - 1 - c.r;
    st.T(k) = e_prime;
    st.Xr(k) = static_cast<uint16_t>(x + y);
    if (y > 0) {
      c.fh_pos = k;
      c.fh_rem = y;
    }
    ++c.r;
  }
  c.cum_nf += x;
  c.cum_f += y;
  if (c.cum_nf == c.nf_target && c.cum_f == c.free_budget) c.walking = false;
}

// Called when the walk reached event 0.  Returns true if a second (free-block) walk is needed.
__device__ __forceinline__ bool chain_walk_restart(ChainRegs& c) {
  if (!c.walking || c.overflow) return false;
  // Second walk already done, or LRU (no free blocks): the whole prefix is cached.
  if (c.free_budget != 0 || c.D == 0) {
    c.walking = false;
    return false;
  }
  // Every non-free block of the prefix fits (NF_all = cum_nf < C): grant free blocks too.
  c.nf_target = c.cum_nf;
  c.free_budget = c.C - c.cum_nf;
  c.r = c.cum_nf = c.cum_f = 0;
  c.fh_pos = 0xFFFFFFFFu;
  c.fh_rem = 0;
  return true;
}

__device__ __forceinline__ void chain_walk_finish(ChainRegs& c) {
  c.walking = false;
  c.head = c.W - c.r;
  c.tail = c.W;
  c.used = c.cum_nf + c.cum_f;
  if (c.fh_pos != 0xFFFFFFFFu) {
    c.fh = c.fh_pos;
    c.frem = c.fh_rem;
  } else {
    c.fh = c.tail;
    c.frem = 0;
  }
}

template <bool AWARE = false, class St>
__device__ __forceinline__ bool chain_compact(ChainRegs& c, const St& st) {
  uint32_t j = 0;
  uint32_t new_fh = 0xFFFFFFFFu;
  const bool fh_dead = (c.fh < c.tail) && st.Xr(c.fh) == 0;
  for (uint32_t k = c.head; k < c.tail; ++k) {
    if (k == c.fh) new_fh = j;
    if (st.Xr(k) != 0) {
      if (j != k) st.template move<AWARE>(j, k);
      ++j;
    }
  }
  if (c.fh >= c.tail) {
    new_fh = j;
  } else if (fh_dead) {  // fh was a tombstone: the next live entry is untouched since insertion
    c.frem = (new_fh < j) ? min(static_cast<uint32_t>(st.Xr(new_fh)), AWARE ? uint32_t(st.Sr(new_fh)) : c.D) : 0u;
  }
  c.head = 0;
  c.tail = j;
  c.fh = new_fh;
  return j < c.W;
}

// Alg. 1 for the request at event index e with sim view (prev, J, La).
// Returns b = J - X_theta.  Sets c.overflow if the state is full.
template <class St>
__device__ __forceinline__ uint32_t chain_request(ChainRegs& c, const St& st, uint32_t e, uint32_t prev, uint32_t J,
                                                  uint32_t La) {
  uint32_t x_old = 0;
  if (prev != TLRU_NONE) {
    uint32_t lo = c.head, n = c.tail - c.head;
    while (n > 0) {  // lower_bound of prev in tau[head, tail)
      uint32_t half = n >> 1;
      uint32_t m = lo + half;
      if (st.T(m) < prev) {
        lo = m + 1;
        n -= half + 1;
      } else {
        n = half;
      }
    }
    if (lo < c.tail && st.T(lo) == prev) {
      x_old = st.Xr(lo);
      st.Xr(lo) = 0;
      if (lo == c.fh) c.frem = 0;
    }
  }
  const uint32_t b = J - x_old;
  // Threshold-LRU: a history below the threshold is not cached (L never
  // decreases, so theta had no entry either: x_old = 0)
  if (La < c.T) return b;
  if (c.tail == c.W) {
    if (!chain_compact(c, st)) {
      c.overflow = true;
      return b;
    }
  }
  // Alg. 1 line 1: X_theta <- L_theta (whole history, Reading #7), tau_theta <- now
  st.T(c.tail) = e;
  st.Xr(c.tail) = static_cast<uint16_t>(La);
  if (c.fh == c.tail) c.frem = min(La, c.D);
  ++c.tail;
  c.used += La - x_old;
  if (c.used > c.C) {  // Alg. 1 line 2
    uint32_t over = c.used - c.C;
    // Phase 1: TEL-safe trimming, oldest tau first, theta last
    while (over > 0 && c.fh < c.tail) {
      uint32_t take = min(c.frem, over);
      if (take > 0) {
        st.Xr(c.fh) = static_cast<uint16_t>(st.Xr(c.fh) - take);
        c.frem -= take;
        over -= take;
        c.ev_trim += take;
      }
      if (c.frem == 0) {
        ++c.fh;
        c.frem = (c.fh < c.tail) ? min(static_cast<uint32_t>(st.Xr(c.fh)), c.D) : 0u;
      }
    }
    // Phase 2: LRU, partial, from the least recently used entry
    while (over > 0) {
      uint32_t x = st.Xr(c.head);
      uint32_t take = min(x, over);
      st.Xr(c.head) = static_cast<uint16_t>(x - take);
      over -= take;
      c.ev_lru += take;
      if (x == take) ++c.head;
    }
    c.used = c.C;
  }
  c.max_occ = max(c.max_occ, c.used);
  return b;
}

// End-Aware / Length-Aware T-LRU (Readings #24-#25) on a whole-trace chain.
// `last`: theta's conversation has no later turn -> its blocks are released and its history is
// not cached; otherwise Alg. 1 with the surplus min(La, Dcur) stored per entry (Length-Aware's
// Dcur = max(xi - q_next, 0) differs per turn, so entries with surplus 0 may follow fh; fh is
// the oldest entry whose surplus may be > 0, and every entry after it is untouched since its
// insertion, so its surplus is S).
template <class St>
__device__ __forceinline__ uint32_t chain_request_aware(ChainRegs& c, const St& st, uint32_t e, uint32_t prev,
                                                        uint32_t J, uint32_t La, bool last, uint32_t Dcur,
                                                        bool forced = false) {
  uint32_t x_old = 0;
  if (prev != TLRU_NONE) {
    uint32_t lo = c.head, n = c.tail - c.head;
    while (n > 0) {
      uint32_t half = n >> 1;
      uint32_t m = lo + half;
      if (st.T(m) < prev) {
        lo = m + 1;
        n -= half + 1;
      } else {
        n = half;
      }
    }
    if (lo < c.tail && st.T(lo) == prev) {
      x_old = st.Xr(lo);
      st.Xr(lo) = 0;
      if (lo == c.fh) c.frem = 0;
    }
  }
  const uint32_t b = J - x_old;
  if (last) {  // terminating turn: release, cache nothing
    c.used -= x_old;
    return b;
  }
  if (c.tail == c.W) {
    if (!chain_compact<true>(c, st)) {
      c.overflow = true;
      return b;
    }
  }
  const uint32_t s0 = min(La, Dcur);
  st.T(c.tail) = e;
  st.Xr(c.tail) = static_cast<uint16_t>(La);
  st.Sr(c.tail) = static_cast<uint16_t>(s0);
  if (c.fh == c.tail) c.frem = s0;
  ++c.tail;
  c.used += La - x_old;
  if (c.used > c.C) {
    uint32_t over = c.used - c.C;
    // forced caching (App. C, Reading #28): theta (the tail entry) is skipped by both phases
    const uint32_t lim = forced ? c.tail - 1 : c.tail;
    while (over > 0 && c.fh < lim) {  // Phase 1, oldest surplus first, theta last
      uint32_t take = min(c.frem, over);
      if (take > 0) {
        st.Xr(c.fh) = static_cast<uint16_t>(st.Xr(c.fh) - take);
        c.frem -= take;
        over -= take;
        c.ev_trim += take;
      }
      if (c.frem == 0) {
        ++c.fh;
        c.frem = (c.fh < c.tail) ? min(static_cast<uint32_t>(st.Xr(c.fh)), static_cast<uint32_t>(st.Sr(c.fh))) : 0u;
      }
    }
    while (over > 0 && c.head < lim) {  // Phase 2, LRU
      uint32_t x = st.Xr(c.head);
      uint32_t take = min(x, over);
      st.Xr(c.head) = static_cast<uint16_t>(x - take);
      over -= take;
      c.ev_lru += take;
      if (x == take) ++c.head;
    }
    if (over > 0) {  // forced: theta alone exceeds C -- its tail blocks (free ones first) go
      const uint32_t t = c.tail - 1;
      st.Xr(t) = static_cast<uint16_t>(st.Xr(t) - over);
      if (c.fh == t) c.frem -= min(c.frem, over);
      c.ev_lru += over;
    }
    c.used = c.C;
  }
  c.max_occ = max(c.max_occ, c.used);
  return b;
}

// ---------------------------------------------------------------------------------------------
// Tail-Optimized Belady (Thm 1; Reading #26) on one chain.  State: entries sorted
// ascending by key = the conversation's NEXT arrival (event index) in [head, tail); T = key,
// X = cached blocks, S = blocks still cached above the exact TEL-safe budget (L + q_next - xi)^+
// (S <= X always; Phase 2 runs only once every S is 0).  Every key is a future event and each
// event is the next arrival of one conversation, so theta's old entry (key == e) is the minimum:
// the head.  Conversations that never return hold only free blocks and are evicted first; they
// are aggregated in c.dead (which of them is trimmed is unobservable: they never return).
// Entries fully trimmed by Phase 1 stay as tombstones (X = 0) until their key event or a
// compaction.  A new key goes to its sorted position, shifting the shorter side (head - 1 or
// tail + 1 must be free; else tombstones are compacted; else the chain overflows).
template <class St>
__device__ __forceinline__ bool belady_insert(ChainRegs& c, const St& st, uint32_t key, uint32_t x, uint32_t s,
                                              uint32_t& pos) {
  uint32_t lo = c.head, n = c.tail - c.head;
  while (n > 0) {  // lower_bound of key in T[head, tail)
    const uint32_t half = n >> 1;
    const uint32_t m = lo + half;
    if (st.T(m) < key) {
      lo = m + 1;
      n -= half + 1;
    } else {
      n = half;
    }
  }
  if (c.head == 0 && c.tail == c.W) {  // full: drop tombstones (order kept)
    uint32_t j = 0, npos = 0;
    for (uint32_t k = 0; k < c.tail; ++k) {
      if (k == lo) npos = j;
      if (st.Xr(k) != 0) {
        if (j != k) st.template move<true>(j, k);
        ++j;
      }
    }
    if (lo == c.tail) npos = j;
    if (j == c.W) return false;
    c.tail = j;
    lo = npos;
    c.p1 = 0xFFFFFFFFu;  // indices remapped: no bound known
  }
  const bool down = c.head > 0 && (c.tail == c.W || lo - c.head <= c.tail - lo);
  if (down) {  // shift [head, lo) one slot towards the front
    for (uint32_t k = c.head; k < lo; ++k) st.template move<true>(k - 1, k);
    if (c.p1 <= lo) --c.p1;  // the zero-surplus run [p1, lo) moved down with them
    --c.head;
    --lo;
  } else {  // shift [lo, tail) one slot towards the back
    for (uint32_t k = c.tail; k > lo; --k) st.template move<true>(k, k - 1);
    if (c.p1 != 0xFFFFFFFFu && c.p1 >= lo) ++c.p1;
    ++c.tail;
  }
  if (s > 0 && c.p1 != 0xFFFFFFFFu && c.p1 <= lo) c.p1 = lo + 1;  // the new entry has surplus
  st.T(lo) = key;
  st.Xr(lo) = static_cast<uint16_t>(x);
  st.Sr(lo) = static_cast<uint16_t>(s);
  pos = lo;
  return true;
}

// Request at event e: J, La from the sim view, nx = theta's next arrival (TLRU_NONE: never),
// s0 = min(La, max(xi - q_next, 0)) = La - (La + q_next - xi)^+ (unused when nx is NONE).
// forced (App. C; Reading #29): the post-decision state holds theta's whole history,
// so theta's blocks take part in neither phase; Phase 2 then skips theta's entry (entries before
// it that it empties stay as tombstones), and only if theta alone exceeds C does it lose its tail
// blocks -- its above-budget ones first (they are the tail) -- counted in ev_lru.
template <class St>
__device__ __forceinline__ uint32_t chain_request_belady(ChainRegs& c, const St& st, uint32_t e, uint32_t J,
                                                         uint32_t La, uint32_t nx, uint32_t s0, bool forced = false) {
  uint32_t x_old = 0;
  if (c.head < c.tail && st.T(c.head) == e) {  // theta's entry: the smallest key
    x_old = st.Xr(c.head);
    c.fsum -= st.Sr(c.head);
    ++c.head;
  }
  const uint32_t b = J - x_old;  // job - x
  c.used += La - x_old;          // X_theta <- L_theta (Reading #7)
  uint32_t tpos = 0xFFFFFFFFu;   // theta's entry (forced: excluded from both phases)
  uint32_t tdead = 0;            // forced: theta's never-returning blocks, held apart from dead
  if (nx == TLRU_NONE) {
    if (forced) tdead = La;
    else c.dead += La;           // budget 0: every block free
  } else {
    if (!belady_insert(c, st, nx, La, s0, tpos)) {
      c.overflow = true;
      return b;
    }
    if (!forced) {
      c.fsum += s0;
      tpos = 0xFFFFFFFFu;
    }
  }
  if (c.used > c.C) {
    uint32_t over = c.used - c.C;
    // Phase 1: blocks above the budget, furthest next arrival first (never-returning first)
    const uint32_t kd = min(c.dead, over);
    c.dead -= kd;
    over -= kd;
    c.ev_trim += kd;
    uint32_t j = min(c.tail, c.p1);
    bool walked = false;
    while (over > 0 && c.fsum > 0 && j > c.head) {
      --j;
      walked = true;
      if (j == tpos) continue;
      const uint32_t s = st.Sr(j);
      if (s == 0) continue;
      const uint32_t take = min(s, over);
      st.Sr(j) = static_cast<uint16_t>(s - take);
      st.Xr(j) = static_cast<uint16_t>(st.Xr(j) - take);
      c.fsum -= take;
      over -= take;
      c.ev_trim += take;
    }
    // every entry above the last one visited has S == 0 now (theta's is counted as surplus)
    if (walked) c.p1 = (j == tpos || st.Sr(j) > 0) ? j + 1 : j;
    // Phase 2: furthest-in-future, partial; every S is 0 here (theta's aside)
    if (tpos == 0xFFFFFFFFu) {
      while (over > 0 && c.tail > c.head) {
        const uint32_t x = st.Xr(c.tail - 1);
        const uint32_t take = min(x, over);
        st.Xr(c.tail - 1) = static_cast<uint16_t>(x - take);
        over -= take;
        c.ev_lru += take;
        if (x == take) --c.tail;
      }
    } else {
      for (uint32_t j = c.tail; over > 0 && j > c.head;) {
        --j;
        if (j == tpos) continue;
        const uint32_t x = st.Xr(j);
        const uint32_t take = min(x, over);
        st.Xr(j) = static_cast<uint16_t>(x - take);
        over -= take;
        c.ev_lru += take;
      }
    }
    if (over > 0) {  // forced: theta alone exceeds C -- its tail blocks go, above-budget first
      if (tpos == 0xFFFFFFFFu) {
        tdead -= over;
      } else {
        const uint32_t s = st.Sr(tpos);
        st.Sr(tpos) = static_cast<uint16_t>(s - min(s, over));
        st.Xr(tpos) = static_cast<uint16_t>(st.Xr(tpos) - over);
      }
      c.ev_lru += over;
    }
    while (c.tail > c.head && st.Xr(c.tail - 1) == 0) --c.tail;
    c.used = c.C;
  }
  if (forced) {  // theta rejoins the state
    if (tpos != 0xFFFFFFFFu) {
      c.fsum += st.Sr(tpos);
      if (c.p1 != 0xFFFFFFFFu && c.p1 <= tpos) c.p1 = tpos + 1;
    }
    c.dead += tdead;
  }
  c.max_occ = max(c.max_occ, c.used);
  return b;
}

}  // namespace tlru
