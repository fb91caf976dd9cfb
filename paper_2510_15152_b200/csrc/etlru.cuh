// etlru.cuh -- Expected-Tail-Optimized LRU (Def. 1; greedy Alg. 2, P:603-650;
// Reading #27) on the GPU: one warp per (instance, time segment), the 32 lanes cooperate on every
// request ("one instance per warp ... warp-level min/scan primitives").  Included by
// sim.cu after its TraceDev / AccDev definitions.
//
// Ranking criterion.  v_i = lambda_i P(L_i + Q_i - xi >= X_i) with the belief
// lambda_i = exp(-mu (t - time_i)) (homogeneous lambda-bar) orders like the static
// score  s_i = mu * time_i + ln P(Q >= X_i - L_i + xi)  (t is common to every i at a decision),
// evaluated as __dadd_rn(__dmul_rn(double(ticks_i), mu_tick), ln_surv[k]) with ln_surv[k] = 0
// for k <= 0 and -inf for k > K.  Evict the minimum of (s, tau), tau = event index of the last
// turn (older first on ties); a conversation's blocks go tail first.
//
// State (W dense unordered slots, 24 B each): key = the order-preserving u64 of the score of the
// slot's last cached block, base = mu * time (double), tau u32, X u16, L u16 (history at the last
// turn).  A request finds theta's slot by a strided ballot over tau == prev and swap-removes it,
// then appends the new slot; while the cache overflows, every lane scans its slots for its best
// and second-best (key, tau), three redux.sync steps give the warp minimum and three more the
// runner-up, and the minimum conversation loses the prefix of its tail blocks that still rank
// below the runner-up, tested 32 blocks at a time by the lanes with one ballot (Alg. 2's
// one-block-at-a-time re-scoring, in bulk).
//
// Time partitioning (verified, as the End-/Length-Aware chains in sim.cu): segment k of an
// instance starts `burn` events early from an empty cache and saves its canonical state (live
// (tau, X) sorted by tau, used) at the segment start (G_k) and end (F_k).  The state determines
// the rest of the run, so segment k is exact iff k = 0 or G_k == F_{k-1}; etlru_fix_kernel re-runs
// every other segment (and any that outgrew its W slots) from the exact F_{k-1} with global-memory
// state, in order, so every output is exact.
#pragma once

namespace tlru {

struct EtItem {  // one ET-LRU instance
  uint32_t inst, trace, C, xi;
  uint64_t boff;
  uint32_t forced, pad;  // forced caching (App. C; Reading #30)
};

struct EtSeg {  // one warp of the segment kernel
  uint32_t item, seg;
};

struct EtModel {
  const double* ln_surv;  // [K + 1] (global)
  uint32_t K;
  double mu_tick;
};

struct EtSegs {  // time partitioning of the ET-LRU chains
  uint32_t seg_len, burn, nseg_max, wsnap;
  uint32_t* snap;            // [item][seg][2][2 + 2 wsnap]: G_k, F_k = {n, used, tau[wsnap], X[wsnap]}
  unsigned long long* segc;  // [item][seg][2]: blocks evicted with P = 0 / the others
  uint32_t* segm;            // [item][seg]: max occupancy
  uint32_t* ovf;             // [item][seg]: 1 = the segment outgrew its slots
};

constexpr int kEtTab = 256;  // table entries kept in shared memory

__host__ __device__ __forceinline__ size_t et_snap_words(uint32_t wsnap) { return 2 + 2 * size_t(wsnap); }

// Order-preserving map of a non-NaN double to u64 (IEEE < becomes unsigned <; scores are never
// -0.0: the model normalises mu and the table, and base >= +0 with round-to-nearest adds).
__device__ __forceinline__ uint64_t et_ord(double v) {
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

struct EtCtx {
  const double* tab_s;  // shared copy of ln_surv[0 .. min(K, kEtTab - 1)]
  const double* tab_g;
  uint32_t K;
  double mu;
  __device__ __forceinline__ double lg(int64_t k) const {
    if (k <= 0) return 0.0;
    if (k > static_cast<int64_t>(K)) return -__longlong_as_double(0x7FF0000000000000ll);  // -inf
    return k < kEtTab ? tab_s[k] : __ldg(tab_g + k);
  }
};

// Warp-wide minimum of (key, tau) (lexicographic; tau unique per slot): three redux steps.
__device__ __forceinline__ void et_warp_min(uint64_t k, uint32_t t, uint64_t& km, uint32_t& tm) {
  const uint32_t hi = __reduce_min_sync(0xFFFFFFFFu, static_cast<uint32_t>(k >> 32));
  const uint32_t lo =
      __reduce_min_sync(0xFFFFFFFFu, static_cast<uint32_t>(k >> 32) == hi ? static_cast<uint32_t>(k) : 0xFFFFFFFFu);
  km = (uint64_t(hi) << 32) | lo;
  tm = __reduce_min_sync(0xFFFFFFFFu, k == km ? t : 0xFFFFFFFFu);
}

struct EtState {
  uint64_t* key;
  double* base;
  uint32_t* tau;
  uint16_t* X;
  uint16_t* L;
  uint32_t cap, n, used, max_occ, C;
  int64_t xi;
  unsigned long long ev_free, ev_other;
  bool overflow;
  bool forced;  // theta is not a candidate while its turn is served (Y_theta = L, App. C)
  // Incremental candidates (inc, the large slot classes): every lane keeps the two smallest
  // (key, tau) of ITS slots (slot s belongs to lane s % 32) -- bk1/bt1 at slot bs1, then bk2/bt2 --
  // so an eviction round needs no scan: only the lanes whose slots changed recompute theirs,
  // the whole warp reading one such lane's <= 32 slots at once (et_rescan).
  bool inc;
  uint64_t bk1, bk2;
  uint32_t bt1, bt2, bs1;

  __device__ __forceinline__ void carve(unsigned char* pool, uint32_t c) {
    cap = c;
    key = reinterpret_cast<uint64_t*>(pool);
    base = reinterpret_cast<double*>(key + c);
    tau = reinterpret_cast<uint32_t*>(base + c);
    X = reinterpret_cast<uint16_t*>(tau + c);
    L = X + c;
  }
  __device__ __forceinline__ void move_slot(uint32_t dst, uint32_t src) {
    key[dst] = key[src];
    base[dst] = base[src];
    tau[dst] = tau[src];
    X[dst] = X[src];
    L[dst] = L[src];
  }
};

#ifndef TLRU_ET_INC_MIN
#define TLRU_ET_INC_MIN 256u
#endif
constexpr uint32_t kEtIncMin = TLRU_ET_INC_MIN;  // slot classes from this size keep incremental candidates

__device__ __forceinline__ bool et_less(uint64_t k, uint32_t t, uint64_t K, uint32_t T) {
  return k < K || (k == K && t < T);
}

// Lane o's two smallest (key, tau) over its slots o, o + 32, ... (< S.n, != ex), read by the whole
// warp (one slot per lane while S.n <= 1024) and reduced with the same redux steps as a round.
__device__ __forceinline__ void et_rescan(EtState& S, uint32_t o, uint32_t ex) {
  const uint32_t lane = threadIdx.x & 31;
  uint64_t a1 = ~0ull, a2 = ~0ull;
  uint32_t u1 = 0xFFFFFFFFu, u2 = 0xFFFFFFFFu, s1 = 0;
  for (uint32_t s = o + 32u * lane; s < S.n; s += 1024u) {
    if (s == ex) continue;
    const uint64_t k = S.key[s];
    const uint32_t t = S.tau[s];
    if (et_less(k, t, a1, u1)) {
      a2 = a1;
      u2 = u1;
      a1 = k;
      u1 = t;
      s1 = s;
    } else if (et_less(k, t, a2, u2)) {
      a2 = k;
      u2 = t;
    }
  }
  uint64_t m1, m2;
  uint32_t n1, n2;
  et_warp_min(a1, u1, m1, n1);
  const int wl = __ffs(__ballot_sync(0xFFFFFFFFu, a1 == m1 && u1 == n1)) - 1;
  const uint32_t ms = __shfl_sync(0xFFFFFFFFu, s1, wl);
  if (static_cast<int>(lane) == wl) {
    a1 = a2;
    u1 = u2;
  }
  et_warp_min(a1, u1, m2, n2);
  if (lane == o) {
    S.bk1 = m1;
    S.bt1 = n1;
    S.bs1 = ms;
    S.bk2 = m2;
    S.bt2 = n2;
  }
}

// Slot s (key k, tau t) joins its owner lane's candidates (a new slot; keys only grow otherwise).
__device__ __forceinline__ void et_offer(EtState& S, uint32_t s, uint64_t k, uint32_t t) {
  if ((threadIdx.x & 31) != (s & 31u)) return;
  if (et_less(k, t, S.bk1, S.bt1)) {
    S.bk2 = S.bk1;
    S.bt2 = S.bt1;
    S.bk1 = k;
    S.bt1 = t;
    S.bs1 = s;
  } else if (et_less(k, t, S.bk2, S.bt2)) {
    S.bk2 = k;
    S.bt2 = t;
  }
}

// Every lane's candidates from scratch (after a snapshot load).
__device__ __forceinline__ void et_cand_init(EtState& S) {
  S.bk1 = S.bk2 = ~0ull;
  S.bt1 = S.bt2 = 0xFFFFFFFFu;
  S.bs1 = 0;
  if (!S.inc) return;
  for (uint32_t s = threadIdx.x & 31; s < S.n; s += 32) et_offer(S, s, S.key[s], S.tau[s]);
}

// One request (event e, sim view ev, time tk).  Returns b = J - X_theta (valid in every lane).
__device__ __forceinline__ uint32_t et_request(EtState& S, const EtCtx& m, uint32_t e, uint64_t ev, uint64_t tk) {
  const int lane = threadIdx.x & 31;
  const uint32_t prev = sim_prev(ev), J = sim_J(ev), La = sim_La(ev);
  // ---- theta's slot (tau == prev): strided ballot, then swap-remove
  uint32_t x_old = 0;
  if (prev != TLRU_NONE) {
    int hit = -1;
#pragma unroll 4
    for (uint32_t s = lane; s < S.n; s += 32)
      if (S.tau[s] == prev) hit = static_cast<int>(s);
    const unsigned bal = __ballot_sync(0xFFFFFFFFu, hit >= 0);
    if (bal) {
      const uint32_t p = static_cast<uint32_t>(__shfl_sync(0xFFFFFFFFu, hit, __ffs(bal) - 1));
      x_old = S.X[p];
      __syncwarp();
      const uint32_t last = S.n - 1;
      if (lane == 0 && p != last) S.move_slot(p, last);
      --S.n;
      __syncwarp();
      if (S.inc) {  // slot p now holds the former last slot
        et_rescan(S, p & 31u, 0xFFFFFFFFu);
        if ((last & 31u) != (p & 31u)) et_rescan(S, last & 31u, 0xFFFFFFFFu);
      }
    }
  }
  const uint32_t b = J - x_old;  // job - x
  // ---- Alg. 2 lines 2-4: L_theta += Q + A, X_theta <- L_theta, lambda_theta <- lambda-bar
  if (S.n == S.cap) {
    S.overflow = true;
    return b;
  }
  {
    const double bs = __dmul_rn(static_cast<double>(tk), m.mu);
    const uint64_t kt = et_ord(__dadd_rn(bs, m.lg(S.xi)));  // X = L: k = xi
    if (lane == 0) {
      S.base[S.n] = bs;
      S.key[S.n] = kt;
      S.tau[S.n] = e;
      S.X[S.n] = static_cast<uint16_t>(La);
      S.L[S.n] = static_cast<uint16_t>(La);
    }
    if (S.inc && !S.forced) et_offer(S, S.n, kt, e);  // forced: theta joins after its turn
  }
  ++S.n;
  S.used += La - x_old;
  uint32_t th = S.forced ? S.n - 1 : 0xFFFFFFFFu;  // forced: theta's slot, excluded below
  __syncwarp();
  // ---- lines 8-12: evict the overflow, minimum ranking criterion first
  while (S.used > S.C) {
    const uint32_t over = S.used - S.C;
    uint64_t k1 = ~0ull, k2 = ~0ull;
    uint32_t t1 = 0xFFFFFFFFu, t2 = 0xFFFFFFFFu, s1 = 0;
    if (S.inc) {
      k1 = S.bk1;
      t1 = S.bt1;
      s1 = S.bs1;
      k2 = S.bk2;
      t2 = S.bt2;
    }
#pragma unroll 4
    for (uint32_t s = lane; !S.inc && s < S.n; s += 32) {
      if (s == th) continue;
      const uint64_t ks = S.key[s];
      const uint32_t ts = S.tau[s];
      if (ks < k1 || (ks == k1 && ts < t1)) {
        k2 = k1;
        t2 = t1;
        k1 = ks;
        t1 = ts;
        s1 = s;
      } else if (ks < k2 || (ks == k2 && ts < t2)) {
        k2 = ks;
        t2 = ts;
      }
    }
    uint64_t kmin, krun;
    uint32_t tmin, trun;
    et_warp_min(k1, t1, kmin, tmin);
    if (kmin == ~0ull) {  // forced: only theta is left and it alone exceeds C -- it loses the excess
      __syncwarp();
      if (lane == 0) {
        const uint32_t xn = S.X[th] - over;
        S.X[th] = static_cast<uint16_t>(xn);
        S.key[th] = et_ord(__dadd_rn(S.base[th], m.lg(int64_t(xn) - int64_t(S.L[th]) + S.xi)));
      }
      S.ev_other += over;
      S.used = S.C;
      __syncwarp();
      break;
    }
    const int wl = __ffs(__ballot_sync(0xFFFFFFFFu, k1 == kmin && t1 == tmin)) - 1;
    const uint32_t j = __shfl_sync(0xFFFFFFFFu, s1, wl);
    if (lane == wl) {  // the runner-up: the winner lane's second or any other lane's best
      k1 = k2;
      t1 = t2;
    }
    et_warp_min(k1, t1, krun, trun);
    // j loses tail blocks while they still rank below the runner-up: lane l tests block X_j - l
    const uint32_t xj = S.X[j];
    const int64_t Lj = S.L[j];
    const double bj = S.base[j];
    const int64_t x = int64_t(xj) - lane;
    bool ok = false, fr = false;
    if (static_cast<uint32_t>(lane) < over && x >= 1) {
      const double g = m.lg(x - Lj + S.xi);
      const uint64_t kv = et_ord(__dadd_rn(bj, g));
      ok = kv < krun || (kv == krun && tmin < trun);
      fr = __double_as_longlong(g) == static_cast<long long>(0xFFF0000000000000ull);  // -inf: TEL-safe
    }
    const unsigned okb = __ballot_sync(0xFFFFFFFFu, ok);
    const uint32_t cnt = okb == 0xFFFFFFFFu ? 32u : static_cast<uint32_t>(__ffs(~okb) - 1);  // a prefix (>= 1)
    const unsigned pm = cnt == 32 ? 0xFFFFFFFFu : ((1u << cnt) - 1u);
    const uint32_t nfree = __popc(__ballot_sync(0xFFFFFFFFu, fr) & pm);
    S.ev_free += nfree;
    S.ev_other += cnt - nfree;
    S.used -= cnt;
    const uint32_t xn = xj - cnt;
    __syncwarp();
    const uint32_t last = S.n - 1;
    if (xn == 0 && j != last && th == last) th = j;  // theta moves into j's slot
    if (lane == 0) {
      if (xn == 0) {
        if (j != last) S.move_slot(j, last);
      } else {
        S.X[j] = static_cast<uint16_t>(xn);
        S.key[j] = et_ord(__dadd_rn(bj, m.lg(int64_t(xn) - Lj + S.xi)));
      }
    }
    if (xn == 0) --S.n;
    __syncwarp();
    if (S.inc) {  // j's key grew or j now holds the former last slot
      et_rescan(S, j & 31u, th);
      if (xn == 0 && (last & 31u) != (j & 31u)) et_rescan(S, last & 31u, th);
    }
  }
  if (S.inc && S.forced && th != 0xFFFFFFFFu) {  // theta is a candidate again after its turn
    __syncwarp();
    et_offer(S, th, S.key[th], S.tau[th]);
  }
  S.max_occ = max(S.max_occ, S.used);
  return b;
}

// Requests [from, to) of the trace; b written to bout (+ boff) unless bout is NULL.
__device__ __forceinline__ void et_run(EtState& S, const EtCtx& m, const TraceDev& tr, uint32_t from, uint32_t to,
                                       uint16_t* bout) {
  const int lane = threadIdx.x & 31;
  for (uint32_t t0 = from; t0 < to && !S.overflow; t0 += 32) {
    const uint32_t nk = min(32u, to - t0);
    uint64_t ev_l = 0, tk_l = 0;
    if (static_cast<uint32_t>(lane) < nk) {
      ev_l = __ldg(tr.sim + t0 + lane);
      tk_l = __ldg(tr.ticks + t0 + lane);
    }
    uint32_t b_mine = 0;
    for (uint32_t k = 0; k < nk && !S.overflow; ++k) {
      const uint64_t ev = __shfl_sync(0xFFFFFFFFu, ev_l, k);
      const uint64_t tk = __shfl_sync(0xFFFFFFFFu, tk_l, k);
      const uint32_t b = et_request(S, m, t0 + k, ev, tk);
      if (lane == static_cast<int>(k)) b_mine = b;
    }
    if (bout && !S.overflow && static_cast<uint32_t>(lane) < nk) bout[t0 + lane] = static_cast<uint16_t>(b_mine);
  }
}

// Canonical state: live (tau, X) sorted by tau (rank by counting), header {n, used}.
__device__ void et_snap_write(uint32_t* out, uint32_t wsnap, const EtState& S) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    out[0] = S.n <= wsnap ? S.n : 0xFFFFFFFFu;  // too large to save: never matches, the fix-up re-runs it
    out[1] = S.used;
  }
  if (S.n > wsnap) return;
  for (uint32_t s = lane; s < S.n; s += 32) {
    const uint32_t t = S.tau[s];
    uint32_t r = 0;
    for (uint32_t u = 0; u < S.n; ++u) r += S.tau[u] < t;
    out[2 + r] = t;
    out[2 + wsnap + r] = S.X[s];
  }
}

__device__ bool et_snap_equal(const uint32_t* a, const uint32_t* b, uint32_t wsnap) {
  if (a[0] == 0xFFFFFFFFu || a[0] != b[0] || a[1] != b[1]) return false;
  bool eq = true;
  for (uint32_t i = threadIdx.x & 31; i < a[0]; i += 32)
    eq = eq && a[2 + i] == b[2 + i] && a[2 + wsnap + i] == b[2 + wsnap + i];
  return __all_sync(0xFFFFFFFFu, eq);
}

// Rebuild a state from a snapshot: L and base follow from tau (the history at that turn, its time).
__device__ void et_snap_load(EtState& S, const EtCtx& m, const TraceDev& tr, const uint32_t* in, uint32_t wsnap) {
  const uint32_t n = in[0];
  for (uint32_t i = threadIdx.x & 31; i < n; i += 32) {
    const uint32_t t = in[2 + i];
    const uint32_t x = in[2 + wsnap + i];
    const uint32_t La = sim_La(tr.sim[t]);
    const double bs = __dmul_rn(static_cast<double>(tr.ticks[t]), m.mu);
    S.tau[i] = t;
    S.X[i] = static_cast<uint16_t>(x);
    S.L[i] = static_cast<uint16_t>(La);
    S.base[i] = bs;
    S.key[i] = et_ord(__dadd_rn(bs, m.lg(int64_t(x) - int64_t(La) + S.xi)));
  }
  S.n = n;
  S.used = in[1];
  __syncwarp();
  et_cand_init(S);
}

__device__ __forceinline__ void et_ctx_init(EtCtx& c, const EtModel& m, double* tab_s) {
  const uint32_t nt = min(m.K + 1, static_cast<uint32_t>(kEtTab));
  for (uint32_t k = threadIdx.x & 31; k < nt; k += 32) tab_s[k] = m.ln_surv[k];
  __syncwarp();
  c.tab_s = tab_s;
  c.tab_g = m.ln_surv;
  c.K = m.K;
  c.mu = m.mu_tick;
}

__device__ __forceinline__ void et_state_init(EtState& S, uint32_t C, uint32_t xi, bool forced) {
  S.n = S.used = S.max_occ = 0;
  S.C = C;
  S.xi = xi;
  S.ev_free = S.ev_other = 0;
  S.overflow = false;
  S.forced = forced;
  S.inc = S.cap >= kEtIncMin;
  et_cand_init(S);
}

// One warp per (instance, segment); W slots in shared memory after the table copy.
template <int W>
__global__ void __launch_bounds__(32) etlru_seg_kernel(const EtSeg* __restrict__ segs, const EtItem* __restrict__ items,
                                                       const TraceDev* __restrict__ traces, EtModel mdl, EtSegs sg,
                                                       uint16_t* __restrict__ bout) {
  extern __shared__ __align__(16) unsigned char smem[];
  const EtSeg sj = segs[blockIdx.x];
  const EtItem it = items[sj.item];
  const TraceDev tr = traces[it.trace];
  EtCtx m;
  et_ctx_init(m, mdl, reinterpret_cast<double*>(smem));
  EtState S;
  S.carve(smem + kEtTab * sizeof(double), W);
  et_state_init(S, it.C, it.xi, it.forced != 0);
  const uint32_t s = sj.seg * sg.seg_len;
  const uint32_t s_end = static_cast<uint32_t>(min(uint64_t(s) + sg.seg_len, tr.E));
  const uint32_t s0 = s > sg.burn ? s - sg.burn : 0u;
  const size_t sw = et_snap_words(sg.wsnap);
  const size_t slot = size_t(sj.item) * sg.nseg_max + sj.seg;
  uint32_t* G = sg.snap + slot * 2 * sw;
  et_run(S, m, tr, s0, s, nullptr);  // burn-in from an empty cache (no output)
  if (sj.seg > 0 && !S.overflow) et_snap_write(G, sg.wsnap, S);
  S.ev_free = S.ev_other = 0;
  S.max_occ = 0;
  et_run(S, m, tr, s, s_end, bout + it.boff);
  if ((threadIdx.x & 31) == 0) {
    sg.segc[2 * slot] = S.ev_free;
    sg.segc[2 * slot + 1] = S.ev_other;
    sg.segm[slot] = S.max_occ;
    sg.ovf[slot] = S.overflow ? 1u : 0u;
  }
  if (!S.overflow) et_snap_write(G + sw, sg.wsnap, S);
}

// Fix-up: one warp per instance walks its segments in order; a segment that overflowed or whose
// start state G_k differs from the exact end state F_{k-1} is re-run from F_{k-1} (empty for
// k = 0) with global-memory state (Wg slots), which also rewrites F_k.  Then the segment counters
// are summed into the instance's accumulators.
__global__ void __launch_bounds__(32) etlru_fix_kernel(const EtItem* __restrict__ items, uint32_t nitems,
                                                       const TraceDev* __restrict__ traces, EtModel mdl, EtSegs sg,
                                                       uint16_t* __restrict__ bout, AccDev* acc,
                                                       unsigned char* gpool, uint32_t Wg, unsigned int* nfixed,
                                                       unsigned int* nfail) {
  __shared__ double tab_s[kEtTab];
  const uint32_t i = blockIdx.x;
  if (i >= nitems) return;
  const int lane = threadIdx.x & 31;
  const EtItem it = items[i];
  const TraceDev tr = traces[it.trace];
  EtCtx m;
  et_ctx_init(m, mdl, tab_s);
  EtState S;
  S.carve(gpool + size_t(i) * Wg * 24, Wg);
  et_state_init(S, it.C, it.xi, it.forced != 0);
  const uint32_t nseg = static_cast<uint32_t>((tr.E + sg.seg_len - 1) / sg.seg_len);
  const size_t sw = et_snap_words(sg.wsnap);
  bool carry = false;  // S holds the exact state at the end of segment k - 1
  for (uint32_t k = 0; k < nseg; ++k) {
    const size_t slot = size_t(i) * sg.nseg_max + k;
    uint32_t* G = sg.snap + slot * 2 * sw;
    const uint32_t* Fp = k > 0 ? sg.snap + (slot - 1) * 2 * sw + sw : nullptr;
    if (!sg.ovf[slot] && (k == 0 || et_snap_equal(G, Fp, sg.wsnap))) {
      carry = false;
      continue;
    }
    if (!carry) {
      et_state_init(S, it.C, it.xi, it.forced != 0);
      if (k > 0) {
        if (Fp[0] == 0xFFFFFFFFu) {  // the previous end state was too large to save
          if (lane == 0) atomicAdd(nfail, 1u);
          return;
        }
        et_snap_load(S, m, tr, Fp, sg.wsnap);
      }
    }
    S.ev_free = S.ev_other = 0;
    S.max_occ = 0;
    const uint32_t s = k * sg.seg_len;
    const uint32_t s_end = static_cast<uint32_t>(min(uint64_t(s) + sg.seg_len, tr.E));
    et_run(S, m, tr, s, s_end, bout + it.boff);
    if (S.overflow) {
      if (lane == 0) atomicAdd(nfail, 1u);
      return;
    }
    if (lane == 0) {
      sg.segc[2 * slot] = S.ev_free;
      sg.segc[2 * slot + 1] = S.ev_other;
      sg.segm[slot] = S.max_occ;
      sg.ovf[slot] = 0;
      atomicAdd(nfixed, 1u);
    }
    et_snap_write(G + sw, sg.wsnap, S);
    __syncwarp();
    carry = true;
  }
  if (lane == 0) {
    unsigned long long ef = 0, eo = 0;
    uint32_t mo = 0;
    for (uint32_t k = 0; k < nseg; ++k) {
      const size_t slot = size_t(i) * sg.nseg_max + k;
      ef += sg.segc[2 * slot];
      eo += sg.segc[2 * slot + 1];
      mo = max(mo, sg.segm[slot]);
    }
    acc[it.inst].ev_trim = ef;
    acc[it.inst].ev_lru = eo;
    acc[it.inst].max_occ = mo;
  }
}

}  // namespace tlru
