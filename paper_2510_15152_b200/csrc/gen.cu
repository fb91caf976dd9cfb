// gen.cu -- K1: synthetic traces from the paper's stochastic conversation model
// (Sec. 5; App. E recipe P:724) and the upload path for host traces.
//
//   count   : one thread per conversation: birth gap, death / turn clocks -> turn count;
//             the few conversations that could reach the context cap L_max are queued
//             and recounted exactly with their lengths (count_fix)
//   scan    : birth ticks = inclusive scan of Exp(lambda_conv) gaps (integer, so
//             order-independent); per-conversation event offsets = exclusive scan
//   slot/draw: one thread per event slot draws its turn gap and prompt / response lengths
//   emit    : one thread per conversation: prefix sums of gaps (time) and lengths (J, L_after)
//   sort    : stable radix sort on the 64-bit arrival tick; conversation order is
//             (conv, turn), so ties come out ordered by (conv, turn) (Reading #9)
//   link    : scatter to time order, prev/next links and the 8-byte sim view
#include <cub/cub.cuh>

#include <algorithm>

#include "common.cuh"
#include "rng.cuh"

namespace tlru {

struct GenDev {  // per-trace constants, by value to the kernels
  uint64_t seed;
  uint32_t N, B, Lmax, max_turns;
  uint32_t safe_turns;  // a conversation with at most this many turns can never hit L_max
  double us_birth, us_turn, us_death;  // 1e6 / rate
  double p_mean, p_sigma, r_mean, r_sigma;
  uint32_t p_lo, p_hi, r_lo, r_hi;
};

// Exact turn count of conversation c: death/turn clocks plus the context-window rule,
// which needs the lengths.  Used only for conversations that may reach L_max.
__device__ __forceinline__ uint32_t conv_count_exact(const GenDev& g, uint32_t c) {
  const U64x4 d00 = turn_draw(g.seed, c, 0, 0);
  const uint64_t life = exp_ticks_of(d00.v[3], g.us_death);  // Exp(mu) lifetime
  const double p_mu = lognormal_mu(g.p_mean, g.p_sigma), r_mu = lognormal_mu(g.r_mean, g.r_sigma);
  uint64_t elapsed = 0;
  uint32_t L = 0, n = 0;
  for (uint32_t k = 0; k < g.max_turns; ++k) {
    const U64x4 d = k ? turn_draw(g.seed, c, k, 0) : d00;
    if (k > 0) {  // Poisson(lambda_turn) turns while alive
      elapsed += exp_ticks_of(d.v[0], g.us_turn);
      if (elapsed >= life) break;
    }
    double zp, zr;
    polar_pair(g.seed, c, k, d, zp, zr);
    const uint32_t pt = lognormal_tokens(zp, p_mu, g.p_sigma, g.p_lo, g.p_hi);
    const uint32_t rt = lognormal_tokens(zr, r_mu, g.r_sigma, g.r_lo, g.r_hi);
    uint32_t q = (pt + g.B - 1) / g.B;
    if (q < 1) q = 1;
    const uint32_t a = (rt + g.B - 1) / g.B;
    if (uint64_t(L) + q + a > g.Lmax) break;  // context-window end
    L += q + a;
    ++n;
  }
  return n;
}

// Turns allowed by the death clock and max_turns alone (no lengths drawn).
__device__ __forceinline__ uint32_t clock_turns(const GenDev& g, uint32_t c, uint64_t life, uint64_t* last_elapsed) {
  uint64_t elapsed = 0, kept = 0;
  uint32_t n = 1;
  for (uint32_t k = 1; k < g.max_turns; ++k) {
    elapsed += exp_ticks_of(turn_draw(g.seed, c, k, 0).v[0], g.us_turn);
    if (elapsed >= life) break;
    kept = elapsed;
    ++n;
  }
  *last_elapsed = kept;
  return n;
}

// Births + death/turn clocks only.  Conversations long enough to possibly reach L_max are
// queued for an exact replay with lengths (gen_count_fix_kernel), so no warp diverges into
// the lognormal sampling here.
__global__ void gen_count_kernel(GenDev g, uint64_t* gaps, uint32_t* counts, unsigned long long* max_elapsed,
                                 uint32_t* queue, uint32_t* nqueue) {
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t Npad = (g.N + 31u) & ~31u;  // whole warps stay in the loop for the warp-aggregated atomics
  unsigned long long mel = 0;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < Npad; c += stride) {
    uint32_t n = 0;
    if (c < g.N) {
      const U64x4 d00 = turn_draw(g.seed, c, 0, 0);
      gaps[c] = exp_ticks_of(d00.v[0], g.us_birth);  // Poisson(lambda_conv) births
      uint64_t el;
      n = clock_turns(g, c, exp_ticks_of(d00.v[3], g.us_death), &el);  // Exp(mu) lifetime
      counts[c] = n;
      mel = el > mel ? el : mel;
    }
    const bool q = c < g.N && n > g.safe_turns;
    const uint32_t slot = warp_push(nqueue, q);
    if (q) queue[slot] = c;
  }
  warp_atomic_max_u64(max_elapsed, mel);
  if (blockIdx.x == 0 && threadIdx.x == 0) counts[g.N] = 0;
}

__global__ void gen_count_fix_kernel(GenDev g, const uint32_t* queue, const uint32_t* nqueue, uint32_t* counts) {
  const uint32_t nq = *nqueue;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += gridDim.x * blockDim.x) {
    const uint32_t c = queue[i];
    counts[c] = conv_count_exact(g, c);
  }
}

// One thread per conversation: label its event slots with (conversation, turn).
__global__ void gen_slot_kernel(GenDev g, const uint32_t* off, uint32_t* cid, uint16_t* turn) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < g.N; c += gridDim.x * blockDim.x) {
    const uint32_t b = off[c], n = off[c + 1] - b;
    for (uint32_t k = 0; k < n; ++k) {
      cid[b + k] = c;
      turn[b + k] = static_cast<uint16_t>(k);
    }
  }
}

// One thread per event slot: the turn's random draws: gap to the previous turn
// (turn > 0) and the prompt / response lengths in blocks (Reading #16).
__global__ void gen_draw_kernel(GenDev g, uint32_t E, const uint32_t* cid, const uint16_t* turn, uint64_t* gapt,
                                uint16_t* q16, uint16_t* a16) {
  const double p_mu = lognormal_mu(g.p_mean, g.p_sigma), r_mu = lognormal_mu(g.r_mean, g.r_sigma);
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < E; j += gridDim.x * blockDim.x) {
    const uint32_t c = cid[j], k = turn[j];
    const U64x4 d = turn_draw(g.seed, c, k, 0);  // one draw: the gap and the first polar pair
    gapt[j] = k ? exp_ticks_of(d.v[0], g.us_turn) : 0ull;
    double zp, zr;
    polar_pair(g.seed, c, k, d, zp, zr);
    const uint32_t pt = lognormal_tokens(zp, p_mu, g.p_sigma, g.p_lo, g.p_hi);
    const uint32_t rt = lognormal_tokens(zr, r_mu, g.r_sigma, g.r_lo, g.r_hi);
    uint32_t q = (pt + g.B - 1) / g.B;
    if (q < 1) q = 1;
    q16[j] = static_cast<uint16_t>(q);
    a16[j] = static_cast<uint16_t>((rt + g.B - 1) / g.B);
  }
}

// One thread per conversation, no random draws: arrival ticks and history prefix sums over its
// slots; J = L_before + q, L_after = J + a.  Slots are allocated from the turn
// clocks alone, so a turn that would push the history past L_max ends the conversation here
// (context-window end): it and the later slots get the sentinel key and sort past the end.
__global__ void gen_emit_kernel(GenDev g, const uint64_t* birth, const uint32_t* off, const uint64_t* gapt,
                                const uint16_t* q16, const uint16_t* a16, uint64_t sentinel, uint64_t* key,
                                uint32_t* val, uint16_t* J16, uint16_t* La16, uint8_t* last8, uint32_t* max_L,
                                uint32_t* nconv, uint32_t* nvalid, unsigned long long* universe) {
  uint32_t maxL = 0, nc = 0, nv = 0;
  unsigned long long U = 0;  // sum of final histories (the universe)
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < g.N; c += gridDim.x * blockDim.x) {
    const uint32_t b = off[c], n = off[c + 1] - b;
    uint64_t t = birth[c];
    uint32_t L = 0, k = 0;
    for (; k < n; ++k) {
      const uint32_t j = b + k;
      const uint32_t q = q16[j], a = a16[j];
      if (L + q + a > g.Lmax) break;  // context-window end
      t += gapt[j];
      key[j] = t;
      val[j] = j;
      L += q;
      J16[j] = static_cast<uint16_t>(L);
      L += a;
      La16[j] = static_cast<uint16_t>(L);
      last8[j] = 0;
    }
    if (k > 0) last8[b + k - 1] = 1;
    for (uint32_t r = k; r < n; ++r) {
      key[b + r] = sentinel;
      val[b + r] = b + r;
    }
    maxL = L > maxL ? L : maxL;
    nc += k > 0;
    nv += k;
    U += L;
  }
  warp_atomic_max_u32(max_L, maxL);
  warp_atomic_add_u32(nconv, nc);
  warp_atomic_add_u32(nvalid, nv);
  warp_atomic_add_u64(universe, U);
}

// ---- time order: bucket sort on the arrival tick (buckets of 2^sh ticks, ~2 events each),
// then each bucket is sorted by (tick, slot) -- slot order is (conversation, turn), so ties come
// out as Reading #9 requires and the result does not depend on the atomics' order.  Slots with
// the sentinel key (context-capped turns) go to the extra last bucket (never read).
__global__ void gen_bucket_count_kernel(uint32_t n, const uint64_t* __restrict__ key, uint32_t sh, uint32_t nb,
                                        uint64_t sentinel, uint32_t* cnt) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const uint64_t k = key[j];
    atomicAdd(&cnt[k == sentinel ? nb : static_cast<uint32_t>(k >> sh)], 1u);
  }
}

__global__ void gen_bucket_place_kernel(uint32_t n, const uint64_t* __restrict__ key, uint32_t sh, uint32_t nb,
                                        uint64_t sentinel, const uint32_t* __restrict__ start, uint32_t* fill,
                                        uint64_t* okey, uint32_t* oval) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const uint64_t k = key[j];
    const uint32_t b = k == sentinel ? nb : static_cast<uint32_t>(k >> sh);
    const uint32_t p = start[b] + atomicAdd(&fill[b], 1u);
    okey[p] = k;
    oval[p] = j;  // the slot index
  }
}

__global__ void gen_bucket_sort_kernel(uint32_t nb, const uint32_t* __restrict__ start, uint64_t* key, uint32_t* val) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
    const uint32_t lo = start[b], hi = start[b + 1];
    for (uint32_t i = lo + 1; i < hi; ++i) {  // insertion sort by (tick, slot)
      const uint64_t k = key[i];
      const uint32_t v = val[i];
      uint32_t j = i;
      while (j > lo && (key[j - 1] > k || (key[j - 1] == k && val[j - 1] > v))) {
        key[j] = key[j - 1];
        val[j] = val[j - 1];
        --j;
      }
      key[j] = k;
      val[j] = v;
    }
  }
}

__global__ void gen_scatter_kernel(uint64_t E, const uint64_t* skey, const uint32_t* sval, const uint32_t* cid,
                                   const uint16_t* q16, const uint16_t* a16, const uint8_t* last8, uint32_t* pos,
                                   uint64_t* time_ticks, uint32_t* conv, uint16_t* prompt, uint16_t* response,
                                   uint8_t* is_last) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < E; i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t j = sval[i];
    pos[j] = static_cast<uint32_t>(i);
    if (time_ticks) time_ticks[i] = skey[i];
    if (conv) conv[i] = cid[j];
    if (prompt) prompt[i] = q16[j];
    if (response) response[i] = a16[j];
    if (is_last) is_last[i] = last8[j];
  }
}

__global__ void gen_link_kernel(uint64_t E, const uint32_t* sval, const uint32_t* cid, const uint32_t* off,
                                const uint16_t* J16, const uint16_t* La16, const uint8_t* last8, const uint32_t* pos,
                                uint64_t* sim, uint32_t* next) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < E; i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t j = sval[i];
    uint32_t prev = (j == off[cid[j]]) ? TLRU_NONE : pos[j - 1];
    next[i] = last8[j] ? TLRU_NONE : pos[j + 1];
    sim[i] = pack_sim(prev, J16[j], La16[j]);
  }
}

// ----------------------------------------------------------------------------- host
static tlru_status validate_gen(const tlru_gen_params* p) {
  if (!p) TLRU_FAIL(TLRU_EINVAL, "params is NULL");
  if (p->num_conversations == 0) TLRU_FAIL(TLRU_EINVAL, "num_conversations must be >= 1");
  if (p->block_tokens == 0) TLRU_FAIL(TLRU_EINVAL, "block_tokens must be >= 1");
  if (!(p->birth_rate > 0) || !(p->turn_rate > 0) || !(p->death_rate > 0))
    TLRU_FAIL(TLRU_EINVAL, "birth_rate, turn_rate and death_rate must be > 0");
  if (!(p->prompt_mean_tokens > 0) || !(p->response_mean_tokens > 0))
    TLRU_FAIL(TLRU_EINVAL, "prompt/response mean tokens must be > 0");
  if (!(p->prompt_sigma_ln >= 0) || !(p->response_sigma_ln >= 0)) TLRU_FAIL(TLRU_EINVAL, "sigma_ln must be >= 0");
  if (p->prompt_min_tokens > p->prompt_max_tokens || p->response_min_tokens > p->response_max_tokens)
    TLRU_FAIL(TLRU_EINVAL, "token clip range is empty");
  if (p->max_history_blocks == 0 || p->max_history_blocks > 65535)
    TLRU_FAIL(TLRU_ERANGE, "max_history_blocks must be in 1..65535");
  if (p->max_turns == 0 || p->max_turns > 65535) TLRU_FAIL(TLRU_EINVAL, "max_turns must be in 1..65535");
  if (uint64_t(p->num_conversations) * p->max_turns >= 0xFFFFFFFFull)
    TLRU_FAIL(TLRU_ERANGE, "num_conversations * max_turns must stay below 2^32 - 1 (u32 event links)");
  return TLRU_OK;
}

static GenDev make_dev(const tlru_gen_params* p) {
  GenDev g;
  g.seed = p->seed;
  g.N = p->num_conversations;
  g.B = p->block_tokens;
  g.Lmax = p->max_history_blocks;
  g.max_turns = p->max_turns;
  {
    const uint64_t qmax = std::max<uint64_t>(1, (uint64_t(p->prompt_max_tokens) + p->block_tokens - 1) / p->block_tokens);
    const uint64_t amax = (uint64_t(p->response_max_tokens) + p->block_tokens - 1) / p->block_tokens;
    g.safe_turns = static_cast<uint32_t>(std::min<uint64_t>(p->max_turns, p->max_history_blocks / (qmax + amax)));
  }
  g.us_birth = 1000000.0 / p->birth_rate;
  g.us_turn = 1000000.0 / p->turn_rate;
  g.us_death = 1000000.0 / p->death_rate;
  g.p_mean = p->prompt_mean_tokens;  // ln(mean) - sigma^2/2 is evaluated on the device (fixed-order dln)
  g.p_sigma = p->prompt_sigma_ln;
  g.r_mean = p->response_mean_tokens;
  g.r_sigma = p->response_sigma_ln;
  g.p_lo = p->prompt_min_tokens;
  g.p_hi = p->prompt_max_tokens;
  g.r_lo = p->response_min_tokens;
  g.r_hi = p->response_max_tokens;
  return g;
}

struct GenWs {
  uint64_t* gaps;   // [N]   then birth ticks (in place is not allowed by cub -> separate)
  uint64_t* birth;  // [N]
  uint32_t* counts; // [N+1]
  uint32_t* off;    // [N+1]
  unsigned long long* max_elapsed;
  uint32_t* max_L;
  uint32_t* nconv;
  uint32_t* queue;   // [N] conversations needing an exact length replay in the count pass
  uint32_t* nqueue;
  uint32_t* nvalid;
  unsigned long long* universe;
  uint16_t* turn;    // [E] turn index of each event slot
  uint64_t* gapt;    // [E] gap ticks to the previous turn
  uint64_t* key[2];
  uint32_t* val[2];
  uint32_t* cid;
  uint16_t *q16, *a16, *J16, *La16;
  uint8_t* last8;
  uint32_t* pos;
  uint32_t* bcnt;    // [cap / 2 + 2] time-bucket counts, then bucket starts (bucket sort)
  uint32_t* bfill;   // [cap / 2 + 2] bucket fill cursors
  void* cub_tmp;
  size_t cub_bytes;
};

static tlru_status carve_gen(Carver& cv, uint32_t N, uint64_t cap, GenWs* w) {
  w->gaps = cv.take<uint64_t>(N);
  w->birth = cv.take<uint64_t>(N);
  w->counts = cv.take<uint32_t>(N + 1);
  w->off = cv.take<uint32_t>(N + 1);
  w->max_elapsed = cv.take<unsigned long long>(1);
  w->max_L = cv.take<uint32_t>(1);
  w->nconv = cv.take<uint32_t>(1);
  w->queue = cv.take<uint32_t>(N);
  w->nqueue = cv.take<uint32_t>(1);
  w->nvalid = cv.take<uint32_t>(1);
  w->universe = cv.take<unsigned long long>(1);
  w->turn = cv.take<uint16_t>(cap);
  w->gapt = cv.take<uint64_t>(cap);
  for (int i = 0; i < 2; ++i) {
    w->key[i] = cv.take<uint64_t>(cap);
    w->val[i] = cv.take<uint32_t>(cap);
  }
  w->cid = cv.take<uint32_t>(cap);
  w->q16 = cv.take<uint16_t>(cap);
  w->a16 = cv.take<uint16_t>(cap);
  w->J16 = cv.take<uint16_t>(cap);
  w->La16 = cv.take<uint16_t>(cap);
  w->last8 = cv.take<uint8_t>(cap);
  w->pos = cv.take<uint32_t>(cap);
  w->bcnt = cv.take<uint32_t>(cap / 2 + 3);
  w->bfill = cv.take<uint32_t>(cap / 2 + 3);
  size_t s1 = 0, s2 = 0, s3 = 0;
  cub::DoubleBuffer<uint64_t> kb(nullptr, nullptr);
  cub::DoubleBuffer<uint32_t> vb(nullptr, nullptr);
  if (cub::DeviceRadixSort::SortPairs(nullptr, s1, kb, vb, static_cast<int>(cap > 0 ? cap : 1)) != cudaSuccess ||
      cub::DeviceScan::InclusiveSum(nullptr, s2, (uint64_t*)nullptr, (uint64_t*)nullptr, static_cast<int>(N)) !=
          cudaSuccess ||
      cub::DeviceScan::ExclusiveSum(nullptr, s3, (uint32_t*)nullptr, (uint32_t*)nullptr, static_cast<int>(N + 1)) !=
          cudaSuccess)
    TLRU_FAIL(TLRU_ECUDA, "cub temp-storage query failed");
  size_t s4 = 0;
  if (cub::DeviceScan::ExclusiveSum(nullptr, s4, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                    static_cast<int>(cap / 2 + 3)) != cudaSuccess)
    TLRU_FAIL(TLRU_ECUDA, "cub temp-storage query failed");
  w->cub_bytes = std::max(std::max(s1, s4), std::max(s2, s3));
  w->cub_tmp = cv.take<char>(w->cub_bytes);
  return TLRU_OK;
}

// Runs count + scans; fills E (host) and the max tick bound.  Synchronizes.
// exact = false: slots from the turn clocks only (an upper bound; context-capped turns are
// dropped later by gen_emit_kernel).  exact = true: the exact event count.
static tlru_status run_count(const tlru_gen_params* p, const GenWs& w, cudaStream_t st, uint64_t* E,
                             uint64_t* max_tick, bool exact) {
  GenDev g = make_dev(p);
  TLRU_CUDA(cudaMemsetAsync(w.max_elapsed, 0, sizeof(unsigned long long), st));
  TLRU_CUDA(cudaMemsetAsync(w.nqueue, 0, sizeof(uint32_t), st));
  gen_count_kernel<<<grid_for(g.N, 128), 128, 0, st>>>(g, w.gaps, w.counts, w.max_elapsed, w.queue, w.nqueue);
  TLRU_CHECK_LAUNCH();
  if (exact) {
    gen_count_fix_kernel<<<grid_for(g.N / 8 + 1, 128), 128, 0, st>>>(g, w.queue, w.nqueue, w.counts);
    TLRU_CHECK_LAUNCH();
  }
  size_t b = w.cub_bytes;
  TLRU_CUDA(cub::DeviceScan::InclusiveSum(w.cub_tmp, b, w.gaps, w.birth, static_cast<int>(g.N), st));
  b = w.cub_bytes;
  TLRU_CUDA(cub::DeviceScan::ExclusiveSum(w.cub_tmp, b, w.counts, w.off, static_cast<int>(g.N + 1), st));
  uint32_t totalE = 0;
  uint64_t last_birth = 0;
  unsigned long long mel = 0;
  TLRU_CUDA(cudaMemcpyAsync(&totalE, w.off + g.N, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  TLRU_CUDA(cudaMemcpyAsync(&last_birth, w.birth + (g.N - 1), sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  TLRU_CUDA(cudaMemcpyAsync(&mel, w.max_elapsed, sizeof(mel), cudaMemcpyDeviceToHost, st));
  TLRU_CUDA(cudaStreamSynchronize(st));
  *E = totalE;
  *max_tick = last_birth + mel;
  return TLRU_OK;
}

// ----------------------------------------------------------------------------- upload path
__global__ void up_init_kernel(uint64_t E, const uint32_t* conv, const uint16_t* q, uint32_t* key, uint32_t* val,
                               unsigned long long* bad_q, unsigned long long* bad_conv) {
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < E; e += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t c = conv[e];
    key[e] = c;
    val[e] = static_cast<uint32_t>(e);
    if (q[e] == 0) atomicMin(bad_q, static_cast<unsigned long long>(e));
    if (c == TLRU_NONE) atomicMin(bad_conv, static_cast<unsigned long long>(e));
  }
}

__global__ void up_weight_kernel(uint64_t E, const uint32_t* sval, const uint16_t* q, const uint16_t* a,
                                 uint32_t* w) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < E; i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t e = sval[i];
    w[i] = uint32_t(q[e]) + uint32_t(a[e]);
  }
}

// In conversation-major order (stable, so time order within a conversation):
// L_after = running sum of q + a, J = L_after - a, prev/next = neighbours.
__global__ void up_link_kernel(uint64_t E, const uint32_t* skey, const uint32_t* sval, const uint32_t* cum,
                               const uint16_t* a, const uint64_t* ticks, uint64_t* sim, uint32_t* next,
                               uint8_t* is_last, uint64_t* time_ticks, unsigned long long* bad_range,
                               unsigned long long* bad_ticks, uint32_t* max_L, uint32_t* nconv,
                               unsigned long long* universe) {
  uint32_t maxL = 0, nc = 0;
  unsigned long long bad = ~0ull, badt = ~0ull, U = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < E; i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t e = sval[i];
    uint32_t La = cum[i];
    uint32_t J = La - a[e];
    if (La > 65535u && e < bad) bad = e;
    bool first = (i == 0) || skey[i - 1] != skey[i];
    bool last = (i + 1 == E) || skey[i + 1] != skey[i];
    uint32_t prev = first ? TLRU_NONE : sval[i - 1];
    uint32_t nx = last ? TLRU_NONE : sval[i + 1];
    sim[e] = pack_sim(prev, J, La);
    next[e] = nx;
    if (is_last) is_last[e] = last ? 1 : 0;
    if (time_ticks) time_ticks[e] = ticks ? ticks[e] : e;
    if (ticks && e > 0 && ticks[e - 1] > ticks[e] && e < badt) badt = e;
    nc += first;
    if (last) {
      maxL = max(maxL, La > 65535u ? 65535u : La);
      U += La;
    }
  }
  warp_atomic_max_u32(max_L, maxL);
  warp_atomic_add_u32(nconv, nc);
  warp_atomic_add_u64(universe, U);
  if (bad != ~0ull) atomicMin(bad_range, bad);
  if (badt != ~0ull) atomicMin(bad_ticks, badt);
}

struct UpWs {
  uint32_t* key[2];
  uint32_t* val[2];
  uint32_t* w;
  uint32_t* cum;
  unsigned long long* flags;  // bad_q, bad_conv, bad_range, bad_ticks, universe
  uint32_t* stats;            // max_L, nconv
  void* cub_tmp;
  size_t cub_bytes;
};

static tlru_status carve_up(Carver& cv, uint64_t E, UpWs* w) {
  uint64_t n = E > 0 ? E : 1;
  for (int i = 0; i < 2; ++i) {
    w->key[i] = cv.take<uint32_t>(n);
    w->val[i] = cv.take<uint32_t>(n);
  }
  w->w = cv.take<uint32_t>(n);
  w->cum = cv.take<uint32_t>(n);
  w->flags = cv.take<unsigned long long>(5);
  w->stats = cv.take<uint32_t>(2);
  size_t s1 = 0, s2 = 0;
  cub::DoubleBuffer<uint32_t> kb(nullptr, nullptr), vb(nullptr, nullptr);
  if (cub::DeviceRadixSort::SortPairs(nullptr, s1, kb, vb, static_cast<int>(n)) != cudaSuccess ||
      cub::DeviceScan::InclusiveSumByKey(nullptr, s2, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                         static_cast<int>(n)) != cudaSuccess)
    TLRU_FAIL(TLRU_ECUDA, "cub temp-storage query failed");
  w->cub_bytes = std::max(s1, s2);
  w->cub_tmp = cv.take<char>(w->cub_bytes);
  return TLRU_OK;
}

}  // namespace tlru

using namespace tlru;

extern "C" tlru_status tlru_trace_max_events(const tlru_gen_params* p, uint64_t* out) {
  clear_error();
  TLRU_TRY(validate_gen(p));
  if (!out) TLRU_FAIL(TLRU_EINVAL, "out is NULL");
  *out = uint64_t(p->num_conversations) * p->max_turns;
  return TLRU_OK;
}

extern "C" tlru_status tlru_gen_workspace_size(const tlru_gen_params* p, uint64_t capacity, size_t* bytes) {
  clear_error();
  TLRU_TRY(validate_gen(p));
  if (!bytes) TLRU_FAIL(TLRU_EINVAL, "bytes is NULL");
  if (capacity >= 0xFFFFFFFFull) TLRU_FAIL(TLRU_ERANGE, "capacity must be < 2^32 - 1");
  Carver cv(nullptr);
  GenWs w;
  TLRU_TRY(carve_gen(cv, p->num_conversations, capacity, &w));
  *bytes = cv.used;
  return TLRU_OK;
}

extern "C" tlru_status tlru_count_events(const tlru_gen_params* p, uint64_t* out, void* ws, size_t ws_bytes,
                                         cudaStream_t stream) {
  clear_error();
  TLRU_TRY(validate_gen(p));
  if (!out) TLRU_FAIL(TLRU_EINVAL, "out is NULL");
  Carver cv(ws);
  GenWs w;
  TLRU_TRY(carve_gen(cv, p->num_conversations, 0, &w));
  TLRU_TRY(check_ws(cv, ws, ws_bytes));
  uint64_t mt;
  return run_count(p, w, stream, out, &mt, true);
}

extern "C" tlru_status tlru_count_event_slots(const tlru_gen_params* p, uint64_t* out, void* ws, size_t ws_bytes,
                                              cudaStream_t stream) {
  clear_error();
  TLRU_TRY(validate_gen(p));
  if (!out) TLRU_FAIL(TLRU_EINVAL, "out is NULL");
  Carver cv(ws);
  GenWs w;
  TLRU_TRY(carve_gen(cv, p->num_conversations, 0, &w));
  TLRU_TRY(check_ws(cv, ws, ws_bytes));
  uint64_t mt;
  return run_count(p, w, stream, out, &mt, false);
}

extern "C" tlru_status tlru_generate_traces(const tlru_gen_params* params, uint32_t n, tlru_trace* traces, void* ws,
                                            size_t ws_bytes, cudaStream_t st) {
  clear_error();
  if (n > 0 && (!params || !traces)) TLRU_FAIL(TLRU_EINVAL, "params/traces is NULL");
  for (uint32_t t = 0; t < n; ++t) {
    const tlru_gen_params* p = params + t;
    tlru_trace* tr = traces + t;
    TLRU_TRY(validate_gen(p));
    if (!tr->sim || !tr->next) TLRU_FAIL(TLRU_EINVAL, "trace %u: sim and next arrays are required", t);
    if (tr->capacity >= 0xFFFFFFFFull) TLRU_FAIL(TLRU_ERANGE, "trace %u: capacity must be < 2^32 - 1", t);
    Carver cv(ws);
    GenWs w;
    TLRU_TRY(carve_gen(cv, p->num_conversations, tr->capacity, &w));
    TLRU_TRY(check_ws(cv, ws, ws_bytes));
    uint64_t E, max_tick;  // E = event slots
    TLRU_TRY(run_count(p, w, st, &E, &max_tick, false));
    if (E > tr->capacity) TLRU_TRY(run_count(p, w, st, &E, &max_tick, true));  // no room for spare slots
    if (E > tr->capacity)
      TLRU_FAIL(TLRU_ERANGE, "trace %u: %llu events exceed capacity %llu", t, (unsigned long long)E,
                (unsigned long long)tr->capacity);
    GenDev g = make_dev(p);
    int end_bit = 1;  // the sentinel key (all ones below end_bit) sorts after every arrival tick
    while (end_bit < 64 && ((max_tick + 1) >> end_bit) != 0) ++end_bit;
    const uint64_t sentinel = end_bit >= 64 ? ~0ull : ((1ull << end_bit) - 1);
    TLRU_CUDA(cudaMemsetAsync(w.max_L, 0, sizeof(uint32_t), st));
    TLRU_CUDA(cudaMemsetAsync(w.nconv, 0, sizeof(uint32_t), st));
    TLRU_CUDA(cudaMemsetAsync(w.nvalid, 0, sizeof(uint32_t), st));
    TLRU_CUDA(cudaMemsetAsync(w.universe, 0, sizeof(unsigned long long), st));
    gen_slot_kernel<<<grid_for(g.N, 128), 128, 0, st>>>(g, w.off, w.cid, w.turn);
    TLRU_CHECK_LAUNCH();
    if (E > 0) {
      gen_draw_kernel<<<grid_for(E, 128), 128, 0, st>>>(g, static_cast<uint32_t>(E), w.cid, w.turn, w.gapt, w.q16,
                                                         w.a16);
      TLRU_CHECK_LAUNCH();
    }
    gen_emit_kernel<<<grid_for(g.N, 128), 128, 0, st>>>(g, w.birth, w.off, w.gapt, w.q16, w.a16, sentinel, w.key[0],
                                                         w.val[0], w.J16, w.La16, w.last8, w.max_L, w.nconv,
                                                         w.nvalid, w.universe);
    TLRU_CHECK_LAUNCH();
    uint32_t stats[3];
    unsigned long long universe = 0;
    TLRU_CUDA(cudaMemcpyAsync(&stats[0], w.max_L, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    TLRU_CUDA(cudaMemcpyAsync(&stats[1], w.nconv, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    TLRU_CUDA(cudaMemcpyAsync(&stats[2], w.nvalid, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    TLRU_CUDA(cudaMemcpyAsync(&universe, w.universe, sizeof(universe), cudaMemcpyDeviceToHost, st));
    TLRU_CUDA(cudaStreamSynchronize(st));
    const uint64_t slots = E;
    E = stats[2];  // events that survive the context cap
    if (E > 0) {
      // bucket width 2^sh ticks: about two events per bucket over [0, max_tick]
      uint32_t sh = 0;
      while (sh < 63 && ((max_tick >> sh) + 1) > slots / 2 + 1) ++sh;
      const uint32_t nb = static_cast<uint32_t>((max_tick >> sh) + 1);  // + 1 sentinel bucket at nb
      const uint32_t n = static_cast<uint32_t>(slots);
      TLRU_CUDA(cudaMemsetAsync(w.bcnt, 0, (nb + 2) * sizeof(uint32_t), st));
      TLRU_CUDA(cudaMemsetAsync(w.bfill, 0, (nb + 2) * sizeof(uint32_t), st));
      gen_bucket_count_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, w.key[0], sh, nb, sentinel, w.bcnt);
      TLRU_CHECK_LAUNCH();
      size_t b = w.cub_bytes;  // in place: starts[b] = exclusive prefix of counts, starts[nb + 1] = n
      TLRU_CUDA(cub::DeviceScan::ExclusiveSum(w.cub_tmp, b, w.bcnt, w.bcnt, static_cast<int>(nb + 2), st));
      gen_bucket_place_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, w.key[0], sh, nb, sentinel, w.bcnt, w.bfill,
                                                                w.key[1], w.val[1]);
      TLRU_CHECK_LAUNCH();
      gen_bucket_sort_kernel<<<grid_for(nb, 256), 256, 0, st>>>(nb, w.bcnt, w.key[1], w.val[1]);
      TLRU_CHECK_LAUNCH();
      gen_scatter_kernel<<<grid_for(E, 256), 256, 0, st>>>(E, w.key[1], w.val[1], w.cid, w.q16, w.a16, w.last8,
                                                           w.pos, tr->time_ticks, tr->conv, tr->prompt, tr->response,
                                                           tr->is_last);
      TLRU_CHECK_LAUNCH();
      gen_link_kernel<<<grid_for(E, 256), 256, 0, st>>>(E, w.val[1], w.cid, w.off, w.J16, w.La16, w.last8, w.pos,
                                                        tr->sim, tr->next);
      TLRU_CHECK_LAUNCH();
    }
    tr->num_events = E;  // known since the stats copy: the rest of the generation stays asynchronous
    tr->max_history = stats[0];
    tr->num_conversations = stats[1];
    tr->universe_blocks = universe;
    tr->flags = 0;
  }
  return TLRU_OK;
}

extern "C" tlru_status tlru_upload_workspace_size(uint64_t E, size_t* bytes) {
  clear_error();
  if (!bytes) TLRU_FAIL(TLRU_EINVAL, "bytes is NULL");
  if (E >= 0xFFFFFFFFull) TLRU_FAIL(TLRU_ERANGE, "E must be < 2^32 - 1");
  Carver cv(nullptr);
  UpWs w;
  TLRU_TRY(carve_up(cv, E, &w));
  *bytes = cv.used;
  return TLRU_OK;
}

extern "C" tlru_status tlru_trace_from_turns(const uint32_t* conv, const uint16_t* q, const uint16_t* a,
                                             const uint64_t* ticks, uint64_t E, tlru_trace* out, void* ws,
                                             size_t ws_bytes, cudaStream_t st) {
  clear_error();
  if (!out) TLRU_FAIL(TLRU_EINVAL, "out is NULL");
  if (E >= 0xFFFFFFFFull) TLRU_FAIL(TLRU_ERANGE, "E must be < 2^32 - 1");
  if (E > out->capacity) TLRU_FAIL(TLRU_ERANGE, "E = %llu exceeds capacity %llu", (unsigned long long)E,
                                   (unsigned long long)out->capacity);
  if (E > 0 && (!conv || !q || !a)) TLRU_FAIL(TLRU_EINVAL, "conv/q/a is NULL");
  if (E > 0 && (!out->sim || !out->next)) TLRU_FAIL(TLRU_EINVAL, "sim and next arrays are required");
  Carver cv(ws);
  UpWs w;
  TLRU_TRY(carve_up(cv, E, &w));
  TLRU_TRY(check_ws(cv, ws, ws_bytes));
  out->num_events = E;
  out->max_history = 0;
  out->num_conversations = 0;
  out->universe_blocks = 0;
  out->flags = ticks ? 0u : TLRU_TRACE_SYNTHETIC_TICKS;
  if (E == 0) return TLRU_OK;
  const unsigned long long init[5] = {~0ull, ~0ull, ~0ull, ~0ull, 0ull};
  TLRU_CUDA(cudaMemcpyAsync(w.flags, init, sizeof(init), cudaMemcpyHostToDevice, st));
  TLRU_CUDA(cudaMemsetAsync(w.stats, 0, 2 * sizeof(uint32_t), st));
  up_init_kernel<<<grid_for(E, 256), 256, 0, st>>>(E, conv, q, w.key[0], w.val[0], w.flags, w.flags + 1);
  TLRU_CHECK_LAUNCH();
  cub::DoubleBuffer<uint32_t> kb(w.key[0], w.key[1]), vb(w.val[0], w.val[1]);
  size_t b = w.cub_bytes;
  TLRU_CUDA(cub::DeviceRadixSort::SortPairs(w.cub_tmp, b, kb, vb, static_cast<int>(E), 0, 32, st));
  up_weight_kernel<<<grid_for(E, 256), 256, 0, st>>>(E, vb.Current(), q, a, w.w);
  TLRU_CHECK_LAUNCH();
  b = w.cub_bytes;
  TLRU_CUDA(cub::DeviceScan::InclusiveSumByKey(w.cub_tmp, b, kb.Current(), w.w, w.cum, static_cast<int>(E),
                                               cub::Equality(), st));
  up_link_kernel<<<grid_for(E, 256), 256, 0, st>>>(E, kb.Current(), vb.Current(), w.cum, a, ticks, out->sim,
                                                   out->next, out->is_last, out->time_ticks, w.flags + 2,
                                                   w.flags + 3, w.stats, w.stats + 1, w.flags + 4);
  TLRU_CHECK_LAUNCH();
  if (out->conv) TLRU_CUDA(cudaMemcpyAsync(out->conv, conv, E * 4, cudaMemcpyDeviceToDevice, st));
  if (out->prompt) TLRU_CUDA(cudaMemcpyAsync(out->prompt, q, E * 2, cudaMemcpyDeviceToDevice, st));
  if (out->response) TLRU_CUDA(cudaMemcpyAsync(out->response, a, E * 2, cudaMemcpyDeviceToDevice, st));
  unsigned long long flags[5];
  uint32_t stats[2];
  TLRU_CUDA(cudaMemcpyAsync(flags, w.flags, sizeof(flags), cudaMemcpyDeviceToHost, st));
  TLRU_CUDA(cudaMemcpyAsync(stats, w.stats, sizeof(stats), cudaMemcpyDeviceToHost, st));
  TLRU_CUDA(cudaStreamSynchronize(st));
  if (flags[1] != ~0ull) TLRU_FAIL(TLRU_EINVAL, "conv[%llu] == TLRU_NONE is reserved", flags[1]);
  if (flags[0] != ~0ull) TLRU_FAIL(TLRU_EINVAL, "q[%llu] == 0: every prompt has at least one block", flags[0]);
  if (flags[2] != ~0ull) TLRU_FAIL(TLRU_ERANGE, "event %llu: L_after exceeds 65535 blocks", flags[2]);
  if (flags[3] != ~0ull) TLRU_FAIL(TLRU_EINVAL, "ticks[%llu] < ticks[%llu]: arrival times must be non-decreasing",
                                   flags[3], flags[3] - 1);
  out->max_history = stats[0];
  out->num_conversations = stats[1];
  out->universe_blocks = flags[4];
  return TLRU_OK;
}
