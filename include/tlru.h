/*
 * tlru.h -- C ABI of libtlru, the B200-native (sm_100a) hot path of
 * arXiv 2510.15152 "Tail-Optimized LRU": batched trace-driven simulation of
 * prompt-cache (KV prefix) eviction under LRU and T-LRU over multi-turn
 * conversation traces.
 *
 * Citations: P:NNN = PAPER.md line NNN with its section / equation / algorithm.
 * "Reading #k" = DESIGN.md "Readings of the paper" item k.
 *
 * Conventions for every call
 *   * Pointers are caller-owned DEVICE memory unless marked "host".  The library
 *     never allocates device memory; scratch comes from the caller's workspace
 *     `ws` (size it with the matching *_workspace_size call; ws must be
 *     256-byte aligned).  `ws == NULL` with a non-zero requirement is TLRU_ERANGE.
 *   * Calls are asynchronous on `stream` unless marked "synchronizes".  Outputs
 *     are valid once the stream is synchronized.  Distinct streams are
 *     thread-safe; one stream must not be used from two threads at once.
 *   * No C++ exception crosses the ABI.  On a non-OK status, tlru_last_error()
 *     returns a thread-local message naming the offending argument / index;
 *     outputs are then unspecified.
 *   * Integers are the contract: uncached-block counts, evictions, TEL in
 *     blocks, SLO counts and percentiles (in blocks) are exact.  Floating point
 *     appears only in tlru_tail's millisecond fields, derived from integers.
 *   * Determinism: identical inputs give identical output bytes for any launch
 *     configuration and any number of GPUs.
 */
#ifndef TLRU_H_
#define TLRU_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TLRU_NONE 0xFFFFFFFFu /* "no previous / next turn" in prev/next links */

typedef enum {
  TLRU_OK = 0,
  TLRU_EINVAL = 1,       /* bad argument or configuration (block_tokens == 0, rate <= 0, q == 0, ...) */
  TLRU_ERANGE = 2,       /* buffer / workspace too small, or a value exceeds its field width (J > 65535) */
  TLRU_ECUDA = 3,        /* CUDA runtime error; tlru_last_error() carries cudaGetErrorString */
  TLRU_EUNSUPPORTED = 4, /* policy family not built (policy > TLRU_POLICY_ETLRU_FORCED) */
  TLRU_ESTATE = 5        /* internal per-chain state pool exhausted with no fallback left */
} tlru_status;

/* Thread-local message for the last non-OK status of this thread ("" if none). */
const char* tlru_last_error(void);

/* Library version string, e.g. "tlru 0.1 sm_100a". */
const char* tlru_version(void);

/* Total kernel launches issued by this library in this process (host counter). */
uint64_t tlru_launch_count(void);

/* ------------------------------------------------------------------------
 * Synthetic traces: the paper's stochastic conversation model (Sec. 5)
 *   - conversations are born by a Poisson(birth_rate) process;
 *   - each conversation lives an Exp(death_rate) time;
 *   - while alive it issues turns by a Poisson(turn_rate) process;
 *     the first turn is at birth (Reading #18);
 *   - each turn draws a prompt length Q and a response length A,
 *     here lognormal in tokens, quantized to blocks of `block_tokens`
 *     (q = max(1, ceil(tokens/B)), a = ceil(tokens/B); Reading #16);
 *   - a turn whose history would exceed max_history_blocks ends the
 *     conversation (context window), as does max_turns.
 * App. E's recipe is the ShareGPT preset.  Random numbers come from
 * Philox4x64-10 keyed by the seed with counter (conv, turn, attempt, 0): attempt 0
 * of a turn gives the gap before it (turn 0: the birth gap), the first Marsaglia
 * polar pair and (turn 0) the death clock; a rejected pair retries with attempt
 * 1, 2, ...; so a trace is a pure function of its parameters (Reading #16).  Time
 * is kept in integer microsecond ticks; events are ordered by (tick, conv, turn).
 * ------------------------------------------------------------------------ */
typedef struct {
  uint64_t seed;
  uint32_t num_conversations;    /* N >= 1 */
  uint32_t block_tokens;         /* tokens per KV block (128 in the BASELINE configs); 0 -> EINVAL */
  double birth_rate;             /* lambda_conv > 0, per second */
  double turn_rate;              /* lambda_turn > 0, per second, homogeneous */
  double death_rate;             /* mu > 0, per second; mean turns = 1 + turn_rate / death_rate */
  double prompt_mean_tokens;     /* lognormal mean > 0 (WildChat: 200) */
  double prompt_sigma_ln;        /* lognormal sigma of ln(tokens) >= 0 */
  double response_mean_tokens;   /* lognormal mean > 0 (paper silent; A is arbitrary) */
  double response_sigma_ln;      /* >= 0 */
  uint32_t prompt_min_tokens;    /* clip range for prompt tokens */
  uint32_t prompt_max_tokens;
  uint32_t response_min_tokens;  /* clip range for response tokens */
  uint32_t response_max_tokens;
  uint32_t max_history_blocks;   /* context cap L_max in blocks, 1..65535 */
  uint32_t max_turns;            /* hard cap on turns per conversation, 1..65535 */
} tlru_gen_params;

/* One event-ordered trace (conversation i issues requests at
 * disjoint times T_i; q_{i,t}, a_{i,t} in blocks).  Event index = tau. */
typedef struct {
  uint64_t capacity;    /* in:  allocated length of every non-NULL array below */
  uint64_t num_events;  /* out: E */
  uint32_t max_history; /* out: max over events of L_after (bounds every J and every b) */
  uint32_t num_conversations; /* out: number of distinct conversation ids */
  uint64_t universe_blocks;   /* out: sum over conversations of their final L_after (the "universe" of
                                 the stack engine's window sums) */
  uint32_t flags;             /* out: TLRU_TRACE_* bits below */
  uint32_t reserved;
  uint64_t* sim;        /* [E] required.  Simulation view, 8 B per request:
                             bits  0..31 prev = event index of the same conversation's previous
                                         turn, or TLRU_NONE for a first turn
                             bits 32..47 J = L_before + q   (job size)
                             bits 48..63 L_after = J + a    (history after the turn, Reading #6) */
  uint32_t* next;       /* [E] required: event index of the next turn of the same conversation,
                             TLRU_NONE if none (used to rebuild cache state at segment starts) */
  uint32_t* conv;       /* [E] nullable export: conversation id (dense, birth order for generated traces) */
  uint16_t* prompt;     /* [E] nullable export: q blocks >= 1 */
  uint16_t* response;   /* [E] nullable export: a blocks >= 0 */
  uint64_t* time_ticks; /* [E] nullable export: arrival time in microseconds (generated traces; the
                             caller's ticks on upload, else event indices and TLRU_TRACE_SYNTHETIC_TICKS) */
  uint8_t* is_last;     /* [E] nullable export: 1 on a conversation's last turn */
} tlru_trace;

/* tlru_trace.flags: time_ticks holds event indices, not arrival times (an upload without
 * ticks).  ET-LRU's beliefs decay with time, so ET-LRU instances on such a trace are
 * TLRU_EINVAL. */
#define TLRU_TRACE_SYNTHETIC_TICKS 1u

/* Host: upper bound N * max_turns on the events of a generated trace. */
tlru_status tlru_trace_max_events(const tlru_gen_params* p /*host*/, uint64_t* out /*host*/);

/* Host: workspace bytes for tlru_count_events / tlru_generate_traces of one trace
 * with N conversations whose trace arrays have `capacity` entries. */
tlru_status tlru_gen_workspace_size(const tlru_gen_params* p /*host*/, uint64_t capacity,
                                    size_t* bytes /*host*/);

/* Exact event count of the trace `p` describes.  Synchronizes `stream`. */
tlru_status tlru_count_events(const tlru_gen_params* p /*host*/, uint64_t* out /*host*/, void* ws,
                              size_t ws_bytes, cudaStream_t stream);

/* Event slots of the trace `p` describes: turns allowed by the birth / death / turn clocks
 * before the context-window rule drops any, so E <= slots.  A trace whose
 * arrays hold >= slots entries is generated with one counting pass; with fewer (but >= E)
 * tlru_generate_traces counts a second time, exactly.  Synchronizes `stream`. */
tlru_status tlru_count_event_slots(const tlru_gen_params* p /*host*/, uint64_t* out /*host*/, void* ws,
                                   size_t ws_bytes, cudaStream_t stream);

/* Generate n traces (one per params entry) into traces[i] (host structs holding
 * device arrays).  capacity < E -> TLRU_ERANGE.  Fills num_events, max_history
 * and num_conversations.  Synchronizes `stream` once per trace (to read E). */
tlru_status tlru_generate_traces(const tlru_gen_params* p /*host[n]*/, uint32_t n,
                                 tlru_trace* traces /*host[n]*/, void* ws, size_t ws_bytes,
                                 cudaStream_t stream);

/* Host: workspace bytes for tlru_trace_from_turns with E requests. */
tlru_status tlru_upload_workspace_size(uint64_t E, size_t* bytes /*host*/);

/* Build the simulation view of an uploaded trace.  conv/q/a are DEVICE arrays
 * in event (time) order; conversation ids are arbitrary u32 except TLRU_NONE.
 * ticks (DEVICE u64[E], nullable) are the arrival times, non-decreasing, in the unit
 * ET-LRU's mu_per_tick uses; they are copied to out->time_ticks.  Without ticks,
 * out->time_ticks (if non-NULL) receives event indices and out->flags gets
 * TLRU_TRACE_SYNTHETIC_TICKS.  The library derives prev, next, J = L_before + q and
 * L_after = J + a and fills out->sim / out->next, copying the non-NULL
 * export arrays, and out->max_history, num_conversations, universe_blocks, flags.
 * q == 0 or decreasing ticks -> TLRU_EINVAL; J or L_after > 65535 -> TLRU_ERANGE
 * (offending event index in tlru_last_error()).  E == 0 is valid.  Synchronizes `stream`. */
tlru_status tlru_trace_from_turns(const uint32_t* conv, const uint16_t* q, const uint16_t* a,
                                  const uint64_t* ticks, uint64_t E,
                                  tlru_trace* out /*host struct, device arrays*/, void* ws,
                                  size_t ws_bytes, cudaStream_t stream);

/* ------------------------------------------------------------------------
 * Batched simulation: Alg. 1 per instance.
 * Per request of conversation theta: b = J - X_theta (uncached blocks,
 * P:154-156); then X_theta <- L_after (optional caching caches the whole
 * history, Reading #7), tau_theta <- now; if sum X > C:
 *   Phase 1 (T-LRU only): evict TEL-safe ("infinitely old", P:62,
 *     P:225) blocks, i.e. each conversation's blocks above its budget
 *     (L + Q_hat - xi)^+ (P:56), oldest tau first, theta last, as many
 *     as needed (Readings #1-#5);
 *   Phase 2: evict from the least recently used conversation,
 *     partially, tail blocks first (Reading #10).
 * LRU = Phase 2 only.  xi and Q_hat are in blocks (xi = xi_s / alpha).
 * Threshold-LRU (the paper's baseline): LRU that caches a
 *   conversation's history only once its length reaches `threshold` blocks
 *   (L_after >= threshold, Reading #23): below it nothing is cached (b = J),
 *   at or above it the whole history is cached and evicted by plain LRU.
 * End-Aware / Length-Aware T-LRU (Readings #24-#25): the trace
 *   supplies the future knowledge -- a turn with no later turn of its
 *   conversation releases theta's blocks (not counted as evictions) and caches
 *   nothing; Length-Aware budgets each cached history with the true next prompt,
 *   surplus = min(L_after, max(xi - q_next, 0)).  Their cache is not the top-C of
 *   the universe, so they always run on the replay engine, as time segments that
 *   start with a burn-in from an empty cache and are verified against their
 *   predecessor's end state (a fix-up kernel re-runs any segment whose start state
 *   was not exact).  In a batch that also holds LRU / T-LRU / Threshold-LRU
 *   instances, those still run on the stack engine (stats.engine = MIXED).
 * Tail-Optimized Belady (Thm 1; proof App. A; Reading
 *   #26): the hindsight policy, clairvoyant through the trace's next links.
 *   theta caches its whole history; on overflow Phase 1 trims blocks above the
 *   exact TEL-safe budget (L + q_next - xi)^+ (0 for a conversation that never
 *   returns), furthest next arrival first; Phase 2 evicts the conversation whose
 *   next arrival is furthest in the future (evicted_lru counts these), partial.
 *   q_hat is ignored.  Replay engine only (like End-/Length-Aware).
 * Expected-Tail-Optimized LRU (Def. 1; greedy Alg. 2, P:603-650;
 *   Reading #27): on overflow, evict blocks one at a time from the minimum of
 *   v_i = lambda_i P(L_i + Q_i - xi >= X_i), belief lambda_i = exp(-mu (t - time_i))
 *   (P:255); equivalently the minimum static score
 *   (double)time_ticks_i * mu_tick + ln_surv[X_i - L_i + xi] (IEEE multiply then add;
 *   ln_surv[k <= 0] = 0, ln_surv[k > K] = -inf), ties -> older last turn.  The model
 *   comes from tlru_set_etlru_model; the trace must carry time_ticks.  evicted_trim
 *   counts blocks with P = 0 (TEL-safe), evicted_lru the rest.  q_hat is ignored.
 *   One warp per instance (replay engine only).
 * T-LRU under forced caching (App. C; Reading #28): Alg. 1 where the
 *   post-decision state must hold theta's whole history -- Phases 1 and 2 skip
 *   theta; only if theta alone exceeds C does it lose tail blocks (counted in
 *   evicted_lru).  With xi <= q_hat it equals LRU.  Replay engine only.
 *   Feasibility: constraint (3) as an equality cannot hold on a request whose
 *   history exceeds the cache (L_after > C); the library does not fail such a
 *   run -- theta keeps its C most recent blocks -- and does not flag it: the
 *   number of such requests of an instance is #{e : L_after_e > C}, a function
 *   of the trace alone (e.g. from the exported q / response arrays).
 * Tail-Optimized Belady under forced caching (App. C: "Theorem 1
 *   continues to hold" with constraint (3) as an equality; Reading #29): the
 *   Tail-Optimized Belady rule with theta excluded from both phases; only if
 *   theta alone exceeds C does it lose tail blocks, above-budget ones first
 *   (counted in evicted_lru).  Its TEL is the forced hindsight optimum.  Replay
 *   engine only.
 * ET-LRU under forced caching (App. C: Y_theta = L; Reading #30):
 *   ET-LRU whose greedy never picks theta while its turn is served; if no other
 *   block is left and the cache still exceeds C, theta loses the excess from its
 *   tail (evicted_lru).  With a fixed prompt length it is forced T-LRU.
 *   Needs the ET-LRU model and real ticks, like ET-LRU.  One warp per instance.
 * ------------------------------------------------------------------------ */
enum {
  TLRU_POLICY_LRU = 0,
  TLRU_POLICY_TLRU = 1,
  TLRU_POLICY_THRESHOLD = 2,
  TLRU_POLICY_END_AWARE = 3,
  TLRU_POLICY_LENGTH_AWARE = 4,
  TLRU_POLICY_TAIL_BELADY = 5,
  TLRU_POLICY_ET_LRU = 6,
  TLRU_POLICY_TLRU_FORCED = 7,
  TLRU_POLICY_BELADY_FORCED = 8,
  TLRU_POLICY_ETLRU_FORCED = 9 /* > 9 -> TLRU_EUNSUPPORTED */
};

typedef struct {
  uint32_t trace;    /* index into traces[] */
  uint32_t policy;   /* TLRU_POLICY_* */
  uint32_t capacity; /* C in blocks, >= 0 */
  uint32_t xi;       /* xi in blocks: T-LRU threshold and TEL threshold (Eq. 3) */
  uint32_t q_hat;    /* Q_hat in blocks, next-prompt estimate */
  uint32_t slo;      /* SLO violation iff b > slo (strict); 16 = 200 ms at 12.5 ms/block */
  uint32_t threshold; /* TLRU_POLICY_THRESHOLD: admission threshold in blocks (1024 tokens = 8 blocks
                         of 128); ignored by the other policies */
} tlru_instance;

typedef struct { /* 72 B, all exact integers */
  uint64_t requests;       /* E of the instance's trace */
  uint64_t sum_uncached;   /* sum b */
  uint64_t tel_blocks;     /* sum max(b - xi, 0)  (Eq. 3) */
  uint64_t slo_violations; /* #{b > slo} */
  uint64_t evicted_trim;   /* blocks evicted by Phase 1 */
  uint64_t evicted_lru;    /* blocks evicted by Phase 2 */
  uint32_t p50, p90, p95, p99;            /* nearest-rank percentiles of b (Reading #11) */
  uint32_t max_uncached, max_occupancy;   /* max b; max sum X after a request (<= capacity) */
} tlru_result;

/* Host: workspace bytes for tlru_simulate_batch on these traces / instances. */
tlru_status tlru_sim_workspace_size(const tlru_trace* traces /*host[nt]*/, uint32_t nt,
                                    const tlru_instance* inst /*host[ni]*/, uint32_t ni,
                                    size_t* bytes /*host*/);

/* Simulate ni instances.  inst is a HOST array (the launch planner groups
 * instances by trace, engine and capacity class on the host).  uncached (device,
 * u16) receives instance i's per-request b at uncached[offsets[i] .. offsets[i] + E_i);
 * offsets is a host array, or NULL for packed offsets (prefix sums of E_i).
 * results (device[ni]) receives one tlru_result per instance.
 * Engine per instance: LRU / T-LRU / Threshold-LRU instances run on the engine
 * tlru_set_sim_engine selects (stack by default) -- except on a trace whose
 * universe_blocks >= 2^32 - 2^16 (the stack engine's 32-bit window sums), which runs
 * on the replay engine; every other policy runs on the replay engine.  A batch
 * that needs both engines runs both, each on its own instances (stats.engine =
 * TLRU_ENGINE_MIXED); the outputs are identical either way.
 * Unknown policy -> TLRU_EUNSUPPORTED; trace index out of range -> TLRU_EINVAL;
 * ET-LRU on a trace without real ticks (TLRU_TRACE_SYNTHETIC_TICKS) -> TLRU_EINVAL.
 * Does not synchronize.  A replay chain that outgrows its on-chip state is re-run
 * from global memory (counted in spilled_chains, never truncated); one that
 * outgrows even that is counted in failed_chains (its b rows are then invalid):
 * callers that cannot rule this out poll tlru_last_sim_stats (the Python binding's
 * simulate_batch does). */
tlru_status tlru_simulate_batch(const tlru_trace* traces /*host[nt]*/, uint32_t nt,
                                const tlru_instance* inst /*host[ni]*/, uint32_t ni, uint16_t* uncached,
                                const uint64_t* offsets /*host[ni] or NULL*/, tlru_result* results, void* ws,
                                size_t ws_bytes, cudaStream_t stream);

/* tlru_simulate_batch that also exports each instance's histogram of b (the one
 * the tail metrics of its tlru_result are computed from): hist (device,
 * nullable) receives row i = #{requests of instance i with b = v} for v = 0 ..
 * hist_bins - 1 at hist[i * hist_bins + v].  hist_bins must exceed every trace's
 * max_history (b <= J <= L_after), else TLRU_ERANGE; bins above the batch's
 * largest max_history are written as 0.  The workspace size is the same as
 * tlru_simulate_batch's.  Row sums fit u32 because E < 2^32. */
tlru_status tlru_simulate_batch_ex(const tlru_trace* traces /*host[nt]*/, uint32_t nt,
                                   const tlru_instance* inst /*host[ni]*/, uint32_t ni, uint16_t* uncached,
                                   const uint64_t* offsets /*host[ni] or NULL*/, tlru_result* results,
                                   uint32_t* hist /*device[ni][hist_bins] or NULL*/, uint32_t hist_bins,
                                   void* ws, size_t ws_bytes, cudaStream_t stream);

/* Tuning / test knobs for tlru_simulate_batch on this thread (host; 0 = automatic).
 * segment_events: events per segment (rounded up to a multiple of 32; the cache
 *   state at each segment start is rebuilt exactly, so results do not depend on it).
 * state_entries: per-chain on-chip state entries W (32, 64, 96, 128, 256, 512 or 1024); chains that
 *   outgrow it are re-run from global memory, so results do not depend on it. */
tlru_status tlru_set_sim_options(uint32_t segment_events, uint32_t state_entries);

/* ET-LRU model for the calling thread's later tlru_simulate_batch calls (Def. 1, P:261-275;
 * Reading #27).  mu_per_tick: belief decay rate per time tick (the trace's time_ticks unit,
 * microseconds for generated traces), finite and >= 0.  ln_surv: HOST array of K + 1 doubles,
 * ln P(Q >= k) for k = 0..K (copied; non-increasing, each <= 0, -inf allowed, no NaN) -> else
 * TLRU_EINVAL; K > 65535 -> TLRU_ERANGE.  A batch with ET-LRU instances and no model set ->
 * TLRU_EINVAL. */
tlru_status tlru_set_etlru_model(double mu_per_tick, const double* ln_surv /*host[K+1]*/, uint32_t K);

/* Engine of tlru_simulate_batch on this thread (host).  Both are exact and give
 * identical bytes (tests/test_gpu_parity.py):
 *   TLRU_ENGINE_REPLAY: K2 -- Alg. 1 replayed request by request, one lane per
 *     instance, per-chain recency state in shared memory, segments rebuilt exactly;
 *   TLRU_ENGINE_STACK: closed form of Alg. 1 from the stack property:
 *     per (trace, D) window sums, every capacity of a trace in one pass; the
 *     eviction counters by telescoping.  Default. */
enum { TLRU_ENGINE_REPLAY = 0, TLRU_ENGINE_STACK = 1, TLRU_ENGINE_MIXED = 2 /* stats only */ };
tlru_status tlru_set_sim_engine(uint32_t engine);

/* Statistics of the last tlru_simulate_batch on this thread.  Reads two device
 * counters from that call's workspace, so the workspace must not have been
 * reused; synchronizes the device. */
typedef struct {
  uint64_t chains;          /* instance x segment work units launched (32 lanes per warp) */
  uint64_t segment_events;  /* events per segment */
  uint64_t spilled_chains;  /* chains re-run with global-memory state (incl. End-/Length-Aware
                               segments re-run by the fix-up) */
  uint64_t failed_chains;   /* chains that overflowed even the global-memory state (must be 0) */
  uint32_t kernels;         /* kernel launches issued */
  uint32_t state_entries;   /* largest on-chip W used (replay engine) */
  uint32_t engine;          /* TLRU_ENGINE_* used */
  uint32_t reserved;
  float k2_ms;              /* device time of the simulation kernels (K2 + spill, or the stack engine;
                               MIXED: both engines and their K3) */
  float k3_ms;              /* device time of the tail-metric kernels (K3; 0 for MIXED) */
  float out_ms;             /* stack engine, fused path: device time from the first to the last
                               s2_out launch (b output + histograms, the dominant kernel); else 0 */
  uint32_t out_launches;    /* s2_out launches in that interval */
} tlru_sim_stats;
tlru_status tlru_last_sim_stats(tlru_sim_stats* out /*host*/);

/* ------------------------------------------------------------------------
 * Tail metrics over request segments (Eq. 1-3).
 * Segment s covers b[seg_offsets[s] .. seg_offsets[s+1]).
 *   TEL_blocks = sum max(b - xi, 0); TEL_ms = sum max(alpha*b - xi_ms, 0) (summed
 *   over b in ascending order, double); SLO = #{b > slo};
 *   p-th percentile: nearest rank k = max(1, ceil(p * n / 100)) on sorted b
 *   (integer arithmetic, p in {50, 90, 95, 99}; Reading #11); *_ms = alpha * b_(k).
 * An empty segment yields n = 0 and zero fields.  max_b (<= 65535) bounds the
 * histogram: a value of b above it makes the call return TLRU_ERANGE (the count
 * of such values is in n_clamped of the affected segments, whose other fields are
 * then unspecified) -- percentiles are never computed from truncated data.  For
 * that check tlru_tail_metrics synchronizes `stream`.
 * ------------------------------------------------------------------------ */
typedef struct {
  uint64_t n, tel_blocks, slo_violations, sum_b;
  uint32_t p50, p90, p95, p99;
  uint32_t max_b, n_clamped; /* n_clamped: values above max_b (0 whenever the call returns TLRU_OK) */
  double tel_ms, p50_ms, p90_ms, p95_ms, p99_ms, mean_ms;
} tlru_tail;

tlru_status tlru_tail_workspace_size(uint32_t ns, uint32_t max_b, size_t* bytes /*host*/);

tlru_status tlru_tail_metrics(const uint16_t* b, const uint64_t* seg_offsets /*device[ns+1]*/, uint32_t ns,
                              const uint32_t* xi /*device[ns]*/, const double* xi_ms /*device[ns]*/,
                              const uint32_t* slo /*device[ns]*/, double alpha_ms_per_block,
                              uint32_t max_b, tlru_tail* out /*device[ns]*/, void* ws, size_t ws_bytes,
                              cudaStream_t stream);

/* ------------------------------------------------------------------------
 * Pooled metrics (row a10; the paper reports percentiles of TTFT pooled over
 * the requests of a configuration): histograms of b are summed per
 * pool -- e.g. one pool per (C, xi, policy) over seeds -- on each GPU, summed
 * across GPUs by the caller's collective (NCCL all_reduce of the u64 counts), and
 * turned into tail metrics.  Sums of histograms are exact, so the pooled metrics
 * equal tlru_tail_metrics over the concatenated b of the pool's instances.
 * ------------------------------------------------------------------------ */

/* Host: workspace bytes of tlru_pool_histograms for ni instances. */
tlru_status tlru_pool_workspace_size(uint32_t ni, size_t* bytes /*host*/);

/* pooled[pool[i] * bins + v] += hist[i * bins + v] for every instance i with
 * pool[i] != TLRU_NONE (TLRU_NONE skips the instance).  pooled is accumulated into
 * (zero it first).  pool[i] >= npool (other than TLRU_NONE) -> TLRU_EINVAL. */
tlru_status tlru_pool_histograms(const uint32_t* hist /*device[ni][bins]*/, uint32_t ni, uint32_t bins,
                                 const uint32_t* pool /*host[ni]*/, uint32_t npool,
                                 uint64_t* pooled /*device[npool][bins]*/, void* ws, size_t ws_bytes,
                                 cudaStream_t stream);

/* Tail metrics of ns histograms (u64 counts, hist[s * bins + v] = #{b = v}) with the
 * definitions of tlru_tail_metrics (xi, xi_ms, slo nullable: 0, 0.0, "no SLO").
 * bins in 1..65536; n_clamped = 0.  No workspace; does not synchronize. */
tlru_status tlru_tail_from_histograms(const uint64_t* hist /*device[ns][bins]*/, uint32_t ns, uint32_t bins,
                                      const uint32_t* xi /*device[ns]*/, const double* xi_ms /*device[ns]*/,
                                      const uint32_t* slo /*device[ns]*/, double alpha_ms_per_block,
                                      tlru_tail* out /*device[ns]*/, cudaStream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* TLRU_H_ */
