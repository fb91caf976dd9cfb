/*
 * tlru_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded CPU oracle for the data-parallel hot path of
 * arXiv 2510.15152 "Tail-Optimized LRU" (T-LRU).  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product path (paper_2510_15152_b200/) never
 * links, imports or calls it; the two share no code, headers or constants.
 *
 * Citations: P:NNN = /root/reference/PAPER.md line NNN (section / equation /
 * algorithm).  "Reading #k" = DESIGN.md section "Readings of the paper", item k.
 *
 * Contents
 *   1. Philox4x64-10 counter-based RNG (Salmon et al. 2011), pinned in tests
 *      against numpy.random.Philox.
 *   2. Deterministic ln / exp written with IEEE basic operations only
 *      (compile with -ffp-contract=off), pinned against libm in tests.
 *   3. The paper's stochastic conversation model (Sec. 5) with the
 *      App. E timing recipe: synthetic trace generation.
 *   4. Trace derivation: J = L_before + q, L_after = J + a, prev links
 *      (Sec. 3 explicit TEL form).
 *   5. Alg. 1 replay (Sec. 4): LRU (Phase 2 only) and T-LRU
 *      (Phase 1 TEL-safe trimming then Phase 2 LRU); Threshold-LRU,
 *      End-/Length-Aware T-LRU, the hindsight Tail-Optimized
 *      Belady (Thm 1) and Expected-Tail-Optimized LRU (Def. 1,
 *      Alg. 2).
 *   6. Metrics: TTFT = alpha*b (Eq. 2), TEL (Eq. 1/3),
 *      nearest-rank percentiles (Reading #11), SLO count (strict >).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define ORACLE_NONE 0xFFFFFFFFu

/* ------------------------------------------------------------------------ */
/* 1. Philox4x64-10                                                          */
/* ------------------------------------------------------------------------ */
static void mulhilo64(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
    unsigned __int128 p = (unsigned __int128)a * (unsigned __int128)b;
    *hi = (uint64_t)(p >> 64);
    *lo = (uint64_t)p;
}

void oracle_philox4x64(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
    uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint64_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += 0x9E3779B97F4A7C15ull;
            k1 += 0xBB67AE8584CAA73Bull;
        }
        uint64_t hi0, lo0, hi1, lo1;
        mulhilo64(0xD2E7470EE14C6C93ull, c0, &hi0, &lo0);
        mulhilo64(0xCA5A826395121157ull, c2, &hi1, &lo1);
        uint64_t n0 = hi1 ^ c1 ^ k0;
        uint64_t n1 = lo1;
        uint64_t n2 = hi0 ^ c3 ^ k1;
        uint64_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Uniform in (0, 1]: ((x >> 11) + 1) * 2^-53 (Reading #16). */
double oracle_u01(uint64_t x) {
    return (double)((x >> 11) + 1) * (1.0 / 9007199254740992.0);
}

/* ------------------------------------------------------------------------ */
/* 2. Deterministic ln / exp (basic IEEE ops only)                           */
/* ------------------------------------------------------------------------ */
static const double LN2_HI = 6.93147180369123816490e-01; /* 0x3fe62e42fee00000 */
static const double LN2_LO = 1.90821492927058770002e-10; /* 0x3dea39ef35793c76 */

/* ln(x) for finite x > 0.  x = m * 2^e with m in [sqrt(1/2), sqrt(2));
   ln m = 2 atanh(s), s = (m-1)/(m+1), series to s^21. */
double oracle_det_ln(double x) {
    uint64_t bits;
    memcpy(&bits, &x, 8);
    int e = (int)((bits >> 52) & 0x7ff) - 1023;
    uint64_t mb = (bits & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull;
    double m;
    memcpy(&m, &mb, 8);
    if (m > 1.4142135623730951) { m = m * 0.5; e += 1; }
    double s = (m - 1.0) / (m + 1.0);
    double s2 = s * s;
    double p = 1.0 / 21.0;
    p = p * s2 + 1.0 / 19.0;
    p = p * s2 + 1.0 / 17.0;
    p = p * s2 + 1.0 / 15.0;
    p = p * s2 + 1.0 / 13.0;
    p = p * s2 + 1.0 / 11.0;
    p = p * s2 + 1.0 / 9.0;
    p = p * s2 + 1.0 / 7.0;
    p = p * s2 + 1.0 / 5.0;
    p = p * s2 + 1.0 / 3.0;
    p = p * s2 + 1.0;
    double lnm = 2.0 * s * p;
    double de = (double)e;
    return de * LN2_HI + (lnm + de * LN2_LO);
}

/* exp(y) for |y| < 700: y = k ln2 + r, |r| <= ln2/2, Taylor to r^13. */
double oracle_det_exp(double y) {
    double k = rint(y / 0.6931471805599453);
    double r = (y - k * LN2_HI) - k * LN2_LO;
    double p = 1.0 / 6227020800.0;        /* 1/13! */
    p = p * r + 1.0 / 479001600.0;        /* 1/12! */
    p = p * r + 1.0 / 39916800.0;         /* 1/11! */
    p = p * r + 1.0 / 3628800.0;          /* 1/10! */
    p = p * r + 1.0 / 362880.0;           /* 1/9!  */
    p = p * r + 1.0 / 40320.0;            /* 1/8!  */
    p = p * r + 1.0 / 5040.0;             /* 1/7!  */
    p = p * r + 1.0 / 720.0;              /* 1/6!  */
    p = p * r + 1.0 / 120.0;              /* 1/5!  */
    p = p * r + 1.0 / 24.0;               /* 1/4!  */
    p = p * r + 1.0 / 6.0;                /* 1/3!  */
    p = p * r + 0.5;                      /* 1/2!  */
    p = p * r + 1.0;
    p = p * r + 1.0;
    return ldexp(p, (int)k);
}

/* ------------------------------------------------------------------------ */
/* 3. Stochastic conversation model -> synthetic trace           */
/* ------------------------------------------------------------------------ */
typedef struct {
    uint64_t seed;
    uint32_t num_conversations;
    uint32_t block_tokens;
    double birth_rate, turn_rate, death_rate;                 /* lambda_conv, lambda_turn, mu */
    double prompt_mean_tokens, prompt_sigma_ln;               /* lognormal */
    double response_mean_tokens, response_sigma_ln;
    uint32_t prompt_min_tokens, prompt_max_tokens;
    uint32_t response_min_tokens, response_max_tokens;
    uint32_t max_history_blocks;                              /* L_max */
    uint32_t max_turns;
} oracle_gen_params;

static const uint64_t KEY_TAG = 0x544C52552D474E31ull; /* "TLRU-GN1" */

/* The random numbers of turn `turn` of conversation `conv` (Reading #16): Philox4x64-10 with
   counter (conv, turn, attempt, 0).  Attempt 0: o[0] = the gap before the turn (turn 0: the
   birth gap), o[1], o[2] = the first polar pair, o[3] = the death clock (turn 0); a rejected
   polar pair retries with attempt 1, 2, ... */
static void draw(uint64_t seed, uint64_t conv, uint64_t turn, uint64_t attempt, uint64_t out[4]) {
    uint64_t ctr[4] = {conv, turn, attempt, 0};
    uint64_t key[2] = {seed, KEY_TAG};
    oracle_philox4x64(ctr, key, out);
}

/* Exponential(rate) gap from one 64-bit draw, in integer microsecond ticks:
   floor(-ln(u) * (1e6/rate)). */
static uint64_t exp_ticks(uint64_t x, double rate) {
    double u = oracle_u01(x);
    double scale = 1000000.0 / rate;
    double g = (0.0 - oracle_det_ln(u)) * scale;
    return (uint64_t)floor(g);
}

/* Two standard normals by the Marsaglia polar method (one accepted pair gives both):
   the prompt's z1 = v1 f and the response's z2 = v2 f. */
static void std_normal_pair(uint64_t seed, uint64_t conv, uint64_t turn, double* z1, double* z2) {
    for (uint64_t a = 0; a < 64; ++a) {
        uint64_t o[4];
        draw(seed, conv, turn, a, o);
        double v1 = 2.0 * oracle_u01(o[1]) - 1.0;
        double v2 = 2.0 * oracle_u01(o[2]) - 1.0;
        double s = v1 * v1 + v2 * v2;
        if (s < 1.0 && s > 0.0) {
            double f = sqrt((-2.0 * oracle_det_ln(s)) / s);
            *z1 = v1 * f;
            *z2 = v2 * f;
            return;
        }
    }
    *z1 = *z2 = 0.0;
}

/* Lognormal token count with the given mean, clipped to [lo, hi], rounded half-up. */
static uint32_t lognormal_tokens(double z, double mean, double sigma, uint32_t lo, uint32_t hi) {
    double mu = oracle_det_ln(mean) - 0.5 * (sigma * sigma);
    double x = oracle_det_exp(mu + sigma * z);
    double t = floor(x + 0.5);
    if (t < (double)lo) t = (double)lo;
    if (t > (double)hi) t = (double)hi;
    return (uint32_t)t;
}

typedef struct {
    uint64_t t;
    uint32_t conv, turn, q, a, last;
} gen_event;

static int cmp_gen_event(const void* x, const void* y) {
    const gen_event* a = (const gen_event*)x;
    const gen_event* b = (const gen_event*)y;
    if (a->t != b->t) return a->t < b->t ? -1 : 1;
    if (a->conv != b->conv) return a->conv < b->conv ? -1 : 1;
    if (a->turn != b->turn) return a->turn < b->turn ? -1 : 1;
    return 0;
}

/* Generate the whole trace.  Returns the number of events E, or -1 on bad
   params / allocation failure.  On success *out points to malloc'ed arrays
   (event order): ticks[E] (u64), conv[E], q[E], a[E], is_last[E] (u32).
   Free with oracle_free. */
int64_t oracle_generate(const oracle_gen_params* p, uint64_t** ticks_out, uint32_t** conv_out,
                        uint32_t** q_out, uint32_t** a_out, uint32_t** last_out) {
    if (p->num_conversations == 0 || p->block_tokens == 0) return -1;
    if (!(p->birth_rate > 0) || !(p->turn_rate > 0) || !(p->death_rate > 0)) return -1;
    if (p->max_turns == 0 || p->max_history_blocks == 0) return -1;
    const uint32_t B = p->block_tokens;
    size_t cap = 1024, n = 0;
    gen_event* ev = (gen_event*)malloc(cap * sizeof(gen_event));
    if (!ev) return -1;
    uint64_t birth = 0;
    for (uint32_t c = 0; c < p->num_conversations; ++c) {
        uint64_t o0[4];
        draw(p->seed, c, 0, 0, o0);
        /* Births: Poisson(lambda_conv) process, gaps Exp(lambda_conv). */
        birth += exp_ticks(o0[0], p->birth_rate);
        /* Death clock Exp(mu). */
        uint64_t life = exp_ticks(o0[3], p->death_rate);
        uint64_t t = birth, elapsed = 0;
        uint32_t L = 0;
        for (uint32_t k = 0; k < p->max_turns; ++k) {
            if (k > 0) {
                /* While active, turns follow a Poisson(lambda_turn) process. */
                uint64_t o[4];
                draw(p->seed, c, k, 0, o);
                uint64_t gap = exp_ticks(o[0], p->turn_rate);
                elapsed += gap;
                if (elapsed >= life) break;
                t += gap;
            }
            /* Random prompt length Q and response length A per turn. */
            double zp, zr;
            std_normal_pair(p->seed, c, k, &zp, &zr);
            uint32_t ptok = lognormal_tokens(zp, p->prompt_mean_tokens, p->prompt_sigma_ln,
                                             p->prompt_min_tokens, p->prompt_max_tokens);
            uint32_t rtok = lognormal_tokens(zr, p->response_mean_tokens, p->response_sigma_ln,
                                             p->response_min_tokens, p->response_max_tokens);
            uint32_t q = (ptok + B - 1) / B;
            if (q < 1) q = 1;
            uint32_t a = (rtok + B - 1) / B;
            if ((uint64_t)L + q + a > p->max_history_blocks) break; /* context window end */
            L += q + a;
            if (n == cap) {
                cap *= 2;
                gen_event* nev = (gen_event*)realloc(ev, cap * sizeof(gen_event));
                if (!nev) { free(ev); return -1; }
                ev = nev;
            }
            ev[n].t = t; ev[n].conv = c; ev[n].turn = k; ev[n].q = q; ev[n].a = a; ev[n].last = 0;
            ++n;
        }
        if (n > 0 && ev[n - 1].conv == c) ev[n - 1].last = 1;
    }
    /* Global time order; ties by conversation id, then turn (Reading #9). */
    qsort(ev, n, sizeof(gen_event), cmp_gen_event);
    uint64_t* ticks = (uint64_t*)malloc((n ? n : 1) * 8);
    uint32_t* conv = (uint32_t*)malloc((n ? n : 1) * 4);
    uint32_t* q = (uint32_t*)malloc((n ? n : 1) * 4);
    uint32_t* a = (uint32_t*)malloc((n ? n : 1) * 4);
    uint32_t* last = (uint32_t*)malloc((n ? n : 1) * 4);
    if (!ticks || !conv || !q || !a || !last) {
        free(ev); free(ticks); free(conv); free(q); free(a); free(last);
        return -1;
    }
    for (size_t i = 0; i < n; ++i) {
        ticks[i] = ev[i].t; conv[i] = ev[i].conv; q[i] = ev[i].q; a[i] = ev[i].a; last[i] = ev[i].last;
    }
    free(ev);
    *ticks_out = ticks; *conv_out = conv; *q_out = q; *a_out = a; *last_out = last;
    return (int64_t)n;
}

void oracle_free(void* p) { free(p); }

/* ------------------------------------------------------------------------ */
/* Dense conversation index: distinct ids sorted, then binary search.        */
/* ------------------------------------------------------------------------ */
static int cmp_u32(const void* x, const void* y) {
    uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
    return a < b ? -1 : (a > b ? 1 : 0);
}

/* Writes dense[E]; returns number of distinct conversations, or -1. */
static int64_t densify(const uint32_t* conv, uint64_t E, uint32_t* dense) {
    uint32_t* ids = (uint32_t*)malloc((E ? E : 1) * 4);
    if (!ids) return -1;
    memcpy(ids, conv, E * 4);
    qsort(ids, E, 4, cmp_u32);
    uint64_t n = 0;
    for (uint64_t i = 0; i < E; ++i)
        if (i == 0 || ids[i] != ids[n - 1]) ids[n++] = ids[i];
    for (uint64_t e = 0; e < E; ++e) {
        uint64_t lo = 0, hi = n;
        while (hi - lo > 1) {
            uint64_t mid = (lo + hi) / 2;
            if (ids[mid] <= conv[e]) lo = mid; else hi = mid;
        }
        dense[e] = (uint32_t)lo;
    }
    free(ids);
    return (int64_t)n;
}

/* ------------------------------------------------------------------------ */
/* 4. Trace derivation: J = L_before + q, L_after = J + a, prev. */
/* ------------------------------------------------------------------------ */
int oracle_derive(const uint32_t* conv, const uint32_t* q, const uint32_t* a, uint64_t E,
                  uint32_t* prev, uint64_t* J, uint64_t* L_after, uint32_t* next) {
    uint32_t* dense = (uint32_t*)malloc((E ? E : 1) * 4);
    if (!dense) return -1;
    int64_t n = densify(conv, E, dense);
    if (n < 0) { free(dense); return -1; }
    uint64_t* L = (uint64_t*)calloc((size_t)(n ? n : 1), 8);
    uint32_t* last = (uint32_t*)malloc((size_t)(n ? n : 1) * 4);
    if (!L || !last) { free(dense); free(L); free(last); return -1; }
    for (int64_t i = 0; i < n; ++i) last[i] = ORACLE_NONE;
    for (uint64_t e = 0; e < E; ++e) {
        uint32_t c = dense[e];
        prev[e] = last[c];
        if (next) {
            next[e] = ORACLE_NONE;
            if (last[c] != ORACLE_NONE) next[last[c]] = (uint32_t)e;
        }
        J[e] = L[c] + q[e];
        L_after[e] = J[e] + a[e];
        L[c] = L_after[e];
        last[c] = (uint32_t)e;
    }
    free(dense); free(L); free(last);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* 5. Alg. 1 replay                                                          */
/* ------------------------------------------------------------------------ */
/* Per-conversation state: X = cached blocks, L = history length,
   tau = timestamp of last turn (event index), surplus = blocks above the
   TEL-safe budget still cached ("free", marked infinitely old).
   Two intrusive doubly-linked lists in ascending tau: `res` holds every
   conversation with X > 0 (Phase 2 scans it), `fre` holds every conversation
   with surplus > 0 (Phase 1 scans it).  An arrival moves theta to both tails
   because it receives the newest tau. */
typedef struct {
    uint64_t X, L, surplus;
    uint64_t tau;
    int64_t res_prev, res_next, fre_prev, fre_next;
    int in_res, in_fre;
} conv_state;

typedef struct {
    int64_t head, tail;
} list_ends;

#define RES 0
#define FRE 1

static void list_remove(conv_state* s, list_ends* l, int which, int64_t i) {
    int64_t pv = which == RES ? s[i].res_prev : s[i].fre_prev;
    int64_t nx = which == RES ? s[i].res_next : s[i].fre_next;
    if (pv >= 0) { if (which == RES) s[pv].res_next = nx; else s[pv].fre_next = nx; }
    else l->head = nx;
    if (nx >= 0) { if (which == RES) s[nx].res_prev = pv; else s[nx].fre_prev = pv; }
    else l->tail = pv;
    if (which == RES) s[i].in_res = 0; else s[i].in_fre = 0;
}

static void list_push_tail(conv_state* s, list_ends* l, int which, int64_t i) {
    if (which == RES) { s[i].res_prev = l->tail; s[i].res_next = -1; s[i].in_res = 1; }
    else { s[i].fre_prev = l->tail; s[i].fre_next = -1; s[i].in_fre = 1; }
    if (l->tail >= 0) { if (which == RES) s[l->tail].res_next = i; else s[l->tail].fre_next = i; }
    else l->head = i;
    l->tail = i;
}

/* Tail-Optimized Belady (Thm 1; its proof App. A), the hindsight
   policy: clairvoyant, it knows each conversation's next arrival and next prompt length
   from the trace.  Reading #26: on arrival theta caches its whole history (optional caching,
   as Alg. 1, Reading #7); only on overflow and only as much as needed (Reading #8):
   Phase 1 trims blocks above each conversation's exact TEL-safe budget
   (L + q_next - xi)^+ (budget 0 for a conversation that never returns),
   furthest next arrival first; Phase 2 evicts from the conversation "whose next requests
   are expected to arrive furthest in the future", partial, tail blocks first.
   Written plainly: the resident conversations live in an unordered array and every
   eviction step scans it for the maximum next arrival (never-returning = +infinity; ties
   among those by lower conversation id, SPEC S:248 -- unobservable: they never return
   and are all free).  Counters as oracle_replay (Phase 1 -> evicted_trim). */
/* forced != 0: Tail-Optimized Belady under forced caching (App. C: "Theorem 1
   continues to hold" with constraint (3) as an equality), Reading #29: the post-decision state
   holds theta's whole history, so theta takes no part in either phase; only if the other
   conversations cannot make room (theta alone exceeds C) does theta lose its tail blocks --
   above-budget blocks first, they are the tail -- counted with the Phase-2 evictions (as forced
   T-LRU, Reading #28). */
static int replay_tail_belady(const uint32_t* dense, int64_t n, const uint32_t* q, const uint32_t* a,
                              const uint64_t* nxt, uint64_t E, uint64_t C, uint64_t xi, int forced,
                              uint64_t* b_out, uint64_t* counters_out) {
    uint64_t* X = (uint64_t*)calloc((size_t)(n ? n : 1), 8);   /* cached blocks x_i */
    uint64_t* L = (uint64_t*)calloc((size_t)(n ? n : 1), 8);   /* history length L_i */
    uint64_t* sur = (uint64_t*)calloc((size_t)(n ? n : 1), 8); /* blocks above the budget */
    uint64_t* nx = (uint64_t*)calloc((size_t)(n ? n : 1), 8);  /* next arrival (UINT64_MAX: never) */
    int64_t* res = (int64_t*)malloc((size_t)(n ? n : 1) * 8);  /* resident conversations */
    unsigned char* in_res = (unsigned char*)calloc((size_t)(n ? n : 1), 1);
    if (!X || !L || !sur || !nx || !res || !in_res) {
        free(X); free(L); free(sur); free(nx); free(res); free(in_res);
        return -1;
    }
    int64_t nres = 0;
    uint64_t used = 0, ev_trim = 0, ev_far = 0, max_occ = 0;
    for (uint64_t t = 0; t < E; ++t) {
        int64_t c = dense[t];
        uint64_t J = L[c] + q[t];
        b_out[t] = J - X[c];                         /* job - x */
        uint64_t L_after = J + a[t];
        used = used - X[c] + L_after;                /* X_theta <- L_theta (Reading #7) */
        X[c] = L_after;
        L[c] = L_after;
        nx[c] = nxt[t];
        /* exact TEL-safe budget: (L + q_next - xi)^+, 0 if theta never returns */
        uint64_t budget = 0;
        if (nxt[t] != (uint64_t)-1) {
            uint64_t need = L_after + q[nxt[t]];
            budget = need > xi ? need - xi : 0;
        }
        sur[c] = L_after > budget ? L_after - budget : 0;
        if (!in_res[c] && X[c] > 0) { res[nres++] = c; in_res[c] = 1; }
        if (used > C) {
            uint64_t over = used - C;
            for (int phase = 1; phase <= 2 && over > 0; ++phase) {
                while (over > 0) {
                    /* the resident conversation with the furthest next arrival that still
                       has evictable blocks (Phase 1: blocks above its budget) */
                    int64_t best = -1;
                    for (int64_t k = 0; k < nres; ++k) {
                        int64_t i = res[k];
                        if (forced && i == c) continue;   /* theta is kept whole */
                        uint64_t avail = phase == 1 ? sur[i] : X[i];
                        if (avail == 0) continue;
                        if (best < 0 || nx[i] > nx[best] || (nx[i] == nx[best] && i < best)) best = i;
                    }
                    if (best < 0) break;
                    uint64_t avail = phase == 1 ? sur[best] : X[best];
                    uint64_t k = avail < over ? avail : over;
                    X[best] -= k;
                    if (phase == 1) { sur[best] -= k; ev_trim += k; } else { ev_far += k; }
                    used -= k;
                    over -= k;
                }
            }
            if (forced && over > 0) {   /* theta alone exceeds C: its tail blocks go */
                uint64_t k = over;
                X[c] -= k;
                sur[c] -= sur[c] < k ? sur[c] : k;
                used -= k;
                over = 0;
                ev_far += k;
            }
            /* drop conversations left with no cached block from the resident array */
            int64_t w = 0;
            for (int64_t k = 0; k < nres; ++k) {
                if (X[res[k]] > 0) res[w++] = res[k];
                else in_res[res[k]] = 0;
            }
            nres = w;
        }
        if (used > max_occ) max_occ = used;
    }
    counters_out[0] = ev_trim;
    counters_out[1] = ev_far;
    counters_out[2] = max_occ;
    free(X); free(L); free(sur); free(nx); free(res); free(in_res);
    return 0;
}

/* policy: 0 = LRU, 1 = T-LRU, 2 = Threshold-LRU (LRU that caches a
   conversation's history only when its length reaches `threshold` blocks; below it
   nothing is cached -- Reading #23: L_after >= threshold), 3 = End-Aware T-LRU and
   4 = Length-Aware T-LRU (with future knowledge taken from the trace itself:
   a conversation's terminating turn releases all its blocks instead of caching its
   history (Reading #24); Length-Aware also budgets with the true next prompt length,
   surplus = min(L, max(xi - q_next, 0)) (Reading #25)).  b_out[E] receives the
   uncached blocks of each request (u64).  counters_out[3] = {evicted_trim,
   evicted_lru, max_occupancy}; released blocks are not evictions.  5 = Tail-Optimized
   Belady (Thm 1, replay_tail_belady above; evicted_lru counts its Phase-2
   furthest-in-future evictions).  7 = T-LRU under forced caching (App. C, Reading #28).
   8 = Tail-Optimized Belady under forced caching (App. C, Reading #29).
   Returns 0, or -1 on allocation failure. */
int oracle_replay(const uint32_t* conv, const uint32_t* q, const uint32_t* a, uint64_t E,
                  int policy, uint64_t C, uint64_t xi, uint64_t q_hat, uint64_t threshold,
                  uint64_t* b_out, uint64_t* counters_out) {
    uint32_t* dense = (uint32_t*)malloc((E ? E : 1) * 4);
    if (!dense) return -1;
    int64_t n = densify(conv, E, dense);
    if (n < 0) { free(dense); return -1; }
    conv_state* s = (conv_state*)calloc((size_t)(n ? n : 1), sizeof(conv_state));
    if (!s) { free(dense); return -1; }
    /* next turn of the same conversation (End-/Length-Aware knowledge, from the trace) */
    uint64_t* nxt = (uint64_t*)malloc((E ? E : 1) * 8);
    int64_t* seen = (int64_t*)malloc((size_t)(n ? n : 1) * 8);
    if (!nxt || !seen) { free(dense); free(s); free(nxt); free(seen); return -1; }
    for (int64_t i = 0; i < n; ++i) seen[i] = -1;
    for (uint64_t t = E; t-- > 0;) {
        nxt[t] = seen[dense[t]] < 0 ? (uint64_t)-1 : (uint64_t)seen[dense[t]];
        seen[dense[t]] = (int64_t)t;
    }
    free(seen);
    if (policy == 5 || policy == 8) {  /* Tail-Optimized Belady (Thm 1); 8: under forced caching */
        int rc = replay_tail_belady(dense, n, q, a, nxt, E, C, xi, policy == 8, b_out, counters_out);
        free(s);
        free(dense);
        free(nxt);
        return rc;
    }
    list_ends res = {-1, -1}, fre = {-1, -1};
    /* Free tail per conversation D = max(xi - q_hat, 0): the blocks at the end
       of the history beyond the TEL-safe budget L + Q_hat - xi (P:56, P:62
       footnote; Readings #2, #4, #6).  LRU has no free blocks. */
    uint64_t D = 0;
    if ((policy == 1 || policy == 3 || policy == 7) && xi > q_hat) D = xi - q_hat;
    /* policy 7: T-LRU under forced caching (App. C; Reading #28): the post-decision
       state must hold theta's whole history (constraint (3) with equality), so Phases 1 and 2
       skip theta; only if theta alone exceeds C does it lose tail blocks (capacity first). */
    const int forced = policy == 7;
    uint64_t used = 0, ev_trim = 0, ev_lru = 0, max_occ = 0;
    for (uint64_t t = 0; t < E; ++t) {
        int64_t c = dense[t];
        /* Uncached blocks of the request: job - x = L + q - X. */
        uint64_t J = s[c].L + q[t];
        b_out[t] = J - s[c].X;
        /* Alg. 1 line 1: L_theta <- L', X_theta <- L_theta, tau_theta <- now.
           Optional caching caches the whole history incl. the response (Reading #7). */
        uint64_t L_after = J + a[t];
        if (policy == 2 && L_after < threshold) {
            /* Threshold-LRU below the threshold: the history is not cached at all.  L
               never decreases, so this conversation was never admitted: X = 0, b = J. */
            s[c].L = L_after;
            continue;
        }
        if ((policy == 3 || policy == 4) && nxt[t] == (uint64_t)-1) {
            /* terminating turn (End-/Length-Aware): "evicts all blocks from
               terminating conversations" -- the history is not cached and the blocks
               theta held are released (Reading #24) */
            used -= s[c].X;
            s[c].X = 0;
            s[c].surplus = 0;
            s[c].L = L_after;
            if (s[c].in_res) list_remove(s, &res, RES, c);
            if (s[c].in_fre) list_remove(s, &fre, FRE, c);
            continue;
        }
        uint64_t Dt = D;
        if (policy == 4) {  /* budget with the true next prompt q_next (Reading #25) */
            uint64_t qn = q[nxt[t]];
            Dt = xi > qn ? xi - qn : 0;
        }
        used = used - s[c].X + L_after;
        s[c].X = L_after;
        s[c].L = L_after;
        s[c].tau = t;
        s[c].surplus = L_after < Dt ? L_after : Dt;
        if (s[c].in_res) list_remove(s, &res, RES, c);
        list_push_tail(s, &res, RES, c);
        if (s[c].in_fre) list_remove(s, &fre, FRE, c);
        if (s[c].surplus > 0) list_push_tail(s, &fre, FRE, c);
        if (used > C) {                          /* Alg. 1 line 2 */
            uint64_t over = used - C;
            /* Phase 1, TEL-safe trimming: evict free blocks,
               ascending tau, theta last, bulk (Readings #1, #3, #5). */
            int64_t i = fre.head;
            while (over > 0 && i >= 0) {
                int64_t nx = s[i].fre_next;
                if (forced && i == c) { i = nx; continue; }   /* theta is kept whole */
                uint64_t k = s[i].surplus < over ? s[i].surplus : over;
                s[i].X -= k; s[i].surplus -= k; used -= k; over -= k; ev_trim += k;
                if (s[i].surplus == 0) list_remove(s, &fre, FRE, i);
                if (s[i].X == 0) list_remove(s, &res, RES, i);
                i = nx;
            }
            /* Phase 2, LRU: evict from argmin tau, partial (Reading #10).
               Reached only with the free list exhausted, so every surplus is 0 here. */
            i = res.head;
            while (over > 0 && i >= 0) {
                int64_t nx = s[i].res_next;
                if (forced && i == c) { i = nx; continue; }
                uint64_t k = s[i].X < over ? s[i].X : over;
                s[i].X -= k; used -= k; over -= k; ev_lru += k;
                if (s[i].X == 0) list_remove(s, &res, RES, i);
                i = nx;
            }
            if (forced && over > 0) {
                /* theta alone exceeds C: its tail blocks go (free ones first, they are the tail) */
                uint64_t k = over;
                s[c].X -= k; used -= k; over = 0; ev_lru += k;
                uint64_t ks = s[c].surplus < k ? s[c].surplus : k;
                s[c].surplus -= ks;
                if (s[c].surplus == 0 && s[c].in_fre) list_remove(s, &fre, FRE, c);
                if (s[c].X == 0) list_remove(s, &res, RES, c);
            }
        }
        if (used > max_occ) max_occ = used;
    }
    counters_out[0] = ev_trim;
    counters_out[1] = ev_lru;
    counters_out[2] = max_occ;
    free(s);
    free(dense);
    free(nxt);
    return 0;
}

/* Expected-Tail-Optimized LRU (Def. 1; greedy Alg. 2), literal:
   after serving theta (L_theta += Q + A, X_theta <- L_theta, lambda_theta <- lambda-bar),
   evict n = overflow blocks one at a time from the conversation with the minimum ranking
   criterion v_i = lambda_i * P(L_i + Q_i - xi >= X_i), re-scoring after every block.
   Reading #27: homogeneous lambda-bar (it cancels) and belief lambda_i = exp(-mu (t - tau_i))
   (P:255), so argmin v_i = argmin of ln v_i + mu t = mu * time_i + ln P(Q >= X_i - L_i + xi),
   evaluated as (double)ticks_i * mu_tick + ln_surv[k] (one IEEE multiply, one add; ticks in
   microseconds, mu_tick = mu per tick); ln_surv[k] = ln P(Q >= k) is the caller's table for
   k = 0..K (k <= 0 -> ln 1 = 0, k > K -> -inf: the block is TEL-safe); ties -> older last
   turn first (then the same conversation's tail block).  evicted_trim counts blocks evicted
   with P = 0 (-inf), evicted_lru the others.  time_i = the tick of conversation i's last turn. */
/* forced != 0: ET-LRU under forced caching (App. C: decision space X_F with
   Y_theta = L -- theta's whole history stays; Reading #30): theta is not a candidate of the
   greedy while serving its own turn; if no other block is left and the cache still exceeds C
   (theta alone holds more than C), theta loses the excess from its tail, counted with the
   P > 0 evictions (evicted_lru, as forced T-LRU, Reading #28). */
int oracle_replay_etlru(const uint32_t* conv, const uint32_t* q, const uint32_t* a, const uint64_t* ticks,
                        uint64_t E, uint64_t C, uint64_t xi, double mu_tick, const double* ln_surv,
                        uint64_t K, int forced, uint64_t* b_out, uint64_t* counters_out) {
    uint32_t* dense = (uint32_t*)malloc((E ? E : 1) * 4);
    if (!dense) return -1;
    int64_t n = densify(conv, E, dense);
    if (n < 0) { free(dense); return -1; }
    uint64_t* X = (uint64_t*)calloc((size_t)(n ? n : 1), 8);
    uint64_t* L = (uint64_t*)calloc((size_t)(n ? n : 1), 8);
    uint64_t* tau = (uint64_t*)calloc((size_t)(n ? n : 1), 8);
    int64_t* res = (int64_t*)malloc((size_t)(n ? n : 1) * 8);
    unsigned char* in_res = (unsigned char*)calloc((size_t)(n ? n : 1), 1);
    if (!X || !L || !tau || !res || !in_res) {
        free(dense); free(X); free(L); free(tau); free(res); free(in_res);
        return -1;
    }
    const double NEG_INF = -1.0 / 0.0;
    int64_t nres = 0;
    uint64_t used = 0, ev_free = 0, ev_other = 0, max_occ = 0;
    for (uint64_t t = 0; t < E; ++t) {
        int64_t c = dense[t];
        uint64_t J = L[c] + q[t];
        b_out[t] = J - X[c];                         /* job - x */
        L[c] = J + a[t];                             /* Alg. 2 line 2 */
        used = used - X[c] + L[c];
        X[c] = L[c];                                 /* Alg. 2 line 3 */
        tau[c] = t;                                  /* line 4: lambda_theta <- lambda-bar */
        if (!in_res[c] && X[c] > 0) { res[nres++] = c; in_res[c] = 1; }
        while (used > C) {                           /* lines 8-12: one block per iteration */
            int64_t best = -1;
            double best_v = 0.0, best_lg = 0.0;
            for (int64_t k = 0; k < nres; ++k) {
                int64_t i = res[k];
                if (X[i] == 0) continue;
                if (forced && i == c) continue;          /* Y_theta = L (App. C) */
                /* P(L_i + Q_i - xi >= X_i) = P(Q_i >= X_i - L_i + xi) */
                int64_t kk = (int64_t)X[i] - (int64_t)L[i] + (int64_t)xi;
                double lg = kk <= 0 ? 0.0 : ((uint64_t)kk > K ? NEG_INF : ln_surv[kk]);
                double v = (double)ticks[tau[i]] * mu_tick + lg;
                if (best < 0 || v < best_v || (v == best_v && tau[i] < tau[best])) {
                    best = i; best_v = v; best_lg = lg;
                }
            }
            if (best < 0) {                             /* forced: theta alone exceeds C */
                uint64_t k = used - C;
                X[c] -= k;
                used = C;
                ev_other += k;
                break;
            }
            X[best] -= 1;
            used -= 1;
            if (best_lg == NEG_INF) ev_free += 1; else ev_other += 1;
        }
        int64_t w = 0;
        for (int64_t k = 0; k < nres; ++k) {
            if (X[res[k]] > 0) res[w++] = res[k];
            else in_res[res[k]] = 0;
        }
        nres = w;
        if (used > max_occ) max_occ = used;
    }
    counters_out[0] = ev_free;
    counters_out[1] = ev_other;
    counters_out[2] = max_occ;
    free(dense); free(X); free(L); free(tau); free(res); free(in_res);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* 6. Metrics                                                                 */
/* ------------------------------------------------------------------------ */
static int cmp_u64(const void* x, const void* y) {
    uint64_t a = *(const uint64_t*)x, b = *(const uint64_t*)y;
    return a < b ? -1 : (a > b ? 1 : 0);
}

/* Tail metrics of one segment of per-request uncached counts b[n].
   ints_out[8]  = {n, tel_blocks, slo_violations, sum_b, p50, p90, p95, p99}
   dbls_out[6]  = {tel_ms, p50_ms, p90_ms, p95_ms, p99_ms, mean_ms}
   TEL_blocks = sum max(b - xi, 0) (Eq. 3); TEL_ms = sum max(alpha*b - xi_ms, 0)
   (Eq. 1) summed over b in ascending order; SLO = #{b > slo};
   percentile p: nearest rank k = max(1, ceil(p_bp * n / 10000)) on sorted b
   (Reading #11); ms values = alpha * b (Eq. 2).  n = 0 gives zeros. */
int oracle_tail(const uint64_t* b, uint64_t n, uint64_t xi, double xi_ms, uint64_t slo,
                double alpha, uint64_t* ints_out, double* dbls_out) {
    memset(ints_out, 0, 8 * sizeof(uint64_t));
    memset(dbls_out, 0, 6 * sizeof(double));
    ints_out[0] = n;
    if (n == 0) return 0;
    uint64_t* s = (uint64_t*)malloc(n * 8);
    if (!s) return -1;
    memcpy(s, b, n * 8);
    qsort(s, n, 8, cmp_u64);
    uint64_t tel = 0, slo_n = 0, sum = 0;
    double tel_ms = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        if (s[i] > xi) tel += s[i] - xi;
        if (s[i] > slo) slo_n += 1;
        sum += s[i];
        double ttft = alpha * (double)s[i];
        if (ttft > xi_ms) tel_ms += ttft - xi_ms;
    }
    static const uint64_t pbp[4] = {5000, 9000, 9500, 9900};
    ints_out[1] = tel; ints_out[2] = slo_n; ints_out[3] = sum;
    dbls_out[0] = tel_ms;
    for (int j = 0; j < 4; ++j) {
        uint64_t k = (pbp[j] * n + 9999) / 10000;
        if (k < 1) k = 1;
        ints_out[4 + j] = s[k - 1];
        dbls_out[1 + j] = alpha * (double)s[k - 1];
    }
    dbls_out[5] = alpha * (double)sum / (double)n;
    free(s);
    return 0;
}
