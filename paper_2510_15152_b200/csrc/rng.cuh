// rng.cuh -- counter-based sampling for the synthetic-trace generator (K1).
//
// The generator spec (Reading #16) fixes every random
// value as a pure function of (seed, conversation, turn, attempt, lane):
//   Philox4x64-10, key = (seed, 0x544C52552D474E31 "TLRU-GN1"),
//   counter = (conv, turn, attempt, 0) -> four 64-bit lanes; attempt 0 of a turn gives
//   lane 0: the gap before the turn (turn 0: the birth gap), lanes 1, 2: the first polar pair,
//   lane 3: the death clock (turn 0); a rejected polar pair retries with attempt 1, 2, ...;
//   one accepted pair (v1, v2) gives both normals: prompt z = v1 f, response z = v2 f;
//   u = ((x >> 11) + 1) * 2^-53 in (0, 1];
//   ln / exp evaluated with a fixed sequence of correctly rounded IEEE double
//   operations (explicit __d*_rn intrinsics: no FMA contraction), so the
//   result does not depend on the math library;
//   Exp(rate) gaps in integer microsecond ticks floor(-ln(u) * (1e6 / rate));
//   standard normals by the Marsaglia polar method (attempt a = 0, 1, ...);
//   lognormal tokens exp(ln(mean) - sigma^2/2 + sigma z), rounded half up and clipped.
#pragma once

#include <stdint.h>

namespace tlru {

struct U64x4 {
  uint64_t v[4];
};

__device__ __forceinline__ U64x4 philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3, uint64_t k0,
                                               uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t m0 = 0xD2E7470EE14C6C93ull, m1 = 0xCA5A826395121157ull;
    uint64_t hi0 = __umul64hi(m0, c0), lo0 = m0 * c0;
    uint64_t hi1 = __umul64hi(m1, c2), lo1 = m1 * c2;
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ull;  // key schedule (bump after each round; the bump after the last is unused)
    k1 += 0xBB67AE8584CAA73Bull;
  }
  U64x4 out;
  out.v[0] = c0;
  out.v[1] = c1;
  out.v[2] = c2;
  out.v[3] = c3;
  return out;
}

__device__ __forceinline__ U64x4 turn_draw(uint64_t seed, uint64_t conv, uint64_t turn, uint64_t attempt) {
  return philox4x64_10(conv, turn, attempt, 0, seed, 0x544C52552D474E31ull);
}

__device__ __forceinline__ double unit_open0(uint64_t x) {  // (0, 1]
  return __dmul_rn(static_cast<double>((x >> 11) + 1ull), 1.0 / 9007199254740992.0);
}

// ln(x), x > 0 finite: x = m 2^e, m in [sqrt(1/2), sqrt(2)); ln m = 2 atanh((m-1)/(m+1)).
__device__ __forceinline__ double dln(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  long long bits = __double_as_longlong(x);
  int e = static_cast<int>((bits >> 52) & 0x7ff) - 1023;
  double m = __longlong_as_double((bits & 0x000FFFFFFFFFFFFFll) | 0x3FF0000000000000ll);
  if (m > 1.4142135623730951) {
    m = __dmul_rn(m, 0.5);
    e += 1;
  }
  double s = __ddiv_rn(__dsub_rn(m, 1.0), __dadd_rn(m, 1.0));
  double s2 = __dmul_rn(s, s);
  double p = 1.0 / 21.0;
  p = __dadd_rn(__dmul_rn(p, s2), 1.0 / 19.0);
  p = __dadd_rn(__dmul_rn(p, s2), 1.0 / 17.0);
  p = __dadd_rn(__dmul_rn(p, s2), 1.0 / 15.0);
  p = __dadd_rn(__dmul_rn(p, s2), 1.0 / 13.0);
  p = __dadd_rn(__dmul_rn(p, s2), 1.0 / 11.0);
  p = __dadd_rn(__dmul_rn(p, s2), 1.0 / 9.0);
  p = __dadd_rn(__dmul_rn(p, s2), 1.0 / 7.0);
  p = __dadd_rn(__dmul_rn(p, s2), 1.0 / 5.0);
  p = __dadd_rn(__dmul_rn(p, s2), 1.0 / 3.0);
  p = __dadd_rn(__dmul_rn(p, s2), 1.0);
  double lnm = __dmul_rn(__dmul_rn(2.0, s), p);
  double de = static_cast<double>(e);
  return __dadd_rn(__dmul_rn(de, ln2_hi), __dadd_rn(lnm, __dmul_rn(de, ln2_lo)));
}

// exp(y), |y| < 700: y = k ln2 + r, Taylor of exp(r) through r^13 in Horner form.
__device__ __forceinline__ double dexp(double y) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  double k = rint(__ddiv_rn(y, 0.6931471805599453));
  double r = __dsub_rn(__dsub_rn(y, __dmul_rn(k, ln2_hi)), __dmul_rn(k, ln2_lo));
  double p = 1.0 / 6227020800.0;
  p = __dadd_rn(__dmul_rn(p, r), 1.0 / 479001600.0);
  p = __dadd_rn(__dmul_rn(p, r), 1.0 / 39916800.0);
  p = __dadd_rn(__dmul_rn(p, r), 1.0 / 3628800.0);
  p = __dadd_rn(__dmul_rn(p, r), 1.0 / 362880.0);
  p = __dadd_rn(__dmul_rn(p, r), 1.0 / 40320.0);
  p = __dadd_rn(__dmul_rn(p, r), 1.0 / 5040.0);
  p = __dadd_rn(__dmul_rn(p, r), 1.0 / 720.0);
  p = __dadd_rn(__dmul_rn(p, r), 1.0 / 120.0);
  p = __dadd_rn(__dmul_rn(p, r), 1.0 / 24.0);
  p = __dadd_rn(__dmul_rn(p, r), 1.0 / 6.0);
  p = __dadd_rn(__dmul_rn(p, r), 0.5);
  p = __dadd_rn(__dmul_rn(p, r), 1.0);
  p = __dadd_rn(__dmul_rn(p, r), 1.0);
  return ldexp(p, static_cast<int>(k));
}

// Exp(rate) waiting time in integer microsecond ticks from one 64-bit lane.
__device__ __forceinline__ uint64_t exp_ticks_of(uint64_t x, double us_per_unit /* = 1e6 / rate */) {
  double u = unit_open0(x);
  double g = __dmul_rn(__dsub_rn(0.0, dln(u)), us_per_unit);
  return static_cast<uint64_t>(floor(g));
}

// Two standard normals of turn (conv, turn) by the Marsaglia polar method: lanes 1, 2 of the
// attempt-0 draw d0, then of attempts 1, 2, ... until accepted.
__device__ __forceinline__ void polar_pair(uint64_t seed, uint64_t conv, uint64_t turn, const U64x4& d0, double& z1,
                                           double& z2) {
  for (uint64_t att = 0; att < 64; ++att) {
    const U64x4 d = att == 0 ? d0 : turn_draw(seed, conv, turn, att);
    double v1 = __dsub_rn(__dmul_rn(2.0, unit_open0(d.v[1])), 1.0);
    double v2 = __dsub_rn(__dmul_rn(2.0, unit_open0(d.v[2])), 1.0);
    double s = __dadd_rn(__dmul_rn(v1, v1), __dmul_rn(v2, v2));
    if (s < 1.0 && s > 0.0) {
      double f = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, dln(s)), s));
      z1 = __dmul_rn(v1, f);
      z2 = __dmul_rn(v2, f);
      return;
    }
  }
  z1 = z2 = 0.0;
}

__device__ __forceinline__ uint32_t lognormal_tokens(double z, double ln_mean_minus_half_var, double sigma,
                                                     uint32_t lo, uint32_t hi) {
  double x = dexp(__dadd_rn(ln_mean_minus_half_var, __dmul_rn(sigma, z)));
  double t = floor(__dadd_rn(x, 0.5));
  if (t < static_cast<double>(lo)) t = static_cast<double>(lo);
  if (t > static_cast<double>(hi)) t = static_cast<double>(hi);
  return static_cast<uint32_t>(t);
}

// ln(mean) - sigma^2 / 2, evaluated in the fixed order of the spec.
__device__ __forceinline__ double lognormal_mu(double mean, double sigma) {
  return __dsub_rn(dln(mean), __dmul_rn(0.5, __dmul_rn(sigma, sigma)));
}

}  // namespace tlru
