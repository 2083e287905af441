// nrmf_crhypot.cuh -- correctly rounded hypot, cr_hypot(a, b) = RN(sqrt(a^2 + b^2)),
// for the A-style top levels (the paper's recommended final
// reduction "Z with A"; A_x = R with cr_hypot).
//
// Exact integer method (no floating-point rounding anywhere before the final
// one): write the operands as integers A, B times powers of two, normalised
// to 53 (24) significant bits, form N = A^2 * 4^d + B^2 exactly in 256-bit
// arithmetic, take an integer square root of N scaled by an even power of two
// to 57-58 bits plus a sticky bit, and round once to nearest-even on the
// format's grid (subnormal quantum included).  Used only above the tile
// level (<= 1/4096 of the nodes), so clarity wins over speed.
//
// Specials (IEEE 754 hypot): +inf if either operand is infinite, else NaN if
// either is NaN; cr_hypot(x, 0) = |x|.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace nrmf {

template <typename F> struct CrFmt;
template <> struct CrFmt<double> {
  static constexpr int P = 53, EMIN = -1074, EMAXP1 = 1024, EBIAS = 1023, MBITS = 52;
  using U = unsigned long long;
};
template <> struct CrFmt<float> {
  static constexpr int P = 24, EMIN = -149, EMAXP1 = 128, EBIAS = 127, MBITS = 23;
  using U = unsigned int;
};

struct U256 {
  unsigned long long w[4];  // little endian
};

__device__ __forceinline__ int clz64(unsigned long long v) { return v ? __clzll(v) : 64; }

__device__ __forceinline__ int bitlen256(const U256& x) {
  for (int i = 3; i >= 0; --i)
    if (x.w[i]) return 64 * i + 64 - clz64(x.w[i]);
  return 0;
}

// x << s (s < 256), bits beyond 256 dropped (never happens here)
__device__ __forceinline__ U256 shl256(const U256& x, int s) {
  U256 r = {{0, 0, 0, 0}};
  const int q = s >> 6, o = s & 63;
  for (int i = 3; i >= 0; --i) {
    const int j = i - q;
    if (j < 0) continue;
    unsigned long long v = x.w[j] << o;
    if (o && j - 1 >= 0) v |= x.w[j - 1] >> (64 - o);
    r.w[i] = v;
  }
  return r;
}

// bits [lo, lo+128) of x as u128 (lo >= 0)
__device__ __forceinline__ unsigned __int128 bits128(const U256& x, int lo) {
  unsigned __int128 r = 0;
  for (int b = 0; b < 128; b += 64) {
    const int bit = lo + b, q = bit >> 6, o = bit & 63;
    unsigned long long v = 0;
    if (q < 4) {
      v = x.w[q] >> o;
      if (o && q + 1 < 4) v |= x.w[q + 1] << (64 - o);
    }
    r |= (unsigned __int128)v << b;
  }
  return r;
}

// any bit of x below position lo set?
__device__ __forceinline__ bool any_below(const U256& x, int lo) {
  for (int i = 0; i < 4; ++i) {
    const int b0 = 64 * i;
    if (b0 >= lo) break;
    const int nb = lo - b0;
    const unsigned long long m = nb >= 64 ? ~0ull : ((1ull << nb) - 1);
    if (x.w[i] & m) return true;
  }
  return false;
}

__device__ __forceinline__ unsigned __int128 isqrt128(unsigned __int128 v) {
  // floor(sqrt(v)) for v < 2^116: double estimate, then exact correction
  unsigned long long r = (unsigned long long)sqrt((double)v);
  while ((unsigned __int128)r * r > v) --r;
  while ((unsigned __int128)(r + 1) * (r + 1) <= v) ++r;
  return r;
}

template <typename F>
__device__ __noinline__ F cr_hypot(F a, F b) {
  using Fm = CrFmt<F>;
  using U = typename Fm::U;
  constexpr int P = Fm::P, MB = Fm::MBITS;
  if (isinf(a) || isinf(b)) return F(INFINITY);
  if (isnan(a) || isnan(b)) return F(NAN);
  // |.| and order by bit pattern (non-negative, non-NaN)
  U ua, ub;
  if constexpr (sizeof(F) == 8) {
    ua = (U)__double_as_longlong(a) & 0x7fffffffffffffffull;
    ub = (U)__double_as_longlong(b) & 0x7fffffffffffffffull;
  } else {
    ua = (U)__float_as_uint(a) & 0x7fffffffu;
    ub = (U)__float_as_uint(b) & 0x7fffffffu;
  }
  const U uM = ua > ub ? ua : ub, um = ua > ub ? ub : ua;
  if (uM == 0) return F(0);
  F Mv;
  if constexpr (sizeof(F) == 8) Mv = __longlong_as_double((long long)uM);
  else Mv = __uint_as_float((unsigned)uM);
  if (um == 0) return Mv;
  // integer significands normalised to P bits: value = sig * 2^e
  auto split = [](U u, unsigned long long& sig, int& e) {
    const int ef = (int)(u >> MB);
    unsigned long long s = (unsigned long long)(u & (((U)1 << MB) - 1));
    if (ef) {
      s |= 1ull << MB;
      e = ef - Fm::EBIAS - MB;
    } else {
      e = Fm::EMIN;
      while (!(s >> MB)) { s <<= 1; --e; }
    }
    sig = s;
  };
  unsigned long long A, B;
  int ea, eb;
  split(uM, A, ea);
  split(um, B, eb);
  const int d = ea - eb;  // >= 0 (M >= m, both normalised to P bits)
  // m < M * 2^(1-d): for d >= P + 7 the exact sqrt(M^2 + m^2) lies within
  // M * 2^(-2P-10) of M, far below half an ulp of M: the result is M
  if (d >= P + 7) return Mv;
  // N = A^2 * 4^d + B^2 (< 2^(2P + 2d) <= 2^(4P+12) <= 2^224), exact
  const unsigned __int128 A2 = (unsigned __int128)A * A, B2 = (unsigned __int128)B * B;
  U256 N = {{(unsigned long long)A2, (unsigned long long)(A2 >> 64), 0, 0}};
  N = shl256(N, 2 * d);
  {
    unsigned __int128 s = (unsigned __int128)N.w[0] + (unsigned long long)B2;
    N.w[0] = (unsigned long long)s;
    s = (unsigned __int128)N.w[1] + (unsigned long long)(B2 >> 64) + (unsigned long long)(s >> 64);
    N.w[1] = (unsigned long long)s;
    unsigned long long c = (unsigned long long)(s >> 64);
    for (int i = 2; i < 4 && c; ++i) {
      s = (unsigned __int128)N.w[i] + c;
      N.w[i] = (unsigned long long)s;
      c = (unsigned long long)(s >> 64);
    }
  }
  // sqrt(a^2 + b^2) = sqrt(N) * 2^eb.  Scale N by 4^-k to 114..115 bits.
  const int bl = bitlen256(N);
  int k = 0;
  while (bl - 2 * k > 115) ++k;
  while (bl - 2 * k < 114) --k;
  unsigned __int128 Np;
  bool sticky;
  if (k >= 0) {
    Np = bits128(N, 2 * k);
    sticky = any_below(N, 2 * k);
  } else {
    Np = bits128(N, 0) << (-2 * k);
    sticky = false;
  }
  const unsigned __int128 r = isqrt128(Np);
  if (r * r != Np) sticky = true;
  // sqrt(N) * 2^eb = (r + f) * 2^(k + eb), f in [0, 1), f > 0 iff sticky
  const unsigned long long r64 = (unsigned long long)r;  // 57..58 bits
  const int rb = 64 - __clzll(r64);
  const int base = k + eb;
  const int e = rb - 1 + base;              // value in [2^e, 2^(e+1))
  int qe = e - (P - 1);
  if (qe < Fm::EMIN) qe = Fm::EMIN;          // subnormal quantum
  const int dd = qe - base;                  // bits of r below the quantum (>= 1)
  unsigned long long mant = dd >= 64 ? 0 : (r64 >> dd);
  const bool guard = dd >= 1 && dd <= 64 && ((r64 >> (dd - 1)) & 1);
  const bool rest = (dd >= 2 && (r64 & ((dd - 1 >= 64) ? ~0ull : ((1ull << (dd - 1)) - 1)))) || sticky;
  if (guard && (rest || (mant & 1))) ++mant;
  if (mant >> P) {  // carried into a new binade
    mant >>= 1;
    ++qe;
  }
  // value = mant * 2^qe, mant < 2^P
  if (mant == 0) return F(0);
  const int top = 63 - __clzll(mant);       // exponent of the leading bit
  if (top + qe >= Fm::EMAXP1) return F(INFINITY);
  if constexpr (sizeof(F) == 8) {
    unsigned long long bits;
    if (mant >> (P - 1)) bits = ((unsigned long long)(qe + P - 1 + Fm::EBIAS) << MB) | (mant & ((1ull << MB) - 1));
    else bits = mant;  // subnormal: qe == EMIN
    return __longlong_as_double((long long)bits);
  } else {
    unsigned bits;
    if (mant >> (P - 1)) bits = ((unsigned)(qe + P - 1 + Fm::EBIAS) << MB) | (unsigned)(mant & ((1ull << MB) - 1));
    else bits = (unsigned)mant;
    return __uint_as_float(bits);
  }
}

}  // namespace nrmf
