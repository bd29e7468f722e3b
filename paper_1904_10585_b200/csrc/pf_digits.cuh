// pf_digits.cuh -- base-128 digit splitting of fp64 values for the exact int8 tensor-core
// products (pf_gemm_i8.cu: A and Y splits; pf_rebuild.cu: digits written by the PFAM update).
// See pf_gemm_i8.cu's header for the representation.
#pragma once
#include "pf_common.cuh"

namespace pf {
namespace i8 {

// Byte offset of digit slice s of A(row, col) in the tiled A8 layout the K1-i8 GEMM streams:
// [tile = row / 128][k-block = col / 64][slice s < S][row % 128][col % 64] -- every TMA box
// (one slice of one 128 x 64-byte tile) is a contiguous 8 KB block of HBM.
PF_DEV size_t a8_offset(int row, int col, int s, int KB, int S) {
  return ((((size_t)(row >> 7) * KB + (col >> 6)) * S + s) << 13) + ((row & 127) << 6) + (col & 63);
}
// exact power of two 2^k as a double (|k| <= 1022)
PF_DEV double pow2(int k) { return __longlong_as_double((long long)(1023 + k) << 52); }
// scale exponent E of a row / column with max |x| = m: |x| 2^-E < 1 (frexp), 0 for m == 0
PF_DEV int scale_exp(double m) {
  if (!(m > 0.0)) return 0;
  int e;
  frexp(m, &e);
  return max(-1000, min(1000, e));
}
// Digits of x relative to the scale 2^E (|x| < 2^E): U = floor(|x| 2^(7S-E)) (U < 2^7S, exact from
// the fp64 bit pattern with integer shifts) in base 128, every digit carrying the sign of x:
// d_s = sign(x) ((U >> 7(S-1-s)) & 127) in [-127, 127], so x = 2^E sum_s d_s 128^-(s+1) + r with
// |r| < 2^(E-7S) -- the truncating digit expansion d_s = trunc(128 r), r <- 128 r - d_s.
// Sign-symmetric digits keep the dropped low-order products (levels > S+1) unbiased; floor digits
// (all low digits >= 0) bias every dropped term the same way, an error growing like K instead of
// sqrt(K) (measured 1000x larger on Gaussian data).  Packed as bytes:
// wlo = (d_{S-1}, d_{S-2}, d_{S-3}, d_{S-4}), whi = (d_{S-5}, ..., d_0) (S - 4 bytes).
template <int S>
PF_DEV void digit_words(double x, int E, uint32_t& wlo, uint32_t& whi) {
  static_assert(S == 6 || S == 7, "S");
  const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
  const int be = (int)((bits >> 52) & 0x7ff);
  unsigned long long m = bits & 0xFFFFFFFFFFFFFull;
  int ex = -1074;                       // x = m 2^ex (subnormal / zero)
  if (be != 0) {
    m |= 1ull << 52;
    ex = be - 1075;
  }
  const int sh = (E - 7 * S) - ex;      // >= 4 since |x| < 2^E and 7S <= 49
  const unsigned long long U = (sh >= 64) ? 0ull : (m >> sh);
  const uint32_t lo = (uint32_t)U & 0x0FFFFFFFu;
  wlo = (lo & 0x7Fu) | ((lo << 1) & 0x7F00u) | ((lo << 2) & 0x7F0000u) | ((lo << 3) & 0x7F000000u);
  const uint32_t h = (uint32_t)(U >> 28);
  whi = (h & 0x7Fu) | ((h << 1) & 0x7F00u) | ((h << 2) & 0x7F0000u);
  if (bits >> 63) {  // negate every byte (no borrow between bytes)
    wlo = __vneg4(wlo);
    whi = __vneg4(whi);
  }
}
// The same digits with U formed in fp64: |x| 2^(7S-E) < 2^7S is exact (a power-of-two scale sc,
// no underflow that could reach 1), and adding 2^52 with round-toward-zero leaves trunc of it in
// the low 52 bits of the sum.  Two fp64 instructions + a funnel shift replace the exponent
// decode and the 64-bit variable shift.  Byte negation: -b = (0x80 - b) ^ 0x80 for b in [0, 127].
template <int S>
PF_DEV void digit_words_sc(double x, double sc, uint32_t& wlo, uint32_t& whi) {
  const double y = __dadd_rz(fabs(x) * sc, 4503599627370496.0);
  const unsigned long long b = (unsigned long long)__double_as_longlong(y);
  const uint32_t l32 = (uint32_t)b, h32 = (uint32_t)(b >> 32);
  // U bits 28..48 (bits 52.. of b hold y's exponent: masked below)
  const uint32_t h = __funnelshift_r(l32, h32, 28);
  // 7-bit groups to bytes in two steps: 14-bit halves to the two 16-bit lanes, then 7-bit
  // groups to the bytes of each lane (shift + LOP3 each; the same bytes as one mask per byte)
  const uint32_t tl = (l32 & 0x3FFFu) | ((l32 << 2) & 0x3FFF0000u);
  wlo = (tl & 0x007F007Fu) | ((tl << 1) & 0x7F007F00u);
  const uint32_t th = (h & 0x3FFFu) | ((h << 2) & 0x007F0000u);
  whi = (th & 0x007F007Fu) | ((th << 1) & 0x00007F00u);
  if (__double_as_longlong(x) < 0) {
    wlo = (0x80808080u - wlo) ^ 0x80808080u;
    whi = (0x80808080u - whi) ^ 0x80808080u;
  }
}
// 4 x 4 byte transpose: t[b] = (byte b of w0, w1, w2, w3)
PF_DEV void transpose4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t (&t)[4]) {
  const uint32_t a = __byte_perm(w0, w1, 0x5140), b = __byte_perm(w2, w3, 0x5140);
  const uint32_t c = __byte_perm(w0, w1, 0x7362), d = __byte_perm(w2, w3, 0x7362);
  t[0] = __byte_perm(a, b, 0x5410);
  t[1] = __byte_perm(a, b, 0x7632);
  t[2] = __byte_perm(c, d, 0x5410);
  t[3] = __byte_perm(c, d, 0x7632);
}
// digit slices of 4 consecutive values: out[s] = bytes (d_s(x0), d_s(x1), d_s(x2), d_s(x3))
template <int S>
PF_DEV void slices4(double x0, double x1, double x2, double x3, int E, uint32_t (&out)[S]) {
  uint32_t l[4], h[4], tl[4], th[4];
  if (E >= 7 * S - 1022) {  // 2^(7S-E) is a normal double: the fp64 form
    const double sc = pow2(7 * S - E);
    digit_words_sc<S>(x0, sc, l[0], h[0]);
    digit_words_sc<S>(x1, sc, l[1], h[1]);
    digit_words_sc<S>(x2, sc, l[2], h[2]);
    digit_words_sc<S>(x3, sc, l[3], h[3]);
  } else {
    digit_words<S>(x0, E, l[0], h[0]);
    digit_words<S>(x1, E, l[1], h[1]);
    digit_words<S>(x2, E, l[2], h[2]);
    digit_words<S>(x3, E, l[3], h[3]);
  }
  transpose4(l[0], l[1], l[2], l[3], tl);
  transpose4(h[0], h[1], h[2], h[3], th);
#pragma unroll
  for (int b = 0; b < 4; ++b) out[S - 1 - b] = tl[b];
#pragma unroll
  for (int b = 0; b < S - 4; ++b) out[S - 5 - b] = th[b];
}
// one value's digits (ragged tails)
template <int S>
PF_DEV int8_t digit(double x, int E, int s) {
  uint32_t lo, hi;
  digit_words<S>(x, E, lo, hi);
  const uint32_t w = (s >= S - 4) ? (lo >> (8 * (S - 1 - s))) : (hi >> (8 * (S - 5 - s)));
  return (int8_t)(w & 0xffu);
}

}  // namespace i8
}  // namespace pf
