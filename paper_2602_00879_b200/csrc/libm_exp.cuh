// fp64 exp bit-identical to the reference's std::exp.
//
// The reference computes every gate in fp64 with std::exp (gating.cpp:17-38),
// i.e. glibc's exp. On x86-64 glibc 2.39 (the image's libm.so.6, Ubuntu
// 2.39-0ubuntu8.5) dispatches exp through an ifunc to its FMA build on any
// host with FMA + AVX2 (every B200 host). That build is the Arm
// optimized-routines algorithm (glibc sysdeps/ieee754/dbl-64/e_exp.c, since
// 2.28):
//
//   exp(x) = 2^(k/N) * exp(r),  N = 128,  x = k ln2/N + r,  |r| <= ln2/2N
//   kd  = fma(x, N/ln2, 0x1.8p52)           (round-to-nearest k, in the low bits)
//   r   = fma(kd', -ln2hi/N, fma(kd', -ln2lo/N, ..))   kd' = kd - 0x1.8p52
//   tmp = tail[k mod N] + r + r^2 (C2 + r C3) + r^4 (C4 + r C5)
//   exp = scale + scale * tmp,  scale = 2^(k/N) as stored bits + (k << 45)
//
// restated here operation for operation, with the FMA contractions that
// build makes (read off its machine code: x*InvLn2N+Shift, both r steps, the
// two inner polynomial terms, the two outer terms and the final
// scale + scale*tmp are fused; r*r and r2*r2 are plain products) and its
// special cases: |x| < 2^-54 -> 1 + x; |x| >= 1024 -> 0 / inf / NaN;
// 512 <= |x| < 1024 -> the rescaled path, whose negative branch rounds into
// the subnormal range once (hi/lo split) exactly as glibc does. Every
// operation is an explicit __fma_rn / __dadd_rn / __dmul_rn so nvcc cannot
// contract or reassociate anything. With it the routing kernels' softmax
// and sigmoid gates, sums and renormalised gates are bit-identical to the
// reference's (tests/test_gpu_parity.py checks gates with atol = 0), and
// near-underflow ties (gates of 0 vs the smallest subnormal) order exactly
// as the reference orders them.
//
// The 2^(k/N) table is generated from first principles by
// tools/gen_exp_table.py (libm_exp_table.inc); the C restatement
// oracle/desmoe_oracle.c:or_glibc_exp is pinned against the host libm over
// every range (tests/test_oracle.py::test_glibc_exp_restatement).
#pragma once

#include <cstdint>

namespace desmoe {

// 2^(k/128) = H[k] (1 + T[k]): {bits(T[k]), bits(H[k]) - (k << 45)}
static __device__ __align__(16) const unsigned long long kExpTab[256] = {
#include "libm_exp_table.inc"
};

namespace libm_exp {
constexpr double kInvLn2N = 0x1.71547652b82fep+7;     // N / ln2
constexpr double kShift = 0x1.8p52;
constexpr double kNegLn2HiN = -0x1.62e42fefa0000p-8;  // -ln2/N, high part
constexpr double kNegLn2LoN = -0x1.cf79abc9e3b3ap-47; // -ln2/N, low part
constexpr double kC2 = 0x1.ffffffffffdbdp-2;
constexpr double kC3 = 0x1.555555555543cp-3;
constexpr double kC4 = 0x1.55555cf172b91p-5;
constexpr double kC5 = 0x1.1111167a4d017p-7;
}  // namespace libm_exp

// glibc exp of x; `tab` = kExpTab or a shared-memory copy of it.
__device__ __forceinline__ double glibc_exp(double x, const unsigned long long* tab) {
  using namespace libm_exp;
  const uint64_t ix = static_cast<uint64_t>(__double_as_longlong(x));
  uint32_t abstop = static_cast<uint32_t>(ix >> 52) & 0x7ffu;
  if (abstop - 0x3c9u >= 0x3fu) {
    if (static_cast<int>(abstop) - 0x3c9 < 0) return __dadd_rn(1.0, x);  // |x| < 2^-54
    if (abstop >= 0x409u) {                                                // |x| >= 1024
      if (ix == 0xfff0000000000000ull) return 0.0;                         // -inf
      if (abstop >= 0x7ffu) return __dadd_rn(1.0, x);                      // inf / NaN
      return (ix >> 63) ? 0.0 : __longlong_as_double(0x7ff0000000000000ll);  // under / overflow
    }
    abstop = 0;  // 512 <= |x| < 1024: the rescaled special case below
  }
  const double kd0 = __fma_rn(x, kInvLn2N, kShift);
  const uint64_t ki = static_cast<uint64_t>(__double_as_longlong(kd0));
  const double kd = __dsub_rn(kd0, kShift);
  double r = __fma_rn(kd, kNegLn2HiN, x);
  r = __fma_rn(kd, kNegLn2LoN, r);
  const uint32_t idx = 2u * static_cast<uint32_t>(ki & 127u);
  const uint64_t top = ki << 45;
  const double tail = __longlong_as_double(static_cast<long long>(tab[idx]));
  uint64_t sbits = tab[idx + 1] + top;
  const double r2 = __dmul_rn(r, r);
  const double p23 = __fma_rn(r, kC3, kC2);
  const double p45 = __fma_rn(r, kC5, kC4);
  double tmp = __fma_rn(p23, r2, __dadd_rn(r, tail));
  tmp = __fma_rn(__dmul_rn(r2, r2), p45, tmp);
  if (abstop != 0) {
    const double scale = __longlong_as_double(static_cast<long long>(sbits));
    return __fma_rn(scale, tmp, scale);
  }
  // specialcase (k outside the normal scale range)
  if ((ki & 0x80000000ull) == 0) {
    sbits -= 1009ull << 52;
    const double scale = __longlong_as_double(static_cast<long long>(sbits));
    return __dmul_rn(__fma_rn(scale, tmp, scale), 0x1p1009);
  }
  sbits += 1022ull << 52;
  const double scale = __longlong_as_double(static_cast<long long>(sbits));
  const double st = __dmul_rn(scale, tmp);
  double y = __dadd_rn(scale, st);
  if (y < 1.0) {
    // round y to its final precision once, before scaling into the
    // subnormal range (no double rounding)
    const double lo0 = __dadd_rn(__dsub_rn(scale, y), st);
    const double hi = __dadd_rn(y, 1.0);
    const double lo = __dadd_rn(__dadd_rn(__dsub_rn(1.0, hi), y), lo0);
    y = __dsub_rn(__dadd_rn(lo, hi), 1.0);
    if (y == 0.0) y = 0.0;  // no -0
  }
  return __dmul_rn(y, 0x1p-1022);
}

}  // namespace desmoe
