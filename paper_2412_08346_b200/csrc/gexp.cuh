// exp() restated from glibc's double-precision exp
// (sysdeps/ieee754/dbl-64/e_exp.c, used by the reference's std::exp inside
// rbf_kernel, optim.cpp:123) so the SVGD kernel values are bit-identical.
//
// exp(x) = 2^(k/N) * exp(r), N = 128, x = k ln2/N + r, |r| <= ln2/(2N);
// exp(r) - 1 ~ r + C2 r^2 + C3 r^3 + C4 r^4 + C5 r^5 evaluated with the same
// fused multiply-adds gcc emits for the x86-64 FMA variant.  The 2^(i/N)
// table is generated (tools/gen_exp_table.py); the four polynomial
// coefficients and the reduction constants are glibc's.  The |x| >= 512
// branch (results below 2^-738 or above 2^738) follows the same structure and
// is not guaranteed to match in the last ulp there; such terms are far below
// the resolution of every sum they enter.
#pragma once

#include "exp_table.cuh"

#include <cstdint>
#include <cstring>

namespace asicp {

__host__ __device__ __forceinline__ double u2d(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(u));
#else
  double d;
  std::memcpy(&d, &u, 8);
  return d;
#endif
}
__host__ __device__ __forceinline__ uint64_t d2u(double d) {
#ifdef __CUDA_ARCH__
  return static_cast<uint64_t>(__double_as_longlong(d));
#else
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
#endif
}
__host__ __device__ __forceinline__ double fmad_(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return __builtin_fma(a, b, c);
#endif
}

__host__ __device__ inline double glibc_exp(double x) {
#ifdef __CUDA_ARCH__
  const uint64_t* T = kExpTabDev;
#else
  const uint64_t* T = kExpTabHost;
#endif
  constexpr double InvLn2N = 0x1.71547652b82fep7;
  constexpr double Shift = 0x1.8p52;
  constexpr double NegLn2hiN = -0x1.62e42fefa0000p-8;
  constexpr double NegLn2loN = -0x1.cf79abc9e3b3ap-47;
  constexpr double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3;
  constexpr double C4 = 0x1.55555cf172b91p-5, C5 = 0x1.1111167a4d017p-7;
  uint32_t abstop = static_cast<uint32_t>(d2u(x) >> 52) & 0x7ff;
  constexpr uint32_t kTiny = 0x3c9;   // top12(0x1p-54)
  constexpr uint32_t kLarge = 0x408;  // top12(512.0)
  if (abstop - kTiny >= kLarge - kTiny) {
    if (static_cast<int32_t>(abstop - kTiny) < 0) return 1.0 + x;
    if (abstop >= 0x409) {  // top12(1024.0)
      if (d2u(x) == 0xfff0000000000000ull) return 0.0;
      if (abstop >= 0x7ff) return 1.0 + x;
      return (d2u(x) >> 63) ? 0.0 : u2d(0x7ff0000000000000ull);
    }
    abstop = 0;
  }
  const double z = InvLn2N * x;
  double kd = z + Shift;
  const uint64_t ki = d2u(kd);
  kd = kd - Shift;
  const double r = fmad_(kd, NegLn2loN, fmad_(kd, NegLn2hiN, x));
  const uint64_t idx = 2 * (ki % 128);
  const uint64_t top = ki << 45;
  const double tail = u2d(T[idx]);
  uint64_t sbits = T[idx + 1] + top;
  const double r2 = r * r;
  const double tmp = fmad_(r2 * r2, fmad_(r, C5, C4), fmad_(r2, fmad_(r, C3, C2), tail + r));
  if (abstop == 0) {
    if ((ki & 0x80000000ull) == 0) {
      sbits -= 1009ull << 52;
      const double scale = u2d(sbits);
      return 0x1p1009 * fmad_(scale, tmp, scale);
    }
    sbits += 1022ull << 52;
    const double scale = u2d(sbits);
    double y = fmad_(scale, tmp, scale);
    if (y < 1.0) {
      double lo = fmad_(scale, tmp, scale - y);
      const double hi = 1.0 + y;
      lo = 1.0 - hi + y + lo;
      y = (hi + lo) - 1.0;
      if (y == 0.0) y = 0.0;
    }
    return 0x1p-1022 * y;
  }
  const double scale = u2d(sbits);
  return fmad_(scale, tmp, scale);
}

}  // namespace asicp
