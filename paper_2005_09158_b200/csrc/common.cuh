// Shared device helpers for the ParaDiag-II kernels (sm_100a).  complex128 = double2 (x = re, y = im).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#define PD_HD __host__ __device__ __forceinline__
#define PD_D __device__ __forceinline__

PD_HD double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
PD_HD double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
PD_HD double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
PD_HD double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
// c + a*b
PD_HD double2 cfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
PD_HD double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
PD_HD double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
PD_HD double2 cneg(double2 a) { return make_double2(-a.x, -a.y); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
PD_HD double2 cmul_mi(double2 a) { return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x); }
PD_HD double2 crcp(double2 a) {
  // 1/a with scaling to avoid overflow/underflow in |a|^2
  double s = fmax(fabs(a.x), fabs(a.y));
  double ax = a.x / s, ay = a.y / s;
  double d = 1.0 / (s * (ax * ax + ay * ay));
  return make_double2(ax * d, -ay * d);
}
PD_HD double2 cdiv(double2 a, double2 b) { return cmul(a, crcp(b)); }
// 1/a with one correctly rounded fp64 reciprocal (no overflow guard: for |a| in ~[1e-150, 1e150])
PD_D double2 crcp_fast(double2 a) {
  const double d = __drcp_rn(fma(a.x, a.x, a.y * a.y));
  return make_double2(a.x * d, -a.y * d);
}
PD_HD double2 czero() { return make_double2(0.0, 0.0); }
