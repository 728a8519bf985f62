// Closed forms of the paper (float64), shared by the metrics kernel (K6) and the host
// entry points fastrs_spheroid_area & co.  Written from PAPER.md §2.1 / §4.1 directly.
#pragma once
#include <math.h>

namespace fastrs {

constexpr double kPi = 3.141592653589793238;

// Spheroid surface area, Eqs. 6-7.  Reading c1: the printed
// "e = 1 - c^2/a^2" is e^2; e is the eccentricity.  Reading c12: branch as printed,
// 1 - e^2 evaluated as (c/a)^2 and e == 0 gives the sphere 4 pi a^2.
__host__ __device__ inline double spheroid_area(double a, double c) {
  if (c < a) {  // oblate, Eq. 6
    const double q = c / a, q2 = q * q;
    const double e = sqrt(1.0 - q2);
    if (e == 0.0) return 4.0 * kPi * a * a;
    return 2.0 * kPi * a * a * (1.0 + q2 * atanh(e) / e);
  }
  const double q = a / c;  // prolate, Eq. 7
  const double e = sqrt(1.0 - q * q);
  if (e == 0.0) return 4.0 * kPi * a * a;
  return 2.0 * kPi * a * a * (1.0 + asin(e) / (q * e));
}

// Ramanujan's first approximation of the ellipse perimeter, Eq. 9.
__host__ __device__ inline double ramanujan_perimeter(double a, double b) {
  return kPi * (3.0 * (a + b) - sqrt((3.0 * a + b) * (a + 3.0 * b)));
}

// 3D: a_s = mean LT, c_s = 3V/(4 pi a_s^2) (Eq. 8), S = pi^(1/3)(6V)^(2/3) / area
// (Eq. 1), written as cbrt(36 pi V^2) / area.
__host__ __device__ inline double c_axis_3d(double V, double a) { return 3.0 * V / (4.0 * kPi * a * a); }
__host__ __device__ inline double sphericity_3d(double V, double a) {
  return cbrt(36.0 * kPi * V * V) / spheroid_area(a, c_axis_3d(V, a));
}

// 2D: a_e = mean LT, b_e = A/(pi a_e) (Eq. 10), P_c = 2 sqrt(pi A) (Eq. 11),
// S = P_c / P_o (Eq. 2) with P_o from Eq. 9.
__host__ __device__ inline double b_axis_2d(double A, double a) { return A / (kPi * a); }
__host__ __device__ inline double sphericity_2d(double A, double a) {
  return 2.0 * sqrt(kPi * A) / ramanujan_perimeter(a, b_axis_2d(A, a));
}

}  // namespace fastrs
