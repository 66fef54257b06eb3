// Radial kernel functions on the device (ifmm/kernels.py:50-170) plus the two
// BASELINE kernels: inv_r (scale / r) and log_r (scale * (ln r + shift)).
// All return 0 at r == 0 (regularised inner branches vanish there; the unit
// diagonal is written explicitly by the near-field assembly).
#pragma once
#include <cuda_runtime.h>

namespace ifmm {

enum KernelId : int {
  K_LOG = 0,
  K_LAPLACE3D = 1,
  K_BIHARMONIC = 2,
  K_BESSEL_Y0 = 3,
  K_INV_QUADRIC = 4,
  K_INV_MULTIQUADRIC = 5,
  K_HELMHOLTZ3D = 6,
  K_GAUSSIAN = 7,
  K_MULTIQUADRIC = 8,
  K_INV_R = 9,
  K_LOG_R = 10,
  K_COUNT = 11,
};

struct KernelParams {
  int id;
  double a, scale, shift;
};

__device__ __forceinline__ double keval(const KernelParams& K, double r) {
  const double a = K.a;
  switch (K.id) {
    case K_INV_R:
      return r > 0.0 ? K.scale / r : 0.0;
    case K_LOG_R:
      return r > 0.0 ? K.scale * (log(r) + K.shift) : 0.0;
    case K_GAUSSIAN:
      return exp(-(r * r) / a);
    case K_MULTIQUADRIC:
      return sqrt(1.0 + r * r / (a * a));
    default:
      break;
  }
  if (r <= 0.0) return 0.0;
  const bool in = r < a;
  switch (K.id) {
    case K_LOG:
      return in ? r * (log(r) - 1.0) / (a * (log(a) - 1.0)) : log(r) / log(a);
    case K_LAPLACE3D:
      return in ? r / a : a / r;
    case K_BIHARMONIC:
      return in ? r * r * r * (3.0 * log(r) - 1.0) / (a * a * a * (3.0 * log(a) - 1.0))
                : r * r * log(r) / (a * a * log(a));
    case K_BESSEL_Y0:
      return in ? (1.0 + y0(a)) / (1.0 + y0(r)) : y0(r) / y0(a);
    case K_INV_QUADRIC:
      return in ? atan(r) / atan(a) : (1.0 + a * a) / (1.0 + r * r);
    case K_INV_MULTIQUADRIC:
      return in ? asinh(r) / asinh(a) : sqrt((1.0 + a * a) / (1.0 + r * r));
    case K_HELMHOLTZ3D:
      return in ? r / a : a * cos(r) / (r * cos(a));
    default:
      return 0.0;
  }
}

// Euclidean distance with the reference's rounding order (no FMA contraction):
// sqrt(sum_d (t_d - s_d)^2), summed in coordinate order.
__device__ __forceinline__ double dist_rn(const double* t, const double* s, int dim) {
  double acc = 0.0;
  for (int d = 0; d < dim; d++) {
    const double df = __dsub_rn(t[d], s[d]);
    acc = d == 0 ? __dmul_rn(df, df) : __dadd_rn(acc, __dmul_rn(df, df));
  }
  return sqrt(acc);
}

}  // namespace ifmm
