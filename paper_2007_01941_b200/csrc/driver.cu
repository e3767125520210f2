// Small host-side numerics and utility kernels of the driver layer:
// rotation canonicalisation (rotation.py:124-137), camera/point step application,
// and the largest eigenvalue of the <= 5x5 Lanczos tridiagonal
// (multigrid.py:281-284, scipy eigh_tridiagonal) by Sturm bisection.
#include <math.h>

#include "common.cuh"
#include "ctx.h"

// aa <- aa * (1 - 2 pi / |aa|) while |aa| > pi (rotation.py:124-137), in place on (n, stride) rows
__global__ void k_canonicalize(double* __restrict__ cams, int n, int stride) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double* a = cams + (int64_t)i * stride;
    for (int it = 0; it < 64; ++it) {
      double th = sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
      if (!(th > M_PI)) break;
      double s = 1.0 - 2.0 * M_PI / th;
      a[0] *= s;
      a[1] *= s;
      a[2] *= s;
    }
  }
}

extern "C" int bamg_canonicalize(bamg_ctx* ctx, double* cams, int32_t n, int32_t stride, void* stream) {
  (void)ctx;
  if (n <= 0) return 0;
  launch(k_canonicalize, grid_for(n, 128), 128, 0, as_stream(stream), cams, n, stride);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// Number of eigenvalues of the symmetric tridiagonal (a, b) strictly below x.
static int sturm_count(const double* a, const double* b, int n, double x) {
  int c = 0;
  double q = 1.0;
  for (int i = 0; i < n; ++i) {
    double bb = (i > 0) ? b[i - 1] * b[i - 1] : 0.0;
    q = (a[i] - x) - (i > 0 ? bb / q : 0.0);
    if (q == 0.0) q = -1e-300;
    if (q < 0.0) ++c;
  }
  return c;
}

extern "C" double bamg_tridiag_max_eig(const double* a_host, const double* b_host, int32_t n) {
  if (n <= 0) return NAN;
  if (n == 1) return a_host[0];
  double lo = INFINITY, hi = -INFINITY;
  for (int i = 0; i < n; ++i) {
    double r = (i > 0 ? fabs(b_host[i - 1]) : 0.0) + (i < n - 1 ? fabs(b_host[i]) : 0.0);
    lo = fmin(lo, a_host[i] - r);
    hi = fmax(hi, a_host[i] + r);
  }
  double span = fmax(fabs(lo), fabs(hi));
  lo -= 1e-14 * span + 1e-300;
  hi += 1e-14 * span + 1e-300;
  for (int it = 0; it < 200; ++it) {
    double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (sturm_count(a_host, b_host, n, mid) >= n) hi = mid;  // all eigenvalues below mid
    else lo = mid;
  }
  return 0.5 * (lo + hi);
}
