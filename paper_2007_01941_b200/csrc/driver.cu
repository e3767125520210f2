// Small host-side numerics and utility kernels of the driver layer:
// rotation canonicalisation (rotation.py:124-137), camera/point step application,
// and the largest eigenvalue of the <= 5x5 Lanczos tridiagonal
// (multigrid.py:281-284, scipy eigh_tridiagonal) by Sturm bisection.
#include <math.h>

#include "common.cuh"
#include "ctx.h"

// aa <- aa * (1 - 2 pi / |aa|) while |aa| > pi (rotation.py:124-137). numpy's
// np.linalg.norm over 3 entries is sqrt((a0^2 + a1^2) + a2^2) with every operation
// rounded; the explicit _rn intrinsics keep nvcc from contracting them into FMAs,
// so the wrap decision near |aa| = pi is the reference's.
__device__ __noinline__ void canon_row(double* a) {
  for (int it = 0; it < 64; ++it) {
    double th = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(a[0], a[0]), __dmul_rn(a[1], a[1])), __dmul_rn(a[2], a[2])));
    if (!(th > M_PI)) break;
    double s = __dsub_rn(1.0, __ddiv_rn(2.0 * M_PI, th));
    a[0] = __dmul_rn(a[0], s);
    a[1] = __dmul_rn(a[1], s);
    a[2] = __dmul_rn(a[2], s);
  }
}

// in place on (n, stride) rows
__global__ void k_canonicalize(double* __restrict__ cams, int n, int stride) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    canon_row(cams + (int64_t)i * stride);
}

// LM trial step on the device (solver.py:276-301): from the device scalars of the
// step -- t = [rhs.dc, dc.S dc, g_p.C^-1 g_p, dc.dc, dp.dp, f, f_new] -- and the
// candidate's behind-camera count:
//   decrease = (t0 - 0.5 t1) + 0.5 t2            (schur.py:176-188)
//   rho = -inf if the candidate is behind a camera or decrease <= 0,
//         else 0.5 (f - f_new) / decrease
//   accepted = rho > min_rho: params <- candidate, rotations canonicalised
// Every thread evaluates the (uniform) decision; the arithmetic is the host's
// IEEE sequence (explicit _rn operations, no contraction). out = [rho, accepted,
// decrease, step_norm, f_new (f when behind), radius']: the trust-region update
// (solver.py:134-149) radius' = radius / max(1/3, 1 - (2 rho - 1)^3) on acceptance,
// radius / 2 otherwise, from the device slot t[7]. The cube is formed in double-double
// and rounded once, like the host's correctly rounded pow(x, 3).
__global__ void k_lm_trial(const double* __restrict__ t, const int* __restrict__ n_behind, double min_rho,
                           double* __restrict__ cams, const double* __restrict__ cand_cams, int nc,
                           double* __restrict__ pts, const double* __restrict__ cand_pts, int npt,
                           double* __restrict__ out) {
  double dec = __dadd_rn(__dsub_rn(t[0], __dmul_rn(0.5, t[1])), __dmul_rn(0.5, t[2]));
  bool behind = *n_behind > 0;
  double f = t[5], fn = behind ? t[5] : t[6];
  double rho = (!behind && dec > 0.0) ? __ddiv_rn(__dmul_rn(0.5, __dsub_rn(f, fn)), dec) : -INFINITY;
  bool acc = rho > min_rho;
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid == 0) {
    out[0] = rho;
    out[1] = acc ? 1.0 : 0.0;
    out[2] = dec;
    out[3] = __dsqrt_rn(__dadd_rn(t[3], t[4]));
    out[4] = fn;
    double rad = t[7];
    if (acc) {
      double u = __dsub_rn(__dmul_rn(2.0, rho), 1.0);
      double hi = __dmul_rn(u, u), lo = __fma_rn(u, u, -hi);
      double p = __dmul_rn(hi, u), e = __fma_rn(hi, u, -p);
      double cube = __dadd_rn(p, __dadd_rn(e, __dmul_rn(lo, u)));
      rad = __ddiv_rn(rad, fmax(1.0 / 3.0, __dsub_rn(1.0, cube)));
    } else {
      rad = __ddiv_rn(rad, 2.0);
    }
    out[5] = rad;
  }
  if (!acc) return;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < (int64_t)npt * 3; i += stride) pts[i] = cand_pts[i];
  for (int64_t i = tid; i < nc; i += stride) {
    const double* c = cand_cams + i * 9;
    double* a = cams + i * 9;
    for (int q = 0; q < 9; ++q) a[q] = c[q];
    canon_row(a);  // rotation.py:124-137, the same code as k_canonicalize
  }
}

extern "C" int bamg_lm_trial(bamg_ctx* ctx, const double* t_dev, const int32_t* n_behind_dev, double min_rho,
                             double* cams, const double* cand_cams, int32_t nc, double* pts, const double* cand_pts,
                             int32_t npt, double* out_dev, void* stream) {
  (void)ctx;
  int64_t work = (int64_t)npt * 3 > nc ? (int64_t)npt * 3 : nc;
  launch(k_lm_trial, grid_for(work > 0 ? work : 1, 256), 256, 0, as_stream(stream), t_dev, n_behind_dev, min_rho,
         cams, cand_cams, (int)nc, pts, cand_pts, (int)npt, out_dev);
  BAMG_LAUNCH_CHECK();
  return 0;
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
