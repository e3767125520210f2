// Device-side synthetic scenes for BASELINE configs 3-5.
//
// The reference ships a host generator (synth.py:92-558: camera frames, visibility,
// pixel noise, centre-preserving perturbation); the repo's numpy scenes.py follows
// SURVEY App. C for the five BASELINE configurations and takes ~25 s at config 4.
// This file generates the same distributions on the GPU, directly into the arrays a
// BundleProblem ingests, in three steps:
//   bamg_scene_layout      cameras (truth + perturbed start), points, requested
//                          cameras per point, camera grid cells
//   bamg_scene_visibility  per point: candidate cameras from the cell lists (city,
//                          large) or the run formula (loop), the candidate filters,
//                          the draw, the final observation filters of _finish, the
//                          ">= 2 cameras" rule; survivors sorted by camera
//   bamg_scene_emit        compaction (kept cameras / points), point-major
//                          observations, pixels = projection + N(0, 1)
// Every random draw is a pure function of (seed, stream, index): a splitmix64
// counter hash, so results do not depend on grid size or scheduling. The scenes are
// NOT bit-identical to the numpy generator's (PCG64 streams); they share its model,
// and tests pin their statistics and determinism, not their digests.
#include <math.h>

#include "common.cuh"

namespace {

enum { KIND_CITY = 3, KIND_LARGE = 4, KIND_LOOP = 5 };
enum {  // random streams
  ST_CLUSTER = 1, ST_CAM_POS, ST_CAM_YAW, ST_CAM_K, ST_CAM_XI, ST_CAM_C0, ST_PT_POS, ST_PT_PICK, ST_PT_INIT,
  ST_PT_LOOP, ST_KEY, ST_PIX
};
#define SCENE_MAX_PICK 32
#define SCENE_CAP 2048  // in-radius candidates cached per point (warp)

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t rbits(uint64_t seed, int stream, uint64_t idx, int k) {
  return mix64(mix64(mix64(seed ^ ((uint64_t)stream << 56)) + idx) + (uint64_t)k * 0xd1342543de82ef95ull);
}
// uniform in (0, 1)
__device__ __forceinline__ double runif(uint64_t seed, int stream, uint64_t idx, int k) {
  return ((double)(rbits(seed, stream, idx, k) >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}
__device__ __forceinline__ double rnorm(uint64_t seed, int stream, uint64_t idx, int k) {
  double u1 = runif(seed, stream, idx, 2 * k), u2 = runif(seed, stream, idx, 2 * k + 1);
  return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}
__device__ int rpoisson(double lam, double u) {  // inversion, lam small
  double p = exp(-lam), c = p;
  int k = 0;
  while (u > c && k < 64) {
    ++k;
    p *= lam / k;
    c += p;
  }
  return k;
}

// rows x_c, y_c, z_c of a camera looking along the horizontal/any direction `look`
// (scenes.look_frames; the frame of pkg/tests/conftest.py:33-41)
__device__ void look_frame(const double look[3], double R[9]) {
  double n = sqrt(look[0] * look[0] + look[1] * look[1] + look[2] * look[2]);
  double z[3] = {-look[0] / n, -look[1] / n, -look[2] / n};
  double x[3] = {-z[1], z[0], 0.0};  // up x z, up = (0,0,1)
  double xn = sqrt(x[0] * x[0] + x[1] * x[1]);
  x[0] /= xn;
  x[1] /= xn;
  double y[3] = {z[1] * x[2] - z[2] * x[1], z[2] * x[0] - z[0] * x[2], z[0] * x[1] - z[1] * x[0]};
  for (int c = 0; c < 3; ++c) {
    R[c] = x[c];
    R[3 + c] = y[c];
    R[6 + c] = z[c];
  }
}

// rotation matrix -> angle-axis through the unit quaternion (largest-component branch)
__device__ void rotvec_of(const double R[9], double aa[3]) {
  double tr = R[0] + R[4] + R[8], q[4];  // w, x, y, z
  if (tr > 0) {
    double s = sqrt(tr + 1.0) * 2;
    q[0] = 0.25 * s;
    q[1] = (R[7] - R[5]) / s;
    q[2] = (R[2] - R[6]) / s;
    q[3] = (R[3] - R[1]) / s;
  } else if (R[0] > R[4] && R[0] > R[8]) {
    double s = sqrt(1.0 + R[0] - R[4] - R[8]) * 2;
    q[0] = (R[7] - R[5]) / s;
    q[1] = 0.25 * s;
    q[2] = (R[1] + R[3]) / s;
    q[3] = (R[2] + R[6]) / s;
  } else if (R[4] > R[8]) {
    double s = sqrt(1.0 + R[4] - R[0] - R[8]) * 2;
    q[0] = (R[2] - R[6]) / s;
    q[1] = (R[1] + R[3]) / s;
    q[2] = 0.25 * s;
    q[3] = (R[5] + R[7]) / s;
  } else {
    double s = sqrt(1.0 + R[8] - R[0] - R[4]) * 2;
    q[0] = (R[3] - R[1]) / s;
    q[1] = (R[2] + R[6]) / s;
    q[2] = (R[5] + R[7]) / s;
    q[3] = 0.25 * s;
  }
  if (q[0] < 0)
    for (int k = 0; k < 4; ++k) q[k] = -q[k];
  double vn = sqrt(q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  double th = 2.0 * atan2(vn, q[0]);
  double sc = vn > 1e-12 ? th / vn : 2.0;
  for (int k = 0; k < 3; ++k) aa[k] = sc * q[1 + k];
}

// Rodrigues matrix of a (small) rotation vector
__device__ void rot_of(const double w[3], double R[9]) {
  double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  double a = th > 1e-9 ? sin(th) / th : 1.0 - th * th / 6.0;
  double b = th > 1e-9 ? (1.0 - cos(th)) / (th * th) : 0.5 - th * th / 24.0;
  double K[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double kk = 0;
      for (int m = 0; m < 3; ++m) kk += K[3 * i + m] * K[3 * m + j];
      R[3 * i + j] = (i == j ? 1.0 : 0.0) + a * K[3 * i + j] + b * kk;
    }
}

struct Layout {
  int kind, nc, npts, n_clusters, gx, gy;
  uint64_t seed;
  double side, cam_sigma, pt_sigma, z_max, lam, cell, org, bridge_frac;
};

__device__ void cluster_centre(const Layout& L, int cl, double c[2]) {
  c[0] = L.side * runif(L.seed, ST_CLUSTER, cl, 0);
  c[1] = L.side * runif(L.seed, ST_CLUSTER, cl, 1);
}

__device__ __forceinline__ int cell_of(const Layout& L, double x, double y) {
  int cx = (int)floor((x - L.org) / L.cell), cy = (int)floor((y - L.org) / L.cell);
  cx = min(max(cx, 0), L.gx - 1);
  cy = min(max(cy, 0), L.gy - 1);
  return cy * L.gx + cx;
}

// cam_rt rows (24): R (9), t (3), R0 (9), t0 (3); truth / init rows (9): aa, t, f, k1, k2
__global__ void k_scene_cameras(Layout L, double* __restrict__ centre, double* __restrict__ cam_rt,
                                double* __restrict__ truth, double* __restrict__ init, uint32_t* __restrict__ cell) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L.nc; i += gridDim.x * blockDim.x) {
    double c[3], look[3];
    if (L.kind == KIND_LOOP) {
      double rad = L.nc / (2.0 * M_PI), phi = i / rad;
      c[0] = rad * cos(phi);
      c[1] = rad * sin(phi);
      c[2] = 0.0;
      look[0] = -sin(phi);
      look[1] = cos(phi);
      look[2] = 0.0;
    } else {
      if (L.kind == KIND_CITY) {
        c[0] = L.side * runif(L.seed, ST_CAM_POS, i, 0);
        c[1] = L.side * runif(L.seed, ST_CAM_POS, i, 1);
      } else {
        double cc[2];
        cluster_centre(L, i / (L.nc / L.n_clusters), cc);
        c[0] = cc[0] + L.cam_sigma * rnorm(L.seed, ST_CAM_POS, i, 0);
        c[1] = cc[1] + L.cam_sigma * rnorm(L.seed, ST_CAM_POS, i, 1);
      }
      c[2] = 1.5;
      double yaw = 2.0 * M_PI * runif(L.seed, ST_CAM_YAW, i, 0);
      look[0] = cos(yaw);
      look[1] = sin(yaw);
      look[2] = 0.0;
    }
    double R[9], t[3];
    look_frame(look, R);
    for (int r = 0; r < 3; ++r) t[r] = -(R[3 * r] * c[0] + R[3 * r + 1] * c[1] + R[3 * r + 2] * c[2]);
    double k1 = 1e-2 * rnorm(L.seed, ST_CAM_K, i, 0), k2 = 1e-2 * rnorm(L.seed, ST_CAM_K, i, 1);
    // start: rotation <- Rot(xi) R, centre + N(0, 1e-2), t recomputed (synth.py:449-463)
    double xi[3], dR[9], R0[9], c0[3], t0[3];
    for (int k = 0; k < 3; ++k) {
      xi[k] = 1e-2 * rnorm(L.seed, ST_CAM_XI, i, k);
      c0[k] = c[k] + 1e-2 * rnorm(L.seed, ST_CAM_C0, i, k);
    }
    rot_of(xi, dR);
    for (int r = 0; r < 3; ++r)
      for (int cc = 0; cc < 3; ++cc) {
        double s = 0;
        for (int m = 0; m < 3; ++m) s += dR[3 * r + m] * R[3 * m + cc];
        R0[3 * r + cc] = s;
      }
    for (int r = 0; r < 3; ++r) t0[r] = -(R0[3 * r] * c0[0] + R0[3 * r + 1] * c0[1] + R0[3 * r + 2] * c0[2]);
    double* o = cam_rt + (int64_t)i * 24;
    for (int k = 0; k < 9; ++k) {
      o[k] = R[k];
      o[12 + k] = R0[k];
    }
    for (int k = 0; k < 3; ++k) {
      o[9 + k] = t[k];
      o[21 + k] = t0[k];
      centre[3 * (int64_t)i + k] = c[k];
    }
    double aa[3], aa0[3];
    rotvec_of(R, aa);
    rotvec_of(R0, aa0);
    double* tr = truth + (int64_t)i * 9;
    double* in = init + (int64_t)i * 9;
    for (int k = 0; k < 3; ++k) {
      tr[k] = aa[k];
      tr[3 + k] = t[k];
      in[k] = aa0[k];
      in[3 + k] = t0[k];
    }
    tr[6] = in[6] = 500.0;
    tr[7] = in[7] = k1;
    tr[8] = in[8] = k2;
    cell[i] = (L.kind == KIND_LOOP) ? 0u : (uint32_t)cell_of(L, c[0], c[1]);
  }
}

// aux (2 per point): loop -- floor(s) and (behind | bridge offset << 8, 0 = no bridge)
__global__ void k_scene_points(Layout L, double* __restrict__ pts, double* __restrict__ pts0,
                               int32_t* __restrict__ n_pick, int32_t* __restrict__ aux) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L.npts; i += (int64_t)gridDim.x * blockDim.x) {
    double X[3];
    int pick;
    if (L.kind == KIND_LOOP) {
      double rad = L.nc / (2.0 * M_PI);
      double s = L.nc * runif(L.seed, ST_PT_POS, i, 0);
      double rr = 10.0 * sqrt(runif(L.seed, ST_PT_POS, i, 1));
      double ang = 2.0 * M_PI * runif(L.seed, ST_PT_POS, i, 2);
      double radial = rr * cos(ang), ps = s / rad;
      X[0] = (rad + radial) * cos(ps);
      X[1] = (rad + radial) * sin(ps);
      X[2] = rr * sin(ang);
      // L = 2 + geometric(0.5), support >= 1: 1 + leading zero run of random bits
      uint64_t b = rbits(L.seed, ST_PT_LOOP, i, 0);
      int g = 1 + (b ? __clzll((long long)b) : 63);
      pick = min(2 + g, SCENE_MAX_PICK - 1);
      int behind = 7 + (int)(rbits(L.seed, ST_PT_LOOP, i, 1) % 4);
      int bridge = 0;
      if (runif(L.seed, ST_PT_LOOP, i, 2) < L.bridge_frac) bridge = 51 + (int)(rbits(L.seed, ST_PT_LOOP, i, 3) % 50);
      aux[2 * i] = (int)floor(s);
      aux[2 * i + 1] = behind | (bridge << 8);
    } else {
      if (L.kind == KIND_CITY) {
        X[0] = L.side * runif(L.seed, ST_PT_POS, i, 0);
        X[1] = L.side * runif(L.seed, ST_PT_POS, i, 1);
      } else {
        double cc[2];
        int cl = (int)(rbits(L.seed, ST_PT_POS, i, 7) % (uint64_t)L.n_clusters);
        cluster_centre(L, cl, cc);
        X[0] = cc[0] + L.pt_sigma * rnorm(L.seed, ST_PT_POS, i, 0);
        X[1] = cc[1] + L.pt_sigma * rnorm(L.seed, ST_PT_POS, i, 1);
      }
      X[2] = L.z_max * runif(L.seed, ST_PT_POS, i, 6);
      pick = min(2 + rpoisson(L.lam, runif(L.seed, ST_PT_PICK, i, 0)), SCENE_MAX_PICK);
      aux[2 * i] = aux[2 * i + 1] = 0;
    }
    n_pick[i] = pick;
    for (int k = 0; k < 3; ++k) {
      pts[3 * i + k] = X[k];
      pts0[3 * i + k] = X[k] + 5e-2 * rnorm(L.seed, ST_PT_INIT, i, k);
    }
  }
}

// _finish's observation filters (scenes.py:100-160): depth >= 1 and |p| <= 2 at the
// truth, in front of the camera (z < -1e-3) at the start
__device__ bool obs_ok(const double* __restrict__ rt, const double X[3], const double X0[3]) {
  double pc[3];
  for (int r = 0; r < 3; ++r) pc[r] = rt[3 * r] * X[0] + rt[3 * r + 1] * X[1] + rt[3 * r + 2] * X[2] + rt[9 + r];
  double depth = -pc[2];
  if (!(depth >= 1.0)) return false;
  double px = pc[0] / depth, py = pc[1] / depth;
  if (!(px * px + py * py <= 4.0)) return false;
  const double* r0 = rt + 12;
  double z0 = r0[6] * X0[0] + r0[7] * X0[1] + r0[8] * X0[2] + r0[11];
  return z0 < -1e-3;
}

__device__ void finish_point(int cnt, int32_t* mine, int32_t* out_cnt) {
  // insertion sort by camera, duplicates removed, fewer than two -> dropped
  for (int a = 1; a < cnt; ++a) {
    int v = mine[a], b = a - 1;
    while (b >= 0 && mine[b] > v) {
      mine[b + 1] = mine[b];
      --b;
    }
    mine[b + 1] = v;
  }
  int m = 0;
  for (int a = 0; a < cnt; ++a)
    if (m == 0 || mine[m - 1] != mine[a]) mine[m++] = mine[a];
  *out_cnt = m >= 2 ? m : 0;
}

__global__ void k_scene_vis_loop(Layout L, const double* __restrict__ cam_rt, const double* __restrict__ pts,
                                 const double* __restrict__ pts0, const int32_t* __restrict__ n_pick,
                                 const int32_t* __restrict__ aux, int32_t* __restrict__ sel,
                                 int32_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L.npts; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t* mine = sel + i * SCENE_MAX_PICK;
    double X[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    double X0[3] = {pts0[3 * i], pts0[3 * i + 1], pts0[3 * i + 2]};
    int s = aux[2 * i], behind = aux[2 * i + 1] & 255, bridge = aux[2 * i + 1] >> 8;
    int m = 0;
    for (int off = 0; off < n_pick[i] + (bridge ? 1 : 0); ++off) {
      int d = off < n_pick[i] ? behind + off : bridge;
      int cam = ((s - d) % L.nc + L.nc) % L.nc;
      if (obs_ok(cam_rt + (int64_t)cam * 24, X, X0)) mine[m++] = cam;
    }
    finish_point(m, mine, cnt + i);
  }
}

// city / large: one warp per point. Candidates = cameras of the 3x3 cells around the
// point within `radius`; the k_nn nearest of them (distance threshold by bisection);
// candidate filters of scenes._nearest_visible / _large_chunk; the draw takes the
// n_pick smallest keys (city: distance, large: a uniform key per (point, camera)).
__global__ void __launch_bounds__(128)
k_scene_vis_cells(Layout L, double radius, int k_nn, const double* __restrict__ centre,
                  const double* __restrict__ cam_rt, const double* __restrict__ pts, const double* __restrict__ pts0,
                  const int32_t* __restrict__ n_pick, const int32_t* __restrict__ cell_ptr,
                  const uint32_t* __restrict__ cell_cams, int32_t* __restrict__ sel, int32_t* __restrict__ cnt,
                  int32_t* __restrict__ info) {
  extern __shared__ __align__(16) unsigned char smem_scene[];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  double* key = reinterpret_cast<double*>(smem_scene) + (size_t)w * SCENE_CAP;
  int32_t* cid = reinterpret_cast<int32_t*>(smem_scene + (size_t)wpb * SCENE_CAP * 8) + (size_t)w * SCENE_CAP;
  for (int64_t i = blockIdx.x * (int64_t)wpb + w; i < L.npts; i += (int64_t)gridDim.x * wpb) {
    double X[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    double X0[3] = {pts0[3 * i], pts0[3 * i + 1], pts0[3 * i + 2]};
    int cx = (int)floor((X[0] - L.org) / L.cell), cy = (int)floor((X[1] - L.org) / L.cell);
    cx = min(max(cx, 0), L.gx - 1);
    cy = min(max(cy, 0), L.gy - 1);
    // 1. in-radius candidates into shared memory (order: cell-major, warp-compacted)
    int n = 0;
    bool over = false;
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        int gx = cx + dx, gy = cy + dy;
        if (gx < 0 || gy < 0 || gx >= L.gx || gy >= L.gy) continue;
        int c = gy * L.gx + gx, lo = cell_ptr[c], hi = cell_ptr[c + 1];
        for (int b = lo; b < hi; b += 32) {
          int j = b + lane;
          int cam = j < hi ? (int)cell_cams[j] : -1;
          double d2 = 1e300;
          if (cam >= 0) {
            double ex = X[0] - centre[3 * (int64_t)cam], ey = X[1] - centre[3 * (int64_t)cam + 1];
            d2 = ex * ex + ey * ey;
          }
          bool in = cam >= 0 && d2 <= radius * radius;
          unsigned m = __ballot_sync(FULL_MASK, in);
          int pos = n + __popc(m & ((1u << lane) - 1));
          if (in) {
            if (pos < SCENE_CAP) {
              key[pos] = d2;
              cid[pos] = cam;
            } else {
              over = true;
            }
          }
          n += __popc(m);
        }
      }
    if (__any_sync(FULL_MASK, over)) {
      if (lane == 0) atomicAdd(info, 1);
      n = SCENE_CAP;
    }
    __syncwarp();
    // 2. distance threshold of the k_nn nearest
    double T = radius * radius;
    if (n > k_nn) {
      double lo = 0.0, hi = T;
      for (int it = 0; it < 48; ++it) {
        double mid = 0.5 * (lo + hi);
        int c = 0;
        for (int j = lane; j < n; j += 32) c += key[j] <= mid;
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(FULL_MASK, c, o);
        if (c <= k_nn) lo = mid;
        else hi = mid;
      }
      T = lo;
    }
    // 3. candidate filters; key <- selection key or +inf
    for (int j = lane; j < n; j += 32) {
      double d2 = key[j], k = 1e300;
      int cam = cid[j];
      if (d2 <= T) {
        const double* rt = cam_rt + (int64_t)cam * 24;
        double rel[3] = {X[0] - centre[3 * (int64_t)cam], X[1] - centre[3 * (int64_t)cam + 1],
                         X[2] - centre[3 * (int64_t)cam + 2]};
        double px = rt[0] * rel[0] + rt[1] * rel[1] + rt[2] * rel[2];
        double py = rt[3] * rel[0] + rt[4] * rel[1] + rt[5] * rel[2];
        double depth = -(rt[6] * rel[0] + rt[7] * rel[1] + rt[8] * rel[2]);
        double d3 = sqrt(rel[0] * rel[0] + rel[1] * rel[1] + rel[2] * rel[2]);
        bool ok = depth >= fmax(1.0, 0.2 * d3);
        if (L.kind == KIND_CITY) ok = ok && fmax(fabs(px), fabs(py)) <= 1.9 * depth;
        else ok = ok && px * px + py * py <= (1.9 * depth) * (1.9 * depth);
        if (ok) k = (L.kind == KIND_CITY) ? d2 : runif(L.seed, ST_KEY, (uint64_t)i * (uint64_t)L.nc + cam, 0);
      }
      key[j] = k;
    }
    __syncwarp();
    // 4. the n_pick smallest keys (ties: lower camera id), final filters on each
    int want = n_pick[i], m = 0;
    int32_t* mine = sel + i * SCENE_MAX_PICK;
    for (int r = 0; r < want; ++r) {
      double best = 1e300;
      int bj = -1, bc = 0x7fffffff;
      for (int j = lane; j < n; j += 32) {
        double k = key[j];
        if (k < best || (k == best && k < 1e300 && cid[j] < bc)) {
          best = k;
          bj = j;
          bc = cid[j];
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        double ob = __shfl_xor_sync(FULL_MASK, best, o);
        int oj = __shfl_xor_sync(FULL_MASK, bj, o), oc = __shfl_xor_sync(FULL_MASK, bc, o);
        if (ob < best || (ob == best && oc < bc)) {
          best = ob;
          bj = oj;
          bc = oc;
        }
      }
      if (!(best < 1e300)) break;
      if (lane == 0) {
        key[bj] = 1e300;
        if (obs_ok(cam_rt + (int64_t)bc * 24, X, X0)) mine[m++] = bc;
      }
      __syncwarp();
    }
    if (lane == 0) finish_point(m, mine, cnt + i);
    __syncwarp();
  }
}

__global__ void k_scene_mark(const int32_t* __restrict__ cnt, const int32_t* __restrict__ sel, int64_t npts,
                             int32_t* __restrict__ cam_used, int32_t* __restrict__ pt_used) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npts; i += (int64_t)gridDim.x * blockDim.x) {
    int c = cnt[i];
    pt_used[i] = c > 0;
    for (int a = 0; a < c; ++a) cam_used[sel[i * SCENE_MAX_PICK + a]] = 1;  // same value from every writer
  }
}

__global__ void k_scene_emit_obs(uint64_t seed, int64_t npts, const int32_t* __restrict__ cnt,
                                 const int32_t* __restrict__ obs_off, const int32_t* __restrict__ sel,
                                 const int32_t* __restrict__ cam_map, const int32_t* __restrict__ pt_map,
                                 const double* __restrict__ cam_rt, const double* __restrict__ truth,
                                 const double* __restrict__ pts, const double* __restrict__ pts0,
                                 int64_t* __restrict__ cam_index, int64_t* __restrict__ pt_index,
                                 double* __restrict__ pixels, double* __restrict__ out_pts,
                                 double* __restrict__ out_pts0) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npts; i += (int64_t)gridDim.x * blockDim.x) {
    int c = cnt[i];
    if (!c) continue;
    int64_t o = obs_off[i], p = pt_map[i];
    double X[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    for (int k = 0; k < 3; ++k) {
      out_pts[3 * p + k] = X[k];
      out_pts0[3 * p + k] = pts0[3 * i + k];
    }
    for (int a = 0; a < c; ++a) {
      int cam = sel[i * SCENE_MAX_PICK + a];
      const double* rt = cam_rt + (int64_t)cam * 24;
      const double* tr = truth + (int64_t)cam * 9;
      double pc[3];
      for (int r = 0; r < 3; ++r) pc[r] = rt[3 * r] * X[0] + rt[3 * r + 1] * X[1] + rt[3 * r + 2] * X[2] + rt[9 + r];
      double qx = -pc[0] / pc[2], qy = -pc[1] / pc[2];
      double n2 = qx * qx + qy * qy;
      double s = tr[6] * (1.0 + tr[7] * n2 + tr[8] * n2 * n2);  // problem.py projection model
      uint64_t id = (uint64_t)i * SCENE_MAX_PICK + a;
      cam_index[o + a] = cam_map[cam];
      pt_index[o + a] = p;
      pixels[2 * (o + a)] = s * qx + rnorm(seed, ST_PIX, id, 0);
      pixels[2 * (o + a) + 1] = s * qy + rnorm(seed, ST_PIX, id, 1);
    }
  }
}

__global__ void k_scene_emit_cams(int nc, const int32_t* __restrict__ cam_used, const int32_t* __restrict__ cam_map,
                                  const double* __restrict__ truth, const double* __restrict__ init,
                                  double* __restrict__ out_truth, double* __restrict__ out_init) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
    if (!cam_used[i]) continue;
    int64_t m = cam_map[i];
    for (int k = 0; k < 9; ++k) {
      out_truth[9 * m + k] = truth[9 * (int64_t)i + k];
      out_init[9 * m + k] = init[9 * (int64_t)i + k];
    }
  }
}

int fill_layout(Layout& L, int kind, int64_t seed, int nc, int64_t npts, const double* p) {
  if (kind != KIND_CITY && kind != KIND_LARGE && kind != KIND_LOOP) {
    bamg_set_error("scene kind %d: 3 (city), 4 (large) or 5 (loop)", kind);
    return BAMG_ERR_UNSUPPORTED;
  }
  if (nc < 2 || npts < 1 || npts > 0x7fffffff / SCENE_MAX_PICK) {
    bamg_set_error("scene size out of range (nc=%d, npts=%lld)", nc, (long long)npts);
    return BAMG_ERR_UNSUPPORTED;
  }
  // params: [side, n_clusters, cam_sigma, pt_sigma, z_max, lam, radius, bridge_frac]
  L.kind = kind;
  L.nc = nc;
  L.npts = (int)npts;
  L.seed = (uint64_t)seed;
  L.side = p[0];
  L.n_clusters = (int)p[1] > 0 ? (int)p[1] : 1;
  L.cam_sigma = p[2];
  L.pt_sigma = p[3];
  L.z_max = p[4];
  L.lam = p[5];
  L.cell = p[6] > 0 ? p[6] : 1.0;
  L.bridge_frac = p[7];
  double margin = (kind == KIND_LARGE) ? 6.0 * (L.cam_sigma + L.pt_sigma) : 0.0;
  L.org = -margin;
  L.gx = L.gy = (kind == KIND_LOOP) ? 1 : (int)ceil((L.side + 2 * margin) / L.cell) + 1;
  if (kind == KIND_LARGE && nc % L.n_clusters) {
    bamg_set_error("large scene: nc must be a multiple of n_clusters");
    return BAMG_ERR_UNSUPPORTED;
  }
  return BAMG_OK;
}

}  // namespace

extern "C" int bamg_scene_grid_cells(int32_t kind, int32_t nc, int64_t npts, const double* params_host) {
  Layout L;
  if (fill_layout(L, kind, 0, nc, npts, params_host) != BAMG_OK) return -1;
  return L.gx * L.gy;
}

extern "C" int bamg_scene_layout(bamg_ctx* ctx, int32_t kind, int64_t seed, int32_t nc, int64_t npts,
                                 const double* params_host, double* cam_centre, double* cam_rt, double* cam_truth,
                                 double* cam_init, uint32_t* cam_cell, double* pts_true, double* pts_init,
                                 int32_t* n_pick, int32_t* aux, void* stream) {
  (void)ctx;
  Layout L;
  int rc = fill_layout(L, kind, seed, nc, npts, params_host);
  if (rc != BAMG_OK) return rc;
  launch(k_scene_cameras, grid_for(nc, 128), 128, 0, as_stream(stream), L, cam_centre, cam_rt, cam_truth, cam_init,
         cam_cell);
  launch(k_scene_points, grid_for(npts, 256), 256, 0, as_stream(stream), L, pts_true, pts_init, n_pick, aux);
  BAMG_LAUNCH_CHECK();
  return BAMG_OK;
}

extern "C" int bamg_scene_visibility(bamg_ctx* ctx, int32_t kind, int64_t seed, int32_t nc, int64_t npts,
                                     const double* params_host, int32_t k_nn, const double* cam_centre,
                                     const double* cam_rt, const double* pts_true, const double* pts_init,
                                     const int32_t* n_pick, const int32_t* aux, const int32_t* cell_ptr,
                                     const uint32_t* cell_cams, int32_t* sel, int32_t* cnt, int32_t* cam_used,
                                     int32_t* pt_used, int32_t* info, void* stream) {
  (void)ctx;
  Layout L;
  int rc = fill_layout(L, kind, seed, nc, npts, params_host);
  if (rc != BAMG_OK) return rc;
  cudaStream_t st = as_stream(stream);
  BAMG_CUDA_CHECK(cudaMemsetAsync(info, 0, sizeof(int32_t), st));
  BAMG_CUDA_CHECK(cudaMemsetAsync(cam_used, 0, sizeof(int32_t) * (size_t)nc, st));
  if (kind == KIND_LOOP) {
    launch(k_scene_vis_loop, grid_for(npts, 128), 128, 0, st, L, cam_rt, pts_true, pts_init, n_pick, aux, sel, cnt);
  } else {
    const int threads = 128;
    size_t smem = (size_t)(threads / 32) * SCENE_CAP * 12;
    BAMG_CUDA_CHECK(cudaFuncSetAttribute(k_scene_vis_cells, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int64_t blocks = ceil_div(npts, threads / 32);
    int grid = (int)(blocks < (int64_t)bamg_num_sms() * 2 ? blocks : (int64_t)bamg_num_sms() * 2);
    launch(k_scene_vis_cells, grid, threads, smem, st, L, params_host[6], (int)k_nn, cam_centre, cam_rt, pts_true,
           pts_init, n_pick, cell_ptr, cell_cams, sel, cnt, info);
  }
  launch(k_scene_mark, grid_for(npts, 256), 256, 0, st, cnt, sel, npts, cam_used, pt_used);
  BAMG_LAUNCH_CHECK();
  return BAMG_OK;
}

extern "C" int bamg_scene_emit(bamg_ctx* ctx, int64_t seed, int32_t nc, int64_t npts, const int32_t* cnt,
                               const int32_t* obs_off, const int32_t* sel, const int32_t* cam_used,
                               const int32_t* cam_map, const int32_t* pt_map, const double* cam_rt,
                               const double* cam_truth, const double* cam_init, const double* pts_true,
                               const double* pts_init, int64_t* cam_index, int64_t* pt_index, double* pixels,
                               double* out_cam_truth, double* out_cam_init, double* out_pts_true,
                               double* out_pts_init, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  launch(k_scene_emit_obs, grid_for(npts, 128), 128, 0, st, (uint64_t)seed, npts, cnt, obs_off, sel, cam_map, pt_map,
         cam_rt, cam_truth, pts_true, pts_init, cam_index, pt_index, pixels, out_pts_true, out_pts_init);
  launch(k_scene_emit_cams, grid_for(nc, 128), 128, 0, st, (int)nc, cam_used, cam_map, cam_truth, cam_init,
         out_cam_truth, out_cam_init);
  BAMG_LAUNCH_CHECK();
  return BAMG_OK;
}
