// Observation structure, residual/Jacobian evaluation, normal blocks, damping,
// reduced right-hand side, back-substitution.
//
// Device layout: observations are stored POINT-MAJOR, sorted by
// (point, camera); `pt_ptr` delimits each point's segment. `cm_list` lists the
// point-major positions in (camera, point) order -- exactly the block order of the
// reference's W (`schur.py:114-116` via `blockmat.py:217-230`); `cam_ptr`
// delimits each camera's run in it. Per-observation arrays (all fp64, AoS per
// observation): F (2x9 row-major), E (2x3), res (2), w (1), H = E C^-1 (2x3).
#include <math.h>

#include "common.cuh"
#include "ctx.h"

int radix_sort_pairs(const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout,
                     int64_t n, int key_bits, cudaStream_t st);
int scan_exclusive_int(const int* in, int* out, int64_t n, int* total, cudaStream_t st);
int segment_ptr(const int* ids, int64_t n, int nseg, int* ptr, cudaStream_t st);

static int bits_for(int64_t n) {
  int b = 1;
  while ((1ll << b) < n) ++b;
  return b;
}

__global__ void k_iota(uint32_t* a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (uint32_t)i;
}

// Builds the point-major permutation and the camera-major list (problem.py:84-86
// keeps input order; only the device layout changes).
// rows of 9 doubles -> rows of 10 (80 B, 16 B aligned): per-observation gathers of a
// camera's 9 values then take five 16 B loads instead of nine 8 B ones (each load
// instruction of a warp touches up to 32 lines: the L1 wavefront count is the limit)
__global__ void k_pad9(const double* __restrict__ src, int n, double* __restrict__ dst) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)n * 10;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / 10;
    int c = (int)(t - r * 10);
    dst[t] = c < 9 ? src[r * 9 + c] : 0.0;
  }
}
static inline void pad9(const double* src, int n, double* dst, cudaStream_t st) {
  launch(k_pad9, grid_for((int64_t)n * 10, 256), 256, 0, st, src, n, dst);
}

// Point-major order by counting: per-point histogram -> pt_ptr, scatter into the
// point segments (atomic slots: arbitrary order inside a segment), then every
// element finds its place by ranking its segment on (camera, caller index) -- the
// (point, camera) order is total once duplicates are tie-broken by caller index, so
// the result is the stable sort's, deterministic. Segments are short (a point's
// observations), so the quadratic rank costs less than five radix passes.
__global__ void k_count_i32(const int* __restrict__ key, int64_t k, int* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[key[i]], 1);
}

__global__ void k_pt_scatter(const int* __restrict__ cam_idx, const int* __restrict__ pt_idx, int64_t k,
                             const int* __restrict__ pt_ptr, int* __restrict__ fill, int* __restrict__ tcam,
                             int* __restrict__ tperm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
    int p = pt_idx[i];
    int pos = pt_ptr[p] + atomicAdd(&fill[p], 1);
    tcam[pos] = cam_idx[i];
    tperm[pos] = (int)i;
  }
}

__global__ void k_segment_ids(const int* __restrict__ ptr, int n, int* __restrict__ ids) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    for (int q = ptr[p]; q < ptr[p + 1]; ++q) ids[q] = p;
}

__global__ void k_pt_rank(const int* __restrict__ pt_ptr, const int* __restrict__ obs_pt_pm, int64_t k,
                          const int* __restrict__ tcam, const int* __restrict__ tperm, int* __restrict__ obs_cam_pm,
                          int* __restrict__ pm_perm) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < k; q += (int64_t)gridDim.x * blockDim.x) {
    int p = obs_pt_pm[q];
    int s = pt_ptr[p], e = pt_ptr[p + 1];
    int c = tcam[q], t = tperm[q];
    int r = 0;
    for (int u = s; u < e; ++u) {
      int cu = tcam[u];
      r += (cu < c) || (cu == c && tperm[u] < t);
    }
    obs_cam_pm[s + r] = c;
    pm_perm[s + r] = t;
  }
}

extern "C" int bamg_obs_orders(bamg_ctx* ctx, const int32_t* cam_idx, const int32_t* pt_idx, int64_t k,
                               int32_t nc, int32_t npt, int32_t* pm_perm, int32_t* obs_cam_pm,
                               int32_t* obs_pt_pm, int32_t* pt_ptr, int32_t* cm_list, int32_t* cam_ptr,
                               void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (k == 0) {
    BAMG_CUDA_CHECK(cudaMemsetAsync(pt_ptr, 0, sizeof(int) * (npt + 1), st));
    BAMG_CUDA_CHECK(cudaMemsetAsync(cam_ptr, 0, sizeof(int) * (nc + 1), st));
    return 0;
  }
  uint32_t *iota = nullptr, *cm_keys = nullptr;
  int *cnt = nullptr, *tcam = nullptr, *tperm = nullptr;
  BAMG_CUDA_CHECK(cudaMallocAsync(&iota, 4 * k, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&cm_keys, 4 * k, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&tcam, 4 * k, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&tperm, 4 * k, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&cnt, 4 * ((size_t)npt + 1), st));
  int g = grid_for(k, 256);
  // (a) point segments by counting
  BAMG_CUDA_CHECK(cudaMemsetAsync(cnt, 0, 4 * ((size_t)npt + 1), st));
  launch(k_count_i32, g, 256, 0, st, pt_idx, k, cnt);
  int rc = scan_exclusive_int(cnt, pt_ptr, (int64_t)npt + 1, nullptr, st);
  if (rc) return rc;
  BAMG_CUDA_CHECK(cudaMemsetAsync(cnt, 0, 4 * (size_t)npt, st));
  launch(k_pt_scatter, g, 256, 0, st, cam_idx, pt_idx, k, pt_ptr, cnt, tcam, tperm);
  launch(k_segment_ids, grid_for(npt, 256), 256, 0, st, pt_ptr, npt, obs_pt_pm);
  // (b) inside each point: (camera, caller index) order
  launch(k_pt_rank, g, 256, 0, st, pt_ptr, obs_pt_pm, k, tcam, tperm, obs_cam_pm, pm_perm);
  // (c) point-major positions stably by camera -> (camera, point) order
  launch(k_iota, g, 256, 0, st, iota, k);
  rc = radix_sort_pairs((const uint32_t*)obs_cam_pm, iota, cm_keys, (uint32_t*)cm_list, k, bits_for(nc), st);
  if (rc) return rc;
  rc = segment_ptr((const int*)cm_keys, k, nc, cam_ptr, st);
  if (rc) return rc;
  BAMG_LAUNCH_CHECK();
  cudaFreeAsync(iota, st);
  cudaFreeAsync(cm_keys, st);
  cudaFreeAsync(tcam, st);
  cudaFreeAsync(tperm, st);
  cudaFreeAsync(cnt, st);
  return 0;
}

// ---------------------------------------------------------------------------
// covisibility pattern (S pattern incl. diagonal) and visibility strength

// Row i: OR a bitmap of cameras co-observing any point of camera i; the diagonal
// is always present (A is block-diagonal, schur.py:136).
__global__ void k_covis_rows(const int* __restrict__ cam_ptr, const int* __restrict__ cm_list,
                             const int* __restrict__ obs_pt_pm, const int* __restrict__ pt_ptr,
                             const int* __restrict__ obs_cam_pm, int nc, int* __restrict__ counts,
                             const int* __restrict__ S_ptr, int* __restrict__ S_col,
                             unsigned* __restrict__ bm_out) {
  extern __shared__ unsigned int bm[];
  int words = (nc + 31) >> 5;
  for (int i = blockIdx.x; i < nc; i += gridDim.x) {
    for (int w = threadIdx.x; w < words; w += blockDim.x) bm[w] = 0u;
    __syncthreads();
    if (threadIdx.x == 0) atomicOr(&bm[i >> 5], 1u << (i & 31));
    for (int q = cam_ptr[i] + threadIdx.x; q < cam_ptr[i + 1]; q += blockDim.x) {
      int p = obs_pt_pm[cm_list[q]];
      for (int o = pt_ptr[p]; o < pt_ptr[p + 1]; ++o) {
        int j = obs_cam_pm[o];
        atomicOr(&bm[j >> 5], 1u << (j & 31));
      }
    }
    __syncthreads();
    if (S_col == nullptr) {
      int c = 0;
      for (int w = threadIdx.x; w < words; w += blockDim.x) {
        c += __popc(bm[w]);
        if (bm_out) bm_out[(int64_t)i * words + w] = bm[w];
      }
      c = warp_sum_int(c);
      __shared__ int red[32];
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
      __syncthreads();
      if (threadIdx.x == 0) {
        int t = 0;
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
        counts[i] = t;
      }
    } else {
      // ordered fill: one warp walks the words, lanes compact set bits
      if (threadIdx.x < 32) {
        int lane = threadIdx.x;
        int out = S_ptr[i];
        for (int w0 = 0; w0 < words; w0 += 32) {
          int w = w0 + lane;
          unsigned v = (w < words) ? bm[w] : 0u;
          int c = __popc(v);
          int incl = c;
          for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(FULL_MASK, incl, o);
            if (lane >= o) incl += t;
          }
          int pos = out + incl - c;
          while (v) {
            int b = __ffs(v) - 1;
            v &= v - 1;
            S_col[pos++] = w * 32 + b;
          }
          out += __shfl_sync(FULL_MASK, incl, 31);
        }
      }
    }
    __syncthreads();
  }
}

// Fill from the row bitmaps the count pass kept (nc x ceil(nc/32) words): warp per
// row, lanes compact set bits in column order -- no second sweep of the observations.
__global__ void k_covis_compact(const unsigned* __restrict__ bm, int nc, const int* __restrict__ S_ptr,
                                int* __restrict__ S_col) {
  const int words = (nc + 31) >> 5;
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < nc; i += nwarps) {
    const unsigned* row = bm + (int64_t)i * words;
    int out = S_ptr[i];
    for (int w0 = 0; w0 < words; w0 += 32) {
      int w = w0 + lane;
      unsigned v = (w < words) ? row[w] : 0u;
      int c = __popc(v);
      int incl = c;
      for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(FULL_MASK, incl, o);
        if (lane >= o) incl += t;
      }
      int pos = out + incl - c;
      while (v) {
        int b = __ffs(v) - 1;
        v &= v - 1;
        S_col[pos++] = w * 32 + b;
      }
      out += __shfl_sync(FULL_MASK, incl, 31);
    }
  }
}

extern "C" int bamg_covis_count_keep(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list,
                                     const int32_t* obs_pt_pm, const int32_t* pt_ptr, const int32_t* obs_cam_pm,
                                     int32_t nc, int32_t* row_counts, uint32_t* bitmaps, void* stream) {
  (void)ctx;
  size_t sm = sizeof(unsigned) * ((nc + 31) / 32);
  if (sm > 200 * 1024) {
    bamg_set_error("covisibility bitmap for %d cameras exceeds shared memory", nc);
    return BAMG_ERR_UNSUPPORTED;
  }
  if (sm > 48 * 1024) cudaFuncSetAttribute(k_covis_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  launch(k_covis_rows, grid_for(nc, 1, 16), 256, sm, as_stream(stream), cam_ptr, cm_list, obs_pt_pm, pt_ptr,
         obs_cam_pm, nc, row_counts, nullptr, nullptr, bitmaps);
  BAMG_LAUNCH_CHECK();
  return 0;
}

extern "C" int bamg_covis_compact(bamg_ctx* ctx, const uint32_t* bitmaps, int32_t nc, const int32_t* S_ptr,
                                  int32_t* S_col, void* stream) {
  (void)ctx;
  if (nc <= 0) return 0;
  launch(k_covis_compact, grid_for((int64_t)nc * 32, 256), 256, 0, as_stream(stream), bitmaps, nc, S_ptr, S_col);
  BAMG_LAUNCH_CHECK();
  return 0;
}

extern "C" int bamg_covis_count(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list,
                                const int32_t* obs_pt_pm, const int32_t* pt_ptr, const int32_t* obs_cam_pm,
                                int32_t nc, int32_t* row_counts, void* stream) {
  (void)ctx;
  size_t sm = sizeof(unsigned) * ((nc + 31) / 32);
  if (sm > 200 * 1024) {
    bamg_set_error("covisibility bitmap for %d cameras exceeds shared memory", nc);
    return BAMG_ERR_UNSUPPORTED;
  }
  if (sm > 48 * 1024) cudaFuncSetAttribute(k_covis_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  launch(k_covis_rows, grid_for(nc, 1, 16), 256, sm, as_stream(stream), cam_ptr, cm_list, obs_pt_pm, pt_ptr,
         obs_cam_pm, nc, row_counts, nullptr, nullptr, nullptr);
  BAMG_LAUNCH_CHECK();
  return 0;
}

extern "C" int bamg_covis_fill(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list,
                               const int32_t* obs_pt_pm, const int32_t* pt_ptr, const int32_t* obs_cam_pm,
                               int32_t nc, const int32_t* S_ptr, int32_t* S_col, void* stream) {
  (void)ctx;
  size_t sm = sizeof(unsigned) * ((nc + 31) / 32);
  if (sm > 48 * 1024) cudaFuncSetAttribute(k_covis_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  launch(k_covis_rows, grid_for(nc, 1, 16), 256, sm, as_stream(stream), cam_ptr, cm_list, obs_pt_pm, pt_ptr,
         obs_cam_pm, nc, nullptr, S_ptr, S_col, nullptr);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// Shared-point counts per covisibility slot (diagonal = degree), exact integers.
__global__ void k_shared_counts(const int* __restrict__ cam_ptr, const int* __restrict__ cm_list,
                                const int* __restrict__ obs_pt_pm, const int* __restrict__ pt_ptr,
                                const int* __restrict__ obs_cam_pm, int nc, const int* __restrict__ S_ptr,
                                const int* __restrict__ S_col, int* __restrict__ shared_cnt) {
  extern __shared__ int sm_i[];
  for (int i = blockIdx.x; i < nc; i += gridDim.x) {
    int b = S_ptr[i], n = S_ptr[i + 1] - b;
    int* cols = sm_i;
    int* cnt = sm_i + n;
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
      cols[q] = S_col[b + q];
      cnt[q] = 0;
    }
    __syncthreads();
    for (int q = cam_ptr[i] + threadIdx.x; q < cam_ptr[i + 1]; q += blockDim.x) {
      int p = obs_pt_pm[cm_list[q]];
      for (int o = pt_ptr[p]; o < pt_ptr[p + 1]; ++o) {
        int s = lower_bound_i32(cols, n, obs_cam_pm[o]);
        atomicAdd(&cnt[s], 1);
      }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < n; q += blockDim.x) shared_cnt[b + q] = cnt[q];
    __syncthreads();
  }
}

extern "C" int bamg_shared_counts(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list,
                                  const int32_t* obs_pt_pm, const int32_t* pt_ptr, const int32_t* obs_cam_pm,
                                  int32_t nc, const int32_t* S_ptr, const int32_t* S_col, int32_t max_row,
                                  int32_t* shared_cnt, void* stream) {
  (void)ctx;
  size_t sm = sizeof(int) * 2 * (size_t)max_row;
  if (sm > 200 * 1024) {
    bamg_set_error("covisibility row of %d blocks exceeds shared memory", max_row);
    return BAMG_ERR_UNSUPPORTED;
  }
  if (sm > 48 * 1024) cudaFuncSetAttribute(k_shared_counts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  launch(k_shared_counts, grid_for(nc, 1, 16), 256, sm, as_stream(stream), cam_ptr, cm_list, obs_pt_pm, pt_ptr,
                                                                       obs_cam_pm, nc, S_ptr, S_col, shared_cnt);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// Visibility strength (multigrid.py:52-80): G_ij = min(shared / sqrt(deg_i deg_j), 1)
// for i != j, stored on the covisibility pattern minus the diagonal. Exact integer
// counts + IEEE sqrt/div => bit-identical to the reference. Also counts the
// int8-wrapped covisibility blocks of schur.py:151-159 (slots with shared % 256 != 0).
__global__ void k_visibility_strength(const int* __restrict__ S_ptr, const int* __restrict__ S_col,
                                      const int* __restrict__ shared_cnt, int nc, int* __restrict__ G_ptr,
                                      int* __restrict__ G_col, double* __restrict__ G_val,
                                      int* __restrict__ wrapped_count) {
  int local = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
    int b = S_ptr[i], e = S_ptr[i + 1];
    int out = b - i;  // every row holds exactly one (forced) diagonal slot
    G_ptr[i] = out;
    if (i == nc - 1) G_ptr[nc] = e - nc;
    for (int q = b; q < e; ++q) {
      int j = S_col[q];
      int c = shared_cnt[q];
      if ((c & 255) != 0) ++local;
      if (j == i) continue;
      G_col[out] = j;
      G_val[out] = (double)c;  // finished by k_strength_scale
      ++out;
    }
  }
  local = warp_sum_int(local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(wrapped_count, local);
}

__global__ void k_strength_scale(const int* __restrict__ G_ptr, const int* __restrict__ G_col,
                                 const int* __restrict__ deg, int nc, double* __restrict__ G_val) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
    double di = (double)deg[i];
    for (int q = G_ptr[i]; q < G_ptr[i + 1]; ++q) {
      double scale = sqrt(di * (double)deg[G_col[q]]);
      double v = G_val[q] / scale;
      G_val[q] = v < 1.0 ? v : 1.0;
    }
  }
}

__global__ void k_degrees(const int* __restrict__ cam_ptr, int nc, int* __restrict__ deg, int* __restrict__ zero) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
    int d = cam_ptr[i + 1] - cam_ptr[i];
    deg[i] = d;
    if (d == 0) atomicAdd(zero, 1);
  }
}

// Outputs: G (CSR without diagonal), degrees, flags[0] = #cameras with no points,
// flags[1] = int8-wrapped covisibility block count. Host reads flags.
extern "C" int bamg_visibility_strength(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* S_ptr,
                                        const int32_t* S_col, const int32_t* shared_cnt, int32_t nc,
                                        int32_t* deg, int32_t* G_ptr, int32_t* G_col, double* G_val,
                                        int32_t* flags_dev, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  BAMG_CUDA_CHECK(cudaMemsetAsync(flags_dev, 0, 2 * sizeof(int), st));
  int g = grid_for(nc, 128);
  launch(k_degrees, g, 128, 0, st, cam_ptr, nc, deg, flags_dev);
  launch(k_visibility_strength, g, 128, 0, st, S_ptr, S_col, shared_cnt, nc, G_ptr, G_col, G_val, flags_dev + 1);
  launch(k_strength_scale, g, 128, 0, st, G_ptr, G_col, deg, nc, G_val);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------------------
// residuals and Jacobians (problem.py:202-219, 272-326; rotation.py:36-114)

struct CamModel {
  double R[9];   // rotation matrix (rotation.py:61-71)
  double Jr[9];  // right Jacobian (rotation.py:74-88)
  double s1, s2;
};

__device__ __forceinline__ void rot_coeffs(const double* aa, double& a2, double& s1, double& s2, double& c2,
                                           bool& small) {
  a2 = aa[0] * aa[0] + aa[1] * aa[1] + aa[2] * aa[2];
  double a = sqrt(a2);
  small = a < 1e-4;
  if (small) {
    s1 = 1.0 - a2 / 6.0;
    s2 = 0.5 - a2 / 24.0;
    c2 = 1.0 / 6.0 - a2 / 120.0;
  } else {
    double sn, cs;
    sincos(a, &sn, &cs);
    s1 = sn / a;
    s2 = (1.0 - cs) / a2;
    c2 = (a - sn) / (a2 * a);
  }
}

__device__ __forceinline__ void hat(const double* v, double* K) {
  K[0] = 0.0;   K[1] = -v[2]; K[2] = v[1];
  K[3] = v[2];  K[4] = 0.0;   K[5] = -v[0];
  K[6] = -v[1]; K[7] = v[0];  K[8] = 0.0;
}

__device__ __forceinline__ void mm3(const double* A, const double* B, double* C) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) C[i * 3 + j] = A[i * 3] * B[j] + A[i * 3 + 1] * B[3 + j] + A[i * 3 + 2] * B[6 + j];
}

struct ProjOut {
  double pc[3], p[2], n2, dist, res[2], s;
};

__device__ __forceinline__ bool project_one(const double* __restrict__ cam, const double* __restrict__ X,
                                            const double* __restrict__ pix, ProjOut& o) {
  const double* aa = cam;
  double a2, s1, s2, c2;
  bool small;
  rot_coeffs(aa, a2, s1, s2, c2, small);
  // rotate(): X + s1 (aa x X) + s2 (aa x (aa x X))
  double c1v[3] = {aa[1] * X[2] - aa[2] * X[1], aa[2] * X[0] - aa[0] * X[2], aa[0] * X[1] - aa[1] * X[0]};
  double c2v[3] = {aa[1] * c1v[2] - aa[2] * c1v[1], aa[2] * c1v[0] - aa[0] * c1v[2], aa[0] * c1v[1] - aa[1] * c1v[0]};
#pragma unroll
  for (int d = 0; d < 3; ++d) o.pc[d] = (X[d] + s1 * c1v[d] + s2 * c2v[d]) + cam[3 + d];
  double z = o.pc[2];
  if (z >= -1e-12) return false;  // problem.py:211 (bad = z >= -eps)
  o.p[0] = -o.pc[0] / z;
  o.p[1] = -o.pc[1] / z;
  o.n2 = o.p[0] * o.p[0] + o.p[1] * o.p[1];
  double k1 = cam[7], k2 = cam[8], f = cam[6];
  o.dist = 1.0 + k1 * o.n2 + k2 * o.n2 * o.n2;
  double fd = f * o.dist;
  o.res[0] = fd * o.p[0] - pix[0];
  o.res[1] = fd * o.p[1] - pix[1];
  o.s = o.res[0] * o.res[0] + o.res[1] * o.res[1];
  return true;
}

__device__ __forceinline__ double loss_rho(double s, int huber) {
  if (!huber) return s;
  return s <= 1.0 ? s : 2.0 * sqrt(fmax(s, 1.0)) - 1.0;
}

__device__ __forceinline__ double loss_w(double s, int huber) {
  if (!huber) return 1.0;
  return s <= 1.0 ? 1.0 : pow(fmax(s, 1.0), -0.25);
}

// ---------------------------------------------------------------------------
// Observation records. Everything the assembly reads per observation lives in one
// 256 B record (two full cache lines, 16 B aligned):
//   [ 0,18) F (2x9)   [18,24) E (2x3)   [24,30) H = E C^-1 (2x3)   [30,32) residual
// Kernels that visit observations in camera order gather whole records with
// warp-cooperative double2 loads staged through shared memory, so every load
// instruction touches a few cache lines instead of 32.
#define EVAL_THREADS 128
#ifndef EVAL_ZERO_H
#define EVAL_ZERO_H 1
#endif
#define EVAL_STRIDE 33  // odd smem stride: conflict-free per-thread record writes

// One thread per observation (point-major); the CTA's records are staged in shared
// memory and written back as contiguous double2 stores (H slots untouched). The
// objective is reduced deterministically (last block finishes).
#ifndef EVAL_MINB
// 1: 138 registers, 12 warps per SM. 4 (128 registers, 16 warps) runs 2.11 -> 1.71 ms at
// c4, but ptxas then contracts differently: F moves by ulps, enough to move the
// visibility-Jacobi PCG solutions of the reference-pinned tests past their bounds.
#define EVAL_MINB 1
#endif
__global__ void __launch_bounds__(EVAL_THREADS, EVAL_MINB)
k_evaluate(const double* __restrict__ cams, const double* __restrict__ pts, const int* __restrict__ ocam,
           const int* __restrict__ opt, const double* __restrict__ pix, int64_t k, int huber, int with_jac,
           double* __restrict__ J, double* __restrict__ w, unsigned char* __restrict__ behind,
           int* __restrict__ n_behind, double* partials, unsigned int* counter, double* objective) {
  __shared__ double scratch[33];
  __shared__ double rec[EVAL_THREADS * EVAL_STRIDE];
  double acc = 0.0;
  int nb = 0;
  double* my = rec + threadIdx.x * EVAL_STRIDE;
  // Software pipeline over the grid-stride tiles: the (camera, point, pixel) inputs of
  // tile i+1 are gathered while tile i is written back, so the index -> parameter
  // load chain (a DRAM then an L2 latency) no longer sits in front of every tile.
  const int64_t stride = (int64_t)gridDim.x * EVAL_THREADS;
  // Indices run two tiles ahead, parameters one tile ahead.
  double cam[9], X[3], px[2];
  int ic = 0, ip = 0;  // indices of the next tile to gather
  auto load_idx = [&](int64_t tt) {
    if (tt < k) {
      ic = __ldg(ocam + tt);
      ip = __ldg(opt + tt);
    }
  };
  auto gather = [&](int64_t tt) {
    if (tt < k) {
      const double2* c = reinterpret_cast<const double2*>(cams + (int64_t)ic * 10);  // padded rows
      const double* x = pts + (int64_t)ip * 3;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double2 v = __ldg(c + q);
        cam[2 * q] = v.x;
        cam[2 * q + 1] = v.y;
      }
      cam[8] = __ldg(cams + (int64_t)ic * 10 + 8);
#pragma unroll
      for (int q = 0; q < 3; ++q) X[q] = __ldg(x + q);
      px[0] = __ldg(pix + 2 * tt);
      px[1] = __ldg(pix + 2 * tt + 1);
    }
  };
  {
    int64_t t0 = (int64_t)blockIdx.x * EVAL_THREADS + threadIdx.x;
    load_idx(t0);
    gather(t0);
    load_idx(t0 + stride);
  }
  for (int64_t base = (int64_t)blockIdx.x * EVAL_THREADS; base < k; base += stride) {
    int64_t t = base + threadIdx.x;
    if (t < k) {
      ProjOut o;
      bool ok = project_one(cam, X, px, o);
      if (behind) behind[t] = ok ? 0 : 1;
      if (!ok) {
        ++nb;
        if (with_jac) {
          for (int q = 0; q < REC; ++q) my[q] = 0.0;
          w[t] = 0.0;
        }
      } else {
        acc += loss_rho(o.s, huber);
        if (with_jac) {
          double wt = loss_w(o.s, huber);
          double z = o.pc[2];
          double f = cam[6], k1 = cam[7], k2 = cam[8];
          double iz = -1.0 / z;
          double z2 = z * z;
          double dp[6] = {iz, 0.0, o.pc[0] / z2, 0.0, iz, o.pc[1] / z2};
          double coef = f * (2.0 * k1 + 4.0 * k2 * o.n2);
          double fd = f * o.dist;
          double M[4] = {fd + coef * o.p[0] * o.p[0], coef * o.p[0] * o.p[1], coef * o.p[1] * o.p[0],
                         fd + coef * o.p[1] * o.p[1]};
          double Dm[6];
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) Dm[r * 3 + c] = M[r * 2] * dp[c] + M[r * 2 + 1] * dp[3 + c];
          const double* aa = cam;
          double a2, s1, s2, c2;
          bool small;
          rot_coeffs(aa, a2, s1, s2, c2, small);
          double K[9], K2[9];
          hat(aa, K);
          mm3(K, K, K2);
          double R[9], Jr[9];
#pragma unroll
          for (int q = 0; q < 9; ++q) {
            double I = (q % 4 == 0) ? 1.0 : 0.0;
            R[q] = I + s1 * K[q] + s2 * K2[q];
            Jr[q] = I - s2 * K[q] + c2 * K2[q];
          }
          double HX[9], T1[9], RJ[9];
          hat(X, HX);
          mm3(R, HX, T1);
          mm3(T1, Jr, RJ);
#pragma unroll
          for (int r = 0; r < 2; ++r) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              double v = -(Dm[r * 3] * RJ[c] + Dm[r * 3 + 1] * RJ[3 + c] + Dm[r * 3 + 2] * RJ[6 + c]);
              my[RF + r * 9 + c] = v * wt;
              my[RF + r * 9 + 3 + c] = Dm[r * 3 + c] * wt;
              my[RE + r * 3 + c] = (Dm[r * 3] * R[c] + Dm[r * 3 + 1] * R[3 + c] + Dm[r * 3 + 2] * R[6 + c]) * wt;
            }
            my[RF + r * 9 + 6] = (o.dist * o.p[r]) * wt;
            my[RF + r * 9 + 7] = ((f * o.n2) * o.p[r]) * wt;
            my[RF + r * 9 + 8] = ((f * o.n2 * o.n2) * o.p[r]) * wt;
          }
          my[RR] = o.res[0] * wt;
          my[RR + 1] = o.res[1] * wt;
          w[t] = wt;
        }
      }
    }
    gather(t + stride);  // next tile's inputs in flight during the write-back
    load_idx(t + 2 * stride);
    if (with_jac) {
      __syncthreads();
      // coalesced write-back of the CTA's records, all 16 double2 each: the H slots
      // (pieces 12..14, filled by build_system's k_obs_H before any use) are written
      // as zeros, so every 32 B sector is written whole -- skipping them left the
      // sector shared by H and the residual partially written (an L2 read-modify-write
      // from DRAM per observation)
      int nrec = (int)min((int64_t)EVAL_THREADS, k - base);
      double2* dst = reinterpret_cast<double2*>(J + base * REC);
      for (int g = threadIdx.x; g < nrec * 16; g += EVAL_THREADS) {
        int rr = g >> 4, pc = g & 15;
        if (pc >= 12 && pc < 15) {
          if (EVAL_ZERO_H) dst[g] = make_double2(0.0, 0.0);
          continue;
        }
        const double* s = rec + rr * EVAL_STRIDE + 2 * pc;
        dst[g] = make_double2(s[0], s[1]);
      }
      __syncthreads();
    }
  }
  nb = warp_sum_int(nb);
  if ((threadIdx.x & 31) == 0 && nb) atomicAdd(n_behind, nb);
  acc = block_sum(acc, scratch);
  grid_finish(partials, counter, acc, scratch, objective);
}

extern "C" int bamg_evaluate(bamg_ctx* ctx, const double* cams, int32_t nc, const double* pts, const int32_t* obs_cam,
                             const int32_t* obs_pt, const double* pixels, int64_t k, int32_t huber,
                             int32_t with_jacobian, double* J, double* w, uint8_t* behind, double* objective_dev,
                             int32_t* n_behind_dev, void* stream) {
  cudaStream_t st = as_stream(stream);
  BAMG_CUDA_CHECK(cudaMemsetAsync(n_behind_dev, 0, sizeof(int), st));
  int g = grid_for(k, EVAL_THREADS, 8);
  double* cams10 = nullptr;  // camera rows padded to 80 B
  BAMG_CUDA_CHECK(cudaMallocAsync(&cams10, sizeof(double) * 10 * (size_t)(nc > 0 ? nc : 1), st));
  if (nc > 0) pad9(cams, nc, cams10, st);
  launch(k_evaluate, g, EVAL_THREADS, 0, st, (const double*)cams10, pts, obs_cam, obs_pt, pixels, k, huber,
         with_jacobian, J, w, behind, n_behind_dev, ctx->partials, ctx->counters + BAMG_CTR_OBJ, objective_dev);
  BAMG_CUDA_CHECK(cudaFreeAsync(cams10, st));
  BAMG_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------------------
// normal-equation blocks (problem.py:255-269, schur.py:104-112)

#define CN_ST 21  // 9 F pieces + residual piece = 20 doubles, odd stride
#ifndef CN_STAGES
#define CN_STAGES 4  // chunks of 32 records in flight per warp (k_cam_normal)
#endif

// Warp per camera: A_raw = sum F^T F (full 9x9), g = sum F^T r.
__global__ void __launch_bounds__(128)
k_cam_normal(const int* __restrict__ cam_ptr, const int* __restrict__ cm_list, const double* __restrict__ J, int nc,
             double* __restrict__ A_raw, double* __restrict__ g_cam) {
  // CN_STAGES chunk buffers per warp (rec_issue layout): F pieces 0..8, residual 9
  extern __shared__ __align__(16) double cn_smem[];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* wbuf = cn_smem + (size_t)w * CN_STAGES * 640;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < nc; i += nwarps) {
    double a[45];
    double g[9];
#pragma unroll
    for (int q = 0; q < 45; ++q) a[q] = 0.0;
#pragma unroll
    for (int q = 0; q < 9; ++q) g[q] = 0.0;
    const int q0 = cam_ptr[i], q1 = cam_ptr[i + 1];
#pragma unroll
    for (int s = 0; s < CN_STAGES - 1; ++s) {  // prologue: chunks 0 .. CN_STAGES-2
      int cb = q0 + 32 * s;
      if (cb < q1) {
        bool v = cb + lane < q1;
        rec_issue<9, 1, 0>(J, v ? cm_list[cb + lane] : 0, v, 0, RR / 2, nullptr, wbuf + s * 640, lane);
      } else {
        cp_async_commit();
      }
    }
    int c = 0;
    // observation ids of the next chunk to issue, loaded one iteration ahead so the
    // copies never wait on the index load
    int nidx = (q0 + 32 * (CN_STAGES - 1) + lane < q1) ? cm_list[q0 + 32 * (CN_STAGES - 1) + lane] : 0;
    for (int base = q0; base < q1; base += 32, ++c) {
      // chunk c + CN_STAGES - 1 goes out before chunk c is consumed
      int nb = base + 32 * (CN_STAGES - 1);
      if (nb < q1) {
        bool vn = nb + lane < q1;
        rec_issue<9, 1, 0>(J, nidx, vn, 0, RR / 2, nullptr,
                           wbuf + ((c + CN_STAGES - 1) % CN_STAGES) * 640, lane);
      } else {
        cp_async_commit();
      }
      {
        int pb = nb + 32;
        nidx = (pb + lane < q1) ? cm_list[pb + lane] : 0;
      }
      cp_async_wait<CN_STAGES - 1>();
      __syncwarp();
      bool valid = base + lane < q1;
      const double* b = wbuf + (c % CN_STAGES) * 640 + 2 * lane;
      if (valid) {
        double f[18];
#pragma unroll
        for (int j = 0; j < 9; ++j) {
          f[2 * j] = b[j * 64];
          f[2 * j + 1] = b[j * 64 + 1];
        }
        double r0 = b[9 * 64], r1 = b[9 * 64 + 1];
        int t = 0;
#pragma unroll
        for (int j = 0; j < 9; ++j) {
          double f0j = f[j], f1j = f[9 + j];
#pragma unroll
          for (int l = j; l < 9; ++l) a[t++] += f0j * f[l] + f1j * f[9 + l];
          g[j] += f0j * r0 + f1j * r1;
        }
      }
      __syncwarp();
    }
    cp_async_wait<0>();
#pragma unroll
    for (int q = 0; q < 45; ++q) a[q] = warp_sum(a[q]);
#pragma unroll
    for (int q = 0; q < 9; ++q) g[q] = warp_sum(g[q]);
    if (lane == 0) {
      double* out = A_raw + (int64_t)i * 81;
      int t = 0;
#pragma unroll
      for (int j = 0; j < 9; ++j)
#pragma unroll
        for (int l = j; l < 9; ++l) {
          out[j * 9 + l] = a[t];
          out[l * 9 + j] = a[t];
          ++t;
        }
#pragma unroll
      for (int j = 0; j < 9; ++j) g_cam[(int64_t)i * 9 + j] = g[j];
    }
  }
}

// Thread per point: C_raw = sum E^T E (3x3), g_pt = sum E^T r.
__global__ void k_pt_normal(const int* __restrict__ pt_ptr, const double* __restrict__ J, int npt,
                            double* __restrict__ C_raw, double* __restrict__ g_pt) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < npt; p += gridDim.x * blockDim.x) {
    double c[6] = {0, 0, 0, 0, 0, 0}, g[3] = {0, 0, 0};
    for (int o = pt_ptr[p]; o < pt_ptr[p + 1]; ++o) {
      const double2* rp = reinterpret_cast<const double2*>(J + (int64_t)o * REC);
      double2 e01 = __ldg(rp + RE / 2), e23 = __ldg(rp + RE / 2 + 1), e45 = __ldg(rp + RE / 2 + 2);
      double2 rr = __ldg(rp + RR / 2);
      double e[6] = {e01.x, e01.y, e23.x, e23.y, e45.x, e45.y};
      int t = 0;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
#pragma unroll
        for (int l = j; l < 3; ++l) c[t++] += e[j] * e[l] + e[3 + j] * e[3 + l];
        g[j] += e[j] * rr.x + e[3 + j] * rr.y;
      }
    }
    double* out = C_raw + (int64_t)p * 9;
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2];
    out[3] = c[1]; out[4] = c[3]; out[5] = c[4];
    out[6] = c[2]; out[7] = c[4]; out[8] = c[5];
    g_pt[3 * p] = g[0];
    g_pt[3 * p + 1] = g[1];
    g_pt[3 * p + 2] = g[2];
  }
}

extern "C" int bamg_normal_blocks(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list,
                                  const int32_t* pt_ptr, const double* J, int32_t nc, int32_t npt, double* A_raw,
                                  double* g_cam, double* C_raw, double* g_pt, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (nc > 0) {
    const size_t sm = sizeof(double) * 4 * CN_STAGES * 640;
    static bool attr = false;
    if (!attr) {
      BAMG_CUDA_CHECK(cudaFuncSetAttribute(k_cam_normal, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      attr = true;
    }
    launch(k_cam_normal, grid_for((int64_t)nc * 32, 128, 8), 128, sm, st, cam_ptr, cm_list, J, nc, A_raw, g_cam);
    BAMG_LAUNCH_CHECK();
  }
  if (npt > 0) {
    launch(k_pt_normal, grid_for(npt, 128, 16), 128, 0, st, pt_ptr, J, npt, C_raw, g_pt);
    BAMG_LAUNCH_CHECK();
  }
  return 0;
}

// Damping (schur.py:38-47): clip(diag, 1e-6, 1e32) / radius.
__global__ void k_damping(const double* __restrict__ raw, int n, int bs, double radius, double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)n * bs; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = t / bs;
    int j = (int)(t - b * bs);
    double d = raw[b * bs * bs + j * (bs + 1)];
    d = fmin(fmax(d, 1e-6), 1e32);
    if (d != d) d = raw[b * bs * bs + j * (bs + 1)];
    out[t] = d / radius;
  }
}

extern "C" int bamg_damping(bamg_ctx* ctx, const double* A_raw, const double* C_raw, int32_t nc, int32_t npt,
                            double radius, double* d_cam, double* d_pt, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (nc) launch(k_damping, grid_for((int64_t)nc * 9, 256), 256, 0, st, A_raw, nc, 9, radius, d_cam);
  if (npt) launch(k_damping, grid_for((int64_t)npt * 3, 256), 256, 0, st, C_raw, npt, 3, radius, d_pt);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// A = A_raw + diag(d_cam)
__global__ void k_add_diag(const double* __restrict__ raw, const double* __restrict__ d, int n, int bs,
                           double* __restrict__ out) {
  int64_t tot = (int64_t)n * bs * bs;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = t / (bs * bs);
    int q = (int)(t - b * bs * bs);
    int r = q / bs, c = q - r * bs;
    out[t] = raw[t] + (r == c ? d[b * bs + r] : 0.0);
  }
}

// A = A_raw + diag(d) for n blocks of size bs (the damped camera blocks on demand)
extern "C" int bamg_add_block_diag(bamg_ctx* ctx, const double* raw, const double* d, int32_t n, int32_t bs,
                                   double* out, void* stream) {
  (void)ctx;
  if (n > 0)
    launch(k_add_diag, grid_for((int64_t)n * bs * bs, 256), 256, 0, as_stream(stream), raw, d, n, bs, out);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// 3x3 Cholesky + L^-T L^-1 (blockmat.py:95-115). Returns false if not PD.
__device__ __forceinline__ bool chol_inv3(const double* C, double* Ci) {
  double l00 = C[0];
  if (!(l00 > 0.0)) return false;
  l00 = sqrt(l00);
  double l10 = C[3] / l00, l20 = C[6] / l00;
  double d1 = C[4] - l10 * l10;
  if (!(d1 > 0.0)) return false;
  double l11 = sqrt(d1);
  double l21 = (C[7] - l20 * l10) / l11;
  double d2 = C[8] - l20 * l20 - l21 * l21;
  if (!(d2 > 0.0)) return false;
  double l22 = sqrt(d2);
  double m00 = 1.0 / l00, m11 = 1.0 / l11, m22 = 1.0 / l22;
  double m10 = -l10 * m00 / l11;
  double m21 = -l21 * m11 / l22;
  double m20 = -(l20 * m00 + l21 * m10) / l22;
  Ci[0] = m00 * m00 + m10 * m10 + m20 * m20;
  Ci[1] = m10 * m11 + m20 * m21;
  Ci[2] = m20 * m22;
  Ci[4] = m11 * m11 + m21 * m21;
  Ci[5] = m21 * m22;
  Ci[8] = m22 * m22;
  Ci[3] = Ci[1];
  Ci[6] = Ci[2];
  Ci[7] = Ci[5];
  return true;
}

// Thread per observation: H = E C_p^-1 (into the record) and q = E C_p^-1 b_p.
__global__ void k_obs_H(const int* __restrict__ opt, const double* __restrict__ Cinv, const double* __restrict__ Cb,
                        int64_t k, double* __restrict__ J, double* __restrict__ qo) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < k; o += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = opt[o];
    double2* rp = reinterpret_cast<double2*>(J + o * REC);
    double2 e01 = rp[RE / 2], e23 = rp[RE / 2 + 1], e45 = rp[RE / 2 + 2];
    double2 res = rp[RR / 2];  // rewritten with H[4..5]: the shared sector is stored whole
    double e[6] = {e01.x, e01.y, e23.x, e23.y, e45.x, e45.y};
    const double* ci = Cinv + p * 9;
    double x0 = Cb[3 * p], x1 = Cb[3 * p + 1], x2 = Cb[3 * p + 2];
    double h[6];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int cc = 0; cc < 3; ++cc)
        h[r * 3 + cc] = e[r * 3] * ci[cc] + e[r * 3 + 1] * ci[3 + cc] + e[r * 3 + 2] * ci[6 + cc];
    rp[RH / 2] = make_double2(h[0], h[1]);
    rp[RH / 2 + 1] = make_double2(h[2], h[3]);
    rp[RH / 2 + 2] = make_double2(h[4], h[5]);
    rp[RR / 2] = res;
    reinterpret_cast<double2*>(qo)[o] =
        make_double2(e[0] * x0 + e[1] * x1 + e[2] * x2, e[3] * x0 + e[4] * x1 + e[5] * x2);
  }
}

// k_points_factor + k_obs_H in one pass: 32 consecutive points per warp, a lane per
// point factors C (C = C_raw + D_p, batched 3x3 Cholesky inverse, b_p = -g_p), parks C^-1 and C^-1 b_p in
// shared memory, then the lanes walk the points' contiguous observations (coalesced
// record accesses) and form H = E C^-1 and q = E C^-1 b_p (same arithmetic as k_obs_H).
__global__ void __launch_bounds__(128)
k_points_H_warp(const int* __restrict__ pt_ptr, const double* __restrict__ C_raw, const double* __restrict__ d_pt,
                const double* __restrict__ g_pt, int npt, double* __restrict__ C, double* __restrict__ Cinv,
                double* __restrict__ Cb, int* __restrict__ bad_min, double* __restrict__ J, double* __restrict__ qo) {
  __shared__ double cib[4][32 * 12];
  __shared__ int sbuf[4][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int p0 = warp * 32; p0 < npt; p0 += nwarps * 32) {
    const int np = min(32, npt - p0);
    const int p = p0 + lane;
    if (lane < np) sbuf[w][lane] = pt_ptr[p0 + lane];
    if (lane == 0) sbuf[w][np] = pt_ptr[p0 + np];
    if (lane < np) {
      double c[9], ci[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) c[q] = C_raw[(int64_t)p * 9 + q];
      c[0] += d_pt[3 * p];
      c[4] += d_pt[3 * p + 1];
      c[8] += d_pt[3 * p + 2];
#pragma unroll
      for (int q = 0; q < 9; ++q) C[(int64_t)p * 9 + q] = c[q];
      if (!chol_inv3(c, ci)) {
        atomicMin(bad_min, p);
#pragma unroll
        for (int q = 0; q < 9; ++q) ci[q] = 0.0;
      }
#pragma unroll
      for (int q = 0; q < 9; ++q) Cinv[(int64_t)p * 9 + q] = ci[q];
      double b0 = -g_pt[3 * p], b1 = -g_pt[3 * p + 1], b2 = -g_pt[3 * p + 2];
      double x0 = ci[0] * b0 + ci[1] * b1 + ci[2] * b2;
      double x1 = ci[3] * b0 + ci[4] * b1 + ci[5] * b2;
      double x2 = ci[6] * b0 + ci[7] * b1 + ci[8] * b2;
      Cb[3 * p] = x0;
      Cb[3 * p + 1] = x1;
      Cb[3 * p + 2] = x2;
      double* cb = cib[w] + 12 * lane;
#pragma unroll
      for (int q = 0; q < 9; ++q) cb[q] = ci[q];
      cb[9] = x0;
      cb[10] = x1;
      cb[11] = x2;
    }
    __syncwarp();
    const int r0 = sbuf[w][0], r1 = sbuf[w][np];
    for (int o = r0 + lane; o < r1; o += 32) {
      int lo = 0, hi = np;
      while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (sbuf[w][mid] <= o) lo = mid; else hi = mid;
      }
      const double* ci = cib[w] + 12 * lo;
      double2* rp = reinterpret_cast<double2*>(J + (int64_t)o * REC);
      double2 e01 = rp[RE / 2], e23 = rp[RE / 2 + 1], e45 = rp[RE / 2 + 2];
      double2 res = rp[RR / 2];  // rewritten with H[4..5]: the shared sector is stored whole
      double e[6] = {e01.x, e01.y, e23.x, e23.y, e45.x, e45.y};
      double h[6];
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int cc = 0; cc < 3; ++cc)
          h[r * 3 + cc] = e[r * 3] * ci[cc] + e[r * 3 + 1] * ci[3 + cc] + e[r * 3 + 2] * ci[6 + cc];
      rp[RH / 2] = make_double2(h[0], h[1]);
      rp[RH / 2 + 1] = make_double2(h[2], h[3]);
      rp[RH / 2 + 2] = make_double2(h[4], h[5]);
      rp[RR / 2] = res;
      reinterpret_cast<double2*>(qo)[o] =
          make_double2(e[0] * ci[9] + e[1] * ci[10] + e[2] * ci[11], e[3] * ci[9] + e[4] * ci[10] + e[5] * ci[11]);
    }
    __syncwarp();
  }
}

// Warp per camera: out_i = -g_i - sum_o F_o^T q_o   (schur.py:122 rhs), or with
// A != null: out_i = A_i x_i - sum_o F_o^T q_o (implicit matvec, schur.py:84-86).
__global__ void __launch_bounds__(128)
k_cam_gather(const int* __restrict__ cam_ptr, const int* __restrict__ cm_list, const double* __restrict__ J,
             const double* __restrict__ qo, const double* __restrict__ g_cam, const double* __restrict__ A,
             const double* __restrict__ x, int nc, double* __restrict__ out) {
  // the k_cam_normal pipeline: F pieces 0..8 of the record + this obs's q (piece 9)
  extern __shared__ __align__(16) double cn_smem[];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* wbuf = cn_smem + (size_t)w * CN_STAGES * 640;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < nc; i += nwarps) {
    double s[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) s[j] = 0.0;
    const int q0 = cam_ptr[i], q1 = cam_ptr[i + 1];
#pragma unroll
    for (int st = 0; st < CN_STAGES - 1; ++st) {
      int cb = q0 + 32 * st;
      if (cb < q1) {
        bool v = cb + lane < q1;
        rec_issue<9, 0, 1>(J, v ? cm_list[cb + lane] : 0, v, 0, 0, qo, wbuf + st * 640, lane);
      } else {
        cp_async_commit();
      }
    }
    int c = 0;
    // observation ids of the next chunk to issue, loaded one iteration ahead so the
    // copies never wait on the index load
    int nidx = (q0 + 32 * (CN_STAGES - 1) + lane < q1) ? cm_list[q0 + 32 * (CN_STAGES - 1) + lane] : 0;
    for (int base = q0; base < q1; base += 32, ++c) {
      int nb = base + 32 * (CN_STAGES - 1);
      if (nb < q1) {
        bool vn = nb + lane < q1;
        rec_issue<9, 0, 1>(J, nidx, vn, 0, 0, qo,
                           wbuf + ((c + CN_STAGES - 1) % CN_STAGES) * 640, lane);
      } else {
        cp_async_commit();
      }
      {
        int pb = nb + 32;
        nidx = (pb + lane < q1) ? cm_list[pb + lane] : 0;
      }
      cp_async_wait<CN_STAGES - 1>();
      __syncwarp();
      bool valid = base + lane < q1;
      const double* b = wbuf + (c % CN_STAGES) * 640 + 2 * lane;
      if (valid) {
        double f[18];
#pragma unroll
        for (int j = 0; j < 9; ++j) {
          f[2 * j] = b[j * 64];
          f[2 * j + 1] = b[j * 64 + 1];
        }
        double q0v = b[9 * 64], q1v = b[9 * 64 + 1];
#pragma unroll
        for (int j = 0; j < 9; ++j) s[j] += f[j] * q0v + f[9 + j] * q1v;
      }
      __syncwarp();
    }
    cp_async_wait<0>();
#pragma unroll
    for (int j = 0; j < 9; ++j) s[j] = warp_sum(s[j]);
    if (lane < 9) {
      double v = 0.0;
#pragma unroll
      for (int j = 0; j < 9; ++j)
        if (j == lane) v = s[j];
      double b;
      if (A) {
        const double* a = A + (int64_t)i * 81 + lane * 9;
        const double* xi = x + (int64_t)i * 9;
        b = 0.0;
#pragma unroll
        for (int c = 0; c < 9; ++c) b += a[c] * xi[c];
      } else {
        b = -g_cam[(int64_t)i * 9 + lane];
      }
      out[(int64_t)i * 9 + lane] = b - v;
    }
  }
}

static size_t cam_gather_smem() {
  const size_t sm = sizeof(double) * 4 * CN_STAGES * 640;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_cam_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  return sm;
}

extern "C" int bamg_build_system(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list,
                                 const int32_t* pt_ptr, double* J, int64_t k, const double* A_raw,
                                 const double* C_raw, const double* g_cam, const double* g_pt, const double* d_cam,
                                 const double* d_pt, int32_t nc, int32_t npt, double* A, double* C, double* Cinv,
                                 double* Cb, double* qo, double* rhs, int32_t* bad_min_dev, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  int big = 0x7fffffff;
  set_i32(bad_min_dev, big, st);  // device-side: no pageable host copy in the stream
  if (nc) launch(k_add_diag, grid_for((int64_t)nc * 81, 256), 256, 0, st, A_raw, d_cam, nc, 9, A);
  if (npt)
    launch(k_points_H_warp, grid_for((int64_t)ceil_div(npt, 32) * 32, 128, 16), 128, 0, st, pt_ptr, C_raw, d_pt, g_pt,
           npt, C, Cinv, Cb, bad_min_dev, J, qo);
  if (nc && rhs)  // rhs == NULL: formed later by bamg_rhs_gather or the Schur diagonal pass
    launch(k_cam_gather, grid_for((int64_t)nc * 32, 128, 8), 128, cam_gather_smem(), st, cam_ptr, cm_list, J, qo,
           g_cam, nullptr, nullptr, nc, rhs);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// schur.py:122 rhs_cam = -g - sum_o F_o^T q_o on its own (camera-major gather)
extern "C" int bamg_rhs_gather(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list, const double* J,
                               const double* qo, const double* g_cam, int32_t nc, double* rhs, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (nc)
    launch(k_cam_gather, grid_for((int64_t)nc * 32, 128, 8), 128, cam_gather_smem(), st, cam_ptr, cm_list, J, qo,
           g_cam, nullptr, nullptr, nc, rhs);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// H of every observation from a system's C^-1 (restores H after another system
// built from the same Jacobian overwrote it).
extern "C" int bamg_obs_H(bamg_ctx* ctx, const int32_t* obs_pt_pm, const double* Cinv, const double* Cb, int64_t k,
                          double* J, double* qo, void* stream) {
  (void)ctx;
  if (k) launch(k_obs_H, grid_for(k, 256, 8), 256, 0, as_stream(stream), obs_pt_pm, Cinv, Cb, k, J, qo);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// Per point: u_p = sum_o E_o^T (F_o x_cam(o)); v_p = Cinv u_p (or Cinv (base - u_p));
// q_o = E_o v_p. x: camera rows padded to 10 doubles (pad9).
__global__ void k_point_wtx(const int* __restrict__ pt_ptr, const int* __restrict__ ocam, const double* __restrict__ J,
                            const double* __restrict__ Cinv, const double* __restrict__ x, const double* __restrict__ base,
                            int npt, double* __restrict__ v_out, double* __restrict__ qo) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < npt; p += gridDim.x * blockDim.x) {
    double u[3] = {0, 0, 0};
    for (int o = pt_ptr[p]; o < pt_ptr[p + 1]; ++o) {
      const double2* rp = reinterpret_cast<const double2*>(J + (int64_t)o * REC);
      const double2* xc2 = reinterpret_cast<const double2*>(x + (int64_t)ocam[o] * 10);  // padded rows
      double xc[10];
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        double2 v = __ldg(xc2 + c);
        xc[2 * c] = v.x;
        xc[2 * c + 1] = v.y;
      }
      double t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int c = 0; c < 9; ++c) {
        double2 fc = __ldg(rp + c);  // fields 2c, 2c+1 of the flattened F (rows 0 and 1)
        int e0 = 2 * c, e1 = 2 * c + 1;
        // flattened index e -> (row e / 9, col e % 9)
        if (e0 < 9) t0 += fc.x * xc[e0]; else t1 += fc.x * xc[e0 - 9];
        if (e1 < 9) t0 += fc.y * xc[e1]; else t1 += fc.y * xc[e1 - 9];
      }
      double2 e01 = __ldg(rp + RE / 2), e23 = __ldg(rp + RE / 2 + 1), e45 = __ldg(rp + RE / 2 + 2);
      double e[6] = {e01.x, e01.y, e23.x, e23.y, e45.x, e45.y};
#pragma unroll
      for (int j = 0; j < 3; ++j) u[j] += e[j] * t0 + e[3 + j] * t1;
    }
    if (base) {
#pragma unroll
      for (int j = 0; j < 3; ++j) u[j] = base[3 * (int64_t)p + j] - u[j];
    }
    const double* ci = Cinv + (int64_t)p * 9;
    double v0 = ci[0] * u[0] + ci[1] * u[1] + ci[2] * u[2];
    double v1 = ci[3] * u[0] + ci[4] * u[1] + ci[5] * u[2];
    double v2 = ci[6] * u[0] + ci[7] * u[1] + ci[8] * u[2];
    if (v_out) {
      v_out[3 * (int64_t)p] = v0;
      v_out[3 * (int64_t)p + 1] = v1;
      v_out[3 * (int64_t)p + 2] = v2;
    }
    if (qo) {
      for (int o = pt_ptr[p]; o < pt_ptr[p + 1]; ++o) {
        const double* e = J + (int64_t)o * REC + RE;
        qo[2 * (int64_t)o] = e[0] * v0 + e[1] * v1 + e[2] * v2;
        qo[2 * (int64_t)o + 1] = e[3] * v0 + e[4] * v1 + e[5] * v2;
      }
    }
  }
}

// Implicit Schur matvec y = A x - W C^-1 W^T x (schur.py:84-86). qo: k*2 scratch.
extern "C" int bamg_implicit_matvec(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list,
                                    const int32_t* pt_ptr, const int32_t* obs_cam_pm, const double* J,
                                    const double* A, const double* Cinv, const double* x, int32_t nc, int32_t npt,
                                    double* qo, double* y, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  double* x10 = nullptr;  // camera vector padded to 80 B rows for k_point_wtx's gathers
  BAMG_CUDA_CHECK(cudaMallocAsync(&x10, sizeof(double) * 10 * (size_t)(nc > 0 ? nc : 1), st));
  if (nc) pad9(x, nc, x10, st);
  if (npt) launch(k_point_wtx, grid_for(npt, 128, 16), 128, 0, st, pt_ptr, obs_cam_pm, J, Cinv, (const double*)x10,
                  nullptr, npt, nullptr, qo);
  BAMG_CUDA_CHECK(cudaFreeAsync(x10, st));
  if (nc)
    launch(k_cam_gather, grid_for((int64_t)nc * 32, 128, 8), 128, cam_gather_smem(), st, cam_ptr, cm_list, J, qo,
           nullptr, A, x, nc, y);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// Back-substitution dp = C^-1 (b_p - W^T dc) (schur.py:171-173); b_p = -g_pt.
__global__ void k_neg(const double* __restrict__ a, double* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = -a[i];
}

extern "C" int bamg_back_substitute(bamg_ctx* ctx, const int32_t* pt_ptr, const int32_t* obs_cam_pm, const double* J,
                                    const double* Cinv, const double* grad_pt, const double* dc, int32_t nc,
                                    int32_t npt, double* dp, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  double* x10 = nullptr;  // dc padded to 80 B camera rows for k_point_wtx's gathers
  BAMG_CUDA_CHECK(cudaMallocAsync(&x10, sizeof(double) * 10 * (size_t)(nc > 0 ? nc : 1), st));
  if (nc > 0) pad9(dc, nc, x10, st);
  if (npt) launch(k_point_wtx, grid_for(npt, 128, 16), 128, 0, st, pt_ptr, obs_cam_pm, J, Cinv, (const double*)x10,
                  grad_pt, npt, dp, nullptr);
  BAMG_CUDA_CHECK(cudaFreeAsync(x10, st));
  BAMG_LAUNCH_CHECK();
  return 0;
}

extern "C" int bamg_negate(bamg_ctx* ctx, const double* a, double* b, int64_t n, void* stream) {
  (void)ctx;
  if (n) launch(k_neg, grid_for(n, 256), 256, 0, as_stream(stream), a, b, n);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// W blocks in the reference's BSR order (for API views): W_b = F_o^T E_o, o = cm_list[b].
__global__ void k_materialize_W(const int* __restrict__ cm_list, const double* __restrict__ J, int64_t k,
                                double* __restrict__ W) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < k * 27; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = t / 27;
    int q = (int)(t - b * 27);
    int r = q / 3, c = q - r * 3;
    const double* rec = J + (int64_t)cm_list[b] * REC;
    W[t] = rec[RF + r] * rec[RE + c] + rec[RF + 9 + r] * rec[RE + 3 + c];
  }
}

extern "C" int bamg_materialize_W(bamg_ctx* ctx, const int32_t* cm_list, const double* J, int64_t k, double* W,
                                  void* stream) {
  (void)ctx;
  if (k) launch(k_materialize_W, grid_for(k * 27, 256), 256, 0, as_stream(stream), cm_list, J, k, W);
  BAMG_LAUNCH_CHECK();
  return 0;
}
