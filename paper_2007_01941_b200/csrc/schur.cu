// Explicit reduced camera matrix S = A - W C^-1 W^T (schur.py:128-144).
//
// W_o = F_o^T E_o, so every point contribution factors through a 2x2 core:
//   W_a C^-1 W_b^T = F_a^T (H_a E_b^T) F_b,   H_a = E_a C_p^-1  (stored per obs).
// Symbolic phase (once per problem; the observation structure is parameter
// independent, solver.py:221-230): every point p with cameras c_1<...<c_m emits the
// upper pairs (a<b) of its segment; a stable radix sort by S block index groups
// them per block while keeping point order inside each block. Numeric phase: one
// warp per camera for the diagonal blocks (A_i minus a symmetric 45-entry
// accumulation), and 3 lanes per upper off-diagonal block (each lane owns three
// columns of the 9x9 block in registers) -- no atomics, fixed summation order, so
// S is bit-reproducible run to run. S_ji is written as S_ij^T (exactly symmetric,
// matching the reference's 0.5 (S + S^T) to roundoff).
#include <algorithm>

#include "common.cuh"
#include "ctx.h"

int radix_sort_pairs(const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout,
                     int64_t n, int key_bits, cudaStream_t st);
int scan_exclusive_int(const int* in, int* out, int64_t n, int* total, cudaStream_t st);
int segment_ptr(const int* ids, int64_t n, int nseg, int* ptr, cudaStream_t st);

__global__ void k_pair_counts(const int* __restrict__ pt_ptr, int npt, int* __restrict__ cnt) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < npt; p += gridDim.x * blockDim.x) {
    int m = pt_ptr[p + 1] - pt_ptr[p];
    cnt[p] = m * (m - 1) / 2;
  }
}

__global__ void k_pair_emit(const int* __restrict__ pt_ptr, const int* __restrict__ ocam,
                            const int* __restrict__ S_ptr, const int* __restrict__ S_col,
                            const int* __restrict__ off, int npt, uint32_t* __restrict__ key,
                            int* __restrict__ oa, int* __restrict__ ob) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < npt; p += gridDim.x * blockDim.x) {
    int s = pt_ptr[p], e = pt_ptr[p + 1];
    int pos = off[p];
    for (int a = s; a < e; ++a) {
      int ca = ocam[a];
      const int* cols = S_col + S_ptr[ca];
      int n = S_ptr[ca + 1] - S_ptr[ca];
      for (int b = a + 1; b < e; ++b) {
        int q = lower_bound_i32(cols, n, ocam[b]);
        key[pos] = (uint32_t)(S_ptr[ca] + q);
        oa[pos] = a;
        ob[pos] = b;
        ++pos;
      }
    }
  }
}

// Packed form of k_pair_emit: the pair is carried through the sort as its value,
// a << 7 | (b - a) (a < 2^25 observations, b - a < 128 inside a point's segment), so
// the sort needs no index payload and no gather afterwards.
__global__ void k_pair_emit_packed(const int* __restrict__ pt_ptr, const int* __restrict__ ocam,
                                   const int* __restrict__ S_ptr, const int* __restrict__ S_col,
                                   const int* __restrict__ off, int npt, uint32_t* __restrict__ key,
                                   uint32_t* __restrict__ val) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < npt; p += gridDim.x * blockDim.x) {
    int s = pt_ptr[p], e = pt_ptr[p + 1];
    int pos = off[p];
    for (int a = s; a < e; ++a) {
      int ca = ocam[a];
      const int* cols = S_col + S_ptr[ca];
      int n = S_ptr[ca + 1] - S_ptr[ca];
      for (int b = a + 1; b < e; ++b) {
        int q = lower_bound_i32(cols, n, ocam[b]);
        key[pos] = (uint32_t)(S_ptr[ca] + q);
        val[pos] = ((uint32_t)a << 7) | (uint32_t)(b - a);
        ++pos;
      }
    }
  }
}

// Same output as k_pair_emit_packed with a thread per observation a instead of per
// point (29 M threads with at most m - 1 pairs each, against 4.5 M with up to
// m (m - 1) / 2): a's pairs start at pair_off[p] + t (m - 1) - t (t - 1) / 2 for a at
// index t of its point's segment; the partner cameras ascend, so each slot search
// starts past the previous one.
__global__ void k_pair_emit_obs(const int* __restrict__ pt_ptr, const int* __restrict__ obs_pt_pm,
                                const int* __restrict__ ocam, const int* __restrict__ S_ptr,
                                const int* __restrict__ S_col, const int* __restrict__ off, int64_t k,
                                uint32_t* __restrict__ key, uint32_t* __restrict__ val) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < k; a += (int64_t)gridDim.x * blockDim.x) {
    int p = obs_pt_pm[a];
    int s = pt_ptr[p], e = pt_ptr[p + 1];
    int t = (int)a - s, m = e - s;
    int64_t pos = (int64_t)off[p] + (int64_t)t * (m - 1) - (int64_t)t * (t - 1) / 2;
    int ca = ocam[a];
    int r0 = S_ptr[ca], n = S_ptr[ca + 1] - r0;
    const int* cols = S_col + r0;
    int q = -1;
    for (int b = (int)a + 1; b < e; ++b, ++pos) {
      q += 1 + lower_bound_i32(cols + q + 1, n - q - 1, ocam[b]);
      key[pos] = (uint32_t)(r0 + q);
      val[pos] = ((uint32_t)a << 7) | (uint32_t)(b - (int)a);
    }
  }
}

__global__ void k_unpack_pairs(const uint32_t* __restrict__ v, int64_t n, int* __restrict__ pa, int* __restrict__ pb) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = v[i];
    int a = (int)(x >> 7);
    pa[i] = a;
    pb[i] = a + (int)(x & 127u);
  }
}

__global__ void k_max_segment(const int* __restrict__ pt_ptr, int npt, int* __restrict__ mx) {
  int m = 0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < npt; p += gridDim.x * blockDim.x)
    m = max(m, pt_ptr[p + 1] - pt_ptr[p]);
  m = warp_max_int(m);
  if ((threadIdx.x & 31) == 0) atomicMax(mx, m);
}

__global__ void k_iota_u32(uint32_t* a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (uint32_t)i;
}

__global__ void k_gather_pairs(const uint32_t* __restrict__ perm, const int* __restrict__ oa,
                               const int* __restrict__ ob, int64_t n, int* __restrict__ pa, int* __restrict__ pb) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t s = perm[i];
    pa[i] = oa[s];
    pb[i] = ob[s];
  }
}

// Per row: diagonal slot, count of upper blocks.
__global__ void k_row_upper(const int* __restrict__ S_ptr, const int* __restrict__ S_col, int nc,
                            int* __restrict__ dpos, int* __restrict__ nup) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
    int b = S_ptr[i], n = S_ptr[i + 1] - b;
    int q = lower_bound_i32(S_col + b, n, i);
    dpos[i] = b + q;
    nup[i] = n - q - 1;
  }
}

__global__ void k_upper_list(const int* __restrict__ S_ptr, const int* __restrict__ S_col, int nc,
                             const int* __restrict__ dpos, const int* __restrict__ up_off, int* __restrict__ up_blk,
                             int* __restrict__ up_row, int* __restrict__ up_tpos) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
    int out = up_off[i];
    for (int q = dpos[i] + 1; q < S_ptr[i + 1]; ++q) {
      int j = S_col[q];
      const int* cj = S_col + S_ptr[j];
      int t = lower_bound_i32(cj, S_ptr[j + 1] - S_ptr[j], i);
      up_blk[out] = q;
      up_row[out] = i;
      up_tpos[out] = S_ptr[j] + t;
      ++out;
    }
  }
}

// Query sizes for the symbolic phase: returns n_pairs and n_upper through out[2]
// (host pointer) after a stream sync.
extern "C" int bamg_schur_symbolic_sizes(bamg_ctx* ctx, const int32_t* pt_ptr, const int32_t* S_ptr,
                                         const int32_t* S_col, int32_t nc, int32_t npt, int32_t* pair_off,
                                         int32_t* dpos, int32_t* up_off, int64_t* out_host, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  int* tot = nullptr;
  BAMG_CUDA_CHECK(cudaMallocAsync(&tot, 2 * sizeof(int), st));
  launch(k_pair_counts, grid_for(npt, 256), 256, 0, st, pt_ptr, npt, pair_off);
  int rc = scan_exclusive_int(pair_off, pair_off, npt, tot, st);
  if (rc) return rc;
  launch(k_row_upper, grid_for(nc, 128), 128, 0, st, S_ptr, S_col, nc, dpos, up_off);
  rc = scan_exclusive_int(up_off, up_off, nc, tot + 1, st);
  if (rc) return rc;
  int h[2];
  BAMG_CUDA_CHECK(cudaMemcpyAsync(h, tot, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  BAMG_CUDA_CHECK(cudaStreamSynchronize(st));
  cudaFreeAsync(tot, st);
  out_host[0] = h[0];
  out_host[1] = h[1];
  return 0;
}

extern "C" int bamg_schur_symbolic(bamg_ctx* ctx, const int32_t* pt_ptr, const int32_t* obs_cam_pm,
                                   const int32_t* obs_pt_pm,
                                   const int32_t* S_ptr, const int32_t* S_col, int32_t nc, int32_t npt,
                                   int64_t nnz, const int32_t* pair_off, int64_t n_pairs, const int32_t* dpos,
                                   const int32_t* up_off, int32_t* pair_a, int32_t* pair_b, int32_t* blk_pair_ptr,
                                   int32_t* up_blk, int32_t* up_row, int32_t* up_tpos, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  launch(k_upper_list, grid_for(nc, 128), 128, 0, st, S_ptr, S_col, nc, dpos, up_off, up_blk, up_row, up_tpos);
  BAMG_LAUNCH_CHECK();
  if (pair_a == nullptr) return 0;  // upper-block list only (row-owned numeric path)
  if (n_pairs == 0) {
    BAMG_CUDA_CHECK(cudaMemsetAsync(blk_pair_ptr, 0, sizeof(int) * (nnz + 1), st));
    return 0;
  }
  // packed path: observation indices below 2^25 and point segments below 128
  {
    int64_t n_obs = 0;
    int h[2] = {0, 0};
    int* dev = nullptr;
    BAMG_CUDA_CHECK(cudaMallocAsync(&dev, 2 * sizeof(int), st));
    BAMG_CUDA_CHECK(cudaMemsetAsync(dev, 0, 2 * sizeof(int), st));
    launch(k_max_segment, grid_for(npt, 256), 256, 0, st, pt_ptr, npt, dev);
    BAMG_CUDA_CHECK(cudaMemcpyAsync(dev + 1, pt_ptr + npt, sizeof(int), cudaMemcpyDeviceToDevice, st));
    BAMG_CUDA_CHECK(cudaMemcpyAsync(h, dev, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    BAMG_CUDA_CHECK(cudaStreamSynchronize(st));
    cudaFreeAsync(dev, st);
    n_obs = h[1];
    if (n_obs < (1ll << 25) && h[0] <= 128) {
      uint32_t *key = nullptr, *val = nullptr, *skey = nullptr, *sval = nullptr;
      BAMG_CUDA_CHECK(cudaMallocAsync(&key, 4 * n_pairs, st));
      BAMG_CUDA_CHECK(cudaMallocAsync(&val, 4 * n_pairs, st));
      BAMG_CUDA_CHECK(cudaMallocAsync(&skey, 4 * n_pairs, st));
      BAMG_CUDA_CHECK(cudaMallocAsync(&sval, 4 * n_pairs, st));
      launch(k_pair_emit_obs, grid_for(n_obs, 256), 256, 0, st, pt_ptr, obs_pt_pm, obs_cam_pm, S_ptr, S_col, pair_off,
             n_obs, key, val);
      int bits = 1;
      while ((1ll << bits) < nnz) ++bits;
      int rc = radix_sort_pairs(key, val, skey, sval, n_pairs, bits, st);
      if (rc) return rc;
      launch(k_unpack_pairs, grid_for(n_pairs, 256), 256, 0, st, (const uint32_t*)sval, n_pairs, pair_a, pair_b);
      rc = segment_ptr((const int*)skey, n_pairs, (int)nnz, blk_pair_ptr, st);
      if (rc) return rc;
      BAMG_LAUNCH_CHECK();
      cudaFreeAsync(key, st);
      cudaFreeAsync(val, st);
      cudaFreeAsync(skey, st);
      cudaFreeAsync(sval, st);
      return 0;
    }
  }
  uint32_t *key = nullptr, *iota = nullptr, *skey = nullptr, *perm = nullptr;
  int *oa = nullptr, *ob = nullptr;
  BAMG_CUDA_CHECK(cudaMallocAsync(&key, 4 * n_pairs, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&iota, 4 * n_pairs, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&skey, 4 * n_pairs, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&perm, 4 * n_pairs, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&oa, 4 * n_pairs, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&ob, 4 * n_pairs, st));
  launch(k_pair_emit, grid_for(npt, 128), 128, 0, st, pt_ptr, obs_cam_pm, S_ptr, S_col, pair_off, npt, key, oa, ob);
  launch(k_iota_u32, grid_for(n_pairs, 256), 256, 0, st, iota, n_pairs);
  BAMG_LAUNCH_CHECK();
  int bits = 1;
  while ((1ll << bits) < nnz) ++bits;
  int rc = radix_sort_pairs(key, iota, skey, perm, n_pairs, bits, st);
  if (rc) return rc;
  launch(k_gather_pairs, grid_for(n_pairs, 256), 256, 0, st, perm, oa, ob, n_pairs, pair_a, pair_b);
  rc = segment_ptr((const int*)skey, n_pairs, (int)nnz, blk_pair_ptr, st);
  if (rc) return rc;
  BAMG_LAUNCH_CHECK();
  cudaFreeAsync(key, st);
  cudaFreeAsync(iota, st);
  cudaFreeAsync(skey, st);
  cudaFreeAsync(perm, st);
  cudaFreeAsync(oa, st);
  cudaFreeAsync(ob, st);
  return 0;
}

// Shared-point counts per covisibility slot from the pair lists (a block's list has
// one pair per shared point): upper slot and its mirror = list length, diagonal =
// the camera's observation count -- what k_shared_counts derives from the
// observations in a separate pass.
__global__ void k_shared_from_pairs(const int* __restrict__ up_blk, const int* __restrict__ up_tpos, int n_up,
                                    const int* __restrict__ blk_ptr, const int* __restrict__ dpos,
                                    const int* __restrict__ cam_ptr, int nc, int* __restrict__ shared) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n_up + nc; u += gridDim.x * blockDim.x) {
    if (u < n_up) {
      int q = up_blk[u];
      int len = blk_ptr[q + 1] - blk_ptr[q];
      shared[q] = len;
      shared[up_tpos[u]] = len;
    } else {
      int i = u - n_up;
      shared[dpos[i]] = cam_ptr[i + 1] - cam_ptr[i];
    }
  }
}

extern "C" int bamg_shared_from_pairs(bamg_ctx* ctx, const int32_t* up_blk, const int32_t* up_tpos, int32_t n_up,
                                      const int32_t* blk_pair_ptr, const int32_t* dpos, const int32_t* cam_ptr,
                                      int32_t nc, int32_t* shared_cnt, void* stream) {
  (void)ctx;
  if (n_up + nc <= 0) return 0;
  launch(k_shared_from_pairs, grid_for((int64_t)n_up + nc, 256), 256, 0, as_stream(stream), up_blk, up_tpos, n_up,
         blk_pair_ptr, dpos, cam_ptr, nc, shared_cnt);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// Work order of the pair-list numeric kernel: upper blocks by descending pair count,
// so the ten blocks sharing a warp have similar trip counts (stable => deterministic).
__global__ void k_up_keys(const int* __restrict__ up_blk, const int* __restrict__ blk_pair_ptr, int n,
                          uint32_t* __restrict__ key, uint32_t* __restrict__ iota) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
    int b = up_blk[u];
    int c = blk_pair_ptr[b + 1] - blk_pair_ptr[b];
    key[u] = 0xFFFFFFu - (uint32_t)min(c, 0xFFFFFF);
    iota[u] = (uint32_t)u;
  }
}

__global__ void k_band_keys(const uint32_t* __restrict__ perm, const int* __restrict__ up_row, int n, int band,
                            uint32_t* __restrict__ key) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x)
    key[u] = (uint32_t)(up_row[perm[u]] / band);
}

__global__ void k_pband_keys(const uint32_t* __restrict__ perm, const int* __restrict__ up_blk,
                             const int* __restrict__ blk_pair_ptr, const int* __restrict__ pair_a, int n, int pband,
                             uint32_t* __restrict__ key) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
    int b = up_blk[perm[u]];
    int q0 = blk_pair_ptr[b], q1 = blk_pair_ptr[b + 1];
    // middle pair's a-side record: the centre of the block's stretch of points
    key[u] = q1 > q0 ? (uint32_t)(pair_a[(q0 + q1) >> 1] / pband) : 0u;
  }
}

__global__ void k_permute3(const uint32_t* __restrict__ perm, int n, int* __restrict__ a, int* __restrict__ b,
                           int* __restrict__ c, int* __restrict__ tmp) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
    tmp[u] = a[perm[u]];
    tmp[n + u] = b[perm[u]];
    tmp[2 * n + u] = c[perm[u]];
  }
}

__global__ void k_copy_i32(const int* __restrict__ src, int* __restrict__ dst, int n) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) dst[u] = src[u];
}

extern "C" int bamg_schur_order_upper(bamg_ctx* ctx, int32_t* up_blk, int32_t* up_row, int32_t* up_tpos,
                                      int32_t n_up, const int32_t* blk_pair_ptr, const int32_t* pair_a,
                                      void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (n_up <= 1) return 0;
  uint32_t *ck = nullptr, *io = nullptr, *sk = nullptr, *pv = nullptr;
  int* tmp = nullptr;
  BAMG_CUDA_CHECK(cudaMallocAsync(&ck, 4 * (size_t)n_up, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&io, 4 * (size_t)n_up, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&sk, 4 * (size_t)n_up, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&pv, 4 * (size_t)n_up, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&tmp, 4 * (size_t)n_up * 3, st));
  // descending pair count (measured at c4: 17 ms vs 31 ms in row order and 23 ms
  // in (row, count) order -- balance beats a-side L2 locality here)
  launch(k_up_keys, grid_for(n_up, 256), 256, 0, st, up_blk, blk_pair_ptr, n_up, ck, io);
  int rc = radix_sort_pairs(ck, io, sk, pv, n_up, 24, st);
  if (rc) return rc;
  // optional row bands (BAMG_SCHUR_BAND rows): blocks of nearby camera rows run
  // together so their observation records stay in L2; count order inside a band
  int band = 0, pband = 0;
  if (const char* e = getenv("BAMG_SCHUR_BAND")) band = atoi(e);
  if (const char* e = getenv("BAMG_SCHUR_PBAND")) pband = atoi(e);
  if (pband > 0 && pair_a) {
    // bands of observation records (point-major): blocks whose pair lists start in
    // the same stretch of points run together
    launch(k_pband_keys, grid_for(n_up, 256), 256, 0, st, pv, up_blk, blk_pair_ptr, pair_a, n_up, pband, ck);
    rc = radix_sort_pairs(ck, pv, sk, io, n_up, 31, st);
    if (rc) return rc;
    std::swap(pv, io);
  } else if (band > 0) {
    launch(k_band_keys, grid_for(n_up, 256), 256, 0, st, pv, up_row, n_up, band, ck);
    rc = radix_sort_pairs(ck, pv, sk, io, n_up, 31, st);
    if (rc) return rc;
    std::swap(pv, io);
  }
  launch(k_permute3, grid_for(n_up, 256), 256, 0, st, pv, n_up, up_blk, up_row, up_tpos, tmp);
  launch(k_copy_i32, grid_for(n_up, 256), 256, 0, st, tmp, up_blk, n_up);
  launch(k_copy_i32, grid_for(n_up, 256), 256, 0, st, tmp + n_up, up_row, n_up);
  launch(k_copy_i32, grid_for(n_up, 256), 256, 0, st, tmp + 2 * n_up, up_tpos, n_up);
  BAMG_LAUNCH_CHECK();
  cudaFreeAsync(ck, st);
  cudaFreeAsync(io, st);
  cudaFreeAsync(sk, st);
  cudaFreeAsync(pv, st);
  cudaFreeAsync(tmp, st);
  return 0;
}

// Diagonal blocks: warp per camera, S_ii = A_i - sum_o F_o^T (H_o E_o^T) F_o.
// Records (F, E, H = pieces 0..14) are gathered 32 at a time into shared memory.
// With RHS the same pass also forms the reduced right-hand side of the camera
// (schur.py:122): rhs_i = -g_i - sum_o F_o^T q_o, q_o = E_o C^-1 b_p staged as piece
// 15 -- the camera-major gather build_system would otherwise run on its own.
#define SD_ST 31
#ifndef SD_STAGES
#define SD_STAGES 2
#endif
template <bool RHS>
__global__ void __launch_bounds__(128)
k_schur_diag(const int* __restrict__ cam_ptr, const int* __restrict__ cm_list, const double* __restrict__ J,
             const double* __restrict__ A, const int* __restrict__ dpos, int nc, const double* __restrict__ qo,
             const double* __restrict__ g_cam, double* __restrict__ rhs, double* __restrict__ S) {
  // SD_STAGES-deep cp.async pipeline of 32-record chunks (pieces 0..14: F, E, H; 15: q)
  extern __shared__ __align__(16) double sd_smem[];
  constexpr int CH = (RHS ? 16 : 15) * 64;
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* wbuf = sd_smem + (size_t)w * SD_STAGES * CH;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < nc; i += nwarps) {
    double acc[45];
#pragma unroll
    for (int q = 0; q < 45; ++q) acc[q] = 0.0;
    double racc[RHS ? 9 : 1];
#pragma unroll
    for (int q = 0; q < (RHS ? 9 : 1); ++q) racc[q] = 0.0;
    const int q0 = cam_ptr[i], q1 = cam_ptr[i + 1];
#pragma unroll
    for (int s = 0; s < SD_STAGES - 1; ++s) {
      int cb = q0 + 32 * s;
      if (cb < q1) {
        bool v = cb + lane < q1;
        rec_issue<15, 0, RHS ? 1 : 0>(J, v ? cm_list[cb + lane] : 0, v, 0, 0, qo, wbuf + s * CH, lane);
      } else {
        cp_async_commit();
      }
    }
    int c = 0;
    // observation ids of the next chunk to issue, loaded one iteration ahead so the
    // copies never wait on the index load
    int nidx = (q0 + 32 * (SD_STAGES - 1) + lane < q1) ? cm_list[q0 + 32 * (SD_STAGES - 1) + lane] : 0;
    for (int base = q0; base < q1; base += 32, ++c) {
      int nb = base + 32 * (SD_STAGES - 1);
      if (nb < q1) {
        bool vn = nb + lane < q1;
        rec_issue<15, 0, RHS ? 1 : 0>(J, nidx, vn, 0, 0, qo,
                            wbuf + ((c + SD_STAGES - 1) % SD_STAGES) * CH, lane);
      } else {
        cp_async_commit();
      }
      {
        int pb = nb + 32;
        nidx = (pb + lane < q1) ? cm_list[pb + lane] : 0;
      }
      cp_async_wait<SD_STAGES - 1>();
      __syncwarp();
      bool valid = base + lane < q1;
      const double* bsrc = wbuf + (c % SD_STAGES) * CH + 2 * lane;
      double f[30];
      if (valid) {
#pragma unroll
        for (int p = 0; p < 15; ++p) {
          f[2 * p] = bsrc[p * 64];
          f[2 * p + 1] = bsrc[p * 64 + 1];
        }
        const double* e = f + RE;
        const double* h = f + RH;
        double g00 = h[0] * e[0] + h[1] * e[1] + h[2] * e[2];
        double g01 = h[0] * e[3] + h[1] * e[4] + h[2] * e[5];
        double g10 = h[3] * e[0] + h[4] * e[1] + h[5] * e[2];
        double g11 = h[3] * e[3] + h[4] * e[4] + h[5] * e[5];
        int t = 0;
#pragma unroll
        for (int j = 0; j < 9; ++j) {
          double a0 = f[j] * g00 + f[9 + j] * g10;
          double a1 = f[j] * g01 + f[9 + j] * g11;
#pragma unroll
          for (int l = j; l < 9; ++l) acc[t++] += a0 * f[l] + a1 * f[9 + l];
        }
        if constexpr (RHS) {
          double q0 = bsrc[15 * 64], q1 = bsrc[15 * 64 + 1];
#pragma unroll
          for (int j = 0; j < 9; ++j) racc[j] += f[j] * q0 + f[9 + j] * q1;
        }
      }
      __syncwarp();
    }
    cp_async_wait<0>();
#pragma unroll
    for (int q = 0; q < 45; ++q) acc[q] = warp_sum(acc[q]);
    if constexpr (RHS) {
#pragma unroll
      for (int q = 0; q < 9; ++q) racc[q] = warp_sum(racc[q]);
      if (lane == 0)
#pragma unroll
        for (int j = 0; j < 9; ++j) rhs[(int64_t)i * 9 + j] = -g_cam[(int64_t)i * 9 + j] - racc[j];
    }
    if (lane == 0) {
      double* out = S + (int64_t)dpos[i] * 81;
      const double* a = A + (int64_t)i * 81;
      int t = 0;
#pragma unroll
      for (int j = 0; j < 9; ++j)
#pragma unroll
        for (int l = j; l < 9; ++l) {
          double v = 0.5 * (a[j * 9 + l] + a[l * 9 + j]) - acc[t++];
          out[j * 9 + l] = v;
          out[l * 9 + j] = v;
        }
    }
  }
}

// Upper off-diagonal blocks from the per-block pair lists: 10 blocks per warp,
// 3 lanes per block (each lane owns three columns of the 9x9 block in registers).
// The a-side (F, H) and b-side (F, E) of a pair sit in one 256 B record each.
// (A variant that staged the ten pairs' records through shared memory with
// cooperative loads measured 2x slower at c4: the extra synchronisation
// serialised the per-pair index -> record latency chain.)
#define OFF_GROUPS 10
#ifndef SCHUR_OFF_MINB
#define SCHUR_OFF_MINB 1  // forcing 5 CTAs/SM (96 regs + spills) measured 8% slower at c4
#endif

__global__ void __launch_bounds__(128, SCHUR_OFF_MINB)
k_schur_offdiag(const int* __restrict__ up_blk, const int* __restrict__ up_tpos, int n_up,
                const int* __restrict__ blk_pair_ptr, const int* __restrict__ pair_a, const int* __restrict__ pair_b,
                const double* __restrict__ J, double* __restrict__ S) {
  int lane = threadIdx.x & 31;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  int grp = lane / 3, c3 = lane - 3 * grp;
  for (int base = warp * OFF_GROUPS; base < n_up; base += nwarps * OFF_GROUPS) {
    int u = base + grp;
    bool active = (grp < OFF_GROUPS) && (u < n_up);
    if (!active) continue;
    int blk = up_blk[u];
    double acc[27];
#pragma unroll
    for (int q = 0; q < 27; ++q) acc[q] = 0.0;
    int c0 = 3 * c3;
    const int fb_lo = (RF + c0) >> 1, fb_hi = (RF + 9 + c0) >> 1;
    const bool lo_odd = (RF + c0) & 1;  // RF even: the high triple has the other parity
    int q = blk_pair_ptr[blk], qe = blk_pair_ptr[blk + 1];
    int na = q < qe ? pair_a[q] : 0, nb = q < qe ? pair_b[q] : 0;
    for (; q < qe; ++q) {
      int64_t oa = na, ob = nb;
      if (q + 1 < qe) {  // next pair's indices in flight during this pair's math
        na = pair_a[q + 1];
        nb = pair_b[q + 1];
      }
      // 16 B loads: the kernel is bound by L1 wavefronts (one per distinct line per
      // load instruction), so fewer, wider loads per pair is what matters.
      const double2* ra = reinterpret_cast<const double2*>(J + oa * REC);
      const double2* rb = reinterpret_cast<const double2*>(J + ob * REC);
      double fa[18], ha[6], eb[6];
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        double2 v = __ldg(ra + RF / 2 + k);
        fa[2 * k] = v.x;
        fa[2 * k + 1] = v.y;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double2 v = __ldg(ra + RH / 2 + k), w = __ldg(rb + RE / 2 + k);
        ha[2 * k] = v.x;
        ha[2 * k + 1] = v.y;
        eb[2 * k] = w.x;
        eb[2 * k + 1] = w.y;
      }
      // this lane's columns c0..c0+2 of both F_b rows, from two aligned pairs each
      double2 p0 = __ldg(rb + fb_lo), p1 = __ldg(rb + fb_lo + 1);
      double2 s0 = __ldg(rb + fb_hi), s1 = __ldg(rb + fb_hi + 1);
      double b0[3], b1[3];
      b0[0] = lo_odd ? p0.y : p0.x;
      b0[1] = lo_odd ? p1.x : p0.y;
      b0[2] = lo_odd ? p1.y : p1.x;
      b1[0] = lo_odd ? s0.x : s0.y;
      b1[1] = lo_odd ? s0.y : s1.x;
      b1[2] = lo_odd ? s1.x : s1.y;
      double g00 = ha[0] * eb[0] + ha[1] * eb[1] + ha[2] * eb[2];
      double g01 = ha[0] * eb[3] + ha[1] * eb[4] + ha[2] * eb[5];
      double g10 = ha[3] * eb[0] + ha[4] * eb[1] + ha[5] * eb[2];
      double g11 = ha[3] * eb[3] + ha[4] * eb[4] + ha[5] * eb[5];
#pragma unroll
      for (int r = 0; r < 9; ++r) {
        double fr0 = fa[r], fr1 = fa[9 + r];
        double a0 = fr0 * g00 + fr1 * g10;
        double a1 = fr0 * g01 + fr1 * g11;
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[r * 3 + c] += a0 * b0[c] + a1 * b1[c];
      }
    }
    double* sij = S + (int64_t)blk * 81;
    double* sji = S + (int64_t)up_tpos[u] * 81;
#pragma unroll
    for (int r = 0; r < 9; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double v = -acc[r * 3 + c];
        sij[r * 9 + c0 + c] = v;
        sji[(c0 + c) * 9 + r] = v;
      }
  }
}

// ---------------------------------------------------------------------------
// Same assignment (10 blocks per warp, 3 lanes per block, same per-block pair order,
// so bit-identical S), but the pair records are streamed into shared memory with
// cp.async through an OFFP_STAGES-deep per-warp pipeline. The register version keeps
// only one pair step in flight per warp and its scattered 8-16 B loads spend L1
// wavefronts per distinct line; here the copies are coalesced 16 B chunks and the
// bytes in flight no longer depend on the register budget. Warps are independent
// (no CTA barrier); the index of step t+1 is fetched while step t's copies issue.
#define OFFP_STAGES 3
#define OFFP_RS 34  // doubles per staged record: 272 B rows put the 10 groups on distinct 16 B banks
#define OFFP_STAGE_DOUBLES (2 * OFF_GROUPS * OFFP_RS)
#define OFFP_WARP_DOUBLES (OFFP_STAGES * OFFP_STAGE_DOUBLES)

// Copy one step's records: lanes 0..19 hold rec = observation index of (group r>>1,
// side r&1) or -1. a side: F (chunks 0-8) + H (12-14); b side: F + E (chunks 0-11).
__device__ __forceinline__ void offp_issue(double* stage, const double* __restrict__ J, int myrec, int lane) {
#pragma unroll
  for (int it = 0; it < 8; ++it) {  // 20 records x 12 chunks = 240 = 7.5 per lane
    int c = lane + 32 * it;
    int r = c / 12;
    int k = c - 12 * r;
    int rec = __shfl_sync(0xffffffffu, myrec, r < 20 ? r : 19);
    if (c < 240 && rec >= 0) {
      int side = r & 1, g = r >> 1;
      int ch = side ? k : (k < 9 ? k : k + 3);
      cp_async16(stage + (side * OFF_GROUPS + g) * OFFP_RS + 2 * ch, J + (int64_t)rec * REC + 2 * ch);
    }
  }
  cp_async_commit();
}

__global__ void __launch_bounds__(128)
k_schur_offdiag_pipe(const int* __restrict__ up_blk, const int* __restrict__ up_tpos, int n_up,
                     const int* __restrict__ blk_pair_ptr, const int* __restrict__ pair_a,
                     const int* __restrict__ pair_b, const double* __restrict__ J, double* __restrict__ S) {
  extern __shared__ __align__(16) double smem_offp[];
  int lane = threadIdx.x & 31;
  double* wsm = smem_offp + (threadIdx.x >> 5) * OFFP_WARP_DOUBLES;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  int grp = lane / 3, c3 = lane - 3 * grp;
  int c0 = 3 * c3;
  const int fb_lo = (RF + c0) >> 1, fb_hi = (RF + 9 + c0) >> 1;
  const bool lo_odd = (RF + c0) & 1;
  const int ig = lane >> 1;
  const int* ilist = (lane & 1) ? pair_b : pair_a;
  for (int base = warp * OFF_GROUPS; base < n_up; base += nwarps * OFF_GROUPS) {
    int u = base + grp;
    bool active = (grp < OFF_GROUPS) && (u < n_up);
    int blk = active ? up_blk[u] : 0;
    int q0 = active ? blk_pair_ptr[blk] : 0;
    int len = active ? blk_pair_ptr[blk + 1] - q0 : 0;
    int maxlen = len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
    // index lanes 0..19 see group ig's pair range
    int src = 3 * ig < 31 ? 3 * ig : 31;
    int iq0 = __shfl_sync(0xffffffffu, q0, src);
    int ilen = __shfl_sync(0xffffffffu, len, src);
    if (lane >= 2 * OFF_GROUPS) ilen = 0;
    int nrec = (ilen > 0) ? ilist[iq0] : -1;  // record index of step 0
#pragma unroll
    for (int t = 0; t < OFFP_STAGES - 1; ++t) {
      int rec = nrec;
      nrec = (t + 1 < ilen) ? ilist[iq0 + t + 1] : -1;
      if (t < maxlen) offp_issue(wsm + t * OFFP_STAGE_DOUBLES, J, rec, lane);
      else cp_async_commit();
    }
    double acc[27];
#pragma unroll
    for (int q = 0; q < 27; ++q) acc[q] = 0.0;
    for (int s = 0; s < maxlen; ++s) {
      int t = s + OFFP_STAGES - 1;
      int rec = nrec;
      nrec = (t + 1 < ilen) ? ilist[iq0 + t + 1] : -1;
      if (t < maxlen) offp_issue(wsm + (t % OFFP_STAGES) * OFFP_STAGE_DOUBLES, J, rec, lane);
      else cp_async_commit();
      cp_async_wait<OFFP_STAGES - 1>();
      __syncwarp();
      if (s < len) {
        const double* stg = wsm + (s % OFFP_STAGES) * OFFP_STAGE_DOUBLES;
        const double2* ra = reinterpret_cast<const double2*>(stg + grp * OFFP_RS);
        const double2* rb = reinterpret_cast<const double2*>(stg + (OFF_GROUPS + grp) * OFFP_RS);
        double fa[18], ha[6], eb[6];
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          double2 v = ra[RF / 2 + k];
          fa[2 * k] = v.x;
          fa[2 * k + 1] = v.y;
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          double2 v = ra[RH / 2 + k], w = rb[RE / 2 + k];
          ha[2 * k] = v.x;
          ha[2 * k + 1] = v.y;
          eb[2 * k] = w.x;
          eb[2 * k + 1] = w.y;
        }
        double2 p0 = rb[fb_lo], p1 = rb[fb_lo + 1];
        double2 s0 = rb[fb_hi], s1 = rb[fb_hi + 1];
        double b0[3], b1[3];
        b0[0] = lo_odd ? p0.y : p0.x;
        b0[1] = lo_odd ? p1.x : p0.y;
        b0[2] = lo_odd ? p1.y : p1.x;
        b1[0] = lo_odd ? s0.x : s0.y;
        b1[1] = lo_odd ? s0.y : s1.x;
        b1[2] = lo_odd ? s1.x : s1.y;
        double g00 = ha[0] * eb[0] + ha[1] * eb[1] + ha[2] * eb[2];
        double g01 = ha[0] * eb[3] + ha[1] * eb[4] + ha[2] * eb[5];
        double g10 = ha[3] * eb[0] + ha[4] * eb[1] + ha[5] * eb[2];
        double g11 = ha[3] * eb[3] + ha[4] * eb[4] + ha[5] * eb[5];
        // S_ab = F_a^T (G F_b): the lane's three columns of G F_b first (12 FMA),
        // then 2 FMA per output -- 78 FMA per lane and pair instead of 102 for
        // (F_a^T G) F_b, which needs all nine rows of F_a^T G in every lane
        double z0[3], z1[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          z0[c] = g00 * b0[c] + g01 * b1[c];
          z1[c] = g10 * b0[c] + g11 * b1[c];
        }
#pragma unroll
        for (int r = 0; r < 9; ++r) {
          double fr0 = fa[r], fr1 = fa[9 + r];
#pragma unroll
          for (int c = 0; c < 3; ++c) acc[r * 3 + c] += fr0 * z0[c] + fr1 * z1[c];
        }
      }
      __syncwarp();
    }
    cp_async_wait<0>();
    __syncwarp();
    if (active) {
      double* sij = S + (int64_t)blk * 81;
      double* sji = S + (int64_t)up_tpos[u] * 81;
#pragma unroll
      for (int r = 0; r < 9; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double v = -acc[r * 3 + c];
          sij[r * 9 + c0 + c] = v;
          sji[(c0 + c) * 9 + r] = v;
        }
    }
  }
}

// ---------------------------------------------------------------------------
// Row-owned off-diagonal assembly. One CTA owns camera row i and accumulates its
// upper blocks S_ij (j > i) in shared memory. It walks camera i's observations in
// point order; for observation a (point p) the partners b > a of p's segment are
// exactly the cameras j > i of p (segments are sorted by camera), contiguous in
// memory. Warp w owns the slots s = w (mod 8), so every block is accumulated by
// one warp in a fixed order (deterministic, no atomics); 27 lanes hold a 9x9
// product (lane = row r, column triple cg). Rows with more upper blocks than the
// shared-memory window are processed in several windows.

#define SR_WARPS 16
#define SR_QCAP 160

struct SrEntry {
  int a, b, slot;
};

// One queue entry's 9x9 contribution (lane r9, columns 3cg..3cg+2) -- loads only.
struct SrTerm {
  double a0, a1, b0[3], b1[3];
};

__device__ __forceinline__ SrTerm sr_load(const SrEntry& en, const double* __restrict__ F, const double* __restrict__ E,
                                          const double* __restrict__ H, int r9, int cg) {
  const double* fa = F + (int64_t)en.a * REC;
  const double* ha = H + (int64_t)en.a * REC;
  const double* eb = E + (int64_t)en.b * REC;
  const double* fb = F + (int64_t)en.b * REC + 3 * cg;
  double g00 = ha[0] * eb[0] + ha[1] * eb[1] + ha[2] * eb[2];
  double g01 = ha[0] * eb[3] + ha[1] * eb[4] + ha[2] * eb[5];
  double g10 = ha[3] * eb[0] + ha[4] * eb[1] + ha[5] * eb[2];
  double g11 = ha[3] * eb[3] + ha[4] * eb[4] + ha[5] * eb[5];
  double f0 = fa[r9], f1 = fa[9 + r9];
  SrTerm t;
  t.a0 = f0 * g00 + f1 * g10;
  t.a1 = f0 * g01 + f1 * g11;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    t.b0[c] = fb[c];
    t.b1[c] = fb[9 + c];
  }
  return t;
}

__device__ __forceinline__ void sr_add(double* acc, const SrEntry& en, const SrTerm& t, int r9, int cg) {
  double* ac = acc + en.slot * 81 + r9 * 9 + 3 * cg;
#pragma unroll
  for (int c = 0; c < 3; ++c) ac[c] += t.a0 * t.b0[c] + t.a1 * t.b1[c];
}

// Drain a warp queue: two entries in flight, accumulated in queue order.
__device__ __forceinline__ void sr_drain(double* acc, const SrEntry* q, int qn, const double* __restrict__ F,
                                         const double* __restrict__ E, const double* __restrict__ H, int lane, int r9,
                                         int cg) {
  if (lane < 27) {
    int t = 0;
    for (; t + 1 < qn; t += 2) {
      SrEntry e0 = q[t], e1 = q[t + 1];
      SrTerm x0 = sr_load(e0, F, E, H, r9, cg);
      SrTerm x1 = sr_load(e1, F, E, H, r9, cg);
      sr_add(acc, e0, x0, r9, cg);
      sr_add(acc, e1, x1, r9, cg);
    }
    if (t < qn) {
      SrEntry e0 = q[t];
      SrTerm x0 = sr_load(e0, F, E, H, r9, cg);
      sr_add(acc, e0, x0, r9, cg);
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(SR_WARPS * 32)
k_schur_rows(const int* __restrict__ cam_ptr, const int* __restrict__ cm_list, const int* __restrict__ pt_ptr,
             const int* __restrict__ obs_cam, const int* __restrict__ obs_pt, const double* __restrict__ F,
             const double* __restrict__ E, const double* __restrict__ H, const int* __restrict__ S_ptr,
             const int* __restrict__ S_col, const int* __restrict__ dpos, const int* __restrict__ up_tpos,
             const int* __restrict__ up_off, int nc, int use_map, int win_cap, unsigned int* __restrict__ next_row,
             double* __restrict__ S) {
  extern __shared__ double sm[];
  double* acc = sm;                                             // [win_cap][81]
  SrEntry* queue = reinterpret_cast<SrEntry*>(acc + (size_t)win_cap * 81);  // [SR_WARPS][SR_QCAP]
  int* cols = reinterpret_cast<int*>(queue + SR_WARPS * SR_QCAP);          // [win_cap] (binary search mode)
  unsigned short* map = reinterpret_cast<unsigned short*>(cols + win_cap);  // [nc] (map mode)
  __shared__ int s_row;
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  SrEntry* q = queue + w * SR_QCAP;
  int r9 = lane / 3, cg = lane - 3 * r9;  // lanes 0..26: output row r9, columns 3cg..3cg+2
  if (use_map)
    for (int j = threadIdx.x; j < nc; j += blockDim.x) map[j] = 0xFFFF;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_row = (int)atomicAdd(next_row, 1u);
    __syncthreads();
    int i = s_row;
    if (i >= nc) break;
    int u0 = dpos[i] + 1;  // first upper slot of the row in S
    int n_up = S_ptr[i + 1] - u0;
    for (int w0 = 0; w0 < n_up; w0 += win_cap) {
      int wn = min(win_cap, n_up - w0);
      for (int t = threadIdx.x; t < wn * 81; t += blockDim.x) acc[t] = 0.0;
      for (int t = threadIdx.x; t < wn; t += blockDim.x) {
        int j = S_col[u0 + w0 + t];
        if (use_map) map[j] = (unsigned short)t;
        else cols[t] = j;
      }
      __syncthreads();
      int qn = 0;
      int c_lo = S_col[u0 + w0], c_hi = S_col[u0 + w0 + wn - 1];
      unsigned lt = (1u << lane) - 1u;
      for (int base = cam_ptr[i]; base < cam_ptr[i + 1]; base += 32) {
        int qq = base + lane;
        int a = -1, e = 0;
        if (qq < cam_ptr[i + 1]) {
          a = cm_list[qq];
          e = pt_ptr[obs_pt[a] + 1];
        }
        // pass 1: how many partners of a this warp owns; pass 2: write them
        // contiguously per lane (queue order = camera-i observation order)
        int own = 0;
        for (int b = a + 1; a >= 0 && b < e; ++b) {
          int j = obs_cam[b];
          if (j < c_lo || j > c_hi) continue;
          int slot = use_map ? (int)map[j] : lower_bound_i32(cols, wn, j);
          if ((slot & (SR_WARPS - 1)) == w) ++own;
        }
        int incl = own;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int t = __shfl_up_sync(FULL_MASK, incl, o);
          if (lane >= o) incl += t;
        }
        int total = __shfl_sync(FULL_MASK, incl, 31);
        if (qn + total > SR_QCAP) {
          sr_drain(acc, q, qn, F, E, H, lane, r9, cg);
          qn = 0;
        }
        if (total > SR_QCAP) {  // pathological point sizes: one lane at a time
          for (int src = 0; src < 32; ++src) {
            int sa = __shfl_sync(FULL_MASK, a, src), se = __shfl_sync(FULL_MASK, e, src);
            for (int b0 = sa + 1; sa >= 0 && b0 < se; b0 += 32) {
              int b = b0 + lane, slot = -1;
              if (b < se) {
                int j = obs_cam[b];
                if (j >= c_lo && j <= c_hi) slot = use_map ? (int)map[j] : lower_bound_i32(cols, wn, j);
              }
              bool mine = slot >= 0 && (slot & (SR_WARPS - 1)) == w;
              unsigned bal = __ballot_sync(FULL_MASK, mine);
              if (mine) q[qn + __popc(bal & lt)] = SrEntry{sa, b, slot};
              qn += __popc(bal);
              if (qn > SR_QCAP - 32) {
                __syncwarp();
                sr_drain(acc, q, qn, F, E, H, lane, r9, cg);
                qn = 0;
              }
            }
          }
          continue;
        }
        int pos = qn + incl - own;
        for (int b = a + 1; a >= 0 && b < e; ++b) {
          int j = obs_cam[b];
          if (j < c_lo || j > c_hi) continue;
          int slot = use_map ? (int)map[j] : lower_bound_i32(cols, wn, j);
          if ((slot & (SR_WARPS - 1)) == w) q[pos++] = SrEntry{a, b, slot};
        }
        qn += total;
        __syncwarp();
      }
      __syncwarp();
      sr_drain(acc, q, qn, F, E, H, lane, r9, cg);
      __syncthreads();
      // write S_ij (j > i) and its transpose S_ji
      int ub = up_off[i] + w0;
      for (int t = threadIdx.x; t < wn * 81; t += blockDim.x) {
        int s = t / 81, e = t - s * 81;
        int rr = e / 9, cc = e - rr * 9;
        double v = -acc[t];
        S[(int64_t)(u0 + w0 + s) * 81 + e] = v;
        S[(int64_t)up_tpos[ub + s] * 81 + cc * 9 + rr] = v;
      }
      if (use_map)
        for (int t = threadIdx.x; t < wn; t += blockDim.x) map[S_col[u0 + w0 + t]] = 0xFFFF;
      __syncthreads();
    }
  }
}

static size_t schur_diag_smem(bool with_rhs) {
  const size_t sm = sizeof(double) * 4 * SD_STAGES * (with_rhs ? 16 : 15) * 64;
  static bool attr[2] = {false, false};
  if (!attr[with_rhs]) {
    if (with_rhs) cudaFuncSetAttribute(k_schur_diag<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    else cudaFuncSetAttribute(k_schur_diag<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr[with_rhs] = true;
  }
  return sm;
}

static void schur_diag_launch(const int* cam_ptr, const int* cm_list, const double* J, const double* A,
                              const int* dpos, int nc, const double* qo, const double* g_cam, double* rhs, double* S,
                              cudaStream_t st) {
  int g = grid_for((int64_t)nc * 32, 128, 8);
  if (rhs)
    launch(k_schur_diag<true>, g, 128, schur_diag_smem(true), st, cam_ptr, cm_list, J, A, dpos, nc, qo, g_cam, rhs, S);
  else
    launch(k_schur_diag<false>, g, 128, schur_diag_smem(false), st, cam_ptr, cm_list, J, A, dpos, nc, qo, g_cam, rhs,
           S);
}

extern "C" int bamg_schur_numeric_rows(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list,
                                       const int32_t* pt_ptr, const int32_t* obs_cam_pm, const int32_t* obs_pt_pm,
                                       const double* J, const double* A, const int32_t* S_ptr, const int32_t* S_col,
                                       const int32_t* dpos, const int32_t* up_off, const int32_t* up_tpos, int32_t nc,
                                       double* S, void* stream) {
  cudaStream_t st = as_stream(stream);
  if (nc <= 0) return 0;
  schur_diag_launch(cam_ptr, cm_list, J, A, dpos, nc, nullptr, nullptr, nullptr, S, st);
  const size_t budget = 200 * 1024;
  size_t fixed = sizeof(SrEntry) * SR_WARPS * SR_QCAP;
  int use_map = (nc <= 40000) ? 1 : 0;
  size_t map_bytes = use_map ? ((sizeof(unsigned short) * (size_t)nc + 15) & ~size_t(15)) : 0;
  int win_cap = (int)((budget - fixed - map_bytes) / (81 * sizeof(double) + sizeof(int)));
  if (win_cap > 512) win_cap = 512;
  if (win_cap < 8) {
    bamg_set_error("schur rows: shared-memory window too small");
    return BAMG_ERR_UNSUPPORTED;
  }
  size_t sm = (size_t)win_cap * 81 * sizeof(double) + fixed + sizeof(int) * (size_t)win_cap + map_bytes;
  BAMG_CUDA_CHECK(cudaFuncSetAttribute(k_schur_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  unsigned* ctr = ctx->counters + BAMG_CTR_MISC;
  BAMG_CUDA_CHECK(cudaMemsetAsync(ctr, 0, sizeof(unsigned), st));
  int blocks = bamg_num_sms() * (sm <= 100 * 1024 ? 2 : 1);
  launch(k_schur_rows, blocks, SR_WARPS * 32, sm, st, cam_ptr, cm_list, pt_ptr, obs_cam_pm, obs_pt_pm, J + RF,
         J + RE, J + RH, S_ptr, S_col, dpos, up_tpos, up_off, nc, use_map, win_cap, ctr, S);
  BAMG_LAUNCH_CHECK();
  return 0;
}

extern "C" int bamg_schur_numeric(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list, const double* J,
                                  const double* A, const int32_t* dpos, int32_t nc, const int32_t* up_blk,
                                  const int32_t* up_tpos, int32_t n_up, const int32_t* blk_pair_ptr,
                                  const int32_t* pair_a, const int32_t* pair_b, const double* qo, const double* g_cam,
                                  double* rhs, double* S, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (nc) schur_diag_launch(cam_ptr, cm_list, J, A, dpos, nc, qo, g_cam, rhs, S, st);
  if (n_up) {
    int64_t warps = ceil_div(n_up, OFF_GROUPS);
    static const int variant = [] {
      const char* e = getenv("BAMG_SCHUR_OFF");
      return (e && e[0] == 'r') ? 1 : 0;  // "reg": the register-only kernel
    }();
    if (variant == 1) {
      launch(k_schur_offdiag, grid_for(warps * 32, 128, 8), 128, 0, st, up_blk, up_tpos, n_up, blk_pair_ptr, pair_a,
             pair_b, J, S);
    } else {
      const size_t sm = 4 * OFFP_WARP_DOUBLES * sizeof(double);
      static bool attr = false;
      if (!attr) {
        BAMG_CUDA_CHECK(cudaFuncSetAttribute(k_schur_offdiag_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        attr = true;
      }
      launch(k_schur_offdiag_pipe, grid_for(warps * 32, 128, 8), 128, sm, st, up_blk, up_tpos, n_up, blk_pair_ptr,
             pair_a, pair_b, J, S);
    }
  }
  BAMG_LAUNCH_CHECK();
  return 0;
}

// ===========================================================================
// Point-chunk phased assembly (schur.py:128-144, same sums in another order).
//
// The block-owned pair lists above read both records of every point pair: 90.5 M
// pairs x ~450 B at config 4, with no reuse in L2 (a record's ~6 uses are spread
// over the whole run: ncu read 46 GB for 7.5 GB of records). Here the points are
// cut into chunks of consecutive points in (first camera, point) order, each chunk
// holding about `chunk_records` observations (a few tens of MB of records), and the
// pairs are sorted by (chunk, S block). A work item is one (chunk, block) segment;
// items run in chunk order, so while a chunk is in flight its records stay in L2
// and every record comes from DRAM about once. A block's running sum travels
// through its own S slot: the first segment stores the partial, later segments
// (later chunks) wait on the block's completion counter, load the partial and add
// theirs, the last one writes -S_ij and its transpose. Every block is summed in one
// fixed order (chunk, then point) by one lane group at a time: deterministic, no
// floating-point atomics.

__global__ void k_point_firstcam(const int* __restrict__ pt_ptr, const int* __restrict__ ocam, int npt, int nc,
                                 uint32_t* __restrict__ key, uint32_t* __restrict__ val) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < npt; p += gridDim.x * blockDim.x) {
    int s = pt_ptr[p], e = pt_ptr[p + 1];
    key[p] = (e - s >= 2) ? (uint32_t)ocam[s] : (uint32_t)nc;  // points without pairs last
    val[p] = (uint32_t)p;
  }
}

__global__ void k_chunk_counts(const uint32_t* __restrict__ order, const int* __restrict__ pt_ptr, int npt,
                               int* __restrict__ cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npt; i += gridDim.x * blockDim.x) {
    int p = (int)order[i];
    int m = pt_ptr[p + 1] - pt_ptr[p];
    cnt[i] = m >= 2 ? m : 0;
  }
}

// chunk c (in first-camera order) runs at position (c mod K) * ceil(n / K) + c / K:
// consecutive chunks in the run are K apart in camera order, so they rarely share an
// S block and a segment seldom waits for the previous chunk's segment of its block
__global__ void k_chunk_assign(const uint32_t* __restrict__ order, const int* __restrict__ cum, int npt,
                               int64_t chunk_records, int n_chunks, int stride, int* __restrict__ ch) {
  int per = (n_chunks + stride - 1) / stride;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npt; i += gridDim.x * blockDim.x) {
    int c = (int)((int64_t)cum[i] / chunk_records);
    ch[order[i]] = (c % stride) * per + c / stride;
  }
}

// pairs of point p keyed (chunk(p) << blk_bits) | S position; value packed a << 7 | (b - a)
// (PACKED) or the pair's emission index (payload for a gather)
template <bool PACKED>
__global__ void k_pair_emit_chunk(const int* __restrict__ pt_ptr, const int* __restrict__ ocam,
                                  const int* __restrict__ S_ptr, const int* __restrict__ S_col,
                                  const int* __restrict__ off, const int* __restrict__ ch, int npt, int blk_bits,
                                  uint32_t* __restrict__ key, uint32_t* __restrict__ val, int* __restrict__ oa,
                                  int* __restrict__ ob) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < npt; p += gridDim.x * blockDim.x) {
    int s = pt_ptr[p], e = pt_ptr[p + 1];
    int pos = off[p];
    uint32_t hi = (uint32_t)ch[p] << blk_bits;
    for (int a = s; a < e; ++a) {
      int ca = ocam[a];
      const int* cols = S_col + S_ptr[ca];
      int n = S_ptr[ca + 1] - S_ptr[ca];
      for (int b = a + 1; b < e; ++b) {
        int q = lower_bound_i32(cols, n, ocam[b]);
        key[pos] = hi | (uint32_t)(S_ptr[ca] + q);
        if (PACKED) {
          val[pos] = ((uint32_t)a << 7) | (uint32_t)(b - a);
        } else {
          val[pos] = (uint32_t)pos;
          oa[pos] = a;
          ob[pos] = b;
        }
        ++pos;
      }
    }
  }
}

__global__ void k_seg_heads(const uint32_t* __restrict__ key, int64_t n, int* __restrict__ head) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    head[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

// heads -> segment starts / keys (sid = exclusive scan of the head flags)
__global__ void k_seg_fill(const uint32_t* __restrict__ key, const int* __restrict__ sid, int64_t n,
                           int* __restrict__ seg_start, uint32_t* __restrict__ seg_key) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (i == 0 || key[i] != key[i - 1]) {
      seg_start[sid[i]] = (int)i;
      seg_key[sid[i]] = key[i];
    }
  }
}

// per segment: block position (sort key of the ordinal pass), row, transposed position
__global__ void k_seg_info(const uint32_t* __restrict__ seg_key, int nseg, int blk_bits,
                           const int* __restrict__ S_ptr, const int* __restrict__ S_col, int nc,
                           uint32_t* __restrict__ blk_key, uint32_t* __restrict__ iota, int* __restrict__ row,
                           int* __restrict__ tpos) {
  uint32_t mask = (blk_bits >= 32) ? 0xFFFFFFFFu : ((1u << blk_bits) - 1u);
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nseg; s += gridDim.x * blockDim.x) {
    int q = (int)(seg_key[s] & mask);
    // row i: last row with S_ptr[i] <= q
    int lo = 0, hi = nc;
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (S_ptr[mid] <= q) lo = mid; else hi = mid;
    }
    int i = lo, j = S_col[q];
    row[s] = i;
    tpos[s] = S_ptr[j] + lower_bound_i32(S_col + S_ptr[j], S_ptr[j + 1] - S_ptr[j], i);
    blk_key[s] = (uint32_t)q;
    iota[s] = (uint32_t)s;
  }
}

// segments sorted by block (stable: chunk order inside a block) -> ordinal and last flag
__global__ void k_seg_ordinal(const uint32_t* __restrict__ bkey, const uint32_t* __restrict__ bseg, int nseg,
                              int* __restrict__ ord2) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nseg; i += gridDim.x * blockDim.x) {
    uint32_t b = bkey[i];
    int d = 0;
    while (i - d - 1 >= 0 && bkey[i - d - 1] == b) ++d;
    bool last = (i + 1 >= nseg) || bkey[i + 1] != b;
    ord2[bseg[i]] = d * 2 + (last ? 1 : 0);
  }
}

// work order keys: pass 1 longest first (8 bits), pass 2 (chunk, row) stable
__global__ void k_seg_lenkey(const int* __restrict__ seg_start, int nseg, int64_t n_pairs, uint32_t* __restrict__ key,
                             uint32_t* __restrict__ iota) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nseg; s += gridDim.x * blockDim.x) {
    int64_t e = (s + 1 < nseg) ? seg_start[s + 1] : n_pairs;
    int len = (int)(e - seg_start[s]);
    key[s] = 255u - (uint32_t)min(len, 255);
    iota[s] = (uint32_t)s;
  }
}

__global__ void k_seg_rowkey(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ seg_key, int nseg,
                             int blk_bits, const int* __restrict__ row, int row_bits, uint32_t* __restrict__ key,
                             int* __restrict__ chunk_of) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nseg; i += gridDim.x * blockDim.x) {
    int s = (int)perm[i];
    uint32_t c = blk_bits >= 32 ? 0u : (seg_key[s] >> blk_bits);
    key[i] = row_bits > 0 ? ((c << row_bits) | (uint32_t)row[s]) : c;
    chunk_of[i] = (int)c;
  }
}

// per chunk: padded segment count (multiple of OFF_GROUPS, so no warp batch spans two
// chunks: a block then never appears twice in one batch)
__global__ void k_chunk_pad(const int* __restrict__ cptr, int nch, int* __restrict__ padded) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nch; c += gridDim.x * blockDim.x) {
    int n = cptr[c + 1] - cptr[c];
    padded[c] = (n + OFF_GROUPS - 1) / OFF_GROUPS * OFF_GROUPS;
  }
}

__global__ void k_work_fill(const uint32_t* __restrict__ perm, const int* __restrict__ chunk_of, int nseg,
                            const int* __restrict__ cptr, const int* __restrict__ wpos, const int* __restrict__ seg_start,
                            const uint32_t* __restrict__ seg_key, const int* __restrict__ tpos,
                            const int* __restrict__ ord2, int64_t n_pairs, int blk_bits, int4* __restrict__ work,
                            int* __restrict__ bad) {
  uint32_t mask = (blk_bits >= 32) ? 0xFFFFFFFFu : ((1u << blk_bits) - 1u);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nseg; i += gridDim.x * blockDim.x) {
    int s = (int)perm[i];
    int c = chunk_of[i];
    int pos = wpos[c] + (i - cptr[c]);
    int64_t e = (s + 1 < nseg) ? seg_start[s + 1] : n_pairs;
    int len = (int)(e - seg_start[s]);
    int o2 = ord2[s];
    if (len >= (1 << 21) || (o2 >> 1) >= (1 << 9)) atomicExch(bad, 1);
    work[pos] = make_int4(seg_start[s], (int)(seg_key[s] & mask), tpos[s],
                          len | ((o2 >> 1) << 21) | ((o2 & 1) << 30));
  }
}

__global__ void k_work_pad_init(int4* __restrict__ work, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    work[i] = make_int4(0, -1, 0, 0);
}

static int bits_of(int64_t n) {
  int b = 1;
  while ((1ll << b) < n) ++b;
  return b;
}

extern "C" int bamg_schur_chunk_pairs(bamg_ctx* ctx, const int32_t* pt_ptr, const int32_t* obs_cam_pm,
                                      const int32_t* S_ptr, const int32_t* S_col, int32_t nc, int32_t npt,
                                      int64_t nnz, int64_t k, const int32_t* pair_off, int64_t n_pairs,
                                      int64_t chunk_records, int32_t* pair_a, int32_t* pair_b, uint32_t* sorted_key,
                                      int64_t* out_host, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  const int blk_bits = bits_of(nnz + 1);
  if (blk_bits > 30) {
    bamg_set_error("schur chunks: %lld S blocks exceed the 30-bit key", (long long)nnz);
    return BAMG_ERR_UNSUPPORTED;
  }
  const int64_t max_chunks = 1ll << (32 - blk_bits);
  if (chunk_records < 1) chunk_records = 1;
  if (ceil_div(k, chunk_records) + 64 > max_chunks) chunk_records = ceil_div(k, max_chunks - 64);
  out_host[0] = 0;
  out_host[1] = ceil_div(k > 0 ? k : 1, chunk_records);
  out_host[2] = blk_bits;
  out_host[3] = chunk_records;
  if (n_pairs == 0 || npt == 0) return 0;
  // 1. chunk of every point: consecutive points in (first camera, point) order
  uint32_t *pk = nullptr, *pv = nullptr, *spk = nullptr, *spv = nullptr;
  int *cum = nullptr, *ch = nullptr, *mx = nullptr;
  BAMG_CUDA_CHECK(cudaMallocAsync(&pk, 4 * (size_t)npt, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&pv, 4 * (size_t)npt, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&spk, 4 * (size_t)npt, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&spv, 4 * (size_t)npt, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&cum, 4 * (size_t)npt + 4, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&ch, 4 * (size_t)npt, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&mx, 8, st));
  launch(k_point_firstcam, grid_for(npt, 256), 256, 0, st, pt_ptr, obs_cam_pm, npt, nc, pk, pv);
  int rc = radix_sort_pairs(pk, pv, spk, spv, npt, bits_of((int64_t)nc + 1), st);
  if (rc) return rc;
  launch(k_chunk_counts, grid_for(npt, 256), 256, 0, st, spv, pt_ptr, npt, cum);
  rc = scan_exclusive_int(cum, cum, npt, nullptr, st);
  if (rc) return rc;
  {
    int stride = 8;
    if (const char* e = getenv("BAMG_SCHUR_CHUNK_STRIDE")) stride = atoi(e) > 0 ? atoi(e) : 1;
    int nch = (int)ceil_div(k > 0 ? k : 1, chunk_records);
    if (stride > nch) stride = nch;
    // positions run up to stride * ceil(nch / stride) - 1
    out_host[1] = (int64_t)stride * ceil_div(nch, stride);
    launch(k_chunk_assign, grid_for(npt, 256), 256, 0, st, spv, cum, npt, chunk_records, nch, stride, ch);
  }
  // 2. pairs keyed (chunk, block), sorted (stable: point order inside a segment)
  int h[2] = {0, 0};
  BAMG_CUDA_CHECK(cudaMemsetAsync(mx, 0, 8, st));
  launch(k_max_segment, grid_for(npt, 256), 256, 0, st, pt_ptr, npt, mx);
  BAMG_CUDA_CHECK(cudaMemcpyAsync(h, mx, sizeof(int), cudaMemcpyDeviceToHost, st));
  BAMG_CUDA_CHECK(cudaStreamSynchronize(st));
  const bool packed = k < (1ll << 25) && h[0] <= 128;
  uint32_t *key = nullptr, *val = nullptr, *sval = nullptr;
  int *oa = nullptr, *ob = nullptr;
  BAMG_CUDA_CHECK(cudaMallocAsync(&key, 4 * n_pairs, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&val, 4 * n_pairs, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&sval, 4 * n_pairs, st));
  if (packed) {
    launch(k_pair_emit_chunk<true>, grid_for(npt, 128), 128, 0, st, pt_ptr, obs_cam_pm, S_ptr, S_col, pair_off, ch,
           npt, blk_bits, key, val, (int*)nullptr, (int*)nullptr);
  } else {
    BAMG_CUDA_CHECK(cudaMallocAsync(&oa, 4 * n_pairs, st));
    BAMG_CUDA_CHECK(cudaMallocAsync(&ob, 4 * n_pairs, st));
    launch(k_pair_emit_chunk<false>, grid_for(npt, 128), 128, 0, st, pt_ptr, obs_cam_pm, S_ptr, S_col, pair_off, ch,
           npt, blk_bits, key, val, oa, ob);
  }
  BAMG_LAUNCH_CHECK();
  rc = radix_sort_pairs(key, val, sorted_key, sval, n_pairs, 32, st);
  if (rc) return rc;
  if (packed) {
    launch(k_unpack_pairs, grid_for(n_pairs, 256), 256, 0, st, (const uint32_t*)sval, n_pairs, pair_a, pair_b);
  } else {
    launch(k_gather_pairs, grid_for(n_pairs, 256), 256, 0, st, sval, oa, ob, n_pairs, pair_a, pair_b);
    cudaFreeAsync(oa, st);
    cudaFreeAsync(ob, st);
  }
  // 3. segment count
  int* head = (int*)val;  // reuse: n_pairs ints
  launch(k_seg_heads, grid_for(n_pairs, 256), 256, 0, st, sorted_key, n_pairs, head);
  int* tot = mx;
  rc = scan_exclusive_int(head, head, n_pairs, tot, st);
  if (rc) return rc;
  BAMG_CUDA_CHECK(cudaMemcpyAsync(h, tot, sizeof(int), cudaMemcpyDeviceToHost, st));
  BAMG_CUDA_CHECK(cudaStreamSynchronize(st));
  BAMG_LAUNCH_CHECK();
  out_host[0] = h[0];
  for (void* p : {(void*)pk, (void*)pv, (void*)spk, (void*)spv, (void*)cum, (void*)ch, (void*)mx, (void*)key,
                  (void*)val, (void*)sval})
    cudaFreeAsync(p, st);
  return 0;
}

extern "C" int bamg_schur_chunk_work(bamg_ctx* ctx, const int32_t* S_ptr, const int32_t* S_col, int32_t nc,
                                     const uint32_t* sorted_key, int64_t n_pairs, int32_t n_seg, int32_t n_chunks,
                                     int32_t blk_bits, int32_t group_rows, int32_t* work, int64_t work_cap,
                                     int64_t* out_host, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  out_host[0] = 0;
  if (n_seg <= 0) return 0;
  int *sid = nullptr, *seg_start = nullptr, *row = nullptr, *tpos = nullptr, *ord2 = nullptr, *chunk_of = nullptr;
  int *cptr = nullptr, *padded = nullptr, *bad = nullptr;
  uint32_t *seg_key = nullptr, *k1 = nullptr, *v1 = nullptr, *k2 = nullptr, *v2 = nullptr;
  BAMG_CUDA_CHECK(cudaMallocAsync(&sid, 4 * n_pairs, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&seg_start, 4 * (size_t)n_seg, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&seg_key, 4 * (size_t)n_seg, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&row, 4 * (size_t)n_seg, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&tpos, 4 * (size_t)n_seg, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&ord2, 4 * (size_t)n_seg, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&chunk_of, 4 * (size_t)n_seg, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&k1, 4 * (size_t)n_seg, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&v1, 4 * (size_t)n_seg, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&k2, 4 * (size_t)n_seg, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&v2, 4 * (size_t)n_seg, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&cptr, 4 * ((size_t)n_chunks + 1), st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&padded, 4 * ((size_t)n_chunks + 1), st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&bad, 8, st));
  BAMG_CUDA_CHECK(cudaMemsetAsync(bad, 0, 8, st));
  launch(k_seg_heads, grid_for(n_pairs, 256), 256, 0, st, sorted_key, n_pairs, sid);
  int rc = scan_exclusive_int(sid, sid, n_pairs, nullptr, st);
  if (rc) return rc;
  launch(k_seg_fill, grid_for(n_pairs, 256), 256, 0, st, sorted_key, sid, n_pairs, seg_start, seg_key);
  // ordinals: segments of a block in chunk order
  launch(k_seg_info, grid_for(n_seg, 256), 256, 0, st, seg_key, n_seg, blk_bits, S_ptr, S_col, nc, k1, v1, row, tpos);
  rc = radix_sort_pairs(k1, v1, k2, v2, n_seg, blk_bits, st);
  if (rc) return rc;
  launch(k_seg_ordinal, grid_for(n_seg, 256), 256, 0, st, k2, v2, n_seg, ord2);
  // work order: (chunk, row) with the longest segments first inside a row
  launch(k_seg_lenkey, grid_for(n_seg, 256), 256, 0, st, seg_start, n_seg, n_pairs, k1, v1);
  rc = radix_sort_pairs(k1, v1, k2, v2, n_seg, 8, st);
  if (rc) return rc;
  const int chunk_bits = bits_of((int64_t)n_chunks + 1);
  int row_bits = group_rows ? bits_of((int64_t)nc + 1) : 0;
  if (chunk_bits + row_bits > 32) row_bits = 0;
  launch(k_seg_rowkey, grid_for(n_seg, 256), 256, 0, st, v2, seg_key, n_seg, blk_bits, row, row_bits, k1, chunk_of);
  rc = radix_sort_pairs(k1, v2, k2, v1, n_seg, chunk_bits + row_bits, st);  // v1 = final order
  if (rc) return rc;
  launch(k_seg_rowkey, grid_for(n_seg, 256), 256, 0, st, v1, seg_key, n_seg, blk_bits, row, 0, k1, chunk_of);
  rc = segment_ptr(chunk_of, n_seg, n_chunks, cptr, st);
  if (rc) return rc;
  launch(k_chunk_pad, grid_for(n_chunks, 256), 256, 0, st, cptr, n_chunks, padded);
  int* tot = bad + 1;
  rc = scan_exclusive_int(padded, padded, n_chunks, tot, st);
  if (rc) return rc;
  int h[2] = {0, 0};
  BAMG_CUDA_CHECK(cudaMemcpyAsync(h, bad, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  BAMG_CUDA_CHECK(cudaStreamSynchronize(st));
  if (h[1] > work_cap) {
    bamg_set_error("schur chunks: work list %d exceeds capacity %lld", h[1], (long long)work_cap);
    return BAMG_ERR_UNSUPPORTED;
  }
  int4* w4 = reinterpret_cast<int4*>(work);
  launch(k_work_pad_init, grid_for(h[1], 256), 256, 0, st, w4, (int64_t)h[1]);
  launch(k_work_fill, grid_for(n_seg, 256), 256, 0, st, v1, chunk_of, n_seg, cptr, padded, seg_start, seg_key, tpos,
         ord2, n_pairs, blk_bits, w4, bad);
  BAMG_CUDA_CHECK(cudaMemcpyAsync(h, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  BAMG_CUDA_CHECK(cudaStreamSynchronize(st));
  BAMG_LAUNCH_CHECK();
  for (void* p : {(void*)sid, (void*)seg_start, (void*)seg_key, (void*)row, (void*)tpos, (void*)ord2,
                  (void*)chunk_of, (void*)k1, (void*)v1, (void*)k2, (void*)v2, (void*)cptr, (void*)padded,
                  (void*)bad})
    cudaFreeAsync(p, st);
  if (h[0]) {
    bamg_set_error("schur chunks: a segment exceeds 2^21 pairs or a block 512 chunks");
    return BAMG_ERR_UNSUPPORTED;
  }
  out_host[0] = h[1];
  return 0;
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Work item (int4): x = first pair, y = S position of the upper block (-1: padding),
// z = transposed position, w = length | ordinal << 21 | last << 30. Warps take
// batches of OFF_GROUPS items from a global counter (dispensed in work order, so a
// segment only ever waits on segments owned by running warps: no deadlock).
// Measured at c4 (profiles/r2/schur_experiments.md): DRAM read 46 -> 14.4 GB, but
// 8.6 ms against the block-owned kernel's 7.6 ms -- 4.5 M short segments (20 pairs
// on average) pay the per-batch latency chain four times as often.
__global__ void __launch_bounds__(128)
k_schur_chunked(const int4* __restrict__ work, int n_work, const int* __restrict__ pair_a,
                const int* __restrict__ pair_b, const double* __restrict__ J, unsigned* __restrict__ done,
                unsigned* __restrict__ next_batch, double* __restrict__ S) {
  extern __shared__ __align__(16) double smem_offp[];
  int lane = threadIdx.x & 31;
  double* wsm = smem_offp + (threadIdx.x >> 5) * OFFP_WARP_DOUBLES;
  int grp = lane / 3, c3 = lane - 3 * grp;
  int c0 = 3 * c3;
  const int fb_lo = (RF + c0) >> 1, fb_hi = (RF + 9 + c0) >> 1;
  const bool lo_odd = (RF + c0) & 1;
  const int ig = lane >> 1;
  const int* ilist = (lane & 1) ? pair_b : pair_a;
  const int n_batches = (n_work + OFF_GROUPS - 1) / OFF_GROUPS;
  for (;;) {
    int bt = 0;
    if (lane == 0) bt = (int)atomicAdd(next_batch, 1u);
    bt = __shfl_sync(FULL_MASK, bt, 0);
    if (bt >= n_batches) break;
    int u = bt * OFF_GROUPS + grp;
    int4 wi = make_int4(0, -1, 0, 0);
    if (grp < OFF_GROUPS && u < n_work) wi = work[u];
    bool active = wi.y >= 0;
    int q0 = wi.x, blk = wi.y;
    int len = active ? (wi.w & ((1 << 21) - 1)) : 0;
    unsigned ord = (unsigned)(wi.w >> 21) & 511u;
    bool last = (wi.w >> 30) & 1;
    int maxlen = len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(FULL_MASK, maxlen, o));
    int src = 3 * ig < 31 ? 3 * ig : 31;
    int iq0 = __shfl_sync(FULL_MASK, q0, src);
    int ilen = __shfl_sync(FULL_MASK, len, src);
    if (lane >= 2 * OFF_GROUPS) ilen = 0;
    int nrec = (ilen > 0) ? ilist[iq0] : -1;
#pragma unroll
    for (int t = 0; t < OFFP_STAGES - 1; ++t) {
      int rec = nrec;
      nrec = (t + 1 < ilen) ? ilist[iq0 + t + 1] : -1;
      if (t < maxlen) offp_issue(wsm + t * OFFP_STAGE_DOUBLES, J, rec, lane);
      else cp_async_commit();
    }
    // the block's running sum from the previous chunk (records are already in flight)
    double acc[27];
    if (active && ord > 0) {
      while (ld_acquire_u32(done + blk) < ord) __nanosleep(64);
      const double* sp = S + (int64_t)blk * 81 + c0;
#pragma unroll
      for (int r = 0; r < 9; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[r * 3 + c] = __ldcg(sp + r * 9 + c);
    } else {
#pragma unroll
      for (int q = 0; q < 27; ++q) acc[q] = 0.0;
    }
    __syncwarp();
    for (int s = 0; s < maxlen; ++s) {
      int t = s + OFFP_STAGES - 1;
      int rec = nrec;
      nrec = (t + 1 < ilen) ? ilist[iq0 + t + 1] : -1;
      if (t < maxlen) offp_issue(wsm + (t % OFFP_STAGES) * OFFP_STAGE_DOUBLES, J, rec, lane);
      else cp_async_commit();
      cp_async_wait<OFFP_STAGES - 1>();
      __syncwarp();
      if (s < len) {
        const double* stg = wsm + (s % OFFP_STAGES) * OFFP_STAGE_DOUBLES;
        const double2* ra = reinterpret_cast<const double2*>(stg + grp * OFFP_RS);
        const double2* rb = reinterpret_cast<const double2*>(stg + (OFF_GROUPS + grp) * OFFP_RS);
        double fa[18], ha[6], eb[6];
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          double2 v = ra[RF / 2 + k];
          fa[2 * k] = v.x;
          fa[2 * k + 1] = v.y;
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          double2 v = ra[RH / 2 + k], w = rb[RE / 2 + k];
          ha[2 * k] = v.x;
          ha[2 * k + 1] = v.y;
          eb[2 * k] = w.x;
          eb[2 * k + 1] = w.y;
        }
        double2 p0 = rb[fb_lo], p1 = rb[fb_lo + 1];
        double2 s0 = rb[fb_hi], s1 = rb[fb_hi + 1];
        double b0[3], b1[3];
        b0[0] = lo_odd ? p0.y : p0.x;
        b0[1] = lo_odd ? p1.x : p0.y;
        b0[2] = lo_odd ? p1.y : p1.x;
        b1[0] = lo_odd ? s0.x : s0.y;
        b1[1] = lo_odd ? s0.y : s1.x;
        b1[2] = lo_odd ? s1.x : s1.y;
        double g00 = ha[0] * eb[0] + ha[1] * eb[1] + ha[2] * eb[2];
        double g01 = ha[0] * eb[3] + ha[1] * eb[4] + ha[2] * eb[5];
        double g10 = ha[3] * eb[0] + ha[4] * eb[1] + ha[5] * eb[2];
        double g11 = ha[3] * eb[3] + ha[4] * eb[4] + ha[5] * eb[5];
        double z0[3], z1[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          z0[c] = g00 * b0[c] + g01 * b1[c];
          z1[c] = g10 * b0[c] + g11 * b1[c];
        }
#pragma unroll
        for (int r = 0; r < 9; ++r) {
          double fr0 = fa[r], fr1 = fa[9 + r];
#pragma unroll
          for (int c = 0; c < 3; ++c) acc[r * 3 + c] += fr0 * z0[c] + fr1 * z1[c];
        }
      }
      __syncwarp();
    }
    cp_async_wait<0>();
    __syncwarp();
    if (active) {
      double* sij = S + (int64_t)blk * 81;
      if (last) {
        double* sji = S + (int64_t)wi.z * 81;
#pragma unroll
        for (int r = 0; r < 9; ++r)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            double v = -acc[r * 3 + c];
            sij[r * 9 + c0 + c] = v;
            sji[(c0 + c) * 9 + r] = v;
          }
      } else {
#pragma unroll
        for (int r = 0; r < 9; ++r)
#pragma unroll
          for (int c = 0; c < 3; ++c) __stcg(sij + r * 9 + c0 + c, acc[r * 3 + c]);
      }
    }
    if (active && !last) __threadfence();
    __syncwarp();
    if (active && !last && c3 == 0) st_release_u32(done + blk, ord + 1);
  }
}

extern "C" int bamg_schur_numeric_chunked(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list,
                                          const double* J, const double* A, const int32_t* dpos, int32_t nc,
                                          const int32_t* work, int32_t n_work, const int32_t* pair_a,
                                          const int32_t* pair_b, uint32_t* done, int64_t nnz, const double* qo,
                                          const double* g_cam, double* rhs, double* S, void* stream) {
  cudaStream_t st = as_stream(stream);
  if (nc) schur_diag_launch(cam_ptr, cm_list, J, A, dpos, nc, qo, g_cam, rhs, S, st);
  if (n_work > 0) {
    BAMG_CUDA_CHECK(cudaMemsetAsync(done, 0, sizeof(uint32_t) * (size_t)nnz, st));
    unsigned* ctr = ctx->counters + BAMG_CTR_MISC;
    BAMG_CUDA_CHECK(cudaMemsetAsync(ctr, 0, sizeof(unsigned), st));
    const size_t sm = 4 * OFFP_WARP_DOUBLES * sizeof(double);
    static int grid = 0;
    if (!grid) {
      BAMG_CUDA_CHECK(cudaFuncSetAttribute(k_schur_chunked, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      int per_sm = 0;
      BAMG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_schur_chunked, 128, sm));
      grid = bamg_num_sms() * (per_sm > 0 ? per_sm : 1);
    }
    int64_t batches = ceil_div(n_work, OFF_GROUPS);
    int g = (int)std::min<int64_t>(grid, ceil_div(batches, 4));
    launch(k_schur_chunked, g, 128, sm, st, reinterpret_cast<const int4*>(work), n_work, pair_a, pair_b, J,
           done, ctr, S);
  }
  BAMG_LAUNCH_CHECK();
  return 0;
}


// ---------------------------------------------------------------------------
// One camera-major pass for everything the camera side of a linear solve needs
// from the observation records (schur.py:38-47, 99-125, 128-144):
//   dA_i  = diag(sum_o F_o^T F_o)                 (normal_diagonal, problem.py:262-269)
//   D_i   = clip(dA_i, 1e-6, 1e32) / radius        (Damping.from_jacobian)
//   S_ii  = sum_o F_o^T (I - H_o E_o^T) F_o + D_i  (= A_i + D_i - sum W C^-1 W^T, one sum)
//   rhs_i = -sum_o F_o^T (r_o + q_o)               (= -g_i - sum W C^-1 b_p)
// Three lanes per observation, ten observations per warp step; lane (g, c) owns
// columns 3c..3c+2 of the 9x9 block (27 accumulators instead of the 45 + 9 + 9 a lane
// per observation would hold, so the pass runs at 4 CTAs / SM instead of 1). The
// records (all 16 pieces) and q stream through a CF_STAGES-deep cp.async pipeline;
// at the end the ten groups' partials are added in group order (deterministic).
// WITH_S = false: only dA / D (the damping of a Jacobian whose S is not assembled).
#define CF_G 10
#define CF_P 17                   // 16 record pieces + q
#define CF_PD (CF_P * CF_G * 2)   // doubles per stage
#ifndef CF_STAGES
#define CF_STAGES 6
#endif

#ifndef CF_MINB
#define CF_MINB 3
#endif
template <bool WITH_S>
__global__ void __launch_bounds__(128, CF_MINB)
k_cam_fused(const int* __restrict__ cam_ptr, const int* __restrict__ cm_list, const double* __restrict__ J,
            const double* __restrict__ qo, int nc, double radius, const int* __restrict__ dpos,
            double* __restrict__ S, double* __restrict__ rhs, double* __restrict__ d_cam,
            double* __restrict__ dA_out) {
  extern __shared__ __align__(16) double cf_smem[];
  const int lane = threadIdx.x & 31;
  double* wbuf = cf_smem + (size_t)(threadIdx.x >> 5) * CF_STAGES * CF_PD;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int g = lane / 3, c = lane - 3 * (lane / 3);
  // copy slots: 10 obs x 17 pieces = 170 chunks, 6 per lane; slot s = lane + 32 it has a
  // fixed (observation, piece), decoded once
  int s_ob[6], s_pc[6], s_dst[6];
#pragma unroll
  for (int it = 0; it < 6; ++it) {
    const int s = lane + 32 * it;
    s_ob[it] = s < CF_P * CF_G ? s / CF_P : (1 << 20);  // no slot
    s_pc[it] = s - CF_P * (s / CF_P);
    s_dst[it] = s_pc[it] * (2 * CF_G) + 2 * s_ob[it];
  }
  auto issue = [&](int q_lo, int q_hi, int idx_lane, double* buf) {
    const int nval = q_hi - q_lo;  // observations of this step (>= 1)
#pragma unroll
    for (int it = 0; it < 6; ++it) {
      const int ob = s_ob[it], pc = s_pc[it];
      const int o = __shfl_sync(FULL_MASK, idx_lane, ob < CF_G ? ob : 0);
      if (ob < nval && (WITH_S || pc < 9)) {
        const double* src = pc < 16 ? J + (int64_t)o * REC + 2 * pc : qo + 2 * (int64_t)o;
        cp_async16(buf + s_dst[it], src);
      }
    }
    cp_async_commit();
  };
  for (int i = warp; i < nc; i += nwarps) {
    const int q0 = cam_ptr[i], q1 = cam_ptr[i + 1];
    double acc[27], dA[3], rr[3];
#pragma unroll
    for (int t = 0; t < 27; ++t) acc[t] = 0.0;
#pragma unroll
    for (int t = 0; t < 3; ++t) dA[t] = rr[t] = 0.0;
    // observation ids: lane l < 10 holds obs l of a step; CF_STAGES - 1 steps issued ahead
    int nidx = 0;
#pragma unroll
    for (int t = 0; t < CF_STAGES - 1; ++t) {
      const int b = q0 + CF_G * t;
      const int id = (lane < CF_G && b + lane < q1) ? cm_list[b + lane] : 0;
      if (b < q1) issue(b, q1, id, wbuf + t * CF_PD);
      else cp_async_commit();
    }
    {
      const int b = q0 + CF_G * (CF_STAGES - 1);
      nidx = (lane < CF_G && b + lane < q1) ? cm_list[b + lane] : 0;
    }
    int st = 0;
    for (int base = q0; base < q1; base += CF_G, ++st) {
      const int nb = base + CF_G * (CF_STAGES - 1);
      if (nb < q1) issue(nb, q1, nidx, wbuf + ((st + CF_STAGES - 1) % CF_STAGES) * CF_PD);
      else cp_async_commit();
      {
        const int b = nb + CF_G;
        nidx = (lane < CF_G && b + lane < q1) ? cm_list[b + lane] : 0;
      }
      cp_async_wait<CF_STAGES - 1>();
      __syncwarp();
      if (g < CF_G && base + g < q1) {
        const double* bf = wbuf + (st % CF_STAGES) * CF_PD + 2 * g;
        auto pcv = [&](int pc) { return *reinterpret_cast<const double2*>(bf + pc * (2 * CF_G)); };
        double f[18];
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          double2 v = pcv(k);
          f[2 * k] = v.x;
          f[2 * k + 1] = v.y;
        }
        // own columns of F (rows 0 and 1), read again from shared memory (element e of
        // the flattened F sits at piece e / 2, half e % 2)
        double f0[3], f1[3];
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const int e0 = 3 * c + t, e1 = 9 + 3 * c + t;
          f0[t] = bf[(e0 >> 1) * (2 * CF_G) + (e0 & 1)];
          f1[t] = bf[(e1 >> 1) * (2 * CF_G) + (e1 & 1)];
          dA[t] += f0[t] * f0[t] + f1[t] * f1[t];
        }
        if constexpr (WITH_S) {
          double e[6], h[6];
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            double2 ve = pcv(RE / 2 + k), vh = pcv(RH / 2 + k);
            e[2 * k] = ve.x;
            e[2 * k + 1] = ve.y;
            h[2 * k] = vh.x;
            h[2 * k + 1] = vh.y;
          }
          const double2 r = pcv(RR / 2), q = pcv(16);
          const double u0 = r.x + q.x, u1 = r.y + q.y;
#pragma unroll
          for (int t = 0; t < 3; ++t) rr[t] += f0[t] * u0 + f1[t] * u1;
          // G' = I - H E^T
          const double m00 = 1.0 - (h[0] * e[0] + h[1] * e[1] + h[2] * e[2]);
          const double m01 = -(h[0] * e[3] + h[1] * e[4] + h[2] * e[5]);
          const double m10 = -(h[3] * e[0] + h[4] * e[1] + h[5] * e[2]);
          const double m11 = 1.0 - (h[3] * e[3] + h[4] * e[4] + h[5] * e[5]);
          double z0[3], z1[3];
#pragma unroll
          for (int t = 0; t < 3; ++t) {
            z0[t] = m00 * f0[t] + m01 * f1[t];
            z1[t] = m10 * f0[t] + m11 * f1[t];
          }
#pragma unroll
          for (int j = 0; j < 9; ++j)
#pragma unroll
            for (int t = 0; t < 3; ++t) acc[j * 3 + t] += f[j] * z0[t] + f[9 + j] * z1[t];
        }
      }
      __syncwarp();
    }
    cp_async_wait<0>();
    __syncwarp();
    // group partials -> shared memory (the stage buffers are free now), added in group order
    constexpr int NV = WITH_S ? 33 : 3;
    double* red = wbuf;  // [CF_G][3][NV]
    if (g < CF_G) {
      double* my = red + (g * 3 + c) * NV;
#pragma unroll
      for (int t = 0; t < 3; ++t) my[t] = dA[t];
      if constexpr (WITH_S) {
#pragma unroll
        for (int t = 0; t < 3; ++t) my[3 + t] = rr[t];
#pragma unroll
        for (int t = 0; t < 27; ++t) my[6 + t] = acc[t];
      }
    }
    __syncwarp();
    // lane l < 9: column l -- its raw diagonal, damping, rhs, and its column of S_ii
    if (lane < 9) {
      const int cc = lane / 3, t = lane - 3 * (lane / 3);
      double da = 0.0, rv = 0.0;
      for (int gg = 0; gg < CF_G; ++gg) {
        const double* p = red + (gg * 3 + cc) * NV;
        da += p[t];
        if constexpr (WITH_S) rv += p[3 + t];
      }
      double d = fmin(fmax(da, 1e-6), 1e32);
      if (d != d) d = da;
      d = d / radius;
      if (d_cam) d_cam[(int64_t)i * 9 + lane] = d;
      if (dA_out) dA_out[(int64_t)i * 9 + lane] = da;
      if constexpr (WITH_S) {
        if (rhs) rhs[(int64_t)i * 9 + lane] = -rv;
        // S_ii[j][l], j <= l, from column l's owner; mirrored to [l][j]
        double* out = S + (int64_t)dpos[i] * 81;
        for (int j = 0; j <= lane; ++j) {
          double v = 0.0;
          for (int gg = 0; gg < CF_G; ++gg) v += red[(gg * 3 + cc) * NV + 6 + j * 3 + t];
          if (j == lane) v += d;
          out[j * 9 + lane] = v;
          out[lane * 9 + j] = v;
        }
      }
    }
    __syncwarp();
  }
}

extern "C" int bamg_camera_pass(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list, const double* J,
                                const double* qo, int32_t nc, double radius, const int32_t* dpos, double* S,
                                double* rhs, double* d_cam, double* dA_raw, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (nc <= 0) return 0;
  const size_t sm = sizeof(double) * 4 * CF_STAGES * CF_PD;
  static bool attr[2] = {false, false};
  const int g = grid_for((int64_t)nc * 32, 128, 16);
  if (S) {
    if (!attr[1]) {
      BAMG_CUDA_CHECK(cudaFuncSetAttribute(k_cam_fused<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      attr[1] = true;
    }
    launch(k_cam_fused<true>, g, 128, sm, st, cam_ptr, cm_list, J, qo, nc, radius, dpos, S, rhs, d_cam, dA_raw);
  } else {
    if (!attr[0]) {
      BAMG_CUDA_CHECK(cudaFuncSetAttribute(k_cam_fused<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      attr[0] = true;
    }
    launch(k_cam_fused<false>, g, 128, sm, st, cam_ptr, cm_list, J, qo, nc, radius, dpos, S, rhs, d_cam, dA_raw);
  }
  BAMG_LAUNCH_CHECK();
  return 0;
}
