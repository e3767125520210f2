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
  k_pair_counts<<<grid_for(npt, 256), 256, 0, st>>>(pt_ptr, npt, pair_off);
  int rc = scan_exclusive_int(pair_off, pair_off, npt, tot, st);
  if (rc) return rc;
  k_row_upper<<<grid_for(nc, 128), 128, 0, st>>>(S_ptr, S_col, nc, dpos, up_off);
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
                                   const int32_t* S_ptr, const int32_t* S_col, int32_t nc, int32_t npt,
                                   int64_t nnz, const int32_t* pair_off, int64_t n_pairs, const int32_t* dpos,
                                   const int32_t* up_off, int32_t* pair_a, int32_t* pair_b, int32_t* blk_pair_ptr,
                                   int32_t* up_blk, int32_t* up_row, int32_t* up_tpos, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  k_upper_list<<<grid_for(nc, 128), 128, 0, st>>>(S_ptr, S_col, nc, dpos, up_off, up_blk, up_row, up_tpos);
  BAMG_LAUNCH_CHECK();
  if (n_pairs == 0) {
    BAMG_CUDA_CHECK(cudaMemsetAsync(blk_pair_ptr, 0, sizeof(int) * (nnz + 1), st));
    return 0;
  }
  uint32_t *key = nullptr, *iota = nullptr, *skey = nullptr, *perm = nullptr;
  int *oa = nullptr, *ob = nullptr;
  BAMG_CUDA_CHECK(cudaMallocAsync(&key, 4 * n_pairs, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&iota, 4 * n_pairs, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&skey, 4 * n_pairs, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&perm, 4 * n_pairs, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&oa, 4 * n_pairs, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&ob, 4 * n_pairs, st));
  k_pair_emit<<<grid_for(npt, 128), 128, 0, st>>>(pt_ptr, obs_cam_pm, S_ptr, S_col, pair_off, npt, key, oa, ob);
  k_iota_u32<<<grid_for(n_pairs, 256), 256, 0, st>>>(iota, n_pairs);
  BAMG_LAUNCH_CHECK();
  int bits = 1;
  while ((1ll << bits) < nnz) ++bits;
  int rc = radix_sort_pairs(key, iota, skey, perm, n_pairs, bits, st);
  if (rc) return rc;
  k_gather_pairs<<<grid_for(n_pairs, 256), 256, 0, st>>>(perm, oa, ob, n_pairs, pair_a, pair_b);
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

// Diagonal blocks: warp per camera, S_ii = A_i - sum_o F_o^T (H_o E_o^T) F_o.
__global__ void __launch_bounds__(128)
k_schur_diag(const int* __restrict__ cam_ptr, const int* __restrict__ cm_list, const double* __restrict__ F,
             const double* __restrict__ E, const double* __restrict__ H, const double* __restrict__ A,
             const int* __restrict__ dpos, int nc, double* __restrict__ S) {
  int lane = threadIdx.x & 31;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < nc; i += nwarps) {
    double acc[45];
#pragma unroll
    for (int q = 0; q < 45; ++q) acc[q] = 0.0;
    for (int q = cam_ptr[i] + lane; q < cam_ptr[i + 1]; q += 32) {
      int64_t o = cm_list[q];
      const double* f = F + o * 18;
      const double* h = H + o * 6;
      const double* e = E + o * 6;
      double g00 = h[0] * e[0] + h[1] * e[1] + h[2] * e[2];
      double g01 = h[0] * e[3] + h[1] * e[4] + h[2] * e[5];
      double g10 = h[3] * e[0] + h[4] * e[1] + h[5] * e[2];
      double g11 = h[3] * e[3] + h[4] * e[4] + h[5] * e[5];
      double f0[9], f1[9];
#pragma unroll
      for (int c = 0; c < 9; ++c) {
        f0[c] = f[c];
        f1[c] = f[9 + c];
      }
      int t = 0;
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        double a0 = f0[j] * g00 + f1[j] * g10;
        double a1 = f0[j] * g01 + f1[j] * g11;
#pragma unroll
        for (int l = j; l < 9; ++l) acc[t++] += a0 * f0[l] + a1 * f1[l];
      }
    }
#pragma unroll
    for (int q = 0; q < 45; ++q) acc[q] = warp_sum(acc[q]);
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

#define OFF_GROUPS 10  // blocks per warp (3 lanes each, lanes 30/31 idle)

__global__ void __launch_bounds__(128)
k_schur_offdiag(const int* __restrict__ up_blk, const int* __restrict__ up_tpos, int n_up,
                const int* __restrict__ blk_pair_ptr, const int* __restrict__ pair_a, const int* __restrict__ pair_b,
                const double* __restrict__ F, const double* __restrict__ E, const double* __restrict__ H,
                double* __restrict__ S) {
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
    for (int q = blk_pair_ptr[blk]; q < blk_pair_ptr[blk + 1]; ++q) {
      int64_t oa = pair_a[q], ob = pair_b[q];
      const double* fa = F + oa * 18;
      const double* ha = H + oa * 6;
      const double* eb = E + ob * 6;
      const double* fb = F + ob * 18;
      double g00 = ha[0] * eb[0] + ha[1] * eb[1] + ha[2] * eb[2];
      double g01 = ha[0] * eb[3] + ha[1] * eb[4] + ha[2] * eb[5];
      double g10 = ha[3] * eb[0] + ha[4] * eb[1] + ha[5] * eb[2];
      double g11 = ha[3] * eb[3] + ha[4] * eb[4] + ha[5] * eb[5];
      double b0[3], b1[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        b0[c] = fb[c0 + c];
        b1[c] = fb[9 + c0 + c];
      }
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

extern "C" int bamg_schur_numeric(bamg_ctx* ctx, const int32_t* cam_ptr, const int32_t* cm_list,
                                  const double* F, const double* E, const double* H, const double* A,
                                  const int32_t* dpos, int32_t nc, const int32_t* up_blk, const int32_t* up_tpos,
                                  int32_t n_up, const int32_t* blk_pair_ptr, const int32_t* pair_a,
                                  const int32_t* pair_b, double* S, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (nc)
    k_schur_diag<<<grid_for((int64_t)nc * 32, 128, 8), 128, 0, st>>>(cam_ptr, cm_list, F, E, H, A, dpos, nc, S);
  if (n_up) {
    int64_t warps = ceil_div(n_up, OFF_GROUPS);
    k_schur_offdiag<<<grid_for(warps * 32, 128, 8), 128, 0, st>>>(up_blk, up_tpos, n_up, blk_pair_ptr, pair_a,
                                                                  pair_b, F, E, H, S);
  }
  BAMG_LAUNCH_CHECK();
  return 0;
}
