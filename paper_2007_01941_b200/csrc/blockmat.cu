// Generic block-sparse API kernels (blockmat.py:152-360): validation, triplet
// assembly with duplicate summation, rectangular / transposed products, block-column
// scaling and the sparse block product. These serve the drop-in API (W, P^T, user
// matrices); the measured path uses the dedicated Schur / Galerkin / V-cycle kernels.
//
// Summation orders follow the reference's third-party kernels so results are
// bit-identical, with every product and sum rounded separately (__dmul_rn /
// __dadd_rn, no FMA contraction):
//   * from_triplets: np.lexsort((cols, rows)) is stable -> duplicates in input
//     order; np.add.reduceat along axis 0 is the first block plus numpy's pairwise
//     sum of the rest (measured against numpy 2.3, tests/test_gpu_blockmat.py);
//   * matvec: scipy bsr_matvec / gemv -- y_r starts at 0, then blocks of the row
//     in column order, inside a block columns in order;
//   * multiply: scipy csr_matmat -- output scalar (r, c) accumulates A[r, k] B[k, c]
//     in ascending scalar k (blocks ascending, then the in-block index); a scalar
//     whose sum is exactly 0 is not stored and a block with no stored scalar is
//     dropped (the re-blocked result keeps blocks with any nonzero, zeros as +0).
#include "common.cuh"
#include "ctx.h"

int radix_sort_pairs(const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout, int64_t n,
                     int key_bits, cudaStream_t st);
int scan_exclusive_int(const int* in, int* out, int64_t n, int* total, cudaStream_t st);
int segment_ptr(const int* ids, int64_t n, int nseg, int* ptr, cudaStream_t st);

static int bits_for(int64_t n) {
  int b = 1;
  while ((1ll << b) < n) ++b;
  return b;
}

// ---------------------------------------------------------------------------
// validation (blockmat.py:174-191)

__global__ void k_bsr_validate(const int* __restrict__ ptr, int nbr, const int* __restrict__ col, int64_t nnz, int nbc,
                               int* __restrict__ flags) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nbr; i += stride)
    if (ptr[i + 1] < ptr[i]) flags[0] = 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += stride)
    if (col[i] < 0 || col[i] >= nbc) flags[1] = 1;
}

extern "C" int bamg_bsr_validate(bamg_ctx* ctx, const int32_t* ptr, int32_t nbr, const int32_t* col, int64_t nnz,
                                 int32_t nbc, int32_t* flags_dev, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  BAMG_CUDA_CHECK(cudaMemsetAsync(flags_dev, 0, 2 * sizeof(int32_t), st));
  int64_t n = nbr > nnz ? nbr : nnz;
  if (n > 0) launch(k_bsr_validate, grid_for(n, 256), 256, 0, st, ptr, nbr, col, nnz, nbc, flags_dev);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------------------
// from_triplets (blockmat.py:195-230)

__global__ void k_trip_keys(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols, int64_t n, int nbr,
                            int nbc, uint32_t* __restrict__ key, uint32_t* __restrict__ iota, int* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = rows[i], c = cols[i];
    if (r < 0 || r >= nbr || c < 0 || c >= nbc) *bad = 1;
    key[i] = (uint32_t)(c < 0 ? 0 : (c >= nbc ? 0 : c));
    iota[i] = (uint32_t)i;
  }
}

__global__ void k_trip_rowkeys(const int64_t* __restrict__ rows, const uint32_t* __restrict__ perm, int64_t n, int nbr,
                               uint32_t* __restrict__ key) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = rows[perm[i]];
    key[i] = (uint32_t)(r < 0 ? 0 : (r >= nbr ? 0 : r));
  }
}

// new[i] = 1 when sorted entry i starts a distinct (row, col)
__global__ void k_trip_heads(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols,
                             const uint32_t* __restrict__ perm, int64_t n, int* __restrict__ head) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t p = perm[i];
    int h = 1;
    if (i > 0) {
      uint32_t q = perm[i - 1];
      h = (rows[p] != rows[q]) || (cols[p] != cols[q]);
    }
    head[i] = h;
  }
}

extern "C" int bamg_triplets_order(bamg_ctx* ctx, const int64_t* rows, const int64_t* cols, int64_t n, int32_t nbr,
                                   int32_t nbc, int32_t* perm, int32_t* seg, int32_t* count_dev, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  BAMG_CUDA_CHECK(cudaMemsetAsync(count_dev, 0, 2 * sizeof(int32_t), st));
  if (n <= 0) return 0;
  uint32_t *k1 = nullptr, *v1 = nullptr, *ks = nullptr, *p1 = nullptr;
  BAMG_CUDA_CHECK(cudaMallocAsync(&k1, 4 * n, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&v1, 4 * n, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&ks, 4 * n, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&p1, 4 * n, st));
  int g = grid_for(n, 256);
  launch(k_trip_keys, g, 256, 0, st, rows, cols, n, nbr, nbc, k1, v1, count_dev + 1);
  // LSD lexsort: stable by column, then stable by row
  int rc = radix_sort_pairs(k1, v1, ks, p1, n, bits_for(nbc), st);
  if (rc) return rc;
  launch(k_trip_rowkeys, g, 256, 0, st, rows, p1, n, nbr, k1);
  rc = radix_sort_pairs(k1, p1, ks, (uint32_t*)perm, n, bits_for(nbr), st);
  if (rc) return rc;
  launch(k_trip_heads, g, 256, 0, st, rows, cols, (const uint32_t*)perm, n, seg);
  rc = scan_exclusive_int(seg, seg, n, count_dev, st);  // seg[i] = heads before i
  if (rc) return rc;
  BAMG_LAUNCH_CHECK();
  cudaFreeAsync(k1, st);
  cudaFreeAsync(v1, st);
  cudaFreeAsync(ks, st);
  cudaFreeAsync(p1, st);
  return 0;
}

// start[u] = first sorted position of unique entry u (seg = exclusive head count)
__global__ void k_trip_starts(const int* __restrict__ seg, int64_t n, int nu, int* __restrict__ start) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int s = seg[i];
    int nxt = (i + 1 < n) ? seg[i + 1] : nu;
    if (nxt != s) start[s] = (int)i;  // position i is the head of unique entry s
    if (i == n - 1) start[nu] = (int)n;
  }
}

// numpy's pairwise_sum (the add reduction's inner loop over a strided axis): below 8
// terms a running sum from +0; up to 128 eight interleaved partial sums combined as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus the tail; beyond, split at a multiple of 8
__device__ double np_pairwise(const double* __restrict__ blocks, const uint32_t* __restrict__ perm, int s, int n,
                              int bsz, int e) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, blocks[(int64_t)perm[s + i] * bsz + e]);
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = blocks[(int64_t)perm[s + j] * bsz + e];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], blocks[(int64_t)perm[s + i + j] * bsz + e]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, blocks[(int64_t)perm[s + i] * bsz + e]);
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise(blocks, perm, s, n2, bsz, e), np_pairwise(blocks, perm, s + n2, n - n2, bsz, e));
}

// np.add.reduceat along axis 0: the segment's first block, plus numpy's pairwise sum
// of the remaining ones (the strided reduction loop)
__global__ void k_trip_sum(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols,
                           const double* __restrict__ blocks, int bsz, const uint32_t* __restrict__ perm,
                           const int* __restrict__ start, int64_t nu, int* __restrict__ urow, int* __restrict__ ucol,
                           double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nu * bsz; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t u = t / bsz;
    int e = (int)(t - u * bsz);
    int s0 = start[u], s1 = start[u + 1];
    uint32_t p = perm[s0];
    double acc = blocks[(int64_t)p * bsz + e];
    if (s1 - s0 > 1) acc = __dadd_rn(acc, np_pairwise(blocks, perm, s0 + 1, s1 - s0 - 1, bsz, e));
    out[t] = acc;
    if (e == 0) {
      urow[u] = (int)rows[p];
      ucol[u] = (int)cols[p];
    }
  }
}

extern "C" int bamg_triplets_reduce(bamg_ctx* ctx, const int64_t* rows, const int64_t* cols, const double* blocks,
                                    int64_t n, int32_t bsz, const int32_t* perm, const int32_t* seg, int64_t nu,
                                    int32_t nbr, int32_t* ptr, int32_t* col_out, double* blocks_out, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (nu <= 0 || n <= 0) {
    BAMG_CUDA_CHECK(cudaMemsetAsync(ptr, 0, sizeof(int32_t) * (nbr + 1), st));
    return 0;
  }
  int *start = nullptr, *urow = nullptr;
  BAMG_CUDA_CHECK(cudaMallocAsync(&start, 4 * (nu + 1), st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&urow, 4 * nu, st));
  launch(k_trip_starts, grid_for(n, 256), 256, 0, st, seg, n, (int)nu, start);
  launch(k_trip_sum, grid_for(nu * bsz, 256), 256, 0, st, rows, cols, blocks, bsz, (const uint32_t*)perm,
         (const int*)start, nu, urow, col_out, blocks_out);
  int rc = segment_ptr(urow, nu, nbr, ptr, st);
  if (rc) return rc;
  BAMG_LAUNCH_CHECK();
  cudaFreeAsync(start, st);
  cudaFreeAsync(urow, st);
  return 0;
}

// ---------------------------------------------------------------------------
// y = M x for any block shape (scipy bsr_matvec order, blockmat.py:295-299)

__global__ void k_bsr_matvec_gen(int rbs, int cbs, const int* __restrict__ ptr, const int* __restrict__ col,
                                 const double* __restrict__ blocks, const double* __restrict__ x, int nbr,
                                 double* __restrict__ y) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)nbr * rbs;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / rbs;
    int r = (int)(t - i * rbs);
    double acc = 0.0;
    for (int q = ptr[i]; q < ptr[i + 1]; ++q) {
      const double* a = blocks + ((int64_t)q * rbs + r) * cbs;
      const double* xb = x + (int64_t)col[q] * cbs;
      for (int c = 0; c < cbs; ++c) acc = __dadd_rn(acc, __dmul_rn(a[c], xb[c]));
    }
    y[t] = acc;
  }
}

extern "C" int bamg_bsr_matvec_gen(bamg_ctx* ctx, int32_t rbs, int32_t cbs, const int32_t* ptr, const int32_t* col,
                                   const double* blocks, const double* x, int32_t nbr, double* y, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if ((int64_t)nbr * rbs > 0)
    launch(k_bsr_matvec_gen, grid_for((int64_t)nbr * rbs, 256), 256, 0, st, rbs, cbs, ptr, col, blocks, x, nbr, y);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------------------
// blockmat.py:321-334 scale_block_columns: out_n = blocks_n @ cb[col_n]  (rbs x cbs @ cbs x k)

__global__ void k_scale_cols(const double* __restrict__ blocks, const double* __restrict__ cb, const int* __restrict__ col,
                             int64_t nnz, int rbs, int cbs, int kk, double* __restrict__ out) {
  int64_t per = (int64_t)rbs * kk;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nnz * per; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t n = t / per;
    int e = (int)(t - n * per);
    int r = e / kk, c = e - r * kk;
    const double* a = blocks + (n * rbs + r) * cbs;
    const double* b = cb + (int64_t)col[n] * cbs * kk + c;
    double acc = 0.0;
    for (int j = 0; j < cbs; ++j) acc = __dadd_rn(acc, __dmul_rn(a[j], b[(int64_t)j * kk]));
    out[t] = acc;
  }
}

extern "C" int bamg_bsr_scale_cols(bamg_ctx* ctx, const double* blocks, const double* col_blocks, const int32_t* col,
                                   int64_t nnz, int32_t rbs, int32_t cbs, int32_t k, double* out, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (nnz * rbs * k > 0)
    launch(k_scale_cols, grid_for(nnz * rbs * k, 256), 256, 0, st, blocks, col_blocks, col, nnz, rbs, cbs, k, out);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------------------
// multiply (blockmat.py:337-353): block SpGEMM in csr_matmat order with its zero-drop.
//   create : candidate products (i, j, A block q, B block t) in emission order
//            (row i, then A's blocks ascending k, then B's row k ascending j), stably
//            sorted by (i, j) -- so each output block's candidates stay in ascending k;
//            *nu_host = distinct (i, j)
//   numeric: per distinct (i, j) the sums, keep flag = any scalar != 0;
//            *nkeep_host = kept blocks
//   finish : the kept blocks as CSR (exact zeros inside kept blocks stored as +0)

__global__ void k_spgemm_rowcount(const int* __restrict__ a_col, int64_t a_nnz, const int* __restrict__ b_ptr,
                                  int* __restrict__ cnt) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < a_nnz; q += (int64_t)gridDim.x * blockDim.x) {
    int k = a_col[q];
    cnt[q] = b_ptr[k + 1] - b_ptr[k];
  }
}

__global__ void k_spgemm_emit(const int* __restrict__ a_ptr, const int* __restrict__ a_col, int a_nbr,
                              const int* __restrict__ b_ptr, const int* __restrict__ b_col, const int* __restrict__ off,
                              uint32_t* __restrict__ jkey, uint32_t* __restrict__ cand_a, uint32_t* __restrict__ cand_b,
                              uint32_t* __restrict__ row_of, uint32_t* __restrict__ iota) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a_nbr; i += gridDim.x * blockDim.x) {
    for (int q = a_ptr[i]; q < a_ptr[i + 1]; ++q) {
      int k = a_col[q];
      int o = off[q];
      for (int t = b_ptr[k]; t < b_ptr[k + 1]; ++t, ++o) {
        jkey[o] = (uint32_t)b_col[t];
        cand_a[o] = (uint32_t)q;
        cand_b[o] = (uint32_t)t;
        row_of[o] = (uint32_t)i;
        iota[o] = (uint32_t)o;
      }
    }
  }
}

__global__ void k_gather_u32(const uint32_t* __restrict__ src, const uint32_t* __restrict__ idx, int64_t n,
                             uint32_t* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

__global__ void k_spgemm_heads(const uint32_t* __restrict__ row_of, const uint32_t* __restrict__ jkey,
                               const uint32_t* __restrict__ perm, int64_t n, int* __restrict__ head) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t p = perm[i];
    int h = 1;
    if (i > 0) {
      uint32_t q = perm[i - 1];
      h = (row_of[p] != row_of[q]) || (jkey[p] != jkey[q]);
    }
    head[i] = h;
  }
}

__global__ void k_spgemm_sum(const uint32_t* __restrict__ perm, const int* __restrict__ start,
                             const uint32_t* __restrict__ cand_a, const uint32_t* __restrict__ cand_b,
                             const uint32_t* __restrict__ row_of, const uint32_t* __restrict__ jkey,
                             const double* __restrict__ A, const double* __restrict__ B, int rbs, int kbs, int cbs,
                             int64_t nu, double* __restrict__ out, int* __restrict__ urow, int* __restrict__ ucol) {
  int64_t per = (int64_t)rbs * cbs;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nu * per; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t u = t / per;
    int e = (int)(t - u * per);
    int r = e / cbs, c = e - r * cbs;
    double acc = 0.0;
    for (int s = start[u]; s < start[u + 1]; ++s) {
      uint32_t p = perm[s];
      const double* a = A + ((int64_t)cand_a[p] * rbs + r) * kbs;
      const double* b = B + (int64_t)cand_b[p] * kbs * cbs + c;
      for (int kk = 0; kk < kbs; ++kk) acc = __dadd_rn(acc, __dmul_rn(a[kk], b[(int64_t)kk * cbs]));
    }
    out[t] = acc;
    if (e == 0) {
      uint32_t p = perm[start[u]];
      urow[u] = (int)row_of[p];
      ucol[u] = (int)jkey[p];
    }
  }
}

__global__ void k_spgemm_keep(const double* __restrict__ vals, int64_t nu, int per, int* __restrict__ keep) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < nu; u += (int64_t)gridDim.x * blockDim.x) {
    int k = 0;
    for (int e = 0; e < per && !k; ++e) k = vals[u * per + e] != 0.0;
    keep[u] = k;
  }
}

__global__ void k_spgemm_compact(const double* __restrict__ vals, const int* __restrict__ urow,
                                 const int* __restrict__ ucol, const int* __restrict__ keep_pos, int64_t nu, int per,
                                 double* __restrict__ out, int* __restrict__ krow, int* __restrict__ kcol) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nu * per; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t u = t / per;
    int e = (int)(t - u * per);
    int pos = keep_pos[u];
    if (keep_pos[u + 1] == pos) continue;  // dropped: every scalar summed to 0
    double v = vals[t];
    out[(int64_t)pos * per + e] = v == 0.0 ? 0.0 : v;
    if (e == 0) {
      krow[pos] = urow[u];
      kcol[pos] = ucol[u];
    }
  }
}

struct bamg_spgemm {
  int64_t n = 0, nu = 0, nkeep = 0;
  int a_nbr = 0, rbs = 0, cbs = 0;
  uint32_t *jkey = nullptr, *ca = nullptr, *cb = nullptr, *row = nullptr, *perm = nullptr;
  int *start = nullptr, *urow = nullptr, *ucol = nullptr, *keep = nullptr;
  double* vals = nullptr;
  ~bamg_spgemm() {
    for (void* p : {(void*)jkey, (void*)ca, (void*)cb, (void*)row, (void*)perm, (void*)start, (void*)urow,
                    (void*)ucol, (void*)keep, (void*)vals})
      if (p) cudaFree(p);
  }
};

extern "C" bamg_spgemm* bamg_spgemm_create(bamg_ctx* ctx, const int32_t* a_ptr, const int32_t* a_col, int32_t a_nbr,
                                           int64_t a_nnz, const int32_t* b_ptr, const int32_t* b_col, int32_t b_nbc,
                                           int64_t* nu_host, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  auto* sp = new bamg_spgemm();
  sp->a_nbr = a_nbr;
  *nu_host = 0;
  auto fail = [&](cudaError_t e) -> bamg_spgemm* {
    bamg_set_error("spgemm: %s", cudaGetErrorString(e));
    delete sp;
    return nullptr;
  };
  cudaError_t e;
  if (a_nnz == 0) return sp;
  int *off = nullptr, *tot = nullptr;
  if ((e = cudaMalloc(&off, 4 * a_nnz)) || (e = cudaMalloc(&tot, 4))) return fail(e);
  launch(k_spgemm_rowcount, grid_for(a_nnz, 256), 256, 0, st, a_col, a_nnz, b_ptr, off);
  if (scan_exclusive_int(off, off, a_nnz, tot, st)) return fail(cudaErrorUnknown);
  int h = 0;
  if ((e = cudaMemcpyAsync(&h, tot, 4, cudaMemcpyDeviceToHost, st)) || (e = cudaStreamSynchronize(st))) return fail(e);
  int64_t n = h;
  sp->n = n;
  if (n > 0) {
    uint32_t *iota = nullptr, *ks = nullptr, *p1 = nullptr, *k2 = nullptr;
    int* head = nullptr;
    if ((e = cudaMalloc(&sp->jkey, 4 * n)) || (e = cudaMalloc(&sp->ca, 4 * n)) || (e = cudaMalloc(&sp->cb, 4 * n)) ||
        (e = cudaMalloc(&sp->row, 4 * n)) || (e = cudaMalloc(&sp->perm, 4 * n)) || (e = cudaMalloc(&iota, 4 * n)) ||
        (e = cudaMalloc(&ks, 4 * n)) || (e = cudaMalloc(&p1, 4 * n)) || (e = cudaMalloc(&k2, 4 * n)) ||
        (e = cudaMalloc(&head, 4 * n)) || (e = cudaMalloc(&sp->start, 4 * (n + 1))))
      return fail(e);
    int g = grid_for(n, 256);
    launch(k_spgemm_emit, grid_for(a_nbr, 128), 128, 0, st, a_ptr, a_col, a_nbr, b_ptr, b_col, (const int*)off,
           sp->jkey, sp->ca, sp->cb, sp->row, iota);
    // LSD: stable by column j, then stable by row i
    if (radix_sort_pairs(sp->jkey, iota, ks, p1, n, bits_for(b_nbc), st)) return fail(cudaErrorUnknown);
    launch(k_gather_u32, g, 256, 0, st, (const uint32_t*)sp->row, (const uint32_t*)p1, n, k2);
    if (radix_sort_pairs(k2, p1, ks, sp->perm, n, bits_for(a_nbr), st)) return fail(cudaErrorUnknown);
    launch(k_spgemm_heads, g, 256, 0, st, (const uint32_t*)sp->row, (const uint32_t*)sp->jkey,
           (const uint32_t*)sp->perm, n, head);
    if (scan_exclusive_int(head, head, n, tot, st)) return fail(cudaErrorUnknown);
    if ((e = cudaMemcpyAsync(&h, tot, 4, cudaMemcpyDeviceToHost, st)) || (e = cudaStreamSynchronize(st))) return fail(e);
    sp->nu = h;
    launch(k_trip_starts, g, 256, 0, st, (const int*)head, n, (int)sp->nu, sp->start);
    if ((e = cudaStreamSynchronize(st))) return fail(e);
    cudaFree(iota);
    cudaFree(ks);
    cudaFree(p1);
    cudaFree(k2);
    cudaFree(head);
  }
  cudaFree(off);
  cudaFree(tot);
  if ((e = cudaGetLastError())) return fail(e);
  *nu_host = sp->nu;
  return sp;
}

extern "C" int bamg_spgemm_numeric(bamg_ctx* ctx, bamg_spgemm* sp, const double* a_blocks, int32_t rbs, int32_t kbs,
                                   const double* b_blocks, int32_t cbs, int64_t* nkeep_host, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  sp->rbs = rbs;
  sp->cbs = cbs;
  *nkeep_host = 0;
  int64_t nu = sp->nu, per = (int64_t)rbs * cbs;
  if (nu == 0) return 0;
  BAMG_CUDA_CHECK(cudaMalloc(&sp->vals, 8 * nu * per));
  BAMG_CUDA_CHECK(cudaMalloc(&sp->urow, 4 * nu));
  BAMG_CUDA_CHECK(cudaMalloc(&sp->ucol, 4 * nu));
  BAMG_CUDA_CHECK(cudaMalloc(&sp->keep, 4 * (nu + 1)));
  launch(k_spgemm_sum, grid_for(nu * per, 256), 256, 0, st, (const uint32_t*)sp->perm, (const int*)sp->start,
         (const uint32_t*)sp->ca, (const uint32_t*)sp->cb, (const uint32_t*)sp->row, (const uint32_t*)sp->jkey,
         a_blocks, b_blocks, rbs, kbs, cbs, nu, sp->vals, sp->urow, sp->ucol);
  launch(k_spgemm_keep, grid_for(nu, 256), 256, 0, st, (const double*)sp->vals, nu, (int)per, sp->keep);
  int rc = scan_exclusive_int(sp->keep, sp->keep, nu + 1, nullptr, st);
  if (rc) return rc;
  int h = 0;
  BAMG_CUDA_CHECK(cudaMemcpyAsync(&h, sp->keep + nu, 4, cudaMemcpyDeviceToHost, st));
  BAMG_CUDA_CHECK(cudaStreamSynchronize(st));
  sp->nkeep = h;
  *nkeep_host = h;
  BAMG_LAUNCH_CHECK();
  return 0;
}

extern "C" int bamg_spgemm_finish(bamg_ctx* ctx, bamg_spgemm* sp, int32_t* ptr, int32_t* col, double* blocks,
                                  void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (sp->nkeep == 0) {
    BAMG_CUDA_CHECK(cudaMemsetAsync(ptr, 0, sizeof(int32_t) * (sp->a_nbr + 1), st));
    return 0;
  }
  int per = sp->rbs * sp->cbs;
  int* krow = nullptr;
  BAMG_CUDA_CHECK(cudaMallocAsync(&krow, 4 * sp->nkeep, st));
  launch(k_spgemm_compact, grid_for(sp->nu * per, 256), 256, 0, st, (const double*)sp->vals, (const int*)sp->urow,
         (const int*)sp->ucol, (const int*)sp->keep, sp->nu, per, blocks, krow, col);
  int rc = segment_ptr(krow, sp->nkeep, sp->a_nbr, ptr, st);
  if (rc) return rc;
  BAMG_LAUNCH_CHECK();
  cudaFreeAsync(krow, st);
  return 0;
}

extern "C" void bamg_spgemm_destroy(bamg_spgemm* sp) { delete sp; }
