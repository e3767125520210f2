// Block-sparse kernels for the solve phase: BSR SpMV (9x9 / 16x16, fused dot),
// fused Chebyshev smoother steps, residual, prolongation / restriction, batched
// block Cholesky + explicit inverse, block-diagonal apply, dense coarse factor.
//
// SpMV mapping: one warp per block row; BS lanes own the BS rows of a block and
// 32/BS lane groups walk the row's blocks in an interleaved order; each lane streams
// its 72 B (BS=9) / 128 B (BS=16) block row through L1 with the x sub-vector
// broadcast, and the groups are combined with a fixed shuffle tree (deterministic).
#include "common.cuh"
#include "ctx.h"

#include <mutex>

template <int BS>
struct Lanes {
  static constexpr int G = 32 / BS;  // lane groups per warp
  static constexpr int USED = G * BS;
};

// Per-warp row product: returns (A x)_r in lanes with lane < BS (r = lane).
template <int BS>
__device__ __forceinline__ double warp_row_product(const int* __restrict__ ptr, const int* __restrict__ col,
                                                   const double* __restrict__ blocks, const double* __restrict__ x,
                                                   int row, int lane) {
  constexpr int G = Lanes<BS>::G;
  int g = lane / BS, r = lane - g * BS;
  double acc = 0.0;
  if (g < G) {
    int b0 = ptr[row], b1 = ptr[row + 1];
    for (int b = b0 + g; b < b1; b += G) {
      const double* a = blocks + (int64_t)b * (BS * BS) + r * BS;
      const double* xv = x + (int64_t)col[b] * BS;
#pragma unroll
      for (int c = 0; c < BS; ++c) acc = fma(__ldg(a + c), __ldg(xv + c), acc);
    }
  }
  // combine groups: lane r += lane r + BS*k
#pragma unroll
  for (int k = 1; k < G; ++k) {
    double t = __shfl_down_sync(FULL_MASK, acc, k * BS);
    if (lane < BS) acc += t;
  }
  return acc;
}

// 16x16 blocks (2 KB, 16 B aligned): the warp streams each block as 4 fully
// coalesced 512 B double2 sweeps. Lane l holds column pair 2(l%8) of rows
// {l/8, 4+l/8, 8+l/8, 12+l/8}; the row sums are reduced over the 8-lane groups
// once per block row, then moved to lane r = row.
template <>
__device__ __forceinline__ double warp_row_product<16>(const int* __restrict__ ptr, const int* __restrict__ col,
                                                       const double* __restrict__ blocks,
                                                       const double* __restrict__ x, int row, int lane) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int b0 = ptr[row], b1 = ptr[row + 1];
  const int cp = 2 * (lane & 7);
  int b = b0;
  for (; b + 1 < b1; b += 2) {  // two blocks in flight
    const double2* A0 = reinterpret_cast<const double2*>(blocks + (int64_t)b * 256) + lane;
    const double2* A1 = reinterpret_cast<const double2*>(blocks + (int64_t)(b + 1) * 256) + lane;
    double2 u0 = __ldg(A0), u1 = __ldg(A0 + 32), u2 = __ldg(A0 + 64), u3 = __ldg(A0 + 96);
    double2 v0 = __ldg(A1), v1 = __ldg(A1 + 32), v2 = __ldg(A1 + 64), v3 = __ldg(A1 + 96);
    double2 xa = __ldg(reinterpret_cast<const double2*>(x + (int64_t)col[b] * 16 + cp));
    double2 xb = __ldg(reinterpret_cast<const double2*>(x + (int64_t)col[b + 1] * 16 + cp));
    a0 = fma(u0.x, xa.x, fma(u0.y, xa.y, a0));
    a1 = fma(u1.x, xa.x, fma(u1.y, xa.y, a1));
    a2 = fma(u2.x, xa.x, fma(u2.y, xa.y, a2));
    a3 = fma(u3.x, xa.x, fma(u3.y, xa.y, a3));
    a0 = fma(v0.x, xb.x, fma(v0.y, xb.y, a0));
    a1 = fma(v1.x, xb.x, fma(v1.y, xb.y, a1));
    a2 = fma(v2.x, xb.x, fma(v2.y, xb.y, a2));
    a3 = fma(v3.x, xb.x, fma(v3.y, xb.y, a3));
  }
  if (b < b1) {
    const double2* A0 = reinterpret_cast<const double2*>(blocks + (int64_t)b * 256) + lane;
    double2 u0 = __ldg(A0), u1 = __ldg(A0 + 32), u2 = __ldg(A0 + 64), u3 = __ldg(A0 + 96);
    double2 xa = __ldg(reinterpret_cast<const double2*>(x + (int64_t)col[b] * 16 + cp));
    a0 = fma(u0.x, xa.x, fma(u0.y, xa.y, a0));
    a1 = fma(u1.x, xa.x, fma(u1.y, xa.y, a1));
    a2 = fma(u2.x, xa.x, fma(u2.y, xa.y, a2));
    a3 = fma(u3.x, xa.x, fma(u3.y, xa.y, a3));
  }
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) {
    a0 += __shfl_xor_sync(FULL_MASK, a0, o);
    a1 += __shfl_xor_sync(FULL_MASK, a1, o);
    a2 += __shfl_xor_sync(FULL_MASK, a2, o);
    a3 += __shfl_xor_sync(FULL_MASK, a3, o);
  }
  // row r = 4k + j lives in accumulator k of lanes 8j..8j+7
  int src = 8 * (lane & 3);
  double s0 = __shfl_sync(FULL_MASK, a0, src);
  double s1 = __shfl_sync(FULL_MASK, a1, src);
  double s2 = __shfl_sync(FULL_MASK, a2, src);
  double s3 = __shfl_sync(FULL_MASK, a3, src);
  int k = (lane >> 2) & 3;
  return k == 0 ? s0 : (k == 1 ? s1 : (k == 2 ? s2 : s3));
}

// y = A x ; optionally dot_out = <x, y> (deterministic, grid_finish).
template <int BS>
__global__ void __launch_bounds__(128)
k_bsr_spmv(const int* __restrict__ ptr, const int* __restrict__ col, const double* __restrict__ blocks,
           const double* __restrict__ x, double* __restrict__ y, int nbr, double* partials, unsigned int* counter,
           double* dot_out) {
  PDL_ENTRY();
  __shared__ double scratch[33];
  int lane = threadIdx.x & 31;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  double dsum = 0.0;
  for (int row = warp; row < nbr; row += nwarps) {
    double v = warp_row_product<BS>(ptr, col, blocks, x, row, lane);
    if (lane < BS) {
      y[(int64_t)row * BS + lane] = v;
      if (dot_out) dsum = fma(x[(int64_t)row * BS + lane], v, dsum);
    }
  }
  if (dot_out) {
    dsum = block_sum(dsum, scratch);
    grid_finish(partials, counter, dsum, scratch, dot_out);
  }
}

// rows x: r = b - A x
template <int BS>
__global__ void __launch_bounds__(128)
k_bsr_residual(const int* __restrict__ ptr, const int* __restrict__ col, const double* __restrict__ blocks,
               const double* __restrict__ x, const double* __restrict__ b, double* __restrict__ r, int nbr) {
  PDL_ENTRY();
  int lane = threadIdx.x & 31;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int row = warp; row < nbr; row += nwarps) {
    double v = warp_row_product<BS>(ptr, col, blocks, x, row, lane);
    if (lane < BS) r[(int64_t)row * BS + lane] = b[(int64_t)row * BS + lane] - v;
  }
}

// Chebyshev step (multigrid.py:308-328), fused with the SpMV and the Jacobi apply:
//   r = b - A x_in   (A == null: r = b)
//   z = D^-1 r
//   divide: d = z / c2          else: d = c1 d + c2 z
//   x_out = x_in + d            (x_in == null: x_out = d)
// x_out must not alias x_in (other rows read x_in).
template <int BS>
__global__ void __launch_bounds__(128)
k_cheb_step(const int* __restrict__ ptr, const int* __restrict__ col, const double* __restrict__ blocks,
            const double* __restrict__ x_in, const double* __restrict__ b, const double* __restrict__ Dinv,
            double* __restrict__ d, double* __restrict__ x_out, int nbr, double c1, double c2, int divide) {
  PDL_ENTRY();
  int lane = threadIdx.x & 31;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int row = warp; row < nbr; row += nwarps) {
    double ax = 0.0;
    if (blocks && x_in) ax = warp_row_product<BS>(ptr, col, blocks, x_in, row, lane);
    int64_t base = (int64_t)row * BS;
    double rr = (lane < BS) ? b[base + lane] - ax : 0.0;
    // z_r = sum_c Dinv[r][c] r_c  (r_c broadcast from lane c)
    double z = 0.0;
    const double* Di = Dinv + (int64_t)row * BS * BS + (lane < BS ? lane : 0) * BS;
#pragma unroll
    for (int c = 0; c < BS; ++c) {
      double rc = __shfl_sync(FULL_MASK, rr, c);
      if (lane < BS) z = fma(Di[c], rc, z);
    }
    if (lane < BS) {
      double dn = divide ? z / c2 : c1 * d[base + lane] + c2 * z;
      d[base + lane] = dn;
      x_out[base + lane] = (x_in ? x_in[base + lane] : 0.0) + dn;
    }
  }
}

static int spmv_grid(int nbr) { return grid_for((int64_t)nbr * 32, 128, 16); }

extern "C" int bamg_bsr_spmv(bamg_ctx* ctx, int32_t bs, const int32_t* ptr, const int32_t* col,
                             const double* blocks, const double* x, double* y, int32_t nbr, double* dot_out_dev,
                             void* stream) {
  cudaStream_t st = as_stream(stream);
  if (nbr <= 0) return 0;
  double* part = ctx ? ctx->partials : nullptr;
  unsigned* ctr = ctx ? ctx->counters + BAMG_CTR_SPMV : nullptr;
  int g = spmv_grid(nbr);
  if (dot_out_dev && g > BAMG_MAX_PARTIALS) g = BAMG_MAX_PARTIALS;
  switch (bs) {
    case 9: launch(k_bsr_spmv<9>, g, 128, 0, st, ptr, col, blocks, x, y, nbr, part, ctr, dot_out_dev); break;
    case 16: launch(k_bsr_spmv<16>, g, 128, 0, st, ptr, col, blocks, x, y, nbr, part, ctr, dot_out_dev); break;
    case 3: launch(k_bsr_spmv<3>, g, 128, 0, st, ptr, col, blocks, x, y, nbr, part, ctr, dot_out_dev); break;
    case 1: launch(k_bsr_spmv<1>, g, 128, 0, st, ptr, col, blocks, x, y, nbr, part, ctr, dot_out_dev); break;
    default: bamg_set_error("bsr_spmv: unsupported square block size %d", bs); return BAMG_ERR_UNSUPPORTED;
  }
  BAMG_LAUNCH_CHECK();
  return 0;
}

extern "C" int bamg_bsr_residual(bamg_ctx* ctx, int32_t bs, const int32_t* ptr, const int32_t* col,
                                 const double* blocks, const double* x, const double* b, double* r, int32_t nbr,
                                 void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (nbr <= 0) return 0;
  int g = spmv_grid(nbr);
  switch (bs) {
    case 9: launch(k_bsr_residual<9>, g, 128, 0, st, ptr, col, blocks, x, b, r, nbr); break;
    case 16: launch(k_bsr_residual<16>, g, 128, 0, st, ptr, col, blocks, x, b, r, nbr); break;
    case 1: launch(k_bsr_residual<1>, g, 128, 0, st, ptr, col, blocks, x, b, r, nbr); break;
    default: bamg_set_error("bsr_residual: unsupported block size %d", bs); return BAMG_ERR_UNSUPPORTED;
  }
  BAMG_LAUNCH_CHECK();
  return 0;
}

extern "C" int bamg_cheb_step(bamg_ctx* ctx, int32_t bs, const int32_t* ptr, const int32_t* col,
                              const double* blocks, const double* x_in, const double* b, const double* Dinv, double* d,
                              double* x_out, int32_t nbr, double c1, double c2, int32_t divide, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (nbr <= 0) return 0;
  int g = spmv_grid(nbr);
  switch (bs) {
    case 9: launch(k_cheb_step<9>, g, 128, 0, st, ptr, col, blocks, x_in, b, Dinv, d, x_out, nbr, c1, c2, divide); break;
    case 16: launch(k_cheb_step<16>, g, 128, 0, st, ptr, col, blocks, x_in, b, Dinv, d, x_out, nbr, c1, c2, divide); break;
    case 1: launch(k_cheb_step<1>, g, 128, 0, st, ptr, col, blocks, x_in, b, Dinv, d, x_out, nbr, c1, c2, divide); break;
    default: bamg_set_error("cheb_step: unsupported block size %d", bs); return BAMG_ERR_UNSUPPORTED;
  }
  BAMG_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------------------
// prolongation / restriction with the tentative prolongator: one bs x 16 block per
// fine node, block column = aggregate (multigrid.py:234-236).

// y_i (+)= P_i xc_agg(i)
// (min-blocks 1 lets ptxas issue the row's eight 16 B loads of P and of xc before
// the fma chain instead of interleaving them at 32 registers)
__global__ void __launch_bounds__(256, 1)
k_prolong(const int* __restrict__ agg, const double* __restrict__ P, const double* __restrict__ xc, int nf, int bs,
          double* __restrict__ y, int accumulate) {
  PDL_ENTRY();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)nf * bs; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / bs;
    int r = (int)(t - i * bs);
    const double2* p = reinterpret_cast<const double2*>(P + (i * bs + r) * 16);
    const double2* xa = reinterpret_cast<const double2*>(xc + (int64_t)__ldg(agg + i) * 16);
    double2 pv[8], xv[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      pv[c] = __ldg(p + c);
      xv[c] = __ldg(xa + c);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s = fma(pv[c].y, xv[c].y, fma(pv[c].x, xv[c].x, s));
    y[t] = accumulate ? y[t] + s : s;
  }
}

// bc_a[c] = sum_{i in a, ascending} sum_r P_i[r][c] r_i[r]
__global__ void k_restrict(const int* __restrict__ agg_ptr, const int* __restrict__ members,
                           const double* __restrict__ P, const double* __restrict__ r, int nagg, int bs,
                           double* __restrict__ bc) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)nagg * 16; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = t >> 4;
    int c = (int)(t & 15);
    double s = 0.0;
    for (int q = agg_ptr[a]; q < agg_ptr[a + 1]; ++q) {
      int64_t i = members[q];
      const double* p = P + i * bs * 16 + c;
      const double* ri = r + i * bs;
      for (int k = 0; k < bs; ++k) s = fma(p[k * 16], ri[k], s);
    }
    bc[t] = s;
  }
}

extern "C" int bamg_prolong(bamg_ctx* ctx, const int32_t* agg, const double* P, const double* xc, int32_t nf,
                            int32_t bs, double* y, int32_t accumulate, void* stream) {
  (void)ctx;
  if (nf <= 0) return 0;
  launch(k_prolong, grid_for((int64_t)nf * bs, 256), 256, 0, as_stream(stream), agg, P, xc, nf, bs, y, accumulate);
  BAMG_LAUNCH_CHECK();
  return 0;
}

extern "C" int bamg_restrict(bamg_ctx* ctx, const int32_t* agg_ptr, const int32_t* members, const double* P,
                             const double* r, int32_t nagg, int32_t bs, double* bc, void* stream) {
  (void)ctx;
  if (nagg <= 0) return 0;
  launch(k_restrict, grid_for((int64_t)nagg * 16, 256), 256, 0, as_stream(stream), agg_ptr, members, P, r, nagg, bs, bc);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------------------
// batched block Cholesky + explicit inverse, bs <= 32 (blockmat.py:95-115):
// warp per block, L in shared memory, inverse = L^-T L^-1.

#define BCH_WARPS 4

__global__ void __launch_bounds__(BCH_WARPS * 32)
k_block_chol_inv(const double* __restrict__ M, int n, int bs, double* __restrict__ Lout, double* __restrict__ inv,
                 int* __restrict__ bad_min) {
  extern __shared__ double shm[];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* L = shm + (size_t)w * 2 * bs * bs;
  double* Li = L + bs * bs;
  int warp = blockIdx.x * BCH_WARPS + w;
  int nwarps = gridDim.x * BCH_WARPS;
  for (int blk = warp; blk < n; blk += nwarps) {
    const double* m = M + (int64_t)blk * bs * bs;
    for (int q = lane; q < bs * bs; q += 32) L[q] = m[q];
    __syncwarp();
    bool ok = true;
    for (int j = 0; j < bs; ++j) {
      // diagonal (lane 0), left-looking
      double d = 0.0;
      if (lane == 0) {
        d = L[j * bs + j];
        for (int k = 0; k < j; ++k) d -= L[j * bs + k] * L[j * bs + k];
      }
      d = __shfl_sync(FULL_MASK, d, 0);
      if (!(d > 0.0)) {
        ok = false;
        break;
      }
      double ljj = sqrt(d);
      int i = lane;
      double v = 0.0;
      if (i > j && i < bs) {
        v = L[i * bs + j];
        for (int k = 0; k < j; ++k) v -= L[i * bs + k] * L[j * bs + k];
        v /= ljj;
      }
      __syncwarp();
      if (i > j && i < bs) L[i * bs + j] = v;
      if (lane == 0) L[j * bs + j] = ljj;
      __syncwarp();
    }
    if (!ok) {
      if (lane == 0) atomicMin(bad_min, blk);
      __syncwarp();
      continue;
    }
    // zero the strict upper triangle of L
    for (int q = lane; q < bs * bs; q += 32) {
      int r = q / bs, c = q - r * bs;
      if (c > r) L[q] = 0.0;
    }
    __syncwarp();
    // Li = L^-1: lane c computes column c by forward substitution
    if (lane < bs) {
      int c = lane;
      for (int i = 0; i < bs; ++i) {
        double v;
        if (i < c) v = 0.0;
        else if (i == c) v = 1.0 / L[c * bs + c];
        else {
          double s = 0.0;
          for (int k = c; k < i; ++k) s += L[i * bs + k] * Li[k * bs + c];
          v = -s / L[i * bs + i];
        }
        Li[i * bs + c] = v;
      }
    }
    __syncwarp();
    double* out = inv + (int64_t)blk * bs * bs;
    for (int q = lane; q < bs * bs; q += 32) {
      int i = q / bs, j = q - i * bs;
      int k0 = i > j ? i : j;
      double s = 0.0;
      for (int k = k0; k < bs; ++k) s += Li[k * bs + i] * Li[k * bs + j];
      out[q] = s;
      if (Lout) Lout[(int64_t)blk * bs * bs + q] = L[q];
    }
    __syncwarp();
  }
}

extern "C" int bamg_block_chol_inv(bamg_ctx* ctx, const double* M, int32_t n, int32_t bs, double* L, double* inv,
                                   int32_t* bad_min_dev, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  int big = 0x7fffffff;
  set_i32(bad_min_dev, big, st);  // device-side: no pageable host copy in the stream
  if (n <= 0) return 0;
  if (bs > 32 || bs < 1) {
    bamg_set_error("block_chol_inv: block size %d outside [1, 32]", bs);
    return BAMG_ERR_UNSUPPORTED;
  }
  size_t sm = sizeof(double) * 2 * bs * bs * BCH_WARPS;
  if (sm > 48 * 1024) cudaFuncSetAttribute(k_block_chol_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  launch(k_block_chol_inv, grid_for(n, BCH_WARPS, 16), BCH_WARPS * 32, sm, st, M, n, bs, L, inv, bad_min_dev);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// y_b = M_b x_b (block-diagonal apply), bs arbitrary
__global__ void k_blockdiag_apply(const double* __restrict__ M, const double* __restrict__ x, int n, int bs,
                                  double* __restrict__ y) {
  PDL_ENTRY();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)n * bs; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = t / bs;
    int r = (int)(t - b * bs);
    const double* m = M + (b * bs + r) * bs;
    const double* xb = x + b * bs;
    double s = 0.0;
    for (int c = 0; c < bs; ++c) s = fma(m[c], xb[c], s);
    y[t] = s;
  }
}

extern "C" int bamg_blockdiag_apply(bamg_ctx* ctx, const double* M, const double* x, int32_t n, int32_t bs,
                                    double* y, void* stream) {
  (void)ctx;
  if (n <= 0) return 0;
  launch(k_blockdiag_apply, grid_for((int64_t)n * bs, 256), 256, 0, as_stream(stream), M, x, n, bs, y);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// diagonal blocks of a square BSR (zero where absent), blockmat.py:270-282
__global__ void k_diag_blocks(const int* __restrict__ ptr, const int* __restrict__ col,
                              const double* __restrict__ blocks, int nbr, int bs, double* __restrict__ D) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)nbr * bs * bs; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / (bs * bs);
    int q = (int)(t - i * bs * bs);
    int b0 = ptr[i], n = ptr[i + 1] - b0;
    int k = lower_bound_i32(col + b0, n, (int)i);
    D[t] = (k < n && col[b0 + k] == i) ? blocks[(int64_t)(b0 + k) * bs * bs + q] : 0.0;
  }
}

extern "C" int bamg_diag_blocks(bamg_ctx* ctx, const int32_t* ptr, const int32_t* col, const double* blocks,
                                int32_t nbr, int32_t bs, double* D, void* stream) {
  (void)ctx;
  if (nbr <= 0) return 0;
  launch(k_diag_blocks, grid_for((int64_t)nbr * bs * bs, 256), 256, 0, as_stream(stream), ptr, col, blocks, nbr, bs, D);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------------------
// coarsest level: densify + symmetrise, single-CTA Cholesky, explicit inverse
// (multigrid.py:431-440, 477-478)

__global__ void k_densify_sym(const int* __restrict__ ptr, const int* __restrict__ col, const double* __restrict__ blocks,
                              int nbr, int bs, double* __restrict__ Dn) {
  int n = nbr * bs;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)n * n; t += (int64_t)gridDim.x * blockDim.x)
    Dn[t] = 0.0;
}

__global__ void k_scatter_dense(const int* __restrict__ ptr, const int* __restrict__ col,
                                const double* __restrict__ blocks, int nbr, int bs, double* __restrict__ Dn) {
  int n = nbr * bs;
  for (int i = blockIdx.x; i < nbr; i += gridDim.x)
    for (int b = ptr[i]; b < ptr[i + 1]; ++b)
      for (int q = threadIdx.x; q < bs * bs; q += blockDim.x) {
        int r = q / bs, c = q - r * bs;
        Dn[(int64_t)(i * bs + r) * n + col[b] * bs + c] = blocks[(int64_t)b * bs * bs + q];
      }
}

__global__ void k_symmetrize(double* __restrict__ Dn, int n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)n * n; t += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(t / n), j = (int)(t - (int64_t)i * n);
    if (j < i) continue;
    double a = Dn[(int64_t)i * n + j], b = Dn[(int64_t)j * n + i];
    double v = 0.5 * (a + b);
    Dn[(int64_t)i * n + j] = v;
    Dn[(int64_t)j * n + i] = v;
  }
}

// In-place lower Cholesky of the n x n matrix in `a` (one CTA); flag[0] = 1 on failure.
__global__ void __launch_bounds__(1024) k_dense_chol(double* a, int n, int* flag) {
  __shared__ double piv;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      double d = a[(int64_t)j * n + j];
      if (!(d > 0.0)) bad = 1;
      piv = sqrt(d);
      a[(int64_t)j * n + j] = piv;
    }
    __syncthreads();
    if (bad) break;
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) a[(int64_t)i * n + j] /= piv;
    __syncthreads();
    int m = n - j - 1;
    for (int64_t t = threadIdx.x; t < (int64_t)m * m; t += blockDim.x) {
      int ii = (int)(t / m), kk = (int)(t - (int64_t)ii * m);
      if (kk > ii) continue;
      int i = j + 1 + ii, k = j + 1 + kk;
      a[(int64_t)i * n + k] -= a[(int64_t)i * n + j] * a[(int64_t)k * n + j];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) flag[0] = bad;
}

// Li = L^-1 (lower), thread per column
__global__ void k_tri_inv(const double* __restrict__ L, int n, double* __restrict__ Li) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    for (int i = 0; i < n; ++i) {
      double v;
      if (i < c) v = 0.0;
      else if (i == c) v = 1.0 / L[(int64_t)c * n + c];
      else {
        double s = 0.0;
        for (int k = c; k < i; ++k) s += L[(int64_t)i * n + k] * Li[(int64_t)k * n + c];
        v = -s / L[(int64_t)i * n + i];
      }
      Li[(int64_t)i * n + c] = v;
    }
  }
}

__global__ void k_ltl(const double* __restrict__ Li, int n, double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)n * n; t += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(t / n), j = (int)(t - (int64_t)i * n);
    int k0 = i > j ? i : j;
    double s = 0.0;
    for (int k = k0; k < n; ++k) s += Li[(int64_t)k * n + i] * Li[(int64_t)k * n + j];
    out[t] = s;
  }
}

// ---- tiled (32x32) dense Cholesky / triangular inverse / L^-T L^-1 -----------
#define DT 32

__device__ __forceinline__ int tile_dim(int n, int t) { return min(DT, n - t * DT); }

// factor diagonal tile k in place (lower); flag on a non-positive pivot
__device__ __forceinline__ void chol_diag_tile(double* a, int n, int k, int* flag) {
  __shared__ double T[DT][DT + 1];
  int tb = tile_dim(n, k);
  int r = threadIdx.x / DT, c = threadIdx.x % DT;
  int64_t base = (int64_t)k * DT * n + (int64_t)k * DT;
  if (r < tb && c < tb) T[r][c] = a[base + (int64_t)r * n + c];
  __syncthreads();
  for (int j = 0; j < tb; ++j) {
    if (threadIdx.x == 0) {
      double d = T[j][j];
      if (!(d > 0.0)) *flag = 1;
      T[j][j] = sqrt(d);
    }
    __syncthreads();
    if (r > j && r < tb && c == j) T[r][j] /= T[j][j];
    __syncthreads();
    if (r > j && r < tb && c > j && c <= r) T[r][c] -= T[r][j] * T[c][j];
    __syncthreads();
  }
  if (r < tb && c < tb) a[base + (int64_t)r * n + c] = (c <= r) ? T[r][c] : 0.0;
}

// L_ik = A_ik L_kk^-T for every tile row i > k (one CTA per tile, warp per row)
__device__ __forceinline__ void chol_trsm_tile(double* a, int n, int k, int bx) {
  __shared__ double Lk[DT][DT + 1];
  __shared__ double X[DT][DT + 1];
  int i = k + 1 + bx;
  int tk = tile_dim(n, k), ti = tile_dim(n, i);
  int r = threadIdx.x / DT, c = threadIdx.x % DT;
  if (r < tk && c < tk) Lk[r][c] = a[(int64_t)(k * DT + r) * n + k * DT + c];
  if (r < ti && c < tk) X[r][c] = a[(int64_t)(i * DT + r) * n + k * DT + c];
  __syncthreads();
  // row r of X solves x L^T = a: x[c] = (a[c] - sum_{j<c} x[j] L[c][j]) / L[c][c]
  if (r < ti) {
    for (int cc = 0; cc < tk; ++cc) {
      double part = (c < cc) ? X[r][c] * Lk[cc][c] : 0.0;
      part = warp_sum(part);
      if (c == cc) X[r][cc] = (X[r][cc] - part) / Lk[cc][cc];
      __syncwarp();
    }
  }
  __syncthreads();
  if (r < ti && c < tk) a[(int64_t)(i * DT + r) * n + k * DT + c] = X[r][c];
}

// A_ij -= L_ik L_jk^T for k < j <= i (one CTA per lower tile of the trailing matrix)
__device__ __forceinline__ void chol_update_tile(double* a, int n, int k, int nt, int t) {
  __shared__ double Li[DT][DT + 1];
  __shared__ double Lj[DT][DT + 1];
  int m = nt - k - 1;
  int ii = (int)((sqrt(8.0 * t + 1.0) - 1.0) / 2.0);
  while ((ii + 1) * (ii + 2) / 2 <= t) ++ii;
  while (ii * (ii + 1) / 2 > t) --ii;
  int jj = t - ii * (ii + 1) / 2;
  if (ii >= m) return;
  int i = k + 1 + ii, j = k + 1 + jj;
  int tk = tile_dim(n, k), ti = tile_dim(n, i), tj = tile_dim(n, j);
  for (int q = threadIdx.x; q < DT * DT; q += blockDim.x) {
    int r = q / DT, c = q % DT;
    Li[r][c] = (r < ti && c < tk) ? a[(int64_t)(i * DT + r) * n + k * DT + c] : 0.0;
    Lj[r][c] = (r < tj && c < tk) ? a[(int64_t)(j * DT + r) * n + k * DT + c] : 0.0;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < DT * DT; q += blockDim.x) {
    int r = q / DT, c = q % DT;
    if (r >= ti || c >= tj) continue;
    double s = 0.0;
#pragma unroll 8
    for (int x = 0; x < DT; ++x) s = fma(Li[r][x], Lj[c][x], s);
    a[(int64_t)(i * DT + r) * n + j * DT + c] -= s;
  }
}

// inverse of each diagonal tile of L (lower), thread per column
__device__ __forceinline__ void tile_inv_diag(const double* __restrict__ L, int n, double* __restrict__ Li, int k) {
  __shared__ double T[DT][DT + 1];
  __shared__ double X[DT][DT + 1];
  int tb = tile_dim(n, k);
  int c = threadIdx.x;
  for (int r = 0; r < tb; ++r) T[r][c] = (c < tb) ? L[(int64_t)(k * DT + r) * n + k * DT + c] : 0.0;
  __syncthreads();
  if (c < tb) {
    for (int r = 0; r < tb; ++r) {
      double v;
      if (r < c) v = 0.0;
      else if (r == c) v = 1.0 / T[c][c];
      else {
        double s = 0.0;
        for (int x = c; x < r; ++x) s += T[r][x] * X[x][c];
        v = -s / T[r][r];
      }
      X[r][c] = v;
    }
  }
  __syncthreads();
  if (c < tb)
    for (int r = 0; r < tb; ++r) Li[(int64_t)(k * DT + r) * n + k * DT + c] = X[r][c];
}

// block column k of L^-1: Li_ik = -Li_ii (sum_{j=k}^{i-1} L_ij Li_jk), i = k+1.. (one CTA per k)
__device__ __forceinline__ void tile_inv_col(const double* __restrict__ L, int n, int nt, double* __restrict__ Li,
                                             int k) {
  __shared__ double A[DT][DT + 1];
  __shared__ double B[DT][DT + 1];
  __shared__ double S[DT][DT + 1];
  int tk = tile_dim(n, k);
  for (int i = k + 1; i < nt; ++i) {
    int ti = tile_dim(n, i);
    for (int q = threadIdx.x; q < DT * DT; q += blockDim.x) S[q / DT][q % DT] = 0.0;
    for (int j = k; j < i; ++j) {
      int tj = tile_dim(n, j);
      __syncthreads();
      for (int q = threadIdx.x; q < DT * DT; q += blockDim.x) {
        int r = q / DT, c = q % DT;
        A[r][c] = (r < ti && c < tj) ? L[(int64_t)(i * DT + r) * n + j * DT + c] : 0.0;
        B[r][c] = (r < tj && c < tk) ? Li[(int64_t)(j * DT + r) * n + k * DT + c] : 0.0;
      }
      __syncthreads();
      for (int q = threadIdx.x; q < DT * DT; q += blockDim.x) {
        int r = q / DT, c = q % DT;
        double s = 0.0;
#pragma unroll 8
        for (int x = 0; x < DT; ++x) s = fma(A[r][x], B[x][c], s);
        S[r][c] += s;
      }
    }
    __syncthreads();
    // Li_ik = -Li_ii S
    for (int q = threadIdx.x; q < DT * DT; q += blockDim.x) {
      int r = q / DT, c = q % DT;
      A[r][c] = (r < ti && c < ti) ? Li[(int64_t)(i * DT + r) * n + i * DT + c] : 0.0;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < DT * DT; q += blockDim.x) {
      int r = q / DT, c = q % DT;
      if (r >= ti || c >= tk) continue;
      double s = 0.0;
      for (int x = 0; x <= r; ++x) s = fma(A[r][x], S[x][c], s);
      Li[(int64_t)(i * DT + r) * n + k * DT + c] = -s;
    }
    __syncthreads();
  }
  // zero the strict upper tiles of column k
  for (int i = 0; i < k; ++i) {
    int ti = tile_dim(n, i);
    for (int q = threadIdx.x; q < DT * DT; q += blockDim.x) {
      int r = q / DT, c = q % DT;
      if (r < ti && c < tk) Li[(int64_t)(i * DT + r) * n + k * DT + c] = 0.0;
    }
  }
}

// inv = Li^T Li, one CTA per output tile (I, J)
__device__ __forceinline__ void tile_ltl(const double* __restrict__ Li, int n, int nt, double* __restrict__ out, int bx) {
  __shared__ double A[DT][DT + 1];
  __shared__ double B[DT][DT + 1];
  int I = bx / nt, J = bx % nt;
  int tI = tile_dim(n, I), tJ = tile_dim(n, J);
  double acc[4] = {0, 0, 0, 0};
  for (int K = max(I, J); K < nt; ++K) {
    int tK = tile_dim(n, K);
    __syncthreads();
    for (int q = threadIdx.x; q < DT * DT; q += blockDim.x) {
      int r = q / DT, c = q % DT;
      A[r][c] = (r < tK && c < tI) ? Li[(int64_t)(K * DT + r) * n + I * DT + c] : 0.0;
      B[r][c] = (r < tK && c < tJ) ? Li[(int64_t)(K * DT + r) * n + J * DT + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int q = threadIdx.x + u * 256;
      int r = q / DT, c = q % DT;
      double s = 0.0;
#pragma unroll 8
      for (int x = 0; x < DT; ++x) s = fma(A[x][r], B[x][c], s);
      acc[u] += s;
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    int q = threadIdx.x + u * 256;
    int r = q / DT, c = q % DT;
    if (r < tI && c < tJ) out[(int64_t)(I * DT + r) * n + J * DT + c] = acc[u];
  }
}

// single-matrix kernels (coarsest level)
__global__ void __launch_bounds__(1024) k_chol_diag(double* a, int n, int k, int* flag) { chol_diag_tile(a, n, k, flag); }
__global__ void __launch_bounds__(1024) k_chol_trsm(double* a, int n, int k) { chol_trsm_tile(a, n, k, blockIdx.x); }
__global__ void __launch_bounds__(256) k_chol_update(double* a, int n, int k, int nt) {
  chol_update_tile(a, n, k, nt, blockIdx.x);
}
__global__ void __launch_bounds__(DT) k_tile_inv_diag(const double* __restrict__ L, int n, double* __restrict__ Li) {
  tile_inv_diag(L, n, Li, blockIdx.x);
}
__global__ void __launch_bounds__(256) k_tile_inv_col(const double* __restrict__ L, int n, int nt,
                                                      double* __restrict__ Li) {
  tile_inv_col(L, n, nt, Li, blockIdx.x);
}
__global__ void __launch_bounds__(256) k_tile_ltl(const double* __restrict__ Li, int n, int nt, double* __restrict__ out) {
  tile_ltl(Li, n, nt, out, blockIdx.x);
}

// dense = sym(BSR); L = chol(dense) (in `work`), inv = L^-T L^-1 -- tiled, many CTAs.
extern "C" int bamg_coarse_factor(bamg_ctx* ctx, const int32_t* ptr, const int32_t* col, const double* blocks,
                                  int32_t nbr, int32_t bs, double* dense, double* work, double* inv,
                                  int32_t* flag_dev, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  int n = nbr * bs;
  if (n <= 0) return 0;
  launch(k_densify_sym, grid_for((int64_t)n * n, 256), 256, 0, st, ptr, col, blocks, nbr, bs, dense);
  launch(k_scatter_dense, grid_for(nbr, 1, 8), 128, 0, st, ptr, col, blocks, nbr, bs, dense);
  launch(k_symmetrize, grid_for((int64_t)n * n, 256), 256, 0, st, dense, n);
  BAMG_CUDA_CHECK(cudaMemcpyAsync(work, dense, sizeof(double) * n * (int64_t)n, cudaMemcpyDeviceToDevice, st));
  BAMG_CUDA_CHECK(cudaMemsetAsync(flag_dev, 0, sizeof(int), st));
  int nt = (n + DT - 1) / DT;
  for (int k = 0; k < nt; ++k) {
    launch(k_chol_diag, 1, 1024, 0, st, work, n, k, flag_dev);
    int m = nt - k - 1;
    if (m > 0) {
      launch(k_chol_trsm, m, 1024, 0, st, work, n, k);
      launch(k_chol_update, m * (m + 1) / 2, 256, 0, st, work, n, k, nt);
    }
  }
  // strict upper tiles of L are stale copies of A: the inverse kernels never read them
  launch(k_tile_inv_diag, nt, DT, 0, st, work, n, dense);
  launch(k_tile_inv_col, nt, 256, 0, st, work, n, nt, dense);
  launch(k_tile_ltl, nt * nt, 256, 0, st, dense, n, nt, inv);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// y = M x for dense n x n (warp per row)
__global__ void k_gemv(const double* __restrict__ M, const double* __restrict__ x, int n, double* __restrict__ y) {
  PDL_ENTRY();
  int lane = threadIdx.x & 31;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < n; i += nwarps) {
    double s = 0.0;
    for (int c = lane; c < n; c += 32) s = fma(M[(int64_t)i * n + c], x[c], s);
    s = warp_sum(s);
    if (lane == 0) y[i] = s;
  }
}

extern "C" int bamg_dense_gemv(bamg_ctx* ctx, const double* M, const double* x, int32_t n, double* y, void* stream) {
  (void)ctx;
  if (n <= 0) return 0;
  launch(k_gemv, grid_for((int64_t)n * 32, 128, 8), 128, 0, as_stream(stream), M, x, n, y);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------------------
// Visibility block-Jacobi (precond.py:59-144): one dense principal submatrix of S
// per camera cluster (clusters from the greedy aggregation with cap 100, members
// ascending), factored with the tiled Cholesky above batched over clusters
// (blockIdx.y = cluster; tiles beyond a cluster's size exit), then inverted
// explicitly (L^-T L^-1) so the apply is one batched gather-GEMV-scatter.
// Cluster c: dim[c] = 9 |members|, row-major dim x dim at off[c] doubles.

// S blocks whose row and column cameras share a cluster land in that cluster's
// matrix (positions by binary search in the ascending member list).
__global__ void k_vj_assemble(const int* __restrict__ S_ptr, const int* __restrict__ S_col,
                              const double* __restrict__ S_blocks, int nc, const int* __restrict__ agg,
                              const int* __restrict__ cptr, const int* __restrict__ mem,
                              const long long* __restrict__ off, const int* __restrict__ dim,
                              double* __restrict__ dense) {
  int lane = threadIdx.x & 31;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < nc; i += nwarps) {
    int c = agg[i];
    int m0 = cptr[c], mlen = cptr[c + 1] - m0;
    int pi = lower_bound_i32(mem + m0, mlen, i);
    int n = dim[c];
    double* M = dense + off[c];
    for (int q = S_ptr[i]; q < S_ptr[i + 1]; ++q) {
      int j = S_col[q];
      if (agg[j] != c) continue;
      int pj = lower_bound_i32(mem + m0, mlen, j);
      const double* B = S_blocks + (int64_t)q * 81;
      for (int e = lane; e < 81; e += 32) {
        int r = e / 9, cc = e - 9 * r;
        M[(int64_t)(9 * pi + r) * n + 9 * pj + cc] = B[e];
      }
    }
  }
}

__device__ __forceinline__ int vj_tiles(int n) { return (n + DT - 1) / DT; }

__global__ void __launch_bounds__(1024) k_bchol_diag(double* a, const long long* off, const int* dim, int k, int* flags) {
  int c = blockIdx.y, n = dim[c];
  if (k >= vj_tiles(n)) return;
  chol_diag_tile(a + off[c], n, k, flags + c);
}
__global__ void __launch_bounds__(1024) k_bchol_trsm(double* a, const long long* off, const int* dim, int k) {
  int c = blockIdx.y, n = dim[c];
  if (k + 1 + (int)blockIdx.x >= vj_tiles(n)) return;
  chol_trsm_tile(a + off[c], n, k, blockIdx.x);
}
__global__ void __launch_bounds__(256) k_bchol_update(double* a, const long long* off, const int* dim, int k) {
  int c = blockIdx.y, n = dim[c], nt = vj_tiles(n);
  int m = nt - k - 1;
  if (m <= 0 || (int)blockIdx.x >= m * (m + 1) / 2) return;
  chol_update_tile(a + off[c], n, k, nt, blockIdx.x);
}
__global__ void __launch_bounds__(DT) k_btile_inv_diag(const double* L, const long long* off, const int* dim, double* Li) {
  int c = blockIdx.y, n = dim[c];
  if ((int)blockIdx.x >= vj_tiles(n)) return;
  tile_inv_diag(L + off[c], n, Li + off[c], blockIdx.x);
}
__global__ void __launch_bounds__(256) k_btile_inv_col(const double* L, const long long* off, const int* dim, double* Li) {
  int c = blockIdx.y, n = dim[c], nt = vj_tiles(n);
  if ((int)blockIdx.x >= nt) return;
  tile_inv_col(L + off[c], n, nt, Li + off[c], blockIdx.x);
}
__global__ void __launch_bounds__(256) k_btile_ltl(const double* Li, const long long* off, const int* dim, double* out) {
  int c = blockIdx.y, n = dim[c], nt = vj_tiles(n);
  if ((int)blockIdx.x >= nt * nt) return;
  tile_ltl(Li + off[c], n, nt, out + off[c], blockIdx.x);
}

// z[members] = inv_c r[members], warp per local row (blockIdx.y = cluster)
__global__ void __launch_bounds__(128)
k_vj_apply(const long long* __restrict__ off, const int* __restrict__ dim, const int* __restrict__ cptr,
           const int* __restrict__ mem, const double* __restrict__ inv, const double* __restrict__ r,
           double* __restrict__ z) {
  int c = blockIdx.y, n = dim[c];
  int lane = threadIdx.x & 31;
  int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int rstride = (gridDim.x * blockDim.x) >> 5;
  const int* mc = mem + cptr[c];
  const double* M = inv + off[c];
  for (; row < n; row += rstride) {
    double s = 0.0;
    for (int j = lane; j < n; j += 32) s = fma(M[(int64_t)row * n + j], r[(int64_t)mc[j / 9] * 9 + j % 9], s);
    s = warp_sum(s);
    if (lane == 0) z[(int64_t)mc[row / 9] * 9 + row % 9] = s;
  }
}

extern "C" int bamg_vj_assemble(bamg_ctx* ctx, const int32_t* S_ptr, const int32_t* S_col, const double* S_blocks,
                                int32_t nc, const int32_t* agg, const int32_t* cptr, const int32_t* mem,
                                const int64_t* off, const int32_t* dim, double* dense, int64_t total, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (nc <= 0) return 0;
  BAMG_CUDA_CHECK(cudaMemsetAsync(dense, 0, sizeof(double) * (size_t)total, st));
  launch(k_vj_assemble, grid_for((int64_t)nc * 32, 128, 8), 128, 0, st, S_ptr, S_col, S_blocks, nc, agg, cptr, mem,
         (const long long*)off, dim, dense);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// work: in A (assembled), out L; tmp: L^-1 scratch; inv: A^-1. flags[c] = 1 if
// cluster c hit a non-positive pivot (precond.py:139-143).
extern "C" int bamg_vj_factor(bamg_ctx* ctx, int32_t ncl, int32_t dim_max, const int64_t* off, const int32_t* dim,
                              double* work, double* tmp, double* inv, int32_t* flags, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (ncl <= 0) return 0;
  if (ncl > 65535) {
    bamg_set_error("vj_factor: %d clusters exceed the grid's y range", ncl);
    return BAMG_ERR_UNSUPPORTED;
  }
  const long long* o = (const long long*)off;
  BAMG_CUDA_CHECK(cudaMemsetAsync(flags, 0, sizeof(int) * (size_t)ncl, st));
  int ntm = (dim_max + DT - 1) / DT;
  for (int k = 0; k < ntm; ++k) {
    launch(k_bchol_diag, dim3(1, ncl), 1024, 0, st, work, o, dim, k, flags);
    int m = ntm - k - 1;
    if (m > 0) {
      launch(k_bchol_trsm, dim3(m, ncl), 1024, 0, st, work, o, dim, k);
      launch(k_bchol_update, dim3(m * (m + 1) / 2, ncl), 256, 0, st, work, o, dim, k);
    }
  }
  launch(k_btile_inv_diag, dim3(ntm, ncl), DT, 0, st, (const double*)work, o, dim, tmp);
  launch(k_btile_inv_col, dim3(ntm, ncl), 256, 0, st, (const double*)work, o, dim, tmp);
  launch(k_btile_ltl, dim3(ntm * ntm, ncl), 256, 0, st, (const double*)tmp, o, dim, inv);
  BAMG_LAUNCH_CHECK();
  return 0;
}

static void vj_apply_launch(int ncl, int dim_max, const long long* off, const int* dim, const int* cptr, const int* mem,
                            const double* inv, const double* r, double* z, cudaStream_t st) {
  int gx = (dim_max + 3) / 4;
  if (gx > 64) gx = 64;
  launch(k_vj_apply, dim3(gx, ncl), 128, 0, st, off, dim, cptr, mem, inv, r, z);
}

struct bamg_vj {
  int ncl, dim_max;
  const long long* off;
  const int *dim, *cptr, *mem;
  const double* inv;
};

extern "C" bamg_vj* bamg_vj_create(int32_t ncl, int32_t dim_max, const int64_t* off, const int32_t* dim,
                                   const int32_t* cptr, const int32_t* mem, const double* inv) {
  return new bamg_vj{ncl, dim_max, (const long long*)off, dim, cptr, mem, inv};
}

extern "C" void bamg_vj_destroy(bamg_vj* v) { delete v; }

static void vj_apply_dev(const bamg_vj* v, const double* r, double* z, cudaStream_t st) {
  vj_apply_launch(v->ncl, v->dim_max, v->off, v->dim, v->cptr, v->mem, v->inv, r, z, st);
}

extern "C" int bamg_vj_apply(bamg_ctx* ctx, const bamg_vj* v, const double* r, double* z, void* stream) {
  (void)ctx;
  if (!v || v->ncl <= 0) return 0;
  vj_apply_dev(v, r, z, as_stream(stream));
  BAMG_LAUNCH_CHECK();
  return 0;
}

// PCG vector updates (solver.py:108-127): x += a p ; r -= a ap ; rr = <r, r>
__global__ void __launch_bounds__(256)
k_pcg_update(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p, const double* __restrict__ ap,
             double a, int64_t n, double* partials, unsigned int* counter, double* rr_out) {
  __shared__ double scratch[33];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] += a * p[i];
    double ri = r[i] - a * ap[i];
    r[i] = ri;
    s = fma(ri, ri, s);
  }
  s = block_sum(s, scratch);
  grid_finish(partials, counter, s, scratch, rr_out);
}

extern "C" int bamg_pcg_update(bamg_ctx* ctx, double* x, double* r, const double* p, const double* ap, double alpha,
                               int64_t n, double* rr_dev, void* stream) {
  cudaStream_t st = as_stream(stream);
  int g = grid_for(n, 256, 4);
  launch(k_pcg_update, g, 256, 0, st, x, r, p, ap, alpha, n, ctx->partials, ctx->counters + BAMG_CTR_PCG0, rr_dev);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// p = z + beta p
__global__ void k_xpby(const double* __restrict__ z, double beta, double* __restrict__ p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}

extern "C" int bamg_xpby(bamg_ctx* ctx, const double* z, double beta, double* p, int64_t n, void* stream) {
  (void)ctx;
  if (n) launch(k_xpby, grid_for(n, 256), 256, 0, as_stream(stream), z, beta, p, n);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// solve-phase runtime (V-cycle program / graph, PCG, Lanczos) shares this TU
// so that it can launch the templated kernels above directly.
#include "vcycle.cuh"
