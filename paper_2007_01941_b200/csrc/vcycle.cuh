// Native solve-phase runtime: the multigrid V-cycle as a fixed kernel program
// (replayed through a CUDA graph), PCG with one host synchronisation per
// iteration, and the 5-step D-Lanczos spectral estimate with a single readback.
//
// Reference semantics: mgcycle (multigrid.py:474-483), ChebyshevSmoother.apply
// (multigrid.py:308-328), pcg + ForcingCriterion (solver.py:38-128),
// estimate_lambda_max (multigrid.py:243-284).
// Included at the end of blas.cu (same translation unit as the kernels it launches).
#include <math.h>

#include <chrono>
#include <vector>

int dot_dev(bamg_ctx* ctx, const double* x, const double* y, int64_t n, double* out, cudaStream_t st);

// ---------------------------------------------------------------------------
// small device-scalar vector kernels

// y = x (copy)
__global__ void k_copy(const double* __restrict__ x, double* __restrict__ y, int64_t n) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i];
}

// PCG x/r update with alpha = rz/pap read from device scalars; rr = <r, r>.
__global__ void __launch_bounds__(256)
k_pcg_update_dev(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                 const double* __restrict__ ap, const double* __restrict__ rz, const double* __restrict__ pap,
                 int64_t n, double* partials, unsigned int* counter, double* rr_out) {
  PDL_ENTRY();
  __shared__ double scratch[33];
  double a = (*rz) / (*pap);
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

// p = z + (rz_new / rz_old) p
__global__ void k_xpby_dev(const double* __restrict__ z, const double* __restrict__ rz_new,
                           const double* __restrict__ rz_old, double* __restrict__ p, int64_t n) {
  PDL_ENTRY();
  double beta = (*rz_new) / (*rz_old);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}

// ---------------------------------------------------------------------------
// Symmetric half-storage 9x9 SpMV for S. S is stored in full (the setup phase
// reads whole rows), but S_ji == S_ij^T bit for bit (schur.cu writes both from one
// value), so the solve phase streams only the upper blocks U_ij (j >= i): positions
// dpos[i]..ptr[i+1]-1 of each row. Two deterministic passes, no atomics:
//   pass 1 (warp per chunk of row i): y_i^up = sum_{j>=i} U_ij x_j, and for j > i the
//          mirror product t = U_ij^T x_i, stored at the position of the mirror block
//          (j, i) (destination order, T_SLOT; evict_last so it stays in L2);
//   pass 2 (warp per row j): y_j = sum_{lower p of row j, column order} T[p] + y_j^up,
//          the row's lower range read contiguously, then the consumer's epilogue
//          (plain / residual / Chebyshev step).
// Bytes per product: (nnz+n)/2 blocks + 2 x 72 B per off-diagonal pair instead of
// nnz blocks -- 0.6x of the full-storage stream.
int scan_exclusive_int(const int* in, int* out, int64_t n, int* total, cudaStream_t st);
extern "C" void bamg_symop_destroy(bamg_symop* S);

struct bamg_symop {
  int bs = 9;              // 9 (S) or 16 (coarse Galerkin operators)
  int nbr = 0;
  int64_t nnzb = 0;
  const int* ptr = nullptr;
  const int* col = nullptr;
  const int* dpos = nullptr;
  int* dpos_own = nullptr; // dpos derived here (pattern-only construction)
  int* tpos = nullptr;     // per full position: mirror position
  double* T = nullptr;     // nnzb x bs, upper off-diagonal positions used
  // pass-1 work units: chunks of <= ch upper blocks of one row (rows' upper
  // parts range from 0 to 2x the mean length, so a warp per row is imbalanced)
  int ch = 24;
  int nch = 0;
  int* ucptr = nullptr;    // nbr + 1: chunk range of each row
  int* cbeg = nullptr;     // nch: first upper position
  int* crow = nullptr;     // nch: row
  double* yup = nullptr;   // nch x bs partial row products
  cudaStream_t alloc_stream = nullptr;
};

// Where the mirrored product of upper block b lives. Destination order (default):
// at the position of its mirror (lower) block, so pass 2 streams each row's lower
// range contiguously with no index indirection, and pass 1's 72 / 128 B stores are
// scattered (fire-and-forget). SYM_SRC_ORDER: at b itself (coalesced stores,
// gathered reads through tpos).
#ifdef SYM_SRC_ORDER
#define T_SLOT(b) (b)
#define T_READ(p) __ldg(tpos + (p))
#else
#define T_SLOT(b) __ldg(tpos + (b))
#define T_READ(p) (p)
#endif

#ifndef SYM_CH
#define SYM_CH 24
#endif
#ifndef SYM_CH16
#define SYM_CH16 8
#endif
#ifndef SYM_MINB
#define SYM_MINB 1
#endif

__global__ void k_sym_chunk_counts(const int* __restrict__ ptr, const int* __restrict__ dpos, int nbr, int CH,
                                   int* __restrict__ cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nbr; i += gridDim.x * blockDim.x)
    cnt[i] = (ptr[i + 1] - dpos[i] + CH - 1) / CH;
}

__global__ void k_sym_chunk_fill(const int* __restrict__ dpos, const int* __restrict__ ucptr, int nbr, int CH,
                                 int* __restrict__ cbeg, int* __restrict__ crow) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nbr; i += gridDim.x * blockDim.x)
    for (int c = ucptr[i]; c < ucptr[i + 1]; ++c) {
      cbeg[c] = dpos[i] + (c - ucptr[i]) * CH;
      crow[c] = i;
    }
}

// pattern-only construction: diagonal slot of every row and the mirror position of
// every block (binary search of i in row j), warp per row
__global__ void k_sym_pattern(const int* __restrict__ ptr, const int* __restrict__ col, int nbr,
                              int* __restrict__ dpos, int* __restrict__ tpos) {
  int lane = threadIdx.x & 31;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < nbr; i += nwarps) {
    int b0 = ptr[i], b1 = ptr[i + 1];
    if (lane == 0) dpos[i] = b0 + lower_bound_i32(col + b0, b1 - b0, i);
    for (int q = b0 + lane; q < b1; q += 32) {
      int j = col[q];
      tpos[q] = ptr[j] + lower_bound_i32(col + ptr[j], ptr[j + 1] - ptr[j], i);
    }
  }
}

__global__ void k_sym_mirror(const int* __restrict__ up_blk, const int* __restrict__ up_tpos, int n_up,
                             int* __restrict__ tpos) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n_up; u += gridDim.x * blockDim.x) {
    tpos[up_blk[u]] = up_tpos[u];
    tpos[up_tpos[u]] = up_blk[u];
  }
}

// pass 1: warp per chunk (<= SYM_CH upper blocks of row i); lane (g, c) =
// (lane / 9, lane % 9) walks blocks cbeg+g, +3, ... and reads column c of U (the 27
// lanes cover three consecutive blocks per step). Writes the chunk's partial row
// product to yup[chunk].
__global__ void __launch_bounds__(128, SYM_MINB)
k_sym9_upper(const int* __restrict__ ptr, const int* __restrict__ col, const int* __restrict__ dpos,
             const int* __restrict__ tpos, const int* __restrict__ cbeg, const int* __restrict__ crow, int nch,
             const double* __restrict__ blocks, const double* __restrict__ x, double* __restrict__ T,
             double* __restrict__ yup, int blk_policy) {
  PDL_ENTRY();
  __shared__ double red[4][27 * 9];
  const uint64_t pb = l2_policy(blk_policy), pt = l2_policy(L2_LAST);
  int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  int g = lane / 9, c = lane - 9 * g;
  for (int ch = warp; ch < nch; ch += nwarps) {
    int row = crow[ch];
    double xi[9], acc[9];
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      xi[r] = __ldg(x + (int64_t)row * 9 + r);
      acc[r] = 0.0;
    }
    if (g < 3) {
      int bd = dpos[row], b0 = cbeg[ch], be = min(b0 + SYM_CH, ptr[row + 1]);
#pragma unroll 2
      for (int b = b0 + g; b < be; b += 3) {
        double xjc = __ldg(x + (int64_t)col[b] * 9 + c);
        const double* U = blocks + (int64_t)b * 81 + c;
        double t = 0.0;
#pragma unroll
        for (int r = 0; r < 9; ++r) {
          double v = ld_pol(U + 9 * r, pb);
          acc[r] = fma(v, xjc, acc[r]);
          t = fma(v, xi[r], t);
        }
        if (b != bd) st_pol(T + (int64_t)T_SLOT(b) * 9 + c, t, pt);
      }
#pragma unroll
      for (int r = 0; r < 9; ++r) red[wib][lane * 9 + r] = acc[r];
    }
    __syncwarp();
    if (lane < 9) {
      double s = 0.0;
      for (int k = 0; k < 27; ++k) s += red[wib][k * 9 + lane];
      yup[(int64_t)ch * 9 + lane] = s;
    }
    __syncwarp();
  }
}

#ifndef SYM_FB
#define SYM_FB 12
#endif
// pass 2 + epilogue. mode 0: out = ax (dot_out: <x_in, ax>, deterministic);
// mode 1: out = b - ax; mode 2: the fused Chebyshev step of k_cheb_step.
template <int FB>
__global__ void __launch_bounds__(128, 1)
k_sym9_finish(const int* __restrict__ ptr, const int* __restrict__ dpos, const int* __restrict__ tpos,
              const double* __restrict__ T,
              const int* __restrict__ ucptr, const double* __restrict__ yup, int nbr, int mode, const double* __restrict__ b,
              const double* __restrict__ Dinv, double* __restrict__ d, const double* __restrict__ x_in,
              double* __restrict__ out, double c1, double c2, int divide, double* partials, unsigned int* counter,
              double* dot_out) {
  PDL_ENTRY();
  __shared__ double scratch[33];
  const uint64_t pt = l2_policy(L2_LAST);
  int lane = threadIdx.x & 31;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  int g = lane / 9, c = lane - 9 * g;
  double dsum = 0.0;
  for (int row = warp; row < nbr; row += nwarps) {
    double s = 0.0;
    if (g < 3) {
      int p = ptr[row] + g, p1 = dpos[row];
      // batches of FB (this lane's p, p+3, ...): indices, then products, then the
      // in-order additions -- same sums, FB loads in flight instead of 1
      for (; p + 3 * (FB - 1) < p1; p += 3 * FB) {
        int tp[FB];
        double v[FB];
#pragma unroll
        for (int u = 0; u < FB; ++u) tp[u] = T_READ(p + 3 * u);
#pragma unroll
        for (int u = 0; u < FB; ++u) v[u] = ld_pol(T + (int64_t)tp[u] * 9 + c, pt);
#pragma unroll
        for (int u = 0; u < FB; ++u) s += v[u];
      }
      for (; p < p1; p += 3) s += ld_pol(T + (int64_t)T_READ(p) * 9 + c, pt);
    }
    double s1 = __shfl_down_sync(FULL_MASK, s, 9);
    double s2 = __shfl_down_sync(FULL_MASK, s, 18);
    int64_t e = (int64_t)row * 9 + (lane < 9 ? lane : 0);
    double up = 0.0;
    if (lane < 9)
      for (int k = ucptr[row]; k < ucptr[row + 1]; ++k) up += yup[(int64_t)k * 9 + lane];
    double ax = (lane < 9) ? (s + s1) + s2 + up : 0.0;
    if (mode == 0) {
      if (lane < 9) {
        out[e] = ax;
        if (dot_out) dsum = fma(x_in[e], ax, dsum);
      }
      continue;
    }
    double rr = (lane < 9) ? b[e] - ax : 0.0;
    if (mode == 1) {
      if (lane < 9) out[e] = rr;
      continue;
    }
    double z = 0.0;
    const double* Di = Dinv + (int64_t)row * 81 + (lane < 9 ? lane : 0) * 9;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      double rk = __shfl_sync(FULL_MASK, rr, k);
      if (lane < 9) z = fma(Di[k], rk, z);
    }
    if (lane < 9) {
      double dn = divide ? z / c2 : c1 * d[e] + c2 * z;
      d[e] = dn;
      out[e] = x_in[e] + dn;
    }
  }
  if (dot_out) {
    dsum = block_sum(dsum, scratch);
    grid_finish(partials, counter, dsum, scratch, dot_out);
  }
}

// 16x16 pass 1: warp per chunk of <= SYM_CH16 upper blocks of row i. Every 2 KB
// block is read as four coalesced 512 B double2 sweeps (lane l: column pair
// cp = 2(l%8) of rows l/8 + 4k, k = 0..3). Row part: a_k += U[r_k][cp..] . x_j[cp..],
// reduced over the 8 lanes of a row once per chunk. Mirror part: t[cp..] =
// sum_k U[r_k][cp..] x_i[r_k], reduced over the 4 lanes sharing cp (xor 8, 16) and
// stored by lanes 0..7 at the mirror block's position (128 B, destination order).
__global__ void __launch_bounds__(128)
k_sym16_upper(const int* __restrict__ ptr, const int* __restrict__ col, const int* __restrict__ dpos,
              const int* __restrict__ tpos, const int* __restrict__ cbeg, const int* __restrict__ crow, int nch, const double* __restrict__ blocks,
              const double* __restrict__ x, double* __restrict__ T, double* __restrict__ yup, int blk_policy) {
  PDL_ENTRY();
  const uint64_t pb = l2_policy(blk_policy), pt = l2_policy(L2_LAST);
  int lane = threadIdx.x & 31;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int cp = 2 * (lane & 7), r0 = lane >> 3;
  for (int ch = warp; ch < nch; ch += nwarps) {
    int row = crow[ch];
    const double* xr = x + (int64_t)row * 16;
    double xi0 = __ldg(xr + r0), xi1 = __ldg(xr + r0 + 4), xi2 = __ldg(xr + r0 + 8), xi3 = __ldg(xr + r0 + 12);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int bd = dpos[row], b0 = cbeg[ch], be = min(b0 + SYM_CH16, ptr[row + 1]);
    for (int b = b0; b < be; ++b) {
      const double2* U = reinterpret_cast<const double2*>(blocks + (int64_t)b * 256) + lane;
      double2 u0 = ld2_pol(U, pb), u1 = ld2_pol(U + 32, pb), u2 = ld2_pol(U + 64, pb), u3 = ld2_pol(U + 96, pb);
      double2 xj = __ldg(reinterpret_cast<const double2*>(x + (int64_t)col[b] * 16 + cp));
      a0 = fma(u0.x, xj.x, fma(u0.y, xj.y, a0));
      a1 = fma(u1.x, xj.x, fma(u1.y, xj.y, a1));
      a2 = fma(u2.x, xj.x, fma(u2.y, xj.y, a2));
      a3 = fma(u3.x, xj.x, fma(u3.y, xj.y, a3));
      double tx = fma(u3.x, xi3, fma(u2.x, xi2, fma(u1.x, xi1, u0.x * xi0)));
      double ty = fma(u3.y, xi3, fma(u2.y, xi2, fma(u1.y, xi1, u0.y * xi0)));
      tx += __shfl_xor_sync(FULL_MASK, tx, 8);
      ty += __shfl_xor_sync(FULL_MASK, ty, 8);
      tx += __shfl_xor_sync(FULL_MASK, tx, 16);
      ty += __shfl_xor_sync(FULL_MASK, ty, 16);
      if (b != bd && lane < 8)
        st2_pol(reinterpret_cast<double2*>(T + (int64_t)T_SLOT(b) * 16) + lane, make_double2(tx, ty), pt);
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
    double v = k == 0 ? s0 : (k == 1 ? s1 : (k == 2 ? s2 : s3));
    if (lane < 16) yup[(int64_t)ch * 16 + lane] = v;
  }
}

// 16x16 pass 2 + epilogue (modes as k_sym9_finish); two rows per warp, lane r of a
// half-warp owns entry r of its row.
#ifndef SYM16_FB
#define SYM16_FB 16
#endif
__global__ void __launch_bounds__(128, 1)
k_sym16_finish(const int* __restrict__ ptr, const int* __restrict__ dpos, const int* __restrict__ tpos,
               const double* __restrict__ T, const int* __restrict__ ucptr, const double* __restrict__ yup, int nbr,
               int mode, const double* __restrict__ b, const double* __restrict__ Dinv, double* __restrict__ d,
               const double* __restrict__ x_in, double* __restrict__ out, double c1, double c2, int divide,
               double* partials, unsigned int* counter, double* dot_out) {
  PDL_ENTRY();
  __shared__ double scratch[33];
  const uint64_t pt = l2_policy(L2_LAST);
  int lane = threadIdx.x & 31;
  int half = lane >> 4, r = lane & 15;
  int row0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 2;
  int stride = ((gridDim.x * blockDim.x) >> 5) * 2;
  double dsum = 0.0;
  for (int base = row0; base < nbr; base += stride) {
    int row = base + half;
    bool ok = row < nbr;
    double ax = 0.0;
    if (ok) {
      double lo = 0.0, up = 0.0;
      int p = ptr[row], p1 = dpos[row];
      // batches of SYM16_FB: the mirror indices, then the products, are loaded before
      // the (in-order, so bit-identical) additions -- a batch of loads in flight, not 1
      for (; p + SYM16_FB <= p1; p += SYM16_FB) {
        int tp[SYM16_FB];
        double v[SYM16_FB];
#pragma unroll
        for (int u = 0; u < SYM16_FB; ++u) tp[u] = T_READ(p + u);
#pragma unroll
        for (int u = 0; u < SYM16_FB; ++u) v[u] = ld_pol(T + (int64_t)tp[u] * 16 + r, pt);
#pragma unroll
        for (int u = 0; u < SYM16_FB; ++u) lo += v[u];
      }
      for (; p < p1; ++p) lo += ld_pol(T + (int64_t)T_READ(p) * 16 + r, pt);
      for (int k = ucptr[row]; k < ucptr[row + 1]; ++k) up += yup[(int64_t)k * 16 + r];
      ax = lo + up;
    }
    int64_t e = (int64_t)(ok ? row : 0) * 16 + r;
    if (mode == 0) {
      if (ok) {
        out[e] = ax;
        if (dot_out) dsum = fma(x_in[e], ax, dsum);
      }
      continue;
    }
    double rr = ok ? b[e] - ax : 0.0;
    if (mode == 1) {
      if (ok) out[e] = rr;
      continue;
    }
    double z = 0.0;
    const double* Di = Dinv + ((int64_t)(ok ? row : 0) * 16 + r) * 16;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      double rc = __shfl_sync(FULL_MASK, rr, c, 16);
      if (ok) z = fma(Di[c], rc, z);
    }
    if (ok) {
      double dn = divide ? z / c2 : c1 * d[e] + c2 * z;
      d[e] = dn;
      out[e] = x_in[e] + dn;
    }
  }
  if (dot_out) {
    dsum = block_sum(dsum, scratch);
    grid_finish(partials, counter, dsum, scratch, dot_out);
  }
}

static int sym_grid(int nbr) { return grid_for((int64_t)nbr * 32, 128, 16); }

// operators whose upper half exceeds ~half of L2 are streamed evict_first, so the
// stream does not displace the resident mirrored products and the small operators
#ifndef SYM_STREAM_BYTES
#define SYM_STREAM_BYTES (64ll << 20)
#endif
static int sym_block_policy(const bamg_symop* S) {
  int64_t up_bytes = (S->nnzb + S->nbr) / 2 * (int64_t)S->bs * S->bs * 8;
  return up_bytes > SYM_STREAM_BYTES ? L2_FIRST : L2_NORMAL;
}

// y = A x through the symmetric operator (bs 9 or 16), with the chosen epilogue.
static void sym_apply(bamg_ctx* ctx, const bamg_symop* S, const double* blocks, const double* x, int mode,
                      const double* b, const double* Dinv, double* d, double* out, double c1, double c2, int divide,
                      double* dot_out, cudaStream_t st) {
  double* part = ctx ? ctx->partials : nullptr;
  unsigned* ctr = ctx ? ctx->counters + BAMG_CTR_SPMV : nullptr;
  if (S->bs == 16) {
    launch_pdl(k_sym16_upper, sym_grid(S->nch), 128, 0, st, S->ptr, S->col, S->dpos, (const int*)S->tpos,
           (const int*)S->cbeg,
           (const int*)S->crow, S->nch, blocks, x, S->T, S->yup, sym_block_policy(S));
    int g = grid_for((int64_t)((S->nbr + 1) / 2) * 32, 128, 16);
    if (dot_out && g > BAMG_MAX_PARTIALS) g = BAMG_MAX_PARTIALS;
    launch_pdl(k_sym16_finish, g, 128, 0, st, S->ptr, S->dpos, (const int*)S->tpos, (const double*)S->T,
           (const int*)S->ucptr, (const double*)S->yup, S->nbr, mode, b, Dinv, d, x, out, c1, c2, divide, part, ctr,
           dot_out);
    return;
  }
  launch_pdl(k_sym9_upper, sym_grid(S->nch), 128, 0, st, S->ptr, S->col, S->dpos, (const int*)S->tpos,
         (const int*)S->cbeg, (const int*)S->crow, S->nch, blocks, x, S->T, S->yup, sym_block_policy(S));
  // one row per warp (the hardware balances CTAs over SMs as rows finish); the
  // fused dot's grid is capped by the partials buffer and strides instead
  int g = (int)ceil_div(S->nbr, 4);
  if (dot_out && g > BAMG_MAX_PARTIALS) g = BAMG_MAX_PARTIALS;
  launch_pdl(k_sym9_finish<SYM_FB>, g, 128, 0, st, S->ptr, S->dpos, (const int*)S->tpos, (const double*)S->T, (const int*)S->ucptr,
         (const double*)S->yup, S->nbr, mode, b, Dinv, d, x, out, c1, c2, divide, part, ctr, dot_out);
}

// shared tail of both constructors: T, the chunk plan (one host readback)
static bamg_symop* symop_finish(bamg_symop* S, cudaStream_t st) {
  auto fail = [&](const char* what) -> bamg_symop* {
    bamg_set_error("symop_create: %s", what);
    bamg_symop_destroy(S);
    return nullptr;
  };
  size_t nn = (size_t)(S->nnzb > 0 ? S->nnzb : 1);
  int nbr = S->nbr;
  if (cudaMallocAsync(&S->T, sizeof(double) * S->bs * nn, st) != cudaSuccess ||
      cudaMallocAsync(&S->ucptr, sizeof(int) * ((size_t)nbr + 1), st) != cudaSuccess)
    return fail("allocation failed");
  if (nbr > 0) {
    launch(k_sym_chunk_counts, grid_for(nbr, 256), 256, 0, st, S->ptr, S->dpos, nbr, S->ch, S->ucptr);
    if (scan_exclusive_int(S->ucptr, S->ucptr, (int64_t)nbr + 1, nullptr, st)) return fail("chunk scan failed");
    if (cudaMemcpyAsync(&S->nch, S->ucptr + nbr, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return fail("chunk count readback failed");
  }
  size_t nc = (size_t)(S->nch > 0 ? S->nch : 1);
  if (cudaMallocAsync(&S->cbeg, sizeof(int) * nc, st) != cudaSuccess ||
      cudaMallocAsync(&S->crow, sizeof(int) * nc, st) != cudaSuccess ||
      cudaMallocAsync(&S->yup, sizeof(double) * S->bs * nc, st) != cudaSuccess)
    return fail("allocation failed");
  if (nbr > 0)
    launch(k_sym_chunk_fill, grid_for(nbr, 256), 256, 0, st, S->dpos, (const int*)S->ucptr, nbr, S->ch, S->cbeg,
           S->crow);
  return S;
}

extern "C" bamg_symop* bamg_symop_create(int32_t nbr, const int32_t* ptr, const int32_t* col, const int32_t* dpos,
                                         const int32_t* up_blk, const int32_t* up_tpos, int32_t n_up, int64_t nnzb,
                                         void* stream) {
  cudaStream_t st = as_stream(stream);
  bamg_symop* S = new bamg_symop();
  S->bs = 9;
  S->ch = SYM_CH;
  S->nbr = nbr;
  S->nnzb = nnzb;
  S->ptr = ptr;
  S->col = col;
  S->dpos = dpos;
  S->alloc_stream = st;
  if (cudaMallocAsync(&S->tpos, sizeof(int) * (size_t)(nnzb > 0 ? nnzb : 1), st) != cudaSuccess) {
    bamg_set_error("symop_create: allocation failed");
    bamg_symop_destroy(S);
    return nullptr;
  }
  if (n_up > 0) launch(k_sym_mirror, grid_for(n_up, 256), 256, 0, st, up_blk, up_tpos, n_up, S->tpos);
  return symop_finish(S, st);
}

extern "C" bamg_symop* bamg_symop_create_pattern(int32_t bs, int32_t nbr, const int32_t* ptr, const int32_t* col,
                                                 int64_t nnzb, void* stream) {
  if (bs != 9 && bs != 16) {
    bamg_set_error("symop_create_pattern: unsupported block size %d", bs);
    return nullptr;
  }
  cudaStream_t st = as_stream(stream);
  bamg_symop* S = new bamg_symop();
  S->bs = bs;
  S->ch = bs == 16 ? SYM_CH16 : SYM_CH;
  S->nbr = nbr;
  S->nnzb = nnzb;
  S->ptr = ptr;
  S->col = col;
  S->alloc_stream = st;
  if (cudaMallocAsync(&S->tpos, sizeof(int) * (size_t)(nnzb > 0 ? nnzb : 1), st) != cudaSuccess ||
      cudaMallocAsync(&S->dpos_own, sizeof(int) * (size_t)(nbr > 0 ? nbr : 1), st) != cudaSuccess) {
    bamg_set_error("symop_create_pattern: allocation failed");
    bamg_symop_destroy(S);
    return nullptr;
  }
  S->dpos = S->dpos_own;
  if (nbr > 0) launch(k_sym_pattern, grid_for((int64_t)nbr * 32, 128, 16), 128, 0, st, ptr, col, nbr, S->dpos_own, S->tpos);
  return symop_finish(S, st);
}

extern "C" void bamg_symop_destroy(bamg_symop* S) {
  if (!S) return;
  void* bufs[] = {S->tpos, S->dpos_own, S->T, S->ucptr, S->cbeg, S->crow, S->yup};
  for (void* b : bufs)
    if (b) cudaFreeAsync(b, S->alloc_stream);
  delete S;
}

extern "C" int32_t bamg_symop_chunks(const bamg_symop* S) { return S ? S->nch : 0; }

extern "C" int bamg_symop_spmv(bamg_ctx* ctx, const bamg_symop* S, const double* blocks, const double* x, double* y,
                               double* dot_out_dev, void* stream) {
  if (!S || S->nbr <= 0) return 0;
  sym_apply(ctx, S, blocks, x, 0, nullptr, nullptr, nullptr, y, 0.0, 0.0, 0, dot_out_dev, as_stream(stream));
  BAMG_LAUNCH_CHECK();
  return 0;
}

extern "C" int bamg_symop_residual(bamg_ctx* ctx, const bamg_symop* S, const double* blocks, const double* x,
                                   const double* b, double* r, void* stream) {
  if (!S || S->nbr <= 0) return 0;
  sym_apply(ctx, S, blocks, x, 1, b, nullptr, nullptr, r, 0.0, 0.0, 0, nullptr, as_stream(stream));
  BAMG_LAUNCH_CHECK();
  return 0;
}

extern "C" int bamg_symop_cheb_step(bamg_ctx* ctx, const bamg_symop* S, const double* blocks, const double* x_in,
                                    const double* b, const double* Dinv, double* d, double* x_out, double c1,
                                    double c2, int32_t divide, void* stream) {
  if (!S || S->nbr <= 0) return 0;
  sym_apply(ctx, S, blocks, x_in, 2, b, Dinv, d, x_out, c1, c2, divide, nullptr, as_stream(stream));
  BAMG_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------------------
// Chunked 16x16 SpMV for the coarse levels. Coarse rows are long (30-80 blocks)
// and few (1-4 K), so a warp per row leaves the SMs latency-bound. Instead every
// warp takes a chunk of <= CH consecutive blocks of ONE row and writes a 16-entry
// partial; a second kernel sums a row's partials in chunk order (deterministic)
// and applies the residual or the fused Chebyshev update.

__device__ __forceinline__ double warp_blocks16(const int* __restrict__ col, const double* __restrict__ blocks,
                                                const double* __restrict__ x, int b, int b1, int lane) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  const int cp = 2 * (lane & 7);
  for (; b + 1 < b1; b += 2) {
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
  int src = 8 * (lane & 3);
  double s0 = __shfl_sync(FULL_MASK, a0, src);
  double s1 = __shfl_sync(FULL_MASK, a1, src);
  double s2 = __shfl_sync(FULL_MASK, a2, src);
  double s3 = __shfl_sync(FULL_MASK, a3, src);
  int k = (lane >> 2) & 3;
  return k == 0 ? s0 : (k == 1 ? s1 : (k == 2 ? s2 : s3));
}

__global__ void __launch_bounds__(128)
k_spmv16_chunks(const int* __restrict__ ptr, const int* __restrict__ col, const double* __restrict__ blocks,
                const double* __restrict__ x, const int* __restrict__ cbeg, const int* __restrict__ crow, int nch,
                int CH, double* __restrict__ partial) {
  PDL_ENTRY();
  int lane = threadIdx.x & 31;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int c = warp; c < nch; c += nwarps) {
    int b0 = cbeg[c];
    int b1 = min(b0 + CH, ptr[crow[c] + 1]);
    double v = warp_blocks16(col, blocks, x, b0, b1, lane);
    if (lane < 16) partial[(int64_t)c * 16 + lane] = v;
  }
}

// Single-pass 16x16 product for the small coarse operators (full storage; every
// level below ROWCTA_MAX_BYTES): CTA per row, warp w takes the w-th quarter of the
// row's blocks, the four partials combine in warp order, and the epilogue of
// k_rows16_finish follows in the same kernel -- one launch per product instead of
// the half-storage pair, whose two latency-bound launches dominate at these sizes.
#ifndef ROWCTA_MAX_BYTES
#define ROWCTA_MAX_BYTES (32ll << 20)
#endif
__global__ void __launch_bounds__(128)
k_row16_cta(const int* __restrict__ ptr, const int* __restrict__ col, const double* __restrict__ blocks,
            const double* __restrict__ x, int nbr, int mode, const double* __restrict__ b,
            const double* __restrict__ Dinv, double* __restrict__ d, double* __restrict__ out, double c1, double c2,
            int divide) {
  PDL_ENTRY();
  __shared__ double part[4][16];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int row = blockIdx.x;
  int b0 = ptr[row], b1 = ptr[row + 1];
  int q = (b1 - b0 + 3) >> 2;
  int lo = min(b0 + w * q, b1), hi = min(lo + q, b1);
  double v = warp_blocks16(col, blocks, x, lo, hi, lane);
  if (lane < 16) part[w][lane] = v;
  __syncthreads();
  if (w != 0) return;
  int r = lane & 15;
  double ax = ((part[0][r] + part[1][r]) + part[2][r]) + part[3][r];
  int64_t e = (int64_t)row * 16 + r;
  double rr = b[e] - ax;
  if (mode == 0) {
    if (lane < 16) out[e] = rr;
    return;
  }
  double z = 0.0;
  const double* Di = Dinv + e * 16;
#pragma unroll
  for (int c = 0; c < 16; ++c) z = fma(Di[c], __shfl_sync(FULL_MASK, rr, c, 16), z);
  if (lane < 16) {
    double dn = divide ? z / c2 : c1 * d[e] + c2 * z;
    d[e] = dn;
    out[e] = x[e] + dn;
  }
}

// Row finish: ax = sum of the row's partials (chunk order); then
//   mode 0: r = b - ax
//   mode 1: fused Chebyshev step (as k_cheb_step): r = b - ax; z = D^-1 r;
//           d = divide ? z / c2 : c1 d + c2 z; x_out = x_in + d
__global__ void __launch_bounds__(128)
k_rows16_finish(const int* __restrict__ cptr, const double* __restrict__ partial, int nbr, int mode,
                const double* __restrict__ b, const double* __restrict__ Dinv, double* __restrict__ d,
                const double* __restrict__ x_in, double* __restrict__ out, double c1, double c2, int divide) {
  PDL_ENTRY();
  int lane = threadIdx.x & 31;
  int half = lane >> 4, r = lane & 15;
  int row0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 2;
  int stride = ((gridDim.x * blockDim.x) >> 5) * 2;
  for (int base = row0; base < nbr; base += stride) {
    int row = base + half;
    bool ok = row < nbr;
    double ax = 0.0;
    if (ok)
      for (int c = cptr[row]; c < cptr[row + 1]; ++c) ax += partial[(int64_t)c * 16 + r];
    int64_t e = (int64_t)row * 16 + r;
    double rr = ok ? b[e] - ax : 0.0;
    if (mode == 0) {
      if (ok) out[e] = rr;
      continue;
    }
    double z = 0.0;
    const double* Di = Dinv + ((int64_t)(ok ? row : 0) * 16 + r) * 16;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      double rc = __shfl_sync(FULL_MASK, rr, c, 16);
      if (ok) z = fma(Di[c], rc, z);
    }
    if (ok) {
      double dn = divide ? z / c2 : c1 * d[e] + c2 * z;
      d[e] = dn;
      out[e] = x_in[e] + dn;
    }
  }
}

// warp per aggregate restriction: bc_a = sum_{i in a} P_i^T r_i. Half-warp h takes
// members h, h + 2, ...; lane c of a half owns column c and sums the BS rows of each
// member's block (per row k the 16 lanes read one coalesced 128 B row of P; r_i is a
// broadcast). Two members per half are loaded before their fma chains, so 4 members'
// loads are in flight per warp; the halves combine once at the end (fixed order).
// (min-blocks 1: without it ptxas holds the kernel at 32 registers and interleaves
// every load with its fma, one member's row in flight at a time)
// CHEB: the coarse level's first smoothing step (x = 0: d = D^-1 b / theta, x = d,
// k_cheb_step without the product) in the same warp, on the 16 values it just formed
// -- one launch per level less, same arithmetic.
template <int BS, bool CHEB = false>
__global__ void __launch_bounds__(128, 1)
k_restrict_warp(const int* __restrict__ agg_ptr, const int* __restrict__ members, const double* __restrict__ P,
                const double* __restrict__ r, int nagg, double* __restrict__ bc, const double* __restrict__ Dinv = nullptr,
                double* __restrict__ dc = nullptr, double* __restrict__ xc = nullptr, double theta = 1.0) {
  PDL_ENTRY();
  int lane = threadIdx.x & 31;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  int c = lane & 15, h = lane >> 4;
  for (int a = warp; a < nagg; a += nwarps) {
    int q = agg_ptr[a] + h, q1 = agg_ptr[a + 1];
    double s = 0.0;
    for (; q + 2 < q1; q += 4) {
      int64_t i0 = __ldg(members + q), i1 = __ldg(members + q + 2);
      double u0[BS], u1[BS], r0[BS], r1[BS];
#pragma unroll
      for (int k = 0; k < BS; ++k) {
        u0[k] = __ldg(P + (i0 * BS + k) * 16 + c);
        u1[k] = __ldg(P + (i1 * BS + k) * 16 + c);
        r0[k] = __ldg(r + i0 * BS + k);
        r1[k] = __ldg(r + i1 * BS + k);
      }
#pragma unroll
      for (int k = 0; k < BS; ++k) s = fma(u0[k], r0[k], s);
#pragma unroll
      for (int k = 0; k < BS; ++k) s = fma(u1[k], r1[k], s);
    }
    if (q < q1) {
      int64_t i0 = __ldg(members + q);
      double u0[BS], r0[BS];
#pragma unroll
      for (int k = 0; k < BS; ++k) {
        u0[k] = __ldg(P + (i0 * BS + k) * 16 + c);
        r0[k] = __ldg(r + i0 * BS + k);
      }
#pragma unroll
      for (int k = 0; k < BS; ++k) s = fma(u0[k], r0[k], s);
    }
    s += __shfl_down_sync(FULL_MASK, s, 16);
    if (lane < 16) bc[(int64_t)a * 16 + c] = s;
    if constexpr (CHEB) {
      double rr = lane < 16 ? s : 0.0;
      double z = 0.0;
      const double* Di = Dinv + (int64_t)a * 256 + (lane < 16 ? lane : 0) * 16;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        double rk = __shfl_sync(FULL_MASK, rr, k);
        if (lane < 16) z = fma(Di[k], rk, z);
      }
      if (lane < 16) {
        double dn = z / theta;
        dc[(int64_t)a * 16 + lane] = dn;
        xc[(int64_t)a * 16 + lane] = 0.0 + dn;
      }
    }
  }
}

// chunk metadata: counts per row, then fill
__global__ void k_chunk_counts(const int* __restrict__ ptr, int nbr, int CH, int* __restrict__ cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nbr; i += gridDim.x * blockDim.x) {
    int len = ptr[i + 1] - ptr[i];
    cnt[i] = (len + CH - 1) / CH;
  }
}

__global__ void k_chunk_fill(const int* __restrict__ ptr, const int* __restrict__ cptr, int nbr, int CH,
                             int* __restrict__ cbeg, int* __restrict__ crow) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nbr; i += gridDim.x * blockDim.x)
    for (int c = cptr[i]; c < cptr[i + 1]; ++c) {
      cbeg[c] = ptr[i] + (c - cptr[i]) * CH;
      crow[c] = i;
    }
}

// ---------------------------------------------------------------------------
// Coarse V-cycle tail as ONE persistent kernel. Below some level every operator is
// small (tens of MB or less): its products, Jacobi steps, restriction, prolongation
// and the coarsest dense solve are each a few microseconds of work behind a
// dependent launch. The plan records those steps as a list of ops once (the same
// recursion that launches them, in recording mode) and replays the list inside one
// cooperative grid, a grid-wide barrier between consecutive ops. Each op computes
// exactly what its kernel computes (same row partition and summation order), so the
// result is bit-identical to the launched form. Vectors written inside the kernel are
// read with ld.global.cg (L2, not the incoherent L1 / read-only paths).
#include <cooperative_groups.h>

enum { TOP_CHEB = 0, TOP_ROW = 1, TOP_RESTRICT = 2, TOP_PROLONG = 3, TOP_GEMV = 4 };

struct TailOp {
  int type = 0, nbr = 0, mode = 0, divide = 0;
  const int* ptr = nullptr;
  const int* col = nullptr;
  const double* blocks = nullptr;
  const double* x = nullptr;  // product / update input (CHEB: may be null)
  const double* b = nullptr;
  const double* Dinv = nullptr;
  double* d = nullptr;
  double* out = nullptr;
  double c1 = 0.0, c2 = 0.0;
  const int* agg_ptr = nullptr;
  const int* members = nullptr;
  const double* P = nullptr;
  const int* agg = nullptr;
  int n_agg = 0, n = 0, bs = 16, pad = 0;
  const double* inv = nullptr;
};

__device__ __forceinline__ double tail_blocks16(const int* __restrict__ col, const double* __restrict__ blocks,
                                                const double* x, int b, int b1, int lane) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  const int cp = 2 * (lane & 7);
  for (; b + 1 < b1; b += 2) {
    const double2* A0 = reinterpret_cast<const double2*>(blocks + (int64_t)b * 256) + lane;
    const double2* A1 = reinterpret_cast<const double2*>(blocks + (int64_t)(b + 1) * 256) + lane;
    double2 u0 = __ldg(A0), u1 = __ldg(A0 + 32), u2 = __ldg(A0 + 64), u3 = __ldg(A0 + 96);
    double2 v0 = __ldg(A1), v1 = __ldg(A1 + 32), v2 = __ldg(A1 + 64), v3 = __ldg(A1 + 96);
    double2 xa = __ldcg(reinterpret_cast<const double2*>(x + (int64_t)__ldg(col + b) * 16 + cp));
    double2 xb = __ldcg(reinterpret_cast<const double2*>(x + (int64_t)__ldg(col + b + 1) * 16 + cp));
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
    double2 xa = __ldcg(reinterpret_cast<const double2*>(x + (int64_t)__ldg(col + b) * 16 + cp));
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
  int src = 8 * (lane & 3);
  double s0 = __shfl_sync(FULL_MASK, a0, src);
  double s1 = __shfl_sync(FULL_MASK, a1, src);
  double s2 = __shfl_sync(FULL_MASK, a2, src);
  double s3 = __shfl_sync(FULL_MASK, a3, src);
  int k = (lane >> 2) & 3;
  return k == 0 ? s0 : (k == 1 ? s1 : (k == 2 ? s2 : s3));
}

// 4-warp group barrier (named barrier 1 + group; barrier 0 stays __syncthreads)
__device__ __forceinline__ void group_sync(int grp) {
  asm volatile("bar.sync %0, 128;" ::"r"(grp + 1) : "memory");
}

// k_row16_cta's row, cooperative over a group of 4 warps (a 128-thread CTA, or one
// of the 4-warp groups of a larger CTA: same partition, same summation order)
__device__ __forceinline__ void tail_row16(const TailOp& o, int row, double (*part)[16], int lane, int w, int grp) {
  int b0 = __ldg(o.ptr + row), b1 = __ldg(o.ptr + row + 1);
  int q = (b1 - b0 + 3) >> 2;
  int lo = min(b0 + w * q, b1), hi = min(lo + q, b1);
  double v = tail_blocks16(o.col, o.blocks, o.x, lo, hi, lane);
  if (lane < 16) part[w][lane] = v;
  group_sync(grp);
  if (w == 0) {
    int r = lane & 15;
    double ax = ((part[0][r] + part[1][r]) + part[2][r]) + part[3][r];
    int64_t e = (int64_t)row * 16 + r;
    double rr = __ldcg(o.b + e) - ax;
    if (o.mode == 0) {
      if (lane < 16) o.out[e] = rr;
    } else {
      double z = 0.0;
      const double* Di = o.Dinv + e * 16;
#pragma unroll
      for (int c = 0; c < 16; ++c) z = fma(__ldg(Di + c), __shfl_sync(FULL_MASK, rr, c, 16), z);
      if (lane < 16) {
        double dn = o.divide ? z / o.c2 : o.c1 * __ldcg(o.d + e) + o.c2 * z;
        o.d[e] = dn;
        o.out[e] = __ldcg(o.x + e) + dn;
      }
    }
  }
  group_sync(grp);
}

// CLUSTER = false: one cooperative grid (128-thread CTAs, grid-wide barrier);
// CLUSTER = true: ONE thread-block cluster of up to 16 CTAs of 512 threads (4-warp
// row groups), cluster barrier between ops -- the coarse levels' data are a few MB,
// read from L2 by 16 SMs at a fraction of a grid barrier's cost.
template <bool CLUSTER>
__global__ void __launch_bounds__(CLUSTER ? 512 : 128) k_vcycle_tail(const TailOp* __restrict__ ops, int nops) {
  namespace cg = cooperative_groups;
  __shared__ double part_all[CLUSTER ? 16 : 4][16];
  const int lane = threadIdx.x & 31, wt = threadIdx.x >> 5, w = wt & 3, grp = wt >> 2;
  const int ngrp = blockDim.x >> 7;
  double(*part)[16] = part_all + 4 * grp;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int k = 0; k < nops; ++k) {
    const TailOp o = ops[k];
    switch (o.type) {
      case TOP_ROW:
        for (int row = blockIdx.x * ngrp + grp; row < o.nbr; row += gridDim.x * ngrp)
          tail_row16(o, row, part, lane, w, grp);
        break;
      case TOP_CHEB:  // k_cheb_step<16> without the product (x_in null)
        for (int row = gwarp; row < o.nbr; row += nwarps) {
          int64_t base = (int64_t)row * 16;
          double rr = (lane < 16) ? __ldcg(o.b + base + lane) : 0.0;
          double z = 0.0;
          const double* Di = o.Dinv + (int64_t)row * 256 + (lane < 16 ? lane : 0) * 16;
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            double rc = __shfl_sync(FULL_MASK, rr, c);
            if (lane < 16) z = fma(__ldg(Di + c), rc, z);
          }
          if (lane < 16) {
            double dn = o.divide ? z / o.c2 : o.c1 * __ldcg(o.d + base + lane) + o.c2 * z;
            o.d[base + lane] = dn;
            o.out[base + lane] = (o.x ? __ldcg(o.x + base + lane) : 0.0) + dn;
          }
        }
        break;
      case TOP_RESTRICT: {  // k_restrict_warp<16>
        int c = lane & 15, h = lane >> 4;
        for (int a = gwarp; a < o.n_agg; a += nwarps) {
          int q = __ldg(o.agg_ptr + a) + h, q1 = __ldg(o.agg_ptr + a + 1);
          double s = 0.0;
          for (; q + 2 < q1; q += 4) {
            int64_t i0 = __ldg(o.members + q), i1 = __ldg(o.members + q + 2);
            double u0[16], u1[16], r0[16], r1[16];
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) {
              u0[kk] = __ldg(o.P + (i0 * 16 + kk) * 16 + c);
              u1[kk] = __ldg(o.P + (i1 * 16 + kk) * 16 + c);
              r0[kk] = __ldcg(o.x + i0 * 16 + kk);
              r1[kk] = __ldcg(o.x + i1 * 16 + kk);
            }
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) s = fma(u0[kk], r0[kk], s);
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) s = fma(u1[kk], r1[kk], s);
          }
          if (q < q1) {
            int64_t i0 = __ldg(o.members + q);
            double u0[16], r0[16];
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) {
              u0[kk] = __ldg(o.P + (i0 * 16 + kk) * 16 + c);
              r0[kk] = __ldcg(o.x + i0 * 16 + kk);
            }
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) s = fma(u0[kk], r0[kk], s);
          }
          s += __shfl_down_sync(FULL_MASK, s, 16);
          if (lane < 16) o.out[(int64_t)a * 16 + c] = s;
        }
        break;
      }
      case TOP_PROLONG: {  // k_prolong, accumulate
        int64_t tot = (int64_t)o.nbr * o.bs;
        for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
             t += (int64_t)gridDim.x * blockDim.x) {
          int64_t i = t / o.bs;
          int r = (int)(t - i * o.bs);
          const double2* pp = reinterpret_cast<const double2*>(o.P + (i * o.bs + r) * 16);
          const double2* xa = reinterpret_cast<const double2*>(o.x + (int64_t)__ldg(o.agg + i) * 16);
          double2 pv[8], xv[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            pv[c] = __ldg(pp + c);
            xv[c] = __ldcg(xa + c);
          }
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < 8; ++c) s = fma(pv[c].y, xv[c].y, fma(pv[c].x, xv[c].x, s));
          o.out[t] = __ldcg(o.out + t) + s;
        }
        break;
      }
      case TOP_GEMV:  // k_gemv
        for (int i = gwarp; i < o.n; i += nwarps) {
          double s = 0.0;
          for (int c = lane; c < o.n; c += 32) s = fma(__ldg(o.inv + (int64_t)i * o.n + c), __ldcg(o.b + c), s);
          s = warp_sum(s);
          if (lane == 0) o.out[i] = s;
        }
        break;
    }
    if (k + 1 < nops) {
      if constexpr (CLUSTER) cg::this_cluster().sync();
      else cg::this_grid().sync();
    }
  }
}

// ---------------------------------------------------------------------------
// MG plan

struct MgLevelPlan {
  int bs = 0, nbr = 0, n = 0;
  // chunked 16x16 SpMV (coarse levels)
  int CH = 0, nch = 0;
  int *cptr = nullptr, *cbeg = nullptr, *crow = nullptr;
  double* partial = nullptr;
  const int* ptr = nullptr;
  const int* col = nullptr;
  const double* blocks = nullptr;
  const double* Dinv = nullptr;
  double theta = 0, delta = 0, sigma = 0;
  int iterations = 2;
  // to the next level
  const double* P = nullptr;
  const int* agg = nullptr;
  const int* agg_ptr = nullptr;
  const int* members = nullptr;
  int n_agg = 0;
  // coarsest
  const double* inv = nullptr;
  // symmetric half-storage operator (bs 9), when set
  const bamg_symop* sym = nullptr;
  // single-pass CTA-per-row products (small 16x16 levels)
  bool rowcta = false;
  // work
  double *b = nullptr, *x = nullptr, *xs = nullptr, *d = nullptr, *r = nullptr;
  // set while the plan records the coarse tail: steps are appended, not launched
  std::vector<TailOp>* rec = nullptr;
};

struct bamg_mg {
  std::vector<MgLevelPlan> lv;
  double* in = nullptr;     // level-0 right-hand side (plan-owned)
  double* out = nullptr;    // level-0 result (plan-owned)
  double* arena = nullptr;  // every work vector, one stream-ordered allocation
  cudaStream_t arena_stream = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  bool dirty = true;
  bool use_graph = false;
  long long graph_kernels = 0;
  // coarse tail (levels >= tail_from) as one persistent kernel
  int tail_mb = -1;  // size cap per level operator (MB); -1: BAMG_VTAIL_MB / default
  int tail_from = -1;
  bool tail_recording = false;
  std::vector<TailOp> tail_host;
  TailOp* tail_ops = nullptr;
  double* tail_result = nullptr;
  int tail_grid = 0;
  bool tail_cluster = true;
};

extern "C" bamg_mg* bamg_mg_create(int32_t n_levels) {
  bamg_mg* m = new bamg_mg();
  m->lv.resize(n_levels);
  return m;
}

// One instantiated V-cycle graph outlives its plan: the next hierarchy (the next LM
// step's, usually with the same levels and kernel kinds) captures its own graph and
// re-targets the parked executable with cudaGraphExecUpdate instead of paying a
// full instantiation (~1 ms of host time for ~60 nodes). Updates affect only later
// launches, so a parked executable may still be in flight.
static std::mutex g_exec_mu;
static cudaGraphExec_t g_parked_exec = nullptr;

static void park_exec(cudaGraphExec_t e) {
  if (!e) return;
  std::lock_guard<std::mutex> lk(g_exec_mu);
  if (g_parked_exec) cudaGraphExecDestroy(g_parked_exec);
  g_parked_exec = e;
}

static cudaGraphExec_t take_parked_exec() {
  std::lock_guard<std::mutex> lk(g_exec_mu);
  cudaGraphExec_t e = g_parked_exec;
  g_parked_exec = nullptr;
  return e;
}

static void mg_free_work(bamg_mg* m) {
  if (m->arena) cudaFreeAsync(m->arena, m->arena_stream);
  m->arena = nullptr;
  if (m->tail_ops) cudaFreeAsync(m->tail_ops, m->arena_stream);
  m->tail_ops = nullptr;
  m->tail_from = -1;
  m->tail_host.clear();
  m->tail_result = nullptr;
  for (auto& L : m->lv) L.b = L.x = L.xs = L.d = L.r = nullptr;
  m->in = m->out = nullptr;
  if (m->exec) park_exec(m->exec);
  if (m->graph) cudaGraphDestroy(m->graph);
  m->exec = nullptr;
  m->graph = nullptr;
}

extern "C" void bamg_mg_destroy(bamg_mg* m) {
  if (!m) return;
  mg_free_work(m);
  delete m;
}

extern "C" int bamg_mg_set_level(bamg_mg* m, int32_t level, int32_t bs, int32_t nbr, const int32_t* ptr,
                                 const int32_t* col, const double* blocks, const double* Dinv, double lower,
                                 double upper, int32_t iterations, const double* P, const int32_t* agg,
                                 const int32_t* agg_ptr, const int32_t* members, int32_t n_agg,
                                 const double* coarse_inv) {
  if (level < 0 || level >= (int)m->lv.size()) {
    bamg_set_error("mg_set_level: level %d out of range", level);
    return BAMG_ERR_UNSUPPORTED;
  }
  if (!coarse_inv && bs != 9 && bs != 16 && bs != 1) {
    bamg_set_error("mg_set_level: unsupported block size %d", bs);
    return BAMG_ERR_UNSUPPORTED;
  }
  MgLevelPlan& L = m->lv[level];
  L.bs = bs;
  L.nbr = nbr;
  L.n = nbr * bs;
  L.ptr = ptr;
  L.col = col;
  L.blocks = blocks;
  L.Dinv = Dinv;
  L.theta = 0.5 * (upper + lower);
  L.delta = 0.5 * (upper - lower);
  L.sigma = L.theta / L.delta;
  L.iterations = iterations;
  L.P = P;
  L.agg = agg;
  L.agg_ptr = agg_ptr;
  L.members = members;
  L.n_agg = n_agg;
  L.inv = coarse_inv;
  m->dirty = true;
  return 0;
}

int scan_exclusive_int(const int* in, int* out, int64_t n, int* total, cudaStream_t st);
static int mg_plan_tail(bamg_mg* m, const std::vector<int>& nnzb, cudaStream_t st);

static int mg_alloc(bamg_mg* m, cudaStream_t st) {
  mg_free_work(m);
  // chunk plan of the 16x16 smoothing levels: CH blocks per warp, enough chunks
  // to cover the SMs several times over
  // block counts: known on the host through a level's symmetric view; read back
  // (one synchronisation) only for levels without one
  std::vector<int> nnzb(m->lv.size(), 0);
  bool need_sync = false;
  for (size_t l = 0; l < m->lv.size(); ++l) {
    MgLevelPlan& L = m->lv[l];
    L.CH = 0;
    L.nch = 0;
    if (L.inv || L.bs != 16 || !L.ptr) continue;
    if (L.sym) {
      nnzb[l] = (int)L.sym->nnzb;
    } else {
      BAMG_CUDA_CHECK(cudaMemcpyAsync(&nnzb[l], L.ptr + L.nbr, sizeof(int), cudaMemcpyDeviceToHost, st));
      need_sync = true;
    }
  }
  if (need_sync) BAMG_CUDA_CHECK(cudaStreamSynchronize(st));
  for (size_t l = 0; l < m->lv.size(); ++l) {
    MgLevelPlan& L = m->lv[l];
    L.rowcta = !L.inv && L.bs == 16 && L.ptr && L.nbr > 0 && (int64_t)nnzb[l] * 2048 <= ROWCTA_MAX_BYTES;
  }
  size_t total = 2 * (size_t)m->lv[0].n;
  size_t itotal = 0;
  for (size_t l = 0; l < m->lv.size(); ++l) {
    MgLevelPlan& L = m->lv[l];
    total += 5 * (size_t)(L.n > 0 ? L.n : 1);
    // chunked full-storage products only where neither the half-storage pair nor
    // the row-CTA kernel runs the level
    if (L.inv || L.bs != 16 || !L.ptr || L.sym || L.rowcta) continue;
    int CH = nnzb[l] / 8192;
    L.CH = CH < 1 ? 1 : (CH > 8 ? 8 : CH);
    itotal += (size_t)L.nbr + 1;
  }
  // chunk counts need a scan before the arrays can be sized: count on the device
  int* counts = nullptr;
  if (itotal) BAMG_CUDA_CHECK(cudaMallocAsync(&counts, sizeof(int) * itotal, st));
  {
    size_t off = 0;
    std::vector<int> nch(m->lv.size(), 0);
    bool any = false;
    for (size_t l = 0; l < m->lv.size(); ++l) {
      MgLevelPlan& L = m->lv[l];
      if (!L.CH) continue;
      launch(k_chunk_counts, grid_for(L.nbr, 256), 256, 0, st, L.ptr, L.nbr, L.CH, counts + off);
      int rc = scan_exclusive_int(counts + off, counts + off, L.nbr + 1, nullptr, st);
      if (rc) return rc;
      BAMG_CUDA_CHECK(cudaMemcpyAsync(&nch[l], counts + off + L.nbr, sizeof(int), cudaMemcpyDeviceToHost, st));
      off += (size_t)L.nbr + 1;
      any = true;
    }
    if (any) BAMG_CUDA_CHECK(cudaStreamSynchronize(st));
    for (size_t l = 0; l < m->lv.size(); ++l) {
      m->lv[l].nch = nch[l];
      if (m->lv[l].CH) {
        itotal += 2 * (size_t)nch[l];
        total += 16 * (size_t)nch[l];
      }
    }
  }
  total += (itotal + 1) / 2 + 1;  // ints live at the end of the arena
  BAMG_CUDA_CHECK(cudaMallocAsync(&m->arena, sizeof(double) * total, st));
  {
    double* pd = m->arena + 2 * (size_t)m->lv[0].n;
    for (auto& L : m->lv) pd += 5 * (size_t)(L.n > 0 ? L.n : 1);
    for (auto& L : m->lv)
      if (L.CH) {
        L.partial = pd;
        pd += 16 * (size_t)L.nch;
      }
    int* pi = reinterpret_cast<int*>(pd);
    size_t off = 0;
    for (auto& L : m->lv) {
      if (!L.CH) continue;
      L.cptr = pi;
      pi += L.nbr + 1;
      BAMG_CUDA_CHECK(cudaMemcpyAsync(L.cptr, counts + off, sizeof(int) * (L.nbr + 1), cudaMemcpyDeviceToDevice, st));
      off += (size_t)L.nbr + 1;
      L.cbeg = pi;
      pi += L.nch;
      L.crow = pi;
      pi += L.nch;
      launch(k_chunk_fill, grid_for(L.nbr, 256), 256, 0, st, L.ptr, L.cptr, L.nbr, L.CH, L.cbeg, L.crow);
    }
  }
  if (counts) BAMG_CUDA_CHECK(cudaFreeAsync(counts, st));
  m->arena_stream = st;
  double* p = m->arena;
  m->in = p;
  p += m->lv[0].n;
  m->out = p;
  p += m->lv[0].n;
  for (size_t l = 0; l < m->lv.size(); ++l) {
    MgLevelPlan& L = m->lv[l];
    size_t n = (size_t)(L.n > 0 ? L.n : 1);
    if (l == 0) L.b = m->in;
    else { L.b = p; p += n; }
    L.x = p; p += n;
    L.xs = p; p += n;
    L.d = p; p += n;
    L.r = p; p += n;
  }
  return mg_plan_tail(m, nnzb, st);
}

template <int BS>
static void cheb_launch(const MgLevelPlan& L, const double* x_in, double* x_out, double c1, double c2, int divide,
                        bool with_A, cudaStream_t st) {
  launch_pdl(k_cheb_step<BS>, spmv_grid(L.nbr), 128, 0, st, L.ptr, L.col, with_A ? L.blocks : nullptr, x_in, L.b, L.Dinv,
         L.d, x_out, L.nbr, c1, c2, divide);
}

static void chunk_spmv(const MgLevelPlan& L, const double* x, cudaStream_t st) {
  launch_pdl(k_spmv16_chunks, grid_for((int64_t)L.nch * 32, 128, 16), 128, 0, st, L.ptr, L.col, L.blocks, x, L.cbeg,
         L.crow, L.nch, L.CH, L.partial);
}

static int finish_grid(int nbr) { return grid_for((int64_t)((nbr + 1) / 2) * 32, 128, 16); }

static void cheb(const MgLevelPlan& L, const double* x_in, double* x_out, double c1, double c2, int divide,
                 bool with_A, cudaStream_t st) {
  if (L.rec) {
    TailOp o;
    o.type = with_A ? TOP_ROW : TOP_CHEB;
    o.mode = 1;
    o.nbr = L.nbr;
    o.ptr = L.ptr;
    o.col = L.col;
    o.blocks = L.blocks;
    o.x = x_in;
    o.b = L.b;
    o.Dinv = L.Dinv;
    o.d = L.d;
    o.out = x_out;
    o.c1 = c1;
    o.c2 = c2;
    o.divide = divide;
    L.rec->push_back(o);
    return;
  }
  if (with_A && L.rowcta) {
    launch_pdl(k_row16_cta, L.nbr, 128, 0, st, L.ptr, L.col, L.blocks, x_in, L.nbr, 1, L.b, L.Dinv, L.d, x_out, c1, c2,
           divide);
    return;
  }
  if (with_A && L.sym) {
    sym_apply(nullptr, L.sym, L.blocks, x_in, 2, L.b, L.Dinv, L.d, x_out, c1, c2, divide, nullptr, st);
    return;
  }
  if (with_A && L.CH) {
    chunk_spmv(L, x_in, st);
    launch_pdl(k_rows16_finish, finish_grid(L.nbr), 128, 0, st, L.cptr, L.partial, L.nbr, 1, L.b, L.Dinv, L.d, x_in,
           x_out, c1, c2, divide);
    return;
  }
  switch (L.bs) {
    case 9: cheb_launch<9>(L, x_in, x_out, c1, c2, divide, with_A, st); break;
    case 16: cheb_launch<16>(L, x_in, x_out, c1, c2, divide, with_A, st); break;
    default: cheb_launch<1>(L, x_in, x_out, c1, c2, divide, with_A, st); break;
  }
}

// Smoother (multigrid.py:308-328); returns the buffer holding the result.
// `final_out` (optional): the buffer the last step writes (the plan's output vector,
// so no copy follows the cycle).
static double* smooth(MgLevelPlan& L, double* x, cudaStream_t st, double* final_out = nullptr,
                      bool first_done = false) {
  double rho = 1.0 / L.sigma;
  double* cur;
  double* spare;
  const bool one = L.iterations <= 1 && final_out;
  if (x == nullptr) {
    double* out = one ? final_out : L.x;
    if (!first_done) cheb(L, nullptr, out, 0.0, L.theta, 1, false, st);  // d = D^-1 b / theta ; x = d
    cur = out;
    spare = L.xs;
  } else {
    double* out = one ? final_out : ((x == L.x) ? L.xs : L.x);
    cheb(L, x, out, 0.0, L.theta, 1, true, st);  // r = b - A x ; d = D^-1 r / theta ; x += d
    cur = out;
    spare = x;
  }
  for (int it = 0; it < L.iterations - 1; ++it) {
    double rho_next = 1.0 / (2.0 * L.sigma - rho);
    if (final_out && it == L.iterations - 2) spare = final_out;
    cheb(L, cur, spare, rho_next * rho, 2.0 * rho_next / L.delta, 0, true, st);
    double* t = cur;
    cur = spare;
    spare = t;
    rho = rho_next;
  }
  return cur;
}

static void residual(const MgLevelPlan& L, const double* x, cudaStream_t st) {
  if (L.rec) {
    TailOp o;
    o.type = TOP_ROW;
    o.mode = 0;
    o.nbr = L.nbr;
    o.ptr = L.ptr;
    o.col = L.col;
    o.blocks = L.blocks;
    o.x = x;
    o.b = L.b;
    o.out = L.r;
    L.rec->push_back(o);
    return;
  }
  if (L.rowcta) {
    launch_pdl(k_row16_cta, L.nbr, 128, 0, st, L.ptr, L.col, L.blocks, x, L.nbr, 0, L.b, nullptr, nullptr, L.r, 0.0, 0.0,
           0);
    return;
  }
  if (L.sym) {
    sym_apply(nullptr, L.sym, L.blocks, x, 1, L.b, nullptr, nullptr, L.r, 0.0, 0.0, 0, nullptr, st);
    return;
  }
  if (L.CH) {
    chunk_spmv(L, x, st);
    launch_pdl(k_rows16_finish, finish_grid(L.nbr), 128, 0, st, L.cptr, L.partial, L.nbr, 0, L.b, nullptr, nullptr,
           nullptr, L.r, 0.0, 0.0, 0);
    return;
  }
  int g = spmv_grid(L.nbr);
  switch (L.bs) {
    case 9: launch_pdl(k_bsr_residual<9>, g, 128, 0, st, L.ptr, L.col, L.blocks, x, L.b, L.r, L.nbr); break;
    case 16: launch_pdl(k_bsr_residual<16>, g, 128, 0, st, L.ptr, L.col, L.blocks, x, L.b, L.r, L.nbr); break;
    default: launch_pdl(k_bsr_residual<1>, g, 128, 0, st, L.ptr, L.col, L.blocks, x, L.b, L.r, L.nbr); break;
  }
}

// V-cycle at level l from x = 0; returns the buffer holding x_l.
static double* vcycle(bamg_mg* m, size_t l, cudaStream_t st, bool first_done = false) {
  MgLevelPlan& L = m->lv[l];
  if ((int)l == m->tail_from && !m->tail_recording) {
    // the recorded coarse tail: one cooperative launch (no PDL edge: every CTA must be
    // resident at once)
    g_bamg_launches.fetch_add(1, std::memory_order_relaxed);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(m->tail_grid);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    if (m->tail_cluster) {
      cfg.blockDim = dim3(512);
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = m->tail_grid;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
    } else {
      cfg.blockDim = dim3(128);
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
    }
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (m->tail_cluster)
      cudaLaunchKernelEx(&cfg, k_vcycle_tail<true>, (const TailOp*)m->tail_ops, (int)m->tail_host.size());
    else
      cudaLaunchKernelEx(&cfg, k_vcycle_tail<false>, (const TailOp*)m->tail_ops, (int)m->tail_host.size());
    return m->tail_result;
  }
  if (L.inv) {
    double* out = l == 0 ? m->out : L.x;
    if (L.rec) {
      TailOp o;
      o.type = TOP_GEMV;
      o.n = L.n;
      o.inv = L.inv;
      o.b = L.b;
      o.out = out;
      L.rec->push_back(o);
      return out;
    }
    launch_pdl(k_gemv, grid_for((int64_t)L.n * 32, 128, 8), 128, 0, st, L.inv, L.b, L.n, out);
    return out;
  }
  double* x = smooth(L, nullptr, st, nullptr, first_done);
  residual(L, x, st);
  MgLevelPlan& C = m->lv[l + 1];
  if (L.rec) {
    TailOp o;
    o.type = TOP_RESTRICT;
    o.agg_ptr = L.agg_ptr;
    o.members = L.members;
    o.P = L.P;
    o.x = L.r;
    o.n_agg = L.n_agg;
    o.out = C.b;
    L.rec->push_back(o);
    double* xc = vcycle(m, l + 1, st);
    TailOp q;
    q.type = TOP_PROLONG;
    q.agg = L.agg;
    q.P = L.P;
    q.x = xc;
    q.nbr = L.nbr;
    q.bs = L.bs;
    q.out = x;
    L.rec->push_back(q);
    return smooth(L, x, st, l == 0 ? m->out : nullptr);
  }
  // the coarse level's first smoothing step rides on the restriction (not into the
  // coarsest solve, nor into a level the recorded tail runs)
  const bool fuse = !C.inv && C.bs == 16 && C.Dinv && C.iterations >= 1 && C.x &&
                    !((int)(l + 1) == m->tail_from && !m->tail_recording);
  const int rg = grid_for((int64_t)L.n_agg * 32, 128, 16);
  if (L.bs == 9) {
    if (fuse)
      launch_pdl(k_restrict_warp<9, true>, rg, 128, 0, st, L.agg_ptr, L.members, L.P, L.r, L.n_agg, C.b, C.Dinv, C.d,
                 C.x, C.theta);
    else
      launch_pdl(k_restrict_warp<9>, rg, 128, 0, st, L.agg_ptr, L.members, L.P, L.r, L.n_agg, C.b, nullptr, nullptr,
                 nullptr, 1.0);
  } else {
    if (fuse)
      launch_pdl(k_restrict_warp<16, true>, rg, 128, 0, st, L.agg_ptr, L.members, L.P, L.r, L.n_agg, C.b, C.Dinv, C.d,
                 C.x, C.theta);
    else
      launch_pdl(k_restrict_warp<16>, rg, 128, 0, st, L.agg_ptr, L.members, L.P, L.r, L.n_agg, C.b, nullptr, nullptr,
                 nullptr, 1.0);
  }
  double* xc = vcycle(m, l + 1, st, fuse);
  launch_pdl(k_prolong, grid_for((int64_t)L.n, 256), 256, 0, st, L.agg, L.P, xc, L.nbr, L.bs, x, 1);
  return smooth(L, x, st, l == 0 ? m->out : nullptr);
}

// Coarse tail: the first level from which every level is a 16x16 operator of at most
// BAMG_VTAIL_MB MB (default 0: off) or the coarsest dense solve, if there is a smoothing
// level among them. Records the tail's steps (the launch recursion in recording
// mode: same buffers, same coefficients) and uploads them.
static int vtail_mb() {
  static int mb = -1;
  if (mb < 0) {
    const char* e = getenv("BAMG_VTAIL_MB");
    mb = e ? atoi(e) : 0;  // off by default: measured slower than the launched levels
  }
  return mb;
}

static int mg_plan_tail(bamg_mg* m, const std::vector<int>& nnzb, cudaStream_t st) {
  m->tail_from = -1;
  const int nl = (int)m->lv.size();
  const int64_t cap = (int64_t)(m->tail_mb >= 0 ? m->tail_mb : vtail_mb()) << 20;
  int from = nl;
  for (int l = nl - 1; l >= 1; --l) {
    const MgLevelPlan& L = m->lv[l];
    bool ok = L.inv ? (l == nl - 1) : (L.bs == 16 && L.ptr && L.Dinv && L.agg_ptr && (int64_t)nnzb[l] * 2048 <= cap);
    if (!ok) break;
    from = l;
  }
  if (cap <= 0 || from >= nl - 1 || !m->lv[nl - 1].inv) return 0;
  for (int l = from; l < nl; ++l) m->lv[l].rec = &m->tail_host;
  m->tail_recording = true;
  m->tail_from = from;
  m->tail_result = vcycle(m, from, st);
  m->tail_recording = false;
  for (int l = from; l < nl; ++l) m->lv[l].rec = nullptr;
  size_t bytes = sizeof(TailOp) * m->tail_host.size();
  BAMG_CUDA_CHECK(cudaMallocAsync(&m->tail_ops, bytes, st));
  BAMG_CUDA_CHECK(cudaMemcpyAsync(m->tail_ops, m->tail_host.data(), bytes, cudaMemcpyHostToDevice, st));
  static int grid = 0, cluster = -1;
  if (cluster < 0) {
    const char* e = getenv("BAMG_VTAIL_MODE");
    cluster = !(e && strcmp(e, "grid") == 0);
  }
  if (!grid) {
    if (cluster) {
      const char* e = getenv("BAMG_VTAIL_CTAS");
      grid = e ? atoi(e) : 16;
      if (grid > 8)
        BAMG_CUDA_CHECK(cudaFuncSetAttribute(k_vcycle_tail<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    } else {
      int per_sm = 0;
      BAMG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_vcycle_tail<false>, 128, 0));
      const char* e = getenv("BAMG_VTAIL_CTAS");
      int want = e ? atoi(e) : 4;
      if (per_sm > want) per_sm = want;
      if (per_sm < 1) per_sm = 1;
      grid = per_sm * bamg_num_sms();
    }
  }
  m->tail_grid = grid;
  m->tail_cluster = cluster != 0;
  return 0;
}

static int mg_record(bamg_mg* m, cudaStream_t st) {
  double* res = vcycle(m, 0, st);
  if (res != m->out)
    BAMG_CUDA_CHECK(cudaMemcpyAsync(m->out, res, sizeof(double) * (size_t)m->lv[0].n, cudaMemcpyDeviceToDevice, st));
  return 0;
}

static int mg_prepare(bamg_mg* m, cudaStream_t st) {
  if (!m->dirty) return 0;
  int rc = mg_alloc(m, st);
  if (rc) return rc;
  m->dirty = false;
  if (!m->use_graph) return 0;
  cudaStream_t cs;
  BAMG_CUDA_CHECK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  BAMG_CUDA_CHECK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  long long before = g_bamg_launches.load();
  rc = mg_record(m, cs);
  m->graph_kernels = g_bamg_launches.load() - before;
  g_bamg_launches.store(before);  // capture is not execution
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(cs, &g);
  cudaStreamDestroy(cs);
  if (rc) return rc;
  BAMG_CUDA_CHECK(e);
  m->graph = g;
  cudaGraphExec_t pe = take_parked_exec();
  if (pe) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(pe, g, &info) == cudaSuccess) {
      m->exec = pe;
      cudaGraphUpload(m->exec, st);  // device-side setup now, not in front of the first launch
      return 0;
    }
    cudaGetLastError();  // clear the update failure; instantiate instead
    cudaGraphExecDestroy(pe);
  }
  BAMG_CUDA_CHECK(cudaGraphInstantiate(&m->exec, g, 0));
  cudaGraphUpload(m->exec, st);
  return 0;
}

// z = M r, one V-cycle (r, z: level-0 device vectors of length n0).
static int mg_apply_dev(bamg_mg* m, const double* r, double* z, cudaStream_t st) {
  int rc = mg_prepare(m, st);
  if (rc) return rc;
  size_t bytes = sizeof(double) * (size_t)m->lv[0].n;
  if (r != m->in) BAMG_CUDA_CHECK(cudaMemcpyAsync(m->in, r, bytes, cudaMemcpyDeviceToDevice, st));
  if (m->use_graph) {
    BAMG_CUDA_CHECK(cudaGraphLaunch(m->exec, st));
    g_bamg_launches.fetch_add(m->graph_kernels);
  } else {
    rc = mg_record(m, st);
    if (rc) return rc;
  }
  if (z != m->out) BAMG_CUDA_CHECK(cudaMemcpyAsync(z, m->out, bytes, cudaMemcpyDeviceToDevice, st));
  BAMG_LAUNCH_CHECK();
  return 0;
}

extern "C" int bamg_mg_set_symmetric(bamg_mg* m, int32_t level, const bamg_symop* sym) {
  if (level < 0 || level >= (int)m->lv.size() || (sym && m->lv[level].bs != sym->bs)) {
    bamg_set_error("mg_set_symmetric: block size of level %d differs from the operator's", level);
    return BAMG_ERR_UNSUPPORTED;
  }
  m->lv[level].sym = sym;
  m->dirty = true;
  return 0;
}

extern "C" int bamg_mg_set_tail(bamg_mg* m, int32_t max_mb) {
  m->tail_mb = max_mb;
  m->dirty = true;
  return 0;
}

extern "C" int bamg_mg_use_graph(bamg_mg* m, int32_t on) {
  m->use_graph = on != 0;
  m->dirty = true;
  return 0;
}

extern "C" int32_t bamg_mg_level_kind(const bamg_mg* m, int32_t level) {
  if (!m || m->dirty || level < 0 || level >= (int)m->lv.size()) return -1;
  const MgLevelPlan& L = m->lv[level];
  if (m->tail_from >= 0 && level >= m->tail_from && !L.inv) return 5;
  if (L.inv) return 4;
  if (L.rowcta) return 1;
  if (L.sym) return 0;
  if (L.CH) return 2;
  return 3;
}

// Work arena, chunk plans and the V-cycle graph (capture + instantiate or re-target)
// ahead of the first application, so the host work can overlap device work.
extern "C" int bamg_mg_prepare(bamg_ctx* ctx, bamg_mg* m, void* stream) {
  (void)ctx;
  return mg_prepare(m, as_stream(stream));
}

extern "C" int bamg_mg_apply(bamg_ctx* ctx, bamg_mg* m, const double* r, double* z, void* stream) {
  (void)ctx;
  return mg_apply_dev(m, r, z, as_stream(stream));
}

// ---------------------------------------------------------------------------
// PCG (solver.py:70-128). Operator: BSR (bs 9/16/1) with fused <p, Ap>.
// Preconditioner: the MG plan, or block-Jacobi inverse blocks (PBJ) when mg == null.
// Outputs (host): iterations, reason (0 residual_tol, 1 forcing, 2 max_iterations),
// rel, q_history[0..iterations], err (0 none, 1 not-SPD, 2 op non-finite,
// 3 curvature, 4 residual non-finite, 5 preconditioner non-finite), err_value, err_iter.

// ---------------------------------------------------------------------------
// The same PCG as ONE CUDA graph with device-side control flow: a WHILE
// conditional node runs the iterations and an IF node inside its body skips the
// preconditioner tail once a stop test fired. The stop tests of solver.py:70-128
// run in single-thread kernels in the reference's order, with every scalar formed
// by separately rounded operations (the host loop's arithmetic, bit for bit); the
// host reads the outcome once, after the solve. No host synchronisation per
// iteration.

struct PcgDev {
  double bnorm, rz, rzn, pap, rr, q, rel, errv;
  int it, done, reason, err, erri, pad0, pad1, pad2;
};

__global__ void k_pcg_g_init(const double* __restrict__ bb, PcgDev* s, double* qh) {
  if (threadIdx.x | blockIdx.x) return;
  double bn = __dsqrt_rn(*bb);
  s->bnorm = bn;
  s->q = 0.0;
  s->rel = 1.0;
  s->it = 0;
  s->err = 0;
  s->erri = 0;
  s->errv = 0.0;
  s->reason = 2;  // max_iterations unless a stop test fires
  s->done = 0;
  qh[0] = 0.0;
  if (bn == 0.0) {  // solver.py:93-94
    s->done = 1;
    s->reason = 0;
    s->rel = 0.0;
  }
}

// iteration-0 checks of <r, M r> (solver.py:97-101), then the loop condition
__global__ void k_pcg_g_rz0(PcgDev* s, int max_it, cudaGraphConditionalHandle hw) {
  if (threadIdx.x | blockIdx.x) return;
  if (!s->done) {
    double rz = s->rz;
    if (!isfinite(rz)) {
      s->err = 5;
      s->done = 1;
    } else if (rz <= 0.0) {
      s->err = 1;
      s->errv = rz;
      s->done = 1;
    }
  }
  cudaGraphSetConditional(hw, (!s->done && max_it > 0) ? 1u : 0u);
}

// after <p, Ap> and the x / r update: curvature, Q, relative residual, residual
// tolerance, forcing (solver.py:104-120, ForcingCriterion.satisfied 52-59)
__global__ void k_pcg_g_check1(PcgDev* s, double* qh, double rtol, double tau, cudaGraphConditionalHandle hw,
                               cudaGraphConditionalHandle hif) {
  PDL_ENTRY();
  if (threadIdx.x | blockIdx.x) return;
  int i = ++s->it;
  double pap = s->pap;
  if (!isfinite(pap)) {
    s->err = 2;
    s->erri = i;
    s->done = 1;
  } else if (pap <= 0.0) {
    s->err = 3;
    s->errv = pap;
    s->erri = i;
    s->done = 1;
  } else {
    double rz = s->rz;
    double alpha = __ddiv_rn(rz, pap);
    double q = __dsub_rn(s->q, __dmul_rn(__dmul_rn(0.5, alpha), rz));
    s->q = q;
    qh[i] = q;
    double rel = __ddiv_rn(__dsqrt_rn(s->rr), s->bnorm);
    s->rel = rel;
    if (!isfinite(rel)) {
      s->err = 4;
      s->erri = i;
      s->done = 1;
    } else if (rel <= rtol) {
      s->reason = 0;
      s->done = 1;
    } else {
      double qc = q, qp = qh[i - 1];
      if (qc != 0.0 && __ddiv_rn(__dmul_rn((double)i, __dsub_rn(qc, qp)), qc) <= tau) {
        s->reason = 1;
        s->done = 1;
      }
    }
  }
  unsigned go = s->done ? 0u : 1u;
  cudaGraphSetConditional(hif, go);
  cudaGraphSetConditional(hw, go);
}

// after z = M r and <r, z>: preconditioner checks (solver.py:121-125), last iteration
__global__ void k_pcg_g_check2(PcgDev* s, int max_it) {
  PDL_ENTRY();
  if (threadIdx.x | blockIdx.x) return;
  double rzn = s->rzn;
  if (!isfinite(rzn)) {
    s->err = 5;
    s->erri = s->it;
    s->done = 1;
  } else if (rzn <= 0.0) {
    s->err = 1;
    s->errv = rzn;
    s->erri = s->it;
    s->done = 1;
  } else if (s->it >= max_it) {
    s->reason = 2;
    s->done = 1;
  }
}

// after p = z + (rz_next / rz) p: rz <- rz_next, loop condition
__global__ void k_pcg_g_next(PcgDev* s, cudaGraphConditionalHandle hw) {
  PDL_ENTRY();
  if (threadIdx.x | blockIdx.x) return;
  s->rz = s->rzn;
  cudaGraphSetConditional(hw, s->done ? 0u : 1u);
}

static cudaGraphExec_t g_pcg_parked = nullptr;  // last PCG executable: re-targeted by the next solve

// A PCG graph built ahead of its launch (bamg_pcg_prepare): the host-side capture and
// re-target then run while the device finishes the setup; bamg_pcg_run launches it
// when called with the same arguments.
struct PcgPlan {
  bool valid = false;
  bamg_mg* mg = nullptr;
  const double* pbj = nullptr;
  const bamg_vj* vj = nullptr;
  int bs = 0, nbr = 0, max_it = 0;
  const int *ptr = nullptr, *col = nullptr;
  const double *blocks = nullptr, *b = nullptr;
  double *x = nullptr, *work = nullptr;
  double tau = 0.0, rtol = 0.0;
  const bamg_symop* sym = nullptr;
  cudaGraphExec_t exec = nullptr;
  PcgDev* dev = nullptr;
  double* qh = nullptr;
  int k_init = 0, k_body = 0, k_tail = 0;
  bool same(bamg_mg* mg_, const double* pbj_, const bamg_vj* vj_, int bs_, int nbr_, const int* ptr_, const int* col_,
            const double* blocks_, const double* b_, double* x_, double tau_, int max_it_, double rtol_, double* work_,
            const bamg_symop* sym_) const {
    return valid && mg == mg_ && pbj == pbj_ && vj == vj_ && bs == bs_ && nbr == nbr_ && ptr == ptr_ && col == col_ &&
           blocks == blocks_ && b == b_ && x == x_ && tau == tau_ && max_it == max_it_ && rtol == rtol_ &&
           work == work_ && sym == sym_;
  }
};
static PcgPlan g_pcg_plan;

static void pcg_plan_drop(cudaStream_t st) {  // an unlaunched plan: keep its executable for re-targeting
  if (!g_pcg_plan.valid) return;
  if (g_pcg_plan.exec) {
    if (g_pcg_parked) cudaGraphExecDestroy(g_pcg_parked);
    g_pcg_parked = g_pcg_plan.exec;
  }
  cudaFreeAsync(g_pcg_plan.dev, st);
  cudaFreeAsync(g_pcg_plan.qh, st);
  g_pcg_plan = PcgPlan();
}

static int pcg_build(bamg_ctx* ctx, bamg_mg* mg, const double* pbj_inv, const bamg_vj* vj, int32_t bs, int32_t nbr,
                     const int32_t* ptr, const int32_t* col, const double* blocks, const double* b, double* x,
                     double tau, int32_t max_it, double rtol, double* work, const bamg_symop* sym, cudaStream_t st) {
  pcg_plan_drop(st);
  int64_t n = (int64_t)nbr * bs;
  double* r = work;
  double* z = work + n;
  if (mg) {
    int rc0 = mg_prepare(mg, st);  // arena + chunk plans before the capture
    if (rc0) return rc0;
    if (mg->lv[0].n == n) {
      r = mg->in;
      z = mg->out;
    }
  }
  double* p = work + 2 * n;
  double* ap = work + 3 * n;
  PcgDev* dev = nullptr;
  double* qh = nullptr;
  double* bb = ctx->scalars + 4;
  BAMG_CUDA_CHECK(cudaMallocAsync(&dev, sizeof(PcgDev), st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&qh, sizeof(double) * ((size_t)max_it + 2), st));
  auto precond = [&](cudaStream_t cs) -> int {
    if (mg) {
      int rc = mg_record(mg, cs);  // kernels of one V-cycle: in = mg->in, result in mg->out
      if (rc) return rc;
      if (r != mg->in || z != mg->out) return BAMG_ERR_UNSUPPORTED;
      return 0;
    }
    if (vj) {
      vj_apply_dev(vj, r, z, cs);
      return 0;
    }
    launch_pdl(k_blockdiag_apply, grid_for(n, 256), 256, 0, cs, pbj_inv, (const double*)r, nbr, bs, z);
    return 0;
  };
  auto spmv_dot = [&](cudaStream_t cs) {
    if (sym) {
      sym_apply(ctx, sym, blocks, p, 0, nullptr, nullptr, nullptr, ap, 0.0, 0.0, 0, &dev->pap, cs);
      return;
    }
    int g = spmv_grid(nbr);
    if (g > BAMG_MAX_PARTIALS) g = BAMG_MAX_PARTIALS;
    unsigned* ctr = ctx->counters + BAMG_CTR_SPMV;
    switch (bs) {
      case 9: launch_pdl(k_bsr_spmv<9>, g, 128, 0, cs, ptr, col, blocks, (const double*)p, ap, nbr, ctx->partials, ctr, &dev->pap); break;
      case 16: launch_pdl(k_bsr_spmv<16>, g, 128, 0, cs, ptr, col, blocks, (const double*)p, ap, nbr, ctx->partials, ctr, &dev->pap); break;
      default: launch_pdl(k_bsr_spmv<1>, g, 128, 0, cs, ptr, col, blocks, (const double*)p, ap, nbr, ctx->partials, ctr, &dev->pap); break;
    }
  };

  // ---- build the graph: init segment, WHILE { check body, IF { preconditioner tail } }
  cudaGraph_t graph = nullptr;
  BAMG_CUDA_CHECK(cudaGraphCreate(&graph, 0));
  cudaGraphConditionalHandle hw, hif;
  BAMG_CUDA_CHECK(cudaGraphConditionalHandleCreate(&hw, graph, 0, cudaGraphCondAssignDefault));
  cudaStream_t cs;
  BAMG_CUDA_CHECK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  long long before = g_bamg_launches.load();
  int rc = 0;
  int k_init = 0, k_body = 0, k_tail = 0;
  cudaGraph_t body = nullptr, tail = nullptr;
  do {
    if (cudaStreamBeginCaptureToGraph(cs, graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal)) { rc = BAMG_ERR_CUDA; break; }
    long long c0 = g_bamg_launches.load();
    cudaMemsetAsync(x, 0, sizeof(double) * n, cs);
    dot_dev(ctx, b, b, n, bb, cs);
    launch_pdl(k_copy, grid_for(n, 256), 256, 0, cs, b, r, n);
    launch(k_pcg_g_init, 1, 32, 0, cs, (const double*)bb, dev, qh);
    if ((rc = precond(cs))) break;
    dot_dev(ctx, r, z, n, &dev->rz, cs);
    launch(k_pcg_g_rz0, 1, 32, 0, cs, dev, max_it, hw);
    launch_pdl(k_copy, grid_for(n, 256), 256, 0, cs, (const double*)z, p, n);
    k_init = (int)(g_bamg_launches.load() - c0);
    // WHILE node after the init segment
    cudaStreamCaptureStatus cst;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    cudaGraph_t cg = nullptr;
    if (cudaStreamGetCaptureInfo(cs, &cst, nullptr, &cg, &deps, &ndeps)) { rc = BAMG_ERR_CUDA; break; }
    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = hw;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wnode;
    if (cudaGraphAddNode(&wnode, cg, deps, ndeps, &wp)) { rc = BAMG_ERR_CUDA; break; }
    body = wp.conditional.phGraph_out[0];
    if (cudaStreamUpdateCaptureDependencies(cs, &wnode, 1, cudaStreamSetCaptureDependencies)) { rc = BAMG_ERR_CUDA; break; }
    if (cudaStreamEndCapture(cs, &graph)) { rc = BAMG_ERR_CUDA; break; }

    // body: S p, <p, S p>, x/r update + |r|^2, checks, IF { M r, <r, z>, checks, p update }
    if (cudaGraphConditionalHandleCreate(&hif, body, 0, cudaGraphCondAssignDefault)) { rc = BAMG_ERR_CUDA; break; }
    if (cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal)) { rc = BAMG_ERR_CUDA; break; }
    c0 = g_bamg_launches.load();
    spmv_dot(cs);
    launch_pdl(k_pcg_update_dev, grid_for(n, 256, 4), 256, 0, cs, x, r, (const double*)p, (const double*)ap,
           (const double*)&dev->rz, (const double*)&dev->pap, n, ctx->partials, ctx->counters + BAMG_CTR_PCG0,
           &dev->rr);
    launch_pdl(k_pcg_g_check1, 1, 32, 0, cs, dev, qh, rtol, tau, hw, hif);
    k_body = (int)(g_bamg_launches.load() - c0);
    if (cudaStreamGetCaptureInfo(cs, &cst, nullptr, &cg, &deps, &ndeps)) { rc = BAMG_ERR_CUDA; break; }
    cudaGraphNodeParams ip = {};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = hif;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    cudaGraphNode_t inode;
    if (cudaGraphAddNode(&inode, cg, deps, ndeps, &ip)) { rc = BAMG_ERR_CUDA; break; }
    tail = ip.conditional.phGraph_out[0];
    if (cudaStreamUpdateCaptureDependencies(cs, &inode, 1, cudaStreamSetCaptureDependencies)) { rc = BAMG_ERR_CUDA; break; }
    if (cudaStreamEndCapture(cs, &body)) { rc = BAMG_ERR_CUDA; break; }

    if (cudaStreamBeginCaptureToGraph(cs, tail, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal)) { rc = BAMG_ERR_CUDA; break; }
    c0 = g_bamg_launches.load();
    if ((rc = precond(cs))) break;
    dot_dev(ctx, r, z, n, &dev->rzn, cs);
    launch_pdl(k_pcg_g_check2, 1, 32, 0, cs, dev, max_it);
    launch_pdl(k_xpby_dev, grid_for(n, 256), 256, 0, cs, (const double*)z, (const double*)&dev->rzn,
           (const double*)&dev->rz, p, n);
    launch_pdl(k_pcg_g_next, 1, 32, 0, cs, dev, hw);
    k_tail = (int)(g_bamg_launches.load() - c0);
    if (cudaStreamEndCapture(cs, &tail)) { rc = BAMG_ERR_CUDA; break; }
  } while (0);
  g_bamg_launches.store(before);  // capture is not execution
  if (rc) {
    cudaStreamCaptureStatus cst;
    if (cudaStreamIsCapturing(cs, &cst) == cudaSuccess && cst != cudaStreamCaptureStatusNone) {
      cudaGraph_t junk = nullptr;
      cudaStreamEndCapture(cs, &junk);
      if (junk && junk != graph) cudaGraphDestroy(junk);
    }
    cudaGetLastError();
    cudaStreamDestroy(cs);
    cudaGraphDestroy(graph);
    cudaFreeAsync(dev, st);
    cudaFreeAsync(qh, st);
    if (rc == BAMG_ERR_CUDA) bamg_set_error("pcg graph capture failed");
    return rc;
  }
  cudaStreamDestroy(cs);
  static const bool timing = getenv("BAMG_PCG_TIMING") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto t0 = now();
  int how = 0;
  cudaGraphExec_t exec = nullptr;
  if (g_pcg_parked) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(g_pcg_parked, graph, &info) == cudaSuccess) {
      exec = g_pcg_parked;
      how = 1;
    } else {
      cudaGetLastError();
      cudaGraphExecDestroy(g_pcg_parked);
      how = 2;
    }
    g_pcg_parked = nullptr;
  }
  auto t1 = now();
  if (!exec) {
    cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
    if (timing)
      fprintf(stderr, "[pcg] update %s %.2f ms, instantiate %.2f ms\n", how == 1 ? "ok" : (how == 2 ? "failed" : "none"),
              std::chrono::duration<double, std::milli>(t1 - t0).count(),
              std::chrono::duration<double, std::milli>(now() - t1).count());
    if (e != cudaSuccess) {
      cudaGraphDestroy(graph);
      cudaFreeAsync(dev, st);
      cudaFreeAsync(qh, st);
      BAMG_CUDA_CHECK(e);
    }
  }
  else if (timing)
    fprintf(stderr, "[pcg] update ok %.2f ms\n", std::chrono::duration<double, std::milli>(t1 - t0).count());
  cudaGraphDestroy(graph);
  PcgPlan& P = g_pcg_plan;
  P.valid = true;
  P.mg = mg;
  P.pbj = pbj_inv;
  P.vj = vj;
  P.bs = bs;
  P.nbr = nbr;
  P.ptr = ptr;
  P.col = col;
  P.blocks = blocks;
  P.b = b;
  P.x = x;
  P.tau = tau;
  P.max_it = max_it;
  P.rtol = rtol;
  P.work = work;
  P.sym = sym;
  P.exec = exec;
  P.dev = dev;
  P.qh = qh;
  P.k_init = k_init;
  P.k_body = k_body;
  P.k_tail = k_tail;
  return 0;
}

static int pcg_graph(bamg_ctx* ctx, bamg_mg* mg, const double* pbj_inv, const bamg_vj* vj, int32_t bs, int32_t nbr,
                     const int32_t* ptr, const int32_t* col, const double* blocks, const double* b, double* x,
                     double tau, int32_t max_it, double rtol, double* work, int32_t* iterations_out,
                     int32_t* reason_out, double* rel_out, double* q_hist, int32_t* err_out, double* err_value_out,
                     int32_t* err_iter_out, const bamg_symop* sym, cudaStream_t st) {
  if (!g_pcg_plan.same(mg, pbj_inv, vj, bs, nbr, ptr, col, blocks, b, x, tau, max_it, rtol, work, sym)) {
    int rc = pcg_build(ctx, mg, pbj_inv, vj, bs, nbr, ptr, col, blocks, b, x, tau, max_it, rtol, work, sym, st);
    if (rc) return rc;
  }
  PcgPlan P = g_pcg_plan;
  g_pcg_plan = PcgPlan();  // consumed
  PcgDev* dev = P.dev;
  double* qh = P.qh;
  BAMG_CUDA_CHECK(cudaGraphLaunch(P.exec, st));
  PcgDev h;
  BAMG_CUDA_CHECK(cudaMemcpyAsync(&h, dev, sizeof(PcgDev), cudaMemcpyDeviceToHost, st));
  BAMG_CUDA_CHECK(cudaStreamSynchronize(st));
  if (g_pcg_parked) cudaGraphExecDestroy(g_pcg_parked);
  g_pcg_parked = P.exec;
  int its = h.it;
  if (its > 0) BAMG_CUDA_CHECK(cudaMemcpy(q_hist + 1, qh + 1, sizeof(double) * (size_t)its, cudaMemcpyDeviceToHost));
  q_hist[0] = 0.0;
  cudaFreeAsync(dev, st);
  cudaFreeAsync(qh, st);
  // launch accounting: init + every body + every executed tail
  int tails = its - ((h.err >= 2 && h.err <= 4) || (h.done && h.err == 0 && h.reason != 2) ? 1 : 0);
  if (tails < 0) tails = 0;
  g_bamg_launches.fetch_add((long long)P.k_init + (long long)its * P.k_body + (long long)tails * P.k_tail);
  *err_out = h.err;
  *err_value_out = h.errv;
  *err_iter_out = h.erri;
  *iterations_out = (h.err == 0 && h.reason == 2) ? max_it : its;
  *reason_out = h.reason;
  *rel_out = h.rel;
  BAMG_LAUNCH_CHECK();
  return 0;
}

// Build (capture / re-target) the PCG graph of a later bamg_pcg_run with the same
// arguments now, so the host work overlaps device work still in flight. Optional.
extern "C" int bamg_pcg_prepare(bamg_ctx* ctx, bamg_mg* mg, const double* pbj_inv, const bamg_vj* vj, int32_t bs,
                                int32_t nbr, const int32_t* ptr, const int32_t* col, const double* blocks,
                                const double* b, double* x, double tau, int32_t max_it, double rtol, double* work,
                                const bamg_symop* sym, void* stream) {
  cudaStream_t st = as_stream(stream);
  if ((sym && bs != sym->bs) || max_it < 0 || (mg && mg_prepare(mg, st) == 0 && mg->lv[0].n != (int64_t)nbr * bs))
    return 0;  // bamg_pcg_run takes another path (or reports the error) itself
  static const bool host_loop = [] {
    const char* e = getenv("BAMG_PCG_HOSTLOOP");
    return e && e[0] == '1';
  }();
  if (host_loop) return 0;
  return pcg_build(ctx, mg, pbj_inv, vj, bs, nbr, ptr, col, blocks, b, x, tau, max_it, rtol, work, sym, st);
}

extern "C" int bamg_pcg_run(bamg_ctx* ctx, bamg_mg* mg, const double* pbj_inv, const bamg_vj* vj, int32_t bs, int32_t nbr,
                            const int32_t* ptr, const int32_t* col, const double* blocks, const double* b, double* x,
                            double tau, int32_t max_it, double rtol, double* work, int32_t* iterations_out,
                            int32_t* reason_out, double* rel_out, double* q_hist, int32_t* err_out,
                            double* err_value_out, int32_t* err_iter_out, const bamg_symop* sym,
                            void* stream) {
  cudaStream_t st = as_stream(stream);
  int64_t n = (int64_t)nbr * bs;
  if (sym && bs != sym->bs) {
    bamg_set_error("pcg_run: symmetric operator block size %d, operator %d", sym->bs, bs);
    return BAMG_ERR_UNSUPPORTED;
  }
  static const bool host_loop = [] {
    const char* e = getenv("BAMG_PCG_HOSTLOOP");
    return e && e[0] == '1';
  }();
  if (!host_loop && max_it >= 0 && (!mg || mg->lv[0].n == n))
    return pcg_graph(ctx, mg, pbj_inv, vj, bs, nbr, ptr, col, blocks, b, x, tau, max_it, rtol, work, iterations_out,
                     reason_out, rel_out, q_hist, err_out, err_value_out, err_iter_out, sym, st);
  double* r = work;
  double* z = work + n;
  if (mg) {
    // the plan's own level-0 input / output vectors: the V-cycle reads r in place and
    // leaves z where the PCG reads it (no copies around every preconditioner application)
    int rc0 = mg_prepare(mg, st);
    if (rc0) return rc0;
    if (mg->lv[0].n == n) {
      r = mg->in;
      z = mg->out;
    }
  }
  double* p = work + 2 * n;
  double* ap = work + 3 * n;
  double* sc = ctx->scalars;      // [0] pap [1] rr [2] rz slot A [3] rz slot B [4] bb
  double* hs = ctx->host_scalars;
  *err_out = 0;
  *err_iter_out = 0;
  *err_value_out = 0.0;
  auto precond = [&](const double* in, double* out) -> int {
    if (mg) return mg_apply_dev(mg, in, out, st);
    if (vj) {
      vj_apply_dev(vj, in, out, st);
      BAMG_LAUNCH_CHECK();
      return 0;
    }
    launch_pdl(k_blockdiag_apply, grid_for(n, 256), 256, 0, st, pbj_inv, in, nbr, bs, out);
    BAMG_LAUNCH_CHECK();
    return 0;
  };
  auto spmv_dot = [&](const double* v, double* out, double* dot) {
    if (sym) {
      sym_apply(ctx, sym, blocks, v, 0, nullptr, nullptr, nullptr, out, 0.0, 0.0, 0, dot, st);
      return;
    }
    int g = spmv_grid(nbr);
    if (g > BAMG_MAX_PARTIALS) g = BAMG_MAX_PARTIALS;
    unsigned* ctr = ctx->counters + BAMG_CTR_SPMV;
    switch (bs) {
      case 9: launch_pdl(k_bsr_spmv<9>, g, 128, 0, st, ptr, col, blocks, v, out, nbr, ctx->partials, ctr, dot); break;
      case 16: launch_pdl(k_bsr_spmv<16>, g, 128, 0, st, ptr, col, blocks, v, out, nbr, ctx->partials, ctr, dot); break;
      default: launch_pdl(k_bsr_spmv<1>, g, 128, 0, st, ptr, col, blocks, v, out, nbr, ctx->partials, ctr, dot); break;
    }
  };
  int rc;
  int q_len = 0;
  q_hist[q_len++] = 0.0;
  BAMG_CUDA_CHECK(cudaMemsetAsync(x, 0, sizeof(double) * n, st));
  rc = dot_dev(ctx, b, b, n, sc + 4, st);
  if (rc) return rc;
  launch_pdl(k_copy, grid_for(n, 256), 256, 0, st, b, r, n);
  BAMG_CUDA_CHECK(cudaMemcpyAsync(hs + 4, sc + 4, sizeof(double), cudaMemcpyDeviceToHost, st));
  BAMG_CUDA_CHECK(cudaStreamSynchronize(st));
  double b_norm = sqrt(hs[4]);
  if (b_norm == 0.0) {
    *iterations_out = 0;
    *reason_out = 0;
    *rel_out = 0.0;
    return 0;
  }
  rc = precond(r, z);
  if (rc) return rc;
  int slot = 2;  // device slot holding the current rz
  rc = dot_dev(ctx, r, z, n, sc + slot, st);
  if (rc) return rc;
  BAMG_CUDA_CHECK(cudaMemcpyAsync(hs + slot, sc + slot, sizeof(double), cudaMemcpyDeviceToHost, st));
  BAMG_CUDA_CHECK(cudaStreamSynchronize(st));
  double rz = hs[slot];
  if (!isfinite(rz)) { *err_out = 5; *err_iter_out = 0; return 0; }
  if (rz <= 0.0) { *err_out = 1; *err_value_out = rz; *err_iter_out = 0; return 0; }
  launch_pdl(k_copy, grid_for(n, 256), 256, 0, st, z, p, n);
  double q_val = 0.0, rel = 1.0;
  bool pending = false;  // an rz_next on the device not yet checked on the host
  for (int i = 1; i <= max_it; ++i) {
    spmv_dot(p, ap, sc + 0);
    launch_pdl(k_pcg_update_dev, grid_for(n, 256, 4), 256, 0, st, x, r, p, ap, sc + slot, sc + 0, n, ctx->partials,
           ctx->counters + BAMG_CTR_PCG0, sc + 1);
    BAMG_CUDA_CHECK(cudaMemcpyAsync(hs, sc, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
    BAMG_CUDA_CHECK(cudaStreamSynchronize(st));
    BAMG_LAUNCH_CHECK();
    if (pending) {  // checks of iteration i-1's <r, M r> (solver.py:121-125)
      double rzn = hs[slot];
      if (!isfinite(rzn)) { *err_out = 5; *err_iter_out = i - 1; *iterations_out = i - 1; return 0; }
      if (rzn <= 0.0) { *err_out = 1; *err_value_out = rzn; *err_iter_out = i - 1; *iterations_out = i - 1; return 0; }
      rz = rzn;
      pending = false;
    }
    double pap = hs[0];
    if (!isfinite(pap)) { *err_out = 2; *err_iter_out = i; *iterations_out = i; return 0; }
    if (pap <= 0.0) { *err_out = 3; *err_value_out = pap; *err_iter_out = i; *iterations_out = i; return 0; }
    double alpha = rz / pap;
    q_val -= 0.5 * alpha * rz;
    q_hist[q_len++] = q_val;
    rel = sqrt(hs[1]) / b_norm;
    *rel_out = rel;
    if (!isfinite(rel)) { *err_out = 4; *err_iter_out = i; *iterations_out = i; return 0; }
    if (rel <= rtol) { *iterations_out = i; *reason_out = 0; return 0; }
    // forcing (solver.py:52-59)
    {
      int k = q_len - 1;
      double qc = q_hist[q_len - 1], qp = q_hist[q_len - 2];
      if (k >= 1 && qc != 0.0 && k * (qc - qp) / qc <= tau) { *iterations_out = i; *reason_out = 1; return 0; }
    }
    rc = precond(r, z);
    if (rc) return rc;
    int nslot = (slot == 2) ? 3 : 2;
    rc = dot_dev(ctx, r, z, n, sc + nslot, st);
    if (rc) return rc;
    launch_pdl(k_xpby_dev, grid_for(n, 256), 256, 0, st, z, sc + nslot, sc + slot, p, n);
    slot = nslot;
    pending = true;
  }
  if (pending) {
    BAMG_CUDA_CHECK(cudaMemcpyAsync(hs + slot, sc + slot, sizeof(double), cudaMemcpyDeviceToHost, st));
    BAMG_CUDA_CHECK(cudaStreamSynchronize(st));
    double rzn = hs[slot];
    if (!isfinite(rzn)) { *err_out = 5; *err_iter_out = max_it; *iterations_out = max_it; return 0; }
    if (rzn <= 0.0) { *err_out = 1; *err_value_out = rzn; *err_iter_out = max_it; *iterations_out = max_it; return 0; }
  }
  *iterations_out = max_it;
  *reason_out = 2;
  *rel_out = rel;
  BAMG_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------------------
// D-Lanczos (multigrid.py:243-284), all steps on the device, one readback.

// z = Dinv u - a q - b qp   (a = s[ia], b = s[ib] or 0)
__global__ void k_lanczos_z(const double* __restrict__ Dinv, const double* __restrict__ u, const double* __restrict__ q,
                            const double* __restrict__ qp, const double* __restrict__ s, int ia, int ib, int nb,
                            int bs, double* __restrict__ z) {
  double a = s[ia];
  double b = ib >= 0 ? s[ib] : 0.0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)nb * bs; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t blk = t / bs;
    int rr = (int)(t - blk * bs);
    const double* m = Dinv + (blk * bs + rr) * bs;
    const double* ub = u + blk * bs;
    double v = 0.0;
    for (int c = 0; c < bs; ++c) v = fma(m[c], ub[c], v);
    z[t] = v - a * q[t] - b * qp[t];
  }
}

// y -= s[i] x
__global__ void k_axpy_dev(const double* __restrict__ x, const double* __restrict__ s, int i, double* __restrict__ y,
                           int64_t n) {
  double a = s[i];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    y[t] = fma(-a, x[t], y[t]);
}

// y = x / sqrt(s[i])
__global__ void k_scale_rsqrt_dev(const double* __restrict__ x, const double* __restrict__ s, int i,
                                  double* __restrict__ y, int64_t n) {
  double b = sqrt(s[i]);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    y[t] = x[t] / b;
}

// s[i] = sqrt(s[i]) in place (single thread)
__global__ void k_sqrt_slot(double* s, int i, int j) {
  if (threadIdx.x == 0 && blockIdx.x == 0) s[j] = sqrt(s[i]);
}

// One modified-Gram-Schmidt step in the D inner product, fused: first finish the
// previous projection (z' = z - s[prev] q_prev, when q_prev != null; written to
// z_out), then out = <w, D z'> with w = q_b, or w = z' (q_b == null: ||z'||_D^2).
// The arithmetic is the unfused sequence's, element for element: the same
// fma(-c, q, z) update as k_axpy_dev, the same per-row fma chain as
// k_blockdiag_apply, and the same thread partition / block tree as k_dot (launch
// with k_dot's grid) -- so the Lanczos scalars are bit-identical to the unfused path.
__global__ void __launch_bounds__(256)
k_reorth_step(const double* __restrict__ D, const double* __restrict__ z_in, double* __restrict__ z_out,
              const double* __restrict__ q_prev, const double* __restrict__ s, int prev,
              const double* __restrict__ qb, int bs, int64_t n, double* partials, unsigned int* counter,
              double* out) {
  __shared__ double scratch[33];
  double c = q_prev ? s[prev] : 0.0;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = i / bs;
    int r = (int)(i - b * bs);
    const double* m = D + (b * bs + r) * bs;
    const double* zb = z_in + b * bs;
    const double* qpb = q_prev ? q_prev + b * bs : nullptr;
    double dz = 0.0;
    for (int cc = 0; cc < bs; ++cc) {
      double zc = qpb ? fma(-c, qpb[cc], zb[cc]) : zb[cc];
      dz = fma(m[cc], zc, dz);
    }
    double zi = q_prev ? fma(-c, q_prev[i], z_in[i]) : z_in[i];
    if (q_prev) z_out[i] = zi;
    acc = fma(qb ? qb[i] : zi, dz, acc);
  }
  acc = block_sum(acc, scratch);
  grid_finish(partials, counter, acc, scratch, out);
}

// v0: seeded start vector (device). D: diagonal blocks, Dinv: their inverses.
// work: (steps + 5) * n doubles. Returns lambda (host) and the Lanczos break
// status through *status (0 ok, 1 non-finite).
extern "C" int bamg_lanczos_lmax(bamg_ctx* ctx, int32_t bs, int32_t nbr, const int32_t* ptr, const int32_t* col,
                                 const double* blocks, const double* D, const double* Dinv, const double* v0,
                                 int32_t steps, double* work, double* lambda_out, int32_t* status,
                                 const bamg_symop* sym, double* ab_out_dev, void* stream) {
  cudaStream_t st = as_stream(stream);
  int64_t n = (int64_t)nbr * bs;
  double* sc = ctx->scalars + 16;  // [0..15] per step: alpha[s]=sc[s], beta2[s]=sc[8+s]; extras at 64+
  double* tmp = ctx->scalars + 64;  // dnorm^2, beta, reorth coefficient slots
  double* basis = work;             // (steps+1) * n
  double* u = work + (int64_t)(steps + 1) * n;
  double* z = u + n;
  double* Dz = z + n;
  double* qprev = Dz + n;
  int g = grid_for(n, 256);
  BAMG_CUDA_CHECK(cudaMemsetAsync(qprev, 0, sizeof(double) * n, st));
  // q0 = v / sqrt(v . D v)
  launch_pdl(k_blockdiag_apply, g, 256, 0, st, D, v0, nbr, bs, Dz);
  int rc = dot_dev(ctx, v0, Dz, n, tmp + 0, st);
  if (rc) return rc;
  launch(k_scale_rsqrt_dev, g, 256, 0, st, v0, tmp, 0, basis, n);
  int sg = spmv_grid(nbr);
  if (sg > BAMG_MAX_PARTIALS) sg = BAMG_MAX_PARTIALS;
  const int rg = grid_for(n, 256, 4);  // k_dot's grid (dot_dev): same partition, same sums
  for (int s = 0; s < steps; ++s) {
    double* q = basis + (int64_t)s * n;
    double* qp = s > 0 ? basis + (int64_t)(s - 1) * n : qprev;
    unsigned* ctr = ctx->counters + BAMG_CTR_SPMV;
    if (sym && sym->bs == bs) sym_apply(ctx, sym, blocks, q, 0, nullptr, nullptr, nullptr, u, 0.0, 0.0, 0, sc + s, st);
    else switch (bs) {
      case 9: launch_pdl(k_bsr_spmv<9>, sg, 128, 0, st, ptr, col, blocks, q, u, nbr, ctx->partials, ctr, sc + s); break;
      case 16: launch_pdl(k_bsr_spmv<16>, sg, 128, 0, st, ptr, col, blocks, q, u, nbr, ctx->partials, ctr, sc + s); break;
      default: launch_pdl(k_bsr_spmv<1>, sg, 128, 0, st, ptr, col, blocks, q, u, nbr, ctx->partials, ctr, sc + s); break;
    }
    // z = D^-1 u - alpha q - beta_prev q_prev   (beta_prev = sqrt(beta2[s-1]))
    if (s > 0) launch(k_sqrt_slot, 1, 1, 0, st, sc, 8 + s - 1, 40 + s - 1);
    launch(k_lanczos_z, g, 256, 0, st, Dinv, u, q, qp, sc, s, s > 0 ? 40 + s - 1 : -1, nbr, bs, z);
    // full reorthogonalisation in the D inner product (modified Gram-Schmidt:
    // z -= q_b <q_b, D z> for b = 0..s), each coefficient fused with the previous
    // subtraction; the last pass finishes the subtraction and forms ||z||_D^2
    double* zc = z;   // current z
    double* zn = Dz;  // the other buffer
    for (int b2 = 0; b2 <= s + 1; ++b2) {
      const double* qprev_b = b2 > 0 ? basis + (int64_t)(b2 - 1) * n : nullptr;
      const double* qb = b2 <= s ? basis + (int64_t)b2 * n : nullptr;
      double* dst = b2 <= s ? tmp + 1 + (b2 & 1) : sc + 8 + s;  // alternate: the kernel reads the previous slot
      launch(k_reorth_step, rg, 256, 0, st, D, (const double*)zc, zn, qprev_b, (const double*)tmp,
             1 + ((b2 + 1) & 1), qb, bs, n, ctx->partials, ctx->counters + BAMG_CTR_DOT, dst);
      if (qprev_b) std::swap(zc, zn);
    }
    launch(k_scale_rsqrt_dev, g, 256, 0, st, zc, sc, 8 + s, basis + (int64_t)(s + 1) * n, n);
  }
  if (ab_out_dev) {  // deferred: the caller reads several levels' scalars at once
    BAMG_CUDA_CHECK(cudaMemcpyAsync(ab_out_dev, sc, 16 * sizeof(double), cudaMemcpyDeviceToDevice, st));
    BAMG_LAUNCH_CHECK();
    return 0;
  }
  double h[16];
  BAMG_CUDA_CHECK(cudaMemcpyAsync(h, sc, 16 * sizeof(double), cudaMemcpyDeviceToHost, st));
  BAMG_CUDA_CHECK(cudaStreamSynchronize(st));
  BAMG_LAUNCH_CHECK();
  return bamg_lanczos_finish(h, steps, lambda_out, status);
}

// host replay of the Lanczos break rule (multigrid.py:268-281) on the 16 device
// scalars [alpha_0..7 | beta^2_0..7], then the Ritz maximum
extern "C" int bamg_lanczos_finish(const double* ab_host, int32_t steps, double* lambda_out, int32_t* status) {
  std::vector<double> al, be;
  *status = 0;
  for (int s = 0; s < steps; ++s) {
    double alpha = ab_host[s], beta2 = ab_host[8 + s];
    al.push_back(alpha);
    if (!isfinite(beta2)) {
      *status = 1;
      return 0;
    }
    if (beta2 <= 0 || sqrt(beta2) < 1e-12 * fabs(alpha)) break;
    be.push_back(sqrt(beta2));
  }
  if (be.size() >= al.size()) be.resize(al.size() - 1);
  if (be.empty()) be.push_back(0.0);
  *lambda_out = bamg_tridiag_max_eig(al.data(), be.data(), (int)al.size());
  return 0;
}
