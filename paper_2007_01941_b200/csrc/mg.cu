// Multigrid setup (multigrid.py:83-237, 371-471; problem.py:332-352):
// operator strength, greedy aggregation (bit-exact, single warp), gauge
// near-nullspace K, per-aggregate Householder QR prolongation (economic + pivoted
// branches), Galerkin P^T A P (symbolic + numeric, deterministic), symmetrise,
// decoupled-dof patch.
#include "common.cuh"
#include "ctx.h"

int radix_sort_pairs(const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout,
                     int64_t n, int key_bits, cudaStream_t st);
int scan_exclusive_int(const int* in, int* out, int64_t n, int* total, cudaStream_t st);
int segment_ptr(const int* ids, int64_t n, int nseg, int* ptr, cudaStream_t st);

// ---------------------------------------------------------------------------
// operator strength (multigrid.py:83-98)

__global__ void k_block_fro(const double* __restrict__ blocks, int64_t nnz, int bb, double* __restrict__ nrm) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nnz; b += (int64_t)gridDim.x * blockDim.x) {
    const double* a = blocks + b * bb;
    double s = 0.0;
    if (bb == 256) {
      // 16x16 blocks (2 KB, 16 B aligned): 16 B loads, eight in flight, the same
      // sequential sum over the entries
      const double2* a2 = reinterpret_cast<const double2*>(a);
      for (int q = 0; q < 128; q += 8) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(a2 + q + u);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          s += v[u].x * v[u].x;
          s += v[u].y * v[u].y;
        }
      }
    } else {
      for (int q = 0; q < bb; ++q) s += a[q] * a[q];
    }
    nrm[b] = sqrt(s);
  }
}

__global__ void k_op_strength(const int* __restrict__ ptr, const int* __restrict__ col, const double* __restrict__ nrm,
                              int n, const double* __restrict__ dnorm, int* __restrict__ G_ptr, int* __restrict__ G_col,
                              double* __restrict__ G_val, int* __restrict__ zero_diag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double di = dnorm[i];
    if (di == 0.0) atomicAdd(zero_diag, 1);
    int out = G_ptr[i];
    for (int q = ptr[i]; q < ptr[i + 1]; ++q) {
      int j = col[q];
      if (j == i) continue;
      double v = nrm[q] / sqrt(di * dnorm[j]);
      G_col[out] = j;
      G_val[out] = v < 1.0 ? v : 1.0;
      ++out;
    }
  }
}

__global__ void k_diag_norm_and_count(const int* __restrict__ ptr, const int* __restrict__ col,
                                      const double* __restrict__ nrm, int n, double* __restrict__ dnorm,
                                      int* __restrict__ offcount) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double d = 0.0;
    int c = 0;
    for (int q = ptr[i]; q < ptr[i + 1]; ++q) {
      if (col[q] == i) d = nrm[q];
      else ++c;
    }
    dnorm[i] = d;
    offcount[i] = c;
  }
}

// G_ptr must hold n+1 ints. Sizes: call with G_col == null to get G_ptr + total.
extern "C" int bamg_operator_strength(bamg_ctx* ctx, const int32_t* ptr, const int32_t* col, const double* blocks,
                                      int32_t n, int64_t nnz, int32_t bs, double* nrm_work, double* dnorm_work,
                                      int32_t* G_ptr, int32_t* G_col, double* G_val, int32_t* flags_dev,
                                      void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (G_col == nullptr) {
    BAMG_CUDA_CHECK(cudaMemsetAsync(flags_dev, 0, sizeof(int) * 2, st));
    launch(k_block_fro, grid_for(nnz, 256), 256, 0, st, blocks, nnz, bs * bs, nrm_work);
    launch(k_diag_norm_and_count, grid_for(n, 128), 128, 0, st, ptr, col, nrm_work, n, dnorm_work, G_ptr);
    BAMG_LAUNCH_CHECK();
    return scan_exclusive_int(G_ptr, G_ptr, n + 1, flags_dev + 1, st);  // G_ptr[n] is scratch -> total
  }
  launch(k_op_strength, grid_for(n, 128), 128, 0, st, ptr, col, nrm_work, n, dnorm_work, G_ptr, G_col, G_val, flags_dev);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------------------
// greedy aggregation (multigrid.py:127-176), one warp, sequential over nodes.
// In-scan choice: among neighbours that are unaggregated or in an aggregate of
// size < max_size, the first in (-G, aggregated?, index) order. Post-pass: the
// (G, -index)-largest neighbour whose aggregate has size <= max_size.

struct Cand {
  double g;
  int un;  // 1 if unaggregated
  int j;
};

__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
  if (a.j < 0) return false;
  if (b.j < 0) return true;
  if (a.g != b.g) return a.g > b.g;
  if (a.un != b.un) return a.un > b.un;
  return a.j < b.j;
}

__device__ __forceinline__ Cand warp_best(Cand c) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Cand t;
    t.g = __shfl_xor_sync(FULL_MASK, c.g, o);
    t.un = __shfl_xor_sync(FULL_MASK, c.un, o);
    t.j = __shfl_xor_sync(FULL_MASK, c.j, o);
    if (better(t, c)) c = t;
  }
  return c;
}

#define AG_K 8

__global__ void __launch_bounds__(32)
k_aggregate(const int* __restrict__ G_ptr, const int* __restrict__ G_col, const double* __restrict__ G_val, int n,
            int max_size, int* __restrict__ agg_g, int* __restrict__ size_g, int use_smem, int* __restrict__ n_agg_out) {
  extern __shared__ int sh[];
  int lane = threadIdx.x;
  int* agg = use_smem ? sh : agg_g;
  int* size = use_smem ? sh + n : size_g;
  for (int i = lane; i < n; i += 32) {
    agg[i] = -1;
    size[i] = 0;
  }
  __syncwarp();
  int nagg = 0;
  // Rows of up to 32*AG_K entries live in registers; the row of the next
  // unaggregated node is loaded while the current node is decided (the
  // decisions themselves only touch shared memory), which hides the global
  // latency that otherwise dominates this sequential scan.
  int pf_node = -1, pf_len = 0;
  int pf_j[AG_K];
  double pf_g[AG_K];
  auto prefetch = [&](int node) {
    pf_node = node;
    int s = G_ptr[node], e = G_ptr[node + 1];
    pf_len = e - s;
#pragma unroll
    for (int t = 0; t < AG_K; ++t) {
      int q = s + lane + 32 * t;
      bool ok = q < e;
      pf_j[t] = ok ? G_col[q] : -1;
      pf_g[t] = ok ? G_val[q] : 0.0;
    }
  };
  if (n > 0) prefetch(0);
  for (int i = 0; i < n; ++i) {
    if (agg[i] >= 0) continue;
    Cand best{0.0, 0, -1};
    if (pf_node != i) prefetch(i);
    int len = pf_len;
    int cj[AG_K];
    double cgv[AG_K];
#pragma unroll
    for (int t = 0; t < AG_K; ++t) {
      cj[t] = pf_j[t];
      cgv[t] = pf_g[t];
    }
    // next candidate: first unaggregated index after i (within 32), else i + 33
    if (i + 1 < n) {
      int k = i + 1 + lane;
      unsigned un = __ballot_sync(FULL_MASK, k < n && agg[k] < 0);
      int nxt = un ? i + 1 + __ffs(un) - 1 : min(i + 33, n - 1);
      prefetch(nxt);
    }
    if (len <= 32 * AG_K) {
#pragma unroll
      for (int t = 0; t < AG_K; ++t) {
        int j = cj[t];
        if (j >= 0) {
          int a = agg[j];
          if ((a < 0) || (size[a] < max_size)) {
            Cand c{cgv[t], a < 0 ? 1 : 0, j};
            if (better(c, best)) best = c;
          }
        }
      }
    } else {
      for (int q = G_ptr[i] + lane; q < G_ptr[i + 1]; q += 32) {
        int j = G_col[q];
        int a = agg[j];
        bool elig = (a < 0) || (size[a] < max_size);
        if (elig) {
          Cand c{G_val[q], a < 0 ? 1 : 0, j};
          if (better(c, best)) best = c;
        }
      }
    }
    best = warp_best(best);
    if (best.j >= 0) {
      int aj = agg[best.j];  // every lane reads the pre-update value
      __syncwarp();
      if (lane == 0) {
        if (aj < 0) {
          agg[i] = nagg;
          agg[best.j] = nagg;
          size[nagg] = 2;
        } else {
          agg[i] = aj;
          size[aj] += 1;
        }
      }
      if (aj < 0) ++nagg;
      __syncwarp();
    }
  }
  // post-pass over leftovers in index order
  for (int i = 0; i < n; ++i) {
    __syncwarp();
    if (agg[i] >= 0) continue;
    Cand best{0.0, 0, -1};
    for (int q = G_ptr[i] + lane; q < G_ptr[i + 1]; q += 32) {
      int j = G_col[q];
      int a = agg[j];
      if (a >= 0 && size[a] <= max_size) {
        Cand c{G_val[q], 0, j};
        if (better(c, best)) best = c;
      }
    }
    best = warp_best(best);
    __syncwarp();
    if (lane == 0) {
      if (best.j >= 0) {
        int a = agg[best.j];
        agg[i] = a;
        size[a] += 1;
      } else {
        agg[i] = nagg;
        size[nagg] = 1;
      }
    }
    if (best.j < 0) ++nagg;
    __syncwarp();
  }
  __syncwarp();
  int mx = 0;
  for (int i = lane; i < n; i += 32) {
    if (use_smem) {
      agg_g[i] = agg[i];
      size_g[i] = size[i];
    }
    if (i < nagg) mx = max(mx, size[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL_MASK, mx, o));
  if (lane == 0) {
    n_agg_out[0] = nagg;
    n_agg_out[1] = mx;
  }
}

// Same greedy scan (identical decisions), restructured around its real cost: the
// rows. The scan visits nodes in index order, so the strength rows it reads are a
// forward walk through the CSR arrays. A ring of AGR_NB batches of AGR_B entries is
// streamed into shared memory with cp.async ahead of the scan (batches of skipped
// nodes are loaded too -- sequential bytes are cheap, latency is not); the decision
// for node i then touches shared memory only (row, agg, size, G_ptr all resident).
#define AGR_B 512
#define AGR_NB 8
#define AGR_R (AGR_B * AGR_NB)

// Each strength row re-ordered by (G desc, column asc) -- the aggregation's own
// candidate key minus its dynamic "unaggregated first" tie-break -- so the scan can
// stop at the first eligible neighbour and only look further along ties of its G.
// Warp per row, bitonic network in shared memory; rows longer than RS_CAP are left
// in column order and flagged in `unsorted` (bit per row) for the full scan.
// Coarse-level operator rows run to a few thousand entries (an aggregate couples to
// the union of its members' neighbours), so the per-warp capacity lives in dynamic
// shared memory: RS_CAP keys + columns per warp, 4 warps per CTA (96 KB).
#define RS_CAP 2048
__global__ void __launch_bounds__(128)
k_rows_sort_desc(const int* __restrict__ G_ptr, const int* __restrict__ G_col, const double* __restrict__ G_val,
                 int n, int* __restrict__ col_s, double* __restrict__ val_s, unsigned* __restrict__ unsorted) {
  extern __shared__ __align__(16) unsigned long long rs_smem[];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long* skw = rs_smem + (size_t)w * RS_CAP;
  int* sjw = reinterpret_cast<int*>(rs_smem + 4 * RS_CAP) + (size_t)w * RS_CAP;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int CAP = RS_CAP;
  for (int row = warp; row < n; row += nwarps) {
    int s = G_ptr[row], L = G_ptr[row + 1] - s;
    if (L > CAP) {
      for (int t = lane; t < L; t += 32) {
        col_s[s + t] = G_col[s + t];
        val_s[s + t] = G_val[s + t];
      }
      if (lane == 0) atomicOr(unsorted + (row >> 5), 1u << (row & 31));
      continue;
    }
    int P = 32;
    while (P < L) P <<= 1;
    for (int t = lane; t < P; t += 32) {
      bool ok = t < L;
      double g = ok ? G_val[s + t] : 0.0;
      // G >= 0: its bit pattern is monotone; complement for descending order
      skw[t] = ok ? ~(unsigned long long)__double_as_longlong(g + 0.0) : ~0ull;
      sjw[t] = ok ? G_col[s + t] : 0x7fffffff;
    }
    __syncwarp();
    for (int k = 2; k <= P; k <<= 1)
      for (int jn = k >> 1; jn > 0; jn >>= 1) {
        for (int t = lane; t < P; t += 32) {
          int p = t ^ jn;
          if (p > t) {
            unsigned long long a = skw[t], b = skw[p];
            int ja = sjw[t], jb = sjw[p];
            bool gt = (a > b) || (a == b && ja > jb);
            if (gt == ((t & k) == 0)) {
              skw[t] = b;
              skw[p] = a;
              sjw[t] = jb;
              sjw[p] = ja;
            }
          }
        }
        __syncwarp();
      }
    for (int t = lane; t < L; t += 32) {
      col_s[s + t] = sjw[t];
      val_s[s + t] = __longlong_as_double((long long)~skw[t]);
    }
    __syncwarp();
  }
}

__device__ __forceinline__ void agr_issue(int bt, int64_t E, const int* __restrict__ G_col,
                                          const double* __restrict__ G_val, int* rcol, double* rval, int lane) {
  int64_t e0 = (int64_t)bt * AGR_B;
  int slot0 = (bt % AGR_NB) * AGR_B;
  constexpr int CC = AGR_B / 4, CV = AGR_B / 2;  // 16 B chunks of columns / values
  if (e0 + AGR_B <= E) {  // full batch (all but the last): plain copies, no bounds arithmetic
    const int* gc = G_col + e0;
    const double* gv = G_val + e0;
#pragma unroll
    for (int c = lane; c < CC; c += 32) cp_async16(rcol + slot0 + 4 * c, gc + 4 * c);
#pragma unroll
    for (int c = lane; c < CV; c += 32) cp_async16(rval + slot0 + 2 * c, gv + 2 * c);
    cp_async_commit();
    return;
  }
#pragma unroll 4
  for (int c = lane; c < CC + CV; c += 32) {
    if (c < CC) {
      int64_t e = e0 + 4 * c;
      int valid = (int)max((int64_t)0, min((int64_t)16, (E - e) * 4));
      cp_async16_zfill(rcol + slot0 + 4 * c, valid ? (const void*)(G_col + e) : (const void*)G_col, valid);
    } else {
      int cc = c - CC;
      int64_t e = e0 + 2 * cc;
      int valid = (int)max((int64_t)0, min((int64_t)16, (E - e) * 8));
      cp_async16_zfill(rval + slot0 + 2 * cc, valid ? (const void*)(G_val + e) : (const void*)G_val, valid);
    }
  }
  cp_async_commit();
}

__global__ void __launch_bounds__(32)
k_aggregate_ring(const int* __restrict__ G_ptr, const int* __restrict__ G_col, const double* __restrict__ G_val,
                 const unsigned* __restrict__ unsorted_g, int n, int max_size, int* __restrict__ agg_g,
                 int* __restrict__ size_g, int* __restrict__ n_agg_out) {
  extern __shared__ __align__(16) double shd[];
  double* rval = shd;                                  // AGR_R
  int* rcol = reinterpret_cast<int*>(rval + AGR_R);    // AGR_R
  int* agg = rcol + AGR_R;                             // n
  int* size = agg + n;                                 // n
  int* ptr = size + n;                                 // n + 1
  unsigned* unsorted = reinterpret_cast<unsigned*>(ptr + n + 1);  // (n + 31) / 32
  int lane = threadIdx.x;
  for (int i = lane; i < n; i += 32) {
    agg[i] = -1;
    size[i] = 0;
  }
  for (int i = lane; i <= n; i += 32) ptr[i] = G_ptr[i];
  for (int i = lane; i < (n + 31) / 32; i += 32) unsorted[i] = unsorted_g[i];
  __syncwarp();
  const int64_t E = ptr[n];
  const int nbt = (int)((E + AGR_B - 1) / AGR_B);
  int issued = 0;
  while (issued < nbt && issued < AGR_NB) agr_issue(issued++, E, G_col, G_val, rcol, rval, lane);
  int nagg = 0;
  for (int i = 0; i < n; ++i) {
    if (agg[i] >= 0) continue;
    int s = ptr[i], e = ptr[i + 1];
    Cand best{0.0, 0, -1};
    bool uniform = false;  // best already warp-uniform (sorted-row path)
    if (e - s <= (AGR_NB - 1) * AGR_B) {
      // recycle batches wholly below s, then wait for the batch holding entry e-1
      int lowb = s / AGR_B;
      while (issued < nbt && issued < lowb + AGR_NB) agr_issue(issued++, E, G_col, G_val, rcol, rval, lane);
      if (e > s) cp_async_wait_dyn(issued - 1 - (e - 1) / AGR_B);
      __syncwarp();
      if (!((unsorted[i >> 5] >> (i & 31)) & 1u)) {
        // sorted row: the answer is the first unaggregated entry among the ties of
        // the first eligible entry's G, else that first eligible entry itself
        bool have = false;
        double gf = 0.0;
        int jf = -1, ju = -1;
        for (int q0 = s; q0 < e; q0 += 32) {
          int q = q0 + lane;
          int slot = q & (AGR_R - 1);
          int j = q < e ? rcol[slot] : -1;
          double g = rval[slot];
          int a = j >= 0 ? agg[j] : -1;
          bool elig = j >= 0 && (a < 0 || size[a] < max_size);
          if (have) elig = elig && (g == gf);
          unsigned m = __ballot_sync(FULL_MASK, elig);
          if (!have) {
            if (!m) continue;
            int f = __ffs(m) - 1;
            gf = __shfl_sync(FULL_MASK, g, f);
            jf = __shfl_sync(FULL_MASK, j, f);
            have = true;
            m = __ballot_sync(FULL_MASK, elig && g == gf);
          }
          unsigned mu = __ballot_sync(FULL_MASK, elig && a < 0) & m;
          if (mu) {
            ju = __shfl_sync(FULL_MASK, j, __ffs(mu) - 1);
            break;
          }
          // ties may continue into the next chunk only if this chunk ends on one
          bool tail = __shfl_sync(FULL_MASK, q < e && g == gf, 31);
          if (!tail) break;
        }
        best.j = ju >= 0 ? ju : jf;
        uniform = true;
      } else
      // 4 entries per lane per round, loads hoisted so the smem chains
      // (column -> agg -> size) of the four overlap
      for (int q0 = s + lane; q0 < e; q0 += 128) {
        int jj[4], aa[4], ss[4];
        double gg[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          int q = q0 + 32 * u;
          int slot = q & (AGR_R - 1);
          jj[u] = q < e ? rcol[slot] : -1;
          gg[u] = rval[slot];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) aa[u] = jj[u] >= 0 ? agg[jj[u]] : -1;
#pragma unroll
        for (int u = 0; u < 4; ++u) ss[u] = aa[u] >= 0 ? size[aa[u]] : 0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (jj[u] >= 0 && (aa[u] < 0 || ss[u] < max_size)) {
            Cand c{gg[u], aa[u] < 0 ? 1 : 0, jj[u]};
            if (better(c, best)) best = c;
          }
      }
    } else {
      for (int q = s + lane; q < e; q += 32) {
        int j = G_col[q];
        int a = agg[j];
        if ((a < 0) || (size[a] < max_size)) {
          Cand c{G_val[q], a < 0 ? 1 : 0, j};
          if (better(c, best)) best = c;
        }
      }
    }
    if (!uniform) best = warp_best(best);
    if (best.j >= 0) {
      int aj = agg[best.j];  // every lane reads the pre-update value
      __syncwarp();
      if (lane == 0) {
        if (aj < 0) {
          agg[i] = nagg;
          agg[best.j] = nagg;
          size[nagg] = 2;
        } else {
          agg[i] = aj;
          size[aj] += 1;
        }
      }
      if (aj < 0) ++nagg;
    }
    __syncwarp();
  }
  cp_async_wait<0>();
  // post-pass over leftovers in index order (few nodes: rows from global memory)
  for (int i = 0; i < n; ++i) {
    __syncwarp();
    if (agg[i] >= 0) continue;
    Cand best{0.0, 0, -1};
    for (int q = ptr[i] + lane; q < ptr[i + 1]; q += 32) {
      int j = G_col[q];
      int a = agg[j];
      if (a >= 0 && size[a] <= max_size) {
        Cand c{G_val[q], 0, j};
        if (better(c, best)) best = c;
      }
    }
    best = warp_best(best);
    __syncwarp();
    if (lane == 0) {
      if (best.j >= 0) {
        int a = agg[best.j];
        agg[i] = a;
        size[a] += 1;
      } else {
        agg[i] = nagg;
        size[nagg] = 1;
      }
    }
    if (best.j < 0) ++nagg;
    __syncwarp();
  }
  __syncwarp();
  int mx = 0;
  for (int i = lane; i < n; i += 32) {
    agg_g[i] = agg[i];
    size_g[i] = size[i];
    if (i < nagg) mx = max(mx, size[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL_MASK, mx, o));
  if (lane == 0) {
    n_agg_out[0] = nagg;
    n_agg_out[1] = mx;  // largest aggregate (sizes the prolongation's shared memory)
  }
}

// Same greedy scan again (identical decisions), built around the observation that
// a visit almost always ends inside the first few entries of the sorted row: the
// first eligible neighbour is the strongest one unless its aggregate is full. Each
// row's top AH_K entries ("head": columns, strengths, row length) are packed once,
// in parallel, into a node-ordered array that the scan streams into shared memory
// in batches of AH_B nodes with cp.async, AH_NB batches ahead. A visit is then
// eight lanes doing one agg/size lookup each plus two ballots; only a visit whose
// head holds no eligible entry, or whose tie run reaches the head's end, scans the
// full sorted row (from global memory), and rows too long to sort take the
// exhaustive scan -- both with the ring kernel's exact rules.
#define AH_K 8
#define AH_B 32
#define AH_NB 4

__global__ void k_agg_heads(const int* __restrict__ G_ptr, const int* __restrict__ col_s,
                            const double* __restrict__ val_s, const unsigned* __restrict__ unsorted, int n,
                            int n_pad, int* __restrict__ hcol, double* __restrict__ hval, int* __restrict__ hlen) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)n_pad * AH_K;
       t += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(t / AH_K), e = (int)(t - (int64_t)i * AH_K);
    int c = -1;
    double g = 0.0;
    if (i < n) {
      int s = G_ptr[i], L = G_ptr[i + 1] - s;
      bool uns = (unsorted[i >> 5] >> (i & 31)) & 1u;
      if (uns) {
        c = e == 0 ? -2 : -1;  // marker: exhaustive scan
      } else if (e < L) {
        c = col_s[s + e];
        g = val_s[s + e];
      }
      if (e == 0) hlen[i] = L;
    } else if (e == 0) {
      hlen[i] = 0;
    }
    hcol[t] = c;
    hval[t] = g;
  }
}

__device__ __forceinline__ void ah_issue(int bt, const int* __restrict__ hcol_g, const double* __restrict__ hval_g,
                                         const int* __restrict__ hlen_g, int* scol, double* sval, int* slen,
                                         int lane) {
  const int slot = bt % AH_NB;
  const int64_t e0 = (int64_t)bt * AH_B * AH_K;
  constexpr int CC = AH_B * AH_K / 4, CV = AH_B * AH_K / 2, CL = AH_B / 4;  // 16 B chunks
#pragma unroll
  for (int c = lane; c < CC; c += 32) cp_async16(scol + slot * AH_B * AH_K + 4 * c, hcol_g + e0 + 4 * c);
#pragma unroll
  for (int c = lane; c < CV; c += 32) cp_async16(sval + slot * AH_B * AH_K + 2 * c, hval_g + e0 + 2 * c);
  if (lane < CL) cp_async16(slen + slot * AH_B + 4 * lane, hlen_g + (int64_t)bt * AH_B + 4 * lane);
  cp_async_commit();
}

__global__ void __launch_bounds__(32)
k_aggregate_head(const int* __restrict__ G_ptr, const int* __restrict__ G_col, const double* __restrict__ G_val,
                 const int* __restrict__ hcol_g, const double* __restrict__ hval_g, const int* __restrict__ hlen_g,
                 int n, int max_size, int* __restrict__ agg_g, int* __restrict__ size_g, int* __restrict__ n_agg_out) {
  extern __shared__ __align__(16) double shh[];
  double* sval = shh;                                           // AH_NB * AH_B * AH_K
  int* scol = reinterpret_cast<int*>(sval + AH_NB * AH_B * AH_K);  // AH_NB * AH_B * AH_K
  int* slen = scol + AH_NB * AH_B * AH_K;                       // AH_NB * AH_B
  int* agg = slen + AH_NB * AH_B;                               // n
  int* size = agg + n;                                          // n
  const int lane = threadIdx.x;
  for (int i = lane; i < n; i += 32) {
    agg[i] = -1;
    size[i] = 0;
  }
  const int nbt = (n + AH_B - 1) / AH_B;
#pragma unroll 1
  for (int b = 0; b < AH_NB; ++b) {
    if (b < nbt) ah_issue(b, hcol_g, hval_g, hlen_g, scol, sval, slen, lane);
    else cp_async_commit();
  }
  __syncwarp();
  int nagg = 0;
  for (int b = 0; b < nbt; ++b) {
    cp_async_wait<AH_NB - 1>();
    __syncwarp();
    const int slot = b % AH_NB;
    const int iend = min(AH_B, n - b * AH_B);
    for (int ii = 0; ii < iend; ++ii) {
      const int i = b * AH_B + ii;
      if (agg[i] >= 0) continue;
      int j = -1;
      double g = 0.0;
      if (lane < AH_K) {
        j = scol[(slot * AH_B + ii) * AH_K + lane];
        g = sval[(slot * AH_B + ii) * AH_K + lane];
      }
      const int len = slen[slot * AH_B + ii];
      int bj = -1;
      bool full_scan = __shfl_sync(FULL_MASK, j, 0) == -2;
      bool row_scan = false;
      if (!full_scan) {
        int a = j >= 0 ? agg[j] : -1;
        bool elig = j >= 0 && (a < 0 || size[a] < max_size);
        unsigned m = __ballot_sync(FULL_MASK, elig);
        if (m) {
          int f = __ffs(m) - 1;
          double gf = __shfl_sync(FULL_MASK, g, f);
          unsigned tie = __ballot_sync(FULL_MASK, elig && g == gf);
          unsigned mu = __ballot_sync(FULL_MASK, elig && g == gf && a < 0);
          if (mu) {
            bj = __shfl_sync(FULL_MASK, j, __ffs(mu) - 1);
          } else {
            // the last head entry continuing the tie run: later entries may hold an
            // unaggregated tie, which would win
            bool tail = __shfl_sync(FULL_MASK, j >= 0 && g == gf, AH_K - 1);
            if (tail && len > AH_K) row_scan = true;
            else bj = __shfl_sync(FULL_MASK, j, f);
            (void)tie;
          }
        } else if (len > AH_K) {
          row_scan = true;
        }
      }
      if (row_scan) {
        // sorted row from global memory, the ring kernel's rule
        const int s = G_ptr[i], e = G_ptr[i + 1];
        bool have = false;
        double gf = 0.0;
        int jf = -1, ju = -1;
        for (int q0 = s; q0 < e; q0 += 32) {
          int q = q0 + lane;
          int jj = q < e ? G_col[q] : -1;
          double gg = q < e ? G_val[q] : 0.0;
          int a = jj >= 0 ? agg[jj] : -1;
          bool elig = jj >= 0 && (a < 0 || size[a] < max_size);
          if (have) elig = elig && (gg == gf);
          unsigned m = __ballot_sync(FULL_MASK, elig);
          if (!have) {
            if (!m) continue;
            int f = __ffs(m) - 1;
            gf = __shfl_sync(FULL_MASK, gg, f);
            jf = __shfl_sync(FULL_MASK, jj, f);
            have = true;
            m = __ballot_sync(FULL_MASK, elig && gg == gf);
          }
          unsigned mu = __ballot_sync(FULL_MASK, elig && a < 0) & m;
          if (mu) {
            ju = __shfl_sync(FULL_MASK, jj, __ffs(mu) - 1);
            break;
          }
          bool tail = __shfl_sync(FULL_MASK, q < e && gg == gf, 31);
          if (!tail) break;
        }
        bj = ju >= 0 ? ju : jf;
      } else if (full_scan) {
        Cand best{0.0, 0, -1};
        for (int q = G_ptr[i] + lane; q < G_ptr[i + 1]; q += 32) {
          int jj = G_col[q];
          int a = agg[jj];
          if ((a < 0) || (size[a] < max_size)) {
            Cand c{G_val[q], a < 0 ? 1 : 0, jj};
            if (better(c, best)) best = c;
          }
        }
        bj = warp_best(best).j;
      }
      if (bj >= 0) {
        int aj = agg[bj];  // every lane reads the pre-update value
        __syncwarp();
        if (lane == 0) {
          if (aj < 0) {
            agg[i] = nagg;
            agg[bj] = nagg;
            size[nagg] = 2;
          } else {
            agg[i] = aj;
            size[aj] += 1;
          }
        }
        if (aj < 0) ++nagg;
      }
      __syncwarp();
    }
    __syncwarp();  // every lane is done with this slot before it is refilled
    if (b + AH_NB < nbt) ah_issue(b + AH_NB, hcol_g, hval_g, hlen_g, scol, sval, slen, lane);
    else cp_async_commit();
  }
  cp_async_wait<0>();
  // post-pass over leftovers in index order (few nodes: rows from global memory)
  for (int i = 0; i < n; ++i) {
    __syncwarp();
    if (agg[i] >= 0) continue;
    Cand best{0.0, 0, -1};
    for (int q = G_ptr[i] + lane; q < G_ptr[i + 1]; q += 32) {
      int j = G_col[q];
      int a = agg[j];
      if (a >= 0 && size[a] <= max_size) {
        Cand c{G_val[q], 0, j};
        if (better(c, best)) best = c;
      }
    }
    best = warp_best(best);
    __syncwarp();
    if (lane == 0) {
      if (best.j >= 0) {
        int a = agg[best.j];
        agg[i] = a;
        size[a] += 1;
      } else {
        agg[i] = nagg;
        size[nagg] = 1;
      }
    }
    if (best.j < 0) ++nagg;
    __syncwarp();
  }
  __syncwarp();
  int mx = 0;
  for (int i = lane; i < n; i += 32) {
    agg_g[i] = agg[i];
    size_g[i] = size[i];
    if (i < nagg) mx = max(mx, size[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL_MASK, mx, o));
  if (lane == 0) {
    n_agg_out[0] = nagg;
    n_agg_out[1] = mx;
  }
}

// ---------------------------------------------------------------------------
// Speculative form of the same scan (identical decisions, fewer dependent steps).
// The 32 nodes of a head batch are decided in parallel, one per lane, from the state
// at the batch start; the batch is then committed in index order. A lane's decision
// depends only on its examined head entries (the first eligible entry, the tie run of
// its strength, the chosen entry) through two facts per entry: assigned or not, and
// whether its aggregate is full. Both change monotonically and only through commits,
// so every commit broadcasts (node, partner, aggregate, became-full) and later lanes
// whose examined entries it touches fall back to the cooperative visit of
// k_aggregate_head at their turn (as do visits that need the sorted row or the
// exhaustive scan). The result equals the sequential scan's decision for decision.

// cooperative visit of node i (the whole warp; state in shared memory)
__device__ __forceinline__ int agg_visit_coop(int i, const int* __restrict__ G_ptr, const int* __restrict__ G_col,
                                              const double* __restrict__ G_val, const int* hc, const double* hv,
                                              int len, const int* agg, const int* size, int max_size, int lane) {
  int j = -1;
  double g = 0.0;
  if (lane < AH_K) {
    j = hc[lane];
    g = hv[lane];
  }
  int bj = -1;
  bool full_scan = __shfl_sync(FULL_MASK, j, 0) == -2;
  bool row_scan = false;
  if (!full_scan) {
    int a = j >= 0 ? agg[j] : -1;
    bool elig = j >= 0 && (a < 0 || size[a] < max_size);
    unsigned m = __ballot_sync(FULL_MASK, elig);
    if (m) {
      int f = __ffs(m) - 1;
      double gf = __shfl_sync(FULL_MASK, g, f);
      unsigned mu = __ballot_sync(FULL_MASK, elig && g == gf && a < 0);
      if (mu) {
        bj = __shfl_sync(FULL_MASK, j, __ffs(mu) - 1);
      } else {
        bool tail = __shfl_sync(FULL_MASK, j >= 0 && g == gf, AH_K - 1);
        if (tail && len > AH_K) row_scan = true;
        else bj = __shfl_sync(FULL_MASK, j, f);
      }
    } else if (len > AH_K) {
      row_scan = true;
    }
  }
  if (row_scan) {
    const int s0 = G_ptr[i], e0 = G_ptr[i + 1];
    bool have = false;
    double gf = 0.0;
    int jf = -1, ju = -1;
    for (int q0 = s0; q0 < e0; q0 += 32) {
      int q = q0 + lane;
      int jj = q < e0 ? G_col[q] : -1;
      double gg = q < e0 ? G_val[q] : 0.0;
      int a = jj >= 0 ? agg[jj] : -1;
      bool elig = jj >= 0 && (a < 0 || size[a] < max_size);
      if (have) elig = elig && (gg == gf);
      unsigned m = __ballot_sync(FULL_MASK, elig);
      if (!have) {
        if (!m) continue;
        int f = __ffs(m) - 1;
        gf = __shfl_sync(FULL_MASK, gg, f);
        jf = __shfl_sync(FULL_MASK, jj, f);
        have = true;
        m = __ballot_sync(FULL_MASK, elig && gg == gf);
      }
      unsigned mu = __ballot_sync(FULL_MASK, elig && a < 0) & m;
      if (mu) {
        ju = __shfl_sync(FULL_MASK, jj, __ffs(mu) - 1);
        break;
      }
      bool tail = __shfl_sync(FULL_MASK, q < e0 && gg == gf, 31);
      if (!tail) break;
    }
    bj = ju >= 0 ? ju : jf;
  } else if (full_scan) {
    Cand best{0.0, 0, -1};
    for (int q = G_ptr[i] + lane; q < G_ptr[i + 1]; q += 32) {
      int jj = G_col[q];
      int a = agg[jj];
      if ((a < 0) || (size[a] < max_size)) {
        Cand c{G_val[q], a < 0 ? 1 : 0, jj};
        if (better(c, best)) best = c;
      }
    }
    bj = warp_best(best).j;
  }
  return bj;
}

__global__ void __launch_bounds__(32)
k_aggregate_spec(const int* __restrict__ G_ptr, const int* __restrict__ G_col, const double* __restrict__ G_val,
                 const int* __restrict__ hcol_g, const double* __restrict__ hval_g, const int* __restrict__ hlen_g,
                 int n, int max_size, int* __restrict__ agg_g, int* __restrict__ size_g, int* __restrict__ n_agg_out) {
  extern __shared__ __align__(16) double shh[];
  double* sval = shh;                                           // AH_NB * AH_B * AH_K
  int* scol = reinterpret_cast<int*>(sval + AH_NB * AH_B * AH_K);  // AH_NB * AH_B * AH_K
  int* slen = scol + AH_NB * AH_B * AH_K;                       // AH_NB * AH_B
  int* sd_ex = slen + AH_NB * AH_B;                             // AH_B * AH_K examined entries
  int* sd_code = sd_ex + AH_B * AH_K;                           // AH_B * AH_K their state code
  int* sd_dec = sd_code + AH_B * AH_K;                          // AH_B decisions (-3: none usable)
  int* agg = sd_dec + AH_B;                                     // n
  int* size = agg + n;                                          // n
  unsigned* pmask = reinterpret_cast<unsigned*>(size + n);      // n: lanes of a round pairing with node j
  unsigned* jmask = pmask + n;                                  // n: lanes of a round joining aggregate a
  const int lane = threadIdx.x;
  for (int i = lane; i < n; i += 32) {
    agg[i] = -1;
    size[i] = 0;
    pmask[i] = 0u;
    jmask[i] = 0u;
  }
  const int nbt = (n + AH_B - 1) / AH_B;
#pragma unroll 1
  for (int b = 0; b < AH_NB; ++b) {
    if (b < nbt) ah_issue(b, hcol_g, hval_g, hlen_g, scol, sval, slen, lane);
    else cp_async_commit();
  }
  __syncwarp();
  int nagg = 0;
  const unsigned lt = (1u << lane) - 1u;
#ifdef AGG_STATS
  int st_turn = 0, st_coop = 0, st_nospec = 0;
#endif
  for (int b = 0; b < nbt; ++b) {
    cp_async_wait<AH_NB - 1>();
    __syncwarp();
    const int slot = b % AH_NB;
    const int iend = min(AH_B, n - b * AH_B);
    const int i_me = b * AH_B + lane;
    const int* hc = scol + (slot * AH_B + lane) * AH_K;
    const double* hv = sval + (slot * AH_B + lane) * AH_K;
    // ---- phase 1: every lane decides its node from the batch-start state and
    // records what the decision read: each examined entry with a state code
    // (-1 unassigned, a assigned to eligible aggregate a, a | 1 << 30 assigned to a
    // full one -- fixed for good, sizes only grow)
    int dec = -3;
    int ex[AH_K], code[AH_K];
#pragma unroll
    for (int e = 0; e < AH_K; ++e) {
      ex[e] = -1;
      code[e] = -1;
    }
    if (lane < iend && agg[i_me] < 0) {
      const int len = slen[slot * AH_B + lane];
      int jj[AH_K];
      double gg[AH_K];
      int aa[AH_K];
#pragma unroll
      for (int e = 0; e < AH_K; ++e) {
        jj[e] = hc[e];
        gg[e] = hv[e];
      }
#pragma unroll
      for (int e = 0; e < AH_K; ++e) aa[e] = jj[e] >= 0 ? agg[jj[e]] : -1;
      bool el[AH_K];
#pragma unroll
      for (int e = 0; e < AH_K; ++e) el[e] = jj[e] >= 0 && (aa[e] < 0 || size[aa[e]] < max_size);
      if (jj[0] != -2) {
        int f = -1;
#pragma unroll
        for (int e = AH_K - 1; e >= 0; --e)
          if (el[e]) f = e;
        int last = AH_K - 1;
        if (f < 0) {
          if (len <= AH_K) dec = -1;  // no eligible neighbour at all: stays unassigned for now
        } else {
          double gf = gg[f];
          int cu = -1;
          last = f;
#pragma unroll
          for (int e = 0; e < AH_K; ++e) {
            if (e >= f && jj[e] >= 0 && gg[e] == gf) {
              if (cu < 0) last = e;
              if (cu < 0 && el[e] && aa[e] < 0) cu = e;
            }
          }
          bool tail = jj[AH_K - 1] >= 0 && gg[AH_K - 1] == gf;
          if (cu >= 0) dec = jj[cu];
          else if (!(tail && len > AH_K)) dec = jj[f];
        }
#pragma unroll
        for (int e = 0; e < AH_K; ++e)
          if (e <= last) {
            ex[e] = jj[e];
            code[e] = aa[e] < 0 ? -1 : (el[e] ? aa[e] : (aa[e] | (1 << 30)));
          }
      }
    }
#pragma unroll
    for (int e = 0; e < AH_K; ++e) {
      sd_ex[lane * AH_K + e] = ex[e];
      sd_code[lane * AH_K + e] = code[e];
    }
    sd_dec[lane] = dec;
    __syncwarp();
    // ---- phase 2: commit in index order, in rounds. A decision stands iff none of
    // the entries it read changed state since the batch start (unassigned ->
    // assigned, eligible -> full; both monotone). A round starts at lane p: every
    // later lane whose decision still stands publishes its effect (pair with node d:
    // pmask[d] |= lane bit; join aggregate a: jmask[a] |= lane bit), then each lane
    // checks the effects of the EARLIER lanes of the round on what it read (an
    // examined node assigned by an earlier lane's own node or pairing, an examined
    // aggregate filled by earlier joins, its own node taken as a partner). Lanes
    // p .. q-1 before the first conflict commit together -- exactly what the
    // one-at-a-time scan does for them -- and lane q is resolved alone with the
    // current state (cooperative visit if its decision no longer stands).
    int p = 0;
    while (p < iend) {
      const bool inr = lane >= p && lane < iend;
      const bool assigned = inr && agg[i_me] >= 0;
      const int d = sd_dec[lane];
      bool pend = inr && !assigned && d != -3;
      if (pend) {
        bool ch = false;
#pragma unroll
        for (int e = 0; e < AH_K; ++e)
          if (ex[e] >= 0) ch |= (code[e] < 0) ? (agg[ex[e]] >= 0) : (!(code[e] >> 30) && size[code[e]] >= max_size);
        pend = !ch;
      }
      int tgt = -1;
      bool pair = false;
      if (pend && d >= 0) {
        const int a = agg[d];
        pair = a < 0;
        tgt = pair ? d : a;
        if (pair) atomicOr(pmask + d, 1u << lane);
        else atomicOr(jmask + a, 1u << lane);
      }
      const unsigned C = __ballot_sync(FULL_MASK, pend && d >= 0);  // lanes whose commit changes state
      __syncwarp();
      bool conflict = inr && !assigned && !pend;
      if (pend) {
        if (pmask[i_me] & lt) conflict = true;  // taken as an earlier lane's partner
#pragma unroll
        for (int e = 0; e < AH_K; ++e) {
          const int j = ex[e];
          if (j < 0) continue;
          const int l = j - b * AH_B;
          if (l >= 0 && l < lane && ((C >> l) & 1u)) conflict = true;  // node of an earlier committer
          if (pmask[j] & lt) conflict = true;                          // an earlier lane's partner
          const int c = code[e];
          if (c >= 0 && !(c >> 30) && __popc(jmask[c] & lt) >= max_size - size[c]) conflict = true;
        }
      }
      const unsigned cm = __ballot_sync(FULL_MASK, conflict);
      const int q = cm ? __ffs(cm) - 1 : iend;
      const unsigned range = (q >= 32 ? 0xffffffffu : ((1u << q) - 1u)) & ~((1u << p) - 1u);
      const unsigned pairs = __ballot_sync(FULL_MASK, pend && d >= 0 && pair) & range;
      __syncwarp();
      if (((range >> lane) & 1u) && pend && d >= 0) {
        if (pair) {
          const int id = nagg + __popc(pairs & lt);
          agg[i_me] = id;
          agg[d] = id;
          size[id] = 2;
        } else {
          agg[i_me] = tgt;
          const unsigned jm = jmask[tgt] & range;
          if (lane == __ffs(jm) - 1) size[tgt] += __popc(jm);
        }
      }
      nagg += __popc(pairs);
      __syncwarp();
      if (pend && d >= 0) {
        if (pair) pmask[d] = 0u;
        else jmask[tgt] = 0u;
      }
      __syncwarp();
#ifdef AGG_STATS
      ++st_turn;
#endif
      if (q < iend) {  // lane q alone, with the current state
        const int ii = q, i = b * AH_B + q;
        if (agg[i] < 0) {
          int bj = sd_dec[ii];
          bool ok = bj != -3;
          if (ok) {
            bool ch = false;
            if (lane < AH_K) {
              const int jx = sd_ex[ii * AH_K + lane], c = sd_code[ii * AH_K + lane];
              if (jx >= 0) ch = (c < 0) ? (agg[jx] >= 0) : (!(c >> 30) && size[c] >= max_size);
            }
            ok = __ballot_sync(FULL_MASK, ch) == 0u;
          }
#ifdef AGG_STATS
          if (!ok) ++st_coop;
#endif
          if (!ok)
            bj = agg_visit_coop(i, G_ptr, G_col, G_val, scol + (slot * AH_B + ii) * AH_K,
                                sval + (slot * AH_B + ii) * AH_K, slen[slot * AH_B + ii], agg, size, max_size, lane);
          if (bj >= 0) {
            const int aj = agg[bj];
            __syncwarp();
            if (lane == 0) {
              if (aj < 0) {
                agg[i] = nagg;
                agg[bj] = nagg;
                size[nagg] = 2;
              } else {
                agg[i] = aj;
                size[aj] += 1;
              }
            }
            if (aj < 0) ++nagg;
          }
        }
        __syncwarp();
      }
      p = q + 1;
    }
    __syncwarp();
    if (b + AH_NB < nbt) ah_issue(b + AH_NB, hcol_g, hval_g, hlen_g, scol, sval, slen, lane);
    else cp_async_commit();
  }
  cp_async_wait<0>();
#ifdef AGG_STATS
  if (lane == 0) printf("agg_spec n=%d turns=%d coop=%d nospec=%d\n", n, st_turn, st_coop, st_nospec);
#endif
  // post-pass over leftovers in index order (multigrid.py:164-175)
  for (int i = 0; i < n; ++i) {
    __syncwarp();
    if (agg[i] >= 0) continue;
    Cand best{0.0, 0, -1};
    for (int q = G_ptr[i] + lane; q < G_ptr[i + 1]; q += 32) {
      int j = G_col[q];
      int a = agg[j];
      if (a >= 0 && size[a] <= max_size) {
        Cand c{G_val[q], 0, j};
        if (better(c, best)) best = c;
      }
    }
    best = warp_best(best);
    __syncwarp();
    if (lane == 0) {
      if (best.j >= 0) {
        int a = agg[best.j];
        agg[i] = a;
        size[a] += 1;
      } else {
        agg[i] = nagg;
        size[nagg] = 1;
      }
    }
    if (best.j < 0) ++nagg;
    __syncwarp();
  }
  __syncwarp();
  int mx = 0;
  for (int i = lane; i < n; i += 32) {
    agg_g[i] = agg[i];
    size_g[i] = size[i];
    if (i < nagg) mx = max(mx, size[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL_MASK, mx, o));
  if (lane == 0) {
    n_agg_out[0] = nagg;
    n_agg_out[1] = mx;
  }
}

// ---------------------------------------------------------------------------
// Low-latency sequential form of the same scan (identical decisions). On the coarse
// levels the neighbours of a node sit a few indices away, so most of a speculative
// batch conflicts and its rounds cost ~500 cycles per node. Here lane 0 alone walks the
// batch's unassigned nodes (a register mask, built by one ballot per batch) and decides
// every node whose top head entry is not tied with the second one: one state load, the
// decision, the stores -- same-thread ordering, no warp synchronisation per node. ncu:
// ~24 instructions per node at ~7.7 cycles each (fixed-latency dependency waits 3.2,
// shared-memory scoreboard 2.9), i.e. the single-warp issue limit of a dependent chain.
// Ties, ineligible tops and unsorted rows take the general head rule (every lane
// redundantly, broadcast loads, no shuffles) or the cooperative row visit of
// k_aggregate_head.
__global__ void __launch_bounds__(32)
k_aggregate_seq(const int* __restrict__ G_ptr, const int* __restrict__ G_col, const double* __restrict__ G_val,
                const int* __restrict__ hcol_g, const double* __restrict__ hval_g, const int* __restrict__ hlen_g,
                int n, int max_size, int* __restrict__ agg_g, int* __restrict__ size_g, int* __restrict__ n_agg_out) {
  extern __shared__ __align__(16) double shh[];
  double* sval = shh;                                              // AH_NB * AH_B * AH_K
  int* scol = reinterpret_cast<int*>(sval + AH_NB * AH_B * AH_K);  // AH_NB * AH_B * AH_K
  int* slen = scol + AH_NB * AH_B * AH_K;                          // AH_NB * AH_B
  int* tops = slen + AH_NB * AH_B;                                 // AH_B: the current batch's top entries
  int* agg = tops + AH_B;                                          // n
  int* size = agg + n;                                             // n
  const int lane = threadIdx.x;
  for (int i = lane; i < n; i += 32) {
    agg[i] = -1;
    size[i] = 0;
  }
  const int nbt = (n + AH_B - 1) / AH_B;
#pragma unroll 1
  for (int b = 0; b < AH_NB; ++b) {
    if (b < nbt) ah_issue(b, hcol_g, hval_g, hlen_g, scol, sval, slen, lane);
    else cp_async_commit();
  }
  __syncwarp();
  int nagg = 0;
#ifdef AGG_STATS
  int st_slow = 0, st_coop = 0, st_none = 0;
#endif
  for (int b = 0; b < nbt; ++b) {
    cp_async_wait<AH_NB - 1>();
    __syncwarp();
    const int slot = b % AH_NB;
    const int iend = min(AH_B, n - b * AH_B);
    const int base = b * AH_B;
    // per batch, all lanes: each node's deciding top entry (-1: tied with the second entry,
    // no entry, or an unsorted row -> the general rule) and the unassigned nodes' mask
    {
      const int j0 = scol[(slot * AH_B + lane) * AH_K];
      const double2 g = *reinterpret_cast<const double2*>(sval + (slot * AH_B + lane) * AH_K);
      tops[lane] = (j0 >= 0 && g.x != g.y) ? j0 : -1;
    }
    unsigned todo = __ballot_sync(FULL_MASK, lane < iend && agg[base + lane] < 0);
    __syncwarp();
    while (todo) {  // warp uniform
      // fast path, lane 0 alone (same-thread ordering, no warp synchronisation per
      // node): an untied top entry wins as soon as it is eligible -- pair if unassigned,
      // join if its aggregate has room. The batch's unassigned nodes are a register
      // mask (a partner inside the batch clears its own bit), so the dependent chain
      // per node is one state load, the decision, the stores.
      int stop = -1, nagg0 = nagg;
      if (lane == 0) {
        unsigned t = todo;
        while (t) {
          const int k = __ffs(t) - 1;
          const int j0 = tops[k];
          if (j0 < 0) {
            stop = k;
            break;
          }
          const int a0 = agg[j0];
          if (a0 < 0) {
            agg[base + k] = nagg0;
            agg[j0] = nagg0;
            size[nagg0] = 2;
            ++nagg0;
            t &= t - 1;
            const unsigned d = (unsigned)(j0 - base);
            if (d < 32u) t &= ~(1u << d);
            continue;
          }
          if (size[a0] < max_size) {
            agg[base + k] = a0;
            size[a0] += 1;
            t &= t - 1;
            continue;
          }
          stop = k;  // its aggregate is full: the general rule looks further
          break;
        }
      }
      stop = __shfl_sync(FULL_MASK, stop, 0);
      nagg = __shfl_sync(FULL_MASK, nagg0, 0);
      __syncwarp();
      if (stop < 0) break;
      // general rule for node `stop`, every lane redundantly (broadcast loads)
#ifdef AGG_STATS
      ++st_slow;
#endif
      const int i = b * AH_B + stop;
      const int* hc = scol + (slot * AH_B + stop) * AH_K;
      const double* hv = sval + (slot * AH_B + stop) * AH_K;
      const int len = slen[slot * AH_B + stop];
      int jj[AH_K], aa[AH_K];
      double gg[AH_K];
#pragma unroll
      for (int e = 0; e < AH_K; ++e) {
        jj[e] = hc[e];
        gg[e] = hv[e];
      }
#pragma unroll
      for (int e = 0; e < AH_K; ++e) aa[e] = jj[e] >= 0 ? agg[jj[e]] : -1;
      int dec = -3;
      if (jj[0] != -2) {
        bool el[AH_K];
#pragma unroll
        for (int e = 0; e < AH_K; ++e) el[e] = jj[e] >= 0 && (aa[e] < 0 || size[aa[e]] < max_size);
        int f = -1;
#pragma unroll
        for (int e = AH_K - 1; e >= 0; --e)
          if (el[e]) f = e;
        if (f < 0) {
          if (len <= AH_K) dec = -1;  // no eligible neighbour: left for the post-pass
        } else {
          double gf = 0.0;
#pragma unroll
          for (int e = 0; e < AH_K; ++e)
            if (e == f) gf = gg[e];
          int cu = -1, jf = -1;
#pragma unroll
          for (int e = AH_K - 1; e >= 0; --e) {
            if (e == f) jf = jj[e];
            if (e >= f && jj[e] >= 0 && gg[e] == gf && el[e] && aa[e] < 0) cu = jj[e];
          }
          const bool tail = jj[AH_K - 1] >= 0 && gg[AH_K - 1] == gf;
          if (cu >= 0) dec = cu;
          else if (!(tail && len > AH_K)) dec = jf;
        }
      }
      int bj = dec;
#ifdef AGG_STATS
      if (dec == -3) ++st_coop;
      if (dec == -1) ++st_none;
#endif
      if (dec == -3) bj = agg_visit_coop(i, G_ptr, G_col, G_val, hc, hv, len, agg, size, max_size, lane);
      if (bj >= 0) {
        const int aj = agg[bj];  // every lane reads the pre-update value
        __syncwarp();
        if (lane == 0) {
          if (aj < 0) {
            agg[i] = nagg;
            agg[bj] = nagg;
            size[nagg] = 2;
          } else {
            agg[i] = aj;
            size[aj] += 1;
          }
        }
        if (aj < 0) ++nagg;
        __syncwarp();
      }
      // the nodes after `stop` that are still unassigned (the visit above may have taken one)
      todo = __ballot_sync(FULL_MASK, lane > stop && lane < iend && agg[base + lane] < 0);
    }
    __syncwarp();  // every lane is done with this slot before it is refilled
    if (b + AH_NB < nbt) ah_issue(b + AH_NB, hcol_g, hval_g, hlen_g, scol, sval, slen, lane);
    else cp_async_commit();
  }
  cp_async_wait<0>();
#ifdef AGG_STATS
  if (lane == 0) printf("agg_seq n=%d slow=%d coop=%d none=%d\n", n, st_slow, st_coop, st_none);
#endif
  // post-pass over leftovers in index order (multigrid.py:164-175); a leftover's visit
  // assigns only itself, so the unassigned set of a 32-node window is read once
  for (int i0 = 0; i0 < n; i0 += 32) {
    __syncwarp();
    unsigned todo = __ballot_sync(FULL_MASK, i0 + lane < n && agg[i0 + lane] < 0);
    while (todo) {
      const int i = i0 + __ffs(todo) - 1;
      todo &= todo - 1;
      Cand best{0.0, 0, -1};
      for (int q = G_ptr[i] + lane; q < G_ptr[i + 1]; q += 32) {
        int j = G_col[q];
        int a = agg[j];
        if (a >= 0 && size[a] <= max_size) {
          Cand c{G_val[q], 0, j};
          if (better(c, best)) best = c;
        }
      }
      best = warp_best(best);
      __syncwarp();
      if (lane == 0) {
        if (best.j >= 0) {
          int a = agg[best.j];
          agg[i] = a;
          size[a] += 1;
        } else {
          agg[i] = nagg;
          size[nagg] = 1;
        }
      }
      if (best.j < 0) ++nagg;
      __syncwarp();
    }
  }
  __syncwarp();
  int mx = 0;
  for (int i = lane; i < n; i += 32) {
    agg_g[i] = agg[i];
    size_g[i] = size[i];
    if (i < nagg) mx = max(mx, size[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL_MASK, mx, o));
  if (lane == 0) {
    n_agg_out[0] = nagg;
    n_agg_out[1] = mx;
  }
}

extern "C" int bamg_aggregate(bamg_ctx* ctx, const int32_t* G_ptr, const int32_t* G_col, const double* G_val,
                              int32_t n, int32_t max_size, int32_t* agg, int32_t* size_work, int32_t* n_agg_dev,
                              int64_t nnz_cap, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (n <= 0) {
    BAMG_CUDA_CHECK(cudaMemsetAsync(n_agg_dev, 0, 2 * sizeof(int), st));
    return 0;
  }
  const int nwords = (n + 31) / 32;
  size_t smr = (size_t)AGR_R * (sizeof(double) + sizeof(int)) + sizeof(int) * (3 * (size_t)n + 1) +
               sizeof(unsigned) * (size_t)nwords;
  static const bool ring_on = [] {
    const char* e = getenv("BAMG_AGG_RING");
    return !(e && e[0] == '0');
  }();
  if (ring_on && smr <= 220 * 1024) {
    size_t ne = (size_t)(nnz_cap > 0 ? nnz_cap : 1);  // sorted copies sized by capacity: no readback
    int* col_s = nullptr;
    double* val_s = nullptr;
    unsigned* uns = nullptr;
    BAMG_CUDA_CHECK(cudaMallocAsync(&val_s, sizeof(double) * ne, st));
    BAMG_CUDA_CHECK(cudaMallocAsync(&col_s, sizeof(int) * ne, st));
    BAMG_CUDA_CHECK(cudaMallocAsync(&uns, sizeof(unsigned) * (size_t)nwords, st));
    BAMG_CUDA_CHECK(cudaMemsetAsync(uns, 0, sizeof(unsigned) * (size_t)nwords, st));
    static bool rs_attr = false;
    const size_t rs_sm = (size_t)4 * RS_CAP * (sizeof(unsigned long long) + sizeof(int));
    if (!rs_attr) {
      BAMG_CUDA_CHECK(cudaFuncSetAttribute(k_rows_sort_desc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs_sm));
      rs_attr = true;
    }
    launch(k_rows_sort_desc, grid_for((int64_t)n * 32, 128, 2), 128, rs_sm, st, G_ptr, G_col, G_val, n, col_s, val_s, uns);
    static size_t attr = 0;
    if (smr > attr) {
      BAMG_CUDA_CHECK(cudaFuncSetAttribute(k_aggregate_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smr));
      attr = smr;
    }
    static const bool head_on = [] {
      const char* e = getenv("BAMG_AGG_HEAD");
      return !(e && e[0] == '0');
    }();
    const int n_pad = ((n + AH_B - 1) / AH_B) * AH_B;
    const size_t smh = (size_t)AH_NB * AH_B * AH_K * (sizeof(double) + sizeof(int)) +
                       (size_t)AH_NB * AH_B * sizeof(int) + (size_t)AH_B * (2 * AH_K + 1) * sizeof(int) +
                       4 * sizeof(int) * (size_t)n;
    static int smem_optin = 0;
    if (!smem_optin) {
      int dev = 0;
      cudaGetDevice(&dev);
      if (cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
        smem_optin = 220 * 1024;
    }
    if (head_on && smh <= (size_t)smem_optin) {
      int *hcol = nullptr, *hlen = nullptr;
      double* hval = nullptr;
      BAMG_CUDA_CHECK(cudaMallocAsync(&hcol, sizeof(int) * (size_t)n_pad * AH_K, st));
      BAMG_CUDA_CHECK(cudaMallocAsync(&hval, sizeof(double) * (size_t)n_pad * AH_K, st));
      BAMG_CUDA_CHECK(cudaMallocAsync(&hlen, sizeof(int) * (size_t)n_pad, st));
      launch(k_agg_heads, grid_for((int64_t)n_pad * AH_K, 256), 256, 0, st, G_ptr, (const int*)col_s,
             (const double*)val_s, (const unsigned*)uns, n, n_pad, hcol, hval, hlen);
      static size_t hattr = 0;
      if (smh > hattr) {
        BAMG_CUDA_CHECK(cudaFuncSetAttribute(k_aggregate_head, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smh));
        hattr = smh;
      }
      static const bool spec_on = [] {
        const char* e = getenv("BAMG_AGG_SPEC");
        return !(e && e[0] == '0');
      }();
      // default: the low-latency sequential scan (config 4: level 0 2.8 -> 1.8 ms, coarse
      // levels 2.5 -> 1.1 ms; config 5: 6.0 -> 1.0 and 3.6 -> 0.8 ms against the
      // speculative rounds, tools/agg_ab.py); BAMG_AGG_SEQ=0 selects the speculative kernel
      static const bool use_seq = [] {
        const char* e = getenv("BAMG_AGG_SEQ");
        return !(e && e[0] == '0');
      }();
      if (use_seq) {
        static size_t qattr = 0;
        if (smh > qattr) {
          BAMG_CUDA_CHECK(cudaFuncSetAttribute(k_aggregate_seq, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smh));
          qattr = smh;
        }
        launch(k_aggregate_seq, 1, 32, smh, st, G_ptr, (const int*)col_s, (const double*)val_s, (const int*)hcol,
               (const double*)hval, (const int*)hlen, n, max_size, agg, size_work, n_agg_dev);
      } else if (spec_on) {
        static size_t sattr = 0;
        if (smh > sattr) {
          BAMG_CUDA_CHECK(cudaFuncSetAttribute(k_aggregate_spec, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smh));
          sattr = smh;
        }
        launch(k_aggregate_spec, 1, 32, smh, st, G_ptr, (const int*)col_s, (const double*)val_s, (const int*)hcol,
               (const double*)hval, (const int*)hlen, n, max_size, agg, size_work, n_agg_dev);
      } else {
        launch(k_aggregate_head, 1, 32, smh, st, G_ptr, (const int*)col_s, (const double*)val_s, (const int*)hcol,
               (const double*)hval, (const int*)hlen, n, max_size, agg, size_work, n_agg_dev);
      }
      BAMG_CUDA_CHECK(cudaFreeAsync(hcol, st));
      BAMG_CUDA_CHECK(cudaFreeAsync(hval, st));
      BAMG_CUDA_CHECK(cudaFreeAsync(hlen, st));
    } else {
      launch(k_aggregate_ring, 1, 32, smr, st, G_ptr, (const int*)col_s, (const double*)val_s, (const unsigned*)uns,
             n, max_size, agg, size_work, n_agg_dev);
    }
    BAMG_CUDA_CHECK(cudaFreeAsync(val_s, st));
    BAMG_CUDA_CHECK(cudaFreeAsync(col_s, st));
    BAMG_CUDA_CHECK(cudaFreeAsync(uns, st));
    BAMG_LAUNCH_CHECK();
    return 0;
  }
  size_t sm = sizeof(int) * 2 * (size_t)n;
  int use_smem = sm <= 200 * 1024;
  if (!use_smem) sm = 0;
  if (sm > 48 * 1024) cudaFuncSetAttribute(k_aggregate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  launch(k_aggregate, 1, 32, sm, st, G_ptr, G_col, G_val, n, max_size, agg, size_work, use_smem, n_agg_dev);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------------------
// gauge near-nullspace (problem.py:332-352), (9 nc) x 16 row-major

__global__ void k_gauge(const double* __restrict__ cams, int nc, double* __restrict__ K) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
    const double* c = cams + (int64_t)i * 9;
    double aa[3] = {c[0], c[1], c[2]};
    double a2 = aa[0] * aa[0] + aa[1] * aa[1] + aa[2] * aa[2];
    double a = sqrt(a2);
    bool small = a < 1e-4;
    double s1, s2, d2;
    if (small) {
      s1 = 1.0 - a2 / 6.0;
      s2 = 0.5 - a2 / 24.0;
      d2 = 1.0 / 12.0 + a2 / 720.0;
    } else {
      double sn, cs;
      sincos(a, &sn, &cs);
      s1 = sn / a;
      s2 = (1.0 - cs) / (a * a);
      double sh, ch;
      sincos(a / 2.0, &sh, &ch);
      d2 = 1.0 / (a * a) - (ch / sh) / (2.0 * a);
    }
    double Kx[9] = {0.0, -aa[2], aa[1], aa[2], 0.0, -aa[0], -aa[1], aa[0], 0.0};
    double K2[9];
    for (int r = 0; r < 3; ++r)
      for (int q = 0; q < 3; ++q) K2[r * 3 + q] = Kx[r * 3] * Kx[q] + Kx[r * 3 + 1] * Kx[3 + q] + Kx[r * 3 + 2] * Kx[6 + q];
    double* out = K + (int64_t)i * 9 * 16;
    for (int q = 0; q < 144; ++q) out[q] = 0.0;
    for (int r = 0; r < 3; ++r)
      for (int q = 0; q < 3; ++q) {
        double I = (r == q) ? 1.0 : 0.0;
        double R = I + s1 * Kx[r * 3 + q] + s2 * K2[r * 3 + q];
        double Ji = I + 0.5 * Kx[r * 3 + q] + d2 * K2[r * 3 + q];
        out[(3 + r) * 16 + q] = -R;
        out[r * 16 + 3 + q] = -Ji;
      }
    for (int r = 0; r < 3; ++r) out[(3 + r) * 16 + 6] = c[3 + r];
    for (int k = 0; k < 9; ++k) out[k * 16 + 7 + k] = 1.0;
  }
}

extern "C" int bamg_gauge_nullspace(bamg_ctx* ctx, const double* cams, int32_t nc, double* K, void* stream) {
  (void)ctx;
  if (nc <= 0) return 0;
  launch(k_gauge, grid_for(nc, 128), 128, 0, as_stream(stream), cams, nc, K);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------------------
// members of each aggregate, ascending (multigrid.py:121-124): stable sort of node
// ids by aggregate id.

__global__ void k_iota_i(uint32_t* a, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = (uint32_t)i;
}

extern "C" int bamg_aggregate_members(bamg_ctx* ctx, const int32_t* agg, int32_t n, int32_t n_agg,
                                      int32_t* agg_ptr, int32_t* members, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (n <= 0) return 0;
  uint32_t *iota = nullptr, *skey = nullptr;
  BAMG_CUDA_CHECK(cudaMallocAsync(&iota, 4 * (size_t)n, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&skey, 4 * (size_t)n, st));
  launch(k_iota_i, grid_for(n, 256), 256, 0, st, iota, n);
  int bits = 1;
  while ((1ll << bits) < n_agg) ++bits;
  int rc = radix_sort_pairs((const uint32_t*)agg, iota, skey, (uint32_t*)members, n, bits, st);
  if (rc) return rc;
  rc = segment_ptr((const int*)skey, n, n_agg, agg_ptr, st);
  if (rc) return rc;
  cudaFreeAsync(iota, st);
  cudaFreeAsync(skey, st);
  return 0;
}

// ---------------------------------------------------------------------------
// tentative prolongation by per-aggregate Householder QR (multigrid.py:179-237).
// One warp per aggregate; local matrix (m x 16, m = members*bs) and Q in smem.
// LAPACK dlarfg convention: beta = -sign(alpha) |(alpha, x)|, tau = (beta-alpha)/beta,
// v = x / (alpha - beta); x == 0 gives tau = 0 (H = I).

#define NS 16

// The per-column dot products of one reflector application are independent, so
// they are accumulated together and their warp reductions interleaved: sixteen
// butterfly trees in flight instead of sixteen back-to-back (the scan is latency
// bound, one warp per aggregate). Every column keeps its own accumulation order and
// tree, so the results are bit-identical to the column-at-a-time loops below.
#ifndef BAMG_QR_BATCH
#define BAMG_QR_BATCH 1
#endif

__device__ __forceinline__ void warp_sum16(double* v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int c = 0; c < 16; ++c) v[c] += __shfl_xor_sync(FULL_MASK, v[c], o);
}

// Shared-memory leading dimension of the QR panels: 17, not 16 -- with 16-double rows
// every column access (lane = row) hit one bank pair (32-way conflicts).
#define QLD 17
// apply H_j (reflector in column j below the diagonal, tau) to columns [from, NS) of A
__device__ __forceinline__ void reflect_cols(double* A, int m, int j, int from, double tau, int lane) {
  double w[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) w[c] = 0.0;
  for (int i = j + 1 + lane; i < m; i += 32) {
    double v = A[i * QLD + j];
#pragma unroll
    for (int c = 0; c < 16; ++c)
      if (c >= from) w[c] += v * A[i * QLD + c];
  }
  warp_sum16(w);
#pragma unroll
  for (int c = 0; c < 16; ++c) w[c] = w[c] + A[j * QLD + c];
  __syncwarp();
  for (int i = j + 1 + lane; i < m; i += 32) {
    double v = A[i * QLD + j];
#pragma unroll
    for (int c = 0; c < 16; ++c)
      if (c >= from) A[i * QLD + c] -= tau * w[c] * v;
  }
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < 16; ++c)
      if (c >= from) A[j * QLD + c] -= tau * w[c];
  }
  __syncwarp();
}

__device__ void householder_step(double* A, int m, int j, int lane, double* tau_out, int ncols_apply_from,
                                 double* diag_out) {
  // column j, rows j..m-1
  double xs = 0.0;
  for (int i = j + 1 + lane; i < m; i += 32) xs += A[i * QLD + j] * A[i * QLD + j];
  xs = warp_sum(xs);
  double alpha = A[j * QLD + j];
  double tau = 0.0, beta = alpha;
  if (xs > 0.0) {
    double xnorm = sqrt(xs);
    beta = -copysign(hypot(alpha, xnorm), alpha);
    tau = (beta - alpha) / beta;
    double scal = 1.0 / (alpha - beta);
    for (int i = j + 1 + lane; i < m; i += 32) A[i * QLD + j] *= scal;
  }
  __syncwarp();
  if (lane == 0) A[j * QLD + j] = beta;
  *tau_out = tau;
  *diag_out = beta;
  __syncwarp();
  if (BAMG_QR_BATCH && tau != 0.0) {
    reflect_cols(A, m, j, ncols_apply_from, tau, lane);
  } else if (tau != 0.0) {
    for (int c = ncols_apply_from; c < NS; ++c) {
      double w = 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) w += A[i * QLD + j] * A[i * QLD + c];
      w = warp_sum(w) + A[j * QLD + c];
      __syncwarp();
      for (int i = j + 1 + lane; i < m; i += 32) A[i * QLD + c] -= tau * w * A[i * QLD + j];
      if (lane == 0) A[j * QLD + c] -= tau * w;
      __syncwarp();
    }
  }
}

// Q[:, :keep] = H_0 ... H_{k-1} I[:, :keep] (reflectors stored below the diagonal of A)
__device__ void form_q(const double* A, const double* tau, int m, int k, int keep, double* Q, int lane) {
  for (int i = lane; i < m; i += 32)
    for (int c = 0; c < NS; ++c) Q[i * QLD + c] = (i == c && c < keep) ? 1.0 : 0.0;
  __syncwarp();
  if (BAMG_QR_BATCH) {
    for (int j = k - 1; j >= 0; --j) {
      const double tj = tau[j];
      if (tj == 0.0) continue;
      double w[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) w[c] = 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) {
        double v = A[i * QLD + j];
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c >= j && c < keep) w[c] += v * Q[i * QLD + c];
      }
      warp_sum16(w);
#pragma unroll
      for (int c = 0; c < 16; ++c) w[c] = Q[j * QLD + c] + w[c];
      __syncwarp();
      for (int i = j + 1 + lane; i < m; i += 32) {
        double v = A[i * QLD + j];
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c >= j && c < keep) Q[i * QLD + c] -= tj * w[c] * v;
      }
      if (lane == 0) {
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c >= j && c < keep) Q[j * QLD + c] -= tj * w[c];
      }
      __syncwarp();
    }
    return;
  }
  for (int j = k - 1; j >= 0; --j) {
    if (tau[j] == 0.0) continue;
    for (int c = j; c < keep; ++c) {
      double w = Q[j * QLD + c];
      double part = 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) part += A[i * QLD + j] * Q[i * QLD + c];
      w += warp_sum(part);
      __syncwarp();
      for (int i = j + 1 + lane; i < m; i += 32) Q[i * QLD + c] -= tau[j] * w * A[i * QLD + j];
      if (lane == 0) Q[j * QLD + c] -= tau[j] * w;
      __syncwarp();
    }
  }
}

__global__ void k_prolong_qr(const int* __restrict__ agg_ptr, const int* __restrict__ members,
                             const double* __restrict__ K, int n_agg, int bs, int m_max, double* __restrict__ Pblocks,
                             double* __restrict__ Kc, int* __restrict__ info /* [n_agg][2]: pivoted, rank */,
                             int* __restrict__ padded_cnt, int size_lo, int size_hi) {
  extern __shared__ double sm[];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int wpb = blockDim.x >> 5;
  double* A = sm + (size_t)w * (2 * m_max * QLD + 2 * NS + NS);
  double* Q = A + m_max * QLD;
  double* tau = Q + m_max * QLD;
  double* dg = tau + NS;
  int* piv = (int*)(dg + NS);  // NS ints packed in the NS-double tail... use separate region
  (void)piv;
  for (int a = blockIdx.x * wpb + w; a < n_agg; a += gridDim.x * wpb) {
    int b0 = agg_ptr[a], nm = agg_ptr[a + 1] - b0;
    if (nm < size_lo || nm > size_hi) continue;  // this launch's size class only
    int m = nm * bs;
    // load
    for (int t = lane; t < m * NS; t += 32) {
      int r = t / NS, c = t - r * NS;
      int node = members[b0 + r / bs];
      A[r * QLD + c] = K[((int64_t)node * bs + (r % bs)) * NS + c];
    }
    __syncwarp();
    int keep = m < NS ? m : NS;
    bool done = false;
    if (m >= NS) {
      // economic QR, no pivoting (scipy.linalg.qr mode="economic")
      for (int j = 0; j < NS; ++j) {
        double tj, dj;
        householder_step(A, m, j, lane, &tj, j + 1, &dj);
        if (lane == 0) {
          tau[j] = tj;
          dg[j] = dj;
        }
        __syncwarp();
      }
      double mn = 1e308, mx = 0.0;
      for (int j = 0; j < NS; ++j) {
        double v = fabs(dg[j]);
        mn = fmin(mn, v);
        mx = fmax(mx, v);
      }
      if (mn > 1e-10 * mx) {
        form_q(A, tau, m, NS, NS, Q, lane);
        // sign fix: s = sign(diag R); P = Q s; Kc = s R
        for (int t = lane; t < m * NS; t += 32) {
          int r = t / NS, c = t - r * NS;
          double s = dg[c] < 0.0 ? -1.0 : 1.0;
          Q[r * QLD + c] *= s;
        }
        double* kc = Kc + (int64_t)a * NS * NS;
        for (int t = lane; t < NS * NS; t += 32) {
          int r = t / NS, c = t - r * NS;
          double s = dg[r] < 0.0 ? -1.0 : 1.0;
          kc[t] = (c >= r) ? s * A[r * QLD + c] : 0.0;
        }
        if (lane == 0) {
          info[2 * a] = 0;
          info[2 * a + 1] = NS;
          padded_cnt[a] = 0;
        }
        done = true;
      } else {
        // reload for the pivoted branch
        __syncwarp();
        for (int t = lane; t < m * NS; t += 32) {
          int r = t / NS, c = t - r * NS;
          int node = members[b0 + r / bs];
          A[r * QLD + c] = K[((int64_t)node * bs + (r % bs)) * NS + c];
        }
        __syncwarp();
      }
    }
    if (!done) {
      // pivoted QR (scipy.linalg.qr pivoting=True, LAPACK geqp3): at step j pick the
      // remaining column with the largest norm of rows j..m-1 (first on ties).
      int perm[NS];
      for (int c = 0; c < NS; ++c) perm[c] = c;
      int k = m < NS ? m : NS;
      for (int j = 0; j < k; ++j) {
        int bestc = j;
        double bestn = -1.0;
        if (BAMG_QR_BATCH) {
          double s[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) s[c] = 0.0;
          for (int i = j + lane; i < m; i += 32) {
#pragma unroll
            for (int c = 0; c < 16; ++c)
              if (c >= j) s[c] += A[i * QLD + c] * A[i * QLD + c];
          }
          warp_sum16(s);
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (c >= j && s[c] > bestn) {
              bestn = s[c];
              bestc = c;
            }
        } else {
          for (int c = j; c < NS; ++c) {
            double s = 0.0;
            for (int i = j + lane; i < m; i += 32) s += A[i * QLD + c] * A[i * QLD + c];
            s = warp_sum(s);
            if (s > bestn) {
              bestn = s;
              bestc = c;
            }
          }
        }
        if (bestc != j) {
          for (int i = lane; i < m; i += 32) {
            double t = A[i * QLD + j];
            A[i * QLD + j] = A[i * QLD + bestc];
            A[i * QLD + bestc] = t;
          }
          int t = perm[j];
          perm[j] = perm[bestc];
          perm[bestc] = t;
        }
        __syncwarp();
        double tj, dj;
        householder_step(A, m, j, lane, &tj, j + 1, &dj);
        if (lane == 0) {
          tau[j] = tj;
          dg[j] = dj;
        }
        __syncwarp();
      }
      double d0 = fabs(dg[0]);
      int rank = 0;
      if (k > 0 && d0 > 0.0)
        for (int j = 0; j < k; ++j)
          if (fabs(dg[j]) > 1e-10 * d0) ++rank;
      form_q(A, tau, m, k, keep, Q, lane);
      double* kc = Kc + (int64_t)a * NS * NS;
      for (int t = lane; t < NS * NS; t += 32) kc[t] = 0.0;
      __syncwarp();
      // r_unpiv[:rank, perm] = R[:rank, :]
      for (int t = lane; t < rank * NS; t += 32) {
        int r = t / NS, c = t - r * NS;
        kc[r * NS + perm[c]] = (c >= r) ? A[r * QLD + c] : 0.0;
      }
      if (lane == 0) {
        info[2 * a] = 1;
        info[2 * a + 1] = rank;
        padded_cnt[a] = NS - keep;
      }
    }
    __syncwarp();
    // scatter P blocks
    for (int t = lane; t < m * NS; t += 32) {
      int r = t / NS, c = t - r * NS;
      int node = members[b0 + r / bs];
      Pblocks[((int64_t)node * bs + (r % bs)) * NS + c] = (c < keep) ? Q[r * QLD + c] : 0.0;
    }
    __syncwarp();
  }
}

extern "C" int bamg_prolongation_qr(bamg_ctx* ctx, const int32_t* agg_ptr, const int32_t* members, const double* K,
                                    int32_t n_agg, int32_t bs, int32_t max_members, double* Pblocks, double* Kc,
                                    int32_t* info, int32_t* padded_cnt, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (n_agg <= 0) return 0;
  // per-warp shared memory sized by the largest aggregate of the launch's size class
  auto run = [&](int lo, int hi) -> int {
    int m_max = hi * bs;
    size_t per_warp = sizeof(double) * (2 * (size_t)m_max * QLD + 3 * NS);
    int wpb = (int)((200 * 1024) / per_warp);
    if (wpb < 1) {
      bamg_set_error("prolongation: aggregate of %d rows exceeds shared memory", m_max);
      return BAMG_ERR_UNSUPPORTED;
    }
    if (wpb > 4) wpb = 4;
    size_t sm = per_warp * wpb;
    if (sm > 48 * 1024) cudaFuncSetAttribute(k_prolong_qr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int blocks = (int)ceil_div(n_agg, wpb);
    int cap = bamg_num_sms() * 8;
    if (blocks > cap) blocks = cap;
    launch(k_prolong_qr, blocks, 32 * wpb, sm, st, agg_ptr, members, K, n_agg, bs, m_max, Pblocks, Kc, info,
           padded_cnt, lo, hi);
    BAMG_LAUNCH_CHECK();
    return 0;
  };
  return run(0, max_members);  // (a small/large split measured slower at c4: 3.7 vs 2.9 ms)
}

// ---------------------------------------------------------------------------
// Galerkin A_c = sym(P^T A P) (multigrid.py:409, 444-455; blockmat.py:337-360).
// Coarse pattern: row a = union over members i of agg(cols of row i) (bitmap).
// Numeric: each fine block (i, j) maps to coarse block (agg i, agg j); fine blocks
// are grouped per coarse block by a stable radix sort (row-major order kept inside),
// then one warp per coarse block accumulates sum P_i^T (A_ij P_j) in registers.

__global__ void k_coarse_rows(const int* __restrict__ agg_ptr, const int* __restrict__ members,
                              const int* __restrict__ ptr, const int* __restrict__ col, const int* __restrict__ agg,
                              int n_agg, int* __restrict__ counts, const int* __restrict__ Cptr, int* __restrict__ Ccol) {
  extern __shared__ unsigned int bm[];
  int words = (n_agg + 31) >> 5;
  for (int a = blockIdx.x; a < n_agg; a += gridDim.x) {
    for (int w = threadIdx.x; w < words; w += blockDim.x) bm[w] = 0u;
    __syncthreads();
    for (int q = agg_ptr[a]; q < agg_ptr[a + 1]; ++q) {
      int i = members[q];
      for (int b = ptr[i] + threadIdx.x; b < ptr[i + 1]; b += blockDim.x) {
        int c = agg[col[b]];
        atomicOr(&bm[c >> 5], 1u << (c & 31));
      }
    }
    __syncthreads();
    if (Ccol == nullptr) {
      int c = 0;
      for (int w = threadIdx.x; w < words; w += blockDim.x) c += __popc(bm[w]);
      c = warp_sum_int(c);
      __shared__ int red[32];
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
      __syncthreads();
      if (threadIdx.x == 0) {
        int t = 0;
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
        counts[a] = t;
      }
    } else if (threadIdx.x < 32) {
      int lane = threadIdx.x;
      int out = Cptr[a];
      for (int w0 = 0; w0 < words; w0 += 32) {
        int w = w0 + lane;
        unsigned v = (w < words) ? bm[w] : 0u;
        int cnt = __popc(v);
        int incl = cnt;
        for (int o = 1; o < 32; o <<= 1) {
          int t = __shfl_up_sync(FULL_MASK, incl, o);
          if (lane >= o) incl += t;
        }
        int pos = out + incl - cnt;
        while (v) {
          int b = __ffs(v) - 1;
          v &= v - 1;
          Ccol[pos++] = w * 32 + b;
        }
        out += __shfl_sync(FULL_MASK, incl, 31);
      }
    }
    __syncthreads();
  }
}

extern "C" int bamg_galerkin_pattern(bamg_ctx* ctx, const int32_t* agg_ptr, const int32_t* members,
                                     const int32_t* ptr, const int32_t* col, const int32_t* agg, int32_t n_agg,
                                     int32_t* Cptr_or_counts, int32_t* Ccol, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  size_t sm = sizeof(unsigned) * ((n_agg + 31) / 32);
  if (sm > 200 * 1024) {
    bamg_set_error("galerkin bitmap for %d aggregates exceeds shared memory", n_agg);
    return BAMG_ERR_UNSUPPORTED;
  }
  if (sm > 48 * 1024) cudaFuncSetAttribute(k_coarse_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (Ccol == nullptr)
    launch(k_coarse_rows, grid_for(n_agg, 1, 16), 128, sm, st, agg_ptr, members, ptr, col, agg, n_agg, Cptr_or_counts,
                                                           nullptr, nullptr);
  else
    launch(k_coarse_rows, grid_for(n_agg, 1, 16), 128, sm, st, agg_ptr, members, ptr, col, agg, n_agg, nullptr,
                                                           Cptr_or_counts, Ccol);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// coarse block index of each fine block
// warp per fine row: lanes take the row's blocks (coalesced column reads and key
// writes), each searching the same coarse row
__global__ void k_fine_to_coarse(const int* __restrict__ ptr, const int* __restrict__ col, const int* __restrict__ agg,
                                 int n, const int* __restrict__ Cptr, const int* __restrict__ Ccol,
                                 uint32_t* __restrict__ key) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
    int a = agg[i];
    int c0 = Cptr[a];
    const int* cc = Ccol + c0;
    int nn = Cptr[a + 1] - c0;
    for (int b = ptr[i] + lane; b < ptr[i + 1]; b += 32) key[b] = (uint32_t)(c0 + lower_bound_i32(cc, nn, agg[col[b]]));
  }
}

__global__ void k_row_of_block(const int* __restrict__ ptr, int n, int* __restrict__ row) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    for (int b = ptr[i]; b < ptr[i + 1]; ++b) row[b] = i;
}

extern "C" int bamg_galerkin_map(bamg_ctx* ctx, const int32_t* ptr, const int32_t* col, const int32_t* agg, int32_t n,
                                 int64_t nnz_fine, const int32_t* Cptr, const int32_t* Ccol, int64_t nnz_coarse,
                                 int32_t* fine_sorted, int32_t* cblk_ptr, int32_t* fine_row, void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (nnz_fine <= 0) return 0;
  uint32_t *key = nullptr, *iota = nullptr, *skey = nullptr;
  BAMG_CUDA_CHECK(cudaMallocAsync(&key, 4 * nnz_fine, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&iota, 4 * nnz_fine, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&skey, 4 * nnz_fine, st));
  launch(k_fine_to_coarse, grid_for((int64_t)n * 32, 128, 16), 128, 0, st, ptr, col, agg, n, Cptr, Ccol, key);
  launch(k_iota_i, grid_for(nnz_fine, 256), 256, 0, st, iota, (int)nnz_fine);
  launch(k_row_of_block, grid_for(n, 128), 128, 0, st, ptr, n, fine_row);
  BAMG_LAUNCH_CHECK();
  int bits = 1;
  while ((1ll << bits) < nnz_coarse) ++bits;
  int rc = radix_sort_pairs(key, iota, skey, (uint32_t*)fine_sorted, nnz_fine, bits, st);
  if (rc) return rc;
  rc = segment_ptr((const int*)skey, nnz_fine, (int)nnz_coarse, cblk_ptr, st);
  if (rc) return rc;
  cudaFreeAsync(key, st);
  cudaFreeAsync(iota, st);
  cudaFreeAsync(skey, st);
  return 0;
}

// Upper coarse blocks (a <= b) of a symmetric coarse pattern as a work list for the
// Galerkin kernels: block position and the position of its mirror (b, a).
__global__ void k_gal_upper_count(const int* __restrict__ Cptr, const int* __restrict__ Ccol, int n,
                                  int* __restrict__ cnt) {
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < n; a += gridDim.x * blockDim.x) {
    int b0 = Cptr[a], nn = Cptr[a + 1] - b0;
    cnt[a] = nn - lower_bound_i32(Ccol + b0, nn, a);
  }
}

// warp per coarse row: lanes take the row's upper blocks (coalesced writes)
__global__ void k_gal_upper_fill(const int* __restrict__ Cptr, const int* __restrict__ Ccol, int n,
                                 const int* __restrict__ off, int* __restrict__ ublk, int* __restrict__ umir) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int a = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < n; a += nw) {
    int b0 = Cptr[a], nn = Cptr[a + 1] - b0;
    int qd = b0 + lower_bound_i32(Ccol + b0, nn, a);
    int o0 = off[a];
    for (int q = qd + lane; q < b0 + nn; q += 32) {
      int b = Ccol[q];
      ublk[o0 + (q - qd)] = q;
      umir[o0 + (q - qd)] = Cptr[b] + lower_bound_i32(Ccol + Cptr[b], Cptr[b + 1] - Cptr[b], a);
    }
  }
}

// Output stage of the Galerkin kernels for an upper coarse block (a, b), a <= b, from
// the four warp partials in `red` (summed in warp order): (a, b) = C and its mirror
// (b, a) = C^T, so the stored operator is exactly symmetric; a diagonal block is
// 0.5 (C + C^T), the symmetrisation of multigrid.py:444-455. The lower blocks are
// never multiplied out (half the Galerkin flops, no separate symmetrisation pass).
__device__ __forceinline__ void galerkin_store_sym(const double (*red)[NS * NS], int64_t cb, int64_t t,
                                                   double* __restrict__ out) {
  double* o = out + cb * NS * NS;
  if (t == cb) {
    for (int e = threadIdx.x; e < NS * NS; e += blockDim.x) {
      int r = e / NS, c = e - r * NS;
      double v = ((red[0][e] + red[1][e]) + red[2][e]) + red[3][e];
      int et = c * NS + r;
      double vt = ((red[0][et] + red[1][et]) + red[2][et]) + red[3][et];
      o[e] = 0.5 * (v + vt);
    }
    return;
  }
  double* y = out + t * NS * NS;
  for (int e = threadIdx.x; e < NS * NS; e += blockDim.x) {
    o[e] = ((red[0][e] + red[1][e]) + red[2][e]) + red[3][e];
    int r = e / NS, c = e - r * NS, et = c * NS + r;
    y[e] = ((red[0][et] + red[1][et]) + red[2][et]) + red[3][et];
  }
}

// CTA per coarse block: its fine blocks are dealt round-robin to the 4 warps; each
// warp stages A_ij, P_j, P_i with coalesced loads into shared memory, forms
// T = A_ij P_j there and accumulates P_i^T T (lane: row lane/2, 8 columns). The
// four partial 16x16 sums are added in warp order (deterministic).
template <int BS>
__global__ void __launch_bounds__(128)
k_galerkin_cta(const int* __restrict__ cblk_ptr, const int* __restrict__ fine_sorted, const int* __restrict__ fine_row,
               const int* __restrict__ col, const double* __restrict__ blocks, const double* __restrict__ P,
               int n_up, const int* __restrict__ ublk, const int* __restrict__ umir, double* __restrict__ out) {
  __shared__ double sA[4][BS * BS];
  __shared__ double sPj[4][BS * NS];
  __shared__ double sPi[4][BS * NS];
  __shared__ double sT[4][BS * (NS + 1)];
  __shared__ double red[4][NS * NS];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int r = lane >> 1, c0 = (lane & 1) * 8;
  double* A = sA[w];
  double* Pj = sPj[w];
  double* Pi = sPi[w];
  double* T = sT[w];
  for (int u = blockIdx.x; u < n_up; u += gridDim.x) {
    const int64_t cb = ublk[u], cmir = umir[u];  // lower blocks: written as mirrors
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    for (int q = cblk_ptr[cb] + w; q < cblk_ptr[cb + 1]; q += 4) {
      int fb = fine_sorted[q];
      int i = fine_row[fb], j = col[fb];
      const double* a = blocks + (int64_t)fb * BS * BS;
      const double* pj = P + (int64_t)j * BS * NS;
      const double* pi = P + (int64_t)i * BS * NS;
      for (int t = lane; t < BS * BS; t += 32) A[t] = __ldg(a + t);
      for (int t = lane; t < BS * NS; t += 32) {
        Pj[t] = __ldg(pj + t);
        Pi[t] = __ldg(pi + t);
      }
      __syncwarp();
      if (r < BS) {  // T[r][c0..c0+7] = sum_k A[r][k] Pj[k][c0..]
        double t8[8];
#pragma unroll
        for (int q2 = 0; q2 < 8; ++q2) t8[q2] = 0.0;
#pragma unroll
        for (int k = 0; k < BS; ++k) {
          double ark = A[r * BS + k];
#pragma unroll
          for (int q2 = 0; q2 < 8; ++q2) t8[q2] = fma(ark, Pj[k * NS + c0 + q2], t8[q2]);
        }
#pragma unroll
        for (int q2 = 0; q2 < 8; ++q2) T[r * (NS + 1) + c0 + q2] = t8[q2];
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < BS; ++k) {
        double pik = Pi[k * NS + r];
#pragma unroll
        for (int q2 = 0; q2 < 8; ++q2) acc[q2] = fma(pik, T[k * (NS + 1) + c0 + q2], acc[q2]);
      }
      __syncwarp();
    }
#pragma unroll
    for (int q2 = 0; q2 < 8; ++q2) red[w][r * NS + c0 + q2] = acc[q2];
    __syncthreads();
    galerkin_store_sym(red, cb, cmir, out);
    __syncthreads();
  }
}

// k_galerkin_cta with the fine-block operands streamed: each warp keeps two stages
// of (A_ij, P_j, P_i) in shared memory and copies the next fine block's operands
// with cp.async while it multiplies the current one. Same operands, same code,
// same order -- bit-identical to k_galerkin_cta.
template <int BS>
__global__ void __launch_bounds__(128)
k_galerkin_pipe(const int* __restrict__ cblk_ptr, const int* __restrict__ fine_sorted, const int* __restrict__ fine_row,
                const int* __restrict__ col, const double* __restrict__ blocks, const double* __restrict__ P,
                int n_up, const int* __restrict__ ublk, const int* __restrict__ umir, double* __restrict__ out) {
  // one stage: A (padded to an even count so P_j / P_i start 16 B aligned) | Pj | Pi.
  // The kernel is bound by L1 wavefronts (ncu: 83% of peak), so P_j and T are read
  // as double2 and P copied in 16 B chunks; the arithmetic is untouched.
  constexpr int SA = BS * BS, SAP = (SA + 1) & ~1, SP = BS * NS, STG = SAP + 2 * SP, TS = NS + 2;
  extern __shared__ __align__(16) double gsm[];
  __shared__ __align__(16) double sT[4][BS * TS];
  __shared__ double red[4][NS * NS];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int r = lane >> 1, c0 = (lane & 1) * 8;
  double* stg = gsm + (size_t)w * 2 * STG;
  double* T = sT[w];
  auto issue = [&](int q, double* dst) {
    int fb = fine_sorted[q];
    int i = fine_row[fb], j = col[fb];
    const double* a = blocks + (int64_t)fb * SA;
    const double* pj = P + (int64_t)j * SP;
    const double* pi = P + (int64_t)i * SP;
    for (int t = lane; t < SA; t += 32) cp_async8(dst + t, a + t);
    for (int t = lane; t < SP / 2; t += 32) {
      cp_async16(dst + SAP + 2 * t, pj + 2 * t);
      cp_async16(dst + SAP + SP + 2 * t, pi + 2 * t);
    }
    cp_async_commit();
  };
  for (int u = blockIdx.x; u < n_up; u += gridDim.x) {
    const int64_t cb = ublk[u], cmir = umir[u];  // lower blocks: written as mirrors
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    const int qb = cblk_ptr[cb], qe = cblk_ptr[cb + 1];
    if (qb + w < qe) issue(qb + w, stg);
    int k = 0;
    for (int q = qb + w; q < qe; q += 4, ++k) {
      if (q + 4 < qe) issue(q + 4, stg + ((k + 1) & 1) * STG);
      else cp_async_commit();
      cp_async_wait<1>();
      __syncwarp();
      const double* A = stg + (k & 1) * STG;
      const double* Pj = A + SAP;
      const double* Pi = A + SAP + SP;
      if (r < BS) {  // T[r][c0..c0+7] = sum_k A[r][k] Pj[k][c0..]
        double t8[8];
#pragma unroll
        for (int q2 = 0; q2 < 8; ++q2) t8[q2] = 0.0;
#pragma unroll
        for (int kk = 0; kk < BS; ++kk) {
          double ark = A[r * BS + kk];
          const double2* pr = reinterpret_cast<const double2*>(Pj + kk * NS + c0);
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            double2 v = pr[h];
            t8[2 * h] = fma(ark, v.x, t8[2 * h]);
            t8[2 * h + 1] = fma(ark, v.y, t8[2 * h + 1]);
          }
        }
        double2* tw = reinterpret_cast<double2*>(T + r * TS + c0);
#pragma unroll
        for (int h = 0; h < 4; ++h) tw[h] = make_double2(t8[2 * h], t8[2 * h + 1]);
      }
      __syncwarp();
#pragma unroll
      for (int kk = 0; kk < BS; ++kk) {
        double pik = Pi[kk * NS + r];
        const double2* tr = reinterpret_cast<const double2*>(T + kk * TS + c0);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          double2 v = tr[h];
          acc[2 * h] = fma(pik, v.x, acc[2 * h]);
          acc[2 * h + 1] = fma(pik, v.y, acc[2 * h + 1]);
        }
      }
      __syncwarp();
    }
    cp_async_wait<0>();
#pragma unroll
    for (int q2 = 0; q2 < 8; ++q2) red[w][r * NS + c0 + q2] = acc[q2];
    __syncthreads();
    galerkin_store_sym(red, cb, cmir, out);
    __syncthreads();
  }
}

// Row and column of every fine block of the coarse-block-sorted list (gathered once,
// so the Galerkin warps read them coalesced instead of through fine_sorted).
__global__ void k_gal_gather_ij(const int* __restrict__ fine_sorted, const int* __restrict__ fine_row,
                                const int* __restrict__ col, int64_t nnz_fine, int* __restrict__ fsi,
                                int* __restrict__ fsj) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz_fine; q += (int64_t)gridDim.x * blockDim.x) {
    int fb = fine_sorted[q];
    fsi[q] = fine_row[fb];
    fsj[q] = col[fb];
  }
}

// Warp per upper coarse block with ONE operand pipeline running across the warp's
// blocks: while fine block q is multiplied, the operands (A_ij, P_j, P_i) of the next
// fine block -- of this coarse block or already of the next one -- are in flight
// (cp.async, two stages), and the (fb, i, j) triples of 32 fine blocks at a time are
// held one per lane (the next coarse block's first 32 are loaded a block ahead). The
// CTA-per-block kernels paid the index chain and the pipeline fill on every coarse
// block. One warp sums a block's fine blocks in list order (deterministic).
template <int BS>
__global__ void __launch_bounds__(128, BS == 9 ? 4 : 3)
k_galerkin_warp(const int* __restrict__ cblk_ptr, const int* __restrict__ fine_sorted, const int* __restrict__ fsi,
                const int* __restrict__ fsj, const double* __restrict__ blocks, const double* __restrict__ P, int n_up,
                const int* __restrict__ ublk, const int* __restrict__ umir, double* __restrict__ out) {
  constexpr int SA = BS * BS, SAP = (SA + 1) & ~1, SP = BS * NS, STG = SAP + 2 * SP, TS = NS + 2;
  constexpr int WSM = 2 * STG + BS * TS + NS * (NS + 1);
  extern __shared__ __align__(16) double gsm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* stg = gsm + (size_t)w * WSM;
  double* T = stg + 2 * STG;
  double* D = T + BS * TS;  // diagonal-block transpose scratch
  const int r = lane >> 1, c0 = (lane & 1) * 8;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (u >= n_up) return;
  auto issue = [&](int fb, int i, int j, double* dst) {
    const double* a = blocks + (int64_t)fb * SA;
    const double* pj = P + (int64_t)j * SP;
    const double* pi = P + (int64_t)i * SP;
    for (int t = lane; t < SA; t += 32) cp_async8(dst + t, a + t);
    for (int t = lane; t < SP / 2; t += 32) {
      cp_async16(dst + SAP + 2 * t, pj + 2 * t);
      cp_async16(dst + SAP + SP + 2 * t, pi + 2 * t);
    }
    cp_async_commit();
  };
  // current block
  int64_t cb = ublk[u], cm = umir[u];
  int q = cblk_ptr[cb], qe = cblk_ptr[cb + 1];
  int base = q;  // first list position held in the index registers
  int xfb = 0, xi = 0, xj = 0;
  if (base + lane < qe) { xfb = fine_sorted[base + lane]; xi = fsi[base + lane]; xj = fsj[base + lane]; }
  // next block (one block ahead)
  int un = u + nwarps;
  int64_t cbn = 0, cmn = 0;
  int qn = 0, qne = 0, nfb = 0, ni = 0, nj = 0;
  auto prefetch_next = [&]() {
    if (un < n_up) {
      cbn = ublk[un];
      cmn = umir[un];
      qn = cblk_ptr[cbn];
      qne = cblk_ptr[cbn + 1];
      if (qn + lane < qne) { nfb = fine_sorted[qn + lane]; ni = fsi[qn + lane]; nj = fsj[qn + lane]; }
    }
  };
  prefetch_next();
  issue(__shfl_sync(FULL_MASK, xfb, 0), __shfl_sync(FULL_MASK, xi, 0), __shfl_sync(FULL_MASK, xj, 0), stg);
  double acc[8];
#pragma unroll
  for (int k2 = 0; k2 < 8; ++k2) acc[k2] = 0.0;
  for (int k = 0;; ++k) {
    const bool last = (q + 1 == qe);
    // the item after q: in this block (refill the index registers every 32), or the
    // first of the next block
    if (!last) {
      int q2 = q + 1;
      if (q2 - base == 32) {
        base = q2;
        if (base + lane < qe) { xfb = fine_sorted[base + lane]; xi = fsi[base + lane]; xj = fsj[base + lane]; }
      }
      int s2 = q2 - base;
      issue(__shfl_sync(FULL_MASK, xfb, s2), __shfl_sync(FULL_MASK, xi, s2), __shfl_sync(FULL_MASK, xj, s2),
            stg + ((k + 1) & 1) * STG);
    } else if (un < n_up) {
      issue(__shfl_sync(FULL_MASK, nfb, 0), __shfl_sync(FULL_MASK, ni, 0), __shfl_sync(FULL_MASK, nj, 0),
            stg + ((k + 1) & 1) * STG);
    } else {
      cp_async_commit();
    }
    cp_async_wait<1>();
    __syncwarp();
    const double* A = stg + (k & 1) * STG;
    const double* Pj = A + SAP;
    const double* Pi = A + SAP + SP;
    if (r < BS) {  // T[r][c0..c0+7] = sum_k A[r][k] Pj[k][c0..]
      double t8[8];
#pragma unroll
      for (int q2 = 0; q2 < 8; ++q2) t8[q2] = 0.0;
#pragma unroll
      for (int kk = 0; kk < BS; ++kk) {
        double ark = A[r * BS + kk];
        const double2* pr = reinterpret_cast<const double2*>(Pj + kk * NS + c0);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          double2 v = pr[h];
          t8[2 * h] = fma(ark, v.x, t8[2 * h]);
          t8[2 * h + 1] = fma(ark, v.y, t8[2 * h + 1]);
        }
      }
      double2* tw = reinterpret_cast<double2*>(T + r * TS + c0);
#pragma unroll
      for (int h = 0; h < 4; ++h) tw[h] = make_double2(t8[2 * h], t8[2 * h + 1]);
    }
    __syncwarp();
#pragma unroll
    for (int kk = 0; kk < BS; ++kk) {
      double pik = Pi[kk * NS + r];
      const double2* tr = reinterpret_cast<const double2*>(T + kk * TS + c0);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        double2 v = tr[h];
        acc[2 * h] = fma(pik, v.x, acc[2 * h]);
        acc[2 * h + 1] = fma(pik, v.y, acc[2 * h + 1]);
      }
    }
    __syncwarp();
    if (!last) {
      ++q;
      continue;
    }
    // block done: (a, b) = C, mirror (b, a) = C^T; diagonal: 0.5 (C + C^T)
    double* o = out + cb * NS * NS;
    if (cm == cb) {
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) D[r * (NS + 1) + c0 + k2] = acc[k2];
      __syncwarp();
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) o[r * NS + c0 + k2] = 0.5 * (acc[k2] + D[(c0 + k2) * (NS + 1) + r]);
      __syncwarp();
    } else {
      double* y = out + cm * NS * NS;
      double2* o2 = reinterpret_cast<double2*>(o + r * NS + c0);
#pragma unroll
      for (int h = 0; h < 4; ++h) o2[h] = make_double2(acc[2 * h], acc[2 * h + 1]);
#pragma unroll
      for (int k2 = 0; k2 < 8; ++k2) y[(c0 + k2) * NS + r] = acc[k2];
    }
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) acc[k2] = 0.0;
    if (un >= n_up) break;
    u = un;
    cb = cbn;
    cm = cmn;
    q = qn;
    qe = qne;
    base = q;
    xfb = nfb;
    xi = ni;
    xj = nj;
    un = u + nwarps;
    prefetch_next();
  }
  cp_async_wait<0>();
}

// +1.0 on padded coarse dofs' diagonal entries (multigrid.py:458-471)
__global__ void k_patch(const int* __restrict__ padded_cnt, const int* __restrict__ Cptr, const int* __restrict__ Ccol,
                        int n_agg, double* __restrict__ B) {
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < n_agg; a += gridDim.x * blockDim.x) {
    int np = padded_cnt[a];
    if (!np) continue;
    int t = Cptr[a] + lower_bound_i32(Ccol + Cptr[a], Cptr[a + 1] - Cptr[a], a);
    if (t >= Cptr[a + 1] || Ccol[t] != a) continue;
    double* X = B + (int64_t)t * NS * NS;
    for (int c = NS - np; c < NS; ++c) X[c * NS + c] += 1.0;
  }
}

extern "C" int bamg_galerkin_numeric(bamg_ctx* ctx, int32_t bs, const int32_t* cblk_ptr, const int32_t* fine_sorted,
                                     const int32_t* fine_row, const int32_t* col, const double* blocks,
                                     const double* P, int64_t nnz_fine, int32_t n_agg, const int32_t* Cptr,
                                     const int32_t* Ccol, int64_t nnz_coarse, const int32_t* padded_cnt, double* out,
                                     void* stream) {
  (void)ctx;
  cudaStream_t st = as_stream(stream);
  if (nnz_coarse <= 0) return 0;
  // upper coarse blocks (the pattern is symmetric: (nnz + n) / 2 of them)
  const int n_up = (int)((nnz_coarse + n_agg) / 2);
  int* ub = nullptr;
  BAMG_CUDA_CHECK(cudaMallocAsync(&ub, sizeof(int) * (2 * (size_t)n_up + n_agg + 1), st));
  int *ublk = ub, *umir = ub + n_up, *uoff = ub + 2 * (size_t)n_up;
  launch(k_gal_upper_count, grid_for(n_agg, 128), 128, 0, st, Cptr, Ccol, n_agg, uoff);
  int rc = scan_exclusive_int(uoff, uoff, (int64_t)n_agg + 1, nullptr, st);
  if (rc) return rc;
  launch(k_gal_upper_fill, grid_for((int64_t)n_agg * 32, 128, 16), 128, 0, st, Cptr, Ccol, n_agg, (const int*)uoff, ublk,
         umir);
  int g = grid_for(n_up, 1, 12);
  static const bool pipe = [] {
    const char* e = getenv("BAMG_GALERKIN_PIPE");
    return !(e && e[0] == '0');
  }();
  static const int gmode = [] {
    const char* e = getenv("BAMG_GALERKIN_WARP");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  // warp pipeline for the 9x9 fine level (1.96 -> 1.12 ms at c4 level 0); the coarse
  // 16x16 levels keep the CTA kernel (0.65 vs 0.70 ms: the 16x16 stages cost the warp
  // kernel occupancy)
  if (gmode == 1 && bs == 9) {
    int* ij = nullptr;
    BAMG_CUDA_CHECK(cudaMallocAsync(&ij, sizeof(int) * 2 * (size_t)(nnz_fine > 0 ? nnz_fine : 1), st));
    int *fsi = ij, *fsj = ij + nnz_fine;
    if (nnz_fine > 0)
      launch(k_gal_gather_ij, grid_for(nnz_fine, 256), 256, 0, st, fine_sorted, fine_row, col, nnz_fine, fsi, fsj);
    const int wsm9 = 2 * ((81 + 1) + 2 * 9 * NS) + 9 * (NS + 2) + NS * (NS + 1);
    const size_t sm9 = sizeof(double) * 4 * wsm9;
    static bool wattr = false;
    if (!wattr) {
      BAMG_CUDA_CHECK(cudaFuncSetAttribute(k_galerkin_warp<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm9));
      wattr = true;
    }
    int64_t warps = n_up < (int64_t)bamg_num_sms() * 24 ? n_up : (int64_t)bamg_num_sms() * 24;
    int gw = (int)ceil_div(warps, 4);
    launch(k_galerkin_warp<9>, gw, 128, sm9, st, cblk_ptr, fine_sorted, (const int*)fsi, (const int*)fsj, blocks, P,
           n_up, (const int*)ublk, (const int*)umir, out);
    cudaFreeAsync(ij, st);
  } else if (pipe) {
    static bool attr = false;
    const size_t sm9 = sizeof(double) * 4 * 2 * (82 + 2 * 9 * NS), sm16 = sizeof(double) * 4 * 2 * (256 + 2 * 16 * NS);
    if (!attr) {
      BAMG_CUDA_CHECK(cudaFuncSetAttribute(k_galerkin_pipe<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm9));
      BAMG_CUDA_CHECK(cudaFuncSetAttribute(k_galerkin_pipe<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm16));
      attr = true;
    }
    switch (bs) {
      case 9: launch(k_galerkin_pipe<9>, g, 128, sm9, st, cblk_ptr, fine_sorted, fine_row, col, blocks, P, n_up,
                     (const int*)ublk, (const int*)umir, out); break;
      case 16: launch(k_galerkin_pipe<16>, g, 128, sm16, st, cblk_ptr, fine_sorted, fine_row, col, blocks, P, n_up,
                      (const int*)ublk, (const int*)umir, out); break;
      default: bamg_set_error("galerkin: unsupported block size %d", bs); return BAMG_ERR_UNSUPPORTED;
    }
  } else {
    switch (bs) {
      case 9: launch(k_galerkin_cta<9>, g, 128, 0, st, cblk_ptr, fine_sorted, fine_row, col, blocks, P, n_up,
                     (const int*)ublk, (const int*)umir, out); break;
      case 16: launch(k_galerkin_cta<16>, g, 128, 0, st, cblk_ptr, fine_sorted, fine_row, col, blocks, P, n_up,
                      (const int*)ublk, (const int*)umir, out); break;
      default: bamg_set_error("galerkin: unsupported block size %d", bs); return BAMG_ERR_UNSUPPORTED;
    }
  }
  launch(k_patch, grid_for(n_agg, 128), 128, 0, st, padded_cnt, Cptr, Ccol, n_agg, out);
  cudaFreeAsync(ub, st);
  BAMG_LAUNCH_CHECK();
  return 0;
}
