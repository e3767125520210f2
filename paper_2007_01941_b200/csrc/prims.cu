// Primitives: stable LSD radix sort, exclusive scan, segment pointers, gathers,
// deterministic reductions, context / error plumbing.
#include <stdarg.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "common.cuh"
#include "ctx.h"

// ---------------------------------------------------------------------------
// error text + device info

static thread_local char g_err[1024] = {0};
std::atomic<long long> g_bamg_launches{0};

extern "C" int64_t bamg_launch_count(void) { return g_bamg_launches.load(std::memory_order_relaxed); }

void bamg_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" int bamg_last_error(char* buf, size_t n) {
  if (!buf || n == 0) return (int)strlen(g_err);
  strncpy(buf, g_err, n - 1);
  buf[n - 1] = 0;
  return (int)strlen(g_err);
}

bool bamg_pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("BAMG_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

__global__ void k_set_i32(int* p, int v) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *p = v;
}
void set_i32(int* p, int v, cudaStream_t st) { launch(k_set_i32, 1, 32, 0, st, p, v); }

int bamg_num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
      sms = 148;
  }
  return sms;
}

extern "C" int bamg_version(void) { return BAMG_ABI_VERSION; }

extern "C" bamg_ctx* bamg_ctx_create(void) {
  bamg_ctx* c = new bamg_ctx();
  memset(c, 0, sizeof(*c));
  if (cudaMalloc(&c->partials, sizeof(double) * BAMG_MAX_PARTIALS) != cudaSuccess) goto fail;
  if (cudaMalloc(&c->counters, sizeof(unsigned int) * BAMG_NUM_COUNTERS) != cudaSuccess) goto fail;
  if (cudaMalloc(&c->scalars, sizeof(double) * BAMG_NUM_SCALARS) != cudaSuccess) goto fail;
  if (cudaMalloc(&c->flags, sizeof(int) * BAMG_NUM_FLAGS) != cudaSuccess) goto fail;
  if (cudaMallocHost(&c->host_scalars, sizeof(double) * BAMG_NUM_SCALARS) != cudaSuccess) goto fail;
  if (cudaMallocHost(&c->host_flags, sizeof(int) * BAMG_NUM_FLAGS) != cudaSuccess) goto fail;
  {
    // stream-ordered scratch (sort keys, pair lists, plan vectors) comes from the
    // device's default pool; keep its memory mapped across synchronisations so
    // repeated solves do not pay page-mapping costs on every allocation
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  cudaMemset(c->counters, 0, sizeof(unsigned int) * BAMG_NUM_COUNTERS);
  cudaMemset(c->scalars, 0, sizeof(double) * BAMG_NUM_SCALARS);
  cudaMemset(c->flags, 0, sizeof(int) * BAMG_NUM_FLAGS);
  if (cudaDeviceSynchronize() != cudaSuccess) goto fail;
  return c;
fail:
  bamg_set_error("bamg_ctx_create: %s", cudaGetErrorString(cudaGetLastError()));
  bamg_ctx_destroy(c);
  return nullptr;
}

extern "C" void bamg_ctx_destroy(bamg_ctx* c) {
  if (!c) return;
  if (c->partials) cudaFree(c->partials);
  if (c->counters) cudaFree(c->counters);
  if (c->scalars) cudaFree(c->scalars);
  if (c->flags) cudaFree(c->flags);
  if (c->host_scalars) cudaFreeHost(c->host_scalars);
  if (c->host_flags) cudaFreeHost(c->host_flags);
  delete c;
}

// ---------------------------------------------------------------------------
// exclusive scan (int32), reduce-then-scan with recursion over block sums

#define SCAN_THREADS 256
#define SCAN_ITEMS 8
#define SCAN_TILE (SCAN_THREADS * SCAN_ITEMS)

__device__ __forceinline__ int block_exclusive_scan_int(int v, int* total, int* sm) {
  // sm: >= 32 ints
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(FULL_MASK, incl, o);
    if (lane >= o) incl += t;
  }
  __syncthreads();
  if (lane == 31) sm[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int w = (lane < (int)(blockDim.x >> 5)) ? sm[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(FULL_MASK, wi, o);
      if (lane >= o) wi += t;
    }
    sm[lane] = wi - w;  // exclusive warp offsets
    if (lane == 31) sm[32] = wi;
  }
  __syncthreads();
  int r = sm[wid] + incl - v;
  *total = sm[32];
  __syncthreads();
  return r;
}

__global__ void k_scan_reduce(const int* __restrict__ in, int64_t n, int* __restrict__ sums) {
  __shared__ double scratch[33];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  int s = 0;
  for (int i = threadIdx.x; i < SCAN_TILE; i += SCAN_THREADS) {
    int64_t g = base + i;
    if (g < n) s += in[g];
  }
  s = warp_sum_int(s);
  __shared__ int ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < SCAN_THREADS / 32; ++w) t += ws[w];
    sums[blockIdx.x] = t;
  }
  (void)scratch;
}

__global__ void k_scan_apply(const int* __restrict__ in, int64_t n, const int* __restrict__ offs,
                             int* __restrict__ out, int* __restrict__ total_out) {
  __shared__ int sm[33];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  int v[SCAN_ITEMS];
  int s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    int64_t g = base + k;
    v[k] = (g < n) ? in[g] : 0;
    s += v[k];
  }
  int tot;
  int ex = block_exclusive_scan_int(s, &tot, sm);
  int run = ex + (offs ? offs[blockIdx.x] : 0);
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    int64_t g = base + k;
    if (g < n) out[g] = run;
    run += v[k];
  }
  if (total_out && blockIdx.x == gridDim.x - 1 && threadIdx.x == SCAN_THREADS - 1) *total_out = run;
}

// out may alias in. If total != nullptr it receives the sum (device int).
int scan_exclusive_int(const int* in, int* out, int64_t n, int* total, cudaStream_t st) {
  if (n <= 0) {
    if (total) BAMG_CUDA_CHECK(cudaMemsetAsync(total, 0, sizeof(int), st));
    return 0;
  }
  int64_t nb = ceil_div(n, SCAN_TILE);
  if (nb == 1) {
    launch(k_scan_apply, 1, SCAN_THREADS, 0, st, in, n, nullptr, out, total);
    BAMG_LAUNCH_CHECK();
    return 0;
  }
  int* sums = nullptr;
  BAMG_CUDA_CHECK(cudaMallocAsync(&sums, sizeof(int) * nb, st));
  launch(k_scan_reduce, (unsigned)nb, SCAN_THREADS, 0, st, in, n, sums);
  BAMG_LAUNCH_CHECK();
  int rc = scan_exclusive_int(sums, sums, nb, nullptr, st);
  if (rc) return rc;
  launch(k_scan_apply, (unsigned)nb, SCAN_THREADS, 0, st, in, n, sums, out, total);
  BAMG_LAUNCH_CHECK();
  BAMG_CUDA_CHECK(cudaFreeAsync(sums, st));
  return 0;
}

extern "C" int bamg_scan_exclusive_i32(bamg_ctx* ctx, const int32_t* in, int32_t* out, int64_t n,
                                       int32_t* total, void* stream) {
  (void)ctx;
  return scan_exclusive_int(in, out, n, total, as_stream(stream));
}

// ---------------------------------------------------------------------------
// stable LSD radix sort of (uint32 key, uint32 value), 8-bit digits.
// Tile = 8 warps x 8 rounds x 32 lanes = 2048 items; within a warp items are
// ranked round by round with __match_any_sync, so ranks follow input order.

// The scatter stages each tile in shared memory in digit order first, so that the
// global writes are runs of consecutive addresses per digit (a tile of 4096 items
// puts ~16 items in each of the 256 buckets) instead of 32 lanes writing to 32
// different buckets; the permutation is the same (stable, input order per digit).
#define RS_WARPS 8
#define RS_ROUNDS 16
#define RS_TILE (RS_WARPS * RS_ROUNDS * 32)

__global__ void __launch_bounds__(RS_WARPS * 32)
k_radix_hist(const uint32_t* __restrict__ keys, int64_t n, int shift, int ntiles,
             int* __restrict__ hist) {
  __shared__ int h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * RS_TILE;
  for (int i = threadIdx.x; i < RS_TILE; i += blockDim.x) {
    int64_t g = base + i;
    if (g < n) atomicAdd(&h[(keys[g] >> shift) & 255u], 1);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += blockDim.x) hist[(int64_t)d * ntiles + blockIdx.x] = h[d];
}

__global__ void __launch_bounds__(RS_WARPS * 32)
k_radix_scatter(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, int64_t n,
                int shift, int ntiles, const int* __restrict__ offs,
                uint32_t* __restrict__ kout, uint32_t* __restrict__ vout) {
  __shared__ int wcount[RS_WARPS][256];
  __shared__ int tile_off[256];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = lane; i < 256; i += 32) wcount[w][i] = 0;
  for (int d = threadIdx.x; d < 256; d += blockDim.x) tile_off[d] = offs[(int64_t)d * ntiles + blockIdx.x];
  __syncwarp();
  int64_t base = (int64_t)blockIdx.x * RS_TILE + (int64_t)w * RS_ROUNDS * 32;
  uint32_t key[RS_ROUNDS], val[RS_ROUNDS];
  int rank[RS_ROUNDS];
  unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < RS_ROUNDS; ++r) {
    int64_t g = base + r * 32 + lane;
    bool ok = g < n;
    key[r] = ok ? kin[g] : 0xffffffffu;
    val[r] = ok ? vin[g] : 0u;
    unsigned d = (key[r] >> shift) & 255u;
    unsigned act = __ballot_sync(FULL_MASK, ok);
    unsigned peers = __match_any_sync(FULL_MASK, ok ? d : 0x1000u + lane);
    peers &= act;
    int before = wcount[w][d & 255u];
    __syncwarp();
    rank[r] = before + __popc(peers & lt);
    if (ok && (peers & lt) == 0) wcount[w][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per-digit exclusive prefix over warps (thread d owns digit d), then a block-wide
  // exclusive scan of the digit totals: where each digit starts in the tile
  static_assert(RS_WARPS * 32 == 256, "one thread per digit");
  __shared__ int dstart[257];
  __shared__ int wtot[RS_WARPS];
  {
    const int d = threadIdx.x;
    int run = 0;
#pragma unroll
    for (int q = 0; q < RS_WARPS; ++q) {
      int c = wcount[q][d];
      wcount[q][d] = run;
      run += c;
    }
    int incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(FULL_MASK, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) wtot[w] = incl;
    __syncthreads();
    int off = 0;
    for (int q = 0; q < w; ++q) off += wtot[q];
    dstart[d] = off + incl - run;
    if (d == 255) dstart[256] = off + incl;
  }
  __syncthreads();
  __shared__ uint32_t skey[RS_TILE];
  __shared__ uint32_t sval[RS_TILE];
#pragma unroll
  for (int r = 0; r < RS_ROUNDS; ++r) {
    int64_t g = base + r * 32 + lane;
    if (g < n) {
      unsigned d = (key[r] >> shift) & 255u;
      int lp = dstart[d] + wcount[w][d] + rank[r];
      skey[lp] = key[r];
      sval[lp] = val[r];
    }
  }
  __syncthreads();
  int cnt = dstart[256];
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    uint32_t k = skey[i];
    unsigned d = (k >> shift) & 255u;
    int64_t pos = (int64_t)tile_off[d] + (i - dstart[d]);
    kout[pos] = k;
    vout[pos] = sval[i];
  }
}

// Sorts by key bits [0, key_bits). kout/vout receive the result; inputs untouched.
int radix_sort_pairs(const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout,
                     int64_t n, int key_bits, cudaStream_t st) {
  if (n <= 0) return 0;
  int passes = key_bits <= 0 ? 1 : (key_bits + 7) / 8;
  int ntiles = (int)ceil_div(n, RS_TILE);
  int* hist = nullptr;
  uint32_t *kb = nullptr, *vb = nullptr;
  BAMG_CUDA_CHECK(cudaMallocAsync(&hist, sizeof(int) * 256 * (int64_t)ntiles, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&kb, sizeof(uint32_t) * n, st));
  BAMG_CUDA_CHECK(cudaMallocAsync(&vb, sizeof(uint32_t) * n, st));
  // ping-pong so that the last pass writes kout/vout
  const uint32_t *ks = kin, *vs = vin;
  for (int p = 0; p < passes; ++p) {
    bool last = (p == passes - 1);
    bool to_out = ((passes - 1 - p) % 2) == 0;
    uint32_t* kd = to_out ? kout : kb;
    uint32_t* vd = to_out ? vout : vb;
    (void)last;
    launch(k_radix_hist, ntiles, RS_WARPS * 32, 0, st, ks, n, 8 * p, ntiles, hist);
    BAMG_LAUNCH_CHECK();
    int rc = scan_exclusive_int(hist, hist, 256 * (int64_t)ntiles, nullptr, st);
    if (rc) return rc;
    launch(k_radix_scatter, ntiles, RS_WARPS * 32, 0, st, ks, vs, n, 8 * p, ntiles, hist, kd, vd);
    BAMG_LAUNCH_CHECK();
    ks = kd;
    vs = vd;
  }
  BAMG_CUDA_CHECK(cudaFreeAsync(hist, st));
  BAMG_CUDA_CHECK(cudaFreeAsync(kb, st));
  BAMG_CUDA_CHECK(cudaFreeAsync(vb, st));
  return 0;
}

extern "C" int bamg_sort_pairs_u32(bamg_ctx* ctx, const uint32_t* kin, const uint32_t* vin,
                                   uint32_t* kout, uint32_t* vout, int64_t n, int key_bits,
                                   void* stream) {
  (void)ctx;
  return radix_sort_pairs(kin, vin, kout, vout, n, key_bits, as_stream(stream));
}

// ---------------------------------------------------------------------------
// segment pointers from sorted segment ids: ptr[s] = first i with id[i] >= s

__global__ void k_segment_ptr(const int* __restrict__ ids, int64_t n, int nseg, int* __restrict__ ptr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
    int prev = (i == 0) ? -1 : ids[i - 1];
    int cur = (i == n) ? nseg : ids[i];
    for (int s = prev + 1; s <= cur; ++s) ptr[s] = (int)i;
  }
}

int segment_ptr(const int* ids, int64_t n, int nseg, int* ptr, cudaStream_t st) {
  launch(k_segment_ptr, grid_for(n + 1, 256), 256, 0, st, ids, n, nseg, ptr);
  BAMG_LAUNCH_CHECK();
  return 0;
}

extern "C" int bamg_segment_ptr(bamg_ctx* ctx, const int32_t* sorted_ids, int64_t n, int32_t nseg,
                                int32_t* ptr, void* stream) {
  (void)ctx;
  return segment_ptr(sorted_ids, n, nseg, ptr, as_stream(stream));
}

// ---------------------------------------------------------------------------
// gathers

__global__ void k_gather_rows_f64(const double* __restrict__ src, const int* __restrict__ idx,
                                  int64_t n, int width, double* __restrict__ dst) {
  int64_t total = n * width;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / width;
    int c = (int)(t - r * width);
    dst[t] = src[(int64_t)idx[r] * width + c];
  }
}

__global__ void k_scatter_rows_f64(const double* __restrict__ src, const int* __restrict__ idx,
                                   int64_t n, int width, double* __restrict__ dst) {
  int64_t total = n * width;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / width;
    int c = (int)(t - r * width);
    dst[(int64_t)idx[r] * width + c] = src[t];
  }
}

__global__ void k_gather_i32(const int* __restrict__ src, const int* __restrict__ idx, int64_t n,
                             int* __restrict__ dst) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    dst[t] = src[idx[t]];
}

extern "C" int bamg_gather_rows_f64(bamg_ctx* ctx, const double* src, const int32_t* idx, int64_t n,
                                    int32_t width, double* dst, void* stream) {
  (void)ctx;
  if (n <= 0) return 0;
  launch(k_gather_rows_f64, grid_for(n * width, 256), 256, 0, as_stream(stream), src, idx, n, width, dst);
  BAMG_LAUNCH_CHECK();
  return 0;
}

extern "C" int bamg_scatter_rows_f64(bamg_ctx* ctx, const double* src, const int32_t* idx, int64_t n,
                                     int32_t width, double* dst, void* stream) {
  (void)ctx;
  if (n <= 0) return 0;
  launch(k_scatter_rows_f64, grid_for(n * width, 256), 256, 0, as_stream(stream), src, idx, n, width, dst);
  BAMG_LAUNCH_CHECK();
  return 0;
}

extern "C" int bamg_gather_i32(bamg_ctx* ctx, const int32_t* src, const int32_t* idx, int64_t n,
                               int32_t* dst, void* stream) {
  (void)ctx;
  if (n <= 0) return 0;
  launch(k_gather_i32, grid_for(n, 256), 256, 0, as_stream(stream), src, idx, n, dst);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------------------
// deterministic vector reductions (fixed grid, fixed order)

#define RED_THREADS 256

__global__ void __launch_bounds__(RED_THREADS)
k_dot(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
      double* partials, unsigned int* counter, double* out) {
  PDL_ENTRY();
  __shared__ double scratch[33];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s = fma(x[i], y[i], s);
  s = block_sum(s, scratch);
  grid_finish(partials, counter, s, scratch, out);
}

__global__ void __launch_bounds__(RED_THREADS)
k_absmax(const double* __restrict__ x, int64_t n, double* partials, unsigned int* counter, double* out) {
  __shared__ double scratch[33];
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double a = fabs(x[i]);
    m = (a > m || a != a) ? a : m;
  }
  // max tree (NaN-propagating)
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    double t = __shfl_xor_sync(FULL_MASK, m, o);
    m = (t > m || t != t) ? t : m;
  }
  if (lane == 0) scratch[wid] = m;
  __syncthreads();
  __shared__ bool am_last;
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < RED_THREADS / 32; ++w) b = (scratch[w] > b || scratch[w] != scratch[w]) ? scratch[w] : b;
    partials[blockIdx.x] = b;
    __threadfence();
    am_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (am_last && threadIdx.x == 0) {
    __threadfence();
    double b = 0.0;
    for (unsigned i = 0; i < gridDim.x; ++i) {
      double v = ((volatile double*)partials)[i];
      b = (v > b || v != v) ? v : b;
    }
    *out = b;
    *counter = 0u;
  }
}

int dot_dev(bamg_ctx* ctx, const double* x, const double* y, int64_t n, double* out, cudaStream_t st) {
  int g = grid_for(n, RED_THREADS, 4);
  launch_pdl(k_dot, g, RED_THREADS, 0, st, x, y, n, ctx->partials, ctx->counters + BAMG_CTR_DOT, out);
  BAMG_LAUNCH_CHECK();
  return 0;
}

extern "C" int bamg_dot(bamg_ctx* ctx, const double* x, const double* y, int64_t n, double* out_dev,
                        void* stream) {
  return dot_dev(ctx, x, y, n, out_dev, as_stream(stream));
}

extern "C" int bamg_absmax(bamg_ctx* ctx, const double* x, int64_t n, double* out_dev, void* stream) {
  cudaStream_t st = as_stream(stream);
  int g = grid_for(n, RED_THREADS, 4);
  launch(k_absmax, g, RED_THREADS, 0, st, x, n, ctx->partials, ctx->counters + BAMG_CTR_DOT, out_dev);
  BAMG_LAUNCH_CHECK();
  return 0;
}

// y = a*x + b*y  (elementwise, n doubles); b == 0 does not read y
__global__ void k_axpby(double a, const double* __restrict__ x, double b, double* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (b == 0.0) ? a * x[i] : a * x[i] + b * y[i];
}

extern "C" int bamg_axpby(bamg_ctx* ctx, double a, const double* x, double b, double* y, int64_t n,
                          void* stream) {
  (void)ctx;
  if (n <= 0) return 0;
  launch(k_axpby, grid_for(n, 256), 256, 0, as_stream(stream), a, x, b, y, n);
  BAMG_LAUNCH_CHECK();
  return 0;
}
