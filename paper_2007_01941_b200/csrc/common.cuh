// Shared device helpers for libbamg_b200 (sm_100a, fp64 block-sparse path).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>
#include <utility>

#include "../../include/bamg_b200.h"

// Every kernel of the library goes through launch(): it counts launches
// (bamg_launch_count) so benchmarks can report exactly how many of OUR kernels
// ran in a timed region.
extern std::atomic<long long> g_bamg_launches;

template <typename... KArgs, typename... Args>
static inline void launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                          Args&&... args) {
  g_bamg_launches.fetch_add(1, std::memory_order_relaxed);
  k<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
}

// Programmatic dependent launch (PDL) for the kernel chains of the V-cycle and PCG
// graphs: launch_pdl sets the programmatic-stream-serialization attribute, so in a
// captured graph the edge to the previous kernel becomes programmatic and the next
// kernel's CTAs are launched while the previous one drains. Every kernel launched
// this way starts with PDL_ENTRY(): griddepcontrol.wait (returns once the
// predecessor grid has completed and its writes are visible -- nothing is read
// early) and launch_dependents (lets the successor's launch begin). BAMG_PDL=0
// turns the attribute off (A/B).
bool bamg_pdl_enabled();
template <typename... KArgs, typename... Args>
static inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  if (!bamg_pdl_enabled()) {
    launch(k, grid, block, smem, st, std::forward<Args>(args)...);
    return;
  }
  g_bamg_launches.fetch_add(1, std::memory_order_relaxed);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}
#define PDL_ENTRY() asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")

#define BAMG_WARP 32
#define FULL_MASK 0xffffffffu

// Thread-local last-error text (bamg_last_error).
void bamg_set_error(const char* fmt, ...);

#define BAMG_CUDA_CHECK(expr)                                                     \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      bamg_set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,                   \
                     cudaGetErrorString(_e));                                     \
      return BAMG_ERR_CUDA;                                                       \
    }                                                                             \
  } while (0)

#define BAMG_LAUNCH_CHECK() BAMG_CUDA_CHECK(cudaGetLastError())

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// grid size for grid-stride loops: a multiple of the SM count (148 on B200)
int bamg_num_sms();
static inline int grid_for(int64_t n, int threads, int per_sm = 8) {
  int64_t want = ceil_div(n, threads);
  int64_t cap = (int64_t)bamg_num_sms() * per_sm;
  if (want < 1) want = 1;
  return (int)(want < cap ? want : cap);
}

// one int32 device slot <- v (a kernel, not a pageable host->device copy)
__global__ void k_set_i32(int* p, int v);
void set_i32(int* p, int v, cudaStream_t st);

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
  return v;
}

__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
  return v;
}

__device__ __forceinline__ int warp_max_int(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(FULL_MASK, v, o));
  return v;
}

// Deterministic block-wide sum (fixed tree). `scratch` >= 32 doubles. All threads
// receive the result.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double t = (threadIdx.x < nw) ? scratch[threadIdx.x] : 0.0;
  if (wid == 0) t = warp_sum(t);
  if (threadIdx.x == 0) scratch[0] = t;
  __syncthreads();
  double r = scratch[0];
  __syncthreads();
  return r;
}

// Last-block-done finisher for deterministic grid reductions: every block writes
// `partial[blockIdx.x]`, the final block sums all partials in index order.
// Returns true in the block that must write the final value (thread 0 holds it).
__device__ __forceinline__ bool grid_finish(double* partials, unsigned int* counter,
                                            double block_value, double* scratch,
                                            double* out_total) {
  __shared__ bool am_last;
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = block_value;
    __threadfence();
    unsigned int t = atomicAdd(counter, 1u);
    am_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  double v = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x)
    v += ((volatile double*)partials)[i];
  v = block_sum(v, scratch);
  if (threadIdx.x == 0) {
    *out_total = v;
    *counter = 0u;  // re-arm for the next launch
  }
  return true;
}

// L2 eviction-priority policies (createpolicy) and hinted loads/stores. The solve
// phase streams operators far larger than L2 (evict_first) while small arrays that
// are written by one kernel and gathered by the next -- the mirrored products of
// the half-storage products -- stay resident (evict_last).
enum { L2_NORMAL = 0, L2_FIRST = 1, L2_LAST = 2 };
__device__ __forceinline__ uint64_t l2_policy(int kind) {
  uint64_t p;
#ifdef NO_L2_HINTS
  kind = L2_NORMAL;
#endif
  if (kind == L2_FIRST)
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else if (kind == L2_LAST)
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_pol(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ld2_pol(const double2* p, uint64_t pol) {
  double2 v;
  asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_pol(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st2_pol(double2* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}

// cp.async (LDGSTS) helpers: 16 B global -> shared copies, L2 only (.cg).
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc) : "memory");
}
// copies src_bytes (0..16) and zero-fills the rest of the 16 B destination
__device__ __forceinline__ void cp_async16_zfill(void* sdst, const void* gsrc, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc), "r"(src_bytes) : "memory");
}
// 8 B copy (L1-cached form; for sources that are only 8 B aligned)
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
// wait until at most `pending` (clamped to 0..7) of this thread's newest groups are in flight
__device__ __forceinline__ void cp_async_wait_dyn(int pending) {
  switch (pending <= 0 ? 0 : (pending >= 7 ? 7 : pending)) {
    case 0: cp_async_wait<0>(); break;
    case 1: cp_async_wait<1>(); break;
    case 2: cp_async_wait<2>(); break;
    case 3: cp_async_wait<3>(); break;
    case 4: cp_async_wait<4>(); break;
    case 5: cp_async_wait<5>(); break;
    case 6: cp_async_wait<6>(); break;
    default: cp_async_wait<7>(); break;
  }
}

// Asynchronous form of gather_records (below) for warp-per-segment gathers: the
// pieces of up to 32 observation records are copied by cp.async into a TRANSPOSED
// shared layout -- piece p of lane l's record at buf + p*64 + 2l (16 B aligned,
// conflict-free reads) -- so a warp can double-buffer: the copies of chunk c+1 are
// in flight while chunk c is consumed. NA pieces from 16 B piece a0 of the record,
// NB from b0. Commits one cp.async group.
template <int NA, int NB, int NX>
__device__ __forceinline__ void rec_issue(const double* __restrict__ J, int o_lane, bool valid, int a0, int b0,
                                          const double* __restrict__ extra, double* buf, int lane);

__device__ __forceinline__ int lower_bound_i32(const int* a, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Observation record layout (256 B, 16 B aligned):
//   [ 0,18) F (2x9)   [18,24) E (2x3)   [24,30) H = E C^-1 (2x3)   [30,32) residual
#define REC 32
#define RF 0
#define RE 18
#define RH 24
#define RR 30

// ---------------------------------------------------------------------------
// warp-cooperative record gather: 32 observations (one per lane) -> shared memory.
// Fetches the double2 pieces [a0, a0+NA) then [b0, b0+NB) of each record, then
// (if `extra` != null) one double2 per observation from a separate (k,2) array;
// slot (l, i) of `buf` (stride ST doubles, odd) receives fetched piece i of lane l.
template <int NA, int NB, int NX, int ST>
__device__ __forceinline__ void gather_records(const double* __restrict__ J, int o_lane, bool valid, int a0, int b0,
                                               const double* __restrict__ extra, double* buf, int lane) {
  constexpr int NP = NA + NB + NX;
  double2 v[NP];
  // all NP loads are issued before any shared-memory store (no serialised latency)
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    int idx = k * 32 + lane;
    int l = idx / NP, i = idx - l * NP;
    int o = __shfl_sync(FULL_MASK, o_lane, l);
    int vv = __shfl_sync(FULL_MASK, (int)valid, l);
    const double2* src;
    if (i < NA) src = reinterpret_cast<const double2*>(J + (int64_t)o * REC) + a0 + i;
    else if (i < NA + NB) src = reinterpret_cast<const double2*>(J + (int64_t)o * REC) + b0 + i - NA;
    else src = reinterpret_cast<const double2*>(extra + (int64_t)o * 2);
    v[k] = vv ? __ldg(src) : make_double2(0.0, 0.0);
  }
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    int idx = k * 32 + lane;
    int l = idx / NP, i = idx - l * NP;
    buf[l * ST + 2 * i] = v[k].x;
    buf[l * ST + 2 * i + 1] = v[k].y;
  }
  __syncwarp();
}

template <int NA, int NB, int NX>
__device__ __forceinline__ void rec_issue(const double* __restrict__ J, int o_lane, bool valid, int a0, int b0,
                                          const double* __restrict__ extra, double* buf, int lane) {
  constexpr int NP = NA + NB + NX;
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    int idx = k * 32 + lane;
    int l = idx / NP, i = idx - l * NP;
    int o = __shfl_sync(FULL_MASK, o_lane, l);
    int vv = __shfl_sync(FULL_MASK, (int)valid, l);
    const double* src = i < NA + NB ? J + (int64_t)o * REC + 2 * (i < NA ? a0 + i : b0 + i - NA)
                                    : extra + (int64_t)o * 2;  // NX: one 16 B piece per obs of `extra`
    if (vv) cp_async16(buf + i * 64 + 2 * l, src);
  }
  cp_async_commit();
}
