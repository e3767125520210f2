// DMMA vs FFMA-pipe A/B for the fp64 block products of the path (north star: "tensor
// cores (DMMA) are used only if ncu shows they help on the batched 9x9 block
// products"). Dev tool, not part of the library:
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/dmma_ab tools/dmma_ab.cu
//   ./tools/dmma_ab            (and under ncu: sm__inst_executed_pipe_*, fp64 pipe activity)
//
// Three measurements, each a batch of independent 16x16x16 fp64 block products (the
// Galerkin coarse-block shape; a 9x9 S block pads to it) per warp:
//   dmma_reg : mma.sync.m8n8k4.f64 on register-resident fragments (tensor-pipe peak)
//   fma_smem : the same products with DFMA, B from shared memory (FP64-pipe peak)
//   dmma_gmem / fma_gmem : operands streamed from HBM (the path's regime: each
//              block product reads 2 KB + 2 KB and writes 2 KB)
#include <cuda_runtime.h>
#include <stdio.h>

#include <vector>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// C(16x16) += A(16x16) B(16x16): 4 output tiles x 4 k-steps of m8n8k4
__device__ __forceinline__ void prod16_dmma(const double (&a)[2][4], const double (&b)[4][2], double (&c)[2][2][2]) {
#pragma unroll
  for (int ti = 0; ti < 2; ++ti)
#pragma unroll
    for (int tj = 0; tj < 2; ++tj)
#pragma unroll
      for (int k = 0; k < 4; ++k) dmma(c[ti][tj][0], c[ti][tj][1], a[ti][k], b[k][tj]);
}

__global__ void k_dmma_reg(const double* __restrict__ A, const double* __restrict__ B, double* out, int reps) {
  int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double a[2][4], b[4][2], c[2][2][2] = {};
#pragma unroll
  for (int ti = 0; ti < 2; ++ti)
#pragma unroll
    for (int k = 0; k < 4; ++k) a[ti][k] = A[(ti * 8 + g) * 16 + k * 4 + t];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int tj = 0; tj < 2; ++tj) b[k][tj] = B[(k * 4 + t) * 16 + tj * 8 + g];
  for (int r = 0; r < reps; ++r) prod16_dmma(a, b, c);
  double s = 0;
#pragma unroll
  for (int ti = 0; ti < 2; ++ti)
#pragma unroll
    for (int tj = 0; tj < 2; ++tj) s += c[ti][tj][0] + c[ti][tj][1];
  if (s == 12345.678) out[0] = s;
}

// lane owns 8 outputs: row lane/2, columns 8*(lane&1)..+8; A row in registers, B in smem
__global__ void k_fma_smem(const double* __restrict__ A, const double* __restrict__ B, double* out, int reps) {
  __shared__ double sb[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sb[i] = B[i];
  __syncthreads();
  int lane = threadIdx.x & 31, row = lane >> 1, c0 = 8 * (lane & 1);
  double ar[16], c[8] = {};
#pragma unroll
  for (int k = 0; k < 16; ++k) ar[k] = A[row * 16 + k];
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int j = 0; j < 8; ++j) c[j] = fma(ar[k], sb[k * 16 + c0 + j], c[j]);
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j];
  if (s == 12345.678) out[0] = s;
}

// streamed: warp w multiplies block pairs (A_i, B_i) -> C_i, i = w, w + nwarps, ...
__global__ void k_dmma_gmem(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C,
                            int nblk) {
  int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < nblk; i += nw) {
    const double* a_ = A + (size_t)i * 256;
    const double* b_ = B + (size_t)i * 256;
    double a[2][4], b[4][2], c[2][2][2] = {};
#pragma unroll
    for (int ti = 0; ti < 2; ++ti)
#pragma unroll
      for (int k = 0; k < 4; ++k) a[ti][k] = a_[(ti * 8 + g) * 16 + k * 4 + t];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int tj = 0; tj < 2; ++tj) b[k][tj] = b_[(k * 4 + t) * 16 + tj * 8 + g];
    prod16_dmma(a, b, c);
    double* c_ = C + (size_t)i * 256;
#pragma unroll
    for (int ti = 0; ti < 2; ++ti)
#pragma unroll
      for (int tj = 0; tj < 2; ++tj) {
        c_[(ti * 8 + g) * 16 + tj * 8 + 2 * t] = c[ti][tj][0];
        c_[(ti * 8 + g) * 16 + tj * 8 + 2 * t + 1] = c[ti][tj][1];
      }
  }
}

__global__ void k_fma_gmem(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C,
                           int nblk) {
  int lane = threadIdx.x & 31, row = lane >> 1, c0 = 8 * (lane & 1);
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < nblk; i += nw) {
    const double* a_ = A + (size_t)i * 256;
    const double* b_ = B + (size_t)i * 256;
    double c[8] = {};
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      double ak = a_[row * 16 + k];
#pragma unroll
      for (int j = 0; j < 8; ++j) c[j] = fma(ak, b_[k * 16 + c0 + j], c[j]);
    }
    double* c_ = C + (size_t)i * 256 + row * 16 + c0;
#pragma unroll
    for (int j = 0; j < 8; ++j) c_[j] = c[j];
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nblk = 1 << 20;  // 1M block products: 2 GB in, 2 GB out... (2 KB each)
  double *A, *B, *C;
  cudaMalloc(&A, sizeof(double) * 256 * (size_t)nblk);
  cudaMalloc(&B, sizeof(double) * 256 * (size_t)nblk);
  cudaMalloc(&C, sizeof(double) * 256 * (size_t)nblk);
  {
    std::vector<double> h(256 * 64);
    for (size_t i = 0; i < h.size(); ++i) h[i] = 1.0 + 1e-3 * (double)(i % 97);
    for (int k = 0; k < nblk / 64; ++k) {
      cudaMemcpy(A + (size_t)k * h.size(), h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
      cudaMemcpy(B + (size_t)k * h.size(), h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
    }
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto fn, double flops, double bytes) {
    fn();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    printf("%-10s %9.3f ms  %8.2f TFLOP/s  %8.1f GB/s\n", name, ms, flops / ms / 1e9, bytes / ms / 1e6);
  };
  const int reps = 2048, warps_per_sm = 16;
  const int grid = sms * warps_per_sm / 4;  // 128-thread CTAs
  double fl_reg = 2.0 * 4096 * reps * (double)grid * 4;
  timeit("dmma_reg", [&] { k_dmma_reg<<<grid, 128>>>(A, B, C, reps); }, fl_reg, 0);
  timeit("fma_smem", [&] { k_fma_smem<<<grid, 128>>>(A, B, C, reps); }, fl_reg, 0);
  double fl = 2.0 * 4096 * nblk, by = 3.0 * 2048 * nblk;
  timeit("dmma_gmem", [&] { k_dmma_gmem<<<sms * 8, 128>>>(A, B, C, nblk); }, fl, by);
  timeit("fma_gmem", [&] { k_fma_gmem<<<sms * 8, 128>>>(A, B, C, nblk); }, fl, by);
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
