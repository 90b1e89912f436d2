// Micro-benchmark (not product code): do DMMA (mma.sync m8n8k4 f64) and scalar
// DFMA run on separate pipes of a B200 SM, i.e. can a kernel that issues both
// exceed the rate of either alone?  Three register-only loops: DMMA only, DFMA
// only, and even warps DMMA / odd warps DFMA in the same CTA.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a fp64_pipes.cu -o fp64_pipes
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// mode 0: all warps DMMA; 1: all warps DFMA; 2: even warps DMMA, odd warps DFMA
__global__ void __launch_bounds__(256, 2) k(int mode, int iters, double* out) {
  const int warp = threadIdx.x >> 5;
  const bool use_dmma = mode == 0 || (mode == 2 && (warp & 1) == 0);
  double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = i;
  if (use_dmma) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 16; i += 2) dmma(acc[i], acc[i + 1], a, b);  // 8 DMMA = 8 * 256 FMA per warp
    }
  } else {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fma(a, acc[i], b);  // 16 DFMA per lane = 512 FMA per warp
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 2, threads = 256, iters = 200000;
  double* out;
  cudaMalloc(&out, sizeof(double) * grid * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode) {
    k<<<grid, threads>>>(mode, 1000, out);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    k<<<grid, threads>>>(mode, iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = double(grid) * threads / 32;
    double fma_total;
    if (mode == 0) fma_total = warps * iters * 8.0 * 256.0;
    else if (mode == 1) fma_total = warps * iters * 512.0;
    else fma_total = warps / 2 * iters * (8.0 * 256.0 + 512.0);
    std::printf("{\"mode\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", mode, ms, 2.0 * fma_total / ms / 1e9);
  }
  return 0;
}
