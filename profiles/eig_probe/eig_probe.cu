// Timing probe (not product code): cuSOLVER symmetric eigensolver variants on
// the c5 subdomain size, to choose the setup's eigensolver call.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a eig_probe.cu -lcusolver -o eig_probe
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

__global__ void fill(int n, double* a, unsigned long long seed) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)n * n) return;
  int i = int(t % n), j = int(t / n);
  int lo = i < j ? i : j, hi = i < j ? j : i;
  unsigned long long z = seed + 0x9E3779B97F4A7C15ull * (unsigned long long)(lo * (long long)n + hi + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  double v = double(z >> 11) * 0x1.0p-53 - 0.5;
  a[t] = (i == j) ? v + 4.0 : v * 0.01;
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 5376;
  const int S = argc > 2 ? atoi(argv[2]) : 8;
  const int M = argc > 3 ? atoi(argv[3]) : 16;  // matrices
  std::vector<cudaStream_t> st(S);
  std::vector<cusolverDnHandle_t> h(S);
  std::vector<cusolverDnParams_t> pr(S);
  for (int i = 0; i < S; ++i) {
    cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
    cusolverDnCreate(&h[i]);
    cusolverDnSetStream(h[i], st[i]);
    cusolverDnCreateParams(&pr[i]);
  }
  std::vector<double*> A(M), W(M);
  for (int m = 0; m < M; ++m) {
    cudaMalloc(&A[m], sizeof(double) * n * n);
    cudaMalloc(&W[m], sizeof(double) * n);
  }
  int* info;
  cudaMalloc(&info, sizeof(int) * M);
  int lw = 0;
  cusolverDnDsyevd_bufferSize(h[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A[0], n, W[0], &lw);
  size_t dws = 0, hws = 0;
  cusolverDnXsyevd_bufferSize(h[0], pr[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A[0], n,
                              CUDA_R_64F, W[0], CUDA_R_64F, &dws, &hws);
  std::vector<double*> work(S);
  std::vector<void*> dwork(S);
  std::vector<std::vector<char>> hwork(S, std::vector<char>(hws + 1));
  for (int i = 0; i < S; ++i) {
    cudaMalloc(&work[i], sizeof(double) * (lw + 1));
    cudaMalloc(&dwork[i], dws + 8);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int lwx = 0, meig = 0;
  cusolverDnDsyevdx_bufferSize(h[0], CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, A[0], n,
                               0.0, 0.0, 1, 80, &meig, W[0], &lwx);
  std::vector<double*> workx(S);
  for (int i = 0; i < S; ++i) cudaMalloc(&workx[i], sizeof(double) * (lwx + 1));
  for (int variant = 0; variant < 4; ++variant) {
    for (int m = 0; m < M; ++m) fill<<<int(((long long)n * n + 255) / 256), 256>>>(n, A[m], m);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    if (variant == 2) {  // one host thread per stream: Dsyevd blocks its calling thread
      std::vector<std::thread> th;
      for (int q = 0; q < S; ++q)
        th.emplace_back([&, q]() {
          for (int m = q; m < M; m += S)
            cusolverDnDsyevd(h[q], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A[m], n, W[m], work[q], lw,
                             info + m);
          cudaStreamSynchronize(st[q]);
        });
      for (auto& t : th) t.join();
    }
    if (variant == 3) {  // the 80 smallest eigenpairs only
      for (int m = 0; m < M; ++m) {
        int q = m % S;
        cusolverDnDsyevdx(h[q], CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, A[m], n, 0.0,
                          0.0, 1, 80, &meig, W[m], workx[q], lwx, info + m);
      }
    }
    for (int m = 0; m < M && variant < 2; ++m) {
      int q = m % S;
      if (variant == 0)
        cusolverDnDsyevd(h[q], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A[m], n, W[m], work[q], lw,
                         info + m);
      else
        cusolverDnXsyevd(h[q], pr[q], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A[m], n,
                         CUDA_R_64F, W[m], CUDA_R_64F, dwork[q], dws, hwork[q].data(), hws, info + m);
    }
    for (int i = 0; i < S; ++i) cudaStreamSynchronize(st[i]);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"variant\": \"%s\", \"n\": %d, \"streams\": %d, \"matrices\": %d, \"ms_per_matrix\": %.2f, \"err\": \"%s\"}\n",
           variant == 0 ? "Dsyevd" : variant == 1 ? "Xsyevd" : variant == 2 ? "Dsyevd_threads" : "Dsyevdx_80", n, S, M, ms / M, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
