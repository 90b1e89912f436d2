// Batched dense Cholesky factorisation, triangular solves and the
// generalized symmetric eigenproblem of the setup (hand-written, sm_100a):
//   cholesky              dense.cpp:226-249   (OneLevel AS / AS+ local factors,
//                                              preconditioner.cpp:20-30; the pencils' MB)
//   forward/backward_solve_multi  dense.cpp:274-297
//   generalized_sym_eig   dense.cpp:211-224   (GenEO pencils, coarse.cpp:98-111):
//       MB = L L^T, C = L^-1 MA L^-T (symmetrised), eig(C) (eig.cu), Y = L^-T Z
// Blocked right-looking algorithms on 64-column panels: the 64 x 64 diagonal
// block is factored and inverted by one CTA per problem in shared memory
// (k_potrf_diag); everything else is grouped FP64 tensor-core GEMMs
// (dgemm.cu) over all problems at once — the panel below the diagonal block
// (L21 = A21 L11^-T), the trailing rank-64 update (A22 -= L21 L21^T, lower
// tiles only), and the block substitutions with the inverted diagonal blocks.
#include <algorithm>
#include <cmath>
#include <vector>

#include "awg_internal.cuh"

namespace awgb {
namespace {

constexpr int kCB = 64;  // panel width

struct CholDev {
  double* A;     // n x n, ld: lower factor on return
  double* DI;    // panels x 64 x 64: inverse of each diagonal block (col-major)
  double* DIT;   // panels x 64 x 64: its transpose (col-major), the GEMM B operand
  int* info;     // 0 or (first non-positive pivot + 1)
  int n, ld;
};

// Cholesky of the diagonal block A(k0:k0+b, k0:k0+b) in shared memory, then
// its inverse (forward substitution against the identity, one column per thread).
constexpr size_t kDiagSmem = size_t(2) * kCB * (kCB + 1) * sizeof(double);
__global__ void __launch_bounds__(256) k_potrf_diag(const CholDev* __restrict__ jobs, int k0) {
  extern __shared__ double dsm[];
  double (*a)[kCB + 1] = reinterpret_cast<double (*)[kCB + 1]>(dsm);
  double (*inv)[kCB + 1] = reinterpret_cast<double (*)[kCB + 1]>(dsm + kCB * (kCB + 1));
  __shared__ int s_bad;
  const CholDev J = jobs[blockIdx.x];
  if (k0 >= J.n) return;
  const int b = min(kCB, J.n - k0), tid = threadIdx.x;
  if (tid == 0) s_bad = -1;
  for (int t = tid; t < kCB * kCB; t += blockDim.x) {
    const int i = t % kCB, j = t / kCB;
    a[i][j] = (i < b && j < b && i >= j) ? J.A[(k0 + i) + (size_t)(k0 + j) * J.ld] : (i == j ? 1.0 : 0.0);
  }
  __syncthreads();
  if (*J.info != 0) return;  // an earlier panel failed: stop (the error reports the first pivot)
  for (int c = 0; c < b; ++c) {
    const double piv = a[c][c];
    if (!(piv > 0.0)) {
      if (tid == 0) s_bad = c;
      __syncthreads();
      break;
    }
    const double l = sqrt(piv);
    __syncthreads();
    if (tid == 0) a[c][c] = l;
    for (int i = c + 1 + tid; i < b; i += blockDim.x) a[i][c] /= l;
    __syncthreads();
    // trailing update of the lower triangle (dense.cpp:238-246 order: column by column)
    for (int t = tid; t < (b - c - 1) * (b - c - 1); t += blockDim.x) {
      const int i = c + 1 + t % (b - c - 1), j = c + 1 + t / (b - c - 1);
      if (i >= j) a[i][j] -= a[i][c] * a[j][c];
    }
    __syncthreads();
  }
  if (s_bad >= 0) {
    if (tid == 0) *J.info = k0 + s_bad + 1;
    return;
  }
  // inverse of the lower triangular block: column j solves L x = e_j
  if (tid < kCB) {
    const int j = tid;
    for (int i = 0; i < kCB; ++i) {
      double v = (i == j) ? 1.0 : 0.0;
      if (i < j || i >= b) {
        inv[i][j] = (i == j) ? 1.0 : 0.0;
        continue;
      }
      for (int k = j; k < i; ++k) v -= a[i][k] * inv[k][j];
      inv[i][j] = v / a[i][i];
    }
  }
  __syncthreads();
  double* DI = J.DI + (size_t)(k0 / kCB) * kCB * kCB;
  double* DIT = J.DIT + (size_t)(k0 / kCB) * kCB * kCB;
  for (int t = tid; t < kCB * kCB; t += blockDim.x) {
    const int i = t % kCB, j = t / kCB;
    DI[i + j * kCB] = inv[i][j];
    DIT[i + j * kCB] = inv[j][i];
    if (i < b && j < b && i >= j) J.A[(k0 + i) + (size_t)(k0 + j) * J.ld] = a[i][j];
  }
}

// row-major copy of the panel L21 (rows k1..n-1, 64 columns) = column-major L21^T:
// out[c + r * 64] = A(k1 + r, k0 + c)
__global__ void k_panel_t(const CholDev* __restrict__ jobs, int k0, double* __restrict__ out, long long stride) {
  const CholDev J = jobs[blockIdx.y];
  const int k1 = k0 + kCB;
  if (k1 >= J.n) return;
  const int m = J.n - k1;
  double* o = out + blockIdx.y * stride;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * kCB;
       t += (long long)gridDim.x * blockDim.x) {
    const int c = int(t % kCB), r = int(t / kCB);
    o[c + (size_t)r * kCB] = J.A[(k1 + r) + (size_t)(k0 + c) * J.ld];
  }
}

__global__ void k_transpose_sq(int n, int ld, const double* __restrict__ in, double* __restrict__ out) {
  __shared__ double t[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int i = bx + threadIdx.x, j = by + k;
    if (i < n && j < n) t[k][threadIdx.x] = in[i + (size_t)j * ld];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int i = by + threadIdx.x, j = bx + k;
    if (i < n && j < n) out[i + (size_t)j * ld] = t[threadIdx.x][k];
  }
}

// out = (a + a^T) / 2 written over `out` from a (dense.cpp:68-75), full square
__global__ void k_symmetrize_into(int n, int ld, const double* __restrict__ a, double* __restrict__ out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)n * n) return;
  const int i = int(t % n), j = int(t / n);
  out[i + (size_t)j * ld] = 0.5 * (a[i + (size_t)j * ld] + a[j + (size_t)i * ld]);
}

__global__ void k_identity_ld(int n, int ld, double* __restrict__ M) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)n * ld) return;
  const int i = int(t % ld), j = int(t / ld);
  M[t] = (i == j && i < n) ? 1.0 : 0.0;
}

}  // namespace

// ---------------------------------------------------------------------------
void CholBatch::factor(Ctx& c, const std::vector<CholJob>& jobs_in) {
  jobs = jobs_in;
  const int J = int(jobs.size());
  nmax = 0;
  for (const auto& j : jobs) {
    nmax = std::max(nmax, j.n);
    if (j.ld % 4) c.fail(AWG_E_ARG, "cholesky: leading dimension must be a multiple of 4");
  }
  npan = (nmax + kCB - 1) / kCB;
  di.alloc(size_t(J) * std::max(npan, 1) * kCB * kCB);
  dit.alloc(size_t(J) * std::max(npan, 1) * kCB * kCB);
  info.alloc(std::max(J, 1));
  info.zero(c.stream);
  std::vector<CholDev> hd(J);
  for (int q = 0; q < J; ++q)
    hd[q] = CholDev{jobs[q].A, di.p + size_t(q) * npan * kCB * kCB, dit.p + size_t(q) * npan * kCB * kCB, info.p + q,
                    jobs[q].n, jobs[q].ld};
  DArr<CholDev> d;
  d.upload(hd, c.stream);
  DArr<double> pt;  // row-major panels (64 x m) per problem
  const long long pstride = (long long)kCB * nmax;
  pt.alloc(size_t(J) * pstride);
  for (int k0 = 0; k0 < nmax; k0 += kCB) {
    ensure_dyn_smem((const void*)k_potrf_diag, kDiagSmem);
    k_potrf_diag<<<J, 256, kDiagSmem, c.stream>>>(d.p, k0);
    ++c.launches;
    check_launch("potrf_diag");
    std::vector<GemmDesc> p1, p2;
    for (int q = 0; q < J; ++q) {
      const CholJob& s = jobs[q];
      const int k1 = k0 + kCB;
      if (k1 >= s.n) continue;
      const int m = s.n - k1;
      double* A21 = s.A + k1 + size_t(k0) * s.ld;
      // L21 = A21 L11^-T  (in place: every tile reads only its own rows)
      p1.push_back({A21, hd[q].DIT + size_t(k0 / kCB) * kCB * kCB, A21, m, kCB, kCB, s.ld, kCB, s.ld, 0, 0});
      // A22 -= L21 L21^T  (lower tiles)
      p2.push_back({A21, pt.p + size_t(q) * pstride, s.A + k1 + size_t(k1) * s.ld, m, m, kCB, s.ld, kCB, s.ld, 1, 1});
    }
    if (p1.empty()) continue;
    GroupedGemm g1, g2;
    g1.set(c, p1);
    g1.run(c);
    dim3 gt(64, J);
    k_panel_t<<<gt, 256, 0, c.stream>>>(d.p, k0, pt.p, pstride);
    ++c.launches;
    g2.set(c, p2);
    g2.run(c);
  }
  std::vector<int> hi = info.download(c.stream);
  for (int q = 0; q < J; ++q)
    if (hi[q] != 0)
      c.fail(AWG_E_NOT_SPD, "matrix not spd: non-positive pivot at index " + std::to_string(hi[q] - 1), hi[q] - 1);
}

// B <- L^-1 B (B: n x nrhs, ldb), right-looking block forward substitution
void CholBatch::solve_lower(Ctx& c, const std::vector<double*>& B, const std::vector<int>& ldb,
                            const std::vector<int>& nrhs) {
  const int J = int(jobs.size());
  for (int k0 = 0; k0 < nmax; k0 += kCB) {
    std::vector<GemmDesc> p1, p2;
    for (int q = 0; q < J; ++q) {
      const CholJob& s = jobs[q];
      if (k0 >= s.n || nrhs[q] == 0) continue;
      const int b = std::min(kCB, s.n - k0);
      double* Bk = B[q] + k0;
      // X_k = L_kk^-1 B_k (in place: a single 64-row tile)
      p1.push_back({di.p + (size_t(q) * npan + k0 / kCB) * kCB * kCB, Bk, Bk, b, nrhs[q], b, kCB, ldb[q], ldb[q], 0, 0});
      const int k1 = k0 + kCB;
      if (k1 < s.n)  // B(k1:, :) -= L(k1:, k0:k1) X_k
        p2.push_back({s.A + k1 + size_t(k0) * s.ld, Bk, B[q] + k1, s.n - k1, nrhs[q], kCB, s.ld, ldb[q], ldb[q], 1, 0});
    }
    if (p1.empty()) continue;
    GroupedGemm g1;
    g1.set(c, p1);
    g1.run(c);
    if (!p2.empty()) {
      GroupedGemm g2;
      g2.set(c, p2);
      g2.run(c);
    }
  }
}

// B <- L^-T B (B: n x nrhs, ldb), left-looking block back substitution
void CholBatch::solve_upper_t(Ctx& c, const std::vector<double*>& B, const std::vector<int>& ldb,
                              const std::vector<int>& nrhs) {
  const int J = int(jobs.size());
  for (int k0 = (npan - 1) * kCB; k0 >= 0; k0 -= kCB) {
    std::vector<GemmDesc> p1, p2;
    for (int q = 0; q < J; ++q) {
      const CholJob& s = jobs[q];
      if (k0 >= s.n || nrhs[q] == 0) continue;
      const int b = std::min(kCB, s.n - k0);
      double* Bk = B[q] + k0;
      const int k1 = k0 + kCB;
      if (k1 < s.n)  // B_k -= L(k1:, k0:k1)^T X(k1:, :)
        p1.push_back({s.A + k1 + size_t(k0) * s.ld, B[q] + k1, Bk, b, nrhs[q], s.n - k1, s.ld, ldb[q], ldb[q], 1, 0});
      // X_k = L_kk^-T B_k  (C = A^T B with A = L_kk^-1; in place, single tile)
      p2.push_back({di.p + (size_t(q) * npan + k0 / kCB) * kCB * kCB, Bk, Bk, b, nrhs[q], b, kCB, ldb[q], ldb[q], 0, 0});
    }
    if (p2.empty()) continue;
    if (!p1.empty()) {
      GroupedGemm g1;
      g1.set(c, p1, /*transpose_a=*/true);
      g1.run(c);
    }
    GroupedGemm g2;
    g2.set(c, p2, /*transpose_a=*/true);
    g2.run(c);
  }
}

// C = sym(L^-1 MA L^-T) over MA (dense.cpp:216-221), T: n x n scratch per problem
void CholBatch::reduce_pencil(Ctx& c, const std::vector<double*>& MA, const std::vector<double*>& T) {
  const int J = int(jobs.size());
  std::vector<int> ld(J), nr(J);
  for (int q = 0; q < J; ++q) {
    ld[q] = jobs[q].ld;
    nr[q] = jobs[q].n;
  }
  solve_lower(c, MA, ld, nr);  // Y = L^-1 MA
  for (int q = 0; q < J; ++q) {
    dim3 g((jobs[q].n + 31) / 32, (jobs[q].n + 31) / 32);
    k_transpose_sq<<<g, dim3(32, 8), 0, c.stream>>>(jobs[q].n, jobs[q].ld, MA[q], T[q]);
    ++c.launches;
  }
  solve_lower(c, T, ld, nr);  // L^-1 Y^T
  for (int q = 0; q < J; ++q) {
    const long long nn = (long long)jobs[q].n * jobs[q].n;
    k_symmetrize_into<<<int((nn + 255) / 256), 256, 0, c.stream>>>(jobs[q].n, jobs[q].ld, T[q], MA[q]);
    ++c.launches;
  }
  check_launch("reduce_pencil");
}

// U = L^-T (AS / AS+ local factors, stored upper triangular) into U (n x n, ld)
void CholBatch::inverse_transpose(Ctx& c, const std::vector<double*>& U, const std::vector<double*>& T) {
  const int J = int(jobs.size());
  std::vector<int> ld(J), nr(J);
  for (int q = 0; q < J; ++q) {
    ld[q] = jobs[q].ld;
    nr[q] = jobs[q].n;
    const long long cnt = (long long)jobs[q].n * jobs[q].ld;
    k_identity_ld<<<int((cnt + 255) / 256), 256, 0, c.stream>>>(jobs[q].n, jobs[q].ld, T[q]);
    ++c.launches;
  }
  solve_lower(c, T, ld, nr);  // L^-1
  for (int q = 0; q < J; ++q) {
    dim3 g((jobs[q].n + 31) / 32, (jobs[q].n + 31) / 32);
    k_transpose_sq<<<g, dim3(32, 8), 0, c.stream>>>(jobs[q].n, jobs[q].ld, T[q], U[q]);
    ++c.launches;
  }
  check_launch("inverse_transpose");
}

}  // namespace awgb
