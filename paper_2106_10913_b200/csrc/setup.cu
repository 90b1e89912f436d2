// GPU setup pipeline of the AWG preconditioner (ProblemContext + h2 +
// second_coarse, harness.cpp:100-124), everything on the device:
//
//   1. B^s = R^s (A ./ M_mu) R^s^T, dense per subdomain          splitting.cpp:37-62
//   2. eigendecomposition of every B^s (cuSOLVER syevd, several   splitting.cpp:88-90
//      streams), in place: the B^s buffer becomes V^s
//   3. classification eps_zero = 1e-12 max|l| n_s, snapping       splitting.cpp:64-84
//   4. NN pencils: MA = Ds^-1 (B^s + V-|L-|V-^T) Ds^-1 (DGEMM rank-q update),
//      MB = R^s A R^s^T + sum_t (shared rows of V-^t)|L-^t|(...)^T (one DGEMM over
//      the concatenated neighbour modes), generalized eigensolve (sygvd:
//      MB = L L^T reduction, Y^T MB Y = I)                        coarse.cpp:69-101, dense.cpp:211-224
//   5. selection (lambda < tau, or the fixed-k rule)              coarse.cpp:26-34
//   6. G = Z^T A+ Z, symmetrize, pivoted factor (reference or exact semantics,
//      cooperative multi-CTA kernel), l11^-1                       coarse.cpp:143-152, dense.cpp:299-346
//   7. W columns: one device PCG on A+ preconditioned by H2 per strictly negative
//      mode (same stopping rule), W^T A W, pivoted factor           preconditioner.cpp:84-128
//   8. INEX core (only in INEX mode)                               preconditioner.cpp:130-147
#include <cooperative_groups.h>
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <numeric>

#include "awg_internal.cuh"

namespace cg = cooperative_groups;

namespace awgb {
namespace {

#define AWG_SOLVER(x)                                                                  \
  do {                                                                                 \
    cusolverStatus_t st_ = (x);                                                        \
    if (st_ != CUSOLVER_STATUS_SUCCESS)                                                \
      throw AwgError(AWG_E_CUDA, std::string(#x) + ": cusolver status " + std::to_string(int(st_))); \
  } while (0)
#define AWG_BLAS(x)                                                                    \
  do {                                                                                 \
    cublasStatus_t st_ = (x);                                                          \
    if (st_ != CUBLAS_STATUS_SUCCESS)                                                  \
      throw AwgError(AWG_E_CUDA, std::string(#x) + ": cublas status " + std::to_string(int(st_))); \
  } while (0)

constexpr int kThreads = 256;

double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// progress trace on stderr with option verbose=1
void trace(const Ctx& c, const std::string& what, double ms) {
  if (c.opt("verbose", 0) == 1) std::fprintf(stderr, "[awg setup] %s: %.1f s\n", what.c_str(), ms / 1e3);
}

// --------------------------------------------------------------------------
// 1. dense local blocks from the CSR.  mode 0: B^s (A_ij / M_mu(ij)), mode 1: R A R^T.
__global__ void k_assemble(int s, int n, int ld, const long long* __restrict__ poff, const int* __restrict__ pidx,
                           const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ va,
                           const int* __restrict__ emult, int mode, double* __restrict__ M) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int* om = pidx + poff[s];
  const int i = om[k];
  for (int e = rp[i]; e < rp[i + 1]; ++e) {
    const int j = ci[e];
    int lo = 0, hi = n - 1, pos = -1;
    while (lo <= hi) {
      const int mid = (lo + hi) >> 1;
      const int v = om[mid];
      if (v == j) {
        pos = mid;
        break;
      }
      if (v < j) lo = mid + 1;
      else hi = mid - 1;
    }
    if (pos >= 0) M[k + (size_t)pos * ld] = mode == 0 ? va[e] / emult[e] : va[e];
  }
}

// 3. eigsplit classification (splitting.cpp:69-80), one warp per subdomain.
__global__ void k_classify(int N, const long long* __restrict__ poff, double* __restrict__ lam, int* __restrict__ m,
                           int* __restrict__ nz, double* __restrict__ eps_out) {
  const int s = blockIdx.x;
  if (s >= N) return;
  const long long p0 = poff[s];
  const int n = int(poff[s + 1] - p0);
  double mx = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) mx = fmax(mx, fabs(lam[p0 + k]));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (threadIdx.x == 0) {
    const double eps = 1e-12 * mx * n;
    int nonpos = 0, zero = 0;
    for (int k = 0; k < n; ++k) {
      if (lam[p0 + k] > eps) break;
      ++nonpos;
      if (fabs(lam[p0 + k]) <= eps) {
        lam[p0 + k] = 0.0;
        ++zero;
      }
    }
    m[s] = nonpos;
    nz[s] = zero;
    eps_out[s] = eps;
  }
}

// U(:, k) = w_k * V(:, k) for the first q columns (rank-q update operand)
__global__ void k_scale_cols(int n, int q, int ld, const double* __restrict__ V, const double* __restrict__ lam,
                             double* __restrict__ U) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (i >= n || k >= q) return;
  U[i + (size_t)k * ld] = (-lam[k]) * V[i + (size_t)k * ld];
}

// M(i,j) *= mu_j * mu_i, then symmetrize (coarse.cpp:86-94); thread per pair i >= j.
__global__ void k_weight_sym(int n, int ld, const int* __restrict__ om, const int* __restrict__ mult,
                             double* __restrict__ M) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)n * n) return;
  const int i = int(t % n), j = int(t / n);
  if (i < j) return;
  const double mi = double(mult[om[i]]), mj = double(mult[om[j]]);
  if (i == j) {
    M[i + (size_t)i * ld] *= mi * mi;
    return;
  }
  const double a = M[i + (size_t)j * ld] * (mj * mi);
  const double b = M[j + (size_t)i * ld] * (mi * mj);
  const double v = 0.5 * (a + b);
  M[i + (size_t)j * ld] = v;
  M[j + (size_t)i * ld] = v;
}

// Neighbour negative modes restricted to Omega^s (splitting.cpp:180-206):
// G(l, c) = V^t(pos_t(om_s[l]), k_c) or 0, and Gw(:, c) = w_c G(:, c).
__global__ void k_gather_neighbour_modes(int n, int ld, const int* __restrict__ om_s, int ncol,
                                         const int* __restrict__ col_t, const int* __restrict__ col_k,
                                         const double* __restrict__ col_w, const double* __restrict__ V,
                                         const long long* __restrict__ voff, const int* __restrict__ ns,
                                         const int* __restrict__ lds, const long long* __restrict__ poff,
                                         const int* __restrict__ pidx, double* __restrict__ G, double* __restrict__ Gw) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (l >= n || c >= ncol) return;
  const int t = col_t[c];
  const int g = om_s[l];
  const int* om_t = pidx + poff[t];
  int lo = 0, hi = ns[t] - 1, pos = -1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int v = om_t[mid];
    if (v == g) {
      pos = mid;
      break;
    }
    if (v < g) lo = mid + 1;
    else hi = mid - 1;
  }
  const double v = pos >= 0 ? V[voff[t] + pos + (size_t)col_k[c] * lds[t]] : 0.0;
  G[l + (size_t)c * ld] = v;
  Gw[l + (size_t)c * ld] = col_w[c] * v;
}

// 5. selection: lambda < tau (coarse.cpp:26-34) or the fixed-k rule.
__global__ void k_select(int N, const long long* __restrict__ poff, const double* __restrict__ plam,
                         const int* __restrict__ m, double tau, int fixed_k, int* __restrict__ ks) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= N) return;
  const long long p0 = poff[s];
  const int n = int(poff[s + 1] - p0);
  int k = 0;
  if (fixed_k > 0) {
    k = min(max(fixed_k, m[s]), n);
    while (k > 0 && k < n && fabs(plam[p0 + k] - plam[p0 + k - 1]) <= 1e-8) ++k;
  } else {
    while (k < n && plam[p0 + k] < tau) ++k;
  }
  ks[s] = k;
}

// z = R^s^T Y_s(:, c)  (coarse.cpp:140)
__global__ void k_scatter_col(int n, const int* __restrict__ om, const double* __restrict__ y, double* __restrict__ z) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l < n) z[om[l]] = y[l];
}

__global__ void k_symmetrize(int n, double* __restrict__ g) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)n * n) return;
  const int i = int(t % n), j = int(t / n);
  if (i <= j) return;
  const double v = 0.5 * (g[i + (size_t)j * n] + g[j + (size_t)i * n]);
  g[i + (size_t)j * n] = v;
  g[j + (size_t)i * n] = v;
}

// 6. Greedy pivoted Cholesky (dense.cpp:299-346) on the full n x n working
// matrix, one elimination step per pass with grid-wide barriers.
//   exact = 0: reference semantics — lower-triangle-only trailing update,
//              full row+column swap (swaps in the stale upper triangle);
//   exact = 1: the trailing update covers the full square (it stays exactly
//              symmetric), which equals refreshing the upper triangle first.
// The update is w(i,j) = fma(-w(j,r), w(i,r), w(i,j)): the reference build
// contracts `w(i,j) -= f * w(i,r)` into one fused multiply-add.
__global__ void k_rrf(int n, double* __restrict__ w, int* __restrict__ perm, int* __restrict__ rank_out,
                      double drop_tol, int exact) {
  cg::grid_group grid = cg::this_grid();
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n; i += nth) perm[i] = int(i);
  __shared__ int s_best;
  double first = 0.0;
  int r = 0;
  grid.sync();
  for (; r < n; ++r) {
    // every block finds the first maximum of the remaining diagonal
    if (threadIdx.x < 32) {
      double bv = -INFINITY;
      int bi = n;
      for (int k = r + threadIdx.x; k < n; k += 32) {
        const double d = w[k + (size_t)k * n];
        if (d > bv) {
          bv = d;
          bi = k;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (threadIdx.x == 0) s_best = bi;
    }
    __syncthreads();
    const int best = s_best;
    const double piv = w[best + (size_t)best * n];
    if (r == 0) first = piv;
    if (piv <= drop_tol * first || piv <= 0.0) break;
    grid.sync();  // all blocks have read the diagonal before it moves
    if (best != r) {
      for (long long k = tid; k < n; k += nth) {
        const double a = w[k + (size_t)r * n];
        w[k + (size_t)r * n] = w[k + (size_t)best * n];
        w[k + (size_t)best * n] = a;
      }
      if (tid == 0) {
        const int t = perm[r];
        perm[r] = perm[best];
        perm[best] = t;
      }
      grid.sync();
      for (long long k = tid; k < n; k += nth) {
        const double a = w[r + (size_t)k * n];
        w[r + (size_t)k * n] = w[best + (size_t)k * n];
        w[best + (size_t)k * n] = a;
      }
      grid.sync();
    }
    const double lkk = sqrt(w[r + (size_t)r * n]);
    const double inv = 1.0 / lkk;
    for (long long i = r + 1 + tid; i < n; i += nth) w[i + (size_t)r * n] *= inv;
    grid.sync();
    if (tid == 0) w[r + (size_t)r * n] = lkk;
    // trailing update: column j handled by one warp-group stripe
    const int m = n - r - 1;
    if (m > 0) {
      const long long total = exact ? (long long)m * m : (long long)m * (m + 1) / 2;
      if (exact) {
        for (long long t = tid; t < total; t += nth) {
          const int jj = int(t / m), ii = int(t % m);
          const int j = r + 1 + jj, i = r + 1 + ii;
          const double f = w[j + (size_t)r * n];
          w[i + (size_t)j * n] = fma(-f, w[i + (size_t)r * n], w[i + (size_t)j * n]);
        }
      } else {
        for (long long jj = blockIdx.x; jj < m; jj += gridDim.x) {
          const int j = r + 1 + int(jj);
          const double f = w[j + (size_t)r * n];
          for (int i = j + threadIdx.x; i < n; i += blockDim.x)
            w[i + (size_t)j * n] = fma(-f, w[i + (size_t)r * n], w[i + (size_t)j * n]);
        }
      }
    }
    grid.sync();
  }
  if (tid == 0) *rank_out = r;
}

__global__ void k_extract_l11(int n, int r, const double* __restrict__ w, double* __restrict__ l) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)r * r) return;
  const int i = int(t % r), j = int(t / r);
  l[t] = (i >= j) ? w[i + (size_t)j * n] : 0.0;
}

// --------------------------------------------------------------------------
struct Solvers {
  // concurrent eigensolves: syevd/sygvd of one subdomain leave most SMs idle
  // in their tridiagonalization phase, so several run side by side
  static constexpr int S = 8;
  cudaStream_t st[S] = {};
  cusolverDnHandle_t sol[S] = {};
  cublasHandle_t blas[S] = {};
  DArr<double> work[S];
  DArr<int> info;
  ~Solvers() {
    for (int i = 0; i < S; ++i) {
      if (sol[i]) cusolverDnDestroy(sol[i]);
      if (blas[i]) cublasDestroy(blas[i]);
      if (st[i]) cudaStreamDestroy(st[i]);
    }
  }
  void init(int nsub) {
    for (int i = 0; i < S; ++i) {
      AWG_CUDA(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
      AWG_SOLVER(cusolverDnCreate(&sol[i]));
      AWG_SOLVER(cusolverDnSetStream(sol[i], st[i]));
      AWG_BLAS(cublasCreate(&blas[i]));
      AWG_BLAS(cublasSetStream(blas[i], st[i]));
    }
    info.alloc(std::max(nsub, 1));
    info.zero(nullptr);
  }
  void sync() {
    for (int i = 0; i < S; ++i) AWG_CUDA(cudaStreamSynchronize(st[i]));
  }
};

void pivoted_factor(Ctx& c, DArr<double>& G, int n, int exact, CoarseFactor& f, int dim) {
  f.clear();
  f.dim = dim;
  if (n == 0) return;
  DArr<int> perm, rk;
  perm.alloc(n);
  rk.alloc(1);
  int threads = 256;
  int per_sm = 0;
  AWG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rrf, threads, 0));
  int blocks = std::max(1, std::min(per_sm, 2) * c.sm_count);
  const long long work = (long long)n * n / 2;
  blocks = int(std::max<long long>(1, std::min<long long>(blocks, (work + threads - 1) / threads)));
  double drop = 1e-10;
  double* wp = G.p;
  int* pp = perm.p;
  int* rp = rk.p;
  void* args[] = {&n, &wp, &pp, &rp, &drop, &exact};
  AWG_CUDA(cudaLaunchCooperativeKernel((void*)k_rrf, dim3(blocks), dim3(threads), args, 0, c.stream));
  ++c.launches;
  int r = 0;
  AWG_CUDA(cudaMemcpyAsync(&r, rk.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  AWG_CUDA(cudaStreamSynchronize(c.stream));
  f.rank = r;
  std::vector<int> hp(n);
  AWG_CUDA(cudaMemcpy(hp.data(), perm.p, sizeof(int) * n, cudaMemcpyDeviceToHost));
  f.h_retained.assign(hp.begin(), hp.begin() + r);
  f.retained.upload(f.h_retained, c.stream);
  DArr<double> l;
  l.alloc(size_t(std::max(r, 1)) * std::max(r, 1));
  if (r) {
    k_extract_l11<<<int(((long long)r * r + 255) / 256), 256, 0, c.stream>>>(n, r, G.p, l.p);
    ++c.launches;
    f.h_l11.resize(size_t(r) * r);
    AWG_CUDA(cudaMemcpyAsync(f.h_l11.data(), l.p, sizeof(double) * r * r, cudaMemcpyDeviceToHost, c.stream));
  }
  k::coarse_inverse(c, l.p, f);
  AWG_CUDA(cudaStreamSynchronize(c.stream));
}

__global__ void k_identity(int n, int ld, double* __restrict__ M) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)n * n) return;
  const int i = int(t % n), j = int(t / n);
  M[i + (size_t)j * ld] = (i == j) ? 1.0 : 0.0;
}

// Dense local blocks of subdomain s on stream q (scratch per stream):
//   a_block      R^s A R^s^T                                      splitting.cpp:161-173
//   aplus_block  R^s A R^s^T + neighbours' restricted V-|L-|V-^T  splitting.cpp:175-209
//   weighted     Ds^-1 (B^s + V-|L-|V-^T) Ds^-1, symmetrized       coarse.cpp:69-96
struct LocalBlocks {
  Ctx& c;
  Solvers& sv;
  std::vector<std::vector<int>> nb;  // neighbours (self included, ascending), splitting.cpp:96-104
  std::vector<int> q_of;             // strictly negative mode count per subdomain
  DArr<double> G1[Solvers::S], G2[Solvers::S];
  std::vector<DArr<int>> d_ct, d_ck;
  std::vector<DArr<double>> d_cw;

  LocalBlocks(Ctx& cc, Solvers& s) : c(cc), sv(s), d_ct(cc.N), d_ck(cc.N), d_cw(cc.N) {
    const int N = c.N;
    nb.assign(N, {});
    std::vector<std::vector<int>> subs(c.n);
    for (int t = 0; t < N; ++t)
      for (long long p = c.h_poff[t]; p < c.h_poff[t + 1]; ++p) subs[c.h_pidx[p]].push_back(t);
    std::vector<char> touch(size_t(N) * N, 0);
    for (int i = 0; i < c.n; ++i)
      for (int a : subs[i])
        for (int b : subs[i]) touch[size_t(a) * N + b] = 1;
    for (int a = 0; a < N; ++a)
      for (int b = 0; b < N; ++b)
        if (touch[size_t(a) * N + b]) nb[a].push_back(b);
    q_of.resize(N);
    for (int t = 0; t < N; ++t) q_of[t] = c.h_m[t] - c.h_nzero[t];
    int ldmax = 1, qn_max = 1;
    for (int t = 0; t < N; ++t) {
      ldmax = std::max(ldmax, c.h_ld[t]);
      int qn = 0;
      for (int u : nb[t]) qn += q_of[u];
      qn_max = std::max(qn_max, qn);
    }
    for (int i = 0; i < Solvers::S; ++i) {
      G1[i].alloc(size_t(ldmax) * qn_max);
      G2[i].alloc(size_t(ldmax) * qn_max);
    }
  }

  void a_block(int s, int q, double* M) {
    const int n = c.h_ns[s], ld = c.h_ld[s];
    AWG_CUDA(cudaMemsetAsync(M, 0, sizeof(double) * ld * n, sv.st[q]));
    k_assemble<<<(n + kThreads - 1) / kThreads, kThreads, 0, sv.st[q]>>>(s, n, ld, c.poff.p, c.pidx.p, c.rp.p,
                                                                          c.ci.p, c.va.p, c.emult.p, 1, M);
    ++c.launches;
  }

  void aplus_block(int s, int q, double* M) {
    a_block(s, q, M);
    const int n = c.h_ns[s], ld = c.h_ld[s];
    std::vector<int> ct, ck;
    std::vector<double> cw;
    for (int t : nb[s])
      for (int k = 0; k < q_of[t]; ++k) {
        ct.push_back(t);
        ck.push_back(k);
        cw.push_back(-c.h_lam[c.h_poff[t] + k]);
      }
    const int qn = int(ct.size());
    if (qn == 0) return;
    d_ct[s].upload(ct, sv.st[q]);
    d_ck[s].upload(ck, sv.st[q]);
    d_cw[s].upload(cw, sv.st[q]);
    dim3 g((n + kThreads - 1) / kThreads, qn);
    k_gather_neighbour_modes<<<g, kThreads, 0, sv.st[q]>>>(n, ld, c.pidx.p + c.h_poff[s], qn, d_ct[s].p, d_ck[s].p,
                                                            d_cw[s].p, c.V.p, c.voff.p, c.ns.p, c.ld.p, c.poff.p,
                                                            c.pidx.p, G1[q].p, G2[q].p);
    ++c.launches;
    const double one = 1.0;
    AWG_BLAS(cublasDgemm(sv.blas[q], CUBLAS_OP_N, CUBLAS_OP_T, n, n, qn, &one, G2[q].p, ld, G1[q].p, ld, &one, M, ld));
  }

  void weighted(int s, int q, double* M) {
    const int n = c.h_ns[s], ld = c.h_ld[s];
    AWG_CUDA(cudaMemsetAsync(M, 0, sizeof(double) * ld * n, sv.st[q]));
    k_assemble<<<(n + kThreads - 1) / kThreads, kThreads, 0, sv.st[q]>>>(s, n, ld, c.poff.p, c.pidx.p, c.rp.p,
                                                                          c.ci.p, c.va.p, c.emult.p, 0, M);
    ++c.launches;
    const int qs = q_of[s];
    const double* Vs = c.V.p + c.h_voff[s];
    if (qs > 0) {
      dim3 g((n + kThreads - 1) / kThreads, qs);
      k_scale_cols<<<g, kThreads, 0, sv.st[q]>>>(n, qs, ld, Vs, c.lam.p + c.h_poff[s], G1[q].p);
      ++c.launches;
      const double one = 1.0;
      AWG_BLAS(cublasDgemm(sv.blas[q], CUBLAS_OP_N, CUBLAS_OP_T, n, n, qs, &one, G1[q].p, ld, Vs, ld, &one, M, ld));
    }
    k_weight_sym<<<int(((long long)n * n + kThreads - 1) / kThreads), kThreads, 0, sv.st[q]>>>(
        n, ld, c.pidx.p + c.h_poff[s], c.mult.p, M);
    ++c.launches;
  }
};

// Subdomains grouped into waves whose per-problem workspace (bytes_of(s))
// fits in a share of the free device memory.
std::vector<std::vector<int>> waves_of(Ctx& c, const std::function<size_t(int)>& bytes_of, double share = 0.6) {
  size_t fr = 0, tot = 0;
  AWG_CUDA(cudaMemGetInfo(&fr, &tot));
  const size_t budget = size_t(double(fr) * share);
  std::vector<std::vector<int>> w(1);
  size_t used = 0;
  for (int s = 0; s < c.N; ++s) {
    const size_t b = bytes_of(s);
    if (!w.back().empty() && used + b > budget) {
      w.emplace_back();
      used = 0;
    }
    w.back().push_back(s);
    used += b;
  }
  return w;
}

// GenEO pencil (generalized_sym_eig, dense.cpp:211-224) of every subdomain in
// `wave`: MB = L L^T (hand-written batched Cholesky), C = sym(L^-1 MA L^-T),
// eigenvalues of C into plam (all n_s), eigenvectors of the `pick` smallest
// (MB-normalised: Y = L^-T Z) into Ycol[s].  MA and MB are destroyed.
void pencil_wave(Ctx& c, const std::vector<int>& wave, const std::vector<double*>& MA, const std::vector<double*>& MB,
                 const std::vector<double*>& T, double* plam, std::vector<DArr<double>>& Ycol, int cap,
                 const std::function<int(int, const double*)>& pick) {
  const int J = int(wave.size());
  std::vector<CholJob> cj(J);
  for (int q = 0; q < J; ++q) cj[q] = {MB[q], c.h_ns[wave[q]], c.h_ld[wave[q]]};
  CholBatch ch;
  ch.factor(c, cj);
  ch.reduce_pencil(c, MA, T);
  // eigenvectors of C land in T (free again), then Y = L^-T Z in place
  std::vector<SyevJob> ej(J);
  for (int q = 0; q < J; ++q) {
    const int s = wave[q];
    ej[q] = {MA[q], c.h_ns[s], c.h_ld[s], plam + c.h_poff[s], T[q], c.h_ld[s], std::min(cap, c.h_ns[s])};
  }
  std::vector<int> nv(J, 0);
  eig_batched(c, ej, [&](int q, const double* w) {
    nv[q] = std::min(pick(wave[q], w), ej[q].nvec);
    return nv[q];
  });
  std::vector<int> ldv(J);
  for (int q = 0; q < J; ++q) ldv[q] = c.h_ld[wave[q]];
  ch.solve_upper_t(c, T, ldv, nv);
  for (int q = 0; q < J; ++q) {
    const int s = wave[q];
    Ycol[s].alloc(size_t(c.h_ld[s]) * std::max(nv[q], 1));
    if (nv[q])
      AWG_CUDA(cudaMemcpyAsync(Ycol[s].p, T[q], sizeof(double) * c.h_ld[s] * nv[q], cudaMemcpyDeviceToDevice,
                               c.stream));
  }
  AWG_CUDA(cudaStreamSynchronize(c.stream));
}

// AS / AS+ one-level factors (OneLevel ctor, preconditioner.cpp:20-30):
// M^s = R A R^T (AS) or R A+ R^T (AS+), M^s = L L^T (cusolver potrf),
// U^s = L^-T (triangular solve against the identity), stored in c.U.
void local_cholesky(Ctx& c, Solvers& sv, LocalBlocks& lb) {
  const int N = c.N;
  c.U.alloc(size_t(c.h_voff[N]));
  c.U.zero(c.stream);
  AWG_CUDA(cudaStreamSynchronize(c.stream));
  if (c.opt("setup_cusolver", 0) == 0) {
    // M^s = L L^T (batched, chol.cu), U^s = L^-T
    auto waves = waves_of(c, [&](int s) { return size_t(2) * c.h_ld[s] * c.h_ns[s] * 8; });
    for (const auto& wave : waves) {
      std::vector<DArr<double>> M(wave.size()), T(wave.size());
      std::vector<CholJob> cj;
      std::vector<double*> U, Tp;
      for (size_t q = 0; q < wave.size(); ++q) {
        const int s = wave[q];
        M[q].alloc(size_t(c.h_ld[s]) * c.h_ns[s]);
        T[q].alloc(size_t(c.h_ld[s]) * c.h_ns[s]);
        const int st = int(q % Solvers::S);
        if (c.one_level == 0) lb.a_block(s, st, M[q].p);
        else lb.aplus_block(s, st, M[q].p);
        cj.push_back({M[q].p, c.h_ns[s], c.h_ld[s]});
        U.push_back(c.U.p + c.h_voff[s]);
        Tp.push_back(T[q].p);
      }
      sv.sync();
      CholBatch ch;
      ch.factor(c, cj);
      ch.inverse_transpose(c, U, Tp);
      AWG_CUDA(cudaStreamSynchronize(c.stream));
    }
    return;
  }
  size_t blk_max = 1;
  int lw_max = 1;
  for (int s = 0; s < N; ++s) {
    blk_max = std::max(blk_max, size_t(c.h_ld[s]) * c.h_ns[s]);
    int lw = 0;
    AWG_SOLVER(cusolverDnDpotrf_bufferSize(sv.sol[0], CUBLAS_FILL_MODE_LOWER, c.h_ns[s], nullptr, c.h_ld[s], &lw));
    lw_max = std::max(lw_max, lw);
  }
  std::vector<DArr<double>> T(Solvers::S);
  for (int i = 0; i < Solvers::S; ++i) {
    T[i].alloc(blk_max);
    sv.work[i].alloc(size_t(lw_max) + 1);
  }
  sv.info.zero(nullptr);
  AWG_CUDA(cudaDeviceSynchronize());
  for (int s = 0; s < N; ++s) {
    const int q = s % Solvers::S;
    const int n = c.h_ns[s], ld = c.h_ld[s];
    if (c.one_level == 0) lb.a_block(s, q, T[q].p);
    else lb.aplus_block(s, q, T[q].p);
    AWG_SOLVER(cusolverDnDpotrf(sv.sol[q], CUBLAS_FILL_MODE_LOWER, n, T[q].p, ld, sv.work[q].p, lw_max,
                                sv.info.p + s));
    double* Us = c.U.p + c.h_voff[s];
    k_identity<<<int(((long long)n * n + kThreads - 1) / kThreads), kThreads, 0, sv.st[q]>>>(n, ld, Us);
    ++c.launches;
    const double one = 1.0;
    AWG_BLAS(cublasDtrsm(sv.blas[q], CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, n, n,
                         &one, T[q].p, ld, Us, ld));
  }
  sv.sync();
  std::vector<int> info(N);
  AWG_CUDA(cudaMemcpy(info.data(), sv.info.p, sizeof(int) * N, cudaMemcpyDeviceToHost));
  for (int s = 0; s < N; ++s)
    if (info[s] > 0)
      c.fail(AWG_E_NOT_SPD, "matrix not spd: non-positive pivot at index " + std::to_string(info[s] - 1),
             info[s] - 1);
}
}  // namespace

void build_local_cholesky(Ctx& c) {
  Solvers sv;
  sv.init(c.N);
  LocalBlocks lb(c, sv);
  local_cholesky(c, sv, lb);
}

// G = W^T A W (preconditioner.cpp:119-126): A W in blocks of columns (one SpMV
// per column), then W^T (A W) as a grouped C = A^T B on the FP64 tensor cores
// (dgemm.cu), split over the n rows so the nm x 512 output still fills every
// SM; the split partials are summed in slice order.
__global__ void k_sum_slices(int S, long long len, const double* __restrict__ part, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len; i += (long long)gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int s = 0; s < S; ++s) a += part[(size_t)s * len + i];
    out[i] = a;
  }
}

static void wtaw(Ctx& c, int nm, double* G) {
  const int Bc = std::min(nm, 512);
  DArr<double> aw;
  aw.alloc(size_t(c.ldw) * Bc);
  aw.zero(c.stream);  // padding rows of each column stay zero
  const int tiles = ((nm + 127) / 128) * ((Bc + 63) / 64);
  int S = std::max(1, std::min(32, (8 * c.sm_count + tiles - 1) / tiles));
  const int kslice = round_up((c.n + S - 1) / S, 16);
  S = (c.n + kslice - 1) / kslice;
  DArr<double> part;
  part.alloc(size_t(S) * nm * Bc);
  GroupedGemm g;
  for (int j0 = 0; j0 < nm; j0 += Bc) {
    const int bc = std::min(Bc, nm - j0);
    for (int j = 0; j < bc; ++j)
      k::spmv(c, c.W.p + size_t(j0 + j) * c.ldw, aw.p + size_t(j) * c.ldw, 0, nullptr, nullptr, nullptr);
    std::vector<GemmDesc> pd;
    for (int sl = 0; sl < S; ++sl) {
      const int k0 = sl * kslice, kl = std::min(kslice, c.n - k0);
      pd.push_back({c.W.p + k0, aw.p + k0, part.p + size_t(sl) * nm * bc, nm, bc, kl, c.ldw, c.ldw, nm});
    }
    g.set(c, pd, /*transpose_a=*/true);
    g.run(c);
    const long long len = (long long)nm * bc;
    k_sum_slices<<<int(std::min<long long>((len + kThreads - 1) / kThreads, 4096)), kThreads, 0, c.stream>>>(
        S, len, part.p, G + size_t(j0) * nm);
    ++c.launches;
    check_launch("wtaw");
  }
}

void run_setup(Ctx& c, const awg_config& cfg) {
  const double t_start = now_ms();
  const int N = c.N;
  c.cfg = cfg;
  c.lu_semantics = cfg.lu_semantics;
  c.have_factors = false;
  c.invalidate_graphs();
  Solvers sv;
  sv.init(N);

  // ---- layout ---------------------------------------------------------------
  c.h_ld.resize(N);
  c.h_voff.assign(N + 1, 0);
  for (int s = 0; s < N; ++s) {
    c.h_ld[s] = round_up(c.h_ns[s], 4);
    c.h_voff[s + 1] = c.h_voff[s] + (long long)c.h_ld[s] * c.h_ns[s];
  }
  c.ns.upload(c.h_ns, c.stream);
  c.ld.upload(c.h_ld, c.stream);
  c.voff.upload(c.h_voff, c.stream);
  c.V.alloc(size_t(c.h_voff[N]));
  c.V.zero(c.stream);
  c.lam.alloc(c.P);
  AWG_CUDA(cudaStreamSynchronize(c.stream));

  // ---- 1+2. B^s and its eigendecomposition ------------------------------------
  double t0 = now_ms();
  if (c.opt("setup_cusolver", 0) == 0) {
    // hand-written batched eigensolver (eig.cu): B^s assembled in place in V^s,
    // eigenvectors through a workspace, copied back over the reflectors
    for (int s = 0; s < N; ++s) {
      const int n = c.h_ns[s];
      k_assemble<<<(n + kThreads - 1) / kThreads, kThreads, 0, c.stream>>>(
          s, n, c.h_ld[s], c.poff.p, c.pidx.p, c.rp.p, c.ci.p, c.va.p, c.emult.p, 0, c.V.p + c.h_voff[s]);
      ++c.launches;
    }
    auto waves = waves_of(c, [&](int s) { return size_t(c.h_ld[s]) * c.h_ns[s] * 8 + (size_t(4) << 20); });
    for (const auto& wave : waves) {
      long long zt = 0;
      for (int s : wave) zt += (long long)c.h_ld[s] * c.h_ns[s];
      DArr<double> Z;
      Z.alloc(size_t(zt));
      std::vector<SyevJob> jobs;
      long long zo = 0;
      for (int s : wave) {
        jobs.push_back({c.V.p + c.h_voff[s], c.h_ns[s], c.h_ld[s], c.lam.p + c.h_poff[s], Z.p + zo, c.h_ld[s], c.h_ns[s]});
        zo += (long long)c.h_ld[s] * c.h_ns[s];
      }
      eig_batched(c, jobs, nullptr);
      AWG_CUDA(cudaMemcpyAsync(c.V.p + c.h_voff[wave.front()], Z.p, sizeof(double) * zt, cudaMemcpyDeviceToDevice,
                               c.stream));  // the wave's blocks are contiguous in V, in the same layout
      AWG_CUDA(cudaStreamSynchronize(c.stream));
    }
  } else {
    int lwork_max = 0;
    int nmax = 0;
    for (int s = 0; s < N; ++s) nmax = std::max(nmax, c.h_ns[s]);
    for (int s = 0; s < N; ++s) {
      int lw = 0;
      AWG_SOLVER(cusolverDnDsyevd_bufferSize(sv.sol[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, c.h_ns[s],
                                             c.V.p + c.h_voff[s], c.h_ld[s], c.lam.p + c.h_poff[s], &lw));
      lwork_max = std::max(lwork_max, lw);
    }
    for (int i = 0; i < Solvers::S; ++i) sv.work[i].alloc(size_t(lwork_max) + 1);
    for (int s = 0; s < N; ++s) {
      const int q = s % Solvers::S;
      const int n = c.h_ns[s];
      k_assemble<<<(n + kThreads - 1) / kThreads, kThreads, 0, sv.st[q]>>>(
          s, n, c.h_ld[s], c.poff.p, c.pidx.p, c.rp.p, c.ci.p, c.va.p, c.emult.p, 0, c.V.p + c.h_voff[s]);
      ++c.launches;
      AWG_SOLVER(cusolverDnDsyevd(sv.sol[q], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n,
                                  c.V.p + c.h_voff[s], c.h_ld[s], c.lam.p + c.h_poff[s], sv.work[q].p, lwork_max,
                                  sv.info.p + s));
    }
    sv.sync();
    std::vector<int> info(N);
    AWG_CUDA(cudaMemcpy(info.data(), sv.info.p, sizeof(int) * N, cudaMemcpyDeviceToHost));
    for (int s = 0; s < N; ++s)
      if (info[s] != 0)
        c.fail(AWG_E_NO_CONVERGENCE, "dense_sym_eig: eigensolver failed on subdomain " + std::to_string(s));
  }
  // ---- 3. classification ------------------------------------------------------------
  {
    DArr<int> m, nz;
    DArr<double> eps;
    m.alloc(N);
    nz.alloc(N);
    eps.alloc(N);
    k_classify<<<N, 32, 0, c.stream>>>(N, c.poff.p, c.lam.p, m.p, nz.p, eps.p);
    ++c.launches;
    c.h_m = m.download(c.stream);
    c.h_nzero = nz.download(c.stream);
    c.h_eps = eps.download(c.stream);
    c.h_lam = c.lam.download(c.stream);
    c.msz.upload(c.h_m, c.stream);
  }
  c.t_setup_ms[0] = now_ms() - t0;
  trace(c, "splitting (B^s + eig)", c.t_setup_ms[0]);

  // ---- 4. pencils + 5. selection (coarse.cpp:98-130) --------------------------------
  // NN / AS+: pencil_nn = (weighted A+^s, R A+ R^T); AS: pencil_as1 = (weighted A+^s,
  // R A R^T) below 1/tau_flat and pencil_as2 = (R A R^T, R A+ R^T) below tau_sharp.
  t0 = now_ms();
  c.one_level = cfg.one_level;
  std::vector<int> ks(N, 0);
  LocalBlocks lb(c, sv);
  if (cfg.use_coarse) {
    const bool as = (cfg.one_level == 0);
    int lw_max = 1;
    size_t blk_max = 1;
    for (int s = 0; s < N; ++s) blk_max = std::max(blk_max, size_t(c.h_ld[s]) * c.h_ns[s]);
    if (c.opt("setup_cusolver", 0) != 0) {  // workspace of the library path only
      for (int s = 0; s < N; ++s) {
        int lw = 0;
        AWG_SOLVER(cusolverDnDsygvd_bufferSize(sv.sol[0], CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                                               CUBLAS_FILL_MODE_LOWER, c.h_ns[s], nullptr, c.h_ld[s], nullptr,
                                               c.h_ld[s], nullptr, &lw));
        lw_max = std::max(lw_max, lw);
      }
    }
    DArr<double> plam, plam2;
    plam.alloc(c.P);
    if (as) plam2.alloc(c.P);
    std::vector<DArr<double>> Ycol(N), Ycol2(N);
    if (c.opt("setup_cusolver", 0) == 0) {
      // how many GenEO vectors each pencil needs (the selection rule of k_select)
      auto count_rule = [&](double tau, int fixed_k) {
        return [&, tau, fixed_k](int s, const double* w) {
          const int n = c.h_ns[s];
          int k = 0;
          if (fixed_k > 0) {
            k = std::min(std::max(fixed_k, c.h_m[s]), n);
            while (k > 0 && k < n && std::fabs(w[k] - w[k - 1]) <= 1e-8) ++k;
          } else {
            while (k < n && w[k] < tau) ++k;
          }
          return k;
        };
      };
      const int cap = 512;
      const int nb = as ? 5 : 3;
      auto waves = waves_of(c, [&](int s) {
        return size_t(nb) * c.h_ld[s] * c.h_ns[s] * 8 + size_t(c.h_ld[s]) * cap * 8 + (size_t(8) << 20);
      });
      for (const auto& wave : waves) {
        const int J = int(wave.size());
        double tw = now_ms();
        std::vector<DArr<double>> B(size_t(J) * nb);
        std::vector<double*> MA(J), MB(J), T(J), AB(J), AB2(J);
        for (int q = 0; q < J; ++q) {
          const int s = wave[q];
          const size_t blk = size_t(c.h_ld[s]) * c.h_ns[s];
          for (int b = 0; b < nb; ++b) B[size_t(q) * nb + b].alloc(blk);
          MA[q] = B[size_t(q) * nb].p;
          MB[q] = B[size_t(q) * nb + 1].p;
          T[q] = B[size_t(q) * nb + 2].p;
          const int st = q % Solvers::S;
          lb.weighted(s, st, MA[q]);
          lb.aplus_block(s, st, MB[q]);
          if (as) {
            AB[q] = B[size_t(q) * nb + 3].p;
            AB2[q] = B[size_t(q) * nb + 4].p;
            lb.a_block(s, st, AB[q]);
            AWG_CUDA(cudaMemcpyAsync(AB2[q], AB[q], sizeof(double) * blk, cudaMemcpyDeviceToDevice, sv.st[st]));
          }
        }
        sv.sync();
        trace(c, "  pencil blocks of " + std::to_string(J) + " subdomains (weighted A+^s, R A+ R^T)", now_ms() - tw);
        tw = now_ms();
        if (!as) {
          const double tau = cfg.one_level == 1 ? 1.0 / cfg.tau_flat : cfg.tau_sharp;
          pencil_wave(c, wave, MA, MB, T, plam.p, Ycol, cap, count_rule(tau, cfg.fixed_k));
        } else {
          // pencil_as1 = (weighted A+^s, R A R^T) below 1/tau_flat; pencil_as2 = (R A R^T, R A+ R^T) below tau_sharp
          pencil_wave(c, wave, MA, AB, T, plam.p, Ycol, cap, count_rule(1.0 / cfg.tau_flat, 0));
          pencil_wave(c, wave, AB2, MB, T, plam2.p, Ycol2, cap, count_rule(cfg.tau_sharp, 0));
        }
        AWG_CUDA(cudaStreamSynchronize(c.stream));
        trace(c, "  pencil reduction + eigensolve + back substitution", now_ms() - tw);
      }
    } else {
    const int nbuf = as ? 4 : 2;
    std::vector<DArr<double>> buf(Solvers::S * nbuf);
    for (int i = 0; i < Solvers::S; ++i) {
      sv.work[i].alloc(size_t(lw_max) + 1);
      for (int b = 0; b < nbuf; ++b) buf[i * nbuf + b].alloc(blk_max);
    }
    DArr<int> info2;
    info2.alloc(N);
    info2.zero(nullptr);
    sv.info.zero(nullptr);
    AWG_CUDA(cudaDeviceSynchronize());
    for (int s = 0; s < N; ++s) {
      const int q = s % Solvers::S;
      cudaStream_t st = sv.st[q];
      const int n = c.h_ns[s], ld = c.h_ld[s];
      double* MA = buf[q * nbuf].p;
      double* MB = buf[q * nbuf + 1].p;
      lb.weighted(s, q, MA);
      int keep = n;
      if (cfg.fixed_k > 0) keep = std::min(n, std::max(cfg.fixed_k, c.h_m[s]) + 64);
      if (!as) {
        lb.aplus_block(s, q, MB);
        AWG_SOLVER(cusolverDnDsygvd(sv.sol[q], CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                    n, MA, ld, MB, ld, plam.p + c.h_poff[s], sv.work[q].p, lw_max, sv.info.p + s));
        Ycol[s].alloc(size_t(ld) * keep);
        AWG_CUDA(cudaMemcpyAsync(Ycol[s].p, MA, sizeof(double) * ld * keep, cudaMemcpyDeviceToDevice, st));
      } else {
        double* AB = buf[q * nbuf + 2].p;
        double* AB2 = buf[q * nbuf + 3].p;
        lb.aplus_block(s, q, MB);
        lb.a_block(s, q, AB);
        AWG_CUDA(cudaMemcpyAsync(AB2, AB, sizeof(double) * ld * n, cudaMemcpyDeviceToDevice, st));
        AWG_SOLVER(cusolverDnDsygvd(sv.sol[q], CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                    n, MA, ld, AB, ld, plam.p + c.h_poff[s], sv.work[q].p, lw_max, sv.info.p + s));
        AWG_SOLVER(cusolverDnDsygvd(sv.sol[q], CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                    n, AB2, ld, MB, ld, plam2.p + c.h_poff[s], sv.work[q].p, lw_max,
                                    info2.p + s));
        Ycol[s].alloc(size_t(ld) * n);
        Ycol2[s].alloc(size_t(ld) * n);
        AWG_CUDA(cudaMemcpyAsync(Ycol[s].p, MA, sizeof(double) * ld * n, cudaMemcpyDeviceToDevice, st));
        AWG_CUDA(cudaMemcpyAsync(Ycol2[s].p, AB2, sizeof(double) * ld * n, cudaMemcpyDeviceToDevice, st));
      }
    }
    sv.sync();
    std::vector<int> info(N), i2(N);
    AWG_CUDA(cudaMemcpy(info.data(), sv.info.p, sizeof(int) * N, cudaMemcpyDeviceToHost));
    AWG_CUDA(cudaMemcpy(i2.data(), info2.p, sizeof(int) * N, cudaMemcpyDeviceToHost));
    for (int s = 0; s < N; ++s)
      for (int v : {info[s], i2[s]}) {
        if (v > c.h_ns[s])
          c.fail(AWG_E_NOT_SPD, "matrix not spd: non-positive pivot at index " + std::to_string(v - c.h_ns[s] - 1),
                 v - c.h_ns[s] - 1);
        if (v != 0) c.fail(AWG_E_NO_CONVERGENCE, "generalized_sym_eig: eigensolver failed");
      }
    }  // cuSOLVER path (option setup_cusolver=1)
    DArr<int> dks, dks2;
    dks.alloc(N);
    if (!as) {
      const double tau = cfg.one_level == 1 ? 1.0 / cfg.tau_flat : cfg.tau_sharp;
      k_select<<<(N + 127) / 128, 128, 0, c.stream>>>(N, c.poff.p, plam.p, c.msz.p, tau, cfg.fixed_k, dks.p);
      ++c.launches;
      ks = dks.download(c.stream);
      c.h_plam = plam.download(c.stream);
    } else {
      dks2.alloc(N);
      k_select<<<(N + 127) / 128, 128, 0, c.stream>>>(N, c.poff.p, plam.p, c.msz.p, 1.0 / cfg.tau_flat, 0, dks.p);
      k_select<<<(N + 127) / 128, 128, 0, c.stream>>>(N, c.poff.p, plam2.p, c.msz.p, cfg.tau_sharp, 0, dks2.p);
      c.launches += 2;
      std::vector<int> m1 = dks.download(c.stream), m2 = dks2.download(c.stream);
      for (int s = 0; s < N; ++s) ks[s] = m1[s] + m2[s];
      c.h_plam = plam.download(c.stream);
      c.h_plam2 = plam2.download(c.stream);
      c.h_ks_as1 = m1;
    }
    c.h_ks = ks;
    // coarse layout, task lists, A- modes, work buffers
    finalize_factors(c);
    c.Y.alloc(size_t(std::max<long long>(c.h_yoff[N], 1)));
    for (int s = 0; s < N; ++s) {
      if (ks[s] == 0) continue;
      const size_t ld = c.h_ld[s];
      if (!as) {
        if (Ycol[s].n < ld * ks[s]) c.fail(AWG_E_STATE, "setup: selected GenEO modes beyond the kept eigenvectors");
        AWG_CUDA(cudaMemcpyAsync(c.Y.p + c.h_yoff[s], Ycol[s].p, sizeof(double) * ld * ks[s], cudaMemcpyDeviceToDevice,
                                 c.stream));
      } else {  // [as1 low modes, as2 low modes] (coarse.cpp:127-130 push order)
        const int m1 = c.h_ks_as1[s], m2 = ks[s] - m1;
        if (m1)
          AWG_CUDA(cudaMemcpyAsync(c.Y.p + c.h_yoff[s], Ycol[s].p, sizeof(double) * ld * m1, cudaMemcpyDeviceToDevice,
                                   c.stream));
        if (m2)
          AWG_CUDA(cudaMemcpyAsync(c.Y.p + c.h_yoff[s] + ld * m1, Ycol2[s].p, sizeof(double) * ld * m2,
                                   cudaMemcpyDeviceToDevice, c.stream));
      }
    }
    AWG_CUDA(cudaStreamSynchronize(c.stream));
  } else {
    c.h_ks = ks;
    finalize_factors(c);
    c.Y.alloc(1);
  }
  if (cfg.one_level != 2) local_cholesky(c, sv, lb);
  AWG_CUDA(cudaStreamSynchronize(c.stream));
  c.t_setup_ms[1] = now_ms() - t0;
  trace(c, "pencils + selection (n0 = " + std::to_string(c.n0) + ")", c.t_setup_ms[1]);

  // ---- 6. coarse operator G = Z^T A+ Z and its pivoted factor ---------------------------
  t0 = now_ms();
  c.k0.clear();
  c.nm = 0;  // H2 only while building the coarse spaces
  if (c.n0 > 0) {
    DArr<double> G, z, az;
    G.alloc(size_t(c.n0) * c.n0);
    z.alloc(c.n);
    az.alloc(c.n);
    int col = 0;
    for (int s = 0; s < N; ++s)
      for (int k = 0; k < ks[s]; ++k, ++col) {
        AWG_CUDA(cudaMemsetAsync(z.p, 0, sizeof(double) * c.n, c.stream));
        k_scatter_col<<<(c.h_ns[s] + kThreads - 1) / kThreads, kThreads, 0, c.stream>>>(
            c.h_ns[s], c.pidx.p + c.h_poff[s], c.Y.p + c.h_yoff[s] + size_t(k) * c.h_ld[s], z.p);
        ++c.launches;
        op_apply(c, AWG_OP_APLUS, z.p, az.p, nullptr);
        k::zT(c, az.p, G.p + size_t(col) * c.n0, nullptr);
      }
    k_symmetrize<<<int(((long long)c.n0 * c.n0 + kThreads - 1) / kThreads), kThreads, 0, c.stream>>>(c.n0, G.p);
    ++c.launches;
    pivoted_factor(c, G, c.n0, cfg.rrf_semantics, c.k0, c.n0);
    k::build_coarse_neg(c);  // A- dots of the coarse columns for the hybrid H2 (apply path only)
    k::build_az(c);          // A Z on ring-extended supports (post-solve half of the hybrid H2)
  }
  c.t_setup_ms[2] = now_ms() - t0;
  trace(c, "coarse operator + pivoted factor (r0 = " + std::to_string(c.k0.rank) + ")", c.t_setup_ms[2]);

  // ---- 7. second coarse space W (preconditioner.cpp:84-128) ------------------------------
  t0 = now_ms();
  c.h_w_inner.clear();
  c.h_neg_weights.clear();
  int nm = 0;
  if (cfg.awg_mode != 0) {
    for (int s = 0; s < N; ++s) nm += c.h_m[s] - c.h_nzero[s];
  }
  c.ldw = round_up(c.n, 4);
  c.kw.clear();
  if (nm > 0) {
    c.W.alloc(size_t(c.ldw) * nm);
    c.W.zero(c.stream);
    std::vector<std::pair<int, int>> modes;
    for (int s = 0; s < N; ++s)
      for (int k = 0; k < c.h_m[s]; ++k) {
        const double lam = c.h_lam[c.h_poff[s] + k];
        if (lam == 0.0) continue;  // kernel columns of B^s are dropped (preconditioner.cpp:103)
        modes.push_back({s, k});
        c.h_neg_weights.push_back(-lam);
      }
    cublasHandle_t hb = nullptr;
    AWG_BLAS(cublasCreate(&hb));
    c.w_batches = 0;
    const long long maxit = (long long)std::max(1, cfg.w_maxit_factor) * c.n;
    try {
      build_w_batched(c, hb, modes, int(std::min<long long>(maxit, 1 << 30)), cfg.w_rtol, c.h_w_inner, 512);
    } catch (...) {
      cublasDestroy(hb);
      throw;
    }
    cublasDestroy(hb);
    const int col = int(modes.size());
    (void)col;
    c.neg_weights.upload(c.h_neg_weights, c.stream);
    c.t_setup_ms[3] = now_ms() - t0;
    trace(c, "W inner PCGs (n_minus = " + std::to_string(nm) + ")", c.t_setup_ms[3]);
    // W^T A W (preconditioner.cpp:119-126)
    t0 = now_ms();
    c.nm = nm;
    c.alloc_work();  // W-sized work buffers
    DArr<double> G;
    G.alloc(size_t(nm) * nm);
    wtaw(c, nm, G.p);
    k_symmetrize<<<int(((long long)nm * nm + kThreads - 1) / kThreads), kThreads, 0, c.stream>>>(nm, G.p);
    ++c.launches;
    pivoted_factor(c, G, nm, cfg.rrf_semantics, c.kw, nm);
    if (cfg.awg_mode == 3) build_core(c);
    c.t_setup_ms[4] = now_ms() - t0;
  }
  c.nm = nm;
  c.alloc_work();
  AWG_CUDA(cudaStreamSynchronize(c.stream));
  c.t_setup_ms[5] = now_ms() - t_start;
}

// The device pivoted factor on a caller-supplied symmetric G (n x n,
// column-major, host memory): the k_rrf run of build_coarse / build_w,
// exposed for direct retained-set parity checks (awg_pivoted_factor).
void pivoted_factor_of(Ctx& c, int n, const double* G_host, int exact, CoarseFactor& f) {
  DArr<double> G;
  G.alloc(size_t(std::max(n, 1)) * std::max(n, 1));
  if (n > 0) {
    AWG_CUDA(cudaMemcpyAsync(G.p, G_host, sizeof(double) * size_t(n) * n, cudaMemcpyHostToDevice, c.stream));
  }
  pivoted_factor(c, G, n, exact, f, n);
}

}  // namespace awgb
