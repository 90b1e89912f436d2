// Batched construction of the second coarse space W (build_w,
// preconditioner.cpp:84-128).
//
// The reference runs one PCG per strictly negative mode, sequentially:
//   W(:, col) = pcg(A+, H2, R^s^T v_k, w_rtol, 10 n)          (:99-116)
// Here B columns run at once as B independent PCGs: every column keeps its own
// alpha, beta, rho, iteration count and stopping decision (the same recursive +
// true residual rule, krylov.cpp:93-102), so per-column semantics are the
// reference's; only the operators are applied to the n x B block at once.  The
// one-level NN solve of a block is two DGEMMs per subdomain (V^s^T X_s and
// V^s U_s, FP64 tensor-core tiles via cuBLAS), so the V^s stream is amortized
// over B right-hand sides.
#include <cublas_v2.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <string>

#include "awg_internal.cuh"

namespace awgb {
namespace {

#define AWG_BLAS(x)                                                                                  \
  do {                                                                                               \
    cublasStatus_t st_ = (x);                                                                        \
    if (st_ != CUBLAS_STATUS_SUCCESS)                                                                \
      throw AwgError(AWG_E_CUDA, std::string(#x) + ": cublas status " + std::to_string(int(st_)));   \
  } while (0)

constexpr int kT = 256;

struct ColState {
  double bnorm, rz, pq, alpha, beta, relres, alpha_prev, beta_prev, true_rel;
  int it, done, converged, past_rtol, need_true, error, fresh, pad1;
  // fresh: the slot was refilled with a new column (R = b, bnorm set); its next
  // loop pass is that column's PCG initialisation (alpha = 0, then z = H r, p = z)
};

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ bool col_off(const int* done, int b) { return done != nullptr && done[b] != 0; }

// Y(:,b) = A X(:,b) (+ epilogues as k_spmv): mode 0 plain, 1 add + AX, 2 sub - (add + AX), 3 sub - AX
__global__ void kb_spmv(int n, int ld, const int* __restrict__ rp, const int* __restrict__ ci,
                        const double* __restrict__ va, const double* __restrict__ X, double* __restrict__ Y, int mode,
                        const double* __restrict__ add, const double* __restrict__ sub, const int* __restrict__ done) {
  const int b = blockIdx.y;
  if (col_off(done, b)) return;
  const size_t o = (size_t)b * ld;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double acc = 0.0;
    acc = csr_row(ci, va, rp[i], rp[i + 1], [&](int j) { return __ldg(X + o + j); });
    double out;
    if (mode == 0) out = acc;
    else if (mode == 1) out = add[o + i] + acc;
    else if (mode == 2) out = sub[o + i] - (add[o + i] + acc);
    else out = sub[o + i] - acc;
    Y[o + i] = out;
  }
}

// block-P layout: subdomain s, column b at boff[s] + b * ld_s
__global__ void kb_gather(long long P, const int* __restrict__ psub, const long long* __restrict__ poff,
                          const int* __restrict__ pidx, const int* __restrict__ lds,
                          const long long* __restrict__ boff, const double* __restrict__ ds, int ldx,
                          const double* __restrict__ X, double* __restrict__ XS, const int* __restrict__ done) {
  const int b = blockIdx.y;
  if (col_off(done, b)) return;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < P; p += (long long)gridDim.x * blockDim.x) {
    const int s = psub[p];
    const int i = int(p - poff[s]);
    double v = X[(size_t)b * ldx + pidx[p]];
    if (ds) v *= ds[p];
    XS[boff[s] + (size_t)b * lds[s] + i] = v;
  }
}

// U(j, b) = 0 for j < n_nonpos(s), U(j, b) / lambda_j otherwise
__global__ void kb_mask(long long P, const int* __restrict__ psub, const long long* __restrict__ poff,
                        const int* __restrict__ lds, const long long* __restrict__ boff, const int* __restrict__ msz,
                        const double* __restrict__ lam, int B, double* __restrict__ U) {
  const int b = blockIdx.y;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < P; p += (long long)gridDim.x * blockDim.x) {
    const int s = psub[p];
    const int j = int(p - poff[s]);
    double* u = U + boff[s] + (size_t)b * lds[s] + j;
    *u = (j < msz[s]) ? 0.0 : *u / lam[p];
  }
}

// Column-blocked forms: thread per (row i, kBB columns of the block), so the
// CSR row / owner entries are read once for kBB columns (they were re-read per
// column from L2: 512 x the CSR arrays per block SpMV).  Per column the
// arithmetic is exactly kb_spmv's / kb_prolong's.
constexpr int kBB = 8;
struct BEnt {  // owner entry q of dof i in the block-P layout: WS(s, loc, b) = WS[base + b * ld]
  long long base;
  int ld, p;
};
__global__ void kb_build_bent(long long P, const int* __restrict__ own_pos, const int* __restrict__ psub,
                              const long long* __restrict__ poff, const int* __restrict__ lds,
                              const long long* __restrict__ boff, BEnt* __restrict__ ent) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < P; q += (long long)gridDim.x * blockDim.x) {
    const int p = own_pos[q];
    const int s = psub[p];
    ent[q] = BEnt{boff[s] + (p - poff[s]), lds[s], p};
  }
}

__device__ __forceinline__ unsigned live_mask(const int* done, int b0, int B) {
  unsigned m = 0;
#pragma unroll
  for (int u = 0; u < kBB; ++u)
    if (b0 + u < B && !col_off(done, b0 + u)) m |= 1u << u;
  return m;
}

__global__ void kb_spmv8(int n, int B, int ld, const int* __restrict__ rp, const int* __restrict__ ci,
                         const double* __restrict__ va, const double* __restrict__ X, double* __restrict__ Y, int mode,
                         const double* __restrict__ add, const double* __restrict__ sub, const int* __restrict__ done) {
  const int b0 = blockIdx.y * kBB;
  const unsigned live = live_mask(done, b0, B);
  if (!live) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double acc[kBB];
#pragma unroll
    for (int u = 0; u < kBB; ++u) acc[u] = 0.0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const double v = va[k];
      const size_t j = ci[k];
#pragma unroll
      for (int u = 0; u < kBB; ++u)
        if (live >> u & 1u) acc[u] = __dadd_rn(acc[u], __dmul_rn(v, __ldg(X + (size_t)(b0 + u) * ld + j)));
    }
#pragma unroll
    for (int u = 0; u < kBB; ++u) {
      if (!(live >> u & 1u)) continue;
      const size_t o = (size_t)(b0 + u) * ld + i;
      double out;
      if (mode == 0) out = acc[u];
      else if (mode == 1) out = add[o] + acc[u];
      else if (mode == 2) out = sub[o] - (add[o] + acc[u]);
      else out = sub[o] - acc[u];
      Y[o] = out;
    }
  }
}

__global__ void kb_prolong8(int n, int B, int ldx, const int* __restrict__ own_off, const BEnt* __restrict__ ent,
                            const double* __restrict__ ds, const double* __restrict__ WS, double* __restrict__ Y,
                            const int* __restrict__ done) {
  const int b0 = blockIdx.y * kBB;
  const unsigned live = live_mask(done, b0, B);
  if (!live) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double acc[kBB];
#pragma unroll
    for (int u = 0; u < kBB; ++u) acc[u] = 0.0;
    for (int q = own_off[i]; q < own_off[i + 1]; ++q) {
      const BEnt e = ent[q];
      const double d = ds ? ds[e.p] : 1.0;
#pragma unroll
      for (int u = 0; u < kBB; ++u) {
        if (!(live >> u & 1u)) continue;
        double w = WS[e.base + (size_t)(b0 + u) * e.ld];
        if (ds) w *= d;
        acc[u] += w;
      }
    }
#pragma unroll
    for (int u = 0; u < kBB; ++u)
      if (live >> u & 1u) Y[(size_t)(b0 + u) * ldx + i] = acc[u];
  }
}

// T(:, j) = V(:, j) / lambda_j  (columns j >= n_nonpos, shifted to start at 0)
__global__ void kb_scale_inv(int n, int ld, const double* __restrict__ V, const double* __restrict__ lam,
                             double* __restrict__ T) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (i < ld) T[i + (size_t)j * ld] = (i < n) ? V[i + (size_t)j * ld] / lam[j] : 0.0;
}

// C(j, b) *= w_j  (the -lambda weights of the negative modes)
__global__ void kb_scale_rows(int m, const double* __restrict__ w, double* __restrict__ C) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < m) C[(size_t)blockIdx.y * m + j] *= w[j];
}

__global__ void kb_take(int r, int n0, int B, const int* __restrict__ ret, const double* __restrict__ src,
                        double* __restrict__ dst) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)r * B) return;
  const int k = int(t % r), b = int(t / r);
  dst[t] = src[(size_t)b * n0 + ret[k]];
}

__global__ void kb_put(int r, int n0, int B, const int* __restrict__ ret, const double* __restrict__ src,
                       double* __restrict__ dst) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)r * B) return;
  const int k = int(t % r), b = int(t / r);
  dst[(size_t)b * n0 + ret[k]] = src[t];
}

// Y = (A - Bm) + D | A + Bm | A - Bm, column-gated
__global__ void kb_axpby(int n, int ld, const double* __restrict__ a, const double* __restrict__ bm,
                         const double* __restrict__ d, double* __restrict__ y, int mode, const int* __restrict__ done) {
  const int b = blockIdx.y;
  if (col_off(done, b)) return;
  const size_t o = (size_t)b * ld;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double v;
    if (mode == 0) v = (a[o + i] - bm[o + i]) + d[o + i];
    else if (mode == 1) v = a[o + i] + bm[o + i];
    else v = a[o + i] - bm[o + i];
    y[o + i] = v;
  }
}

// per-column partial dot products: part[b * G + g]
__global__ void kb_dot(int n, int ld, const double* __restrict__ x, const double* __restrict__ y,
                       double* __restrict__ part, int mode, const double* __restrict__ bm) {
  // mode 0: <x, y>;  mode 1: ||bm - y||^2 (true residual);  x unused in mode 1
  __shared__ double sred[32];
  const int b = blockIdx.y;
  const size_t o = (size_t)b * ld;
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (mode == 0) acc = fma(x[o + i], y[o + i], acc);
    else {
      const double d = bm[o + i] - y[o + i];
      acc = fma(d, d, acc);
    }
  }
  acc = wsum(acc);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sred[w];
    part[(size_t)b * gridDim.x + blockIdx.x] = s;
  }
}

__device__ double sum_parts(const double* part, int G, int b) {
  double s = 0.0;
  for (int g = 0; g < G; ++g) s += part[(size_t)b * G + g];
  return s;
}

// ---- per-column PCG scalar steps (the k_pcg_* logic of ops.cu, per column) --------
// slots the host refilled (fresh[b]): ||b|| from the block dot, state reset
__global__ void kc_fresh(int B, ColState* st, const double* part, int G, int* done, const int* fresh) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B || !fresh[b]) return;
  ColState c{};
  const double s = sum_parts(part, G, b);
  c.bnorm = sqrt(s);
  c.done = (s == 0.0);
  c.converged = (s == 0.0);
  c.fresh = !c.done;
  st[b] = c;
  done[b] = c.done;
}

__global__ void kc_clear(int B, ColState* st, int* done) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  ColState c{};
  c.done = 1;
  st[b] = c;
  done[b] = 1;
}

__global__ void kc_rz(int B, ColState* st, const double* part, int G, int* done, int initial) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  ColState& c = st[b];
  if (c.done) return;
  const double rz = sum_parts(part, G, b);
  if (initial || c.fresh) {
    if (rz <= 0.0) {
      c.error = PCG_BAD_PRECOND;
      c.done = 1;
    }
    c.rz = rz;
    c.beta = 0.0;
    c.fresh = 0;
  } else if (rz <= 0.0) {
    if (!c.past_rtol) c.error = PCG_BAD_PRECOND;
    c.done = 1;
  } else {
    const double beta = rz / c.rz;
    c.beta = beta;
    c.rz = rz;
    c.beta_prev = beta;
    c.alpha_prev = c.alpha;
  }
  done[b] = c.done;
}

__global__ void kc_alpha(int B, ColState* st, const double* part, int G, int* done) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  ColState& c = st[b];
  if (c.done) return;
  if (c.fresh) {  // initialisation pass: x and r stay as set
    c.alpha = 0.0;
    return;
  }
  const double pq = sum_parts(part, G, b);
  c.pq = pq;
  if (pq <= 0.0) {
    if (!c.past_rtol) c.error = PCG_BAD_OPERATOR;
    c.done = 1;
  } else {
    c.alpha = c.rz / pq;
  }
  done[b] = c.done;
}

// X += alpha P; R -= alpha Q (gated per column); partial ||R||^2
__global__ void kb_update(int n, int ld, const ColState* st, double* __restrict__ X, double* __restrict__ R,
                          const double* __restrict__ P, const double* __restrict__ Q, double* __restrict__ part) {
  __shared__ double sred[32];
  const int b = blockIdx.y;
  const size_t o = (size_t)b * ld;
  const bool active = !st[b].done;
  const double alpha = st[b].alpha;
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double ri = R[o + i];
    if (active) {
      X[o + i] = fma(alpha, P[o + i], X[o + i]);
      ri = fma(-alpha, Q[o + i], ri);
      R[o + i] = ri;
    }
    acc = fma(ri, ri, acc);
  }
  acc = wsum(acc);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sred[w];
    part[(size_t)b * gridDim.x + blockIdx.x] = s;
  }
}

__global__ void kc_relres(int B, ColState* st, const double* part, int G, double rtol, int maxit, int* done,
                          int* any_true) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  ColState& c = st[b];
  if (c.done || c.fresh) {
    c.need_true = 0;
    return;
  }
  const double relres = sqrt(sum_parts(part, G, b)) / c.bnorm;
  c.it += 1;
  c.relres = relres;
  c.need_true = (relres <= rtol);
  if (c.need_true) {
    c.past_rtol = 1;
    atomicOr(any_true, 1);
  }
  if (!c.need_true && c.it == maxit) c.done = 1;
  done[b] = c.done;
}

__global__ void kc_true(int B, ColState* st, const double* part, int G, double rtol, int maxit, int* done) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  ColState& c = st[b];
  if (c.done || !c.need_true) return;
  const double tr = sqrt(sum_parts(part, G, b)) / c.bnorm;
  c.true_rel = tr;
  if (tr <= rtol || fabs(tr - c.relres) <= 1e-8) {
    c.converged = 1;
    c.done = 1;
  } else if (c.it == maxit) {
    c.done = 1;
  }
  done[b] = c.done;
}

__global__ void kb_p(int n, int ld, const ColState* st, const double* __restrict__ Z, double* __restrict__ P,
                     int initial) {
  const int b = blockIdx.y;
  if (st[b].done) return;
  const double beta = st[b].beta;
  const size_t o = (size_t)b * ld;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    P[o + i] = initial ? Z[o + i] : fma(beta, P[o + i], Z[o + i]);
}

// ---------------------------------------------------------------------------
struct Block {
  int B = 0, ld = 0, G = 0;
  DArr<double> X, R, Z, Pm, Q, Bm, T, C0, C1, C2, C3, C4, C5;
  DArr<double> XS, WS;  // block-P layout
  DArr<double> Pinv;    // optional P^s = V+ L+^-1 V+^T (NN), V layout
  GroupedGemm pgemm;    // P^s X^s over all subdomains (empty: per-subdomain cuBLAS, option wbuild_cublas=1)
  DArr<double> zx, zr, zt, zc, negc, part;
  DArr<ColState> st;
  DArr<int> done, any_true;
  DArr<long long> boff;
  std::vector<long long> h_boff;
  DArr<BEnt> bent;  // owner entries in the block-P layout (kb_prolong8)
};

// Per-subdomain products of one block operation as ONE cuBLAS grouped-batched
// DGEMM call (one group per subdomain): the per-call overhead of N separate
// DGEMMs dominated these skinny products (q_s or k_s <= ~50 columns).
struct GroupedCall {
  std::vector<cublasOperation_t> ta, tb;
  std::vector<int> m, n, k, lda, ldb, ldc, gs;
  std::vector<double> al, be;
  std::vector<const double*> ha, hb;
  std::vector<double*> hc;
  DArr<const double*> A, B;
  DArr<double*> C;
  void add(cublasOperation_t opa, int mm, int nn, int kk, const double* a, int la, const double* b, int lb, double* cc,
           int lc) {
    ta.push_back(opa);
    tb.push_back(CUBLAS_OP_N);
    m.push_back(mm);
    n.push_back(nn);
    k.push_back(kk);
    lda.push_back(la);
    ldb.push_back(lb);
    ldc.push_back(lc);
    gs.push_back(1);
    al.push_back(1.0);
    be.push_back(0.0);
    ha.push_back(a);
    hb.push_back(b);
    hc.push_back(cc);
  }
  void upload(cudaStream_t st) {
    A.upload(ha, st);
    B.upload(hb, st);
    C.upload(hc, st);
  }
  void run(cublasHandle_t h) const {
    if (m.empty()) return;
    AWG_BLAS(cublasDgemmGroupedBatched(h, ta.data(), tb.data(), m.data(), n.data(), k.data(), al.data(), A.p,
                                       lda.data(), B.p, ldb.data(), be.data(), C.p, ldc.data(), int(m.size()),
                                       gs.data()));
  }
};

struct BlockOps {
  Ctx& c;
  Block& k;
  cublasHandle_t h;
  const CoarseFactor& k0;
  std::vector<int> qs, negoff, koff;  // per subdomain: negative modes, their offset, coarse column offset
  // phase profile of one block pass (option verbose=2): events between phases
  std::vector<std::pair<std::string, cudaEvent_t>> marks;
  bool prof = false;
  void mark(const char* name) {
    if (!prof) return;
    cudaEvent_t e;
    AWG_CUDA(cudaEventCreate(&e));
    AWG_CUDA(cudaEventRecord(e, c.stream));
    marks.push_back({name, e});
  }
  void report() {
    if (marks.size() < 2) return;
    AWG_CUDA(cudaEventSynchronize(marks.back().second));
    std::string line = "[awg setup]   W pass profile (ms):";
    for (size_t i = 1; i < marks.size(); ++i) {
      float ms = 0.f;
      AWG_CUDA(cudaEventElapsedTime(&ms, marks[i - 1].second, marks[i].second));
      line += " " + marks[i].first + "=" + std::to_string(ms);
    }
    std::fprintf(stderr, "%s\n", line.c_str());
    for (auto& m : marks) cudaEventDestroy(m.second);
    marks.clear();
    prof = false;
  }

  GroupedCall g_negdot, g_negcomb, g_zdot, g_zcomb;  // V-^T XS, V- C, Y^T XS, Y C over all subdomains
  bool any_q0 = false, any_k0 = false;              // subdomains without negative modes / coarse columns
  BlockOps(Ctx& cc, Block& kk, cublasHandle_t hh, const CoarseFactor& f) : c(cc), k(kk), h(hh), k0(f) {
    qs.resize(c.N);
    negoff.assign(c.N + 1, 0);
    koff.assign(c.N + 1, 0);
    for (int s = 0; s < c.N; ++s) {
      qs[s] = c.h_m[s] - c.h_nzero[s];
      negoff[s + 1] = negoff[s] + qs[s];
      koff[s + 1] = koff[s] + c.h_ks[s];
    }
    const int B = k.B, n0 = c.n0;
    for (int s = 0; s < c.N; ++s) {
      const int ns = c.h_ns[s], L = c.h_ld[s];
      double* xs = k.XS.p + k.h_boff[s];
      double* ws = k.WS.p + k.h_boff[s];
      if (qs[s] > 0) {
        const double* v = c.V.p + c.h_voff[s];
        g_negdot.add(CUBLAS_OP_T, qs[s], B, ns, v, L, xs, L, k.negc.p + negoff[s], c.nneg);
        g_negcomb.add(CUBLAS_OP_N, ns, B, qs[s], v, L, k.negc.p + negoff[s], c.nneg, ws, L);
      }
      if (c.h_ks[s] > 0) {
        const double* y = c.Y.p + c.h_yoff[s];
        g_zdot.add(CUBLAS_OP_T, c.h_ks[s], B, ns, y, L, xs, L, k.zx.p + koff[s], n0);
        g_zcomb.add(CUBLAS_OP_N, ns, B, c.h_ks[s], y, L, k.zc.p + koff[s], n0, ws, L);
      }
    }
    for (int s = 0; s < c.N; ++s) {
      any_q0 |= qs[s] == 0;
      any_k0 |= c.h_ks[s] == 0;
    }
    for (GroupedCall* g : {&g_negdot, &g_negcomb, &g_zdot, &g_zcomb}) g->upload(c.stream);
  }

  dim3 grid_n() const { return dim3(std::max(1, std::min((c.n + kT - 1) / kT, 148 * 2)), k.B); }
  dim3 grid_bb() const {
    return dim3(std::max(1, std::min((c.n + kT - 1) / kT, 148 * 2)), (k.B + kBB - 1) / kBB);
  }
  void prolong(const double* ds, const double* WS, double* Y, const int* done) {
    kb_prolong8<<<grid_bb(), kT, 0, c.stream>>>(c.n, k.B, k.ld, c.own_off.p, k.bent.p, ds, WS, Y, done);
    ++c.launches;
  }
  dim3 grid_p() const {
    return dim3(std::max(1, int(std::min<long long>((c.P + kT - 1) / kT, 148 * 2))), k.B);
  }

  void spmv(const double* X, double* Y, int mode, const double* add, const double* sub, const int* done) {
    kb_spmv8<<<grid_bb(), kT, 0, c.stream>>>(c.n, k.B, k.ld, c.rp.p, c.ci.p, c.va.p, X, Y, mode, add, sub, done);
    ++c.launches;
  }
  // A- X = sum_s R^s^T V-^s |L-^s| V-^s^T R^s X: the strictly negative modes of s are
  // the first q_s columns of V^s (ascending spectrum, splitting.cpp:129-137), so both
  // products are per-subdomain DGEMMs on the gathered block (V-^s read once per batch)
  void aminus(const double* X, double* Y, const int* done) {
    if (c.nneg == 0) {
      AWG_CUDA(cudaMemsetAsync(Y, 0, sizeof(double) * k.ld * k.B, c.stream));
      return;
    }
    kb_gather<<<grid_p(), kT, 0, c.stream>>>(c.P, c.psub.p, c.poff.p, c.pidx.p, c.ld.p, k.boff.p, nullptr, k.ld, X,
                                             k.XS.p, done);
    mark("am.gather");
    // WS is rewritten (beta = 0) on every row the prolongation reads, except
    // for subdomains without negative modes: zero it only then
    if (any_q0) AWG_CUDA(cudaMemsetAsync(k.WS.p, 0, sizeof(double) * k.WS.n, c.stream));
    mark("am.memset");
    g_negdot.run(h);  // V-^s^T R^s X, every subdomain
    mark("am.dots");
    kb_scale_rows<<<dim3((c.nneg + kT - 1) / kT, k.B), kT, 0, c.stream>>>(c.nneg, c.neg_w.p, k.negc.p);
    g_negcomb.run(h);  // V-^s C_s
    mark("am.comb");
    prolong(nullptr, k.WS.p, Y, done);
    mark("am.prolong");
    c.launches += 3;
  }
  void aplus(const double* X, double* Y, const int* done) {
    aminus(X, Y, done);
    spmv(X, Y, 1, Y, nullptr, done);
  }
  // coarse_correct on the block: Z^T X and Z C as per-subdomain DGEMMs with Y_s
  void q(const double* X, double* Y, const int* done) {
    const int n0 = c.n0, r = k0.rank, B = k.B;
    kb_gather<<<grid_p(), kT, 0, c.stream>>>(c.P, c.psub.p, c.poff.p, c.pidx.p, c.ld.p, k.boff.p, nullptr, k.ld, X,
                                             k.XS.p, done);
    ++c.launches;
    g_zdot.run(h);  // Y_s^T R^s X
    AWG_CUDA(cudaMemsetAsync(k.zc.p, 0, sizeof(double) * n0 * B, c.stream));
    if (r > 0) {
      kb_take<<<int(((long long)r * B + kT - 1) / kT), kT, 0, c.stream>>>(r, n0, B, k0.retained.p, k.zx.p, k.zr.p);
      const double one = 1.0, zero = 0.0;
      // t = L^-1 b_r, y = L^-T t  (rank_revealing_solve, dense.cpp:348-366)
      AWG_BLAS(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, r, B, r, &one, k0.linv.p, r, k.zr.p, r, &zero, k.zt.p, r));
      AWG_BLAS(cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, r, B, r, &one, k0.linv.p, r, k.zt.p, r, &zero, k.zr.p, r));
      kb_put<<<int(((long long)r * B + kT - 1) / kT), kT, 0, c.stream>>>(r, n0, B, k0.retained.p, k.zr.p, k.zc.p);
      c.launches += 2;
    }
    if (any_k0) AWG_CUDA(cudaMemsetAsync(k.WS.p, 0, sizeof(double) * k.WS.n, c.stream));
    g_zcomb.run(h);  // Y_s C_s
    prolong(nullptr, k.WS.p, Y, done);
    c.launches += 3;
  }
  // OneLevel::apply on the block: NN = R^T D V mask(1/lam) V^T D R, AS/AS+ =
  // R^T U U^T R with U = L^-T (triangular products as DTRMM)
  void h1(const double* X, double* Y, const int* done) {
    const bool nn = (c.one_level == 2);
    kb_gather<<<grid_p(), kT, 0, c.stream>>>(c.P, c.psub.p, c.poff.p, c.pidx.p, c.ld.p, k.boff.p,
                                             nn ? c.ds.p : nullptr, k.ld, X, k.XS.p, done);
    const double one = 1.0, zero = 0.0;
    if (nn && k.Pinv.p) {  // P^s X^s for every subdomain, P^s = V+ L+^-1 V+^T
      if (k.pgemm.ntiles) {
        k.pgemm.run(c);  // one grouped FP64 tensor-core launch (dgemm.cu)
      } else {
        for (int s = 0; s < c.N; ++s) {
          const int n = c.h_ns[s], L = c.h_ld[s];
          AWG_BLAS(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, k.B, n, &one, k.Pinv.p + c.h_voff[s], L,
                               k.XS.p + k.h_boff[s], L, &zero, k.WS.p + k.h_boff[s], L));
        }
      }
      prolong(c.ds.p, k.WS.p, Y, done);
      c.launches += 2;
      return;
    }
    for (int s = 0; s < c.N; ++s) {
      const int n = c.h_ns[s], L = c.h_ld[s];
      if (nn) {
        AWG_BLAS(cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, n, k.B, n, &one, c.V.p + c.h_voff[s], L,
                             k.XS.p + k.h_boff[s], L, &zero, k.WS.p + k.h_boff[s], L));
      } else {
        AWG_BLAS(cublasDtrmm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, n, k.B,
                             &one, c.U.p + c.h_voff[s], L, k.XS.p + k.h_boff[s], L, k.WS.p + k.h_boff[s], L));
      }
    }
    if (nn)
      kb_mask<<<grid_p(), kT, 0, c.stream>>>(c.P, c.psub.p, c.poff.p, c.ld.p, k.boff.p, c.msz.p, c.lam.p, k.B,
                                             k.WS.p);
    for (int s = 0; s < c.N; ++s) {
      const int n = c.h_ns[s], L = c.h_ld[s];
      if (nn) {
        AWG_BLAS(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, k.B, n, &one, c.V.p + c.h_voff[s], L,
                             k.WS.p + k.h_boff[s], L, &zero, k.XS.p + k.h_boff[s], L));
      } else {
        AWG_BLAS(cublasDtrmm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, k.B,
                             &one, c.U.p + c.h_voff[s], L, k.WS.p + k.h_boff[s], L, k.XS.p + k.h_boff[s], L));
      }
    }
    prolong(nn ? c.ds.p : nullptr, k.XS.p, Y, done);
    c.launches += nn ? 3 : 2;
  }
  // TwoLevel::apply (preconditioner.cpp:64-82)
  void h2(const double* X, double* Y, const int* done) {
    if (c.n0 == 0) {
      h1(X, Y, done);
      return;
    }
    q(X, k.C0.p, done);
    mark("h2.q");
    if (c.cfg.composition == 0) {
      h1(X, k.C1.p, done);
      axpby(k.C1.p, k.C0.p, nullptr, Y, 1, done);
      return;
    }
    aminus(k.C0.p, k.C1.p, done);
    spmv(k.C0.p, k.C2.p, 2, k.C1.p, X, done);
    mark("h2.aplus");
    h1(k.C2.p, k.C3.p, done);
    mark("h2.h1");
    aplus(k.C3.p, k.C4.p, done);
    mark("h2.aplus2");
    q(k.C4.p, k.C5.p, done);
    mark("h2.q2");
    axpby(k.C3.p, k.C5.p, k.C0.p, Y, 0, done);
    mark("h2.axpby");
  }
  void axpby(const double* a, const double* b, const double* d, double* y, int mode, const int* done) {
    kb_axpby<<<grid_n(), kT, 0, c.stream>>>(c.n, k.ld, a, b, d, y, mode, done);
    ++c.launches;
  }
  void dot(const double* x, const double* y, int mode, const double* bm) {
    kb_dot<<<dim3(k.G, k.B), kT, 0, c.stream>>>(c.n, k.ld, x, y, k.part.p, mode, bm);
    ++c.launches;
  }
};

}  // namespace

// Solve A+ W(:, j) = R^s^T v_k for the given columns (block of rhs already in
// k.Bm), H2 preconditioned; returns per-column iteration counts.
void build_w_batched(Ctx& c, cublasHandle_t h, const std::vector<std::pair<int, int>>& modes, int maxit,
                     double rtol, std::vector<int>& iters, int max_block) {
  const int total = int(modes.size());
  iters.assign(total, 0);
  if (total == 0) return;
  size_t free_b = 0, tot_b = 0;
  AWG_CUDA(cudaMemGetInfo(&free_b, &tot_b));
  // bytes per batched column: 13 n-blocks, 2 restricted blocks, coarse and mode scratch
  const size_t per_col =
      sizeof(double) * (size_t(c.ldw) * 13 + size_t(c.P + 4 * c.N) * 2 + size_t(c.n0) * 4 + c.nneg + 256);
  Block k;
  // NN: precompute P^s = V+^s (L+^s)^-1 V+^s^T when it fits next to a block of
  // >= 256 columns — halves the DGEMM work of every block one-level solve
  const size_t pinv_bytes = sizeof(double) * size_t(c.h_voff[c.N]);
  if (c.one_level == 2 && free_b > pinv_bytes + 256 * per_col * 10 / 7 + (size_t(2) << 30)) {
    k.Pinv.alloc(size_t(c.h_voff[c.N]));
    size_t tmax = 1;
    for (int s = 0; s < c.N; ++s) tmax = std::max(tmax, size_t(c.h_ld[s]) * c.h_ns[s]);
    DArr<double> T;
    T.alloc(tmax);
    AWG_BLAS(cublasSetStream(h, c.stream));
    const double one = 1.0, zero = 0.0;
    for (int s = 0; s < c.N; ++s) {
      const int n = c.h_ns[s], L = c.h_ld[s], m = c.h_m[s];
      const double* Vs = c.V.p + c.h_voff[s];
      if (n - m > 0) {
        kb_scale_inv<<<dim3((n + kT - 1) / kT, n - m), kT, 0, c.stream>>>(n, L, Vs + size_t(m) * L,
                                                                          c.lam.p + c.h_poff[s] + m, T.p);
        AWG_BLAS(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, n, n, n - m, &one, T.p, L, Vs + size_t(m) * L, L, &zero,
                             k.Pinv.p + c.h_voff[s], L));
        ++c.launches;
      } else {
        AWG_CUDA(cudaMemsetAsync(k.Pinv.p + c.h_voff[s], 0, sizeof(double) * L * n, c.stream));
      }
    }
    AWG_CUDA(cudaStreamSynchronize(c.stream));
    AWG_CUDA(cudaMemGetInfo(&free_b, &tot_b));
  }
  int B = int(std::min<size_t>(size_t(max_block), (free_b * 7 / 10) / std::max<size_t>(per_col, 1)));
  B = std::max(1, std::min(B, total));
  // whole 64-column tiles of the grouped GEMM (c5: memory allows 416 columns =
  // 6.5 tiles, i.e. 7 tiles of DMMA work per 6.5 of columns; 384 run 5% faster)
  if (B >= 128 && B < total) B = B / 64 * 64;
  k.B = B;
  k.ld = c.ldw;
  k.G = std::max(1, std::min((c.n + kT - 1) / kT, 148));
  for (DArr<double>* m : {&k.X, &k.R, &k.Z, &k.Pm, &k.Q, &k.Bm, &k.T, &k.C0, &k.C1, &k.C2, &k.C3, &k.C4, &k.C5})
    m->alloc(size_t(k.ld) * B);
  k.h_boff.assign(c.N + 1, 0);
  for (int s = 0; s < c.N; ++s) k.h_boff[s + 1] = k.h_boff[s] + (long long)c.h_ld[s] * B;
  k.boff.upload(k.h_boff, c.stream);
  k.bent.alloc(size_t(std::max<long long>(c.P, 1)));
  kb_build_bent<<<int(std::min<long long>((c.P + kT - 1) / kT, 4096)), kT, 0, c.stream>>>(
      c.P, c.own_pos.p, c.psub.p, c.poff.p, c.ld.p, k.boff.p, k.bent.p);
  k.XS.alloc(size_t(k.h_boff[c.N]));
  k.WS.alloc(size_t(k.h_boff[c.N]));
  k.XS.zero(c.stream);
  k.WS.zero(c.stream);
  k.zx.alloc(size_t(std::max(c.n0, 1)) * B);
  k.zc.alloc(size_t(std::max(c.n0, 1)) * B);
  k.zr.alloc(size_t(std::max(c.k0.rank, 1)) * B);
  k.zt.alloc(size_t(std::max(c.k0.rank, 1)) * B);
  k.negc.alloc(size_t(std::max(c.nneg, 1)) * B);
  k.part.alloc(size_t(k.G) * B);
  k.st.alloc(B);
  k.done.alloc(B);
  k.any_true.alloc(1);
  AWG_BLAS(cublasSetStream(h, c.stream));
  if (k.Pinv.p) {
    if (c.opt("wbuild_cublas", 0) == 0) {
      std::vector<GemmDesc> pd;
      for (int s = 0; s < c.N; ++s) {
        const int n = c.h_ns[s], L = c.h_ld[s];
        pd.push_back({k.Pinv.p + c.h_voff[s], k.XS.p + k.h_boff[s], k.WS.p + k.h_boff[s], n, B, n, L, L, L});
      }
      k.pgemm.set(c, pd);
    }
  }
  BlockOps ops(c, k, h, c.k0);
  const int cb = (B + 127) / 128;
  std::vector<ColState> hs(B);
  // Continuous batching: B slots, each running one column's PCG with its own
  // alpha, beta and stopping state; a slot whose column finished is refilled
  // with the next column at once, so the block DGEMMs never carry finished
  // columns while work remains (per-column semantics are unchanged: a refilled
  // slot spends one pass on its initialisation, r = b, z = H2 r, p = z).
  std::vector<int> slot(B, -1), fresh(B, 0);
  DArr<int> d_fresh;
  d_fresh.alloc(B);
  int next = 0, finished = 0, passes = 0;
  kc_clear<<<cb, 128, 0, c.stream>>>(B, k.st.p, k.done.p);
  ++c.launches;
  auto refill = [&]() {
    bool any = false;
    for (int j = 0; j < B; ++j) {
      fresh[j] = 0;
      if (slot[j] >= 0 || next >= total) continue;
      const int s = modes[next].first, kk = modes[next].second;
      double* bj = k.Bm.p + size_t(j) * k.ld;
      AWG_CUDA(cudaMemsetAsync(bj, 0, sizeof(double) * k.ld, c.stream));
      k::scatter_col(c, s, c.V.p + c.h_voff[s] + size_t(kk) * c.h_ld[s], bj);
      AWG_CUDA(cudaMemsetAsync(k.X.p + size_t(j) * k.ld, 0, sizeof(double) * k.ld, c.stream));
      AWG_CUDA(cudaMemcpyAsync(k.R.p + size_t(j) * k.ld, bj, sizeof(double) * k.ld, cudaMemcpyDeviceToDevice,
                               c.stream));
      slot[j] = next++;
      fresh[j] = 1;
      any = true;
    }
    if (!any) return;
    d_fresh.upload(fresh, c.stream);
    ops.dot(k.R.p, k.R.p, 0, nullptr);
    kc_fresh<<<cb, 128, 0, c.stream>>>(B, k.st.p, k.part.p, k.G, k.done.p, d_fresh.p);
    ++c.launches;
  };
  refill();
  const dim3 gn = ops.grid_n();
  const bool prof_pass = c.opt("verbose", 0) == 2;
  while (finished < total) {
    ops.prof = prof_pass && passes == 5;
    ops.mark("start");
    ops.aplus(k.Pm.p, k.Q.p, k.done.p);
    ops.mark("aplus");
    ops.dot(k.Pm.p, k.Q.p, 0, nullptr);
    kc_alpha<<<cb, 128, 0, c.stream>>>(B, k.st.p, k.part.p, k.G, k.done.p);
    kb_update<<<dim3(k.G, B), kT, 0, c.stream>>>(c.n, k.ld, k.st.p, k.X.p, k.R.p, k.Pm.p, k.Q.p, k.part.p);
    AWG_CUDA(cudaMemsetAsync(k.any_true.p, 0, sizeof(int), c.stream));
    kc_relres<<<cb, 128, 0, c.stream>>>(B, k.st.p, k.part.p, k.G, rtol, maxit, k.done.p, k.any_true.p);
    c.launches += 3;
    int any = 0;
    AWG_CUDA(cudaMemcpyAsync(&any, k.any_true.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    AWG_CUDA(cudaStreamSynchronize(c.stream));
    if (any) {  // true residual b - A+ x for the columns that reached rtol
      ops.aplus(k.X.p, k.T.p, k.done.p);
      ops.dot(nullptr, k.T.p, 1, k.Bm.p);
      kc_true<<<cb, 128, 0, c.stream>>>(B, k.st.p, k.part.p, k.G, rtol, maxit, k.done.p);
      ++c.launches;
    }
    ops.mark("update+relres");
    ops.h2(k.R.p, k.Z.p, k.done.p);
    ops.dot(k.R.p, k.Z.p, 0, nullptr);
    kc_rz<<<cb, 128, 0, c.stream>>>(B, k.st.p, k.part.p, k.G, k.done.p, 0);
    kb_p<<<gn, kT, 0, c.stream>>>(c.n, k.ld, k.st.p, k.Z.p, k.Pm.p, 0);
    c.launches += 2;
    ops.mark("rz+p");
    ops.report();
    ++passes;
    AWG_CUDA(cudaMemcpyAsync(hs.data(), k.st.p, sizeof(ColState) * B, cudaMemcpyDeviceToHost, c.stream));
    AWG_CUDA(cudaStreamSynchronize(c.stream));
    for (int j = 0; j < B; ++j) {
      if (slot[j] < 0 || !hs[j].done) continue;
      if (hs[j].error) c.fail(AWG_E_BREAKDOWN, "build_w: inner PCG breakdown");
      if (!hs[j].converged) c.fail(AWG_E_NO_CONVERGENCE, "build_w: inner PCG for a W column did not converge");
      iters[slot[j]] = hs[j].it;
      AWG_CUDA(cudaMemcpyAsync(c.W.p + size_t(slot[j]) * c.ldw, k.X.p + size_t(j) * k.ld, sizeof(double) * c.n,
                               cudaMemcpyDeviceToDevice, c.stream));
      slot[j] = -1;
      ++finished;
    }
    refill();
    if (passes % 250 == 0) {
      if (c.opt("verbose", 0) == 1)
        std::fprintf(stderr, "[awg setup]   W block pass %d: %d of %d columns done (B = %d)\n", passes, finished,
                     total, B);
    }
  }
  c.w_batches += passes;
  AWG_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace awgb
