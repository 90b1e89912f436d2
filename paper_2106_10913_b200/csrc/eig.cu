// Batched dense symmetric eigensolver for the setup (hand-written, sm_100a):
// the B^s eigendecompositions of the splitting (dense_sym_eig, dense.cpp:117-209,
// called from eigsplit, splitting.cpp:64-84) and the standard problems the
// GenEO pencils reduce to (generalized_sym_eig, dense.cpp:211-224).  The
// reference runs cyclic Jacobi; any accurate symmetric eigensolver produces
// the same spectra (parity on eigenvalues, mode counts and
// basis-invariant operators).  Three stages, one problem per CTA where the
// stage is sequential, grouped FP64 tensor-core GEMMs (dgemm.cu) where it is
// not:
//
// 1. Householder tridiagonalisation Q^T A Q = T (LAPACK's dsytrd / dlatrd
//    algorithm, lower storage, panels of kNB = 64 columns).  k_latrd (one
//    persistent CTA per problem) reduces the panel's columns one by one; the
//    symmetric matrix-vector product of each column streams the trailing
//    lower triangle column by column from HBM into shared memory with TMA
//    bulk copies (cp.async.bulk + mbarrier ring, the single-pass local solve's
//    pipeline) and uses each column for both halves of the product (the dot
//    into w_c and the rank-1 update w += A(:,c) v_c), so the triangle is read
//    once per column.  The rank-2k update of the trailing matrix after each
//    panel (A22 -= V W^T + W V^T) is one grouped DMMA GEMM over all problems,
//    lower tiles only.
// 2. Eigenvalues of T by bisection on Sturm counts (thread per eigenvalue),
//    eigenvectors of T by the twisted factorisation (thread per vector, in place
//    in the output column: no scratch), and inverse iteration with
//    reorthogonalisation (LAPACK dstein's scheme) for clusters of close
//    eigenvalues, where single twisted vectors would not be orthogonal.
// 3. Back-transformation Z <- Q Z with the compact WY form of blocks of 128
//    reflectors (Q_b = I - V_b T_b V_b^T; T_b from the Gram matrix V_b^T V_b and
//    the taus, LAPACK dlarft): grouped DMMA GEMMs over all problems.
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cfloat>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <functional>
#include <vector>

#include "awg_internal.cuh"

namespace awgb {
namespace {

constexpr int kNB = 64;        // panel width
constexpr int kLT = 480;       // k_latrd row-owning (consumer) threads: 15 warps + 1 producer warp,
constexpr int kLW = kLT / 32;  // 512 threads in all (128 registers per thread)
constexpr size_t kLatrdSmemCap = size_t(217) * 1024;  // + ~10 KB static (part, mbarriers) <= 227 KB

struct EigDev {
  double* A;     // n x n, ld (lower referenced; reflectors on return)
  double* VW;    // ld x 2 kNB: panel V (columns 0..kNB-1) and W (kNB..2kNB-1)
  double* Bt;    // (2 kNB) x n, column-major: row-major [W V] (the rank-2k update's B operand)
  double* d;     // n: diagonal of T
  double* e;     // n: off-diagonal of T (e[j] = T(j+1, j))
  double* tau;   // n
  int n, ld;
};

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_arm(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void cp_async16(double* dst, const double* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// 1. Panel reduction (dlatrd, lower).  Columns j = k0 .. k0 + jmax - 1.
// 15 consumer warps own the rows cyclically (row i = tid + kLT * k, k < R, in
// registers); a 17th warp is the copy producer of the symmetric product's TMA
// ring (nslot column slots of L doubles, full / empty mbarriers: no CTA barrier
// per column).  Shared memory: the ring + v (L doubles).
constexpr int kLThreads = kLT + 32;

__device__ __forceinline__ void mb_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void bar_consumers() { asm volatile("bar.sync 1, %0;" ::"n"(kLT) : "memory"); }

// kTC per-lane partials -> lanes l < kTC hold the warp sum of partial l
constexpr int kStages = 5;          // shared-memory ring depth (tiles)
constexpr int kTC = 8;              // columns per tile
constexpr int kTile = kTC * kLT;    // doubles per ring slot (30 KB)
__device__ __forceinline__ double transpose_reduce8(double (&v)[kTC], int lane) {
  // fold the lane halves until kTC lanes remain per column, then exchange
#pragma unroll
  for (int o = 16; o >= kTC; o >>= 1)
#pragma unroll
    for (int k = 0; k < kTC; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
#pragma unroll
  for (int st = kTC / 2; st >= 1; st >>= 1) {
    const bool up = (lane & st) != 0;
#pragma unroll
    for (int k = 0; k < st; ++k) {
      const double send = up ? v[k] : v[k + st];
      const double keep = up ? v[k + st] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, st);
    }
  }
  return v[0];  // lane l: column l % kTC
}

template <int R>
__global__ void __launch_bounds__(kLThreads, 1) k_latrd(const EigDev* __restrict__ jobs, int k0, int L, int nslot,
                                                        unsigned long long* __restrict__ prof, int probe) {
  extern __shared__ __align__(128) double esm[];
  __shared__ double red[16];
  __shared__ double part[2][kLW][kTC];
  __shared__ double s_rowv[kNB], s_roww[kNB], s_s1[kNB], s_s2[kNB];
  __shared__ double s_scal[4];
  __shared__ __align__(8) unsigned long long full[8], empty[8];
  __shared__ unsigned s_nfill;
  const EigDev J = jobs[blockIdx.x];
  const int n = J.n, ld = J.ld, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (k0 >= n - 1) return;
  const bool cons = tid < kLT;  // row owner (the producer warp owns no rows)
  const int jmax = min(kNB, n - 1 - k0);
  double* vsm = esm + (size_t)nslot * kTile;
  double* Vp = J.VW;
  double* Wp = J.VW + (size_t)kNB * ld;
  auto bsum = [&](double v) {  // CTA-wide sum (the producer warp contributes 0; every thread gets it)
    v = wsum(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double a = red[lane & 15];
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    return a;
  };
  if (tid == 0) {
    for (int b = 0; b < nslot; ++b) {
      mb_init(&full[b], 1);
      mb_init(&empty[b], kLW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // zero the panel (unused columns must be zero for the rank-2k update)
  if (cons) {
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int i = tid + kLT * k;
      if (i < n) {
        for (int p = 0; p < 2 * kNB; ++p) {
          J.VW[i + (size_t)p * ld] = 0.0;
          J.Bt[(size_t)i * 2 * kNB + p] = 0.0;
        }
      }
    }
  }
  for (int t = tid; t < nslot * kTile; t += kLThreads) esm[t] = 0.0;  // finite from the start
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zero fill before the first bulk copies
  __syncthreads();
  unsigned g = 0;  // ring fills so far: slot g % nslot, fill round g / nslot

  for (int jj = 0; jj < jmax; ++jj) {
    const int j = k0 + jj;
    long long tc0 = clock64();
    // (1) column j of the trailing matrix with the panel's earlier updates:
    //     a = A(j:n, j) - V(j:n, 0:jj) W(j, 0:jj)^T - W(j:n, 0:jj) V(j, 0:jj)^T
    if (tid < jj) {
      s_rowv[tid] = Vp[j + (size_t)tid * ld];
      s_roww[tid] = Wp[j + (size_t)tid * ld];
    }
    __syncthreads();
    double ar[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int i = tid + kLT * k;
      double a = 0.0;
      if (cons && i >= j && i < n) {
        // independent partial sums: the panel loads of a row go out together
        double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
        int p = 0;
        for (; p + 2 <= jj; p += 2) {
          c0 = fma(Vp[i + (size_t)p * ld], s_roww[p], c0);
          c1 = fma(Wp[i + (size_t)p * ld], s_rowv[p], c1);
          c2 = fma(Vp[i + (size_t)(p + 1) * ld], s_roww[p + 1], c2);
          c3 = fma(Wp[i + (size_t)(p + 1) * ld], s_rowv[p + 1], c3);
        }
        if (p < jj) {
          c0 = fma(Vp[i + (size_t)p * ld], s_roww[p], c0);
          c1 = fma(Wp[i + (size_t)p * ld], s_rowv[p], c1);
        }
        a = J.A[i + (size_t)j * ld] - ((c0 + c2) + (c1 + c3));
        if (i == j) s_scal[0] = a;      // diagonal d_j
        if (i == j + 1) s_scal[1] = a;  // alpha
      }
      ar[k] = a;
    }
    // (2) Householder reflector of a(j+1:n) (dlarfg): H = I - tau v v^T, v(j+1) = 1
    double ss = 0.0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int i = tid + kLT * k;
      if (cons && i > j + 1 && i < n) ss = fma(ar[k], ar[k], ss);
    }
    const double xnorm2 = bsum(ss);  // (its barriers also publish s_scal)
    const double dj = s_scal[0], alpha = s_scal[1];
    double beta, tau, scale;
    if (xnorm2 == 0.0) {
      beta = alpha;
      tau = 0.0;
      scale = 0.0;
    } else {
      beta = -copysign(sqrt(fma(alpha, alpha, xnorm2)), alpha);
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    double vr[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int i = tid + kLT * k;
      const double v = (i == j + 1) ? 1.0 : (i > j + 1 && i < n ? ar[k] * scale : 0.0);
      vr[k] = cons ? v : 0.0;
      if (cons && i < n) {
        vsm[i] = v;
        Vp[i + (size_t)jj * ld] = v;
        if (i > j) J.A[i + (size_t)j * ld] = v;  // reflector storage (explicit 1 at j + 1)
      }
    }
    __syncthreads();  // vsm complete before the product reads v_c
    long long tc1 = clock64();
    // (3) y = A(j+1:n, j+1:n) v over the stored lower triangle (not yet
    //     updated by this panel): column c contributes the dot
    //     sum_{i > c} A(i, c) v_i to y_c and A(i, c) v_c to y_i (i >= c).
    double yr[R];
#pragma unroll
    for (int k = 0; k < R; ++k) yr[k] = 0.0;
    const int c_begin = j + 1;
    // Tiles of kTC columns x kLT rows (row chunk k = rows kLT k .. kLT k + kLT - 1,
    // exactly the rows thread t owns as slot k): one fill = kTC bulk copies of
    // the columns' chunk segments, issued in parallel by the producer warp's
    // lanes.  Consumers loop over column groups and, inside, over their row
    // chunks (unrolled: y and v of chunk k stay in registers); the dot partials
    // of a group are reduced once after all its chunks.  Producer and consumers
    // walk the same (group, chunk) sequence.  (Measured against cp.async staged
    // by every thread with a CTA barrier per tile: 5.7 vs 3.6 s for 16 B^s-sized
    // problems of order 4,482.)
    unsigned nfill = 0;
    if (!cons) {
      if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int G0 = c_begin; G0 < n; G0 += kTC) {
        const int K = min(kTC, n - G0);
        for (int k = G0 / kLT; k * kLT < n; ++k) {
          const unsigned gq = g + nfill, b = gq % nslot, round = gq / nslot;
          const int r0 = k * kLT, rows = min(kLT, n - r0);
          const unsigned bytes = unsigned((rows + 1) & ~1) * 8u;
          if (lane == 0) {
            if (round > 0) mb_wait(&empty[b], (round - 1) & 1);
            mb_arm(&full[b], bytes * unsigned(K));
          }
          __syncwarp();
          if (lane < K)
            bulk_copy(esm + (size_t)b * kTile + (size_t)lane * kLT, J.A + r0 + (size_t)(G0 + lane) * ld, bytes, &full[b]);
          ++nfill;
        }
      }
      __syncwarp();
    } else {
      for (int G0 = c_begin; G0 < n; G0 += kTC) {
        const int kstart = G0 / kLT;
        double acc[kTC], vcol[kTC];
#pragma unroll
        for (int u = 0; u < kTC; ++u) {
          acc[u] = 0.0;
          vcol[u] = (G0 + u < n) ? vsm[G0 + u] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < R; ++k) {
          if (k >= kstart && k * kLT < n) {  // uniform
            const unsigned gq = g + nfill, b = gq % nslot;
            mb_wait(&full[b], (gq / nslot) & 1);
            const double* tile = esm + (size_t)b * kTile + tid;
            const int i = tid + kLT * k;
            const double vi = vr[k];
            double y = yr[k];
            if (probe == 1) {
              // timing probe only (option eig_probe = 1): no arithmetic
            } else if (k * kLT >= G0 + kTC) {
              // every row of the chunk lies strictly below the group's columns.  Rows
              // >= n and columns >= n need no mask: their slot entries are stale but
              // finite (the ring starts zeroed), v_i = 0 for i >= n and v_c = 0 for
              // c >= n, and those rows / columns are never written out
#pragma unroll
              for (int u = 0; u < kTC; ++u) {
                const double a = tile[u * kLT];
                y = fma(a, vcol[u], y);
                acc[u] = fma(a, vi, acc[u]);
              }
            } else {
#pragma unroll
              for (int u = 0; u < kTC; ++u) {
                const int c = G0 + u;
                const double a = (i >= c) ? tile[u * kLT] : 0.0;  // rows above the diagonal: stale
                y = fma(a, vcol[u], y);
                acc[u] = (i > c) ? fma(a, vi, acc[u]) : acc[u];
              }
            }
            yr[k] = y;
            __syncwarp();
            if (lane == 0) mb_arrive(&empty[b]);
            ++nfill;
          }
        }
        const double wpart = transpose_reduce8(acc, lane);  // lanes l < kTC: this warp's dot for column G0 + l
        const int pb = ((G0 - c_begin) / kTC) & 1;
        if (lane < kTC) part[pb][warp][lane] = wpart;
        bar_consumers();
        if (warp == 0 && lane < kTC && G0 + lane < n) {
          double sdot = 0.0;
#pragma unroll
          for (int w = 0; w < kLW; ++w) sdot += part[pb][w][lane];
          Wp[G0 + lane + (size_t)jj * ld] = sdot;  // parked in W(:, jj) until (4)
        }
      }
    }
    // every thread advances the fill counter by the same count
    if (tid == 0) s_nfill = nfill;
    __syncthreads();
    g += s_nfill;
    __syncthreads();
    long long tc2 = clock64();
    // (4) w = tau (y - V (W^T v) - W (V^T v)); w += (-tau/2 w^T v) v
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int i = tid + kLT * k;
      if (cons && i > j && i < n) yr[k] += Wp[i + (size_t)jj * ld];
    }
    for (int p = warp; p < 2 * jj; p += kLW + 1) {  // s1 = W^T v, s2 = V^T v over rows > j
      const double* colp = (p < jj) ? Wp + (size_t)p * ld : Vp + (size_t)(p - jj) * ld;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int i = j + 1 + lane;
      for (; i + 96 < n; i += 128) {
        a0 = fma(colp[i], vsm[i], a0);
        a1 = fma(colp[i + 32], vsm[i + 32], a1);
        a2 = fma(colp[i + 64], vsm[i + 64], a2);
        a3 = fma(colp[i + 96], vsm[i + 96], a3);
      }
      for (; i < n; i += 32) a0 = fma(colp[i], vsm[i], a0);
      const double acc = wsum((a0 + a1) + (a2 + a3));
      if (lane == 0) {
        if (p < jj) s_s1[p] = acc;
        else s_s2[p - jj] = acc;
      }
    }
    __syncthreads();
    double wv = 0.0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int i = tid + kLT * k;
      double y = 0.0;
      if (cons && i > j && i < n) {
        double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
        int p = 0;
        for (; p + 2 <= jj; p += 2) {
          c0 = fma(Vp[i + (size_t)p * ld], s_s1[p], c0);
          c1 = fma(Wp[i + (size_t)p * ld], s_s2[p], c1);
          c2 = fma(Vp[i + (size_t)(p + 1) * ld], s_s1[p + 1], c2);
          c3 = fma(Wp[i + (size_t)(p + 1) * ld], s_s2[p + 1], c3);
        }
        if (p < jj) {
          c0 = fma(Vp[i + (size_t)p * ld], s_s1[p], c0);
          c1 = fma(Wp[i + (size_t)p * ld], s_s2[p], c1);
        }
        y = (yr[k] - ((c0 + c2) + (c1 + c3))) * tau;
      }
      yr[k] = y;
      wv = fma(y, vr[k], wv);
    }
    const double alpha2 = -0.5 * tau * bsum(wv);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int i = tid + kLT * k;
      if (cons && i < n) {
        const double w = (i > j) ? fma(alpha2, vr[k], yr[k]) : 0.0;
        Wp[i + (size_t)jj * ld] = w;
        J.Bt[(size_t)i * 2 * kNB + jj] = w;
        J.Bt[(size_t)i * 2 * kNB + kNB + jj] = vr[k];
      }
    }
    if (prof && tid == 0) {  // cycle profile (option verbose >= 2): steps 1-2, 3, 4
      const long long tc3 = clock64();
      atomicAdd(&prof[0], (unsigned long long)(tc1 - tc0));
      atomicAdd(&prof[1], (unsigned long long)(tc2 - tc1));
      atomicAdd(&prof[2], (unsigned long long)(tc3 - tc2));
    }
    if (tid == 0) {  // (the block-reflector factors T are formed by the back-transformation)
      J.d[j] = dj;
      J.e[j] = beta;
      J.tau[j] = tau;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// 1b. Split form of the panel reduction for batches with fewer problems than
// SMs (c2: 16 subdomains, c3: 64).  k_latrd keeps one CTA per problem, so 16
// problems use 16 of 148 SMs while the symmetric product, 85% of the work,
// streams each trailing triangle through one SM.  Here one column step is two
// launches: k_symv_part splits the column groups of the product over C CTAs
// per problem (cyclically: column lengths fall linearly) — each CTA owns the
// whole dot of its columns (parked in W(:, jj) as in k_latrd) and writes a
// partial of the rank-1 half for all rows —, then k_col_step (one CTA per
// problem) sums the partials in CTA order, finishes w of that column (step 4)
// and forms the next column and its reflector (steps 1-2).  Same arithmetic per
// phase as k_latrd; only y's summation is regrouped by CTA.  Fixed C per
// batch: results are deterministic.
template <int R>
__global__ void __launch_bounds__(kLThreads, 1) k_symv_part(const EigDev* __restrict__ jobs, int k0, int jj, int C,
                                                            int L, int nslot, double* __restrict__ ypart) {
  extern __shared__ __align__(128) double esm[];
  __shared__ double part[2][kLW][kTC];
  __shared__ __align__(8) unsigned long long full[8], empty[8];
  const int q = blockIdx.x / C, cta = blockIdx.x % C;
  const EigDev J = jobs[q];
  const int n = J.n, ld = J.ld, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (k0 >= n - 1) return;
  const int jmax = min(kNB, n - 1 - k0);
  if (jj >= jmax) return;
  const int j = k0 + jj;
  const bool cons = tid < kLT;
  double* vsm = esm + (size_t)nslot * kTile;
  const double* Vj = J.VW + (size_t)jj * ld;      // this column's reflector v (zero above row j + 1)
  double* Wj = J.VW + (size_t)(kNB + jj) * ld;    // dots parked here
  if (tid == 0) {
    for (int b = 0; b < nslot; ++b) {
      mb_init(&full[b], 1);
      mb_init(&empty[b], kLW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int t = tid; t < nslot * kTile; t += kLThreads) esm[t] = 0.0;  // stale slot entries must be finite
  for (int i = tid; i < L; i += kLThreads) vsm[i] = (i < n) ? Vj[i] : 0.0;
  double vr[R], yr[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int i = tid + kLT * k;
    vr[k] = (cons && i < n) ? Vj[i] : 0.0;
    yr[k] = 0.0;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const int c_begin = j + 1;
  const int gstep = kTC * C;
  unsigned nfill = 0;
  if (!cons) {
    for (int G0 = c_begin + kTC * cta; G0 < n; G0 += gstep) {
      const int K = min(kTC, n - G0);
      for (int k = G0 / kLT; k * kLT < n; ++k) {
        const unsigned b = nfill % nslot, round = nfill / nslot;
        const int r0 = k * kLT, rows = min(kLT, n - r0);
        const unsigned bytes = unsigned((rows + 1) & ~1) * 8u;
        if (lane == 0) {
          if (round > 0) mb_wait(&empty[b], (round - 1) & 1);
          mb_arm(&full[b], bytes * unsigned(K));
        }
        __syncwarp();
        if (lane < K)
          bulk_copy(esm + (size_t)b * kTile + (size_t)lane * kLT, J.A + r0 + (size_t)(G0 + lane) * ld, bytes, &full[b]);
        ++nfill;
      }
    }
    __syncwarp();
  } else {
    int gi = 0;
    for (int G0 = c_begin + kTC * cta; G0 < n; G0 += gstep, ++gi) {
      const int kstart = G0 / kLT;
      double acc[kTC], vcol[kTC];
#pragma unroll
      for (int u = 0; u < kTC; ++u) {
        acc[u] = 0.0;
        vcol[u] = (G0 + u < n) ? vsm[G0 + u] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if (k >= kstart && k * kLT < n) {  // uniform
          const unsigned b = nfill % nslot;
          mb_wait(&full[b], (nfill / nslot) & 1);
          const double* tile = esm + (size_t)b * kTile + tid;
          const int i = tid + kLT * k;
          const double vi = vr[k];
          double y = yr[k];
          if (k * kLT >= G0 + kTC) {  // the chunk lies strictly below the group's columns (see k_latrd)
#pragma unroll
            for (int u = 0; u < kTC; ++u) {
              const double a = tile[u * kLT];
              y = fma(a, vcol[u], y);
              acc[u] = fma(a, vi, acc[u]);
            }
          } else {
#pragma unroll
            for (int u = 0; u < kTC; ++u) {
              const int c = G0 + u;
              const double a = (i >= c) ? tile[u * kLT] : 0.0;
              y = fma(a, vcol[u], y);
              acc[u] = (i > c) ? fma(a, vi, acc[u]) : acc[u];
            }
          }
          yr[k] = y;
          __syncwarp();
          if (lane == 0) mb_arrive(&empty[b]);
          ++nfill;
        }
      }
      const double wpart = transpose_reduce8(acc, lane);
      const int pb = gi & 1;
      if (lane < kTC) part[pb][warp][lane] = wpart;
      bar_consumers();
      if (warp == 0 && lane < kTC && G0 + lane < n) {
        double sdot = 0.0;
#pragma unroll
        for (int w = 0; w < kLW; ++w) sdot += part[pb][w][lane];
        Wj[G0 + lane] = sdot;
      }
    }
    double* yp = ypart + ((size_t)q * C + cta) * L;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int i = tid + kLT * k;
      if (i < n) yp[i] = yr[k];
    }
  }
}

template <int R>
__global__ void __launch_bounds__(kLThreads, 1) k_col_step(const EigDev* __restrict__ jobs, int k0, int jj, int C, int L,
                                                           const double* __restrict__ ypart) {
  extern __shared__ __align__(128) double vsm[];  // L doubles
  __shared__ double red[16];
  __shared__ double s_rowv[kNB], s_roww[kNB], s_s1[kNB], s_s2[kNB];
  __shared__ double s_scal[4];
  const EigDev J = jobs[blockIdx.x];
  const int n = J.n, ld = J.ld, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (k0 >= n - 1) return;
  const bool cons = tid < kLT;
  const int jmax = min(kNB, n - 1 - k0);
  double* Vp = J.VW;
  double* Wp = J.VW + (size_t)kNB * ld;
  auto bsum = [&](double v) {
    v = wsum(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double a = red[lane & 15];
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    return a;
  };
  if (jj == 0) {  // new panel: unused columns must be zero for the rank-2k update
    if (cons) {
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int i = tid + kLT * k;
        if (i < n) {
          for (int p = 0; p < 2 * kNB; ++p) {
            J.VW[i + (size_t)p * ld] = 0.0;
            J.Bt[(size_t)i * 2 * kNB + p] = 0.0;
          }
        }
      }
    }
    __syncthreads();
  }
  // ---- finish column jj - 1: step (4) of k_latrd on the summed product
  if (jj > 0 && jj - 1 < jmax) {
    const int jp = jj - 1, j = k0 + jp;
    const double tau = J.tau[j];
    double vr[R], yr[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int i = tid + kLT * k;
      double v = 0.0, y = 0.0;
      if (cons && i < n) {
        v = Vp[i + (size_t)jp * ld];
        vsm[i] = v;
        if (i > j) {
          const double* yp = ypart + (size_t)blockIdx.x * C * L + i;
          for (int cta = 0; cta < C; ++cta) y += yp[(size_t)cta * L];
          y += Wp[i + (size_t)jp * ld];
        }
      }
      vr[k] = v;
      yr[k] = y;
    }
    __syncthreads();
    for (int p = warp; p < 2 * jp; p += kLW + 1) {  // s1 = W^T v, s2 = V^T v over rows > j
      const double* colp = (p < jp) ? Wp + (size_t)p * ld : Vp + (size_t)(p - jp) * ld;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int i = j + 1 + lane;
      for (; i + 96 < n; i += 128) {
        a0 = fma(colp[i], vsm[i], a0);
        a1 = fma(colp[i + 32], vsm[i + 32], a1);
        a2 = fma(colp[i + 64], vsm[i + 64], a2);
        a3 = fma(colp[i + 96], vsm[i + 96], a3);
      }
      for (; i < n; i += 32) a0 = fma(colp[i], vsm[i], a0);
      const double acc = wsum((a0 + a1) + (a2 + a3));
      if (lane == 0) {
        if (p < jp) s_s1[p] = acc;
        else s_s2[p - jp] = acc;
      }
    }
    __syncthreads();
    double wv = 0.0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int i = tid + kLT * k;
      double y = 0.0;
      if (cons && i > j && i < n) {
        double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
        int p = 0;
        for (; p + 2 <= jp; p += 2) {
          c0 = fma(Vp[i + (size_t)p * ld], s_s1[p], c0);
          c1 = fma(Wp[i + (size_t)p * ld], s_s2[p], c1);
          c2 = fma(Vp[i + (size_t)(p + 1) * ld], s_s1[p + 1], c2);
          c3 = fma(Wp[i + (size_t)(p + 1) * ld], s_s2[p + 1], c3);
        }
        if (p < jp) {
          c0 = fma(Vp[i + (size_t)p * ld], s_s1[p], c0);
          c1 = fma(Wp[i + (size_t)p * ld], s_s2[p], c1);
        }
        y = (yr[k] - ((c0 + c2) + (c1 + c3))) * tau;
      }
      yr[k] = y;
      wv = fma(y, vr[k], wv);
    }
    const double alpha2 = -0.5 * tau * bsum(wv);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int i = tid + kLT * k;
      if (cons && i < n) {
        const double w = (i > j) ? fma(alpha2, vr[k], yr[k]) : 0.0;
        Wp[i + (size_t)jp * ld] = w;
        J.Bt[(size_t)i * 2 * kNB + jp] = w;
        J.Bt[(size_t)i * 2 * kNB + kNB + jp] = vr[k];
      }
    }
    __syncthreads();  // W(:, jp) complete before the next column's row reads
  }
  if (jj >= jmax) return;
  // ---- start column jj: steps (1)-(2) of k_latrd
  const int j = k0 + jj;
  if (tid < jj) {
    s_rowv[tid] = Vp[j + (size_t)tid * ld];
    s_roww[tid] = Wp[j + (size_t)tid * ld];
  }
  __syncthreads();
  double ar[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int i = tid + kLT * k;
    double a = 0.0;
    if (cons && i >= j && i < n) {
      double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
      int p = 0;
      for (; p + 2 <= jj; p += 2) {
        c0 = fma(Vp[i + (size_t)p * ld], s_roww[p], c0);
        c1 = fma(Wp[i + (size_t)p * ld], s_rowv[p], c1);
        c2 = fma(Vp[i + (size_t)(p + 1) * ld], s_roww[p + 1], c2);
        c3 = fma(Wp[i + (size_t)(p + 1) * ld], s_rowv[p + 1], c3);
      }
      if (p < jj) {
        c0 = fma(Vp[i + (size_t)p * ld], s_roww[p], c0);
        c1 = fma(Wp[i + (size_t)p * ld], s_rowv[p], c1);
      }
      a = J.A[i + (size_t)j * ld] - ((c0 + c2) + (c1 + c3));
      if (i == j) s_scal[0] = a;
      if (i == j + 1) s_scal[1] = a;
    }
    ar[k] = a;
  }
  double ss = 0.0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int i = tid + kLT * k;
    if (cons && i > j + 1 && i < n) ss = fma(ar[k], ar[k], ss);
  }
  const double xnorm2 = bsum(ss);
  const double dj = s_scal[0], alpha = s_scal[1];
  double beta, tau, scale;
  if (xnorm2 == 0.0) {
    beta = alpha;
    tau = 0.0;
    scale = 0.0;
  } else {
    beta = -copysign(sqrt(fma(alpha, alpha, xnorm2)), alpha);
    tau = (beta - alpha) / beta;
    scale = 1.0 / (alpha - beta);
  }
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int i = tid + kLT * k;
    const double v = (i == j + 1) ? 1.0 : (i > j + 1 && i < n ? ar[k] * scale : 0.0);
    if (cons && i < n) {
      Vp[i + (size_t)jj * ld] = v;
      if (i > j) J.A[i + (size_t)j * ld] = v;
    }
  }
  if (tid == 0) {
    J.d[j] = dj;
    J.e[j] = beta;
    J.tau[j] = tau;
  }
}

// the last diagonal entry: A(n-1, n-1) after its final panel's rank-2 update
// (that panel ends at column n-2, so its trailing matrix is this one entry:
// A(n-1,n-1) - 2 V(n-1,:) W(n-1,:)^T; done here instead of a 1 x 1 GEMM)
__global__ void k_last_diag(const EigDev* __restrict__ jobs) {
  const EigDev J = jobs[blockIdx.x];
  if (threadIdx.x != 0 || J.n <= 0) return;
  const int n = J.n;
  double a = J.A[(n - 1) + (size_t)(n - 1) * J.ld];
  if (n >= 2) {
    const double* Vp = J.VW;
    const double* Wp = J.VW + (size_t)kNB * J.ld;
    for (int p = 0; p < kNB; ++p) a -= 2.0 * Vp[(n - 1) + (size_t)p * J.ld] * Wp[(n - 1) + (size_t)p * J.ld];
  }
  J.d[n - 1] = a;
}

// ---------------------------------------------------------------------------
// 2. Tridiagonal eigenproblem.
struct TriDev {
  const double* d;
  const double* e;
  double* w;      // n eigenvalues, ascending (output)
  double* wu;     // n: unsorted scratch
  double* Z;      // n x nvec eigenvectors of T (ldz)
  double* scr;    // 5 n scratch (cluster inverse iteration)
  int n, ldz, nvec;
};

__device__ double tnorm_of(const double* d, const double* e, int n) {
  double m = 0.0;
  for (int i = 0; i < n; ++i) {
    const double r = fabs(d[i]) + (i > 0 ? fabs(e[i - 1]) : 0.0) + (i < n - 1 ? fabs(e[i]) : 0.0);
    m = fmax(m, r);
  }
  return m;
}

constexpr double kPivmin = 1e-290;

// number of eigenvalues of T strictly below x (Sturm sequence of the LDL^T of T - x)
__device__ __forceinline__ int sturm(const double* d, const double* e2, int n, double x) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < kPivmin) q = -kPivmin;
  cnt += q < 0.0;
  for (int i = 1; i < n; ++i) {
    q = (d[i] - x) - e2[i - 1] / q;
    if (fabs(q) < kPivmin) q = -kPivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

// thread per eigenvalue index; d and e^2 staged in shared memory (one problem per CTA row)
__global__ void k_bisect(const TriDev* __restrict__ jobs, int per_cta) {
  extern __shared__ double tsm[];
  const TriDev J = jobs[blockIdx.y];
  const int n = J.n;
  const int k = blockIdx.x * per_cta + threadIdx.x;
  if (blockIdx.x * per_cta >= n) return;
  double* d = tsm;
  double* e2 = tsm + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    d[i] = J.d[i];
    e2[i] = (i < n - 1) ? J.e[i] * J.e[i] : 0.0;
  }
  __syncthreads();
  if (k >= n || threadIdx.x >= per_cta) return;
  double lo = INFINITY, hi = -INFINITY;
  for (int i = 0; i < n; ++i) {
    const double r = (i > 0 ? fabs(J.e[i - 1]) : 0.0) + (i < n - 1 ? fabs(J.e[i]) : 0.0);
    lo = fmin(lo, d[i] - r);
    hi = fmax(hi, d[i] + r);
  }
  const double tn = fmax(fabs(lo), fabs(hi));
  lo -= 2.0 * DBL_EPSILON * tn + kPivmin;
  hi += 2.0 * DBL_EPSILON * tn + kPivmin;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (hi - lo <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + kPivmin) break;
    if (sturm(d, e2, n, mid) > k) hi = mid;
    else lo = mid;
  }
  J.wu[k] = 0.5 * (lo + hi);
}

// per problem: ascending sort of the bisection results (bitonic, in shared memory)
__global__ void k_sort_eigs(const TriDev* __restrict__ jobs, int pow2) {
  extern __shared__ double ssm[];
  const TriDev J = jobs[blockIdx.x];
  const int n = J.n;
  for (int i = threadIdx.x; i < pow2; i += blockDim.x) ssm[i] = i < n ? J.wu[i] : INFINITY;
  __syncthreads();
  for (int k = 2; k <= pow2; k <<= 1)
    for (int jx = k >> 1; jx > 0; jx >>= 1) {
      for (int i = threadIdx.x; i < pow2; i += blockDim.x) {
        const int l = i ^ jx;
        if (l > i) {
          const bool up = (i & k) == 0;
          const double a = ssm[i], b = ssm[l];
          if ((a > b) == up) {
            ssm[i] = b;
            ssm[l] = a;
          }
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < n; i += blockDim.x) J.w[i] = ssm[i];
}

// eigenvector of T for eigenvalue w[p] by the twisted factorisation
// T - lam = L+ D+ L+^T = U- D- U-^T, twist r = argmin |gamma_r|,
// gamma_r = D+_r + D-_r - (d_r - lam); z_r = 1, z_i = -(e_i / D+_i) z_{i+1}
// upwards, z_{i+1} = -(e_i / D-_{i+1}) z_i downwards.  In place in column p.
__global__ void k_twisted(const TriDev* __restrict__ jobs, int per_cta) {
  const TriDev J = jobs[blockIdx.y];
  const int p = blockIdx.x * per_cta + threadIdx.x;
  if (threadIdx.x >= per_cta || p >= J.nvec) return;
  const int n = J.n;
  const double* d = J.d;
  const double* e = J.e;
  const double lam = J.w[p];
  double* z = J.Z + (size_t)p * J.ldz;
  auto guard = [](double v) { return fabs(v) < kPivmin ? -kPivmin : v; };
  if (n == 1) {
    z[0] = 1.0;
    return;
  }
  // backward: D-_i into z[i]
  double dm = guard(d[n - 1] - lam);
  z[n - 1] = dm;
  for (int i = n - 2; i >= 0; --i) {
    dm = guard((d[i] - lam) - e[i] * e[i] / dm);
    z[i] = dm;
  }
  // forward: D+_i, gamma_i, argmin; z[i] <- D+_i
  double dp = guard(d[0] - lam);
  double best = fabs(dp + z[0] - (d[0] - lam));
  int r = 0;
  z[0] = dp;
  for (int i = 1; i < n; ++i) {
    dp = guard((d[i] - lam) - e[i - 1] * e[i - 1] / dp);
    const double gam = fabs(dp + z[i] - (d[i] - lam));
    if (gam < best) {
      best = gam;
      r = i;
    }
    z[i] = dp;
  }
  // D-_i again below the twist
  dm = guard(d[n - 1] - lam);
  if (n - 1 > r) z[n - 1] = dm;
  for (int i = n - 2; i > r; --i) {
    dm = guard((d[i] - lam) - e[i] * e[i] / dm);
    z[i] = dm;
  }
  // the vector
  double nrm = 1.0, zi = 1.0;
  for (int i = r - 1; i >= 0; --i) {
    zi = -(e[i] / z[i]) * zi;
    z[i] = zi;
    nrm = fma(zi, zi, nrm);
  }
  zi = 1.0;
  for (int i = r; i < n - 1; ++i) {
    zi = -(e[i] / z[i + 1]) * zi;
    z[i + 1] = zi;
    nrm = fma(zi, zi, nrm);
  }
  z[r] = 1.0;
  const double s = 1.0 / sqrt(nrm);
  for (int i = 0; i < n; ++i) z[i] *= s;
  J.wu[p] = isfinite(nrm) && nrm < 1e280 ? 0.0 : 1.0;  // 1: recompute by inverse iteration (k_clusters)
}

// Tight clusters (consecutive eigenvalues closer than kClusterTol * ||T||):
// twisted vectors of nearly equal eigenvalues can coincide, so their columns
// are recomputed by inverse iteration with reorthogonalisation against the
// cluster's earlier members in every step (LAPACK dstein), on the LU
// factorisation with partial pivoting of T - lam (dlagtf / dlagts).  One CTA
// per problem walks its clusters in order.  Every other pair of vectors is
// orthogonal to ~eps ||T|| / gap <= 1e-6 and is finished by the windowed
// Newton-Schulz step below.
constexpr double kClusterTol = 1e-10;
// Clusters of at most kSmallCluster vectors go to k_clusters_small (thread per
// cluster); larger ones stay with the CTA-per-problem walk below.
constexpr int kSmallCluster = 32;

// A problem's small clusters go to the thread-per-cluster kernel only when
// there are enough of them to fill warps (a lone thread is ~6x slower per
// vector than the CTA walk: a pencil's single zero cluster of ~20 vectors is
// faster on the CTA); both kernels take the same decision from the same walk.
constexpr int kMinThreadClusters = 64;
__device__ int count_small_clusters(const TriDev& J, double tol) {
  int cnt = 0, walk = 0;
  while (walk < J.nvec) {
    int q = walk + 1;
    while (q < J.n && J.w[q] - J.w[q - 1] < tol) ++q;
    const int sz = min(q, J.nvec) - walk;
    if ((sz >= 2 || J.wu[walk] != 0.0) && sz <= kSmallCluster) ++cnt;
    walk = q;
  }
  return cnt;
}

// Thread per cluster.  c2's B^s (1e6 contrast: ||T|| ~ 4e6, so the cluster
// gap is 4e-4 while ~3,700 eigenvalues lie in (0.1, 10)) have ~3,300 of their
// ~4,600 eigenvalues in ~1,000 clusters of 2-14 vectors: inverse iteration is
// serial along n, but the clusters are independent, so each thread takes
// whole clusters (cluster index = t mod T within its problem) and runs the
// same dstein scheme as k_clusters alone: dlagtf, four dlagts solves per
// vector, modified Gram-Schmidt against the cluster's earlier vectors.  The
// LU scratch is interleaved by thread (element i of thread t at (a L + i) T + t),
// so lock-stepped lanes store and load contiguous doubles; z is the output
// column itself.
__global__ void k_clusters_small(const TriDev* __restrict__ jobs, int T, int L, double* __restrict__ scratch) {
  const TriDev J = jobs[blockIdx.y];
  const int n = J.n, nv = J.nvec;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (n < 2 || nv < 2 || t >= T) return;
  double* S = scratch + (size_t)blockIdx.y * 5 * L * T + t;
  const size_t LT = (size_t)L * T;
  double* u1 = S;
  double* u2 = S + LT;
  double* u3 = S + 2 * LT;
  double* lm = S + 3 * LT;
  double* pv = S + 4 * LT;  // pivot flags (0.0 / 1.0)
  const double tn = tnorm_of(J.d, J.e, n);
  const double tol = kClusterTol * tn;
  const double small = DBL_EPSILON * tn + kPivmin;
  if (count_small_clusters(J, tol) < kMinThreadClusters) return;  // k_clusters takes them
  int walk = 0, ci = 0;  // eigenvalue index and small-cluster count of the walk so far
  for (int target = t;; target += T) {
    // advance the walk to this thread's next cluster; every lane then works on
    // its own cluster at the same time
    int p = -1, qend = 0;
    while (walk < nv) {
      int q = walk + 1;
      while (q < n && J.w[q] - J.w[q - 1] < tol) ++q;
      const int qe = min(q, nv);
      const int sz = qe - walk;
      const bool mine = (sz >= 2 || J.wu[walk] != 0.0) && sz <= kSmallCluster;
      const int start = walk;
      walk = q;
      if (mine) {
        if (ci++ == target) {
          p = start;
          qend = qe;
          break;
        }
      }
    }
    if (p < 0) return;
    for (int m = p; m < qend; ++m) {
      double lam = J.w[m];
      if (m > p && lam - J.w[m - 1] < 10.0 * DBL_EPSILON * tn) lam = J.w[m - 1] + 10.0 * DBL_EPSILON * tn * (m - p);
      {  // LU of T - lam with partial pivoting (dlagtf)
        double r0 = J.d[0] - lam, r1 = J.e[0], r2 = 0.0;
        for (int i = 0; i < n - 1; ++i) {
          const double n0 = J.e[i], n1 = J.d[i + 1] - lam, n2 = (i + 1 < n - 1) ? J.e[i + 1] : 0.0;
          const size_t o = (size_t)i * T;
          if (fabs(r0) >= fabs(n0)) {
            const double l = (r0 != 0.0) ? n0 / r0 : 0.0;
            u1[o] = (r0 != 0.0) ? r0 : small;
            u2[o] = r1;
            u3[o] = r2;
            lm[o] = l;
            pv[o] = 0.0;
            r0 = n1 - l * r1;
            r1 = n2 - l * r2;
            r2 = 0.0;
          } else {
            const double l = r0 / n0;
            u1[o] = n0;
            u2[o] = n1;
            u3[o] = n2;
            lm[o] = l;
            pv[o] = 1.0;
            r0 = r1 - l * n1;
            r1 = r2 - l * n2;
            r2 = 0.0;
          }
        }
        u1[(size_t)(n - 1) * T] = (r0 != 0.0) ? r0 : small;
      }
      double* z = J.Z + (size_t)m * J.ldz;
      for (int i = 0; i < n; ++i) {  // the same deterministic start vector as k_clusters
        unsigned long long h = (unsigned long long)(i + 1) * 0x9E3779B97F4A7C15ull + (unsigned long long)(m + 1);
        h ^= h >> 31;
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 29;
        z[i] = double(h >> 11) * 0x1.0p-53 - 0.5;
      }
      for (int it = 0; it < 4; ++it) {
        // solve (T - lam) x = z in place: P L U (dlagts)
        double zi = z[0];
        for (int i = 0; i < n - 1; ++i) {
          double zn = z[i + 1];
          const size_t o = (size_t)i * T;
          if (pv[o] != 0.0) {
            const double tmp = zi;
            zi = zn;
            zn = tmp;
          }
          z[i] = zi;
          zi = zn - lm[o] * zi;
        }
        z[n - 1] = zi;
        double mx = 0.0, z1 = 0.0, z2 = 0.0;  // z[i + 1], z[i + 2]
        for (int i = n - 1; i >= 0; --i) {
          const size_t o = (size_t)i * T;
          double v = z[i];
          if (i + 1 < n) v -= u2[o] * z1;
          if (i + 2 < n) v -= u3[o] * z2;
          double piv0 = u1[o];
          if (fabs(piv0) < small) piv0 = copysign(small, piv0);
          v /= piv0;
          z[i] = v;
          mx = fmax(mx, fabs(v));
          if (mx > 1e150) {  // rescale (dlagts overflow guard)
            for (int k = i; k < n; ++k) z[k] *= 1e-150;
            mx *= 1e-150;
            v *= 1e-150;
            z1 *= 1e-150;
          }
          z2 = z1;
          z1 = v;
        }
        // reorthogonalise against the cluster's earlier (final) members, then normalise
        for (int o = p; o < m; ++o) {
          const double* zo = J.Z + (size_t)o * J.ldz;
          double a0 = 0.0, a1 = 0.0;
          int i = 0;
          for (; i + 1 < n; i += 2) {
            a0 = fma(zo[i], z[i], a0);
            a1 = fma(zo[i + 1], z[i + 1], a1);
          }
          if (i < n) a0 = fma(zo[i], z[i], a0);
          const double dotp = a0 + a1;
          for (i = 0; i < n; ++i) z[i] = fma(-dotp, zo[i], z[i]);
        }
        double a0 = 0.0, a1 = 0.0;
        int i = 0;
        for (; i + 1 < n; i += 2) {
          a0 = fma(z[i], z[i], a0);
          a1 = fma(z[i + 1], z[i + 1], a1);
        }
        if (i < n) a0 = fma(z[i], z[i], a0);
        const double nrm = sqrt(a0 + a1);
        const double sc = nrm > 0.0 ? 1.0 / nrm : 0.0;
        for (i = 0; i < n; ++i) z[i] *= sc;
      }
    }
  }
}

__global__ void k_clusters(const TriDev* __restrict__ jobs) {
  __shared__ double red[8];
  __shared__ int s_cl[2];
  const TriDev J = jobs[blockIdx.x];
  const int n = J.n, nv = J.nvec, tid = threadIdx.x;
  if (n < 2 || nv < 2) return;
  double* u1 = J.scr;
  double* u2 = J.scr + n;
  double* u3 = J.scr + 2 * n;
  double* lm = J.scr + 3 * n;
  int* piv = reinterpret_cast<int*>(J.scr + 4 * n);
  const double tn = tnorm_of(J.d, J.e, n);
  const double tol = kClusterTol * tn;
  const double small = DBL_EPSILON * tn + kPivmin;
  auto bsum = [&](double v) {
    const int lane = tid & 31, warp = tid >> 5;
    v = wsum(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double a = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a += red[w];
    return a;
  };
  // (clusters of <= kSmallCluster vectors and broken-down single vectors were
  // done by k_clusters_small when the problem has enough of them)
  const bool threads_took_small = count_small_clusters(J, tol) >= kMinThreadClusters;
  int p = 0;
  while (p < nv) {
    // cluster [p, q): consecutive gaps below tol
    int q = p + 1;
    while (q < n && J.w[q] - J.w[q - 1] < tol) ++q;
    const int qend = min(q, nv);
    if (qend - p > kSmallCluster || (!threads_took_small && (qend - p >= 2 || J.wu[p] != 0.0))) {
      for (int m = p; m < qend; ++m) {
        // separate equal eigenvalues slightly so the factorisations differ (dstein's pertol)
        double lam = J.w[m];
        if (m > p && lam - J.w[m - 1] < 10.0 * DBL_EPSILON * tn) lam = J.w[m - 1] + 10.0 * DBL_EPSILON * tn * (m - p);
        if (tid == 0) {  // LU of T - lam with partial pivoting (banded, 3 diagonals of U)
          double r0 = J.d[0] - lam, r1 = (n > 1) ? J.e[0] : 0.0, r2 = 0.0;
          for (int i = 0; i < n - 1; ++i) {
            const double n0 = J.e[i], n1 = J.d[i + 1] - lam, n2 = (i + 1 < n - 1) ? J.e[i + 1] : 0.0;
            if (fabs(r0) >= fabs(n0)) {
              const double l = (r0 != 0.0) ? n0 / r0 : 0.0;
              u1[i] = (r0 != 0.0) ? r0 : small;
              u2[i] = r1;
              u3[i] = r2;
              lm[i] = l;
              piv[i] = 0;
              r0 = n1 - l * r1;
              r1 = n2 - l * r2;
              r2 = 0.0;
            } else {
              const double l = r0 / n0;
              u1[i] = n0;
              u2[i] = n1;
              u3[i] = n2;
              lm[i] = l;
              piv[i] = 1;
              r0 = r1 - l * n1;
              r1 = r2 - l * n2;
              r2 = 0.0;
            }
          }
          u1[n - 1] = (r0 != 0.0) ? r0 : small;
        }
        double* z = J.Z + (size_t)m * J.ldz;
        // deterministic start vector
        for (int i = tid; i < n; i += blockDim.x) {
          unsigned long long h = (unsigned long long)(i + 1) * 0x9E3779B97F4A7C15ull + (unsigned long long)(m + 1);
          h ^= h >> 31;
          h *= 0xBF58476D1CE4E5B9ull;
          h ^= h >> 29;
          z[i] = double(h >> 11) * 0x1.0p-53 - 0.5;
        }
        __syncthreads();
        for (int it = 0; it < 4; ++it) {
          if (tid == 0) {  // solve (T - lam) x = z in place: P L U
            for (int i = 0; i < n - 1; ++i) {
              if (piv[i]) {
                const double t = z[i];
                z[i] = z[i + 1];
                z[i + 1] = t;
              }
              z[i + 1] -= lm[i] * z[i];
            }
            double mx = 0.0;
            for (int i = n - 1; i >= 0; --i) {
              double v = z[i];
              if (i + 1 < n) v -= u2[i] * z[i + 1];
              if (i + 2 < n) v -= u3[i] * z[i + 2];
              double piv0 = u1[i];
              if (fabs(piv0) < small) piv0 = copysign(small, piv0);
              v /= piv0;
              z[i] = v;
              mx = fmax(mx, fabs(v));
              if (mx > 1e150) {  // rescale (dlagts overflow guard)
                for (int t = i; t < n; ++t) z[t] *= 1e-150;
                mx *= 1e-150;
              }
            }
          }
          __syncthreads();
          // reorthogonalise against the cluster's earlier (final) members, then normalise
          for (int o = p; o < m; ++o) {
            const double* zo = J.Z + (size_t)o * J.ldz;
            double a = 0.0;
            for (int i = tid; i < n; i += blockDim.x) a = fma(zo[i], z[i], a);
            const double dotp = bsum(a);
            for (int i = tid; i < n; i += blockDim.x) z[i] = fma(-dotp, zo[i], z[i]);
            __syncthreads();
          }
          double a = 0.0;
          for (int i = tid; i < n; i += blockDim.x) a = fma(z[i], z[i], a);
          const double nrm = sqrt(bsum(a));
          const double s = nrm > 0.0 ? 1.0 / nrm : 0.0;
          for (int i = tid; i < n; i += blockDim.x) z[i] *= s;
          __syncthreads();
        }
      }
    }
    if (tid == 0) s_cl[0] = q;
    __syncthreads();
    p = s_cl[0];
    __syncthreads();
  }
}

// Newton-Schulz orthogonalisation of column windows of Z: Z_w <- Z_w (3I - G)/2
// with G = Z_w^T Z_w.  The twisted / inverse-iteration vectors each have a
// residual ~ eps ||T||, and the off-diagonal of G pairs vectors i, j with
// ~eps ||T|| / |lam_i - lam_j|, so the correction mixes a vector only with
// close eigenvalues and keeps every residual ~ eps ||T|| while the window
// becomes orthonormal (two steps: 1e-6 -> 1e-12 -> rounding).  Windows of
// consecutive eigenvalues, two overlapping passes (offset W / 2).
__global__ void k_ns_h(int count, const int* __restrict__ wsz, int W, double* __restrict__ G) {
  const int q = blockIdx.y;
  if (q >= count) return;
  const int m = wsz[q];
  double* g = G + (size_t)q * W * W;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m * m; t += gridDim.x * blockDim.x) {
    const int i = t % m, j = t / m;
    g[i + (size_t)j * W] = ((i == j) ? 1.5 : 0.0) - 0.5 * g[i + (size_t)j * W];
  }
}

__global__ void k_copy_cols(int count, const double* const* __restrict__ src, double* const* __restrict__ dst,
                            const int* __restrict__ rows, const int* __restrict__ cols, const int* __restrict__ lds,
                            const int* __restrict__ ldd) {
  const int q = blockIdx.y;
  const long long cnt = (long long)rows[q] * cols[q];
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < cnt; t += (long long)gridDim.x * blockDim.x) {
    const int i = int(t % rows[q]), j = int(t / rows[q]);
    dst[q][i + (size_t)j * ldd[q]] = src[q][i + (size_t)j * lds[q]];
  }
}

// ---------------------------------------------------------------------------
// 3. Back-transformation helpers: the clean panel V_p (rows k0 .. n-1,
// column jj holds the reflector of column k0 + jj: zero above row k0 + jj + 1).
constexpr int kBT = 2 * kNB;  // reflectors per back-transformation block (two panels)

__global__ void k_panel_v(const EigDev* __restrict__ jobs, int k0, double* __restrict__ vbuf, long long vstride) {
  const EigDev J = jobs[blockIdx.y];
  if (k0 >= J.n - 1) return;
  const int jmax = min(kBT, J.n - 1 - k0);
  const int m = J.n - k0;
  double* out = vbuf + blockIdx.y * vstride;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * kBT;
       t += (long long)gridDim.x * blockDim.x) {
    const int r = int(t % m), jj = int(t / m);
    double v = 0.0;
    if (jj < jmax && r >= jj + 1) v = J.A[(k0 + r) + (size_t)(k0 + jj) * J.ld];
    out[r + (size_t)jj * J.ld] = v;
  }
}

// T of a block of kBT reflectors (dlarft, forward, columnwise) from the Gram
// matrix G = V^T V and the taus: T(c, c) = tau_c,
// T(0:c, c) = -tau_c T(0:c, 0:c) G(0:c, c).  One CTA per problem.
__global__ void k_larft(const EigDev* __restrict__ jobs, int k0, const double* __restrict__ gram,
                        double* __restrict__ tbig) {
  extern __shared__ double msm[];
  double* T = msm;               // kBT x kBT
  double* h = msm + kBT * kBT;   // kBT
  const EigDev J = jobs[blockIdx.x];
  if (k0 >= J.n - 1) return;
  const int nr = min(kBT, J.n - 1 - k0);  // reflectors in this block
  const double* G = gram + (size_t)blockIdx.x * kBT * kBT;  // read from L2
  for (int t = threadIdx.x; t < kBT * kBT; t += blockDim.x) T[t] = 0.0;
  __syncthreads();
  for (int c = 0; c < nr; ++c) {
    const double tau = J.tau[k0 + c];
    // h(p) = sum_{q = p..c-1} T(p, q) G(q, c)
    for (int p = threadIdx.x; p < c; p += blockDim.x) {
      double a = 0.0;
      for (int q = p; q < c; ++q) a = fma(T[p + q * kBT], G[q + c * kBT], a);
      h[p] = a;
    }
    __syncthreads();
    for (int p = threadIdx.x; p < c; p += blockDim.x) T[p + c * kBT] = -tau * h[p];
    if (threadIdx.x == 0) T[c + c * kBT] = tau;
    __syncthreads();
  }
  double* out = tbig + (size_t)blockIdx.x * kBT * kBT;
  for (int t = threadIdx.x; t < kBT * kBT; t += blockDim.x) out[t] = T[t];
}

int rows_per_thread(int nmax) {
  const int R = (nmax + kLT - 1) / kLT;  // n <= 5,760
  return R <= 1 ? 1 : R <= 2 ? 2 : R <= 4 ? 4 : R <= 8 ? 8 : R <= 11 ? 11 : R <= 12 ? 12 : -1;
}

template <int R>
void launch_latrd(Ctx& c, const EigDev* jobs, int count, int k0, int L, int nslot, size_t smem,
                  unsigned long long* prof) {
  ensure_dyn_smem((const void*)k_latrd<R>, smem);
  k_latrd<R><<<count, kLThreads, smem, c.stream>>>(jobs, k0, L, nslot, prof, int(c.opt("eig_probe", 0)));
  ++c.launches;
  check_launch("latrd");
}

// one panel in split form: (finish column jj - 1, start column jj), product of column jj, ...
template <int R>
void launch_panel_split(Ctx& c, const EigDev* jobs, int count, int k0, int C, int L, int nslot, size_t smem,
                        double* ypart) {
  ensure_dyn_smem((const void*)k_symv_part<R>, smem);
  ensure_dyn_smem((const void*)k_col_step<R>, size_t(L) * 8);
  for (int jj = 0; jj <= kNB; ++jj) {
    k_col_step<R><<<count, kLThreads, size_t(L) * 8, c.stream>>>(jobs, k0, jj, C, L, ypart);
    if (jj < kNB) k_symv_part<R><<<count * C, kLThreads, smem, c.stream>>>(jobs, k0, jj, C, L, nslot, ypart);
  }
  c.launches += 2 * kNB + 1;
  check_launch("latrd (split)");
}

}  // namespace

// jobs: A (n x n, ld, lower), w (n eigenvalues ascending), Z (n x nvec, ldz):
// the eigenvectors of the nvec smallest eigenvalues.  A is destroyed.
void eig_batched(Ctx& c, const std::vector<SyevJob>& jobs_in, const std::function<int(int, const double*)>& pick) {
  std::vector<SyevJob> jobs = jobs_in;
  const int J = int(jobs.size());
  if (J == 0) return;
  int nmax = 0, ldmax = 0;
  for (const auto& j : jobs) {
    nmax = std::max(nmax, j.n);
    ldmax = std::max(ldmax, j.ld);
    if (j.ld % 4 || j.ldz % 2) c.fail(AWG_E_ARG, "eig: leading dimensions must be multiples of 4 (A) and 2 (Z)");
  }
  const int R = rows_per_thread(nmax);
  if (R < 0) c.fail(AWG_E_ARG, "eig: matrix larger than 5,760 rows");
  // ---- workspace
  const int npan = (nmax - 1 + kNB - 1) / kNB;
  std::vector<long long> off(J + 1, 0);
  DArr<double> vw, bt, dd, ee, tt, wu, scr, vbuf, xb, xb2;
  vw.alloc(size_t(J) * ldmax * 2 * kNB);
  bt.alloc(size_t(J) * 2 * kNB * ldmax);
  dd.alloc(size_t(J) * ldmax);
  ee.alloc(size_t(J) * ldmax);
  tt.alloc(size_t(J) * ldmax);
  wu.alloc(size_t(J) * ldmax);
  scr.alloc(size_t(J) * 5 * ldmax);
  ee.zero(c.stream);
  std::vector<EigDev> ed(J);
  std::vector<TriDev> td(J);
  int nvmax = 0;
  for (int q = 0; q < J; ++q) {
    const SyevJob& s = jobs[q];
    ed[q] = EigDev{s.A, vw.p + size_t(q) * ldmax * 2 * kNB, bt.p + size_t(q) * 2 * kNB * ldmax, dd.p + size_t(q) * ldmax,
                   ee.p + size_t(q) * ldmax, tt.p + size_t(q) * ldmax, s.n, s.ld};
    // the panel buffers use the problem's own ld (their row stride); ld <= ldmax
    td[q] = TriDev{ed[q].d, ed[q].e, s.w, wu.p + size_t(q) * ldmax, s.Z, scr.p + size_t(q) * 5 * ldmax, s.n, s.ldz,
                   s.nvec};
    nvmax = std::max(nvmax, s.nvec);
  }
  DArr<EigDev> d_ed;
  DArr<TriDev> d_td;
  d_ed.upload(ed, c.stream);
  d_td.upload(td, c.stream);

  // phase timing on stderr with option verbose >= 1
  const bool verbose = c.opt("verbose", 0) >= 1;
  double tph = 0.0;
  auto phase = [&](const char* what) {
    if (!verbose) return;
    AWG_CUDA(cudaStreamSynchronize(c.stream));
    const double t = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    if (tph > 0.0) std::fprintf(stderr, "[awg eig] %d problems (n <= %d): %s %.1f ms\n", J, nmax, what, t - tph);
    tph = t;
  };
  phase("start");
  // ---- 1. tridiagonalisation
  const int L = round_up(ldmax, 2);
  const int nslot = int(std::min<size_t>(8, (kLatrdSmemCap - size_t(L) * 8) / (size_t(kTile) * 8)));  // <= 8 mbarriers
  if (nslot < 2) c.fail(AWG_E_ARG, "eig: matrix too large for the shared-memory ring");
  const size_t smem = size_t(nslot) * kTile * 8 + size_t(L) * 8;
  DArr<unsigned long long> prof;
  if (c.opt("verbose", 0) >= 2) {
    prof.alloc(4);
    prof.zero(c.stream);
  }
  // Split form (1b) by default: the symmetric products of one column step run
  // as J C CTAs in one launch (measured: 5.9 TB/s at 128 CTAs, 91% of the copy
  // peak, where k_latrd's one CTA per problem leaves SMs idle below 148
  // problems and runs 216 problems as 148 + 68).  C: the largest count <= 16
  // whose last wave is >= 95% full (else the fullest).  Option eig_split = 0
  // keeps one CTA per problem (k_latrd), k >= 1 forces C = k.
  int C = 1;
  {
    double best = 0.0;
    for (int cc = 1; cc <= 16; ++cc) {
      const double waves = double(J) * cc / c.sm_count;
      const double eff = waves / std::ceil(waves);
      if (eff >= 0.95 || eff > best + 1e-9) {
        if (eff >= 0.95 || best < 0.95) C = cc;
        best = std::max(best, eff);
      }
    }
  }
  const bool split_form = c.opt("eig_split", -1) != 0;
  if (c.opt("eig_split", -1) > 0) C = int(std::min(16LL, c.opt("eig_split", -1)));
  DArr<double> ypart;
  if (split_form) ypart.alloc(size_t(J) * C * L);
  for (int k0 = 0; k0 < nmax - 1; k0 += kNB) {
    if (split_form) {
      switch (R) {
        case 1: launch_panel_split<1>(c, d_ed.p, J, k0, C, L, nslot, smem, ypart.p); break;
        case 2: launch_panel_split<2>(c, d_ed.p, J, k0, C, L, nslot, smem, ypart.p); break;
        case 4: launch_panel_split<4>(c, d_ed.p, J, k0, C, L, nslot, smem, ypart.p); break;
        case 8: launch_panel_split<8>(c, d_ed.p, J, k0, C, L, nslot, smem, ypart.p); break;
        case 11: launch_panel_split<11>(c, d_ed.p, J, k0, C, L, nslot, smem, ypart.p); break;
        default: launch_panel_split<12>(c, d_ed.p, J, k0, C, L, nslot, smem, ypart.p); break;
      }
    } else
    switch (R) {
      case 1: launch_latrd<1>(c, d_ed.p, J, k0, L, nslot, smem, prof.p); break;
      case 2: launch_latrd<2>(c, d_ed.p, J, k0, L, nslot, smem, prof.p); break;
      case 4: launch_latrd<4>(c, d_ed.p, J, k0, L, nslot, smem, prof.p); break;
      case 8: launch_latrd<8>(c, d_ed.p, J, k0, L, nslot, smem, prof.p); break;
      case 11: launch_latrd<11>(c, d_ed.p, J, k0, L, nslot, smem, prof.p); break;
      default: launch_latrd<12>(c, d_ed.p, J, k0, L, nslot, smem, prof.p); break;
    }
    // A22 -= V W^T + W V^T on rows / columns >= k1 (lower tiles)
    std::vector<GemmDesc> pd;
    for (int q = 0; q < J; ++q) {
      const int n = jobs[q].n;
      if (k0 >= n - 1) continue;
      const int k1 = k0 + std::min(kNB, n - 1 - k0);
      const int m = n - k1;
      if (m <= 1) continue;  // the final panel (k1 = n - 1): k_last_diag
      pd.push_back({ed[q].VW + k1, ed[q].Bt + size_t(k1) * 2 * kNB, jobs[q].A + k1 + size_t(k1) * jobs[q].ld, m, m,
                    2 * kNB, jobs[q].ld, 2 * kNB, jobs[q].ld, 1, 1});
    }
    if (!pd.empty()) {
      GroupedGemm g;
      g.set(c, pd);
      g.run(c);
    }
  }
  k_last_diag<<<J, 32, 0, c.stream>>>(d_ed.p);
  ++c.launches;
  if (prof.p) {
    std::vector<unsigned long long> hp = prof.download(c.stream);
    std::fprintf(stderr, "[awg eig] k_latrd cycles summed over CTAs: column+reflector %.3e, symmetric product %.3e, w %.3e\n",
                 double(hp[0]), double(hp[1]), double(hp[2]));
  }
  phase("tridiagonalisation");

  // ---- 2. tridiagonal eigenvalues and vectors
  {
    const int per = 128;
    dim3 gb((nmax + per - 1) / per, J);
    const size_t sm = size_t(2) * nmax * 8;
    ensure_dyn_smem((const void*)k_bisect, sm);
    k_bisect<<<gb, per, sm, c.stream>>>(d_td.p, per);
    int pow2 = 1;
    while (pow2 < nmax) pow2 <<= 1;
    ensure_dyn_smem((const void*)k_sort_eigs, size_t(pow2) * 8);
    k_sort_eigs<<<J, 1024, size_t(pow2) * 8, c.stream>>>(d_td.p, pow2);
    if (pick) {  // the caller chooses how many eigenvectors each problem needs from its spectrum
      std::vector<double> hw(nmax);
      nvmax = 0;
      for (int q = 0; q < J; ++q) {
        AWG_CUDA(cudaMemcpyAsync(hw.data(), jobs[q].w, sizeof(double) * jobs[q].n, cudaMemcpyDeviceToHost, c.stream));
        AWG_CUDA(cudaStreamSynchronize(c.stream));
        const int nv = pick(q, hw.data());
        if (nv > jobs[q].nvec) c.fail(AWG_E_STATE, "eig: more eigenvectors requested than the output holds");
        jobs[q].nvec = nv;
        td[q].nvec = nv;
        nvmax = std::max(nvmax, nv);
      }
      d_td.upload(td, c.stream);
    }
    if (nvmax > 0) {
      dim3 gt((nvmax + per - 1) / per, J);
      k_twisted<<<gt, per, 0, c.stream>>>(d_td.p, per);
      // small clusters: thread per cluster, T threads per problem with an
      // interleaved LU scratch of 5 L doubles per thread (at most 8 GB in all)
      const size_t per_t = size_t(J) * 5 * ldmax * 8;
      size_t free_b = 0, tot_b = 0;
      AWG_CUDA(cudaMemGetInfo(&free_b, &tot_b));
      const size_t budget = std::min<size_t>(size_t(8) << 30, free_b / 4);
      const int T = int(std::max<size_t>(32, std::min<size_t>(1024, budget / per_t / 32 * 32)));
      DArr<double> cscr;
      cscr.alloc(size_t(J) * 5 * ldmax * T);
      k_clusters_small<<<dim3((T + 63) / 64, J), 64, 0, c.stream>>>(d_td.p, T, ldmax, cscr.p);
      k_clusters<<<J, 256, 0, c.stream>>>(d_td.p);
      AWG_CUDA(cudaStreamSynchronize(c.stream));  // cscr goes out of scope
    }
    c.launches += 5;
    check_launch("tridiagonal eigensolver");
  }
  phase("tridiagonal eigenpairs");
  if (nvmax > 1) {
    constexpr int W = 256;
    DArr<double> G, tmp;
    G.alloc(size_t(J) * W * W);
    tmp.alloc(size_t(J) * ldmax * W);
    for (int pass = 0; pass < 2; ++pass) {
      const int off = pass ? W / 2 : 0;
      for (int w0 = off; w0 < nvmax; w0 += W) {
        std::vector<GemmDesc> pg, pz;
        std::vector<int> wsz(J, 0), rows(J, 0), cols(J, 0), lds(J, 0), ldd(J, 0);
        std::vector<double*> src(J, nullptr), dst(J, nullptr);
        for (int q = 0; q < J; ++q) {
          const SyevJob& sj = jobs[q];
          const int m = std::min(W, sj.nvec - w0);
          if (m < 2 || (pass == 1 && sj.nvec <= W)) continue;  // a single window already covered all
          double* Zw = sj.Z + (size_t)w0 * sj.ldz;
          double* Gq = G.p + size_t(q) * W * W;
          double* Tq = tmp.p + size_t(q) * ldmax * W;
          wsz[q] = m;
          pg.push_back({Zw, Zw, Gq, m, m, sj.n, sj.ldz, sj.ldz, W, 0, 0});
          pz.push_back({Zw, Gq, Tq, sj.n, m, m, sj.ldz, W, sj.ldz, 0, 0});
          src[q] = Tq;
          dst[q] = Zw;
          rows[q] = sj.n;
          cols[q] = m;
          lds[q] = sj.ldz;
          ldd[q] = sj.ldz;
        }
        if (pg.empty()) continue;
        DArr<int> d_wsz, d_rows, d_cols, d_lds, d_ldd;
        DArr<double*> d_src, d_dst;
        d_wsz.upload(wsz, c.stream);
        d_rows.upload(rows, c.stream);
        d_cols.upload(cols, c.stream);
        d_lds.upload(lds, c.stream);
        d_ldd.upload(ldd, c.stream);
        d_src.upload(src, c.stream);
        d_dst.upload(dst, c.stream);
        GroupedGemm gg, gz;
        gg.set(c, pg, /*transpose_a=*/true);
        gz.set(c, pz);
        for (int step = 0; step < 2; ++step) {
          gg.run(c);                                                  // G = Z_w^T Z_w
          k_ns_h<<<dim3(64, J), 256, 0, c.stream>>>(J, d_wsz.p, W, G.p);  // H = (3I - G) / 2
          gz.run(c);                                                  // tmp = Z_w H
          k_copy_cols<<<dim3(256, J), 256, 0, c.stream>>>(J, d_src.p, d_dst.p, d_rows.p, d_cols.p, d_lds.p, d_ldd.p);
          c.launches += 2;
        }
        AWG_CUDA(cudaStreamSynchronize(c.stream));  // the per-window descriptor arrays go out of scope
      }
    }
    check_launch("newton-schulz");
  }
  phase("orthogonalisation");

  // ---- 3. Z <- Q Z, two-panel blocks in reverse order:
  //      Z(k0:n, :) -= V_b (T_b (V_b^T Z(k0:n, :)))   (K = 128 reflectors per GEMM)
  if (nvmax > 0) {
    vbuf.alloc(size_t(J) * ldmax * kBT);
    xb.alloc(size_t(J) * kBT * nvmax);
    xb2.alloc(size_t(J) * kBT * nvmax);
    DArr<double> gram, tbig;
    gram.alloc(size_t(J) * kBT * kBT);
    tbig.alloc(size_t(J) * kBT * kBT);
    const int nblk = (npan + 1) / 2;
    for (int blk = nblk - 1; blk >= 0; --blk) {
      const int k0 = blk * kBT;
      dim3 gv(64, J);
      k_panel_v<<<gv, 256, 0, c.stream>>>(d_ed.p, k0, vbuf.p, (long long)ldmax * kBT);
      ++c.launches;
      std::vector<GemmDesc> p0, p1, p2, p3;
      for (int q = 0; q < J; ++q) {
        const SyevJob& s = jobs[q];
        if (k0 >= s.n - 1 || s.nvec == 0) continue;
        const int m = s.n - k0;
        double* V = vbuf.p + size_t(q) * ldmax * kBT;
        double* X = xb.p + size_t(q) * kBT * nvmax;
        double* X2 = xb2.p + size_t(q) * kBT * nvmax;
        double* Zk = s.Z + k0;
        // G = V^T V
        p0.push_back({V, V, gram.p + size_t(q) * kBT * kBT, kBT, kBT, m, s.ld, s.ld, kBT, 0, 0});
        // X = V^T Z   (128 x nvec)
        p1.push_back({V, Zk, X, kBT, s.nvec, m, s.ld, s.ldz, kBT, 0, 0});
        // X2 = T X
        p2.push_back({tbig.p + size_t(q) * kBT * kBT, X, X2, kBT, s.nvec, kBT, kBT, kBT, kBT, 0, 0});
        // Z -= V X2
        p3.push_back({V, X2, Zk, m, s.nvec, kBT, s.ld, kBT, s.ldz, 1, 0});
      }
      if (p1.empty()) continue;
      GroupedGemm g0, g1, g2, g3;
      g0.set(c, p0, /*transpose_a=*/true);
      g0.run(c);
      const size_t msmem = size_t(kBT * kBT + kBT) * 8;
      ensure_dyn_smem((const void*)k_larft, msmem);
      k_larft<<<J, 256, msmem, c.stream>>>(d_ed.p, k0, gram.p, tbig.p);
      ++c.launches;
      g1.set(c, p1, /*transpose_a=*/true);
      g1.run(c);
      g2.set(c, p2);
      g2.run(c);
      g3.set(c, p3);
      g3.run(c);
    }
  }
  phase("back-transformation");
  AWG_CUDA(cudaStreamSynchronize(c.stream));
}

namespace {
__global__ void k_fill_sym(int n, int ld, int kind, unsigned long long seed, double* __restrict__ A) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)n * n) return;
  const int i = int(t % n), j = int(t / n);
  const int a = min(i, j), b = max(i, j);
  double v;
  if (kind == 3) {  // graph Laplacian of an m x m grid, edge weights 10^U(-3,3) (graded, clustered spectrum)
    const int m = int(llrint(sqrt(double(n))));
    auto wgt = [&](int p, int r) {  // weight of the grid edge {p, r}
      const int lo = min(p, r), hi = max(p, r);
      unsigned long long h = seed * 0x9E3779B97F4A7C15ull + (unsigned long long)lo * 0xD1B54A32D192ED03ull + hi;
      h ^= h >> 31;
      h *= 0xBF58476D1CE4E5B9ull;
      h ^= h >> 29;
      return pow(10.0, 6.0 * (double(h >> 11) * 0x1.0p-53) - 3.0);
    };
    const int ax = a % m, ay = a / m, bx = b % m, by = b / m;
    if (a == b) {
      v = 1e-3;
      if (ax > 0) v += wgt(a, a - 1);
      if (ax < m - 1) v += wgt(a, a + 1);
      if (ay > 0) v += wgt(a, a - m);
      if (ay < m - 1) v += wgt(a, a + m);
    } else {
      v = ((ay == by && bx - ax == 1) || (ax == bx && by - ay == 1)) ? -wgt(a, b) : 0.0;
    }
  } else if (kind == 1) {  // 5-point Laplacian on an m x m grid
    const int m = int(llrint(sqrt(double(n))));
    const int ax = a % m, ay = a / m, bx = b % m, by = b / m;
    v = (a == b) ? 4.0 : ((ay == by && bx - ax == 1) || (ax == bx && by - ay == 1)) ? -1.0 : 0.0;
  } else {
    unsigned long long h = seed + (unsigned long long)a * 0x9E3779B97F4A7C15ull + (unsigned long long)b * 0xD1B54A32D192ED03ull;
    h ^= h >> 31;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 29;
    v = double(h >> 11) * 0x1.0p-53 - 0.5;
    if (kind == 2 && a == b) v += 1e-6 * pow(1e6, double(a) / n) * n;
  }
  A[i + (size_t)j * ld] = v;
}
__global__ void k_maxabs_diff(long long cnt, const double* __restrict__ a, const double* __restrict__ b,
                              unsigned long long* __restrict__ out) {
  double m = 0.0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < cnt; t += (long long)gridDim.x * blockDim.x)
    m = fmax(m, fabs(a[t] - (b ? b[t] : 0.0)));
  atomicMax(out, __double_as_longlong(m));
}
// R = A Z - Z diag(w), column-scaled residual; and G = Z^T Z - I
__global__ void k_resid_prep(int n, int ld, const double* __restrict__ w, double* __restrict__ AZ,
                             const double* __restrict__ Z, double* __restrict__ G) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)n * n) return;
  const int i = int(t % n), j = int(t / n);
  AZ[i + (size_t)j * ld] -= w[j] * Z[i + (size_t)j * ld];
  if (i == j) G[i + (size_t)j * ld] -= 1.0;
}
}  // namespace

// Check / benchmark hook (awg_bench_eig): `count` seeded symmetric matrices
// of order n — kind 0: random entries; kind 1: the 5-point Laplacian of an
// m x m grid (n = m^2; exactly repeated eigenvalues); kind 2: random with a
// graded spectrum; kind 3: weighted grid Laplacian, weights 10^U(-3,3) — through eig_batched, against cuSOLVER Dsyevd on the same
// matrices.  out: [0] max |w - w_ref| / ||A||, [1] max ||A z - w z|| / ||A||,
// [2] max |Z^T Z - I|, [3] ms eig_batched, [4] ms cuSOLVER (all count).
void eig_check(Ctx& c, int n, int count, int kind, unsigned long long seed, double* out) {
  const int ld = round_up(n, 4);
  const size_t blk = size_t(ld) * n;
  DArr<double> A0, A, Z, w, wref, AZ, G;
  A0.alloc(blk * count);
  A.alloc(blk * count);
  Z.alloc(blk * count);
  w.alloc(size_t(n) * count);
  wref.alloc(size_t(n) * count);
  AZ.alloc(blk);
  G.alloc(blk);
  A0.zero(c.stream);
  for (int q = 0; q < count; ++q)
    k_fill_sym<<<int(((long long)n * n + 255) / 256), 256, 0, c.stream>>>(n, ld, kind, seed + q, A0.p + blk * q);
  AWG_CUDA(cudaMemcpyAsync(A.p, A0.p, sizeof(double) * blk * count, cudaMemcpyDeviceToDevice, c.stream));
  std::vector<SyevJob> jobs;
  for (int q = 0; q < count; ++q) jobs.push_back({A.p + blk * q, n, ld, w.p + size_t(n) * q, Z.p + blk * q, ld, n});
  cudaEvent_t e0, e1;
  AWG_CUDA(cudaEventCreate(&e0));
  AWG_CUDA(cudaEventCreate(&e1));
  AWG_CUDA(cudaEventRecord(e0, c.stream));
  eig_batched(c, jobs, nullptr);
  AWG_CUDA(cudaEventRecord(e1, c.stream));
  AWG_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  AWG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  out[3] = ms;
  // reference: cuSOLVER on copies
  cusolverDnHandle_t h;
  cublasHandle_t bh;
  if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS || cublasCreate(&bh) != CUBLAS_STATUS_SUCCESS)
    c.fail(AWG_E_CUDA, "eig_check: library handles");
  cusolverDnSetStream(h, c.stream);
  cublasSetStream(bh, c.stream);
  int lw = 0;
  cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A0.p, ld, wref.p, &lw);
  DArr<double> work;
  DArr<int> info;
  work.alloc(size_t(lw) + 1);
  info.alloc(1);
  DArr<double> Aref;
  Aref.alloc(blk);
  AWG_CUDA(cudaEventRecord(e0, c.stream));
  for (int q = 0; q < count; ++q) {
    AWG_CUDA(cudaMemcpyAsync(Aref.p, A0.p + blk * q, sizeof(double) * blk, cudaMemcpyDeviceToDevice, c.stream));
    cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, Aref.p, ld, wref.p + size_t(n) * q, work.p,
                     lw, info.p);
  }
  AWG_CUDA(cudaEventRecord(e1, c.stream));
  AWG_CUDA(cudaEventSynchronize(e1));
  AWG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  out[4] = ms;
  // errors
  DArr<unsigned long long> mx;
  mx.alloc(4);
  mx.zero(c.stream);
  double anorm = 0.0;
  {
    std::vector<double> hw = wref.download(c.stream);
    for (double v : hw) anorm = std::max(anorm, std::fabs(v));
  }
  k_maxabs_diff<<<256, 256, 0, c.stream>>>((long long)n * count, w.p, wref.p, mx.p);
  const double one = 1.0, zero = 0.0;
  for (int q = 0; q < count; ++q) {
    const double* Aq = A0.p + blk * q;
    const double* Zq = Z.p + blk * q;
    cublasDsymm(bh, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, n, n, &one, Aq, ld, Zq, ld, &zero, AZ.p, ld);
    cublasDgemm(bh, CUBLAS_OP_T, CUBLAS_OP_N, n, n, n, &one, Zq, ld, Zq, ld, &zero, G.p, ld);
    k_resid_prep<<<int(((long long)n * n + 255) / 256), 256, 0, c.stream>>>(n, ld, w.p + size_t(n) * q, AZ.p, Zq, G.p);
    k_maxabs_diff<<<256, 256, 0, c.stream>>>((long long)blk, AZ.p, nullptr, mx.p + 1);
    k_maxabs_diff<<<256, 256, 0, c.stream>>>((long long)blk, G.p, nullptr, mx.p + 2);
  }
  std::vector<unsigned long long> hm = mx.download(c.stream);
  double v[3];
  for (int i = 0; i < 3; ++i) std::memcpy(&v[i], &hm[i], 8);
  out[0] = v[0] / std::max(anorm, 1e-300);
  out[1] = v[1] / std::max(anorm, 1e-300);
  out[2] = v[2];
  cusolverDnDestroy(h);
  cublasDestroy(bh);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

}  // namespace awgb
