// Apply-path kernels of the AWG preconditioner (sm_100a, fp64, HBM-bound).
//
// Every kernel takes a `gate` pointer: when non-null and *gate != 0 the kernel
// returns immediately.  The PCG driver points it at its device-side `done`
// flag, so iterations can be enqueued ahead of the host's convergence check
// without changing any state after the stopping rule fired.
//
// Summation-order notes (parity): the CSR SpMV accumulates in ascending
// column order with separately rounded multiply and add exactly like the
// reference build of sparse.cpp:49-56 (bit-identical results); the
// prolongation sums subdomain contributions in ascending s like
// OneLevel::apply (preconditioner.cpp:37-55).  Dense dot products use
// fixed-shape warp trees (deterministic, not sequential): the parity bar for
// the applies is 1e-11 relative.
#include <cublas_v2.h>

#include <algorithm>
#include <cstdlib>

#include "awg_internal.cuh"
#include "pcg_device.cuh"

namespace awgb {
namespace {

constexpr int kThreads = 256;
constexpr int kCoarseStage = 4096;  // retained pivots staged in shared memory by k_coarse_solve (32 KB)

// first statement of every solve-path kernel: wait for the predecessor grid
// (programmatic dependent launch), then honour the device-side PCG gate
__device__ __forceinline__ bool gated(const int* gate) {
  pdl_wait();
  return gate != nullptr && *gate != 0;
}

// The short coarse-chain kernels (Z^T x / A- dots, K+ GEMV, Z c prolongation)
// release their dependents at entry: the successor grid is scheduled while
// this one runs and still waits in pdl_wait() for its completion and memory
// flush, so only the launch latency overlaps.  Off by default (option pdl_early=1):
// measured neutral on c2 (profiles/r01c/knobs_c2.json, 0.511 vs 0.509-0.513 ms
// per iteration), and the isolated Q / H3 applies slower by 1-2 us.
// Not used after the single-pass kernel: waiting successor CTAs next to the
// persistent local solve cost more than they hide.  Before it (the pt SpMV,
// AWG_PDL_LOCAL) the trigger lets the local solve's CTAs start their constant
// V^s copies while the SpMV drains.
__device__ __forceinline__ bool gated_early(const int* gate, int early) {
  if (early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  return gated(gate);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

int grid_for(const Ctx& c, long long work, int threads = kThreads) {
  long long g = (work + threads - 1) / threads;
  long long cap = (long long)c.sm_count * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return int(g);
}

// ---------------------------------------------------------------------------
// CSR SpMV  (sparse.cpp:49-56), thread per row, fused epilogues:
//   mode 0: y = A x      mode 1: y = add + A x   (A+ = A- x + A x, splitting.cpp:142-147)
//   mode 2: y = sub - (add + A x)                (projector transpose, coarse.cpp:180-191)
//   mode 3: y = sub - A x                        (Pi3^T, preconditioner.cpp:173-183)
__global__ void k_spmv(const int* __restrict__ gate, int n, const int* __restrict__ rp,
                       const int* __restrict__ ci, const double* __restrict__ va,
                       const double* __restrict__ x, double* __restrict__ y, int mode,
                       const double* __restrict__ add, const double* __restrict__ sub) {
  if (gated(gate)) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int k0 = rp[i], k1 = rp[i + 1];
    double acc = 0.0;
    // mul then add, not contracted: GCC emits vmulsd + vaddsd for this loop in
    // the reference build (sparse.cpp:53), so the result is bit-identical.
    acc = csr_row(ci, va, k0, k1, [&](int j) { return __ldg(x + j); });
    double out;
    if (mode == 0) out = acc;
    else if (mode == 1) out = add[i] + acc;
    else if (mode == 2) out = sub[i] - (add[i] + acc);
    else out = sub[i] - acc;
    y[i] = out;
  }
}

// Prolongation of a block-sparse combination, evaluated at dof i:
//   sum over subdomains s containing i (ascending) of sum_q coef[q] M_s(loc, col(q))
// — the k_block_combine + k_prolong pair fused.  G lanes share a row: lane t
// takes q = t, t + G, ... of every owner (G independent load streams instead
// of one serial chain of up to 4 x 48 loads); the lanes' sums meet in a fixed
// xor butterfly, so every lane holds the same, run-to-run identical value.
struct BlockSum {
  const int* own_off;
  const OwnEnt* ent;  // owner entries resolved against (M, moff, coff) — owner_tables()
  const int* ccol;    // column of coefficient q (nullptr: q - coff[s])
  const double* M;
  const double* coef;
  template <int G>
  __device__ __forceinline__ double at(int i, int t, bool active) const {
    double acc = 0.0;
    if (active) {
      for (int qo = own_off[i]; qo < own_off[i + 1]; ++qo) {
        const OwnEnt e = ent[qo];
        const double* Ms = M + e.mbase;
        const int L = e.L;
        const int q0 = e.q0, q1 = e.q1;
        double u0 = 0.0, u1 = 0.0;
        int q = q0 + t;
        for (; q + G < q1; q += 2 * G) {
          const int c0 = ccol ? ccol[q] : (q - q0);
          const int c1 = ccol ? ccol[q + G] : (q + G - q0);
          u0 = fma(coef[q], Ms[(size_t)c0 * L], u0);
          u1 = fma(coef[q + G], Ms[(size_t)c1 * L], u1);
        }
        if (q < q1) u0 = fma(coef[q], Ms[(size_t)(ccol ? ccol[q] : (q - q0)) * L], u0);
        acc += u0 + u1;
      }
    }
#pragma unroll
    for (int o = G / 2; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    return acc;
  }
};

// A+ x = A- x + A x with the A- prolongation fused (splitting.cpp:142-147):
//   mode 1: y = am + A x;  mode 2: y = sub - (am + A x)
template <int G>
__global__ void k_spmv_aplus(const int* __restrict__ gate, int n, const int* __restrict__ rp,
                             const int* __restrict__ ci, const double* __restrict__ va,
                             const double* __restrict__ x, double* __restrict__ y, int mode,
                             const double* __restrict__ sub, BlockSum am, int early) {
  if (gated_early(gate, early)) return;
  // G lanes per row; the loop runs warp-uniformly (the lanes meet in shuffles)
  const int t = threadIdx.x & (G - 1);
  const int stride = int((gridDim.x * (long long)blockDim.x) / G);
  for (int i = int((blockIdx.x * (long long)blockDim.x + threadIdx.x) / G);; i += stride) {
    const bool active = i < n;
    if (!__any_sync(0xffffffffu, active)) break;
    const double m = am.at<G>(i, t, active);
    if (active && t == 0) {
      double acc = 0.0;
      acc = csr_row(ci, va, rp[i], rp[i + 1], [&](int j) { return __ldg(x + j); });
      const double a = m + acc;
      y[i] = (mode == 1) ? a : sub[i] - a;
    }
  }
}

// Z c with the composition that consumes it fused into the epilogue (the
// k_axpby steps of TwoLevel::apply / AwgPreconditioner::apply, same operation
// order, so bit-identical to running them separately):
//   a == nullptr: y = Z c
//   a != nullptr: y = (a - Z c) + d           hybrid H2 (preconditioner.cpp:79-81)
//   e != nullptr: y = ((a - Z c) + d) + e     ... + W KW+ W^T x   (AD, :185-192)
struct Combine {
  const double* a;
  const double* d;
  const double* e;
  RzFuse rz;  // rz.st != nullptr: also <r, y> into the PCG state (the PCG's beta step)
};

template <int G>
__global__ void k_prolong_sum(const int* __restrict__ gate, int n, BlockSum bs, double* __restrict__ y,
                              Combine cb, int early) {
  if (gated_early(gate, early)) return;
  const int t = threadIdx.x & (G - 1);
  const int stride = int((gridDim.x * (long long)blockDim.x) / G);
  double rz = 0.0;
  for (int i = int((blockIdx.x * (long long)blockDim.x + threadIdx.x) / G);; i += stride) {
    const bool active = i < n;
    if (!__any_sync(0xffffffffu, active)) break;
    const double v = bs.at<G>(i, t, active);
    if (active && t == 0) {
      double out = v;
      if (cb.a) {
        out = (cb.a[i] - v) + cb.d[i];
        if (cb.e) out = out + cb.e[i];
      }
      y[i] = out;
      if (cb.rz.st) rz = fma(cb.rz.r[i], out, rz);
    }
  }
  // rz = <r, z> and the beta step (krylov.cpp:105-115), fused: k_pcg_rz's work
  if (cb.rz.st)
    pcgdev::grid_reduce(rz, cb.rz.part, cb.rz.count, [&](double v) { pcgdev::rz_finish(cb.rz.st, v, 0); });
}

// xs[p] = x[pidx[p]] (* scale[p])      restrict_to (splitting.cpp:220-223) and the D^s
// scaling of OneLevel::apply (preconditioner.cpp:48-49)
__global__ void k_gather(const int* __restrict__ gate, long long total, const int* __restrict__ pidx,
                         const double* __restrict__ x, const double* __restrict__ scale,
                         double* __restrict__ xs) {
  if (gated(gate)) return;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < total;
       p += (long long)gridDim.x * blockDim.x) {
    double v = __ldg(x + pidx[p]);
    if (scale) v *= scale[p];
    xs[p] = v;
  }
}

// y[i] = sum over subdomains s containing i (ascending s) of w[p(s,i)]
// (prolong_add, splitting.cpp:225-228, in OneLevel's ascending-s order)
__global__ void k_prolong(const int* __restrict__ gate, int n, const int* __restrict__ own_off,
                          const int* __restrict__ own_pos, const double* __restrict__ w,
                          double* __restrict__ y) {
  if (gated(gate)) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int q = own_off[i]; q < own_off[i + 1]; ++q) acc += w[own_pos[q]];
    y[i] = acc;
  }
}

// ---------------------------------------------------------------------------
// Batched NN local solve, first half (local_Aplus_pinv_apply, splitting.cpp:211-218,
// with OneLevel's restriction and D^s scaling, preconditioner.cpp:41-49, fused):
//   uh[p_s + j] = (V^s(:, j) . (D^s x[Omega^s])) / lambda_j   for j >= n_nonpos(s)
// One CTA per (s, column chunk); the scaled restriction is staged once in shared
// memory; one warp per column, 16-byte coalesced loads down the column, 4 loads
// in flight per lane.
// TRI = true: the AS / AS+ one-level (Cholesky factor form, preconditioner.cpp:43-46):
// V is U^s = L^-T (upper triangular, zeros below the diagonal stored), column j
// is read over rows 0..j only, no D^s and no eigenvalue division (lam = nullptr).
template <int NW, bool TRI>
__global__ void __launch_bounds__(NW * 32) k_nn_gemvT(const int* __restrict__ gate, const GemvTTask* __restrict__ tasks,
                                                   const double* __restrict__ V, const long long* __restrict__ voff,
                                                   const int* __restrict__ ns, const int* __restrict__ ld,
                                                   const long long* __restrict__ poff, const int* __restrict__ pidx,
                                                   const double* __restrict__ ds, const double* __restrict__ x,
                                                   const double* __restrict__ lam, double* __restrict__ uh) {
  if (gated(gate)) return;
  extern __shared__ double sx[];
  const GemvTTask t = tasks[blockIdx.x];
  const int s = t.s, n = ns[s], L = ld[s];
  const long long p0 = poff[s];
  for (int i = threadIdx.x; i < L; i += blockDim.x)
    sx[i] = (i < n) ? (ds ? __ldg(x + pidx[p0 + i]) * ds[p0 + i] : __ldg(x + pidx[p0 + i])) : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* Vs = V + voff[s];
  const double2* sx2 = reinterpret_cast<const double2*>(sx);
  for (int j = t.j0 + warp; j < t.j1; j += NW) {
    const int npair = TRI ? min(L >> 1, (j >> 1) + 1) : (L >> 1);
    const double2* col = reinterpret_cast<const double2*>(Vs + (size_t)j * L);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int q = lane;
    for (; q + 96 < npair; q += 128) {
      const double2 v0 = __ldcs(col + q), v1 = __ldcs(col + q + 32), v2 = __ldcs(col + q + 64),
                    v3 = __ldcs(col + q + 96);
      const double2 x0 = sx2[q], x1 = sx2[q + 32], x2 = sx2[q + 64], x3 = sx2[q + 96];
      a0 = fma(v0.x, x0.x, a0); a0 = fma(v0.y, x0.y, a0);
      a1 = fma(v1.x, x1.x, a1); a1 = fma(v1.y, x1.y, a1);
      a2 = fma(v2.x, x2.x, a2); a2 = fma(v2.y, x2.y, a2);
      a3 = fma(v3.x, x3.x, a3); a3 = fma(v3.y, x3.y, a3);
    }
    for (; q < npair; q += 32) {
      const double2 v0 = __ldcs(col + q);
      const double2 x0 = sx2[q];
      a0 = fma(v0.x, x0.x, a0); a0 = fma(v0.y, x0.y, a0);
    }
    const double sum = warp_sum((a0 + a1) + (a2 + a3));
    if (lane == 0) uh[p0 + j] = TRI ? sum : sum / lam[p0 + j];
  }
}

// Second half, split over column chunks: part[kc * P + p_s + i] =
//   sum_{j in chunk kc, j >= n_nonpos(s)} V^s(i, j) uh[p_s + j]
// One CTA per (s, 2*blockDim row panel, column chunk); each thread owns two
// adjacent rows (16-byte loads, a warp reads 512 contiguous bytes of a column
// per step), 8 column loads in flight per thread; the chunk of uh_s is staged
// in shared memory.  D^s and the chunk sum are applied by k_prolong_nn.
__global__ void __launch_bounds__(kThreads) k_nn_gemv(const int* __restrict__ gate, const GemvTask* __restrict__ tasks,
                                                   const double* __restrict__ V, const long long* __restrict__ voff,
                                                   const int* __restrict__ ns, const int* __restrict__ ld,
                                                   const long long* __restrict__ poff, long long P,
                                                   const double* __restrict__ uh, double* __restrict__ part) {
  if (gated(gate)) return;
  extern __shared__ double su[];
  const GemvTask t = tasks[blockIdx.x];
  const int s = t.s, n = ns[s], L = ld[s];
  const int j0 = t.j0, j1 = t.j1;
  const long long p0 = poff[s];
  for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) su[j - j0] = uh[p0 + j];
  __syncthreads();
  const int i = t.i0 + 2 * threadIdx.x;
  if (i >= n) return;
  const double* Vs = V + voff[s] + i;
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
  int j = j0;
  for (; j + 8 <= j1; j += 8) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(reinterpret_cast<const double2*>(Vs + (size_t)(j + u) * L));
#pragma unroll
    for (int u = 0; u < 8; u += 2) {
      const double c0 = su[j + u - j0], c1 = su[j + u + 1 - j0];
      a0 = fma(v[u].x, c0, a0);
      a1 = fma(v[u].y, c0, a1);
      b0 = fma(v[u + 1].x, c1, b0);
      b1 = fma(v[u + 1].y, c1, b1);
    }
  }
  for (; j < j1; ++j) {
    const double2 v0 = __ldcs(reinterpret_cast<const double2*>(Vs + (size_t)j * L));
    const double c0 = su[j - j0];
    a0 = fma(v0.x, c0, a0);
    a1 = fma(v0.y, c0, a1);
  }
  double* out = part + (size_t)t.kc * P + p0;
  out[i] = a0 + b0;
  if (i + 1 < n) out[i + 1] = a1 + b1;
}

// ---------------------------------------------------------------------------
// Single-pass local solve: y_s = sum_j V(:, j) (V(:, j) . xs) / lambda_j over the
// CTA's column range — the same V mask(1/lam) V^T product as gemvT + gemv, but
// each column (or column pair) is brought into shared memory ONCE by a TMA bulk
// copy (cp.async.bulk + mbarrier, up to kFusedMaxBuf buffers in flight) and
// used there for both the dot and the rank-1 update, so V^s is streamed from
// HBM once per apply instead of twice.  The restriction (D^s R^s x) and the
// partial y live in registers (rows tid + kFusedT * k, k < R).  The loops carry
// no bounds checks or branches (a branch per row made the first version
// latency-bound: ~1,900 cycles per column on the dependent chains, see
// profiles/README.md).  Partials land in the split-K layout of k_nn_gemv;
// k_prolong_nn sums them in fixed order.
// TRI: the AS / AS+ factor U^s = L^-T (no eigenvalue division, no D^s).
constexpr int kFusedT = 512;
constexpr int kFusedMaxBuf = 6;  // deepest copy pipeline
constexpr size_t kFusedSmemCap = size_t(224) * 1024;  // dynamic shared memory per CTA

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// In-kernel launch timer (live inside the timed solve; bench.py's roofline):
// tmr[0] earliest CTA start, tmr[1] latest CTA end, tmr[2] CTAs done,
// tmr[3] accumulated ns, tmr[4] launches.  The last CTA folds this launch's
// span (first CTA start -> last CTA end) into the total and re-arms.
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void kernel_timer_end(unsigned long long* tmr) {
  atomicMax(&tmr[1], globaltimer_ns());
  __threadfence();
  if (atomicAdd(&tmr[2], 1ull) == gridDim.x - 1) {
    __threadfence();
    const unsigned long long t0 = atomicAdd(&tmr[0], 0ull), t1 = atomicAdd(&tmr[1], 0ull);
    tmr[3] += t1 - t0;
    tmr[4] += 1;
    tmr[0] = ~0ull;
    tmr[1] = 0;
    tmr[2] = 0;
    __threadfence();
  }
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arm(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

// V^s is streamed once per apply and is far larger than L2: its lines are
// marked evict-first so the index arrays, coarse blocks and vectors of the
// small kernels around the local solve stay L2-resident across iterations
__device__ __forceinline__ unsigned long long l2_evict_first() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                          unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <bool TRI, int R, int CPB, bool HOLD>
__global__ void __launch_bounds__(kFusedT, 1) k_nn_fused(const int* __restrict__ gate, const GemvTask* __restrict__ tasks,
                                                         const double* __restrict__ V, const long long* __restrict__ voff,
                                                         const int* __restrict__ ns, const int* __restrict__ ld,
                                                         const long long* __restrict__ poff,
                                                         const int* __restrict__ pidx, const double* __restrict__ ds,
                                                         const double* __restrict__ x, const double* __restrict__ rlam,
                                                         long long P, double* __restrict__ part, int ntasks,
                                                         int* __restrict__ queue, const int* __restrict__ cta_off, int nbuf, int ldmax,
                                                         int smem_doubles, int prefetch, int prewait,
                                                         unsigned long long* __restrict__ tmr) {
  extern __shared__ __align__(128) double fsm[];
  __shared__ __align__(8) unsigned long long bar[kFusedMaxBuf];
  __shared__ double red[2][CPB][kFusedT / 32];
  __shared__ int s_task;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Rows are read without bounds checks (no branches in the hot loops): rows
  // past a column's end read the next column or the zeroed tail, which meet
  // xr = 0 in the dot and land in rows of yr that are never written out; TRI
  // masks by value.  So the whole buffer area starts finite.
  for (int i = tid; i < smem_doubles; i += kFusedT) fsm[i] = 0.0;
  if (tid == 0) {
    for (int b = 0; b < nbuf; ++b) mbar_init(&bar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // order the zero fill (generic proxy) before the first bulk copies (async proxy)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const size_t bstride = (size_t)CPB * ldmax;  // buffer b starts at fsm + b * bstride
  const unsigned long long pol = l2_evict_first();
  // Persistent CTAs (one per SM).  NN: CTA b runs its own static task range
  // [cta_off[b], cta_off[b + 1]) — equal byte shares, so no SM idles at the
  // end (profiles/r01e/knobs_static_c2.json); AS / AS+ and option fused_static=0
  // (cta_off == nullptr): column chunks pulled from an atomic queue.  The chunk -> partial-slot map
  // is fixed by the task list, so the result does not depend on which CTA ran
  // which chunk.  A step covers CPB columns; g counts
  // the steps this CTA has consumed: buffer g % nbuf, mbarrier parity
  // (g / nbuf) & 1.  One barrier per step: red is double-buffered, and the
  // buffer of the previous step is refilled right after the barrier.
  // Cross-task prefetch: thread 0 claims the CTA's NEXT task while the current
  // one runs and issues its first steps into the ring as soon as buffers free
  // up, so the copy pipeline does not drain at task boundaries (the global step
  // count g, buffer g % nbuf and parity (g / nbuf) & 1 simply run on).
  auto issue = [&](const double* Vs, int L, int j0, int j1, int p, unsigned gbase) {
    const int j = j0 + CPB * p;
    const int cols = min(CPB, j1 - j);
    const unsigned b = (gbase + p) % nbuf;
    if (!TRI) {
      const unsigned bytes = unsigned(cols) * unsigned(L) * 8u;
      mbar_arm(&bar[b], bytes);
      bulk_load(fsm + b * bstride, Vs + (size_t)j * L, bytes, &bar[b], pol);
    } else {
      // upper-triangular U^s: column c holds rows 0..c; copy an even row count
      unsigned rows[CPB], total = 0;
#pragma unroll
      for (int c = 0; c < CPB; ++c) {
        rows[c] = c < cols ? unsigned(min(L, (j + c + 2) & ~1)) : 0u;
        total += rows[c];
      }
      mbar_arm(&bar[b], total * 8u);
#pragma unroll
      for (int c = 0; c < CPB; ++c)
        if (rows[c])
          bulk_load(fsm + b * bstride + (size_t)c * L, Vs + (size_t)(j + c) * L, rows[c] * 8u, &bar[b], pol);
    }
  };
  unsigned g = 0;
  // static split: this CTA's own task range, no queue
  const int lim = cta_off ? cta_off[blockIdx.x + 1] : ntasks;
  // prewait (static split): V^s is constant, so the first task's first copies
  // are issued before griddepcontrol.wait — under the predecessor's early
  // trigger they land while it finishes.  A gated launch drains them first.
  __syncthreads();  // zero fill and barrier init before any copy
  int issued0 = 0;
  if (prewait && cta_off) {
    const int c0 = cta_off[blockIdx.x];
    if (c0 < lim) {
      const GemvTask t0 = tasks[c0];
      issued0 = min(nbuf, (t0.j1 - t0.j0 + CPB - 1) / CPB);
      if (tid == 0)
        for (int p = 0; p < issued0; ++p) issue(V + voff[t0.s], ld[t0.s], t0.j0, t0.j1, p, 0u);
    }
  }
  if (gated(gate)) {
    for (int b = 0; b < issued0; ++b) mbar_wait(&bar[b], 0);
    return;
  }
  if (tmr && tid == 0) atomicMin(&tmr[0], globaltimer_ns());
  if (tid == 0) s_task = cta_off ? cta_off[blockIdx.x] : atomicAdd(queue, 1);
  __syncthreads();
  int cur = s_task;
  // thread 0 only: steps of the current task already issued; the next task
  int pre = issued0, nxt = lim, pre_n = 0, nstep_n = 0, j0_n = 0, j1_n = 0, s_n = 0, L_n = 0, fstage = 0;
  const double* V_n = V;
  // the next task's descriptor is a chain of dependent loads (queue -> task ->
  // ld / voff): one link per step, so thread 0 never stalls the CTA for the
  // whole chain at once
  auto advance = [&]() {
    if (fstage == 0) {
      nxt = cta_off ? cur + 1 : atomicAdd(queue, 1);
      fstage = nxt < lim ? 1 : 3;
    } else if (fstage == 1) {
      const GemvTask tn = tasks[nxt];
      j0_n = tn.j0;
      j1_n = tn.j1;
      s_n = tn.s;
      nstep_n = (tn.j1 - tn.j0 + CPB - 1) / CPB;
      fstage = 2;
    } else if (fstage == 2) {
      L_n = ld[s_n];
      V_n = V + voff[s_n];
      fstage = 3;
    }
  };
  while (cur < lim) {
    const GemvTask t = tasks[cur];
    const int s = t.s, n = ns[s], L = ld[s];
    const long long p0 = poff[s];
    const double* Vs = V + voff[s];
    const int nstep = (t.j1 - t.j0 + CPB - 1) / CPB;
    if (tid == 0) {
      for (int p = pre; p < nbuf && p < nstep; ++p) issue(Vs, L, t.j0, t.j1, p, g);
      nxt = lim;
      pre_n = 0;
      fstage = 0;
    }
    double xr[R], yr[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int i = tid + k * kFusedT;
      double v = 0.0;
      if (i < n) v = TRI ? __ldg(x + pidx[p0 + i]) : __ldg(x + pidx[p0 + i]) * ds[p0 + i];
      xr[k] = v;
      yr[k] = 0.0;
    }
    for (int p = 0; p < nstep; ++p) {
      const int j = t.j0 + CPB * p;
      const unsigned gp = g + p;
      double rl[CPB];  // issued before the wait: off the post-barrier critical path
#pragma unroll
      for (int c = 0; c < CPB; ++c) rl[c] = (!TRI && j + c < t.j1) ? __ldg(rlam + p0 + j + c) : 0.0;
      mbar_wait(&bar[gp % nbuf], (gp / nbuf) & 1);
      const double* cb = fsm + (gp % nbuf) * bstride;
      // dots: two interleaved accumulators per column, fixed order.  HOLD: the
      // column values stay in registers for the update (shared memory is read
      // once per element instead of twice: the MIO pipe, not HBM, was the
      // throttle at power-capped SM clocks)
      double cv[HOLD ? CPB : 1][HOLD ? R : 1];
#pragma unroll
      for (int c = 0; c < CPB; ++c) {
        const double* col = cb + (size_t)c * L;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int k = 0; k < R; ++k) {
          double v = col[tid + k * kFusedT];
          if (TRI) v = (tid + k * kFusedT <= j + c) ? v : 0.0;
          if (HOLD) cv[HOLD ? c : 0][HOLD ? k : 0] = v;
          if (k & 1)
            a1 = fma(v, xr[k], a1);
          else
            a0 = fma(v, xr[k], a0);
        }
        const double acc = warp_sum(a0 + a1);
        if (lane == 0) red[gp & 1][c][warp] = acc;
      }
      __syncthreads();
      // the previous step's buffer is no longer read by anyone (with HOLD this
      // step's buffer is already consumed too: refill it now) — with this
      // task's next step, or past its end with the next task's
      if (tid == 0 && (HOLD || p >= 1)) {
        const int q = HOLD ? p + nbuf : p - 1 + nbuf;
        if (q < nstep) {
          issue(Vs, L, t.j0, t.j1, q, g);
        } else if (prefetch && fstage == 3 && nxt < lim && q - nstep == pre_n && pre_n < nstep_n) {
          issue(V_n, L_n, j0_n, j1_n, pre_n, g + nstep);
          ++pre_n;
        }
      }
      if (tid == 0) advance();
      // the 16 warp partials: lane l reads partial l & 15 (one shared load per
      // warp instead of 16 broadcast loads per thread), then an xor butterfly
      // over 16 lanes — the fixed tree ((r0+r8)+(r4+r12)) + ((r2+r10)+(r6+r14))
      // + ..., identical in every lane and run
      double d[CPB];
#pragma unroll
      for (int c = 0; c < CPB; ++c) {
        double a = red[gp & 1][c][lane & 15];
#pragma unroll
        for (int o = 8; o >= 1; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        const bool live = (j + c < t.j1);
        d[c] = live ? (TRI ? a : a * rl[c]) : 0.0;
      }
#pragma unroll
      for (int c = 0; c < CPB; ++c) {
        const double* col = cb + (size_t)c * L;
#pragma unroll
        for (int k = 0; k < R; ++k) {
          double v;
          if (HOLD) {
            v = cv[HOLD ? c : 0][HOLD ? k : 0];
          } else {
            v = col[tid + k * kFusedT];
            if (TRI) v = (tid + k * kFusedT <= j + c) ? v : 0.0;
          }
          yr[k] = fma(v, d[c], yr[k]);
        }
      }
    }
    double* out = part + (size_t)t.kc * P + p0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int i = tid + k * kFusedT;
      if (i < n) out[i] = yr[k];
    }
    g += nstep;
    // every thread is past this task's last buffer read before the next task's
    // remaining first steps are issued into it
    __syncthreads();
    if (tid == 0) {
      while (fstage < 3) advance();
      s_task = nxt;
      pre = pre_n;
    }
    __syncthreads();
    cur = s_task;
  }
  // the queue resets itself: the last CTA out (queue[1] counts finished CTAs,
  // each after its last queue[0] access) rewinds both counters for the next launch
  if (tid == 0 && atomicAdd(queue + 1, 1) == int(gridDim.x) - 1) {
    atomicExch(queue, 0);
    atomicExch(queue + 1, 0);
  }
  if (tmr && tid == 0) kernel_timer_end(tmr);
}

// y[i] = sum over s containing i (ascending s) of D^s_i * (sum_kc part[kc][p(s,i)])
template <int G>
__global__ void k_prolong_nn(const int* __restrict__ gate, int n, const int* __restrict__ own_off,
                             const int2* __restrict__ own_nkc, long long P, const double* __restrict__ part,
                             const double* __restrict__ ds, double* __restrict__ y) {
  if (gated(gate)) return;
  // G lanes per row split the chunk partials (kc = t, t + G, ...); fixed butterfly
  const int t = threadIdx.x & (G - 1);
  const int stride = int((gridDim.x * (long long)blockDim.x) / G);
  for (int i = int((blockIdx.x * (long long)blockDim.x + threadIdx.x) / G);; i += stride) {
    const bool active = i < n;
    if (!__any_sync(0xffffffffu, active)) break;
    double acc = 0.0;
    if (active) {
      for (int q = own_off[i]; q < own_off[i + 1]; ++q) {
        const int2 e = own_nkc[q];
        const int p = e.x, kcs = e.y;
        double w0 = 0.0, w1 = 0.0;
        int kc = t;
        for (; kc + G < kcs; kc += 2 * G) {
          w0 += part[(size_t)kc * P + p];
          w1 += part[(size_t)(kc + G) * P + p];
        }
        if (kc < kcs) w0 += part[(size_t)kc * P + p];
        const double w = w0 + w1;
        acc += ds ? w * ds[p] : w;
      }
    }
#pragma unroll
    for (int o = G / 2; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (active && t == 0) y[i] = acc;
  }
}



// ---------------------------------------------------------------------------
// A- x (splitting.cpp:119-140): per strictly negative mode (s,k):
//   c = (-lambda_k) * (v_k . x[Omega^s]);   u_s = sum_k c_k v_k;   y = sum_s R^s^T u_s
// (the dots are k_bs_gemvT below; the combination is fused into the consumer)
// u[p] = sum over the negative modes of s(p), ascending k, of c_k v_k[i]
// (Y-combine for Z c uses the same kernel on the Y blocks).
__global__ void k_block_combine(const int* __restrict__ gate, long long P, const int* __restrict__ psub,
                                const long long* __restrict__ poff, const int* __restrict__ coff,
                                const int* __restrict__ ccol, const double* __restrict__ M,
                                const long long* __restrict__ moff, const int* __restrict__ ld,
                                const double* __restrict__ coef, double* __restrict__ u) {
  if (gated(gate)) return;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < P;
       p += (long long)gridDim.x * blockDim.x) {
    const int s = psub[p];
    const int i = int(p - poff[s]);
    const double* Ms = M + moff[s] + i;
    const int L = ld[s];
    double acc = 0.0;
    for (int q = coff[s]; q < coff[s + 1]; ++q) {
      const int col = ccol ? ccol[q] : (q - coff[s]);
      acc = fma(coef[q], Ms[(size_t)col * L], acc);
    }
    u[p] = acc;
  }
}


// Block-sparse GEMV^T: out[q] = w[q] * sum_i M_s(i, col(q)) x[pidx_s[i]] for the
// columns q in [coff[s], coff[s+1]) of every subdomain s — Z^T x (Y_s blocks,
// coarse.cpp:136-141 + matvec_transpose) and the A- dots (V^s columns
// k < n_nonpos, splitting.cpp:124-132).  One CTA per (s, 512-row chunk,
// group of 8 columns): the gathered x rows sit in registers, the 16 column
// loads of a thread are all in flight at once (one memory round trip per CTA),
// per-warp sums meet in shared memory and per-chunk partials go to `part`; the
// last CTA of s (of nch[s] x its column groups) sums the chunks in chunk order
// (run-to-run identical, same order as before the column split).
constexpr int kBsCols = 8;
__global__ void __launch_bounds__(256) k_bs_gemvT(const int* __restrict__ gate, const int* __restrict__ task_s,
                                                  const int* __restrict__ task_c, const int* __restrict__ nch,
                                                  int maxch, const int* __restrict__ coff,
                                                  const int* __restrict__ ccol, const double* __restrict__ M,
                                                  const long long* __restrict__ moff, const int* __restrict__ ns,
                                                  const int* __restrict__ ld, const long long* __restrict__ poff,
                                                  const int* __restrict__ pidx, const double* __restrict__ x,
                                                  const double* __restrict__ w, double* __restrict__ part,
                                                  int* __restrict__ cnt, double* __restrict__ out, int early) {
  if (gated_early(gate, early)) return;
  __shared__ double red[8][kBsCols];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int s = task_s[blockIdx.x], ch = task_c[blockIdx.x];
  const int q0 = coff[s], nc = coff[s + 1] - q0;
  const int cb = blockIdx.y * kBsCols;
  if (cb >= nc) return;  // not counted: the arrival target is nch[s] x ceil(nc / 8)
  const int ncb = min(kBsCols, nc - cb);
  const int n = ns[s], L = ld[s];
  const int ia = ch * kBsRows + tid, ib = ia + 256;
  const long long p0 = poff[s];
  const double* Ms = M + moff[s];
  double va[kBsCols], vb[kBsCols];
#pragma unroll
  for (int u = 0; u < kBsCols; ++u) {
    const bool ok = u < ncb;
    const int col = ok ? (ccol ? ccol[q0 + cb + u] : cb + u) : 0;
    const double* m = Ms + (size_t)col * L;
    va[u] = (ok && ia < n) ? m[ia] : 0.0;
    vb[u] = (ok && ib < n) ? m[ib] : 0.0;
  }
  const double xa = ia < n ? __ldg(x + pidx[p0 + ia]) : 0.0;
  const double xb = ib < n ? __ldg(x + pidx[p0 + ib]) : 0.0;
#pragma unroll
  for (int u = 0; u < kBsCols; ++u) {
    const double a = warp_sum(fma(vb[u], xb, va[u] * xa));
    if (lane == 0) red[warp][u] = a;
  }
  __syncthreads();
  if (tid < ncb) {
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) a += red[k][tid];
    part[(size_t)(q0 + cb + tid) * maxch + ch] = a;
  }
  __threadfence();
  __syncthreads();
  const int ncg = (nc + kBsCols - 1) / kBsCols;
  if (tid == 0) s_last = (atomicAdd(cnt + s, 1) == nch[s] * ncg - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // chunk sums in chunk order; the loads of 8 chunks are issued together (no
  // serial chain of kch dependent L2 round trips), the adds stay sequential
  const int kch = nch[s];
  for (int q = tid; q < nc; q += blockDim.x) {
    const double* pq = part + (size_t)(q0 + q) * maxch;
    double a = 0.0;
    for (int k0 = 0; k0 < kch; k0 += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = (k0 + u < kch) ? __ldcg(pq + k0 + u) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (k0 + u < kch) a += v[u];
    }
    out[q0 + q] = w ? w[q0 + q] * a : a;
  }
  if (tid == 0) cnt[s] = 0;
}

// ---------------------------------------------------------------------------
// rank_revealing_solve (dense.cpp:348-366): b_r = b[retained]; y = L^-T L^-1 b_r;
// x = 0, x[retained] = y.  L^-T L^-1 = K^+ is formed once at setup (k_gram), so
// the solve is ONE symmetric GEMV: warp per output entry, reading row pos[i]
// of K^+ (coalesced) against the gathered b_r (L1/L2 resident).
// Rows i >= dim (when m2t is set): out2[i - dim] = M2(i - dim, :) b_r with M2
// stored transposed (r x nq, column-major): the A- dots of Z K+ b, precomputed
// as M2 = M1 K+ (build_coarse_neg), so the hybrid H2's A+ (Z c) needs no
// separate dot kernel over Z c.
__global__ void k_coarse_solve(const int* __restrict__ gate, int dim, int r, const double* __restrict__ kinv,
                               const int* __restrict__ pos, const int* __restrict__ ret,
                               const double* __restrict__ b, double* __restrict__ x, int early, int nq,
                               const double* __restrict__ m2t, double* __restrict__ out2,
                               int nd, const double* __restrict__ m2, const double* __restrict__ dvec) {
  if (gated_early(gate, early)) return;
  // b_r = b[retained] staged once per CTA (kCoarseStage doubles of static
  // shared memory) instead of two dependent loads per element in every warp
  __shared__ double sb[kCoarseStage];
  const bool staged = r <= kCoarseStage;
  if (staged) {
    for (int j = threadIdx.x; j < r; j += blockDim.x) sb[j] = __ldg(b + ret[j]);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= dim + (m2t ? nq : 0)) return;
  const int k = i < dim ? pos[i] : 0;
  double acc = 0.0;
  if (k >= 0) {
    const double* row = i < dim ? kinv + (size_t)k * r : m2t + (size_t)(i - dim) * r;
    double a1 = 0.0;
    int j = lane;
    if (staged) {
      for (; j + 32 < r; j += 64) {
        acc = fma(row[j], sb[j], acc);
        a1 = fma(row[j + 32], sb[j + 32], a1);
      }
      if (j < r) acc = fma(row[j], sb[j], acc);
    } else {
      for (; j + 32 < r; j += 64) {
        acc = fma(row[j], __ldg(b + ret[j]), acc);
        a1 = fma(row[j + 32], __ldg(b + ret[j + 32]), a1);
      }
      if (j < r) acc = fma(row[j], __ldg(b + ret[j]), acc);
    }
    if (dvec && i < dim) {  // + (M1 K+)^T d at the retained position k (column k of m2, nd x r)
      const double* col = m2 + (size_t)k * nd;
      for (j = lane; j + 32 < nd; j += 64) {
        acc = fma(col[j], __ldg(dvec + j), acc);
        a1 = fma(col[j + 32], __ldg(dvec + j + 32), a1);
      }
      if (j < nd) acc = fma(col[j], __ldg(dvec + j), acc);
    }
    acc = warp_sum(acc + a1);
  }
  if (lane == 0) {
    if (i < dim) x[i] = acc;
    else out2[i - dim] = acc;
  }
}

// g(i, j) = sum_k a(k, i) a(k, j) for a column-major lower r x r (so k >= max(i, j))
__global__ void k_gram(int r, const double* __restrict__ a, double* __restrict__ g) {
  __shared__ double as[32][33], bs[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k0 = max(i0, j0); k0 < r; k0 += 32) {
    for (int yy = ty; yy < 32; yy += 8) {
      const int k = k0 + yy;
      as[yy][tx] = (k < r && i0 + tx < r) ? a[k + (size_t)(i0 + tx) * r] : 0.0;
      bs[yy][tx] = (k < r && j0 + tx < r) ? a[k + (size_t)(j0 + tx) * r] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      const double bv = bs[kk][tx];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(as[kk][ty + 8 * q], bv, acc[q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = i0 + ty + 8 * q, j = j0 + tx;
    if (i < r && j < r) g[i + (size_t)j * r] = acc[q];
  }
}

__global__ void k_retained_set(int r, const int* __restrict__ ret, int* __restrict__ pos) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < r) pos[ret[k]] = k;
}


__global__ void k_scatter(int n, const int* __restrict__ om, const double* __restrict__ y, double* __restrict__ z) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l < n) z[om[l]] = y[l];
}

__global__ void k_zero(const int* __restrict__ gate, int n, double* __restrict__ y) {
  if (gated(gate)) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] = 0.0;
}

// L^-1 of a lower-triangular r x r column-major l (setup; thread per column,
// forward substitution against the identity, row-major scratch then transpose).

__global__ void k_tri_inverse_rm(int r, const double* __restrict__ l, double* __restrict__ xrm) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= r) return;
  for (int k = 0; k < j; ++k) xrm[(size_t)k * r + j] = 0.0;
  for (int k = j; k < r; ++k) {
    double acc = (k == j) ? 1.0 : 0.0;
    for (int m = j; m < k; ++m) acc -= l[k + (size_t)m * r] * xrm[(size_t)m * r + j];
    xrm[(size_t)k * r + j] = acc / l[k + (size_t)k * r];
  }
}

__global__ void k_transpose(int r, const double* __restrict__ a, double* __restrict__ b) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
    const int row = by + yy, col = bx + threadIdx.x;
    if (row < r && col < r) tile[yy][threadIdx.x] = a[(size_t)row * r + col];
  }
  __syncthreads();
  for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
    const int row = bx + yy, col = by + threadIdx.x;
    if (row < r && col < r) b[(size_t)row * r + col] = tile[threadIdx.x][yy];
  }
}

// ---------------------------------------------------------------------------
// Tall-skinny W (n x nm, column-major, ld): split-K W^T x, then W c.
// CTA per (row chunk of CH rows, group of 32 columns): the x chunk is staged
// in shared memory (zero past n), one warp per column, 16-byte loads, 4 in flight
// per lane; part[chunk * nm + j] holds the chunk's partial dot.  CH = 4096, or
// 1024 when that leaves fewer than 4 CTAs per SM (small W: c2's 262 columns
// over 65,536 rows were 144 CTAs at 3.6 TB/s).
template <int CH>
__global__ void __launch_bounds__(kThreads) k_dense_gemvT_part(const int* __restrict__ gate, int n, int nm, int ldw,
                                                            const double* __restrict__ W, const double* __restrict__ x,
                                                            double* __restrict__ part) {
  if (gated(gate)) return;
  __shared__ double2 sx2[CH / 2];
  double* sx = reinterpret_cast<double*>(sx2);
  const int r0 = blockIdx.y * CH;
  const int rows = min(CH, ldw - r0);  // ldw is a multiple of 4: pad rows of W are zero
  for (int i = threadIdx.x; i < CH; i += blockDim.x) sx[i] = (r0 + i < n) ? x[r0 + i] : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int npair = rows >> 1;
  const int jend = min(nm, (int)(blockIdx.x + 1) * 32);
  for (int j = blockIdx.x * 32 + warp; j < jend; j += 8) {
    const double2* col = reinterpret_cast<const double2*>(W + (size_t)j * ldw + r0);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int q = lane;
    for (; q + 96 < npair; q += 128) {
      const double2 v0 = __ldcs(col + q), v1 = __ldcs(col + q + 32), v2 = __ldcs(col + q + 64),
                    v3 = __ldcs(col + q + 96);
      const double2 x0 = sx2[q], x1 = sx2[q + 32], x2 = sx2[q + 64], x3 = sx2[q + 96];
      a0 = fma(v0.x, x0.x, a0); a0 = fma(v0.y, x0.y, a0);
      a1 = fma(v1.x, x1.x, a1); a1 = fma(v1.y, x1.y, a1);
      a2 = fma(v2.x, x2.x, a2); a2 = fma(v2.y, x2.y, a2);
      a3 = fma(v3.x, x3.x, a3); a3 = fma(v3.y, x3.y, a3);
    }
    for (; q < npair; q += 32) {
      const double2 v0 = __ldcs(col + q);
      const double2 x0 = sx2[q];
      a0 = fma(v0.x, x0.x, a0); a0 = fma(v0.y, x0.y, a0);
    }
    const double sum = warp_sum((a0 + a1) + (a2 + a3));
    if (lane == 0) part[(size_t)blockIdx.y * nm + j] = sum;
  }
}

__global__ void k_colsum(const int* __restrict__ gate, int nm, int nchunks, const double* __restrict__ part,
                         double* __restrict__ out) {
  if (gated(gate)) return;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nm) return;
  double acc = 0.0;
  for (int c = 0; c < nchunks; ++c) acc += part[(size_t)c * nm + j];
  out[j] = acc;
}

// y = W c, CTA per (512-row panel, column chunk kc of nkc): two rows per thread
// (16-byte loads), 8 columns in flight; with nkc > 1 the chunk results go to
// part[kc * ldw + i] and k_chunk_sum adds them in fixed order.
__global__ void __launch_bounds__(kThreads) k_dense_gemv(const int* __restrict__ gate, int n, int nm, int ldw, int nkc,
                                                      const double* __restrict__ W, const double* __restrict__ c,
                                                      double* __restrict__ y, double* __restrict__ part) {
  if (gated(gate)) return;
  extern __shared__ double scoef[];
  const int kc = blockIdx.y;
  const int j0 = int((long long)nm * kc / nkc), j1 = int((long long)nm * (kc + 1) / nkc);
  for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) scoef[j - j0] = c[j];
  __syncthreads();
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (i >= n) return;
  const double* w = W + i;
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
  int j = j0;
  for (; j + 8 <= j1; j += 8) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(reinterpret_cast<const double2*>(w + (size_t)(j + u) * ldw));
#pragma unroll
    for (int u = 0; u < 8; u += 2) {
      const double c0 = scoef[j + u - j0], c1 = scoef[j + u + 1 - j0];
      a0 = fma(v[u].x, c0, a0);
      a1 = fma(v[u].y, c0, a1);
      b0 = fma(v[u + 1].x, c1, b0);
      b1 = fma(v[u + 1].y, c1, b1);
    }
  }
  for (; j < j1; ++j) {
    const double2 v0 = __ldcs(reinterpret_cast<const double2*>(w + (size_t)j * ldw));
    const double c0 = scoef[j - j0];
    a0 = fma(v0.x, c0, a0);
    a1 = fma(v0.y, c0, a1);
  }
  double* out = (nkc == 1) ? y : part + (size_t)kc * ldw;
  out[i] = a0 + b0;
  if (i + 1 < n) out[i + 1] = a1 + b1;
}

__global__ void k_chunk_sum(const int* __restrict__ gate, int n, int ldw, int nkc, const double* __restrict__ part,
                            double* __restrict__ y) {
  if (gated(gate)) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int kc = 0; kc < nkc; ++kc) acc += part[(size_t)kc * ldw + i];
    y[i] = acc;
  }
}

// ---------------------------------------------------------------------------
// INEX core solve (preconditioner.cpp:208-216): LU with partial pivoting
// (dense.cpp:368-393) and its solve; lu_semantics 0 reproduces the reference
// back substitution (dense.cpp:404-409, reads lu(i,k) below the diagonal),
// 1 the exact one (reads lu(k,i)).  Single CTA: n_minus is small.
__global__ void k_lu_solve(const int* __restrict__ gate, int m, const double* __restrict__ lu,
                           const int* __restrict__ perm, const double* __restrict__ b, double* __restrict__ x,
                           int exact) {
  if (gated(gate)) return;
  extern __shared__ double sy[];
  for (int i = threadIdx.x; i < m; i += blockDim.x) sy[i] = b[perm[i]];
  __syncthreads();
  for (int k = 0; k < m; ++k) {
    const double f0 = sy[k];
    __syncthreads();
    if (f0 != 0.0)
      for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) sy[i] -= f0 * lu[i + (size_t)k * m];
    __syncthreads();
  }
  // back substitution: sequential in k, parallel dot per k
  __shared__ double red[32];
  for (int k = m - 1; k >= 0; --k) {
    double part = 0.0;
    for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) {
      const double a = exact ? lu[k + (size_t)i * m] : lu[i + (size_t)k * m];
      part = fma(a, sy[i], part);
    }
    part = warp_sum(part);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
      double acc = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) acc += red[w];
      sy[k] = (sy[k] - acc) / lu[k + (size_t)k * m];
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) x[i] = sy[i];
}

// elementwise compositions
//   mode 0: y = (a - b) + d      (TwoLevel hybrid: Pi hp + corr, preconditioner.cpp:79-81)
//   mode 1: y = a + b            (additive / AD sums)
//   mode 2: y = a - b            (projectors)
__global__ void k_axpby(const int* __restrict__ gate, int n, const double* __restrict__ a,
                        const double* __restrict__ b, const double* __restrict__ d, double* __restrict__ y,
                        int mode) {
  if (gated(gate)) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double v;
    if (mode == 0) v = (a[i] - b[i]) + d[i];
    else if (mode == 1) v = a[i] + b[i];
    else v = a[i] - b[i];
    y[i] = v;
  }
}


// owner-entry tables (see OwnEnt): entry q of the owner lists, p = own_pos[q]
__global__ void k_own_ent(long long P, const int* __restrict__ own_pos, const int* __restrict__ psub,
                          const long long* __restrict__ poff, const long long* __restrict__ moff,
                          const int* __restrict__ ld, const int* __restrict__ coff, OwnEnt* __restrict__ ent) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < P; q += (long long)gridDim.x * blockDim.x) {
    const int p = own_pos[q];
    const int s = psub[p];
    OwnEnt e;
    e.mbase = moff[s] + (p - poff[s]);
    e.L = ld[s];
    e.q0 = coff[s];
    e.q1 = coff[s + 1];
    e.pad = 0;
    ent[q] = e;
  }
}

__global__ void k_own_nkc(long long P, const int* __restrict__ own_pos, const int* __restrict__ psub,
                          const int* __restrict__ nkc, int2* __restrict__ out) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < P; q += (long long)gridDim.x * blockDim.x) {
    const int p = own_pos[q];
    out[q] = make_int2(p, nkc[psub[p]]);
  }
}

}  // namespace

// ===========================================================================
namespace k {

void owner_tables(Ctx& c) {
  const long long P = std::max<long long>(c.P, 1);
  const int g = grid_for(c, c.P);
  c.ent_neg.alloc(P);
  c.ent_z.alloc(P);
  k_own_ent<<<g, kThreads, 0, c.stream>>>(c.P, c.own_pos.p, c.psub.p, c.poff.p, c.voff.p, c.ld.p, c.negoff.p,
                                          c.ent_neg.p);
  k_own_ent<<<g, kThreads, 0, c.stream>>>(c.P, c.own_pos.p, c.psub.p, c.poff.p, c.yoff.p, c.ld.p, c.koff.p,
                                          c.ent_z.p);
  c.launches += 2;
  for (LocalPlan* pl : {&c.plan_nn, &c.plan_as}) {
    if (pl->nkc.p) {
      pl->own_nkc.alloc(P);
      k_own_nkc<<<g, kThreads, 0, c.stream>>>(c.P, c.own_pos.p, c.psub.p, pl->nkc.p, pl->own_nkc.p);
      ++c.launches;
    }
    if (pl->fused && pl->nkc_f.p) {
      pl->own_nkc_f.alloc(P);
      k_own_nkc<<<g, kThreads, 0, c.stream>>>(c.P, c.own_pos.p, c.psub.p, pl->nkc_f.p, pl->own_nkc_f.p);
      ++c.launches;
    }
  }
  check_launch("owner_tables");
}

void spmv(Ctx& c, const double* x, double* y, int mode, const double* add, const double* sub, const int* gate) {
  launch(c, k_spmv, grid_for(c, c.n), kThreads, 0, gate, c.n, c.rp.p, c.ci.p, c.va.p, x, y, mode, add, sub);
  ++c.launches;
  check_launch("spmv");
}

void gather(Ctx& c, const double* x, const double* scale, double* xs, const int* gate) {
  launch(c, k_gather, grid_for(c, c.P), kThreads, 0, gate, c.P, c.pidx.p, x, scale, xs);
  ++c.launches;
  check_launch("gather");
}

void prolong(Ctx& c, const double* w, double* y, const int* gate) {
  launch(c, k_prolong, grid_for(c, c.n), kThreads, 0, gate, c.n, c.own_off.p, c.own_pos.p, w, y);
  ++c.launches;
  check_launch("prolong");
}

static size_t nn_smem(Ctx& c) {
  int ldmax = 0;
  for (int v : c.h_ld) ldmax = std::max(ldmax, v);
  const size_t smem = size_t(ldmax) * sizeof(double);
  ensure_dyn_smem((const void*)k_nn_gemvT<8, false>, smem);
  ensure_dyn_smem((const void*)k_nn_gemvT<8, true>, smem);
  return smem;
}

// The one-level factor in use: NN (V^s, eigenvalue mask, D^s) or AS/AS+ (U^s = L^-T).
static const LocalPlan& plan(const Ctx& c) { return c.one_level == 2 ? c.plan_nn : c.plan_as; }

void nn_gemvT(Ctx& c, const double* x, const int* gate) {
  const size_t smem = nn_smem(c);
  const LocalPlan& pl = plan(c);
  if (!pl.tT.n) return;
  if (c.one_level == 2)
    launch(c, (k_nn_gemvT<8, false>), int(pl.tT.n), 256, smem, gate, pl.tT.p, c.V.p, c.voff.p, c.ns.p, c.ld.p,
                                                                c.poff.p, c.pidx.p, c.ds.p, x, c.lam.p, c.uh.p);
  else
    launch(c, (k_nn_gemvT<8, true>), int(pl.tT.n), 256, smem, gate, pl.tT.p, c.U.p, c.voff.p, c.ns.p, c.ld.p,
                                                               c.poff.p, c.pidx.p, nullptr, x, nullptr, c.uh.p);
  ++c.launches;
  check_launch("nn_gemvT");
}

void nn_gemv(Ctx& c, const int* gate) {
  const LocalPlan& pl = plan(c);
  if (!pl.t.n) return;
  launch(c, k_nn_gemv, int(pl.t.n), kThreads, size_t(pl.cols_max) * sizeof(double), 
      gate, pl.t.p, c.one_level == 2 ? c.V.p : c.U.p, c.voff.p, c.ns.p, c.ld.p, c.poff.p, c.P, c.uh.p,
      c.wpart_nn.p);
  ++c.launches;
  check_launch("nn_gemv");
}


// split-K partial sum + D^s + prolongation (k_prolong_nn), lanes per row by size
static void prolong_nn(Ctx& c, const int2* own_nkc, int kcmax, double* y, const int* gate) {
  const double* ds = c.one_level == 2 ? c.ds.p : nullptr;
  const int G = c.n > 300000 ? 1 : (kcmax >= 16 ? 8 : 4);
  if (G == 8)
    launch(c, k_prolong_nn<8>, grid_for(c, 8LL * c.n), kThreads, 0, gate, c.n, c.own_off.p, own_nkc, c.P,
           c.wpart_nn.p, ds, y);
  else if (G == 4)
    launch(c, k_prolong_nn<4>, grid_for(c, 4LL * c.n), kThreads, 0, gate, c.n, c.own_off.p, own_nkc, c.P,
           c.wpart_nn.p, ds, y);
  else
    launch(c, k_prolong_nn<1>, grid_for(c, c.n), kThreads, 0, gate, c.n, c.own_off.p, own_nkc, c.P, c.wpart_nn.p,
           ds, y);
}

void nn_prolong(Ctx& c, double* y, const int* gate) {
  const LocalPlan& pl = plan(c);
  prolong_nn(c, pl.own_nkc.p, pl.kcmax, y, gate);
  ++c.launches;
  check_launch("prolong_nn");
}

// single-pass NN local solve into the split-K partials (see k_nn_fused)
template <bool TRI, int R, int CPB, bool HOLD>
void launch_fused(Ctx& c, const LocalPlan& pl, const double* F, const double* D, const double* x, const int* gate,
                  int grid, size_t smem, int nbuf, int ldmax) {
  ensure_dyn_smem((const void*)k_nn_fused<TRI, R, CPB, HOLD>, kFusedSmemCap);
  launch(c, k_nn_fused<TRI, R, CPB, HOLD>, grid, kFusedT, smem, gate, pl.tf.p, F, c.voff.p, c.ns.p, c.ld.p, c.poff.p,
         c.pidx.p, D, x, TRI ? nullptr : c.rlam.p, c.P, c.wpart_nn.p, int(pl.tf.n), c.fused_queue.p,
         pl.static_grid ? pl.cta_off.p : nullptr, nbuf, ldmax,
         int(smem / sizeof(double)), int(c.fused_prefetch), int(c.pdl_local && pl.static_grid > 0),
         c.fused_timer.p);
}

template <bool TRI, int CPB, bool HOLD>
void launch_fused_r(Ctx& c, const LocalPlan& pl, const double* F, const double* D, const double* x, const int* gate,
                    int grid, size_t smem, int nbuf, int ldmax, int R) {
  switch (R) {
    case 2: launch_fused<TRI, 2, CPB, HOLD>(c, pl, F, D, x, gate, grid, smem, nbuf, ldmax); break;
    case 4: launch_fused<TRI, 4, CPB, HOLD>(c, pl, F, D, x, gate, grid, smem, nbuf, ldmax); break;
    case 8: launch_fused<TRI, 8, CPB, HOLD>(c, pl, F, D, x, gate, grid, smem, nbuf, ldmax); break;
    case 10: launch_fused<TRI, 10, CPB, HOLD>(c, pl, F, D, x, gate, grid, smem, nbuf, ldmax); break;
    case 11: launch_fused<TRI, 11, CPB, HOLD>(c, pl, F, D, x, gate, grid, smem, nbuf, ldmax); break;
    default: launch_fused<TRI, 12, CPB, HOLD>(c, pl, F, D, x, gate, grid, smem, nbuf, ldmax); break;
  }
}

void nn_fused(Ctx& c, const double* x, const int* gate) {
  const bool nn = (c.one_level == 2);
  const LocalPlan& pl = plan(c);
  int ldmax = 0;
  for (int v : c.h_ld) ldmax = std::max(ldmax, v);
  // rows per thread: the smallest instantiated R with R * kFusedT >= ldmax
  const int need = (ldmax + kFusedT - 1) / kFusedT;
  const int R = need <= 2 ? 2 : need <= 4 ? 4 : need <= 8 ? 8 : need <= 10 ? 10 : need <= 11 ? 11 : 12;
  // copy pipeline: CPB columns per buffer, as many buffers as fit (<= kFusedMaxBuf),
  // plus the tail that unchecked rows of the last buffer may reach.  Without
  // HOLD (profiles/README.md): two-column steps win while >= 3 two-column
  // buffers fit (c2, ld 4612) and lose to 4 one-column buffers at ld 5632 (c5).
  // With HOLD a buffer is refilled one step earlier (see below).
  const size_t tail = size_t(std::max(0, R * kFusedT - ldmax)) * sizeof(double);
  const bool hold = c.fused_hold && nn;  // NN only (the triangular AS variant spills with it at R = 12)
  const size_t fit1 = (kFusedSmemCap - tail) / (size_t(ldmax) * sizeof(double));  // one-column buffers that fit
  int cpb;
  int nbuf_pref = 0;
  if (hold) {
    // measured (profiles/r01b/sweep_hold2.json): c2 (6 one-column buffers fit)
    // 0.381 ms with 3 x 1 column vs 0.384 with 3 x 2; c5 (5 fit) 6.81 ms with
    // 2 x 2 columns vs 6.90 with 3 x 1
    cpb = fit1 >= 6 ? 1 : 2;
    nbuf_pref = cpb == 1 ? 3 : 0;
  } else {
    cpb = fit1 / 2 >= 3 ? 2 : 1;
  }
  if (c.fused_cpb == 1 || c.fused_cpb == 2) cpb = c.fused_cpb;
  const size_t buf_bytes = size_t(cpb) * ldmax * sizeof(double);
  int nbuf = int(std::min<size_t>(kFusedMaxBuf, (kFusedSmemCap - tail) / buf_bytes));
  if (nbuf_pref > 0) nbuf = std::min(nbuf, nbuf_pref);
  if (c.fused_nbuf > 0) nbuf = std::min(nbuf, c.fused_nbuf);
  if (nbuf < 2) c.fail(AWG_E_STATE, "single-pass local solve: subdomain too large for the copy pipeline");
  const size_t smem = size_t(nbuf) * buf_bytes + tail;
  if (!pl.tf.n) return;
  if (!c.fused_queue.p) {
    c.fused_queue.alloc(2);  // (next task, CTAs finished); reset by the kernel itself
    c.fused_queue.zero(c.stream);
  }
  if (!c.fused_timer.p) {
    static const unsigned long long init[5] = {~0ull, 0, 0, 0, 0};
    c.fused_timer.alloc(5);
    AWG_CUDA(cudaMemcpyAsync(c.fused_timer.p, init, sizeof(init), cudaMemcpyHostToDevice, c.stream));
  }
  // persistent CTAs: one per SM, less the SMs left to the concurrent W branch
  const int grid =
      pl.static_grid ? pl.static_grid : std::min(int(pl.tf.n), std::max(1, c.sm_count - c.fused_reserve));
  const double* F = nn ? c.V.p : c.U.p;
  const double* D = nn ? c.ds.p : nullptr;
  if (nn && cpb == 2)
    hold ? launch_fused_r<false, 2, true>(c, pl, F, D, x, gate, grid, smem, nbuf, ldmax, R)
         : launch_fused_r<false, 2, false>(c, pl, F, D, x, gate, grid, smem, nbuf, ldmax, R);
  else if (nn)
    hold ? launch_fused_r<false, 1, true>(c, pl, F, D, x, gate, grid, smem, nbuf, ldmax, R)
         : launch_fused_r<false, 1, false>(c, pl, F, D, x, gate, grid, smem, nbuf, ldmax, R);
  else if (cpb == 2)
    hold ? launch_fused_r<true, 2, true>(c, pl, F, D, x, gate, grid, smem, nbuf, ldmax, R)
         : launch_fused_r<true, 2, false>(c, pl, F, D, x, gate, grid, smem, nbuf, ldmax, R);
  else
    hold ? launch_fused_r<true, 1, true>(c, pl, F, D, x, gate, grid, smem, nbuf, ldmax, R)
         : launch_fused_r<true, 1, false>(c, pl, F, D, x, gate, grid, smem, nbuf, ldmax, R);
  ++c.launches;
  check_launch("nn_fused");
}

void h1(Ctx& c, const double* x, double* y, const int* gate) {
  const LocalPlan& pl = plan(c);
  if (pl.fused) {
    nn_fused(c, x, gate);
    prolong_nn(c, pl.own_nkc_f.p, pl.kcmax_f, y, gate);
    ++c.launches;
    check_launch("prolong_nn");
    return;
  }
  nn_gemvT(c, x, gate);
  nn_gemv(c, gate);
  nn_prolong(c, y, gate);
}

struct BsIndex {  // row index sets of a block family (default: the subdomains' Omega^s)
  const int* ns;
  const int* ld;
  const long long* poff;
  const int* pidx;
};
static void bs_gemvT(Ctx& c, BsPlan& b, const int* coff, const int* ccol, const double* M, const long long* moff,
                     const double* x, const double* w, double* out, const int* gate, const BsIndex* ix = nullptr) {
  if (b.ntask == 0) return;
  const BsIndex dflt{c.ns.p, c.ld.p, c.poff.p, c.pidx.p};
  if (!ix) ix = &dflt;
  launch(c, k_bs_gemvT, dim3(b.ntask, b.ncg), 256, 0, gate, b.ts.p, b.tc.p, b.nch.p, b.maxch, coff, ccol, M, moff, ix->ns,
                                            ix->ld, ix->poff, ix->pidx, x, w, b.part.p, b.cnt.p, out, c.pdl_early);
  ++c.launches;
  check_launch("bs_gemvT");
}

static void neg_dot(Ctx& c, const double* x, const int* gate) {
  bs_gemvT(c, c.bs_neg, c.negoff.p, c.neg_k.p, c.V.p, c.voff.p, x, c.neg_w.p, c.neg_c.p, gate);
}

// lanes per dof of the block-sparse prolongations (AWG_ROWS_GROUP overrides: 1, 4 or 8)
static int rows_group(const Ctx& c) {
  if (c.rows_group == 1 || c.rows_group == 4 || c.rows_group == 8) return c.rows_group;
  return c.n <= 300000 ? 4 : 1;
}

void aminus(Ctx& c, const double* x, double* y, const int* gate) {
  if (c.nneg == 0) {
    launch(c, k_zero, grid_for(c, c.n), kThreads, 0, gate, c.n, y);
    ++c.launches;
    check_launch("zero");
    return;
  }
  neg_dot(c, x, gate);
  launch(c, k_block_combine, grid_for(c, c.P), kThreads, 0, gate, c.P, c.psub.p, c.poff.p, c.negoff.p, c.neg_k.p,
                                                               c.V.p, c.voff.p, c.ld.p, c.neg_c.p, c.wl.p);
  ++c.launches;
  check_launch("neg_combine");
  prolong(c, c.wl.p, y, gate);
}

static BlockSum neg_sum(const Ctx& c) {
  return BlockSum{c.own_off.p, c.ent_neg.p, c.neg_k.p, c.V.p, c.neg_c.p};
}

// y = A+ x (mode 1) or y = sub - A+ x (mode 2): the A- dots, then one fused
// SpMV + A- prolongation kernel
void aplus(Ctx& c, const double* x, double* y, int mode, const double* sub, const int* gate, bool neg_ready) {
  if (c.nneg > 0 && !neg_ready) neg_dot(c, x, gate);
  BlockSum bs = neg_sum(c);
  if (rows_group(c) == 8)
    launch(c, k_spmv_aplus<8>, grid_for(c, 8LL * c.n), kThreads, 0, gate, c.n, c.rp.p, c.ci.p, c.va.p, x, y, mode,
           sub, bs, c.trigger_next);
  else if (rows_group(c) == 4)
    launch(c, k_spmv_aplus<4>, grid_for(c, 4LL * c.n), kThreads, 0, gate, c.n, c.rp.p, c.ci.p, c.va.p, x, y, mode,
                                                                       sub, bs, c.trigger_next);
  else
    launch(c, k_spmv_aplus<1>, grid_for(c, c.n), kThreads, 0, gate, c.n, c.rp.p, c.ci.p, c.va.p, x, y, mode, sub,
                                                                bs, c.trigger_next);
  ++c.launches;
  check_launch("spmv_aplus");
}

void rr_solve(Ctx& c, const CoarseFactor& f, const double* b, double* x, const int* gate) {
  const int wpb = kThreads / 32;
  if (f.rank == 0) {
    launch(c, k_zero, grid_for(c, f.dim), kThreads, 0, gate, f.dim, x);
    ++c.launches;
    return;
  }
  launch(c, k_coarse_solve, (f.dim + wpb - 1) / wpb, kThreads, 0, gate, f.dim, f.rank, f.kinv.p, f.pos.p,
                                                                     f.retained.p, b, x, c.pdl_early, 0,
         (const double*)nullptr, (double*)nullptr, 0, (const double*)nullptr, (const double*)nullptr);
  ++c.launches;
  check_launch("coarse_solve");
}

// Q x into y and, in the same coarse-solve launch, the A- dots of y into
// neg_c (the coefficients k::aplus's SpMV consumes with neg_ready = true).
// Returns false (nothing enqueued) when M2 is not available.
bool coarse_q_neg(Ctx& c, const double* x, double* y, const int* gate) {
  if (!c.m2t.p || c.n0 == 0 || c.k0.rank == 0) return false;
  zT(c, x, c.cz.p, gate);
  double* coef = c.cz.p + c.n0;
  const int wpb = kThreads / 32;
  const CoarseFactor& f = c.k0;
  launch(c, k_coarse_solve, (f.dim + c.nneg + wpb - 1) / wpb, kThreads, 0, gate, f.dim, f.rank, f.kinv.p, f.pos.p,
         f.retained.p, (const double*)c.cz.p, coef, c.pdl_early, c.nneg, (const double*)c.m2t.p, c.neg_c.p, 0,
         (const double*)nullptr, (const double*)nullptr);
  ++c.launches;
  check_launch("coarse_solve_neg");
  const BlockSum bs{c.own_off.p, c.ent_z.p, nullptr, c.Y.p, coef};
  const Combine cb{nullptr, nullptr, nullptr, RzFuse{}};
  if (rows_group(c) == 4)
    launch(c, k_prolong_sum<4>, grid_for(c, 4LL * c.n), kThreads, 0, gate, c.n, bs, y, cb, c.pdl_early);
  else
    launch(c, k_prolong_sum<1>, grid_for(c, c.n), kThreads, 0, gate, c.n, bs, y, cb, c.pdl_early);
  ++c.launches;
  check_launch("z_prolong");
  return true;
}

void coarse_q(Ctx& c, const double* x, double* y, const int* gate) {
  if (c.n0 == 0) {
    launch(c, k_zero, grid_for(c, c.n), kThreads, 0, gate, c.n, y);
    ++c.launches;
    return;
  }
  coarse_q_combine(c, x, y, nullptr, nullptr, nullptr, nullptr, gate);
}

static void z_combine(Ctx& c, const double* coef, double* y, const double* a, const double* d, const double* e,
                      cudaEvent_t wait_before_combine, const int* gate);

void coarse_q_combine(Ctx& c, const double* x, double* y, const double* a, const double* d, const double* e,
                      cudaEvent_t wait_before_combine, const int* gate) {
  if (c.n0 == 0) c.fail(AWG_E_STATE, "coarse_q: empty coarse space");
  zT(c, x, c.cz.p, gate);
  double* coef = c.cz.p + c.n0;  // second half of cz holds the solved coefficients
  rr_solve(c, c.k0, c.cz.p, coef, gate);
  z_combine(c, coef, y, a, d, e, wait_before_combine, gate);
}

// The post-solve half of the hybrid H2 without A+ hp:
//   Z^T A+ hp = (A Z)^T hp + Z^T A- hp,  Z^T A- hp = M1^T (V-^T R hp)
// (M1(q, j) = |lambda_q| v_q^T R z_j, build_coarse_neg), so c2 = K+ (Z^T A+ hp)_r = K+ g_r + (M1 K+)^T d with
// g = (A Z)^T hp and d = V-^T R hp from ONE block-sparse GEMV^T launch over both
// families and the second term inside the coarse-solve launch: 3 kernels where
// A- dots + A+ SpMV + Z^T + solve + combine were 5.  Same sums regrouped
// (rounding-level differences only).
void coarse_q_combine_az(Ctx& c, const double* hp, double* y, const double* corr, const double* extra,
                         cudaEvent_t wait_before_combine, const int* gate) {
  if (!c.az_on) c.fail(AWG_E_STATE, "coarse_q_combine_az: A Z not built");
  const BsIndex ix{c.az_ns.p, c.az_ld.p, c.az_poff.p, c.az_pidx.p};
  bs_gemvT(c, c.bs_az, c.az_coff.p, c.az_ccol.p, c.V.p, c.az_moff.p, hp, nullptr, c.az_out.p, gate, &ix);
  double* coef = c.cz.p + c.n0;
  const CoarseFactor& f = c.k0;
  const int wpb = kThreads / 32;
  launch(c, k_coarse_solve, (f.dim + wpb - 1) / wpb, kThreads, 0, gate, f.dim, f.rank, f.kinv.p, f.pos.p, f.retained.p,
         (const double*)(c.az_out.p + c.nneg), coef, c.pdl_early, 0, (const double*)nullptr, (double*)nullptr, c.nneg,
         (const double*)c.m2.p, (const double*)c.az_out.p);
  ++c.launches;
  check_launch("coarse_solve_az");
  z_combine(c, coef, y, hp, corr, extra, wait_before_combine, gate);
}

static void z_combine(Ctx& c, const double* coef, double* y, const double* a, const double* d, const double* e,
                      cudaEvent_t wait_before_combine, const int* gate) {
  if (wait_before_combine) AWG_CUDA(cudaStreamWaitEvent(c.stream, wait_before_combine, 0));
  // Z c: block-sparse combination fused with the prolongation and the composition
  const BlockSum bs{c.own_off.p, c.ent_z.p, nullptr, c.Y.p, coef};
  Combine cb{a, d, e, RzFuse{}};
  if (c.rz_fuse.st && a && y == c.rz_fuse.z) {  // the last kernel of the PCG's preconditioner apply
    cb.rz = c.rz_fuse;
    c.rz_fused = true;
  }
  if (rows_group(c) == 8)
    launch(c, k_prolong_sum<8>, grid_for(c, 8LL * c.n), kThreads, 0, gate, c.n, bs, y, cb, c.pdl_early);
  else if (rows_group(c) == 4)
    launch(c, k_prolong_sum<4>, grid_for(c, 4LL * c.n), kThreads, 0, gate, c.n, bs, y, cb, c.pdl_early);
  else
    launch(c, k_prolong_sum<1>, grid_for(c, c.n), kThreads, 0, gate, c.n, bs, y, cb, c.pdl_early);
  ++c.launches;
  check_launch("z_prolong");
}

void zT(Ctx& c, const double* x, double* out, const int* gate) {
  bs_gemvT(c, c.bs_z, c.koff.p, nullptr, c.Y.p, c.yoff.p, x, nullptr, out, gate);
}

static void w_transpose_apply(Ctx& c, const double* x, double* out, const int* gate) {
  const int groups = (c.nm + 31) / 32;
  const int ch = (long long)groups * ((c.ldw + 4095) / 4096) >= 4LL * c.sm_count ? 4096 : 1024;
  const int nch = (c.ldw + ch - 1) / ch;
  dim3 grid(groups, nch);
  if (ch == 4096)
    launch(c, k_dense_gemvT_part<4096>, grid, kThreads, 0, gate, c.n, c.nm, c.ldw, c.W.p, x, c.wpart.p);
  else
    launch(c, k_dense_gemvT_part<1024>, grid, kThreads, 0, gate, c.n, c.nm, c.ldw, c.W.p, x, c.wpart.p);
  ++c.launches;
  check_launch("dense_gemvT_part");
  launch(c, k_colsum, (c.nm + kThreads - 1) / kThreads, kThreads, 0, gate, c.nm, nch, c.wpart.p, out);
  ++c.launches;
  check_launch("colsum");
}

static void w_apply(Ctx& c, const double* coef, double* y, const int* gate) {
  const int nkc = w_chunks(c);
  const int chunk = (c.nm + nkc - 1) / nkc + 1;
  const size_t smem = size_t(chunk) * sizeof(double);
  if (smem > 48 * 1024) ensure_dyn_smem((const void*)k_dense_gemv, smem);
  dim3 grid((c.n + 2 * kThreads - 1) / (2 * kThreads), nkc);
  launch(c, k_dense_gemv, grid, kThreads, smem, gate, c.n, c.nm, c.ldw, nkc, c.W.p, coef, y, c.wpart2.p);
  ++c.launches;
  check_launch("dense_gemv");
  if (nkc > 1) {
    launch(c, k_chunk_sum, grid_for(c, c.n), kThreads, 0, gate, c.n, c.ldw, nkc, c.wpart2.p, y);
    ++c.launches;
    check_launch("chunk_sum");
  }
}

void wT(Ctx& c, const double* x, double* out, const int* gate) { w_transpose_apply(c, x, out, gate); }

void scatter_col(Ctx& c, int s, const double* col, double* z) {
  const int n = c.h_ns[s];
  k_scatter<<<(n + kThreads - 1) / kThreads, kThreads, 0, c.stream>>>(n, c.pidx.p + c.h_poff[s], col, z);
  ++c.launches;
  check_launch("scatter");
}
void w_apply_public(Ctx& c, const double* coef, double* y, const int* gate) { w_apply(c, coef, y, gate); }

void second_q(Ctx& c, const double* x, double* y, const int* gate) {
  if (c.nm == 0) {
    launch(c, k_zero, grid_for(c, c.n), kThreads, 0, gate, c.n, y);
    ++c.launches;
    return;
  }
  second_q_coef(c, x, gate);
  second_q_apply(c, y, gate);
}

void second_q_coef(Ctx& c, const double* x, const int* gate) {
  w_transpose_apply(c, x, c.cw.p, gate);
  rr_solve(c, c.kw, c.cw.p, c.cw.p + c.nm, gate);
}

void second_q_apply(Ctx& c, double* y, const int* gate) { w_apply(c, c.cw.p + c.nm, y, gate); }

void inex_q(Ctx& c, const double* x, double* y, const int* gate) {
  double* wx = c.cw.p;
  double* coef = c.cw.p + c.nm;
  w_transpose_apply(c, x, wx, gate);
  launch(c, k_lu_solve, 1, 1024, size_t(c.nm) * sizeof(double), gate, c.nm, c.core_lu.p, c.core_perm.p, wx, coef,
                                                                   c.lu_semantics);
  ++c.launches;
  check_launch("lu_solve");
  w_apply(c, coef, y, gate);
}

void axpby(Ctx& c, int n, const double* a, const double* b, const double* d, double* y, int mode, const int* gate) {
  launch(c, k_axpby, grid_for(c, n), kThreads, 0, gate, n, a, b, d, y, mode);
  ++c.launches;
  check_launch("axpby");
}

// L^-1 (column-major, linv: the block W build multiplies by it), K^+ = L^-T L^-1
// (kinv, the apply-time solve) and the retained positions
void coarse_inverse(Ctx& c, const double* l, CoarseFactor& f) {
  const int r = f.rank;
  f.linv.alloc(size_t(std::max(r, 1)) * std::max(r, 1));
  f.kinv.alloc(size_t(std::max(r, 1)) * std::max(r, 1));
  f.pos.alloc(std::max(f.dim, 1));
  AWG_CUDA(cudaMemsetAsync(f.pos.p, 0xff, sizeof(int) * std::max(f.dim, 1), c.stream));  // -1
  if (r == 0) {
    AWG_CUDA(cudaStreamSynchronize(c.stream));
    return;
  }
  DArr<double> linvT;  // row-major L^-1 (k_tri_inverse_rm), transposed into linv
  linvT.alloc(size_t(r) * r);
  k_tri_inverse_rm<<<(r + 127) / 128, 128, 0, c.stream>>>(r, l, linvT.p);
  ++c.launches;
  check_launch("tri_inverse");
  dim3 grid((r + 31) / 32, (r + 31) / 32);
  k_transpose<<<grid, dim3(32, 8), 0, c.stream>>>(r, linvT.p, f.linv.p);
  ++c.launches;
  check_launch("transpose");
  k_gram<<<grid, dim3(32, 8), 0, c.stream>>>(r, f.linv.p, f.kinv.p);
  ++c.launches;
  check_launch("gram");
  k_retained_set<<<(r + 255) / 256, 256, 0, c.stream>>>(r, f.retained.p, f.pos.p);
  ++c.launches;
  check_launch("retained_pos");
  AWG_CUDA(cudaStreamSynchronize(c.stream));
}

// M2 for coarse_q_neg: M1(q, jj) = A- dot q of coarse column retained[jj]
// (the dots k_bs_gemvT forms for A+ (Z c), one column at a time), M2 = M1 K+.
// option coarse_neg=0 disables (the hybrid H2 then runs the dot kernel on Z c).
void build_coarse_neg(Ctx& c) {
  c.m2t.release();
  if (c.opt("coarse_neg", 1) == 0) return;
  const int r = c.k0.rank, nq = c.nneg;
  if (nq == 0 || c.n0 == 0 || r == 0) return;
  // measured (profiles/r01e/knobs_coarse_neg_c{3,5}.json, ms per PCG iteration):
  // M2 at 0.7 MB (c2) and 35 MB (c3: 3.68 -> 3.62) wins; at 69 MB (c5: 13.71 ->
  // 13.95) the doubled coarse-solve launch on the critical chain loses to the
  // dot kernel over Z c, so the precomputed dots stop at 48 MB
  if (double(nq) * r * 8.0 > 48.0 * 1024.0 * 1024.0) return;
  std::vector<int> cs, ck;
  for (int s = 0; s < c.N; ++s)
    for (int k = 0; k < c.h_ks[s]; ++k) {
      cs.push_back(s);
      ck.push_back(k);
    }
  DArr<double> M1, t;
  M1.alloc(size_t(nq) * r);
  t.alloc(c.n);
  for (int jj = 0; jj < r; ++jj) {
    const int j = c.k0.h_retained[jj], s = cs[j], k = ck[j];
    AWG_CUDA(cudaMemsetAsync(t.p, 0, sizeof(double) * c.n, c.stream));
    scatter_col(c, s, c.Y.p + c.h_yoff[s] + size_t(k) * c.h_ld[s], t.p);
    neg_dot(c, t.p, nullptr);
    AWG_CUDA(cudaMemcpyAsync(M1.p + size_t(jj) * nq, c.neg_c.p, sizeof(double) * nq, cudaMemcpyDeviceToDevice,
                             c.stream));
  }
  c.m2t.alloc(size_t(r) * nq);
  cublasHandle_t h = nullptr;
  if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) c.fail(AWG_E_CUDA, "build_coarse_neg: cublasCreate");
  cublasSetStream(h, c.stream);
  const double one = 1.0, zero = 0.0;
  // M2^T (r x nq) = K+ (r x r, symmetric) M1^T
  const cublasStatus_t st =
      cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, r, nq, r, &one, c.k0.kinv.p, r, M1.p, nq, &zero, c.m2t.p, r);
  AWG_CUDA(cudaStreamSynchronize(c.stream));
  cublasDestroy(h);
  if (st != CUBLAS_STATUS_SUCCESS) c.fail(AWG_E_CUDA, "build_coarse_neg: DGEMM");
}

// ---------------------------------------------------------------------------
// A Z on ring-extended supports for coarse_q_combine_az.
namespace {
// AZ_s(e, k) = sum_j A(E_s[e], j) Y_s(loc_s(j), k): thread per (e, k); Omega^s is sorted (binary search)
__global__ void k_az_block(int ne, int lde, const int* __restrict__ eidx, int ns, int lds, const int* __restrict__ om,
                           const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ va,
                           const double* __restrict__ Ys, double* __restrict__ AZs) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x, k = blockIdx.y;
  if (e >= ne) return;
  const int i = eidx[e];
  double acc = 0.0;
  for (int p = rp[i]; p < rp[i + 1]; ++p) {
    const int j = ci[p];
    int lo = 0, hi = ns;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (om[mid] < j) lo = mid + 1;
      else hi = mid;
    }
    if (lo < ns && om[lo] == j) acc = fma(va[p], Ys[lo + (size_t)k * lds], acc);
  }
  AZs[e + (size_t)k * lde] = acc;
}
// m2(q, k) = m2t(k, q): M1 K+ (nq x r) from (K+ M1^T), so that the coarse solve reads column k coalesced
__global__ void k_m2_transpose(int r, int nq, const double* __restrict__ m2t, double* __restrict__ m2) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)r * nq) return;
  const int q = int(t % nq), k = int(t / nq);
  m2[t] = m2t[k + (size_t)q * r];
}
}  // namespace

void build_az(Ctx& c) {
  c.az_on = false;
  c.AZ.release();
  c.m2.release();
  // measured (profiles/r02e/knobs_coarse_az_c{2,3}.json, ms per PCG iteration): c3 3.676 -> 3.643
  // (H3 apply 3.721 -> 3.643); c2 0.4824 -> 0.4851 — there the post-solve chain already
  // overlaps the W branch on the side stream, and the wider dots kernel costs more than
  // the two kernels it saves.  Automatic: on from 16 MB of M2 (option coarse_az = 0 / 1 forces).
  if (!c.m2t.p || c.n0 == 0 || c.k0.rank == 0 || c.nneg == 0) return;
  const long long knob = c.opt("coarse_az", -1);
  if (knob == 0 || (knob < 0 && 8.0 * c.k0.rank * c.nneg < 16.0 * 1024.0 * 1024.0)) return;
  const int N = c.N, n = c.n;
  // E_s = Omega^s plus the columns its rows couple to (A's pattern is symmetric)
  std::vector<int> mark(n, -1), eidx;
  std::vector<long long> eoff(N + 1, 0), azoff(N + 1, 0);
  std::vector<int> ne(N, 0), lde(N, 0);
  for (int s = 0; s < N; ++s) {
    if (c.h_ks[s] > 0) {
      const size_t first = eidx.size();
      for (long long p = c.h_poff[s]; p < c.h_poff[s + 1]; ++p) {
        const int i = c.h_pidx[p];
        if (mark[i] != s) {
          mark[i] = s;
          eidx.push_back(i);
        }
        for (int a = c.h_rp[i]; a < c.h_rp[i + 1]; ++a) {
          const int j = c.h_ci[a];
          if (mark[j] != s) {
            mark[j] = s;
            eidx.push_back(j);
          }
        }
      }
      std::sort(eidx.begin() + first, eidx.end());
      ne[s] = int(eidx.size() - first);
      lde[s] = round_up(ne[s], 4);
    }
    eoff[s + 1] = (long long)eidx.size();
    azoff[s + 1] = azoff[s] + (long long)lde[s] * c.h_ks[s];
  }
  if (azoff[N] == 0) return;
  c.AZ.alloc(size_t(azoff[N]));
  c.AZ.zero(c.stream);
  DArr<int> d_e;
  d_e.upload(eidx, c.stream);
  for (int s = 0; s < N; ++s) {
    if (c.h_ks[s] == 0) continue;
    k_az_block<<<dim3((ne[s] + 255) / 256, c.h_ks[s]), 256, 0, c.stream>>>(
        ne[s], lde[s], d_e.p + eoff[s], c.h_ns[s], c.h_ld[s], c.pidx.p + c.h_poff[s], c.rp.p, c.ci.p, c.va.p,
        c.Y.p + c.h_yoff[s], c.AZ.p + azoff[s]);
    ++c.launches;
  }
  check_launch("az_block");
  // M1 K+ for the second term of the coarse solve
  const int r = c.k0.rank, nq = c.nneg;
  c.m2.alloc(size_t(nq) * r);
  k_m2_transpose<<<int(((long long)r * nq + 255) / 256), 256, 0, c.stream>>>(r, nq, c.m2t.p, c.m2.p);
  ++c.launches;
  check_launch("m2_transpose");
  // combined family arrays: s < N the A- modes on Omega^s, N + s the (A Z)_s blocks on E_s
  std::vector<int> ns2(2 * N), ld2(2 * N), coff2(2 * N + 1, 0), ccol2, pidx2(c.h_pidx);
  std::vector<long long> poff2(2 * N), moff2(2 * N);
  pidx2.insert(pidx2.end(), eidx.begin(), eidx.end());
  const long long P = (long long)c.h_pidx.size();
  const long long az_base = c.AZ.p - c.V.p;  // element offset between the two allocations
  for (int s = 0; s < N; ++s) {
    ns2[s] = c.h_ns[s];
    ld2[s] = c.h_ld[s];
    poff2[s] = c.h_poff[s];
    moff2[s] = c.h_voff[s];
    for (int k = 0; k < c.h_m[s]; ++k)
      if (c.h_lam[c.h_poff[s] + k] != 0.0) ccol2.push_back(k);
    coff2[s + 1] = int(ccol2.size());
  }
  if (coff2[N] != nq) c.fail(AWG_E_STATE, "build_az: A- mode count changed");
  for (int s = 0; s < N; ++s) {
    ns2[N + s] = ne[s];
    ld2[N + s] = lde[s];
    poff2[N + s] = P + eoff[s];
    moff2[N + s] = az_base + azoff[s];
    for (int k = 0; k < c.h_ks[s]; ++k) ccol2.push_back(k);
    coff2[N + s + 1] = int(ccol2.size());
  }
  c.az_ns.upload(ns2, c.stream);
  c.az_ld.upload(ld2, c.stream);
  c.az_poff.upload(poff2, c.stream);
  c.az_moff.upload(moff2, c.stream);
  c.az_coff.upload(coff2, c.stream);
  c.az_ccol.upload(ccol2, c.stream);
  c.az_pidx.upload(pidx2, c.stream);
  BsPlan& b = c.bs_az;
  std::vector<int> ts, tc, nch(2 * N, 0);
  b.maxch = 1;
  int maxcols = 1;
  for (int s = 0; s < 2 * N; ++s) {
    const int cols = coff2[s + 1] - coff2[s];
    if (cols == 0) continue;
    maxcols = std::max(maxcols, cols);
    nch[s] = (ns2[s] + kBsRows - 1) / kBsRows;
    b.maxch = std::max(b.maxch, nch[s]);
    for (int ch = 0; ch < nch[s]; ++ch) {
      ts.push_back(s);
      tc.push_back(ch);
    }
  }
  b.ntask = int(ts.size());
  b.ncg = (maxcols + 7) / 8;
  b.ts.upload(ts, c.stream);
  b.tc.upload(tc, c.stream);
  b.nch.upload(nch, c.stream);
  b.cnt.alloc(2 * N);
  AWG_CUDA(cudaMemsetAsync(b.cnt.p, 0, sizeof(int) * 2 * N, c.stream));
  b.part.alloc(size_t(nq + c.n0) * b.maxch);
  c.az_out.alloc(size_t(nq + c.n0));
  AWG_CUDA(cudaStreamSynchronize(c.stream));
  c.invalidate_graphs();
  c.az_on = true;
}

}  // namespace k
}  // namespace awgb
