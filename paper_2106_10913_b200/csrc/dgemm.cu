// Grouped FP64 GEMM on the B200's FP64 tensor cores (DMMA.8x8x4), for the
// dense contractions of the setup: the block one-level solve of the W build
// (P^s X^s for every subdomain s in one launch, preconditioner.cpp:97-113 with
// OneLevel::apply, preconditioner.cpp:32-57) and the P^s = V+ L+^-1 V+^T
// products that feed it.
//
// Why grouped: one subdomain's product (n_s ~ 5,400 rows x B <= 512 columns)
// is ~130 CTA tiles of 128 x 128 — less than one wave on 148 SMs, so
// per-subdomain library calls leave SMs idle at every tail; one launch over
// all (subdomain, tile) pairs keeps every SM busy until the last wave.
//
// Tiling (default): CTA tile 128 x 64, K-tile 16, 8 warps as 4 (m) x 2 (n),
// warp tile 32 x 32 = 4 x 4 DMMA 8x8x4 fragments (32 fp64 accumulators per
// lane, 126 registers), two CTAs per SM: four warps per scheduler.
// Operands staged by cp.async (16-byte chunks, zero-filled outside the
// matrix) through a 4-stage shared-memory ring; row strides padded so the
// fragment loads are bank-conflict free:
//   A tile as [k][m] with 132 doubles per k (1056 B = 32 B mod 128 B)
//   B tile as [n][k] with 20 doubles per n  (160 B = 32 B mod 128 B)
// Every product is column-major C = A B (A: M x K, B: K x N), or C -= A B
// (GemmDesc::sub), optionally only on the tiles touching the lower triangle.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "awg_internal.cuh"

namespace awgb {
namespace {

constexpr int kBM = 128;

template <int BN, int BK, int ST, int WM = 64, bool TA = false>
struct GCfg {
  static constexpr int kWM = kBM / WM;          // warps along m
  static constexpr int kWarps = kWM * (BN / 32);  // kWM (m) x BN/32 (n) warps of WM x 32
  static constexpr int kT = 32 * kWarps;
  // A tile: [k][m] with kBM + 4 doubles per k (1056 B = 32 B mod 128 B); for
  // C = A^T B (TA, A stored K x M) it is [m][k] like the B tile
  static constexpr int kALd = TA ? BK + 4 : kBM + 4;
  static constexpr int kBLd = BK + 4;   // doubles per n column of the B tile (160 / 288 B = 32 B mod 128 B)
  static constexpr int kAStage = (TA ? kBM : BK) * kALd, kBStage = BN * kBLd;
  static constexpr size_t kSmem = size_t(ST) * (kAStage + kBStage) * sizeof(double);
  static constexpr int kAChunks = BK * kBM / 2, kBChunks = BN * BK / 2;  // 16-byte chunks per tile
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async16(double* dst, const double* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int BN, int BK, int ST, int MINB, int WM, bool TA>
__global__ void __launch_bounds__(GCfg<BN, BK, ST, WM, TA>::kT, MINB)
    k_dgemm_grouped(const GemmDesc* __restrict__ probs, const GemmTile* __restrict__ tiles) {
  using C = GCfg<BN, BK, ST, WM, TA>;
  constexpr int MI = WM / 8;  // 8 x 8 fragments along m per warp
  extern __shared__ __align__(128) double gsm[];
  double* As = gsm;                      // ST x A tile
  double* Bs = gsm + ST * C::kAStage;    // ST x [BN][kBLd]
  const GemmTile t = tiles[blockIdx.x];
  const GemmDesc pr = probs[t.prob];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m0 = t.m0, n0 = t.n0;
  const int KT = (pr.K + BK - 1) / BK;

  // producer addressing, hoisted.  A (no transpose): every chunk of a thread
  // has the same rows (m), columns k0 + kk0 + u * kAStep.  A^T and B: the same
  // rows (k), columns m0 + mm0 + u * step / n0 + nn0 + u * kBStep.  Bounds in
  // M and N are fixed per tile; the K bound only matters on the last K-tile.
  constexpr int kAStep = TA ? C::kT / (BK / 2) : C::kT / 64, kBStep = C::kT / (BK / 2);
  const int kc2 = 2 * (tid % (BK / 2)), row0 = tid / (BK / 2);  // B (and A^T) chunk coordinates
  const int mA = m0 + 2 * (tid & 63), kk0 = tid >> 6;            // A chunk coordinates
  int a_bytes = 0;
  unsigned a_ok = 0;
  const double* a_ptr;
  double* a_dst;
  if constexpr (TA) {
#pragma unroll
    for (int u = 0; u < C::kAChunks / C::kT; ++u) a_ok |= (m0 + row0 + u * kAStep < pr.M) ? (1u << u) : 0u;
    a_ptr = pr.A + (size_t)(m0 + row0) * pr.lda + kc2;
    a_dst = As + row0 * C::kALd + kc2;
  } else {
    a_bytes = 8 * max(0, min(2, pr.M - mA));
    a_ptr = pr.A + (size_t)kk0 * pr.lda + mA;
    a_dst = As + kk0 * C::kALd + 2 * (tid & 63);
  }
  const double* b_ptr = pr.B + (size_t)(n0 + row0) * pr.ldb + kc2;
  unsigned b_ok = 0;
#pragma unroll
  for (int u = 0; u < C::kBChunks / C::kT; ++u) b_ok |= (n0 + row0 + u * kBStep < pr.N) ? (1u << u) : 0u;
  double* b_dst = Bs + row0 * C::kBLd + kc2;
  auto load = [&](int kt, int stage) {
    const int k0 = kt * BK;
    const bool full = k0 + BK <= pr.K;
#pragma unroll
    for (int u = 0; u < C::kAChunks / C::kT; ++u) {
      int bytes;
      const double* src;
      if constexpr (TA) {
        bytes = ((a_ok >> u) & 1u) ? 16 : 0;
        if (!full && bytes) bytes = 8 * max(0, min(2, pr.K - (k0 + kc2)));
        src = a_ptr + (size_t)u * kAStep * pr.lda + k0;
      } else {
        bytes = a_bytes;
        if (!full && k0 + kk0 + u * kAStep >= pr.K) bytes = 0;
        src = a_ptr + (size_t)(k0 + u * kAStep) * pr.lda;
      }
      cp_async16(a_dst + stage * C::kAStage + u * kAStep * C::kALd, bytes ? src : pr.A, bytes);
    }
#pragma unroll
    for (int u = 0; u < C::kBChunks / C::kT; ++u) {
      int bytes = ((b_ok >> u) & 1u) ? 16 : 0;
      if (!full && bytes) bytes = 8 * max(0, min(2, pr.K - (k0 + kc2)));
      cp_async16(b_dst + stage * C::kBStage + u * kBStep * C::kBLd,
                 bytes ? b_ptr + (size_t)u * kBStep * pr.ldb + k0 : pr.B, bytes);
    }
  };

  double acc[MI][4][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < KT) load(s, s);
    cp_commit();
  }
  const int wm = (warp % C::kWM) * WM, wn = (warp / C::kWM) * 32;
  const int fr = lane >> 2, fc = lane & 3;  // fragment row (groupID) / column (thread in group)
  for (int kt = 0; kt < KT; ++kt) {
    cp_wait<ST - 2>();
    __syncthreads();
    if (kt + ST - 1 < KT) load(kt + ST - 1, (kt + ST - 1) % ST);
    cp_commit();
    // A fragment (m = fr, k = fc) and B fragment (k = fc, n = fr) of each 8x8x4 step
    const double* as = TA ? As + (kt % ST) * C::kAStage + (wm + fr) * C::kALd + fc
                          : As + (kt % ST) * C::kAStage + fc * C::kALd + wm + fr;
    const double* bs = Bs + (kt % ST) * C::kBStage + (wn + fr) * C::kBLd + fc;
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      double a[MI], b[4];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = TA ? as[i * 8 * C::kALd + k4 * 4] : as[k4 * 4 * C::kALd + i * 8];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = bs[j * 8 * C::kBLd + k4 * 4];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_wait<0>();
  // epilogue: fragment (i, j) holds C(m0 + wm + 8i + fr, n0 + wn + 8j + 2fc + e)
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int n = n0 + wn + 8 * j + 2 * fc + e;
      if (n >= pr.N) continue;
      double* cn = pr.C + (size_t)n * pr.ldc;
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int m = m0 + wm + 8 * i + fr;
        if (m < pr.M) cn[m] = pr.sub ? cn[m] - acc[i][j][e] : acc[i][j][e];
      }
    }
}

// tile variants (option dgemm_variant; measured in profiles/r01/dgemm_variants.json):
// 0 = 128x64, K 16, 4 stages, 2 CTAs/SM;
// 1 = 128x128, K 16, 4 stages; 2 = 128x128, K 32, 3 stages; 3 = 128x64, K 32, 3 stages;
// warp tile 32 x 32 instead of 64 x 32: 4 = 128x64 (8 warps, 2 CTAs/SM; default —
// 4 warps per scheduler keep the DMMA pipe fed), 5 = 128x128
// (16 warps).  (3 CTAs/SM of 32 x 32 warps spills.)
int gemm_variant(const Ctx& c) { return int(c.opt("dgemm_variant", 4)); }
int gemm_bn(const Ctx& c) {
  const int v = gemm_variant(c);
  return (v == 1 || v == 2 || v == 5) ? 128 : 64;
}

template <int BN, int BK, int ST, int MINB, int WM = 64, bool TA = false>
void launch_gemm(Ctx& c, int ntiles, const GemmDesc* d, const GemmTile* t) {
  using C = GCfg<BN, BK, ST, WM, TA>;
  ensure_dyn_smem((const void*)k_dgemm_grouped<BN, BK, ST, MINB, WM, TA>, C::kSmem);
  k_dgemm_grouped<BN, BK, ST, MINB, WM, TA><<<ntiles, C::kT, C::kSmem, c.stream>>>(d, t);
}

}  // namespace

void GroupedGemm::set(Ctx& c, const std::vector<GemmDesc>& probs, bool transpose_a) {
  ta = transpose_a;
  std::vector<GemmTile> tl;
  flops = 0.0;
  for (int p = 0; p < int(probs.size()); ++p) {
    const GemmDesc& d = probs[p];
    if (d.M <= 0 || d.N <= 0) continue;
    if ((d.lda | d.ldb) & 1) c.fail(AWG_E_ARG, "grouped dgemm: leading dimensions must be even (16-byte chunks)");
    if ((reinterpret_cast<uintptr_t>(d.A) | reinterpret_cast<uintptr_t>(d.B)) & 15)
      c.fail(AWG_E_ARG, "grouped dgemm: operands must be 16-byte aligned");
    flops += 2.0 * d.M * d.N * std::max(d.K, 0);
    // n tiles of one A panel are adjacent in launch order: they run together and
    // share the panel through L2 (A is read from HBM once; B^s stays L2-resident)
    const int bn = ta ? 64 : gemm_bn(c);
    for (int m0 = 0; m0 < d.M; m0 += kBM)
      for (int n0 = 0; n0 < d.N; n0 += bn)
        if (!d.lower || m0 + kBM > n0) tl.push_back({p, m0, n0, 0});
  }
  desc.upload(probs, c.stream);
  tiles.upload(tl, c.stream);
  ntiles = int(tl.size());
}

void GroupedGemm::run(Ctx& c) const {
  if (ntiles == 0) return;
  if (ta) {  // C = A^T B: default tiling only
    launch_gemm<64, 16, 3, 2, 32, true>(c, ntiles, desc.p, tiles.p);  // 3 stages: two CTAs per SM fit
    ++c.launches;
    check_launch("dgemm_grouped_tn");
    return;
  }
  switch (gemm_variant(c)) {
    case 1: launch_gemm<128, 16, 4, 1>(c, ntiles, desc.p, tiles.p); break;
    case 2: launch_gemm<128, 32, 3, 1>(c, ntiles, desc.p, tiles.p); break;
    case 3: launch_gemm<64, 32, 3, 1>(c, ntiles, desc.p, tiles.p); break;
    case 5: launch_gemm<128, 16, 3, 1, 32>(c, ntiles, desc.p, tiles.p); break;
    case 0: launch_gemm<64, 16, 4, 2>(c, ntiles, desc.p, tiles.p); break;
    default: launch_gemm<64, 16, 4, 2, 32>(c, ntiles, desc.p, tiles.p); break;
  }
  ++c.launches;
  check_launch("dgemm_grouped");
}

}  // namespace awgb

// ---------------------------------------------------------------------------
// awg_bench_dgemm: correctness against cuBLAS and the throughput of both on
// the same operands (profiles/dgemm_bench.py).
#include <cublas_v2.h>

namespace awgb {
namespace {
__global__ void k_fill_seeded(size_t n, unsigned long long seed, double* x) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long z = seed + 0x9E3779B97F4A7C15ull * (i + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    x[i] = double(z >> 11) * 0x1.0p-53 * 2.0 - 1.0;
  }
}
__global__ void k_maxabs2(size_t n, const double* a, const double* b, unsigned long long* out) {
  double d = 0.0, r = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    d = fmax(d, fabs(a[i] - b[i]));
    r = fmax(r, fabs(b[i]));
  }
  // non-negative doubles order like their bit patterns
  atomicMax(out, (unsigned long long)__double_as_longlong(d));
  atomicMax(out + 1, (unsigned long long)__double_as_longlong(r));
}
}  // namespace

void bench_grouped_dgemm(Ctx& c, int m, int n, int k, int count, bool ta, int reps, double* out) {
  // A is m x k (lda = round_up(m, 4)) or, with ta, k x m (lda = round_up(k, 4)) and C = A^T B
  const int lda = ta ? round_up(k, 4) : round_up(m, 4), ldb = round_up(k, 4), ldc = round_up(m, 4);
  const size_t sa = size_t(lda) * (ta ? m : k), sb = size_t(ldb) * n, sc = size_t(ldc) * n;
  DArr<double> A, B, C1, C2;
  A.alloc(sa * count);
  B.alloc(sb * count);
  C1.alloc(sc * count);
  C2.alloc(sc * count);
  k_fill_seeded<<<1024, 256, 0, c.stream>>>(sa * count, 1, A.p);
  k_fill_seeded<<<1024, 256, 0, c.stream>>>(sb * count, 2, B.p);
  C1.zero(c.stream);
  C2.zero(c.stream);
  std::vector<GemmDesc> probs;
  for (int q = 0; q < count; ++q)
    probs.push_back({A.p + sa * q, B.p + sb * q, C1.p + sc * q, m, n, k, lda, ldb, ldc});
  GroupedGemm g;
  g.set(c, probs, ta);
  cublasHandle_t h = nullptr;
  if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) c.fail(AWG_E_CUDA, "bench_dgemm: cublasCreate");
  cublasSetStream(h, c.stream);
  const double one = 1.0, zero = 0.0;
  auto lib = [&]() {
    for (int q = 0; q < count; ++q)
      cublasDgemm(h, ta ? CUBLAS_OP_T : CUBLAS_OP_N, CUBLAS_OP_N, m, n, k, &one, A.p + sa * q, lda, B.p + sb * q, ldb, &zero,
                  C2.p + sc * q, ldc);
  };
  cudaEvent_t e0, e1;
  AWG_CUDA(cudaEventCreate(&e0));
  AWG_CUDA(cudaEventCreate(&e1));
  float ms_g = 0.f, ms_l = 0.f;
  g.run(c);
  lib();
  AWG_CUDA(cudaEventRecord(e0, c.stream));
  for (int r = 0; r < reps; ++r) g.run(c);
  AWG_CUDA(cudaEventRecord(e1, c.stream));
  AWG_CUDA(cudaEventSynchronize(e1));
  AWG_CUDA(cudaEventElapsedTime(&ms_g, e0, e1));
  AWG_CUDA(cudaEventRecord(e0, c.stream));
  for (int r = 0; r < reps; ++r) lib();
  AWG_CUDA(cudaEventRecord(e1, c.stream));
  AWG_CUDA(cudaEventSynchronize(e1));
  AWG_CUDA(cudaEventElapsedTime(&ms_l, e0, e1));
  cublasDestroy(h);
  DArr<unsigned long long> mx;
  mx.alloc(2);
  mx.zero(c.stream);
  k_maxabs2<<<1024, 256, 0, c.stream>>>(sc * count, C1.p, C2.p, mx.p);
  const std::vector<unsigned long long> hm = mx.download(c.stream);
  double d, r;
  std::memcpy(&d, &hm[0], 8);
  std::memcpy(&r, &hm[1], 8);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  out[0] = r > 0 ? d / r : d;
  out[1] = ms_g / reps;
  out[2] = ms_l / reps;
  out[3] = g.flops / (out[1] * 1e9);
  out[4] = g.flops / (out[2] * 1e9);
}

}  // namespace awgb
