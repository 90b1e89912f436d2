// C ABI (include/awg_cuda.h): context lifecycle, problem input with the
// reference's validation semantics, factor loading, operator dispatch, PCG.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <numeric>
#include <string>

#include "awg_internal.cuh"

using namespace awgb;

namespace awgb {
namespace {

// Stored-entry multiplicities M_mu(i,j) = #{s : i,j in Omega^s}
// (entry_multiplicities, splitting.cpp:20-33): for each owner subdomain of
// row i, binary search j in the sorted Omega^s.  Records violations of the
// minimal overlap condition for pairs j >= i (check_minimal_overlap,
// partition.cpp:137-156).
__global__ void k_entry_mult(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                             const int* __restrict__ own_off, const int* __restrict__ own_pos,
                             const int* __restrict__ psub, const long long* __restrict__ poff,
                             const int* __restrict__ pidx, int* __restrict__ emult,
                             unsigned long long* __restrict__ first_bad, int* __restrict__ nbad) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    for (int e = rp[i]; e < rp[i + 1]; ++e) {
      const int j = ci[e];
      int count = 0;
      for (int q = own_off[i]; q < own_off[i + 1]; ++q) {
        const int s = psub[own_pos[q]];
        long long lo = poff[s], hi = poff[s + 1] - 1;
        while (lo <= hi) {
          const long long mid = (lo + hi) >> 1;
          const int v = pidx[mid];
          if (v == j) {
            ++count;
            break;
          }
          if (v < j) lo = mid + 1;
          else hi = mid - 1;
        }
      }
      emult[e] = count;
      if (count == 0 && j >= i) {
        atomicAdd(nbad, 1);
        atomicMin(first_bad, (unsigned long long)i * (unsigned long long)n + (unsigned long long)j);
      }
    }
  }
}

// core = Lambda_-^-1 - V_-^T W   (AwgPreconditioner ctor, preconditioner.cpp:134-146);
// warp per entry (i, j).
__global__ void k_core(int nm, const int* __restrict__ neg_s, const int* __restrict__ neg_k,
                       const double* __restrict__ V, const long long* __restrict__ voff, const int* __restrict__ ns,
                       const int* __restrict__ ld, const long long* __restrict__ poff, const int* __restrict__ pidx,
                       const double* __restrict__ W, int ldw, const double* __restrict__ negw,
                       double* __restrict__ core) {
  const int lane = threadIdx.x & 31;
  const long long e = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (e >= (long long)nm * nm) return;
  const int i = int(e % nm), j = int(e / nm);
  const int s = neg_s[i], n = ns[s];
  const double* v = V + voff[s] + (size_t)neg_k[i] * ld[s];
  const int* idx = pidx + poff[s];
  const double* w = W + (size_t)j * ldw;
  double acc = 0.0;
  for (int l = lane; l < n; l += 32) acc = fma(v[l], w[idx[l]], acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) core[i + (size_t)j * nm] = -acc + (i == j ? 1.0 / negw[j] : 0.0);
}

// synthetic factor values for kernel timing (awg_synthetic_factors)
__global__ void k_fill_hash(size_t count, unsigned long long seed, double* __restrict__ v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long z = seed + 0x9E3779B97F4A7C15ull * (i + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    v[i] = double(z >> 11) * 0x1.0p-53 - 0.5;
  }
}

// lu_factor (dense.cpp:368-393): partial pivoting, first maximum, full row
// swaps; single CTA (n_minus is small).
__global__ void k_lu_factor(int m, double* __restrict__ a, int* __restrict__ perm, int* __restrict__ singular) {
  __shared__ int piv;
  for (int i = threadIdx.x; i < m; i += blockDim.x) perm[i] = i;
  __syncthreads();
  for (int k = 0; k < m; ++k) {
    if (threadIdx.x == 0) {
      int p = k;
      for (int i = k + 1; i < m; ++i)
        if (fabs(a[i + (size_t)k * m]) > fabs(a[p + (size_t)k * m])) p = i;
      piv = p;
      if (a[p + (size_t)k * m] == 0.0) *singular = 1;
    }
    __syncthreads();
    if (*singular) return;
    const int p = piv;
    if (p != k) {
      for (int j = threadIdx.x; j < m; j += blockDim.x) {
        const double t = a[k + (size_t)j * m];
        a[k + (size_t)j * m] = a[p + (size_t)j * m];
        a[p + (size_t)j * m] = t;
      }
      if (threadIdx.x == 0) {
        const int t = perm[k];
        perm[k] = perm[p];
        perm[p] = t;
      }
    }
    __syncthreads();
    const double inv = 1.0 / a[k + (size_t)k * m];
    for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) a[i + (size_t)k * m] *= inv;
    __syncthreads();
    for (int j = k + 1; j < m; ++j) {
      const double f = a[k + (size_t)j * m];
      if (f == 0.0) continue;
      for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) a[i + (size_t)j * m] -= a[i + (size_t)k * m] * f;
    }
    __syncthreads();
  }
}

void upload_padded(DArr<double>& dst, const std::vector<long long>& off, long long total, const double* src,
                   const std::vector<int>& rows, const std::vector<int>& lds, const std::vector<int>& cols,
                   cudaStream_t st) {
  dst.alloc(size_t(std::max<long long>(total, 1)));
  dst.zero(st);
  size_t s_off = 0;
  for (size_t s = 0; s < rows.size(); ++s) {
    if (cols[s] > 0 && rows[s] > 0)
      AWG_CUDA(cudaMemcpy2DAsync(dst.p + off[s], sizeof(double) * lds[s], src + s_off, sizeof(double) * rows[s],
                                 sizeof(double) * rows[s], cols[s], cudaMemcpyHostToDevice, st));
    s_off += size_t(rows[s]) * cols[s];
  }
}

void set_factor(Ctx& c, CoarseFactor& f, int dim, int r, const int* ret, const double* l11) {
  f.dim = dim;
  f.rank = r;
  f.h_retained.assign(ret, ret + r);
  f.h_l11.assign(l11, l11 + size_t(r) * r);
  f.retained.upload(f.h_retained, c.stream);
  DArr<double> l;
  if (r) l.upload(f.h_l11, c.stream);
  k::coarse_inverse(c, l.p, f);
}

}  // namespace

void finalize_factors(Ctx& c) {
  const int N = c.N;
  // local layout
  c.h_ld.resize(N);
  c.h_voff.assign(N + 1, 0);
  c.h_yoff.assign(N + 1, 0);
  for (int s = 0; s < N; ++s) {
    c.h_ld[s] = round_up(c.h_ns[s], 4);
    c.h_voff[s + 1] = c.h_voff[s] + (long long)c.h_ld[s] * c.h_ns[s];
    c.h_yoff[s + 1] = c.h_yoff[s] + (long long)c.h_ld[s] * c.h_ks[s];
  }
  c.ns.upload(c.h_ns, c.stream);
  c.ld.upload(c.h_ld, c.stream);
  c.msz.upload(c.h_m, c.stream);
  c.voff.upload(c.h_voff, c.stream);
  c.yoff.upload(c.h_yoff, c.stream);
  {
    std::vector<double> rl(c.h_lam.size(), 0.0);
    for (size_t i = 0; i < rl.size(); ++i)
      if (c.h_lam[i] > 0.0) rl[i] = 1.0 / c.h_lam[i];
    c.rlam.upload(rl, c.stream);
  }
  // local-solve task lists: NN always (V^s columns j >= n_nonpos), AS/AS+ when configured
  auto build_plan = [&](LocalPlan& pl, bool tri) {
    std::vector<GemvTTask> tT;
    std::vector<GemvTask> t;
    std::vector<int> nkc(N, 0);
    pl.kcmax = 1;
    for (int s = 0; s < N; ++s) {
      const int jstart = tri ? 0 : c.h_m[s];
      for (int j0 = jstart; j0 < c.h_ns[s]; j0 += 64) tT.push_back({s, j0, std::min(j0 + 64, c.h_ns[s]), 0});
      // split-K over column chunks of gemv_cols (the last chunk takes the remainder)
      const int cols = c.h_ns[s] - jstart;
      const int kcs = std::max(1, cols / c.gemv_cols);
      nkc[s] = kcs;
      pl.kcmax = std::max(pl.kcmax, kcs);
      for (int kc = 0; kc < kcs; ++kc) {
        const int j0 = jstart + int((long long)cols * kc / kcs);
        const int j1 = jstart + int((long long)cols * (kc + 1) / kcs);
        for (int i0 = 0; i0 < c.h_ns[s]; i0 += c.rows_per_gemv) {
          // upper-triangular U^s: columns j < i0 are zero for the whole panel; an
          // empty task still writes its (zero) partial slot
          const int jj0 = tri ? std::max(j0, std::min(i0, j1)) : j0;
          t.push_back({s, i0, jj0, j1, kc, 0});
        }
      }
    }
    pl.tT.upload(tT, c.stream);
    pl.t.upload(t, c.stream);
    pl.nkc.upload(nkc, c.stream);
    pl.cols_max = 1;
    for (const auto& tk : t) pl.cols_max = std::max(pl.cols_max, tk.j1 - tk.j0);
    // single-pass plan (NN): column ranges sized for >= 4 CTAs per SM in total
    int ldmax = 0;
    long long cols_total = 0;
    for (int s = 0; s < N; ++s) {
      ldmax = std::max(ldmax, c.h_ld[s]);
      cols_total += c.h_ns[s] - (tri ? 0 : c.h_m[s]);
    }
    pl.fused = ldmax <= 6144 && c.use_fused;
    if (pl.fused) {
      const long long target = std::max<long long>((long long)c.fused_chunks_per_sm * c.sm_count, N);  // queue granularity
      // >= 128 columns per task keeps the per-task restriction gather and partial
      // write (about 3 columns' worth of traffic) below ~3%
      const int cs = int(std::max<long long>(c.fused_min_cols, (cols_total + target - 1) / target));
      std::vector<GemvTask> tf, tail;
      std::vector<int> nkf(N, 0);
      pl.kcmax_f = 1;
      for (int s = 0; s < N; ++s) {
        const int jstart = tri ? 0 : c.h_m[s];
        int cols = c.h_ns[s] - jstart;
        // guided tail (NN): the last tail_pct% of each subdomain's columns in
        // quarter-size tasks, queued after every bulk task, so the persistent
        // CTAs finish together
        const int cs_tail = std::max(32, cs / 4);
        int tcols = (!tri && c.fused_tail_pct > 0) ? (cols * c.fused_tail_pct / 100) / cs_tail * cs_tail : 0;
        if (tcols >= cols) tcols = 0;
        cols -= tcols;
        const int kcs = std::max(1, (cols + cs / 2) / cs);
        for (int kc = 0; kc < kcs; ++kc) {
          // triangular factor: equal-area chunks (column j costs j + 1 rows)
          const double f0 = tri ? std::sqrt(double(kc) / kcs) : double(kc) / kcs;
          const double f1 = tri ? std::sqrt(double(kc + 1) / kcs) : double(kc + 1) / kcs;
          const int j0 = jstart + int(cols * f0);
          const int j1 = kc + 1 == kcs ? jstart + cols : jstart + int(cols * f1);
          tf.push_back({s, 0, j0, j1, kc, 0});
        }
        int kc = kcs;
        for (int j0 = jstart + cols; j0 < jstart + cols + tcols; j0 += cs_tail, ++kc)
          tail.push_back({s, 0, j0, j0 + cs_tail, kc, 0});
        nkf[s] = kc;
        pl.kcmax_f = std::max(pl.kcmax_f, kc);
      }
      tf.insert(tf.end(), tail.begin(), tail.end());
      pl.static_grid = 0;
      pl.cta_off.release();
      if (!tri && c.fused_static) {
        // static split (NN): the subdomains' column lists laid end to end and
        // cut into G shares of equal column counts, each CTA's share split at
        // subdomain ends into tasks, so no SM idles at the end as in the work
        // queue's last round.  Equal columns, not equal bytes: every column
        // costs a CTA the same R rows per thread of shared-memory traffic and
        // FMAs whatever its ld_s, and equal-byte shares measured 2% slower
        // (option fused_static_cols=0, profiles/r01f/knobs_static_cols_c2.json).
        // Not for the triangular U^s (AS / AS+): there a column moves j + 1
        // rows but still costs a full column of compute, and equal-byte shares
        // measured 18% slower than the queue (profiles/r01f/knobs_static_as_c2.json)
        const int G = int(std::max<long long>(1, std::min<long long>(cols_total, std::max(1, c.sm_count - c.fused_reserve))));
        const bool cols_only = c.opt("fused_static_cols", 1) != 0;  // 0: equal bytes instead (A/B)
        auto cost = [&](int s, int) -> long long { return cols_only ? 1LL : c.h_ld[s]; };
        long long T = 0;
        for (int s = 0; s < N; ++s)
          for (int j = c.h_m[s]; j < c.h_ns[s]; ++j) T += cost(s, j);
        tf.clear();
        std::fill(nkf.begin(), nkf.end(), 0);
        std::vector<int> off(G + 1, 0);
        int b = 0;
        long long acc = 0;
        for (int s = 0; s < N; ++s) {
          int j0 = c.h_m[s];
          for (int j = j0; j < c.h_ns[s]; ++j) {
            acc += cost(s, j);
            while (b < G - 1 && acc * G >= T * (b + 1)) {  // CTA b's share ends after column j
              if (j + 1 > j0) tf.push_back({s, 0, j0, j + 1, nkf[s]++, 0});
              j0 = j + 1;
              off[++b] = int(tf.size());
            }
          }
          if (c.h_ns[s] > j0) tf.push_back({s, 0, j0, c.h_ns[s], nkf[s]++, 0});
        }
        for (int bb = b + 1; bb <= G; ++bb) off[bb] = int(tf.size());
        pl.kcmax_f = 1;
        for (int v : nkf) pl.kcmax_f = std::max(pl.kcmax_f, v);
        pl.cta_off.upload(off, c.stream);
        pl.static_grid = G;
      }
      pl.tf.upload(tf, c.stream);
      pl.nkc_f.upload(nkf, c.stream);
    }
  };
  c.one_level = c.cfg.one_level;
  build_plan(c.plan_nn, false);
  if (c.one_level != 2) build_plan(c.plan_as, true);
  const int kcmax = std::max({c.plan_nn.kcmax, c.plan_nn.fused ? c.plan_nn.kcmax_f : 1,
                              c.one_level != 2 ? c.plan_as.kcmax : 1,
                              (c.one_level != 2 && c.plan_as.fused) ? c.plan_as.kcmax_f : 1});
  c.wpart_nn.alloc(size_t(kcmax) * std::max<long long>(c.P, 1));
  c.wpart_nn.zero(c.stream);
  // A- modes: k < n_nonpos with lambda != 0 (splitting.cpp:129-131), ascending (s, k)
  std::vector<int> ns_, nk_, noff(N + 1, 0);
  std::vector<double> nw_;
  for (int s = 0; s < N; ++s) {
    for (int k = 0; k < c.h_m[s]; ++k) {
      const double lam = c.h_lam[c.h_poff[s] + k];
      if (lam == 0.0) continue;
      ns_.push_back(s);
      nk_.push_back(k);
      nw_.push_back(-lam);
    }
    noff[s + 1] = int(ns_.size());
  }
  c.nneg = int(ns_.size());
  c.neg_s.upload(ns_, c.stream);
  c.neg_k.upload(nk_, c.stream);
  c.neg_w.upload(nw_, c.stream);
  c.negoff.upload(noff, c.stream);
  c.neg_c.alloc(std::max(c.nneg, 1));
  // coarse columns
  std::vector<int> zs, zl, koff(N + 1, 0);
  for (int s = 0; s < N; ++s) {
    for (int k = 0; k < c.h_ks[s]; ++k) {
      zs.push_back(s);
      zl.push_back(k);
    }
    koff[s + 1] = int(zs.size());
  }
  c.n0 = int(zs.size());
  c.zcol_s.upload(zs, c.stream);
  c.zcol_loc.upload(zl, c.stream);
  c.koff.upload(koff, c.stream);
  auto build_bs = [&](BsPlan& b, const std::vector<int>& off) {
    std::vector<int> ts, tc, nch(N, 0);
    b.maxch = 1;
    for (int s = 0; s < N; ++s) {
      if (off[s + 1] == off[s]) continue;
      nch[s] = (c.h_ns[s] + kBsRows - 1) / kBsRows;
      b.maxch = std::max(b.maxch, nch[s]);
      for (int ch = 0; ch < nch[s]; ++ch) {
        ts.push_back(s);
        tc.push_back(ch);
      }
    }
    b.ntask = int(ts.size());
    int maxcols = 1;
    for (int s = 0; s < N; ++s) maxcols = std::max(maxcols, off[s + 1] - off[s]);
    b.ncg = (maxcols + 7) / 8;
    b.ts.upload(ts, c.stream);
    b.tc.upload(tc, c.stream);
    b.nch.upload(nch, c.stream);
    b.cnt.alloc(N);
    AWG_CUDA(cudaMemsetAsync(b.cnt.p, 0, sizeof(int) * N, c.stream));
    b.part.alloc(size_t(std::max(off[N], 1)) * b.maxch);
  };
  build_bs(c.bs_neg, noff);
  build_bs(c.bs_z, koff);
  k::owner_tables(c);
  c.alloc_work();
  AWG_CUDA(cudaStreamSynchronize(c.stream));
}

void build_core(Ctx& c) {
  if (c.nm == 0) return;
  c.core_lu.alloc(size_t(c.nm) * c.nm);
  c.core_perm.alloc(c.nm);
  const long long pairs = (long long)c.nm * c.nm;
  k_core<<<int((pairs + 7) / 8), 256, 0, c.stream>>>(c.nm, c.neg_s.p, c.neg_k.p, c.V.p, c.voff.p, c.ns.p, c.ld.p,
                                                    c.poff.p, c.pidx.p, c.W.p, c.ldw, c.neg_weights.p,
                                                    c.core_lu.p);
  DArr<int> sing;
  sing.alloc(1);
  sing.zero(c.stream);
  k_lu_factor<<<1, 1024, 0, c.stream>>>(c.nm, c.core_lu.p, c.core_perm.p, sing.p);
  c.launches += 2;
  check_launch("core");
  int h = 0;
  AWG_CUDA(cudaMemcpyAsync(&h, sing.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  AWG_CUDA(cudaStreamSynchronize(c.stream));
  if (h) c.fail(AWG_E_ARG, "lu_factor: singular matrix");
}

}  // namespace awgb

// ===========================================================================
namespace {

template <class F>
int guarded(awg_ctx* ctx, F f) {
  if (!ctx) return AWG_E_ARG;
  Ctx& c = ctx->c;
  try {
    if (c.device >= 0) cudaSetDevice(c.device);
    f(c);
    c.err.clear();
    c.err_index = -1;
    return AWG_OK;
  } catch (const AwgError& e) {
    c.err = e.what();
    c.err_index = e.index;
    return e.code;
  } catch (const std::bad_alloc&) {
    c.err = "host allocation failed";
    return AWG_E_CUDA;
  } catch (const std::exception& e) {
    c.err = e.what();
    return AWG_E_CUDA;
  }
}

void check_config(Ctx& c, const awg_config& cfg) {
  if (cfg.one_level < 0 || cfg.one_level > 2) c.fail(AWG_E_ARG, "one_level must be 0 (AS), 1 (AS_PLUS) or 2 (NN)");
  if (cfg.fixed_k > 0 && cfg.one_level != 2) c.fail(AWG_E_ARG, "fixed-k selection is defined for the NN pencil only");
  // ThresholdSpec ranges (coarse.cpp:9-24)
  if (cfg.use_coarse && cfg.one_level == 1 && !(cfg.tau_flat > 1.0))
    c.fail(AWG_E_ARG, "AS_PLUS threshold requires tau_flat > 1");
  if (cfg.use_coarse && cfg.one_level == 0 && (!(cfg.tau_sharp > 0.0 && cfg.tau_sharp < 1.0) || !(cfg.tau_flat > 1.0)))
    c.fail(AWG_E_ARG, "AS threshold requires 0 < tau_sharp < 1 and tau_flat > 1");
  if (cfg.composition != 0 && cfg.composition != 1) c.fail(AWG_E_ARG, "composition must be 0 or 1");
  if (cfg.awg_mode < 0 || cfg.awg_mode > 3) c.fail(AWG_E_ARG, "awg_mode must be 0..3");
  if (cfg.use_coarse && cfg.one_level == 2 && cfg.fixed_k <= 0 && !(cfg.tau_sharp > 0.0 && cfg.tau_sharp < 1.0))
    c.fail(AWG_E_ARG, "NN threshold requires 0 < tau_sharp < 1");
}

}  // namespace

extern "C" {

int awg_create(awg_ctx** out, int device) {
  if (!out) return AWG_E_ARG;
  *out = nullptr;
  awg_ctx* ctx = new (std::nothrow) awg_ctx();
  if (!ctx) return AWG_E_CUDA;
  Ctx& c = ctx->c;
  c.device = device;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    c.device = -1;
    c.err = "no CUDA device visible (the AWG path has no CPU fallback)";
    *out = ctx;
    return AWG_E_CUDA;
  }
  int rc = guarded(ctx, [&](Ctx& cc) {
    AWG_CUDA(cudaSetDevice(device));
    // the solve's critical path (main stream) outranks the concurrent W branch
    // (side stream); graph kernel nodes keep these priorities (ops.cu)
    int lo = 0, hi = 0;
    AWG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    AWG_CUDA(cudaStreamCreateWithPriority(&cc.stream, cudaStreamNonBlocking, hi));
    AWG_CUDA(cudaStreamCreateWithPriority(&cc.side, cudaStreamNonBlocking, lo));
    AWG_CUDA(cudaEventCreateWithFlags(&cc.ev_fork, cudaEventDisableTiming));
    AWG_CUDA(cudaEventCreateWithFlags(&cc.ev_join, cudaEventDisableTiming));
    AWG_CUDA(cudaEventCreateWithFlags(&cc.ev_mid, cudaEventDisableTiming));
    AWG_CUDA(cudaDeviceGetAttribute(&cc.sm_count, cudaDevAttrMultiProcessorCount, device));
  });
  *out = ctx;
  return rc;
}

void awg_destroy(awg_ctx* ctx) {
  if (!ctx) return;
  if (ctx->c.device >= 0) {
    cudaSetDevice(ctx->c.device);
    if (ctx->c.stream) cudaStreamSynchronize(ctx->c.stream);
  }
  cudaStream_t s = ctx->c.stream, side = ctx->c.side;
  cudaEvent_t e0 = ctx->c.ev_fork, e1 = ctx->c.ev_join, e2 = ctx->c.ev_mid;
  delete ctx;
  if (s) cudaStreamDestroy(s);
  if (side) cudaStreamDestroy(side);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (e2) cudaEventDestroy(e2);
}

const char* awg_last_error(const awg_ctx* ctx) { return ctx ? ctx->c.err.c_str() : "null context"; }
int awg_last_error_index(const awg_ctx* ctx) { return ctx ? ctx->c.err_index : -1; }
long long awg_launch_count(const awg_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

int awg_set_option(awg_ctx* ctx, const char* name, long long value) {
  return guarded(ctx, [&](Ctx& c) {
    if (!name) c.fail(AWG_E_ARG, "set_option: null name");
    const std::string k = name;
    const int v = int(value);
    if (k == "pdl") c.use_pdl = v != 0;
    else if (k == "nn_two_pass") c.use_fused = v == 0;
    else if (k == "fused_cpb") c.fused_cpb = v;
    else if (k == "fused_hold") c.fused_hold = v != 0;
    else if (k == "fused_prefetch") c.fused_prefetch = v != 0;
    else if (k == "fused_static") c.fused_static = v != 0;
    else if (k == "pcg_adaptive") c.pcg_adaptive = v != 0;
    else if (k == "pdl_local") c.pdl_local = v != 0;
    else if (k == "rows_group") c.rows_group = v;
    else if (k == "pdl_early") c.pdl_early = v != 0 ? 1 : 0;
    else if (k == "w_split") c.w_split = v;
    else if (k == "fused_nbuf") c.fused_nbuf = v;
    else if (k == "fused_chunks") c.fused_chunks_per_sm = std::max(1, v);
    else if (k == "fused_reserve") c.fused_reserve = std::max(0, v);
    else if (k == "fused_min_cols") c.fused_min_cols = std::max(8, v);
    else if (k == "fused_tail") c.fused_tail_pct = std::max(0, std::min(90, v));
    else if (k == "fused_static_cols" || k == "synth_nm" || k == "dgemm_variant" || k == "coarse_neg" ||
             k == "verbose" || k == "wbuild_cublas" || k == "setup_cusolver" || k == "eig_probe" || k == "eig_split" || k == "coarse_az")
      c.opts[k] = value;
    else
      c.fail(AWG_E_ARG, "set_option: unknown option " + k);
  });
}

int awg_pivoted_factor(awg_ctx* ctx, int n, const double* G, int exact, int* rank, int* retained, double* l11) {
  return guarded(ctx, [&](Ctx& c) {
    if (n < 0 || (n > 0 && !G) || !rank) c.fail(AWG_E_ARG, "pivoted_factor: bad arguments");
    CoarseFactor f;
    pivoted_factor_of(c, n, G, exact ? 1 : 0, f);
    *rank = f.rank;
    if (retained) std::copy(f.h_retained.begin(), f.h_retained.end(), retained);
    if (l11) std::copy(f.h_l11.begin(), f.h_l11.end(), l11);
  });
}

int awg_coarse_solve(awg_ctx* ctx, int which, const double* b, double* x) {
  return guarded(ctx, [&](Ctx& c) {
    if (!c.have_factors) c.fail(AWG_E_STATE, "coarse_solve: preconditioner not set up");
    if (which != 0 && which != 1) c.fail(AWG_E_ARG, "coarse_solve: which must be 0 (K0) or 1 (KW)");
    const CoarseFactor& f = which == 0 ? c.k0 : c.kw;
    if (!b || !x) c.fail(AWG_E_ARG, "coarse_solve: null vector");
    if (f.dim == 0) return;
    DArr<double> db, dx;
    db.alloc(f.dim);
    dx.alloc(f.dim);
    AWG_CUDA(cudaMemcpyAsync(db.p, b, sizeof(double) * f.dim, cudaMemcpyHostToDevice, c.stream));
    k::rr_solve(c, f, db.p, dx.p, nullptr);
    AWG_CUDA(cudaMemcpyAsync(x, dx.p, sizeof(double) * f.dim, cudaMemcpyDeviceToHost, c.stream));
    AWG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int awg_bench_eig(awg_ctx* ctx, int n, int count, int kind, unsigned long long seed, double* out) {
  return guarded(ctx, [&](Ctx& c) {
    if (n < 2 || count < 1 || !out) c.fail(AWG_E_ARG, "bench_eig: bad arguments");
    eig_check(c, n, count, kind, seed, out);
  });
}

int awg_set_matrix(awg_ctx* ctx, int n, const int* rp, const int* ci, const double* va) {
  return guarded(ctx, [&](Ctx& c) {
    if (c.device < 0) c.fail(AWG_E_CUDA, "no CUDA device");
    if (n <= 0 || !rp || !ci || !va) c.fail(AWG_E_ARG, "set_matrix: bad arguments");
    if (rp[0] != 0) c.fail(AWG_E_ARG, "set_matrix: row_offsets[0] must be 0");
    for (int i = 0; i < n; ++i) {
      if (rp[i + 1] < rp[i]) c.fail(AWG_E_ARG, "set_matrix: row_offsets not monotone");
      for (int k = rp[i]; k < rp[i + 1]; ++k) {
        if (ci[k] < 0 || ci[k] >= n) c.fail(AWG_E_ARG, "set_matrix: column index out of range");
        if (k > rp[i] && ci[k] <= ci[k - 1]) c.fail(AWG_E_ARG, "set_matrix: column indices not strictly increasing");
      }
    }
    c.n = n;
    c.nnz = rp[n];
    c.asm_kind = -1;
    c.h_rhs_asm.clear();
    c.h_rp.assign(rp, rp + n + 1);
    c.h_ci.assign(ci, ci + c.nnz);
    c.h_va.assign(va, va + c.nnz);
    c.rp.upload(c.h_rp, c.stream);
    c.ci.upload(c.h_ci, c.stream);
    c.va.upload(c.h_va, c.stream);
    c.have_factors = false;
    c.N = 0;
    AWG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int awg_set_partition(awg_ctx* ctx, int N, const long long* off, const int* idx) {
  return guarded(ctx, [&](Ctx& c) {
    if (c.n == 0) c.fail(AWG_E_STATE, "set_partition: set the matrix first");
    if (N <= 0 || !off || !idx) c.fail(AWG_E_ARG, "set_partition: bad arguments");
    if (off[0] != 0) c.fail(AWG_E_ARG, "set_partition: offsets[0] must be 0");
    const int n = c.n;
    std::vector<int> mult(n, 0);
    std::vector<int> ns(N);
    for (int s = 0; s < N; ++s) {
      if (off[s + 1] <= off[s]) c.fail(AWG_E_ARG, "set_partition: empty subdomain " + std::to_string(s));
      ns[s] = int(off[s + 1] - off[s]);
      for (long long p = off[s]; p < off[s + 1]; ++p) {
        if (idx[p] < 0 || idx[p] >= n) c.fail(AWG_E_ARG, "partition index out of range");
        if (p > off[s] && idx[p] <= idx[p - 1]) c.fail(AWG_E_ARG, "set_partition: indices must be sorted and unique");
        ++mult[idx[p]];
      }
    }
    for (int i = 0; i < n; ++i)
      if (mult[i] == 0) c.fail(AWG_E_OVERLAP, "partition does not cover dof " + std::to_string(i), i);
    const long long P = off[N];
    c.N = N;
    c.P = P;
    c.h_ns = ns;
    c.h_poff.assign(off, off + N + 1);
    c.h_pidx.assign(idx, idx + P);
    c.h_mult = mult;
    std::vector<int> psub(P), own_off(n + 1, 0), own_pos(P);
    std::vector<double> ds(P);
    for (int s = 0; s < N; ++s)
      for (long long p = off[s]; p < off[s + 1]; ++p) {
        psub[p] = s;
        ds[p] = 1.0 / mult[idx[p]];
        ++own_off[idx[p] + 1];
      }
    for (int i = 0; i < n; ++i) own_off[i + 1] += own_off[i];
    std::vector<int> fill(own_off.begin(), own_off.end() - 1);
    for (long long p = 0; p < P; ++p) own_pos[fill[idx[p]]++] = int(p);
    c.pidx.upload(c.h_pidx, c.stream);
    c.poff.upload(c.h_poff, c.stream);
    c.psub.upload(psub, c.stream);
    c.ds.upload(ds, c.stream);
    c.own_off.upload(own_off, c.stream);
    c.own_pos.upload(own_pos, c.stream);
    c.mult.upload(mult, c.stream);
    // minimal overlap / entry multiplicities on the device
    c.emult.alloc(c.nnz);
    DArr<unsigned long long> first;
    DArr<int> nbad;
    first.alloc(1);
    nbad.alloc(1);
    AWG_CUDA(cudaMemsetAsync(first.p, 0xff, sizeof(unsigned long long), c.stream));
    nbad.zero(c.stream);
    k_entry_mult<<<std::max(1, std::min((n + 255) / 256, c.sm_count * 8)), 256, 0, c.stream>>>(
        n, c.rp.p, c.ci.p, c.own_off.p, c.own_pos.p, c.psub.p, c.poff.p, c.pidx.p, c.emult.p, first.p, nbad.p);
    ++c.launches;
    check_launch("entry_mult");
    unsigned long long hf = 0;
    int hb = 0;
    AWG_CUDA(cudaMemcpyAsync(&hf, first.p, sizeof(hf), cudaMemcpyDeviceToHost, c.stream));
    AWG_CUDA(cudaMemcpyAsync(&hb, nbad.p, sizeof(hb), cudaMemcpyDeviceToHost, c.stream));
    AWG_CUDA(cudaStreamSynchronize(c.stream));
    if (hb > 0) {
      const long long fi = (long long)(hf / (unsigned long long)n), fj = (long long)(hf % (unsigned long long)n);
      c.fail(AWG_E_OVERLAP, "external partition violates minimal overlap on " + std::to_string(hb) +
                                " pair(s), first (" + std::to_string(fi) + "," + std::to_string(fj) + ")");
    }
    c.have_factors = false;
  });
}

int awg_load_factors(awg_ctx* ctx, const awg_config* cfg, const awg_factors* f) {
  return guarded(ctx, [&](Ctx& c) {
    if (c.N == 0) c.fail(AWG_E_STATE, "load_factors: set matrix and partition first");
    if (!cfg || !f || !f->lam || !f->V || !f->n_nonpos || !f->n_zero || !f->ks)
      c.fail(AWG_E_ARG, "load_factors: missing arrays");
    check_config(c, *cfg);
    c.cfg = *cfg;
    c.lu_semantics = cfg->lu_semantics;
    const int N = c.N;
    c.h_m.assign(f->n_nonpos, f->n_nonpos + N);
    c.h_nzero.assign(f->n_zero, f->n_zero + N);
    c.h_ks.assign(f->ks, f->ks + N);
    if (!cfg->use_coarse) std::fill(c.h_ks.begin(), c.h_ks.end(), 0);
    c.h_lam.assign(f->lam, f->lam + c.P);
    c.h_eps.assign(N, 0.0);
    c.h_plam.clear();
    c.lam.upload(c.h_lam, c.stream);
    finalize_factors(c);
    std::vector<int> ns = c.h_ns;
    upload_padded(c.V, c.h_voff, c.h_voff[N], f->V, ns, c.h_ld, ns, c.stream);
    long long n0 = 0;
    for (int s = 0; s < N; ++s) n0 += c.h_ks[s];
    if (n0 > 0) {
      if (!f->Y || !f->k0_retained || !f->k0_l11) c.fail(AWG_E_ARG, "load_factors: coarse factors missing");
      upload_padded(c.Y, c.h_yoff, c.h_yoff[N], f->Y, ns, c.h_ld, c.h_ks, c.stream);
      set_factor(c, c.k0, int(n0), f->r0, f->k0_retained, f->k0_l11);
    } else {
      c.k0.clear();
    }
    c.nm = (cfg->awg_mode != 0) ? f->n_minus : 0;
    if (c.nm > 0 && c.nm != c.nneg)
      c.fail(AWG_E_ARG, "load_factors: n_minus does not match the strictly negative modes of lam / n_nonpos");
    c.ldw = round_up(c.n, 4);
    if (c.nm > 0) {
      if (!f->W || !f->kw_retained || !f->kw_l11) c.fail(AWG_E_ARG, "load_factors: W factors missing");
      std::vector<long long> woff = {0};
      upload_padded(c.W, woff, (long long)c.ldw * c.nm, f->W, {c.n}, {c.ldw}, {c.nm}, c.stream);
      set_factor(c, c.kw, c.nm, f->rw, f->kw_retained, f->kw_l11);
      if (f->neg_weights) {
        c.h_neg_weights.assign(f->neg_weights, f->neg_weights + c.nm);
        c.neg_weights.upload(c.h_neg_weights, c.stream);
      }
    }
    c.alloc_work();
    if (cfg->awg_mode == 3 && c.nm > 0) {
      if (!f->neg_weights) c.fail(AWG_E_ARG, "load_factors: INEX needs neg_weights");
      build_core(c);
    }
    // AS / AS+: the local Cholesky factors are computed here from A (and the
    // loaded V^s for the A+ blocks); Cholesky factors are unique
    if (c.one_level != 2) build_local_cholesky(c);
    k::build_coarse_neg(c);
    k::build_az(c);
    AWG_CUDA(cudaStreamSynchronize(c.stream));
    c.have_factors = true;
  });
}

int awg_synthetic_factors(awg_ctx* ctx, int m_per_sub, unsigned long long seed) {
  return guarded(ctx, [&](Ctx& c) {
    if (c.N == 0) c.fail(AWG_E_STATE, "synthetic_factors: set matrix and partition first");
    awg_config cfg{};
    cfg.one_level = 2;
    cfg.composition = 1;
    cfg.use_coarse = 0;
    cfg.awg_mode = 0;
    cfg.tau_sharp = 0.1;
    cfg.tau_flat = 10.0;
    cfg.w_rtol = 1e-10;
    c.cfg = cfg;
    const int N = c.N;
    c.h_m.assign(N, 0);
    c.h_nzero.assign(N, 0);
    c.h_ks.assign(N, 0);
    c.h_lam.assign(c.P, 1.0);
    for (int s = 0; s < N; ++s) {
      c.h_m[s] = c.h_nzero[s] = std::max(0, std::min(m_per_sub, c.h_ns[s]));
      for (int j = 0; j < c.h_ns[s]; ++j) c.h_lam[c.h_poff[s] + j] = j < c.h_m[s] ? 0.0 : 1.0 + 1e-3 * j;
    }
    c.h_eps.assign(N, 0.0);
    c.lam.upload(c.h_lam, c.stream);
    finalize_factors(c);
    c.V.alloc(size_t(c.h_voff[N]));
    k_fill_hash<<<c.sm_count * 8, 256, 0, c.stream>>>(c.V.n, seed, c.V.p);
    ++c.launches;
    check_launch("fill_hash");
    c.Y.alloc(1);
    c.k0.clear();
    c.kw.clear();
    // optional synthetic W (n x option synth_nm, hash-filled) for timing the
    // W^T x / W c kernels at full scale without the setup (time_kernel 3, 4)
    c.nm = int(std::max(0LL, c.opt("synth_nm", 0)));
    c.ldw = round_up(c.n, 4);
    if (c.nm) {
      c.W.alloc(size_t(c.ldw) * c.nm);
      k_fill_hash<<<c.sm_count * 8, 256, 0, c.stream>>>(c.W.n, seed + 1, c.W.p);
      check_launch("fill_hash W");
    }
    c.alloc_work();
    AWG_CUDA(cudaStreamSynchronize(c.stream));
    c.have_factors = true;
  });
}

int awg_setup(awg_ctx* ctx, const awg_config* cfg) {
  return guarded(ctx, [&](Ctx& c) {
    if (c.N == 0) c.fail(AWG_E_STATE, "setup: set matrix and partition first");
    if (!cfg) c.fail(AWG_E_ARG, "setup: null config");
    check_config(c, *cfg);
    run_setup(c, *cfg);
    c.have_factors = true;
  });
}

int awg_apply(awg_ctx* ctx, int op, const double* x, double* y, int ptr_kind) {
  return guarded(ctx, [&](Ctx& c) {
    if (op != AWG_OP_A && !c.have_factors) c.fail(AWG_E_STATE, "apply: preconditioner not set up");
    if (c.n == 0) c.fail(AWG_E_STATE, "apply: no matrix");
    if (!x || !y) c.fail(AWG_E_ARG, "apply: null vector");
    if (!c.pb.p || c.pb.n != size_t(c.n)) c.alloc_work();
    if (ptr_kind == AWG_PTR_HOST) {
      AWG_CUDA(cudaMemcpyAsync(c.pb.p, x, sizeof(double) * c.n, cudaMemcpyHostToDevice, c.stream));
      op_apply(c, op, c.pb.p, c.pz.p, nullptr);
      AWG_CUDA(cudaMemcpyAsync(y, c.pz.p, sizeof(double) * c.n, cudaMemcpyDeviceToHost, c.stream));
    } else {
      op_apply(c, op, x, y, nullptr);
    }
    AWG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int awg_time_apply(awg_ctx* ctx, int op, int reps, double* ms) {
  return guarded(ctx, [&](Ctx& c) {
    if (!c.have_factors) c.fail(AWG_E_STATE, "time_apply: preconditioner not set up");
    if (reps < 1 || !ms) c.fail(AWG_E_ARG, "time_apply: bad arguments");
    cudaEvent_t e0, e1;
    AWG_CUDA(cudaEventCreate(&e0));
    AWG_CUDA(cudaEventCreate(&e1));
    op_apply(c, op, c.pb.p, c.pz.p, nullptr);
    AWG_CUDA(cudaEventRecord(e0, c.stream));
    for (int r = 0; r < reps; ++r) op_apply(c, op, c.pb.p, c.pz.p, nullptr);
    AWG_CUDA(cudaEventRecord(e1, c.stream));
    AWG_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    AWG_CUDA(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms = double(t) / reps;
  });
}

int awg_bench_dgemm(awg_ctx* ctx, int m, int n, int k, int count, int transpose_a, int reps, double* out) {
  return guarded(ctx, [&](Ctx& c) {
    if (m < 1 || n < 1 || k < 1 || count < 1 || reps < 1 || !out) c.fail(AWG_E_ARG, "bench_dgemm: bad arguments");
    bench_grouped_dgemm(c, m, n, k, count, transpose_a != 0, reps, out);
  });
}

int awg_time_kernel(awg_ctx* ctx, int which, int reps, double* ms, double* bytes) {
  return guarded(ctx, [&](Ctx& c) {
    if (!c.have_factors) c.fail(AWG_E_STATE, "time_kernel: preconditioner not set up");
    if (reps < 1 || !ms || !bytes) c.fail(AWG_E_ARG, "time_kernel: bad arguments");
    double b = 0.0;
    long long vcols = 0, P = 0;
    for (int s = 0; s < c.N; ++s) {
      vcols += (long long)c.h_ns[s] * (c.h_ns[s] - c.h_m[s]);
      P += c.h_ns[s];
    }
    std::function<void()> launch;
    switch (which) {
      case 0:  // V^T reads + x gathered (x, idx, D) + uh written (columns >= m)
        b = 8.0 * vcols + 20.0 * P + 8.0 * P;
        launch = [&] { k::nn_gemvT(c, c.pb.p, nullptr); };
        break;
      case 1:  // V reads + uh read + partials written
        b = 8.0 * vcols + 8.0 * P * 2;
        launch = [&] { k::nn_gemv(c, nullptr); };
        break;
      case 2:  // values + col indices + row offsets + x + y
        b = 12.0 * c.nnz + 4.0 * (c.n + 1) + 16.0 * c.n;
        launch = [&] { k::spmv(c, c.pb.p, c.pz.p, 0, nullptr, nullptr, nullptr); };
        break;
      case 3:
        if (c.nm == 0) c.fail(AWG_E_STATE, "time_kernel: no W");
        b = 8.0 * c.n * c.nm + 8.0 * c.n + 8.0 * c.nm;
        launch = [&] { k::wT(c, c.pb.p, c.cw.p, nullptr); };
        break;
      case 4:
        if (c.nm == 0) c.fail(AWG_E_STATE, "time_kernel: no W");
        b = 8.0 * c.n * c.nm + 8.0 * c.n + 8.0 * c.nm;
        launch = [&] { k::w_apply_public(c, c.cw.p, c.pz.p, nullptr); };
        break;
      case 5:  // single-pass NN: V once + x gathered + partial slots written
        if (!(c.one_level == 2 ? c.plan_nn.fused : c.plan_as.fused))
          c.fail(AWG_E_STATE, "time_kernel: single-pass local solve not available");
        b = 8.0 * vcols + 20.0 * P + 8.0 * P * c.plan_nn.kcmax_f;
        launch = [&] { k::nn_fused(c, c.pb.p, nullptr); };
        break;
      default:
        c.fail(AWG_E_ARG, "time_kernel: unknown kernel");
    }
    cudaEvent_t e0, e1;
    AWG_CUDA(cudaEventCreate(&e0));
    AWG_CUDA(cudaEventCreate(&e1));
    launch();
    AWG_CUDA(cudaEventRecord(e0, c.stream));
    for (int r = 0; r < reps; ++r) launch();
    AWG_CUDA(cudaEventRecord(e1, c.stream));
    AWG_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    AWG_CUDA(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms = double(t) / reps;
    *bytes = b;
  });
}

int awg_pcg(awg_ctx* ctx, const double* b, double* x, double rtol, int maxit, int ptr_kind, awg_solve_report* rep) {
  return guarded(ctx, [&](Ctx& c) {
    if (!c.have_factors) c.fail(AWG_E_STATE, "pcg: preconditioner not set up");
    if (!b || !x || !rep) c.fail(AWG_E_ARG, "pcg: null argument");
    if (ptr_kind == AWG_PTR_HOST) {
      AWG_CUDA(cudaMemcpyAsync(c.pb.p, b, sizeof(double) * c.n, cudaMemcpyHostToDevice, c.stream));
      run_pcg(c, c.pb.p, rtol, maxit, rep);
      AWG_CUDA(cudaMemcpyAsync(x, c.px.p, sizeof(double) * c.n, cudaMemcpyDeviceToHost, c.stream));
    } else {
      run_pcg(c, b, rtol, maxit, rep);
      AWG_CUDA(cudaMemcpyAsync(x, c.px.p, sizeof(double) * c.n, cudaMemcpyDeviceToDevice, c.stream));
    }
    AWG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int awg_query(awg_ctx* ctx, awg_stats* st) {
  return guarded(ctx, [&](Ctx& c) {
    if (!st) c.fail(AWG_E_ARG, "query: null");
    std::memset(st, 0, sizeof(*st));
    st->n = c.n;
    st->nnz = c.nnz;
    st->n_sub = c.N;
    st->n0 = c.n0;
    st->r0 = c.k0.rank;
    st->n_minus = c.nm;
    st->rw = c.kw.rank;
    for (int s = 0; s < c.N && s < (int)c.h_ns.size(); ++s) {
      const long long n_s = c.h_ns[s];
      st->sum_ns += n_s;
      st->sum_ns2 += n_s * n_s;
      if (s < (int)c.h_ks.size()) st->sum_ns_ks += n_s * c.h_ks[s];
      if (s < (int)c.h_m.size()) {
        st->sum_ns_ms += n_s * c.h_m[s];
        st->sum_ns_qs += n_s * (c.h_m[s] - c.h_nzero[s]);
      }
    }
    for (int i = 0; i < 8; ++i) st->t_setup_ms[i] = c.t_setup_ms[i];
    for (int v : c.h_w_inner) st->w_inner_total += v;
    st->w_batches = c.w_batches;
    st->nn_single_pass = ((c.one_level == 2 && c.plan_nn.fused) || (c.one_level != 2 && c.plan_as.fused)) ? 1 : 0;
    {
      const LocalPlan& lp = c.one_level == 2 ? c.plan_nn : c.plan_as;
      st->nn_static_split = (lp.fused && lp.static_grid > 0) ? 1 : 0;
    }
    st->coarse_az = c.az_on ? 1 : 0;
  });
}

int awg_get_history(awg_ctx* ctx, int which, double* out, int cap) {
  if (!ctx) return -1;
  Ctx& c = ctx->c;
  const std::vector<double>& v = which == 0 ? c.h_hist_res : which == 1 ? c.h_hist_diag : c.h_hist_off;
  const int k = std::min<int>(cap, int(v.size()));
  if (out) std::copy(v.begin(), v.begin() + k, out);
  return int(v.size());
}

int awg_kernel_timer(awg_ctx* ctx, int reset, double* ms_total, long long* launches) {
  return guarded(ctx, [&](Ctx& c) {
    unsigned long long h[5] = {~0ull, 0, 0, 0, 0};
    AWG_CUDA(cudaStreamSynchronize(c.stream));
    if (c.fused_timer.p) AWG_CUDA(cudaMemcpy(h, c.fused_timer.p, sizeof(h), cudaMemcpyDeviceToHost));
    if (ms_total) *ms_total = double(h[3]) * 1e-6;
    if (launches) *launches = (long long)h[4];
    if (reset && c.fused_timer.p) {
      const unsigned long long init[5] = {~0ull, 0, 0, 0, 0};
      AWG_CUDA(cudaMemcpy(c.fused_timer.p, init, sizeof(init), cudaMemcpyHostToDevice));
    }
  });
}

int awg_assemble_fd(awg_ctx* ctx, int dims, const int* shape, const double* cell_coef) {
  std::vector<int> rp, ci;
  std::vector<double> va;
  int rc = guarded(ctx, [&](Ctx& c) {
    if (c.device < 0) c.fail(AWG_E_CUDA, "no CUDA device");
    assemble_fd(c, dims, shape, cell_coef, rp, ci, va);
  });
  if (rc != AWG_OK) return rc;
  rc = awg_set_matrix(ctx, int(rp.size()) - 1, rp.data(), ci.data(), va.data());
  if (rc == AWG_OK) {
    ctx->c.asm_kind = 0;
    ctx->c.asm_dims = dims;
    for (int a = 0; a < 3; ++a) ctx->c.asm_shape[a] = a < dims ? shape[a] : 1;
  }
  return rc;
}

int awg_assemble_elasticity(awg_ctx* ctx, int nodes_x, int nodes_y, int layer_thickness, int n_materials,
                            const double* young, const double* poisson, const double* load) {
  std::vector<int> rp, ci;
  std::vector<double> va, b;
  int rc = guarded(ctx, [&](Ctx& c) {
    if (c.device < 0) c.fail(AWG_E_CUDA, "no CUDA device");
    assemble_elasticity(c, nodes_x, nodes_y, layer_thickness, n_materials, young, poisson, load, rp, ci, va, b);
  });
  if (rc != AWG_OK) return rc;
  rc = awg_set_matrix(ctx, int(rp.size()) - 1, rp.data(), ci.data(), va.data());
  if (rc == AWG_OK) {
    ctx->c.asm_kind = 1;
    ctx->c.asm_dims = 2;
    ctx->c.asm_shape[0] = nodes_x;
    ctx->c.asm_shape[1] = nodes_y;
    ctx->c.asm_shape[2] = 1;
    ctx->c.h_rhs_asm = b;
  }
  return rc;
}

int awg_partition_owner(awg_ctx* ctx, const int* owner, int n_sub, int overlap) {
  std::vector<long long> off;
  std::vector<int> idx;
  int rc = guarded(ctx, [&](Ctx& c) {
    if (c.n == 0) c.fail(AWG_E_STATE, "partition: set or assemble the matrix first");
    if (!owner) c.fail(AWG_E_ARG, "partition: bad arguments");
    partition_closure(c, std::vector<int>(owner, owner + c.n), n_sub, overlap, off, idx);
  });
  if (rc != AWG_OK) return rc;
  return awg_set_partition(ctx, n_sub, off.data(), idx.data());
}

int awg_partition_boxes(awg_ctx* ctx, const int* boxes, int overlap) {
  std::vector<int> owner;
  int nsub = 0;
  int rc = guarded(ctx, [&](Ctx& c) {
    if (c.asm_kind < 0) c.fail(AWG_E_STATE, "partition_boxes: the matrix was not assembled on the device");
    if (!boxes) c.fail(AWG_E_ARG, "partition_boxes: bad arguments");
    const int dims = c.asm_dims;
    nsub = 1;
    for (int a = 0; a < dims; ++a) {
      if (boxes[a] < 1 || boxes[a] > c.asm_shape[a]) c.fail(AWG_E_ARG, "partition_boxes: bad box counts");
      nsub *= boxes[a];
    }
    owner.resize(c.n);
    if (c.asm_kind == 0) {
      // cells lexicographic (x fastest), box index per axis coord // (shape / boxes)
      const int nx = c.asm_shape[0], ny = c.asm_shape[1];
      for (int i = 0; i < c.n; ++i) {
        const int co[3] = {i % nx, (i / nx) % ny, i / (nx * ny)};
        int o = 0, mult = 1;
        for (int a = 0; a < dims; ++a) {
          o += (co[a] / (c.asm_shape[a] / boxes[a])) * mult;
          mult *= boxes[a];
        }
        owner[i] = o;
      }
    } else {
      // nodal boxes of the Q1 mesh; both dofs of a free node follow the node
      const int nx = c.asm_shape[0], ny = c.asm_shape[1];
      const int bw = nx / boxes[0], bh = ny / boxes[1];
      for (int i = 0; i < c.n; ++i) {
        const int f = i >> 1, ix = f % (nx - 1) + 1, iy = f / (nx - 1);
        owner[i] = ix / bw + boxes[0] * (iy / bh);
      }
    }
    for (int o : owner)
      if (o >= nsub) c.fail(AWG_E_ARG, "partition_boxes: grid not divisible by the box counts");
  });
  if (rc != AWG_OK) return rc;
  return awg_partition_owner(ctx, owner.data(), nsub, overlap);
}

int awg_get_array(awg_ctx* ctx, int which, void* out, long long cap, long long* n_elems) {
  return guarded(ctx, [&](Ctx& c) {
    std::vector<double> dv;
    std::vector<int> iv;
    bool is_int = false;
    switch (which) {
      case 0: dv = c.h_lam; break;
      case 1: iv = c.h_m; is_int = true; break;
      case 2: iv = c.h_nzero; is_int = true; break;
      case 3: iv = c.h_ks; is_int = true; break;
      case 4: dv = c.h_plam; break;
      case 5: iv = c.h_mult; is_int = true; break;
      case 6: iv = c.k0.h_retained; is_int = true; break;
      case 7: dv = c.k0.h_l11; break;
      case 8: iv = c.kw.h_retained; is_int = true; break;
      case 9: dv = c.kw.h_l11; break;
      // the large device arrays go straight into `out` (no host staging copy:
      // V^s is 50 GB at c5): count first, then copy whatever fits in cap
      case 10:
      case 13:
      case 14: {
        long long cnt = 0;
        if (which == 10) cnt = (long long)c.n * c.nm;
        for (int s = 0; which != 10 && s < c.N; ++s)
          cnt += (long long)c.h_ns[s] * (which == 13 ? c.h_ks[s] : c.h_ns[s]);
        if (n_elems) *n_elems = cnt;
        if (!out) return;
        double* o = static_cast<double*>(out);
        long long pos = 0;
        auto put = [&](const double* src, long long spitch, int rows, int cols) {
          // rows x cols column-major block with device pitch spitch -> packed at o + pos
          const int fit = int(std::max(0LL, std::min<long long>(cols, (cap - pos) / std::max(rows, 1))));
          if (rows > 0 && fit > 0)
            AWG_CUDA(cudaMemcpy2D(o + pos, sizeof(double) * rows, src, sizeof(double) * spitch,
                                  sizeof(double) * rows, fit, cudaMemcpyDeviceToHost));
          pos += (long long)rows * cols;
        };
        if (which == 10) {
          put(c.W.p, c.ldw, c.n, c.nm);
        } else {
          for (int s = 0; s < c.N; ++s) {
            if (which == 13) put(c.Y.p + c.h_yoff[s], c.h_ld[s], c.h_ns[s], c.h_ks[s]);
            else put(c.V.p + c.h_voff[s], c.h_ld[s], c.h_ns[s], c.h_ns[s]);
          }
        }
        return;
      }
      case 11: dv = c.h_neg_weights; break;
      case 12: iv = c.h_w_inner; is_int = true; break;
      case 15: dv = c.h_eps; break;
      case 16: dv = c.h_rhs_asm; break;
      case 17: iv = c.h_rp; is_int = true; break;
      case 18: iv = c.h_ci; is_int = true; break;
      case 19: dv = c.h_va; break;
      case 20:
        for (long long o : c.h_poff) iv.push_back(int(o));
        is_int = true;
        break;
      case 21: iv = c.h_pidx; is_int = true; break;
      default: c.fail(AWG_E_ARG, "get_array: unknown array");
    }
    const long long cnt = is_int ? (long long)iv.size() : (long long)dv.size();
    if (n_elems) *n_elems = cnt;
    if (out) {
      const long long k = std::min(cap, cnt);
      if (is_int) std::memcpy(out, iv.data(), sizeof(int) * k);
      else std::memcpy(out, dv.data(), sizeof(double) * k);
    }
  });
}

}  // extern "C"
