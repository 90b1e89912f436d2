// Operator composition (H1, H2, H3, projectors) and the device-resident PCG.
//
// Composition follows the reference exactly, operation by operation:
//   TwoLevel::apply        preconditioner.cpp:64-82 (hybrid: Pi^T, H1, Pi, + Qx;
//                          Q x is computed once and reused for Pi^T, which the
//                          reference recomputes bit-identically, coarse.cpp:188)
//   AwgPreconditioner      preconditioner.cpp:185-221 (AD, HYB, INEX), apply_pi3(_transpose) :161-183
//   pcg                    krylov.cpp:36-124, including the recursive/true residual
//                          stopping rule (:93-102), breakdown handling (:79-82, :107-110)
//                          and the Lanczos coefficients (:90-91)
#include <cmath>
#include <functional>
#include <cstring>

#include "awg_internal.cuh"
#include "pcg_device.cuh"

namespace awgb {

namespace {

constexpr int kThreads = 256;

using pcgdev::grid_reduce;

__global__ void k_pcg_init(PcgState* st, int n, const double* __restrict__ b, double* __restrict__ x,
                           double* __restrict__ r, double* part, unsigned* count) {
  pdl_wait();
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double bi = b[i];
    x[i] = 0.0;
    r[i] = bi;
    acc = fma(bi, bi, acc);
  }
  grid_reduce(acc, part, count, [&](double s) {
    st->bnorm = sqrt(s);
    st->it = 0;
    st->error = 0;
    st->past_rtol = 0;
    st->need_true = 0;
    st->converged = (s == 0.0);
    st->done = (s == 0.0);
  });
}

// rz = <r, z>; the initial check (krylov.cpp:51-53) or the beta step (:105-115).
__global__ void k_pcg_rz(PcgState* st, int n, const double* __restrict__ r, const double* __restrict__ z,
                         double* part, unsigned* count, int initial) {
  pdl_wait();
  if (st->done) return;
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) acc = fma(r[i], z[i], acc);
  grid_reduce(acc, part, count, [&](double rz) { pcgdev::rz_finish(st, rz, initial); });
}

// p = z + beta p   (p = z on the first step: beta = 0 and p zeroed)
__global__ void k_pcg_p(const PcgState* st, int n, const double* __restrict__ z, double* __restrict__ p, int initial) {
  pdl_wait();
  if (st->done) return;
  const double beta = st->beta;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = initial ? z[i] : fma(beta, p[i], z[i]);
}

// q = A p (or A+ p = A- p + A p when `add` holds A- p) and <p, q> (krylov.cpp:77-83)
__global__ void k_pcg_spmv_dot(PcgState* st, int n, const int* __restrict__ rp, const int* __restrict__ ci,
                               const double* __restrict__ va, const double* __restrict__ p, double* __restrict__ q,
                               const double* __restrict__ add, double* part, unsigned* count) {
  pdl_wait();
  if (st->done) return;
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    s = csr_row(ci, va, rp[i], rp[i + 1], [&](int j) { return __ldg(p + j); });
    if (add) s = add[i] + s;
    q[i] = s;
    acc = fma(p[i], s, acc);
  }
  grid_reduce(acc, part, count, [&](double pq) {
    st->pq = pq;
    if (pq <= 0.0) {
      if (!st->past_rtol) st->error = PCG_BAD_OPERATOR;
      st->done = 1;
      return;
    }
    st->alpha = st->rz / pq;
  });
}

// p = z + beta p_old formed inside the SpMV (the k_pcg_p step fused): every
// row evaluates fma(beta, p_old[j], z[j]) for its columns — bit for bit the
// p that k_pcg_p would have stored — and writes its own p_new[i]; then
// q = A p_new and <p_new, q> (krylov.cpp:77-83, 111-115).  p_old / p_new
// alternate between two buffers across iterations.
__global__ void k_pcg_spmv_dot_p(PcgState* st, int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                 const double* __restrict__ va, const double* __restrict__ z,
                                 const double* __restrict__ pold, double* __restrict__ pnew,
                                 double* __restrict__ q, double* part, unsigned* count) {
  pdl_wait();
  if (st->done) return;
  const double beta = st->beta;
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    s = csr_row(ci, va, rp[i], rp[i + 1], [&](int j) { return fma(beta, __ldg(pold + j), __ldg(z + j)); });
    const double pi = fma(beta, pold[i], z[i]);
    pnew[i] = pi;
    q[i] = s;
    acc = fma(pi, s, acc);
  }
  grid_reduce(acc, part, count, [&](double pq) {
    st->pq = pq;
    if (pq <= 0.0) {
      if (!st->past_rtol) st->error = PCG_BAD_OPERATOR;
      st->done = 1;
      return;
    }
    st->alpha = st->rz / pq;
  });
}

// x += alpha p; r -= alpha q; relres = ||r|| / ||b||, history and Lanczos
// coefficients (krylov.cpp:84-92)
__global__ void k_pcg_update(PcgState* st, int n, double* __restrict__ x, double* __restrict__ r,
                             const double* __restrict__ p, const double* __restrict__ q, double* part,
                             unsigned* count, double* hres, double* hdiag, double* hoff) {
  pdl_wait();
  if (st->done) return;
  const double alpha = st->alpha;
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    acc = fma(ri, ri, acc);
  }
  grid_reduce(acc, part, count, [&](double rr) {
    const double relres = sqrt(rr) / st->bnorm;
    const int it = st->it + 1;
    st->it = it;
    st->relres = relres;
    hres[it - 1] = relres;
    hdiag[it - 1] = 1.0 / alpha + (it > 1 ? st->beta_prev / st->alpha_prev : 0.0);
    if (it > 1) hoff[it - 2] = sqrt(st->beta_prev) / st->alpha_prev;
    st->need_true = (relres <= st->rtol);
    if (st->need_true) st->past_rtol = 1;
    if (!st->need_true && it == st->maxit) st->done = 1;
  });
}

// Recomputed residual ||b - A x|| / ||b|| and the acceptance rule (krylov.cpp:93-103).
__global__ void k_pcg_true(PcgState* st, int n, const int* __restrict__ rp, const int* __restrict__ ci,
                           const double* __restrict__ va, const double* __restrict__ x, const double* __restrict__ b,
                           const double* __restrict__ add, double* part, unsigned* count) {
  pdl_wait();
  const int force = st->force_true;
  if (!force && (st->done || !st->need_true)) return;
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    s = csr_row(ci, va, rp[i], rp[i + 1], [&](int j) { return __ldg(x + j); });
    if (add) s = add[i] + s;
    const double d = b[i] - s;
    acc = fma(d, d, acc);
  }
  grid_reduce(acc, part, count, [&](double dd) {
    const double tr = sqrt(dd) / st->bnorm;
    st->true_rel = tr;
    if (force) {
      st->final_rel = tr;
      return;
    }
    if (tr <= st->rtol || fabs(tr - st->relres) <= 1e-8) {
      st->converged = 1;
      st->done = 1;
      st->final_rel = tr;
      st->rec_exit = st->relres;
    } else if (st->it == st->maxit) {
      st->done = 1;
    }
  });
}

__global__ void k_set_force(PcgState* st, int v) {
  pdl_wait();
  st->force_true = v;
}

// skip flag for work that only the true-residual check needs
__global__ void k_true_gate(const PcgState* st, int* flag) {
  pdl_wait();
  flag[0] = (st->force_true || (!st->done && st->need_true)) ? 0 : 1;
}

int red_grid(const Ctx& c) {
  int g = (c.n + kThreads - 1) / kThreads;
  return std::max(1, std::min(g, c.sm_count * 4));
}

// Extreme eigenvalues of the symmetric tridiagonal Lanczos matrix by Sturm
// bisection (the reference uses dense Jacobi on it, krylov.cpp:126-139;
// report-only quantity).
int sturm_count(const std::vector<double>& d, const std::vector<double>& e, double x) {
  int cnt = 0;
  double q = 1.0;
  for (size_t i = 0; i < d.size(); ++i) {
    const double e2 = i ? e[i - 1] * e[i - 1] : 0.0;
    q = d[i] - x - (i ? e2 / q : 0.0);
    if (q == 0.0) q = -1e-300;
    if (q < 0.0) ++cnt;
  }
  return cnt;
}

double tridiag_eig(const std::vector<double>& d, const std::vector<double>& e, int k) {
  double lo = d[0], hi = d[0];
  for (size_t i = 0; i < d.size(); ++i) {
    const double r = (i ? std::fabs(e[i - 1]) : 0.0) + (i + 1 < d.size() ? std::fabs(e[i]) : 0.0);
    lo = std::min(lo, d[i] - r);
    hi = std::max(hi, d[i] + r);
  }
  for (int iter = 0; iter < 200; ++iter) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (sturm_count(d, e, mid) > k) hi = mid;
    else lo = mid;
  }
  return 0.5 * (lo + hi);
}

}  // namespace

// ---------------------------------------------------------------------------
int w_chunks(const Ctx& c) {
  // 512-row panels; split the n_minus columns until ~4 CTAs per SM exist,
  // keeping at least 128 columns per chunk
  const int panels = (c.n + 511) / 512;
  const int want = (4 * c.sm_count + panels - 1) / panels;
  return std::max(1, std::min(want, c.nm / 128));
}

void Ctx::alloc_work() {
  invalidate_graphs();
  const size_t nn = size_t(n);
  for (DArr<double>* b : {&t0, &t1, &t2, &t3, &t4, &t5, &t6, &t7, &t8}) b->alloc(nn);
  xs.alloc(P);
  uh.alloc(P);
  wl.alloc(P);
  const size_t cdim = size_t(std::max(n0, nm)) * 2 + 2;
  cz.alloc(cdim);
  cw.alloc(cdim);
  const int nch = (round_up(n, 4) + 1023) / 1024;  // W^T x row chunks (1024 or 4096 rows, k::wT)
  wpart.alloc(size_t(std::max(nm, 1)) * nch);
  wpart2.alloc(size_t(w_chunks(*this)) * round_up(n, 4));
  red.alloc(size_t(sm_count) * 16);
  red_count.alloc(1);
  red_count.zero(stream);
  pcg.alloc(1);
  for (DArr<double>* b : {&px, &pr, &pz, &pp, &pp2, &pq, &pb, &pt}) b->alloc(nn);
}

static void h1(Ctx& c, const double* x, double* y, const int* gate) { k::h1(c, x, y, gate); }

static void aplus(Ctx& c, const double* x, double* y, const int* gate) { k::aplus(c, x, y, 1, nullptr, gate); }

// H2 x into y.  With `extra` set (the AD branch's W KW+ W^T x, ready once
// `extra_ready` has fired) the hybrid composition's last kernel also adds it:
// y = ((hp - Q A+ hp) + corr) + extra, the reference's two sums in order.
static void h2(Ctx& c, const double* x, double* y, const int* gate, const double* extra = nullptr,
               cudaEvent_t extra_ready = nullptr, const std::function<void()>& after_h1 = {}) {
  auto add_extra = [&](const double* h2y) {
    if (extra_ready) AWG_CUDA(cudaStreamWaitEvent(c.stream, extra_ready, 0));
    k::axpby(c, c.n, h2y, extra, nullptr, y, 1, gate);
  };
  if (c.n0 == 0) {
    h1(c, x, extra ? c.t1.p : y, gate);
    if (extra) add_extra(c.t1.p);
    return;
  }
  // corr (and, for the hybrid form, the A- dots of corr in the same coarse-solve launch)
  const bool neg_ready = c.cfg.composition != 0 && k::coarse_q_neg(c, x, c.t0.p, gate);
  if (!neg_ready) k::coarse_q(c, x, c.t0.p, gate);
  if (c.cfg.composition == 0) {
    h1(c, x, c.t1.p, gate);
    k::axpby(c, c.n, c.t1.p, c.t0.p, nullptr, extra ? c.t2.p : y, 1, gate);
    if (extra) add_extra(c.t2.p);
    return;
  }
  c.trigger_next = (c.pdl_local && c.use_pdl) ? 1 : 0;  // the local solve may start its copies early
  k::aplus(c, c.t0.p, c.t2.p, 2, x, gate, neg_ready);  // pt = x - A+ corr
  c.trigger_next = 0;
  h1(c, c.t2.p, c.t3.p, gate);                     // hp
  if (after_h1) after_h1();  // enqueues work that must follow the local solve
  if (c.az_on) {  // Z^T A+ hp from the precomputed A Z and M1: no A+ hp, two kernels fewer
    k::coarse_q_combine_az(c, c.t3.p, y, c.t0.p, extra, extra_ready, gate);
    return;
  }
  aplus(c, c.t3.p, c.t4.p, gate);                  // A+ hp
  // (hp - Q A+ hp) + corr [+ extra], fused into the Z c prolongation
  k::coarse_q_combine(c, c.t4.p, y, c.t3.p, c.t0.p, extra, extra_ready, gate);
}

void op_apply(Ctx& c, int op, const double* x, double* y, const int* gate) {
  if (x == y) c.fail(AWG_E_ARG, "apply: x and y must not alias (operators.hpp:7)");
  const bool have_w = c.nm > 0;
  switch (op) {
    case AWG_OP_A:
      k::spmv(c, x, y, 0, nullptr, nullptr, gate);
      return;
    case AWG_OP_AMINUS:
      k::aminus(c, x, y, gate);
      return;
    case AWG_OP_APLUS:
      aplus(c, x, y, gate);
      return;
    case AWG_OP_H1:
      h1(c, x, y, gate);
      return;
    case AWG_OP_Q:
      k::coarse_q(c, x, y, gate);
      return;
    case AWG_OP_QW:
      k::second_q(c, x, y, gate);
      return;
    case AWG_OP_H2:
      h2(c, x, y, gate);
      return;
    case AWG_OP_PI3:
      if (!have_w) {
        AWG_CUDA(cudaMemcpyAsync(y, x, sizeof(double) * c.n, cudaMemcpyDeviceToDevice, c.stream));
        return;
      }
      k::spmv(c, x, c.t6.p, 0, nullptr, nullptr, gate);
      k::second_q(c, c.t6.p, c.t7.p, gate);
      k::axpby(c, c.n, x, c.t7.p, nullptr, y, 2, gate);
      return;
    case AWG_OP_PI3T:
      if (!have_w) {
        AWG_CUDA(cudaMemcpyAsync(y, x, sizeof(double) * c.n, cudaMemcpyDeviceToDevice, c.stream));
        return;
      }
      k::second_q(c, x, c.t6.p, gate);
      k::spmv(c, c.t6.p, y, 3, nullptr, x, gate);
      return;
    case AWG_OP_H3: {
      const int mode = c.cfg.awg_mode;
      if (mode == 0 || !have_w) {
        h2(c, x, y, gate);
        return;
      }
      if (mode == 1) {  // AD: W KW^+ W^T x and H2 x are independent — run them concurrently
        // Split (small W): W^T x and the KW solve overlap the latency-bound
        // coarse chain before the local solve, W c the one after it, so the
        // W streams do not take HBM bandwidth from the single-pass local solve.
        // Large W (c3, c5): the whole branch overlaps everything (pure
        // bandwidth sharing is better there).
        // (the split needs h2's hybrid branch, whose after_h1 hook runs the
        // second half: never split without it, whatever the knob says)
        const bool can_split = c.n0 > 0 && c.cfg.composition != 0;
        const bool split = can_split && (c.w_split >= 0 ? c.w_split == 1 : 8.0 * c.n * c.nm <= 512.0 * (1 << 20));
        AWG_CUDA(cudaEventRecord(c.ev_fork, c.stream));
        AWG_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
        cudaStream_t main = c.stream;
        c.stream = c.side;
        if (split) k::second_q_coef(c, x, gate);
        else k::second_q(c, x, c.t6.p, gate);
        c.stream = main;
        std::function<void()> tail;
        if (split) {
          tail = [&]() {  // on main right after the local solve: release W c on the side stream
            AWG_CUDA(cudaEventRecord(c.ev_mid, c.stream));
            AWG_CUDA(cudaStreamWaitEvent(c.side, c.ev_mid, 0));
            c.stream = c.side;
            k::second_q_apply(c, c.t6.p, gate);
            c.stream = main;
            AWG_CUDA(cudaEventRecord(c.ev_join, c.side));
          };
        } else {
          AWG_CUDA(cudaEventRecord(c.ev_join, c.side));
        }
        h2(c, x, y, gate, c.t6.p, c.ev_join, tail);  // joins the branch before its last kernel
      } else if (mode == 2) {  // HYB
        k::second_q(c, x, c.t6.p, gate);                 // corr
        k::spmv(c, c.t6.p, c.t7.p, 3, nullptr, x, gate);  // pt = x - A corr
        h2(c, c.t7.p, c.t8.p, gate);                     // hp
        k::spmv(c, c.t8.p, c.t7.p, 0, nullptr, nullptr, gate);
        k::second_q(c, c.t7.p, c.t1.p, gate);  // QW A hp (t1 is free once h2 returned)
        k::axpby(c, c.n, c.t8.p, c.t1.p, c.t6.p, y, 0, gate);
      } else {  // INEX
        k::inex_q(c, x, c.t6.p, gate);
        h2(c, x, c.t7.p, gate);
        k::axpby(c, c.n, c.t7.p, c.t6.p, nullptr, y, 1, gate);
      }
      return;
    }
    default:
      c.fail(AWG_E_ARG, "apply: unknown operator");
  }
}

// ---------------------------------------------------------------------------
void run_pcg(Ctx& c, const double* b_dev, double rtol, int maxit, awg_solve_report* rep, int op_a, int op_h) {
  if (!(rtol > 0.0 && rtol < 1.0)) c.fail(AWG_E_ARG, "pcg: rtol must be in (0,1)");
  if (maxit < 1) c.fail(AWG_E_ARG, "pcg: maxit must be positive");
  const int n = c.n;
  if (c.hist_cap < maxit) {
    c.hist_res.alloc(maxit);
    c.hist_diag.alloc(maxit);
    c.hist_off.alloc(maxit);
    c.hist_cap = maxit;
    c.invalidate_graphs();
  }
  if (!c.pcg_flag.p) c.pcg_flag.alloc(1);
  PcgState h{};
  h.rtol = rtol;
  h.maxit = maxit;
  AWG_CUDA(cudaMemcpyAsync(c.pcg.p, &h, sizeof(h), cudaMemcpyHostToDevice, c.stream));
  if (b_dev != c.pb.p)
    AWG_CUDA(cudaMemcpyAsync(c.pb.p, b_dev, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
  PcgState* st = c.pcg.p;
  const int* gate = &st->done;
  const int g = red_grid(c);
  const bool aplus = (op_a == AWG_OP_APLUS);
  double* am = c.t8.p;  // A- p / A- x scratch (H2 uses t0..t5; H3 also t6..t8, never with A+)
  if (aplus && op_h == AWG_OP_H3) c.fail(AWG_E_ARG, "pcg: A+ operator pairs with H2 only");
  cudaEvent_t e0, e1;
  AWG_CUDA(cudaEventCreate(&e0));
  AWG_CUDA(cudaEventCreate(&e1));
  AWG_CUDA(cudaEventRecord(e0, c.stream));

  // Fused form (A operator): p = z + beta p is formed inside the next SpMV
  // (two alternating p buffers, zero before the first step so p_1 = z), and
  // <r, z> is folded into the preconditioner's last kernel when it can take it.
  // With A+ the A- product needs p first, so p and rz stay separate kernels.
  const bool fuse = !aplus;
  launch(c, k_pcg_init, g, kThreads, 0, st, n, c.pb.p, c.px.p, c.pr.p, c.red.p, c.red_count.p);
  ++c.launches;
  op_apply(c, op_h, c.pr.p, c.pz.p, gate);
  launch(c, k_pcg_rz, g, kThreads, 0, st, n, c.pr.p, c.pz.p, c.red.p, c.red_count.p, 1);
  ++c.launches;
  if (fuse) {
    AWG_CUDA(cudaMemsetAsync(c.pp.p, 0, sizeof(double) * n, c.stream));
    AWG_CUDA(cudaMemsetAsync(c.pp2.p, 0, sizeof(double) * n, c.stream));
  } else {
    launch(c, k_pcg_p, g, kThreads, 0, st, n, c.pz.p, c.pp.p, 1);
    ++c.launches;
  }
  check_launch("pcg init");

  auto iteration = [&](double* pold, double* pnew) {
    if (fuse) {
      launch(c, k_pcg_spmv_dot_p, g, kThreads, 0, st, n, c.rp.p, c.ci.p, c.va.p, c.pz.p, pold, pnew, c.pq.p,
             c.red.p, c.red_count.p);
    } else {
      k::aminus(c, c.pp.p, am, gate);
      launch(c, k_pcg_spmv_dot, g, kThreads, 0, st, n, c.rp.p, c.ci.p, c.va.p, c.pp.p, c.pq.p, am, c.red.p,
             c.red_count.p);
      pnew = c.pp.p;
    }
    launch(c, k_pcg_update, g, kThreads, 0, st, n, c.px.p, c.pr.p, pnew, c.pq.p, c.red.p, c.red_count.p,
                                               c.hist_res.p, c.hist_diag.p, c.hist_off.p);
    c.launches += 2;
    if (aplus) {
      launch(c, k_true_gate, 1, 1, 0, st, c.pcg_flag.p);
      ++c.launches;
      k::aminus(c, c.px.p, am, c.pcg_flag.p);
    }
    launch(c, k_pcg_true, g, kThreads, 0, st, n, c.rp.p, c.ci.p, c.va.p, c.px.p, c.pb.p, aplus ? am : nullptr,
                                             c.red.p, c.red_count.p);
    ++c.launches;
    if (fuse) {
      c.rz_fuse = RzFuse{st, c.pr.p, c.pz.p, c.red.p, c.red_count.p};
      c.rz_fused = false;
    }
    op_apply(c, op_h, c.pr.p, c.pz.p, gate);
    c.rz_fuse = RzFuse{};
    if (!(fuse && c.rz_fused)) {
      launch(c, k_pcg_rz, g, kThreads, 0, st, n, c.pr.p, c.pz.p, c.red.p, c.red_count.p, 0);
      ++c.launches;
    }
    if (!fuse) {
      launch(c, k_pcg_p, g, kThreads, 0, st, n, c.pz.p, c.pp.p, 0);
      ++c.launches;
    }
    check_launch("pcg iteration");
  };

  // Enqueue iterations in batches; the device-side `done` flag turns every
  // kernel after the stopping point into a no-op, so overshooting is free of
  // side effects.  One CUDA graph holds two iterations (the p buffers swap
  // roles between them); it is cached per operator pair until buffers or
  // factors change.
  const int key = op_a * 16 + op_h;
  constexpr int kItersPerGraph = 2;
  cudaGraphExec_t exec = nullptr;
  auto it_cached = c.graphs.find(key);
  if (it_cached != c.graphs.end()) {
    exec = it_cached->second;
  } else {
    cudaGraph_t graph = nullptr;
    const long long before = c.launches;
    AWG_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    iteration(c.pp.p, c.pp2.p);
    iteration(c.pp2.p, c.pp.p);
    AWG_CUDA(cudaStreamEndCapture(c.stream, &graph));
    AWG_CUDA(cudaGraphInstantiate(&exec, graph, c.use_priority ? cudaGraphInstantiateFlagUseNodePriority : 0));
    cudaGraphDestroy(graph);
    c.graphs[key] = exec;
    c.graph_launches[key] = c.launches - before;
    c.launches = before;
  }
  const long long per_graph = c.graph_launches[key];
  // Iterations enqueued before the next host check: doubling up to 16, but
  // capped by the iterations the recent convergence rate still needs to reach
  // rtol — every iteration enqueued past the stop runs ~20 gated no-op
  // kernels, and a 16-iteration batch could overshoot by up to 15 (c2: ~1% of
  // the solve).  Host-side scheduling only: the device state decides.
  int batch = 2;
  int issued = 0;
  int prev_it = 0;
  double prev_rel = 0.0;
  while (true) {
    for (int b = 0; b < batch && issued < maxit; b += kItersPerGraph, issued += kItersPerGraph) {
      AWG_CUDA(cudaGraphLaunch(exec, c.stream));
      c.launches += per_graph;
    }
    AWG_CUDA(cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    AWG_CUDA(cudaStreamSynchronize(c.stream));
    if (h.done || issued >= maxit) break;
    int next = std::min(batch * 2, 16);
    if (c.pcg_adaptive && prev_rel > 0.0 && h.it > prev_it && h.relres > rtol && h.relres < prev_rel) {
      const double per_it = std::log(h.relres / prev_rel) / double(h.it - prev_it);  // < 0
      const double need = std::log(rtol / h.relres) / per_it;                      // iterations left
      if (need >= 0.0 && need < next) next = std::max(kItersPerGraph, int(std::ceil(need)));
    }
    prev_rel = h.relres;
    prev_it = h.it;
    batch = next;
  }

  if (!h.converged && h.it > 0 && !h.error) {
    launch(c, k_set_force, 1, 1, 0, st, 1);
    c.launches += 1;
    if (aplus) k::aminus(c, c.px.p, am, nullptr);
    launch(c, k_pcg_true, g, kThreads, 0, st, n, c.rp.p, c.ci.p, c.va.p, c.px.p, c.pb.p, aplus ? am : nullptr,
                                             c.red.p, c.red_count.p);
    launch(c, k_set_force, 1, 1, 0, st, 0);
    c.launches += 2;
    AWG_CUDA(cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
  }
  AWG_CUDA(cudaEventRecord(e1, c.stream));
  AWG_CUDA(cudaStreamSynchronize(c.stream));
  float ms = 0.f;
  AWG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (h.error == PCG_BAD_OPERATOR) c.fail(AWG_E_BREAKDOWN, "pcg: operator not spd (<p, Ap> <= 0)");
  if (h.error == PCG_BAD_PRECOND) c.fail(AWG_E_BREAKDOWN, "pcg: preconditioner not spd (<r, Hr> <= 0)");

  const int it = h.it;
  c.h_hist_res.assign(it, 0.0);
  c.h_hist_diag.assign(it, 0.0);
  c.h_hist_off.assign(it > 1 ? it - 1 : 0, 0.0);
  if (it) {
    AWG_CUDA(cudaMemcpy(c.h_hist_res.data(), c.hist_res.p, sizeof(double) * it, cudaMemcpyDeviceToHost));
    AWG_CUDA(cudaMemcpy(c.h_hist_diag.data(), c.hist_diag.p, sizeof(double) * it, cudaMemcpyDeviceToHost));
    if (it > 1)
      AWG_CUDA(cudaMemcpy(c.h_hist_off.data(), c.hist_off.p, sizeof(double) * (it - 1), cudaMemcpyDeviceToHost));
  }
  std::memset(rep, 0, sizeof(*rep));
  rep->iterations = it;
  rep->converged = h.converged;
  rep->solve_ms = ms;
  if (h.converged && it == 0) return;  // b == 0
  rep->final_relative_residual = h.final_rel;
  rep->recurrence_residual_at_exit = h.converged ? h.rec_exit : (it ? c.h_hist_res.back() : 0.0);
  // fill_ritz (krylov.cpp:21-32)
  if (it == 1) {
    rep->ritz_min = rep->ritz_max = c.h_hist_diag[0];
    rep->kappa_estimate = 1.0;
  } else if (it > 1) {
    rep->ritz_min = tridiag_eig(c.h_hist_diag, c.h_hist_off, 0);
    rep->ritz_max = tridiag_eig(c.h_hist_diag, c.h_hist_off, it - 1);
    rep->kappa_estimate = rep->ritz_max / rep->ritz_min;
  }
}

}  // namespace awgb
