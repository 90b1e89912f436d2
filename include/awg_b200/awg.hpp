// awg_b200/awg.hpp — C++ host API of the B200-native AWG-PCG path.
//
// Header-only layer over the C ABI (include/awg_cuda.h) that keeps the shape of
// the reference's proj/include/awg API so a caller can switch by changing the
// include and the namespace:
//
//   reference (proj/include/awg/...)                       here
//   SparseSymMatrix, read_matrix_market (sparse.hpp:12-55) SparseSymMatrix, read_matrix_market
//   read_vector (sparse.hpp:55)                             read_vector
//   Partition, read_partition (partition.hpp:14-61)         Partition, read_partition
//   PreconditionerConfig, OneLevelKind, Composition,        same names and defaults
//     AwgMode (preconditioner.hpp:17-31)
//   ProblemContext (harness.hpp:73-98)                      ProblemContext (owns the GPU context)
//   Splitting::apply_Aplus / apply_Aminus                   ProblemContext::splitting()
//   OneLevel / TwoLevel / AwgPreconditioner ::apply         same, via ProblemContext
//   coarse_correct (coarse.hpp:72)                          coarse_correct
//   pcg(apply_a, apply_h, b, rtol, maxit) (krylov.hpp:34)   pcg(ctx, b, rtol, maxit) — apply_a = A,
//                                                          apply_h = H3, as run_with_context does
//   SolveReport (krylov.hpp:14-28)                          SolveReport
//   NotSpdError (dense.hpp:58-63), std::runtime_error,      same exception types
//     std::invalid_argument
//
// Vectors are host std::vector<double> (copied to and from HBM per call), or
// raw device pointers through the *_device overloads.
#pragma once

#include <algorithm>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../awg_cuda.h"

namespace awg_b200 {

struct NotSpdError : std::runtime_error {
  int pivot_index;
  NotSpdError(const std::string& m, int k) : std::runtime_error(m), pivot_index(k) {}
};

struct SparseSymMatrix {
  int n = 0;
  std::vector<int> row_offsets;
  std::vector<int> col_indices;
  std::vector<double> values;
  int nnz() const { return static_cast<int>(col_indices.size()); }
};

struct Partition {
  std::vector<std::vector<int>> omega;
  int n = 0;
  int count() const { return static_cast<int>(omega.size()); }
  int size_of(int s) const { return static_cast<int>(omega[s].size()); }
};

enum class OneLevelKind { AS = 0, AS_PLUS = 1, NN = 2 };
enum class Composition { ADDITIVE = 0, HYBRID = 1 };
enum class AwgMode { NONE = 0, AD = 1, HYB = 2, INEX = 3 };

struct PreconditionerConfig {
  OneLevelKind one_level = OneLevelKind::NN;
  Composition composition = Composition::HYBRID;
  bool use_coarse = true;
  double tau_sharp = 0.1;
  double tau_flat = 10.0;
  AwgMode awg = AwgMode::AD;
  double w_rtol = 1e-10;
  // extensions: fixed-k GenEO rule and factor semantics
  int fixed_k = 0;
  bool exact_rank_revealing = false;
  bool exact_lu = false;
  int w_maxit_factor = 10;
};

struct SolveReport {
  int iterations = 0;
  bool converged = false;
  std::vector<double> residual_history;
  double final_relative_residual = 0.0;
  double recurrence_residual_at_exit = 0.0;
  std::vector<double> lanczos_diag;
  std::vector<double> lanczos_offdiag;
  double ritz_min = 0.0;
  double ritz_max = 0.0;
  double kappa_estimate = 0.0;
  double solve_ms = 0.0;
};

// The reference's file readers (read_matrix_market / read_vector /
// read_partition, sparse.cpp:89-138, partition.cpp:212-233) stay with the
// reference caller: it parses its files as before and hands the resulting
// SparseSymMatrix / vector / Partition to ProblemContext below.

// ---- the device-backed problem context -----------------------------------------
class ProblemContext {
 public:
  ProblemContext(const SparseSymMatrix& a, const std::vector<double>& b, const Partition& p, int device = 0)
      : a_(a), b_(b), part_(p) {
    if (static_cast<int>(b.size()) != a.n) throw std::runtime_error("external problem: rhs size does not match matrix");
    awg_ctx* raw = nullptr;
    const int rc = awg_create(&raw, device);
    ctx_.reset(raw);
    check(rc);
    check(awg_set_matrix(raw, a.n, a.row_offsets.data(), a.col_indices.data(), a.values.data()));
    std::vector<long long> off(p.count() + 1, 0);
    std::vector<int> idx;
    for (int s = 0; s < p.count(); ++s) {
      off[s + 1] = off[s] + p.size_of(s);
      idx.insert(idx.end(), p.omega[s].begin(), p.omega[s].end());
    }
    check(awg_set_partition(raw, p.count(), off.data(), idx.data()));
  }

  const SparseSymMatrix& a() const { return a_; }
  const std::vector<double>& rhs() const { return b_; }
  const Partition& partition() const { return part_; }

  // h2 + second_coarse (harness.cpp:105-124), built on the device
  void setup(const PreconditionerConfig& cfg) {
    awg_config c = to_c(cfg);
    check(awg_setup(ctx_.get(), &c));
    cfg_ = cfg;
  }

  std::vector<double> apply(int op, const std::vector<double>& x) const {
    if (static_cast<int>(x.size()) != a_.n) throw std::invalid_argument("apply: dimension mismatch");
    std::vector<double> y(x.size());
    check(awg_apply(ctx_.get(), op, x.data(), y.data(), AWG_PTR_HOST));
    return y;
  }
  void apply_device(int op, const double* x, double* y) const {
    check(awg_apply(ctx_.get(), op, x, y, AWG_PTR_DEVICE));
  }

  std::pair<std::vector<double>, SolveReport> pcg(const std::vector<double>& b, double rtol, int maxit) const {
    std::vector<double> x(b.size());
    awg_solve_report r{};
    check(awg_pcg(ctx_.get(), b.data(), x.data(), rtol, maxit, AWG_PTR_HOST, &r));
    SolveReport rep;
    rep.iterations = r.iterations;
    rep.converged = r.converged != 0;
    rep.final_relative_residual = r.final_relative_residual;
    rep.recurrence_residual_at_exit = r.recurrence_residual_at_exit;
    rep.ritz_min = r.ritz_min;
    rep.ritz_max = r.ritz_max;
    rep.kappa_estimate = r.kappa_estimate;
    rep.solve_ms = r.solve_ms;
    rep.residual_history = history(0);
    rep.lanczos_diag = history(1);
    rep.lanczos_offdiag = history(2);
    return {std::move(x), std::move(rep)};
  }

  awg_stats stats() const {
    awg_stats s{};
    check(awg_query(ctx_.get(), &s));
    return s;
  }

  awg_ctx* raw() const { return ctx_.get(); }

 private:
  struct Del {
    void operator()(awg_ctx* c) const { awg_destroy(c); }
  };

  std::vector<double> history(int which) const {
    const int k = awg_get_history(ctx_.get(), which, nullptr, 0);
    std::vector<double> v(k > 0 ? k : 0);
    if (k > 0) awg_get_history(ctx_.get(), which, v.data(), k);
    return v;
  }

  static awg_config to_c(const PreconditionerConfig& cfg) {
    awg_config c{};
    c.one_level = static_cast<int>(cfg.one_level);
    c.composition = static_cast<int>(cfg.composition);
    c.use_coarse = cfg.use_coarse ? 1 : 0;
    c.tau_sharp = cfg.tau_sharp;
    c.tau_flat = cfg.tau_flat;
    c.fixed_k = cfg.fixed_k;
    c.awg_mode = static_cast<int>(cfg.awg);
    c.w_rtol = cfg.w_rtol;
    c.w_maxit_factor = cfg.w_maxit_factor;
    c.rrf_semantics = cfg.exact_rank_revealing ? 1 : 0;
    c.lu_semantics = cfg.exact_lu ? 1 : 0;
    return c;
  }

  void check(int rc) const {
    if (rc == AWG_OK) return;
    const std::string msg = ctx_ ? awg_last_error(ctx_.get()) : "awg_create failed";
    switch (rc) {
      case AWG_E_NOT_SPD:
        throw NotSpdError(msg, awg_last_error_index(ctx_.get()));
      case AWG_E_ARG:
        throw std::invalid_argument(msg);
      default:
        throw std::runtime_error(msg);
    }
  }

  SparseSymMatrix a_;
  std::vector<double> b_;
  Partition part_;
  PreconditionerConfig cfg_;
  std::unique_ptr<awg_ctx, Del> ctx_;
};

// ---- reference-shaped operator views --------------------------------------------
struct Splitting {
  const ProblemContext* ctx;
  std::vector<double> apply_Aplus(const std::vector<double>& x) const { return ctx->apply(AWG_OP_APLUS, x); }
  std::vector<double> apply_Aminus(const std::vector<double>& x) const { return ctx->apply(AWG_OP_AMINUS, x); }
};
struct OneLevel {
  const ProblemContext* ctx;
  std::vector<double> apply(const std::vector<double>& x) const { return ctx->apply(AWG_OP_H1, x); }
};
struct TwoLevel {
  const ProblemContext* ctx;
  std::vector<double> apply(const std::vector<double>& x) const { return ctx->apply(AWG_OP_H2, x); }
};
struct AwgPreconditioner {
  const ProblemContext* ctx;
  std::vector<double> apply(const std::vector<double>& x) const { return ctx->apply(AWG_OP_H3, x); }
  std::vector<double> apply_pi3(const std::vector<double>& x) const { return ctx->apply(AWG_OP_PI3, x); }
  std::vector<double> apply_pi3_transpose(const std::vector<double>& x) const {
    return ctx->apply(AWG_OP_PI3T, x);
  }
};

inline std::vector<double> coarse_correct(const ProblemContext& ctx, const std::vector<double>& x) {
  return ctx.apply(AWG_OP_Q, x);
}
inline std::vector<double> spmv(const ProblemContext& ctx, const std::vector<double>& x) {
  return ctx.apply(AWG_OP_A, x);
}
inline std::pair<std::vector<double>, SolveReport> pcg(const ProblemContext& ctx, const std::vector<double>& b,
                                                       double rtol, int maxit) {
  return ctx.pcg(b, rtol, maxit);
}

}  // namespace awg_b200
