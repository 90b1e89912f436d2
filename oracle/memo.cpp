// Memoising wrappers around three pure reference functions (TEST
// INFRASTRUCTURE ONLY — never linked into the product).
//
// The reference is single-threaded; its setup at BASELINE config c2 is 8-12 h
// on one core, dominated by independent per-subdomain work:
//   dense_sym_eig        dense.cpp:117-209  (eigsplit of every B^s, splitting.cpp:64-84)
//   generalized_sym_eig  dense.cpp:211-224  (GenEO pencils, coarse.cpp:98-111)
//   pcg                  krylov.cpp:36-124  (build_w's inner solves, preconditioner.cpp:97-113)
// oracle/Makefile renames the reference's own definitions of these three
// symbols (objcopy --redefine-sym, so the reference objects are otherwise
// untouched) to ref_orig_*, and this file provides the public symbols: each
// call hashes its complete input (matrix bytes / right-hand side bytes plus
// rtol and maxit), returns the stored result when a cache entry exists, and
// otherwise runs the reference's own function and stores its result.  Every
// function is deterministic (one thread, same binary), so a cache hit is
// bit-identical to recomputation.  This lets several worker processes
// (ref_driver --phase ...) fill the cache for disjoint subdomains / W columns
// in parallel, after which one ordinary ref_driver run replays the stock
// composition (ProblemContext + run_with_context) end to end.
//
// The pcg key does not include the operators: callers must not share one cache
// directory across different problems (the driver uses one directory per run).
// Each entry records the seconds the reference spent computing it, so the
// serial reference setup time is the sum over entries.
#include <unistd.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "awg/dense.hpp"
#include "awg/krylov.hpp"

namespace awg {
EigenDecomposition ref_orig_dense_sym_eig(const DenseMatrix& m);
EigenDecomposition ref_orig_generalized_sym_eig(const DenseMatrix& ma, const DenseMatrix& mb);
std::pair<std::vector<double>, SolveReport> ref_orig_pcg(const ApplyFn& apply_a, const ApplyFn& apply_h,
                                                          const std::vector<double>& b, double rtol, int maxit);
}  // namespace awg

namespace {

using awg::DenseMatrix;
using awg::EigenDecomposition;
using awg::SolveReport;

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct Hasher {  // FNV-1a 64 over bytes, two lanes with different seeds
  uint64_t a = 0xcbf29ce484222325ull, b = 0x84222325cbf29ce4ull;
  void add(const void* p, size_t n) {
    const unsigned char* c = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) {
      a = (a ^ c[i]) * 0x100000001b3ull;
      b = (b ^ c[i]) * 0x100000001b3ull + 0x9e37;
    }
  }
  void add(const DenseMatrix& m) {
    add(&m.rows, sizeof m.rows);
    add(&m.cols, sizeof m.cols);
    add(m.a.data(), m.a.size() * sizeof(double));
  }
  std::string key(const char* tag) const {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%s_%016llx%016llx", tag, (unsigned long long)a, (unsigned long long)b);
    return buf;
  }
};

const char* memo_dir() {
  const char* d = std::getenv("AWG_MEMO_DIR");
  return (d && *d) ? d : nullptr;
}

constexpr int kMinDim = 200;  // small problems (Ritz tridiagonals, tiny cases) are not cached

struct File {
  FILE* f = nullptr;
  explicit File(const std::string& p, const char* mode) : f(std::fopen(p.c_str(), mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

template <class T>
bool rd(FILE* f, T* p, size_t n) {
  return std::fread(p, sizeof(T), n, f) == n;
}
template <class T>
void wr(FILE* f, const T* p, size_t n) {
  if (std::fwrite(p, sizeof(T), n, f) != n) {
    std::perror("memo write");
    std::exit(4);
  }
}
void wr_vec(FILE* f, const std::vector<double>& v) {
  uint64_t n = v.size();
  wr(f, &n, 1);
  wr(f, v.data(), v.size());
}
bool rd_vec(FILE* f, std::vector<double>& v) {
  uint64_t n = 0;
  if (!rd(f, &n, 1)) return false;
  v.resize(n);
  return rd(f, v.data(), n);
}

bool load_eig(const std::string& path, EigenDecomposition& e) {
  File f(path, "rb");
  if (!f.f) return false;
  double secs = 0;
  int rc[2];
  if (!rd(f.f, &secs, 1) || !rd(f.f, rc, 2)) return false;
  if (!rd_vec(f.f, e.eigenvalues)) return false;
  e.eigenvectors = DenseMatrix(rc[0], rc[1]);
  return rd(f.f, e.eigenvectors.a.data(), e.eigenvectors.a.size());
}

void store_eig(const std::string& path, const EigenDecomposition& e, double secs) {
  const std::string tmp = path + ".tmp" + std::to_string(::getpid());
  {
    File f(tmp, "wb");
    if (!f.f) {
      std::perror("memo open");
      std::exit(4);
    }
    int rc[2] = {e.eigenvectors.rows, e.eigenvectors.cols};
    wr(f.f, &secs, 1);
    wr(f.f, rc, 2);
    wr_vec(f.f, e.eigenvalues);
    wr(f.f, e.eigenvectors.a.data(), e.eigenvectors.a.size());
  }
  std::rename(tmp.c_str(), path.c_str());
}

template <class Fn>
EigenDecomposition memo_eig(const char* tag, Hasher h, int dim, Fn&& compute) {
  const char* dir = memo_dir();
  if (!dir || dim < kMinDim) return compute();
  const std::string path = std::string(dir) + "/" + h.key(tag);
  EigenDecomposition e;
  if (load_eig(path, e)) return e;
  const double t0 = now_s();
  e = compute();
  const double secs = now_s() - t0;
  store_eig(path, e, secs);
  std::fprintf(stderr, "[memo] %s n=%d computed in %.1f s\n", tag, dim, secs);
  return e;
}

}  // namespace

namespace awg {

EigenDecomposition dense_sym_eig(const DenseMatrix& m) {
  Hasher h;
  h.add(m);
  return memo_eig("eig", h, m.rows, [&] { return ref_orig_dense_sym_eig(m); });
}

EigenDecomposition generalized_sym_eig(const DenseMatrix& ma, const DenseMatrix& mb) {
  Hasher h;
  h.add(ma);
  h.add(mb);
  return memo_eig("geig", h, ma.rows, [&] { return ref_orig_generalized_sym_eig(ma, mb); });
}

std::pair<std::vector<double>, SolveReport> pcg(const ApplyFn& apply_a, const ApplyFn& apply_h,
                                                const std::vector<double>& b, double rtol, int maxit) {
  const char* dir = memo_dir();
  const char* on = std::getenv("AWG_MEMO_PCG");
  if (!dir || !on || std::strcmp(on, "1") != 0 || int(b.size()) < kMinDim)
    return ref_orig_pcg(apply_a, apply_h, b, rtol, maxit);
  Hasher h;
  h.add(b.data(), b.size() * sizeof(double));
  h.add(&rtol, sizeof rtol);
  h.add(&maxit, sizeof maxit);
  const std::string path = std::string(dir) + "/" + h.key("pcg");
  {
    File f(path, "rb");
    if (f.f) {
      std::pair<std::vector<double>, SolveReport> out;
      SolveReport& r = out.second;
      double secs = 0;
      int conv = 0;
      bool ok = rd(f.f, &secs, 1) && rd(f.f, &r.iterations, 1) && rd(f.f, &conv, 1) &&
                rd(f.f, &r.final_relative_residual, 1) && rd(f.f, &r.recurrence_residual_at_exit, 1) &&
                rd(f.f, &r.ritz_min, 1) && rd(f.f, &r.ritz_max, 1) && rd(f.f, &r.kappa_estimate, 1) &&
                rd_vec(f.f, r.residual_history) && rd_vec(f.f, r.lanczos_diag) &&
                rd_vec(f.f, r.lanczos_offdiag) && rd_vec(f.f, out.first);
      r.converged = conv != 0;
      if (ok) return out;
    }
  }
  const double t0 = now_s();
  auto out = ref_orig_pcg(apply_a, apply_h, b, rtol, maxit);
  const double secs = now_s() - t0;
  const SolveReport& r = out.second;
  const std::string tmp = path + ".tmp" + std::to_string(::getpid());
  {
    File f(tmp, "wb");
    int conv = r.converged ? 1 : 0;
    wr(f.f, &secs, 1);
    wr(f.f, &r.iterations, 1);
    wr(f.f, &conv, 1);
    wr(f.f, &r.final_relative_residual, 1);
    wr(f.f, &r.recurrence_residual_at_exit, 1);
    wr(f.f, &r.ritz_min, 1);
    wr(f.f, &r.ritz_max, 1);
    wr(f.f, &r.kappa_estimate, 1);
    wr_vec(f.f, r.residual_history);
    wr_vec(f.f, r.lanczos_diag);
    wr_vec(f.f, r.lanczos_offdiag);
    wr_vec(f.f, out.first);
  }
  std::rename(tmp.c_str(), path.c_str());
  std::fprintf(stderr, "[memo] pcg n=%zu it=%d computed in %.1f s\n", b.size(), r.iterations, secs);
  return out;
}

}  // namespace awg
