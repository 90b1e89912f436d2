// C++ caller of the host API (include/awg_b200/awg.hpp), written the way the
// reference's run_with_context (proj/src/harness.cpp:131-139) drives its
// library: a problem in, preconditioner build, PCG with H3 — on the GPU.
// The problem comes as one binary dump written by tests/test_host_api.py
// (the reference caller would use its own file readers instead).
//   host_api_main <prefix> <tau|-k K> [exact]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "awg_b200/awg.hpp"

namespace {
// <prefix>.bin: int32 n, nnz, N; int32 row_offsets[n+1], col_indices[nnz];
// f64 values[nnz], b[n]; int32 part_offsets[N+1], part_indices[...]
template <class T>
std::vector<T> take(std::FILE* f, size_t count) {
  std::vector<T> v(count);
  if (count && std::fread(v.data(), sizeof(T), count, f) != count) throw std::runtime_error("truncated problem dump");
  return v;
}
void load_dump(const std::string& path, awg_b200::SparseSymMatrix& a, std::vector<double>& b, awg_b200::Partition& p) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw std::runtime_error("cannot open " + path);
  const auto hdr = take<int>(f, 3);
  a.n = hdr[0];
  a.row_offsets = take<int>(f, size_t(hdr[0]) + 1);
  a.col_indices = take<int>(f, size_t(hdr[1]));
  a.values = take<double>(f, size_t(hdr[1]));
  b = take<double>(f, size_t(hdr[0]));
  const auto off = take<int>(f, size_t(hdr[2]) + 1);
  const auto idx = take<int>(f, size_t(off.back()));
  std::fclose(f);
  p.n = a.n;
  for (int s = 0; s < hdr[2]; ++s) p.omega.emplace_back(idx.begin() + off[s], idx.begin() + off[s + 1]);
}
}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: host_api_main <prefix> <tau> | <prefix> -k <K> [exact]\n");
    return 2;
  }
  using namespace awg_b200;
  const std::string prefix = argv[1];
  PreconditionerConfig cfg;
  int argi = 2;
  if (std::strcmp(argv[2], "-k") == 0) {
    cfg.fixed_k = std::atoi(argv[3]);
    argi = 4;
  } else {
    cfg.tau_sharp = std::atof(argv[2]);
    argi = 3;
  }
  if (argc > argi && std::strcmp(argv[argi], "exact") == 0) cfg.exact_rank_revealing = true;
  try {
    SparseSymMatrix a;
    std::vector<double> b;
    Partition p;
    load_dump(prefix + ".bin", a, b, p);
    ProblemContext ctx(a, b, p);
    ctx.setup(cfg);
    auto [x, rep] = pcg(ctx, ctx.rhs(), 1e-8, 10000);
    AwgPreconditioner h3{&ctx};
    std::vector<double> y = h3.apply(b);
    const awg_stats st = ctx.stats();
    std::printf("{\"iterations\": %d, \"converged\": %d, \"kappa\": %.17g, \"n0\": %d, \"n_minus\": %d, "
                "\"x0\": %.17g, \"y0\": %.17g}\n",
                rep.iterations, rep.converged ? 1 : 0, rep.kappa_estimate, st.n0, st.n_minus, x[0], y[0]);
    FILE* f = std::fopen((prefix + ".x").c_str(), "w");
    for (double v : x) std::fprintf(f, "%.17g\n", v);
    std::fclose(f);
  } catch (const NotSpdError& e) {
    std::fprintf(stderr, "NotSpdError(%d): %s\n", e.pivot_index, e.what());
    return 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
