// C++ caller of the host API (include/awg_b200/awg.hpp), written the way the
// reference's run_with_context (proj/src/harness.cpp:131-139) drives its
// library: external files in, preconditioner build, PCG with H3 — on the GPU.
//   host_api_main <prefix> <tau|-k K> [exact]
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "awg_b200/awg.hpp"

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
    SparseSymMatrix a = read_matrix_market(prefix + ".mtx");
    std::vector<double> b = read_vector(prefix + ".rhs");
    Partition p = read_partition(prefix + ".part", a.n);
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
