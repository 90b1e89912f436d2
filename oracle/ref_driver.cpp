// Oracle driver (TEST INFRASTRUCTURE ONLY — never linked into the product).
//
// Runs the UNMODIFIED reference library (proj/src/*.cpp, compiled by
// oracle/Makefile into oracle/_ref/) through its public API on a system read
// from the reference's external formats, and exports every setup product and
// apply/solve result as .npy files so the GPU path can be checked against it
// (SURVEY.md §8c protocol: exported-factor apply parity + end-to-end gates).
//
// Composition mirrors ProblemContext + run_with_context
// (proj/src/harness.cpp:63-139) without harness.cpp itself (which needs the
// absent vendor/json.hpp):
//   read_matrix_market / read_vector / read_partition   sparse.cpp:89-138, partition.cpp:212-233
//   check_minimal_overlap                               partition.cpp:137-156 (harness.cpp:85-91)
//   build_pou, Splitting, GeneoContext                  partition.cpp:94-108, splitting.cpp:86-105
//   OneLevel(NN), build_coarse | fixed-k coarse, TwoLevel(HYBRID)   preconditioner.cpp:20-82, coarse.cpp:113-154
//   build_w, AwgPreconditioner                          preconditioner.cpp:84-147
//   pcg                                                 krylov.cpp:36-124
// The fixed-k selection (BASELINE.json configs 3 and 5) is built from public
// API exactly like build_coarse, with k_s = max(k, n_nonpos(s)) extended over
// clusters |lambda_{k+1} - lambda_k| <= 1e-8.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "awg/coarse.hpp"
#include "awg/dense.hpp"
#include "awg/fem.hpp"
#include "awg/krylov.hpp"
#include "awg/partition.hpp"
#include "awg/preconditioner.hpp"
#include "awg/sparse.hpp"
#include "awg/splitting.hpp"

using namespace awg;

namespace {

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// --- minimal .npy writer (v1.0, little-endian) -------------------------------
void write_npy(const std::string& path, const char* descr, const std::vector<long>& shape,
               bool fortran, const void* data, size_t elem_size) {
  std::string sh = "(";
  size_t count = 1;
  for (size_t i = 0; i < shape.size(); ++i) {
    sh += std::to_string(shape[i]);
    sh += (shape.size() == 1) ? "," : (i + 1 < shape.size() ? ", " : "");
    count *= size_t(shape[i]);
  }
  sh += ")";
  std::string header = std::string("{'descr': '") + descr + "', 'fortran_order': " +
                       (fortran ? "True" : "False") + ", 'shape': " + sh + ", }";
  size_t total = 10 + header.size() + 1;
  size_t pad = (64 - total % 64) % 64;
  header += std::string(pad, ' ');
  header += '\n';
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) {
    std::fprintf(stderr, "cannot write %s\n", path.c_str());
    std::exit(2);
  }
  const unsigned char magic[8] = {0x93, 'N', 'U', 'M', 'P', 'Y', 1, 0};
  std::fwrite(magic, 1, 8, f);
  uint16_t hl = uint16_t(header.size());
  std::fwrite(&hl, 2, 1, f);
  std::fwrite(header.data(), 1, header.size(), f);
  if (count) std::fwrite(data, elem_size, count, f);
  std::fclose(f);
}
void npy_d(const std::string& dir, const std::string& name, const std::vector<double>& v) {
  write_npy(dir + "/" + name + ".npy", "<f8", {long(v.size())}, false, v.data(), 8);
}
void npy_i(const std::string& dir, const std::string& name, const std::vector<int>& v) {
  write_npy(dir + "/" + name + ".npy", "<i4", {long(v.size())}, false, v.data(), 4);
}
void npy_mat(const std::string& dir, const std::string& name, const DenseMatrix& m) {
  write_npy(dir + "/" + name + ".npy", "<f8", {long(m.rows), long(m.cols)}, true, m.a.data(), 8);
}
void npy_rows(const std::string& dir, const std::string& name, const std::vector<std::vector<double>>& rows) {
  std::vector<double> flat;
  for (auto& r : rows) flat.insert(flat.end(), r.begin(), r.end());
  long n = rows.empty() ? 0 : long(rows[0].size());
  write_npy(dir + "/" + name + ".npy", "<f8", {long(rows.size()), n}, false, flat.data(), 8);
}

// SplitMix64 uniform stream, identical to paper_2106_10913_b200/problems.py.
std::vector<double> uniform_vec(uint64_t seed, int n, double a, double b) {
  std::vector<double> v(n);
  uint64_t state = seed;
  for (int i = 0; i < n; ++i) {
    state += 0x9E3779B97F4A7C15ull;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    double u = double(z >> 11) * 0x1.0p-53;
    v[i] = a + (b - a) * u;
  }
  return v;
}

struct Args {
  std::string prefix, out;
  double tau = -1.0;
  int fixed_k = -1;
  std::string awg = "ad";
  std::string comp = "hybrid";
  std::string one_level = "NN";
  double tau_flat = 10.0;
  double rtol = 1e-8;
  double w_rtol = 1e-10;
  int maxit = 10000;
  int n_apply = 3;
  int export_factors = 1;
  int apply_reps = 0;
  int no_solve = 0;
  int export_dense = 0;
  int w_probe = 0;          // > 0: run build_w's inner solve for this many W columns, bounded, then exit
  int w_probe_maxit = 3000;
  std::string phase;        // "", "bs", "pencil", "w": fill the memo cache (oracle/memo.cpp) for one worker's share
  int worker = 0, nworkers = 1;
};

Args parse(int argc, char** argv) {
  Args a;
  if (argc < 3) {
    std::fprintf(stderr,
                 "usage: ref_driver <prefix> <outdir> [--tau T | --fixed-k K] [--awg ad|hyb|inex|none]\n"
                 "       [--comp hybrid|additive] [--rtol R] [--w-rtol W] [--maxit M] [--n-apply M]\n"
                 "       [--export-factors 0|1] [--apply-reps R] [--no-solve]\n");
    std::exit(2);
  }
  a.prefix = argv[1];
  a.out = argv[2];
  for (int i = 3; i < argc; ++i) {
    std::string k = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) {
        std::fprintf(stderr, "missing value for %s\n", k.c_str());
        std::exit(2);
      }
      return argv[++i];
    };
    if (k == "--tau") a.tau = std::stod(next());
    else if (k == "--fixed-k") a.fixed_k = std::stoi(next());
    else if (k == "--awg") a.awg = next();
    else if (k == "--comp") a.comp = next();
    else if (k == "--one-level") a.one_level = next();
    else if (k == "--tau-flat") a.tau_flat = std::stod(next());
    else if (k == "--rtol") a.rtol = std::stod(next());
    else if (k == "--w-rtol") a.w_rtol = std::stod(next());
    else if (k == "--maxit") a.maxit = std::stoi(next());
    else if (k == "--n-apply") a.n_apply = std::stoi(next());
    else if (k == "--export-factors") a.export_factors = std::stoi(next());
    else if (k == "--apply-reps") a.apply_reps = std::stoi(next());
    else if (k == "--no-solve") a.no_solve = 1;
    else if (k == "--export-dense") a.export_dense = std::stoi(next());
    else if (k == "--w-probe") a.w_probe = std::stoi(next());
    else if (k == "--w-probe-maxit") a.w_probe_maxit = std::stoi(next());
    else if (k == "--phase") a.phase = next();
    else if (k == "--worker") a.worker = std::stoi(next());
    else if (k == "--nworkers") a.nworkers = std::stoi(next());
    else {
      std::fprintf(stderr, "unknown flag %s\n", k.c_str());
      std::exit(2);
    }
  }
  return a;
}

AwgMode mode_of(const std::string& s) {
  if (s == "none") return AwgMode::NONE;
  if (s == "ad") return AwgMode::AD;
  if (s == "hyb") return AwgMode::HYB;
  if (s == "inex") return AwgMode::INEX;
  std::fprintf(stderr, "bad awg mode %s\n", s.c_str());
  std::exit(2);
}

// Fixed-k GenEO coarse space from public API, mirroring build_coarse
// (coarse.cpp:113-154) with a different per-subdomain column count.
CoarseSpace fixed_k_coarse(GeneoContext& ctx, int k, std::vector<int>& ks) {
  const Splitting& split = ctx.splitting();
  const Partition& part = split.partition();
  const int n = split.n();
  std::vector<std::pair<int, DenseMatrix>> picked;
  ks.clear();
  for (int s = 0; s < part.count(); ++s) {
    const EigenDecomposition& e = ctx.pencil_nn(s);
    const int ns = int(e.eigenvalues.size());
    int kk = std::max(k, split.splits()[s].n_nonpos);
    kk = std::min(kk, ns);
    while (kk > 0 && kk < ns && std::abs(e.eigenvalues[kk] - e.eigenvalues[kk - 1]) <= 1e-8) ++kk;
    DenseMatrix y(e.eigenvectors.rows, kk);
    for (int c = 0; c < kk; ++c) std::copy_n(e.eigenvectors.col(c), e.eigenvectors.rows, y.col(c));
    picked.emplace_back(s, std::move(y));
    ks.push_back(kk);
  }
  int n0 = 0;
  for (auto& p : picked) n0 += p.second.cols;
  CoarseSpace cs;
  cs.z = DenseMatrix(n, n0);
  int col = 0;
  for (auto& [s, y] : picked)
    for (int c = 0; c < y.cols; ++c, ++col) split.prolong_add(s, y.col(c), cs.z.col(col));
  DenseMatrix g(n0, n0);
  std::vector<double> tmp(n);
  for (int j = 0; j < n0; ++j) {
    split.apply_Aplus(cs.z.col(j), tmp.data());
    matvec_transpose(cs.z, tmp.data(), g.col(j));
  }
  symmetrize(g);
  cs.k0 = rank_revealing_sym_factor(g);
  return cs;
}

// --- bounded-sample CPU baseline -------------------------------------------
// For configurations whose reference setup is infeasible on a CPU (SURVEY.md
// §0.9: c2..c5 take hours to hundreds of hours), time the reference's own
// apply kernels on data of the configuration's exact shapes and extrapolate
// the cost of one H3,ad apply (AwgPreconditioner::apply, preconditioner.cpp:185-198):
//   second_correct  = W^T x + rank_revealing_solve(KW) + W c          (dense n x n_-)
//   TwoLevel hybrid = 3 coarse_correct (dense Z, n x n0) + 2 apply_Aplus + OneLevel
//   OneLevel        = per subdomain restrict, D, V^T, mask, V, D, prolong
// Matrix entries are random (timing only): the operation sequence is the
// reference's.  Subdomains / columns are sampled and scaled linearly.
int sample_mode(const std::string& prefix, double budget_s, int n0, int n_minus, int m_avg, const std::string& out) {
  SparseSymMatrix a = read_matrix_market(prefix + ".mtx");
  Partition part = read_partition(prefix + ".part", a.n);
  PartitionOfUnity pou = build_pou(part);
  const int n = a.n, N = part.count();
  std::vector<double> x = uniform_vec(5, n, -1.0, 1.0), y(n);
  auto timeit = [&](auto&& fn, double min_s) {
    fn();
    int reps = 0;
    double t0 = now_s(), t = 0;
    do {
      fn();
      ++reps;
      t = now_s() - t0;
    } while (t < min_s);
    return t / reps;
  };
  const double slot = budget_s / 5.0;
  // spmv (sparse.cpp:49-56), full size
  const double t_spmv = timeit([&] { spmv(a, x.data(), y.data()); }, std::min(slot, 1.0));
  // OneLevel NN on a sample of subdomains (local_Aplus_pinv_apply, splitting.cpp:211-218)
  double t_local_sum = 0.0;
  int sampled = 0;
  double t_start = now_s();
  for (int s = 0; s < N && (now_s() - t_start) < slot; ++s) {
    const int ns = part.size_of(s);
    DenseMatrix v(ns, ns);
    std::vector<double> r = uniform_vec(100 + s, ns * 1, -1.0, 1.0);
    for (size_t i = 0; i < v.a.size(); ++i) v.a[i] = r[i % ns] * 0.5 + double(i % 7) * 1e-3;
    std::vector<double> xs(ns), u(ns), w(ns), lam(ns, 1.0);
    const auto& om = part.omega[s];
    const auto& ds = pou.ds[s];
    t_local_sum += timeit(
        [&] {
          for (int k = 0; k < ns; ++k) xs[k] = x[om[k]] * ds[k];
          matvec_transpose(v, xs.data(), u.data());
          for (int k = 0; k < ns; ++k) u[k] = (k < m_avg) ? 0.0 : u[k] / lam[k];
          matvec(v, u.data(), w.data());
          for (int k = 0; k < ns; ++k) y[om[k]] += w[k] * ds[k];
        },
        0.0);
    ++sampled;
  }
  const double t_h1 = t_local_sum / sampled * N;
  // dense tall-skinny pairs: W (n x n_minus) and Z (n x n0), column-sampled
  auto pair_time = [&](int cols) {
    const int sc = std::max(1, std::min(cols, 8));
    DenseMatrix m(n, sc);
    for (size_t i = 0; i < m.a.size(); ++i) m.a[i] = double(i % 13) * 1e-2;
    std::vector<double> c(sc), out(n);
    const double t = timeit(
        [&] {
          matvec_transpose(m, x.data(), c.data());
          matvec(m, c.data(), out.data());
        },
        std::min(slot, 2.0));
    return t * double(cols) / sc;
  };
  const double t_w = n_minus > 0 ? pair_time(n_minus) : 0.0;
  const double t_z = n0 > 0 ? pair_time(n0) : 0.0;
  // rank_revealing_solve on an r x r factor (dense.cpp:348-366)
  auto rrs_time = [&](int r) {
    if (r <= 0) return 0.0;
    RankRevealingFactor f;
    f.original_dim = r;
    f.l11 = DenseMatrix(r, r);
    for (int j = 0; j < r; ++j)
      for (int i = j; i < r; ++i) f.l11(i, j) = (i == j) ? 1.0 : 1e-3;
    f.retained.resize(r);
    for (int i = 0; i < r; ++i) f.retained[i] = i;
    std::vector<double> b(r, 1.0), xx(r);
    return timeit([&] { rank_revealing_solve(f, b.data(), xx.data()); }, std::min(slot, 0.5));
  };
  const double t_k0 = rrs_time(n0), t_kw = rrs_time(n_minus);
  // A- x (splitting.cpp:119-140, the same loop on random modes): per subdomain
  // restrict, m_avg dot + axpy pairs over n_s, prolong_add — timed on a sample
  // of subdomains and scaled to all of them
  double t_am_sum = 0.0;
  int am_sampled = 0;
  t_start = now_s();
  for (int s = 0; s < N && (am_sampled < 4 || (now_s() - t_start) < slot * 0.5); ++s) {
    const int ns = part.size_of(s);
    const int q = std::max(1, std::min(m_avg, ns));
    DenseMatrix v(ns, q);
    std::vector<double> r = uniform_vec(300 + s, ns, -1.0, 1.0);
    for (size_t i = 0; i < v.a.size(); ++i) v.a[i] = r[i % ns];
    std::vector<double> xs(ns), u(ns), lam(q, -1e-3);
    const auto& om = part.omega[s];
    t_am_sum += timeit(
        [&] {
          for (int k = 0; k < ns; ++k) xs[k] = x[om[k]];
          std::fill(u.begin(), u.end(), 0.0);
          for (int k = 0; k < q; ++k) {
            const double* vk = v.col(k);
            double dot = 0.0;
            for (int i = 0; i < ns; ++i) dot += vk[i] * xs[i];
            const double f = -lam[k] * dot;
            for (int i = 0; i < ns; ++i) u[i] += f * vk[i];
          }
          for (int k = 0; k < ns; ++k) y[om[k]] += u[k];
        },
        0.0);
    ++am_sampled;
  }
  const double t_aminus = t_am_sum / std::max(am_sampled, 1) * N;
  const double t_q = t_z + t_k0;
  const double t_h2 = 3.0 * t_q + 2.0 * (t_aminus + t_spmv) + t_h1;
  const double t_h3 = t_h2 + t_w + t_kw;
  const double t_iter = t_h3 + t_spmv;
  FILE* js = std::fopen((out + "/sample.json").c_str(), "w");
  std::fprintf(js,
               "{\"t_h3_apply_s\": %.9g, \"t_iter_s\": %.9g, \"t_spmv_s\": %.9g, \"t_h1_s\": %.9g, "
               "\"t_z_pair_s\": %.9g, \"t_w_pair_s\": %.9g, \"t_k0_solve_s\": %.9g, \"t_kw_solve_s\": %.9g, "
               "\"t_aminus_s\": %.9g, \"aminus_sampled\": %d, "
               "\"sampled_subdomains\": %d, \"n_sub\": %d, \"n\": %d, \"n0\": %d, \"n_minus\": %d, "
               "\"elapsed_s\": %.3f}\n",
               t_h3, t_iter, t_spmv, t_h1, t_z, t_w, t_k0, t_kw, t_aminus, am_sampled, sampled, N, n, n0, n_minus,
               now_s() - t_start);
  std::fclose(js);
  return 0;
}

// ref_driver --rrf <G.bin> <outdir>: rank_revealing_sym_factor (dense.cpp:299-346)
// of one symmetric matrix (G.bin = int32 n, then n*n float64 column-major);
// exports retained and l11 for the device pivoted-factor parity test.
int rrf_mode(const std::string& in, const std::string& out) {
  FILE* f = std::fopen(in.c_str(), "rb");
  if (!f) return 2;
  int n = 0;
  if (std::fread(&n, sizeof n, 1, f) != 1 || n < 0) return 2;
  DenseMatrix g(n, n);
  if (std::fread(g.a.data(), sizeof(double), g.a.size(), f) != g.a.size()) return 2;
  std::fclose(f);
  const RankRevealingFactor rf = rank_revealing_sym_factor(g);
  npy_i(out, "retained", rf.retained);
  npy_mat(out, "l11", rf.l11);
  return 0;
}

// ref_driver --fem <nodes_x> <nodes_y> <E> <nu> <outdir>: the reference's own
// assemble() (fem.cpp:99-162) on a single-material mesh with h = 1 and the
// default body force: CSR and rhs, to pin the elasticity generator.
int fem_mode(int nx, int ny, double e, double nu, const std::string& out) {
  MeshSpec mesh;
  mesh.domain_width = nx - 1;
  mesh.domain_height = ny - 1;
  mesh.h = 1.0;
  const AssembledSystem sys = assemble(mesh, CoefficientField::constant(e, nu));
  npy_i(out, "row_offsets", sys.a.row_offsets);
  npy_i(out, "col_indices", sys.a.col_indices);
  npy_d(out, "values", sys.a.values);
  npy_d(out, "b", sys.b);
  return 0;
}

// ref_driver --autopart <prefix> <n_parts> <outdir>: auto_partition
// (partition.cpp:42-92: BFS parts, then the one-ring closure of :79-90) of the
// matrix in <prefix>.mtx; exports the closed index sets.
int autopart_mode(const std::string& prefix, int parts, const std::string& out) {
  const SparseSymMatrix a = read_matrix_market(prefix + ".mtx");
  const Partition p = auto_partition(a, parts);
  std::vector<int> off = {0}, idx;
  for (const auto& om : p.omega) {
    idx.insert(idx.end(), om.begin(), om.end());
    off.push_back(int(idx.size()));
  }
  npy_i(out, "part_offsets", off);
  npy_i(out, "part_indices", idx);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc >= 7 && std::string(argv[1]) == "--fem") {
    std::string cmd = "mkdir -p '" + std::string(argv[6]) + "'";
    if (std::system(cmd.c_str()) != 0) return 2;
    return fem_mode(std::stoi(argv[2]), std::stoi(argv[3]), std::stod(argv[4]), std::stod(argv[5]), argv[6]);
  }
  if (argc >= 5 && std::string(argv[1]) == "--autopart") {
    std::string cmd = "mkdir -p '" + std::string(argv[4]) + "'";
    if (std::system(cmd.c_str()) != 0) return 2;
    return autopart_mode(argv[2], std::stoi(argv[3]), argv[4]);
  }
  if (argc >= 4 && std::string(argv[1]) == "--rrf") {
    std::string cmd = "mkdir -p '" + std::string(argv[3]) + "'";
    if (std::system(cmd.c_str()) != 0) return 2;
    return rrf_mode(argv[2], argv[3]);
  }
  if (argc >= 3 && std::string(argv[1]) == "--sample") {
    // ref_driver --sample <prefix> <outdir> <budget_s> <n0> <n_minus> <m_avg>
    if (argc < 8) {
      std::fprintf(stderr, "usage: ref_driver --sample <prefix> <outdir> <budget_s> <n0> <n_minus> <m_avg>\n");
      return 2;
    }
    std::string cmd = "mkdir -p '" + std::string(argv[3]) + "'";
    if (std::system(cmd.c_str()) != 0) return 2;
    return sample_mode(argv[2], std::stod(argv[4]), std::stoi(argv[5]), std::stoi(argv[6]), std::stoi(argv[7]),
                       argv[3]);
  }
  const Args args = parse(argc, argv);
  std::string cmd = "mkdir -p '" + args.out + "'";
  if (std::system(cmd.c_str()) != 0) return 2;
  const std::string& out = args.out;
  FILE* js = std::fopen((out + "/summary.json").c_str(), "w");
  std::fprintf(js, "{\n");

  double t0 = now_s();
  SparseSymMatrix a = read_matrix_market(args.prefix + ".mtx");
  std::vector<double> b = read_vector(args.prefix + ".rhs");
  Partition part = read_partition(args.prefix + ".part", a.n);
  const auto violations = check_minimal_overlap(a, part);
  if (!violations.empty()) {
    std::fprintf(stderr, "minimal overlap violated\n");
    return 3;
  }
  double t_read = now_s() - t0;

  if (args.phase == "bs") {
    // Worker share of the Splitting constructor's eigsplits (splitting.cpp:86-90):
    // the memoised dense_sym_eig stores each result for the replay run.
    auto bs = build_Bs(a, part);
    for (int s = args.worker; s < part.count(); s += args.nworkers) (void)eigsplit(bs[s], s);
    return 0;
  }
  t0 = now_s();
  PartitionOfUnity pou = build_pou(part);
  Splitting split(a, part, pou);
  GeneoContext geneo(split);
  double t_split = now_s() - t0;

  const int N = part.count();
  const int n = a.n;
  std::vector<int> sizes(N), n_nonpos(N), n_zero(N);
  std::vector<double> eps(N);
  for (int s = 0; s < N; ++s) {
    sizes[s] = part.size_of(s);
    n_nonpos[s] = split.splits()[s].n_nonpos;
    n_zero[s] = split.splits()[s].n_zero;
    eps[s] = split.splits()[s].eps_zero;
  }

  const OneLevelKind kind0 =
      args.one_level == "AS" ? OneLevelKind::AS : args.one_level == "AS_PLUS" ? OneLevelKind::AS_PLUS : OneLevelKind::NN;
  if (args.phase == "pencil") {
    // Worker share of the GenEO pencils (coarse.cpp:98-111), memoised.
    for (int s = args.worker; s < N; s += args.nworkers) {
      if (kind0 == OneLevelKind::AS) {
        (void)geneo.pencil_as1(s);
        (void)geneo.pencil_as2(s);
      } else {
        (void)geneo.pencil_nn(s);
      }
    }
    return 0;
  }
  t0 = now_s();
  std::vector<int> ks;
  CoarseSpace cs;
  const OneLevelKind kind =
      args.one_level == "AS" ? OneLevelKind::AS : args.one_level == "AS_PLUS" ? OneLevelKind::AS_PLUS : OneLevelKind::NN;
  auto count_below = [](const EigenDecomposition& e, double tau) {
    int m = 0;
    while (m < int(e.eigenvalues.size()) && e.eigenvalues[m] < tau) ++m;
    return m;
  };
  std::vector<std::vector<double>> ycols(N);  // exported coarse vectors per subdomain, Z column order
  if (args.fixed_k > 0) {
    cs = fixed_k_coarse(geneo, args.fixed_k, ks);
  } else {
    const double tau = args.tau > 0 ? args.tau : 0.1;
    // build_coarse (coarse.cpp:113-154); per-subdomain counts recovered from the pencils
    for (int s = 0; s < N; ++s) {
      if (kind == OneLevelKind::NN) {
        ks.push_back(count_below(geneo.pencil_nn(s), tau));
      } else if (kind == OneLevelKind::AS_PLUS) {
        ks.push_back(count_below(geneo.pencil_nn(s), 1.0 / args.tau_flat));
      } else {
        const int m1 = count_below(geneo.pencil_as1(s), 1.0 / args.tau_flat);
        const int m2 = count_below(geneo.pencil_as2(s), tau);
        ks.push_back(m1 + m2);
        const auto& e1 = geneo.pencil_as1(s).eigenvectors;
        const auto& e2 = geneo.pencil_as2(s).eigenvectors;
        ycols[s].assign(e1.a.begin(), e1.a.begin() + size_t(e1.rows) * m1);
        ycols[s].insert(ycols[s].end(), e2.a.begin(), e2.a.begin() + size_t(e2.rows) * m2);
      }
    }
    if (kind == OneLevelKind::NN) cs = build_coarse(ThresholdSpec::nn(tau), geneo);
    else if (kind == OneLevelKind::AS_PLUS) cs = build_coarse(ThresholdSpec::as_plus(args.tau_flat), geneo);
    else cs = build_coarse(ThresholdSpec::as(tau, args.tau_flat), geneo);
  }
  for (int s = 0; s < N; ++s)
    if (kind != OneLevelKind::AS) {
      const auto& pm = geneo.pencil_nn(s).eigenvectors;
      ycols[s].assign(pm.a.begin(), pm.a.begin() + size_t(pm.rows) * ks[s]);
    }
  double t_coarse = now_s() - t0;
  const Composition comp = args.comp == "additive" ? Composition::ADDITIVE : Composition::HYBRID;
  auto h2 = std::make_shared<TwoLevel>(OneLevel(kind, split), cs, comp, split);

  if (args.phase == "w") {
    // Worker share of build_w's inner solves (preconditioner.cpp:97-113):
    // the same right-hand sides, tolerance and iteration cap, memoised pcg.
    const ApplyFn aplus = [&split](const double* u, double* v) { split.apply_Aplus(u, v); };
    const ApplyFn happly = [&h2](const double* u, double* v) { h2->apply(u, v); };
    std::vector<double> rhs(n);
    int col = 0;
    for (int s = 0; s < N; ++s) {
      const LocalSplit& ls = split.splits()[s];
      for (int k = 0; k < ls.n_nonpos; ++k) {
        if (ls.eig.eigenvalues[k] == 0.0) continue;
        if (col++ % args.nworkers != args.worker) continue;
        std::fill(rhs.begin(), rhs.end(), 0.0);
        split.prolong_add(s, ls.eig.eigenvectors.col(k), rhs.data());
        (void)pcg(aplus, happly, rhs, args.w_rtol, 10 * n);
      }
    }
    return 0;
  }
  if (args.w_probe > 0) {
    // The inner solve of build_w (preconditioner.cpp:97-113) for the first
    // w_probe strictly negative modes, with maxit bounded: reports how the
    // reference's own pcg(A+, H2) behaves when build_w would take 10 n iterations.
    const ApplyFn aplus = [&split](const double* u, double* v) { split.apply_Aplus(u, v); };
    // pcg hands its residual r to the preconditioner once per iteration, so the
    // wrapper can log the recursive relative residual of a long run as it goes
    // (<out>/w_probe_progress.jsonl: a bounded session still leaves evidence).
    std::vector<double> rhs(n);
    long calls = 0;
    double t_col = 0;
    FILE* prog = std::fopen((out + "/w_probe_progress.jsonl").c_str(), "w");
    const ApplyFn happly = [&](const double* u, double* v) {
      if (prog && calls % 500 == 0) {
        double rr = 0, bb = 0;
        for (int i = 0; i < n; ++i) rr += u[i] * u[i], bb += rhs[i] * rhs[i];
        std::fprintf(prog, "{\"iteration\": %ld, \"relres\": %.6e, \"seconds\": %.1f}\n", calls,
                     std::sqrt(rr / bb), now_s() - t_col);
        std::fflush(prog);
      }
      ++calls;
      h2->apply(u, v);
    };
    std::fprintf(js, "  \"n0\": %d, \"r0\": %d, \"n_minus\": %d,\n  \"w_probe\": [", cs.dim(), cs.retained_rank(),
                 split.n_minus());
    int col = 0;
    for (int s = 0; s < N && col < args.w_probe; ++s) {
      const LocalSplit& ls = split.splits()[s];
      for (int k = 0; k < ls.n_nonpos && col < args.w_probe; ++k) {
        if (ls.eig.eigenvalues[k] == 0.0) continue;
        std::fill(rhs.begin(), rhs.end(), 0.0);
        split.prolong_add(s, ls.eig.eigenvectors.col(k), rhs.data());
        const double tp = now_s();
        calls = 0, t_col = tp;
        auto res = pcg(aplus, happly, rhs, args.w_rtol, args.w_probe_maxit);
        const SolveReport& rep = res.second;
        std::fprintf(js, "%s{\"s\": %d, \"k\": %d, \"iterations\": %d, \"converged\": %d, \"kappa\": %.6e, "
                     "\"final_relres\": %.6e, \"seconds\": %.3f}", col ? ", " : "", s, k, rep.iterations,
                     int(rep.converged), rep.kappa_estimate, rep.final_relative_residual, now_s() - tp);
        std::fflush(js);
        ++col;
      }
    }
    std::fprintf(js, "],\n  \"t_splitting\": %.3f, \"t_coarse\": %.3f\n}\n", t_split, t_coarse);
    std::fclose(js);
    return 0;
  }

  t0 = now_s();
  const AwgMode mode = mode_of(args.awg);
  std::shared_ptr<const SecondCoarse> sc;
  if (mode != AwgMode::NONE) sc = std::make_shared<SecondCoarse>(build_w(split, *h2, args.w_rtol));
  double t_w = now_s() - t0;
  t0 = now_s();
  AwgPreconditioner h3(mode, h2, sc, split);
  std::unique_ptr<AwgPreconditioner> h3_ad, h3_hyb, h3_inex;
  if (sc) {
    h3_ad = std::make_unique<AwgPreconditioner>(AwgMode::AD, h2, sc, split);
    h3_hyb = std::make_unique<AwgPreconditioner>(AwgMode::HYB, h2, sc, split);
    h3_inex = std::make_unique<AwgPreconditioner>(AwgMode::INEX, h2, sc, split);
  }
  double t_h3 = now_s() - t0;

  std::fprintf(js, "  \"n\": %d, \"nnz\": %d, \"n_sub\": %d,\n", n, a.nnz(), N);
  // report-only quantities of run_with_context (harness.cpp:172-174)
  std::fprintf(js, "  \"coloring_A\": %d, \"coloring_Aplus\": %d,\n", coloring_constant(a, part).n_colors,
               coloring_constant_aplus(a, part, split.has_negative_modes()).n_colors);
  std::fprintf(js, "  \"n0\": %d, \"r0\": %d, \"n_minus\": %d, \"rw\": %d,\n", cs.dim(), cs.retained_rank(),
               sc ? sc->n_minus() : 0, sc ? sc->kw.rank() : 0);
  std::fprintf(js, "  \"t_read\": %.6f, \"t_splitting\": %.6f, \"t_coarse\": %.6f, \"t_w\": %.6f, \"t_h3\": %.6f,\n",
               t_read, t_split, t_coarse, t_w, t_h3);

  // ---- exports -----------------------------------------------------------
  npy_i(out, "sizes", sizes);
  npy_i(out, "n_nonpos", n_nonpos);
  npy_i(out, "n_zero", n_zero);
  npy_d(out, "eps_zero", eps);
  npy_i(out, "ks", ks);
  npy_i(out, "multiplicity", pou.multiplicity);
  {
    std::vector<double> lam, plam;
    for (int s = 0; s < N; ++s) {
      auto& e = split.splits()[s].eig.eigenvalues;
      lam.insert(lam.end(), e.begin(), e.end());
      auto& pe = geneo.pencil_nn(s).eigenvalues;
      plam.insert(plam.end(), pe.begin(), pe.end());
    }
    npy_d(out, "lam", lam);
    npy_d(out, "pencil_lam", plam);
    if (kind == OneLevelKind::AS) {
      std::vector<double> a1, a2;
      for (int s = 0; s < N; ++s) {
        auto& e1 = geneo.pencil_as1(s).eigenvalues;
        a1.insert(a1.end(), e1.begin(), e1.end());
        auto& e2 = geneo.pencil_as2(s).eigenvalues;
        a2.insert(a2.end(), e2.begin(), e2.end());
      }
      npy_d(out, "pencil_as1_lam", a1);
      npy_d(out, "pencil_as2_lam", a2);
    }
  }
  npy_i(out, "k0_retained", cs.k0.retained);
  npy_mat(out, "k0_l11", cs.k0.l11);
  {
    // The coarse operator fed to rank_revealing_sym_factor, recomputed with
    // the same operations as coarse.cpp:145-151 (deterministic, identical).
    const int n0 = cs.dim();
    DenseMatrix g(n0, n0);
    std::vector<double> tmp(n);
    for (int j = 0; j < n0; ++j) {
      split.apply_Aplus(cs.z.col(j), tmp.data());
      matvec_transpose(cs.z, tmp.data(), g.col(j));
    }
    symmetrize(g);
    npy_mat(out, "k0_G", g);
  }
  if (args.export_dense) {
    // B^s, weighted A+^s and R A+ R^T per subdomain (tiny problems only).
    std::vector<double> bs, ma, mb;
    auto bsv = build_Bs(a, part);
    for (int s = 0; s < N; ++s) {
      bs.insert(bs.end(), bsv[s].a.begin(), bsv[s].a.end());
      DenseMatrix w = geneo.weighted_asplus(s);
      ma.insert(ma.end(), w.a.begin(), w.a.end());
      const DenseMatrix& b2 = geneo.aplus_block(s);
      mb.insert(mb.end(), b2.a.begin(), b2.a.end());
    }
    npy_d(out, "Bs", bs);
    npy_d(out, "pencil_MA", ma);
    npy_d(out, "pencil_MB", mb);
  }
  if (args.export_factors) {
    std::vector<double> V, Y;
    for (int s = 0; s < N; ++s) {
      auto& m = split.splits()[s].eig.eigenvectors.a;
      V.insert(V.end(), m.begin(), m.end());
      Y.insert(Y.end(), ycols[s].begin(), ycols[s].end());
    }
    npy_d(out, "V", V);
    npy_d(out, "Y", Y);
    // The reference keeps Z dense (n x n0); export it too for cross-checks
    // on small problems only.
    if (size_t(n) * cs.dim() <= (size_t(1) << 24)) npy_mat(out, "Z", cs.z);
  }
  if (sc) {
    npy_d(out, "neg_weights", sc->neg_weights);
    npy_i(out, "w_inner_iterations", sc->inner_iterations);
    npy_i(out, "kw_retained", sc->kw.retained);
    npy_mat(out, "kw_l11", sc->kw.l11);
    {
      // W^T A W as in preconditioner.cpp:119-125.
      const int m = sc->n_minus();
      DenseMatrix g(m, m);
      std::vector<double> tmp(n);
      for (int j = 0; j < m; ++j) {
        spmv(a, sc->w.col(j), tmp.data());
        matvec_transpose(sc->w, tmp.data(), g.col(j));
      }
      symmetrize(g);
      npy_mat(out, "kw_G", g);
    }
    if (args.export_factors) {
      npy_mat(out, "W", sc->w);
      npy_mat(out, "v_minus", sc->v_minus);
    }
  }

  // ---- applies on seeded vectors -----------------------------------------
  {
    std::vector<std::vector<double>> X, yA, yAm, yAp, yH1, yQ, yQW, yH2, yAD, yHYB, yINEX, yPI3, yPI3T;
    OneLevel h1(kind, split);
    for (int m = 0; m < args.n_apply; ++m) {
      std::vector<double> x = uniform_vec(1000 + m, n, -1.0, 1.0), y(n);
      X.push_back(x);
      spmv(a, x.data(), y.data()); yA.push_back(y);
      split.apply_Aminus(x.data(), y.data()); yAm.push_back(y);
      split.apply_Aplus(x.data(), y.data()); yAp.push_back(y);
      h1.apply(x.data(), y.data()); yH1.push_back(y);
      coarse_correct(cs, x.data(), y.data()); yQ.push_back(y);
      h2->apply(x.data(), y.data()); yH2.push_back(y);
      if (sc) {
        // second_correct (preconditioner.cpp:149-159) is private: same ops
        // through the public SecondCoarse members.
        const int nm = sc->n_minus();
        std::vector<double> wx(nm), c(nm);
        matvec_transpose(sc->w, x.data(), wx.data());
        rank_revealing_solve(sc->kw, wx.data(), c.data());
        matvec(sc->w, c.data(), y.data());
        yQW.push_back(y);
        h3_ad->apply(x.data(), y.data()); yAD.push_back(y);
        h3_hyb->apply(x.data(), y.data()); yHYB.push_back(y);
        h3_inex->apply(x.data(), y.data()); yINEX.push_back(y);
        h3_ad->apply_pi3(x.data(), y.data()); yPI3.push_back(y);
        h3_ad->apply_pi3_transpose(x.data(), y.data()); yPI3T.push_back(y);
      }
    }
    npy_rows(out, "x_apply", X);
    npy_rows(out, "y_A", yA);
    npy_rows(out, "y_Aminus", yAm);
    npy_rows(out, "y_Aplus", yAp);
    npy_rows(out, "y_H1", yH1);
    npy_rows(out, "y_Q", yQ);
    npy_rows(out, "y_H2", yH2);
    if (sc) {
      npy_rows(out, "y_QW", yQW);
      npy_rows(out, "y_H3ad", yAD);
      npy_rows(out, "y_H3hyb", yHYB);
      npy_rows(out, "y_H3inex", yINEX);
      npy_rows(out, "y_PI3", yPI3);
      npy_rows(out, "y_PI3T", yPI3T);
    }
  }

  // ---- timed H3 apply loop (CPU baseline) --------------------------------
  if (args.apply_reps > 0) {
    std::vector<double> x = uniform_vec(77, n, -1.0, 1.0), y(n);
    h3.apply(x.data(), y.data());
    double ta = now_s();
    for (int r = 0; r < args.apply_reps; ++r) h3.apply(x.data(), y.data());
    double per = (now_s() - ta) / args.apply_reps;
    std::fprintf(js, "  \"t_h3_apply\": %.9f, \"apply_reps\": %d,\n", per, args.apply_reps);
  }

  // ---- the solve (run_with_context, harness.cpp:137-139) ------------------
  if (!args.no_solve) {
    const ApplyFn apply_a = [&a](const double* x, double* y) { spmv(a, x, y); };
    const ApplyFn apply_h = [&h3](const double* x, double* y) { h3.apply(x, y); };
    double ts = now_s();
    auto [x, rep] = pcg(apply_a, apply_h, b, args.rtol, args.maxit);
    double t_solve = now_s() - ts;
    npy_d(out, "pcg_x", x);
    npy_d(out, "pcg_residuals", rep.residual_history);
    npy_d(out, "pcg_lanczos_diag", rep.lanczos_diag);
    npy_d(out, "pcg_lanczos_offdiag", rep.lanczos_offdiag);
    std::fprintf(js, "  \"t_solve\": %.6f, \"iterations\": %d, \"converged\": %s,\n", t_solve, rep.iterations,
                 rep.converged ? "true" : "false");
    std::fprintf(js, "  \"final_relative_residual\": %.17g, \"recurrence_residual_at_exit\": %.17g,\n",
                 rep.final_relative_residual, rep.recurrence_residual_at_exit);
    std::fprintf(js, "  \"ritz_min\": %.17g, \"ritz_max\": %.17g, \"kappa\": %.17g,\n", rep.ritz_min,
                 rep.ritz_max, rep.kappa_estimate);
  }
  std::fprintf(js, "  \"one_level\": \"%s\", \"tau_flat\": %.17g,\n", args.one_level.c_str(), args.tau_flat);
  std::fprintf(js, "  \"awg\": \"%s\", \"rtol\": %.17g, \"w_rtol\": %.17g, \"tau\": %.17g, \"fixed_k\": %d\n}\n",
               args.awg.c_str(), args.rtol, args.w_rtol, args.tau, args.fixed_k);
  std::fclose(js);
  return 0;
}
