// TEST INFRASTRUCTURE ONLY.  Strong definition of
// awg::rank_revealing_sym_factor that replaces the reference's (weakened in a
// copy of dense.o by oracle/Makefile) to build the "probe-fixed" oracle of
// identical greedy pivot rule and drop rule
// (proj/src/dense.cpp:320-328), but the trailing matrix is kept symmetric
// before every row/column swap, so the result is a true pivoted Cholesky
// factor (the shipped version swaps in stale upper-triangle values,
// dense.cpp:313-318 with :334-338).
#include <cmath>
#include <numeric>
#include <stdexcept>

#include "awg/dense.hpp"

namespace awg {

RankRevealingFactor rank_revealing_sym_factor(const DenseMatrix& m, double drop_tol) {
  if (m.rows != m.cols) throw std::invalid_argument("rank_revealing_sym_factor: not square");
  const int n = m.rows;
  RankRevealingFactor out;
  out.original_dim = n;
  if (n == 0) return out;
  DenseMatrix w = m;
  symmetrize(w);
  std::vector<int> perm(n);
  std::iota(perm.begin(), perm.end(), 0);
  double first = 0.0;
  int r = 0;
  for (; r < n; ++r) {
    int best = r;
    for (int k = r + 1; k < n; ++k)
      if (w(k, k) > w(best, best)) best = k;
    const double piv = w(best, best);
    if (r == 0) first = piv;
    if (piv <= drop_tol * first || piv <= 0.0) break;
    // Refresh the trailing upper triangle from the (updated) lower one.
    for (int j = r; j < n; ++j)
      for (int i = j + 1; i < n; ++i) w(j, i) = w(i, j);
    if (best != r) {
      std::swap(perm[r], perm[best]);
      for (int k = 0; k < n; ++k) std::swap(w(k, r), w(k, best));
      for (int k = 0; k < n; ++k) std::swap(w(r, k), w(best, k));
    }
    const double lkk = std::sqrt(w(r, r));
    w(r, r) = lkk;
    const double inv = 1.0 / lkk;
    for (int i = r + 1; i < n; ++i) w(i, r) *= inv;
    for (int j = r + 1; j < n; ++j) {
      const double f = w(j, r);
      if (f == 0.0) continue;
      for (int i = j; i < n; ++i) w(i, j) -= f * w(i, r);
    }
  }
  out.retained.assign(perm.begin(), perm.begin() + r);
  out.l11 = DenseMatrix(r, r);
  for (int j = 0; j < r; ++j)
    for (int i = j; i < r; ++i) out.l11(i, j) = w(i, j);
  return out;
}

}  // namespace awg
