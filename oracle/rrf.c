/* TEST INFRASTRUCTURE ONLY — C restatement of rank_revealing_sym_factor
 * (proj/src/dense.cpp:299-346) for the oracle.  Written in C so the trailing
 * update uses the same fused multiply-add contraction as the reference build
 * (GCC, -ffp-contract=fast): the pivot order of this factorization is decided
 * by near-ties and is therefore rounding-sensitive.
 *
 * w: n x n column-major working copy (already symmetrized), overwritten;
 * perm: n ints; returns the rank r; the factor is w[0:r,0:r] (lower).
 * exact = 0: reference semantics (stale upper triangle swapped in, :313-318);
 * exact = 1: the trailing upper triangle is refreshed before each swap. */
#include <math.h>

int awg_oracle_rrf(double* w, int n, double drop_tol, int exact, int* perm) {
#define W(i, j) w[(long)(i) + (long)(j) * n]
  for (int i = 0; i < n; ++i) perm[i] = i;
  double first = 0.0;
  int r = 0;
  for (; r < n; ++r) {
    int best = r;
    for (int k = r + 1; k < n; ++k)
      if (W(k, k) > W(best, best)) best = k;
    const double piv = W(best, best);
    if (r == 0) first = piv;
    if (piv <= drop_tol * first || piv <= 0.0) break;
    if (exact)
      for (int j = r; j < n; ++j)
        for (int i = j + 1; i < n; ++i) W(j, i) = W(i, j);
    if (best != r) {
      int t = perm[r];
      perm[r] = perm[best];
      perm[best] = t;
      for (int k = 0; k < n; ++k) {
        double a = W(k, r);
        W(k, r) = W(k, best);
        W(k, best) = a;
      }
      for (int k = 0; k < n; ++k) {
        double a = W(r, k);
        W(r, k) = W(best, k);
        W(best, k) = a;
      }
    }
    const double lkk = sqrt(W(r, r));
    W(r, r) = lkk;
    const double inv = 1.0 / lkk;
    for (int i = r + 1; i < n; ++i) W(i, r) *= inv;
    for (int j = r + 1; j < n; ++j) {
      const double f = W(j, r);
      if (f == 0.0) continue;
      for (int i = j; i < n; ++i) W(i, j) -= f * W(i, r);
    }
  }
  return r;
#undef W
}
