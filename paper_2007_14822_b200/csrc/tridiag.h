// tridiag.h -- host-side eigen-solver for the Lanczos tridiagonal T_j (j <= a few hundred).
// Implicit-shift QL (the EISPACK tql2 scheme, written out here): eigenvalues plus the
// rotations applied either to the full eigenvector matrix (final Ritz vector) or to the
// last row only (per-step residual estimate beta_j |y_j[last]|).  A different algorithm
// from the oracle's Sturm bisection, so the two cross-check.
#pragma once
#include <cmath>
#include <vector>

namespace heff {

// d: diagonal (n), e: off-diagonal (n-1, e[i] = T[i][i+1]).  On return d holds the
// eigenvalues (unsorted).  z: row-major nrows x n, rotations are applied to its columns
// (pass the identity for eigenvectors in columns, or the unit row e_{n-1}^T for last components).
inline bool tql_implicit(int n, std::vector<double>& d, std::vector<double> e, double* z, int nrows) {
  if (n == 0) return true;
  e.resize(n);
  e[n - 1] = 0.0;
  const double eps = 2.220446049250313e-16;
  for (int l = 0; l < n; ++l) {
    int iter = 0;
    int m;
    do {
      for (m = l; m < n - 1; ++m) {
        const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
        if (std::fabs(e[m]) <= eps * dd) break;
      }
      if (m != l) {
        if (++iter > 60) return false;
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = d[m] - d[l] + e[l] / (g + (g >= 0.0 ? std::fabs(r) : -std::fabs(r)));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        bool underflow = false;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = std::hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[m] = 0.0;
            underflow = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          for (int k = 0; k < nrows; ++k) {
            double* zk = z + (size_t)k * n;
            f = zk[i + 1];
            zk[i + 1] = s * zk[i] + c * f;
            zk[i] = c * zk[i] - s * f;
          }
        }
        if (underflow) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
  return true;
}

// Lowest eigenvalue of T and the last component of its eigenvector (per-step check).
inline bool tridiag_lowest_last(int n, const double* alpha, const double* beta, double* theta, double* ylast) {
  std::vector<double> d(alpha, alpha + n), e(beta, beta + (n > 0 ? n - 1 : 0));
  std::vector<double> z(n, 0.0);
  z[n - 1] = 1.0;
  if (!tql_implicit(n, d, e, z.data(), 1)) return false;
  int k = 0;
  for (int i = 1; i < n; ++i)
    if (d[i] < d[k]) k = i;
  *theta = d[k];
  *ylast = z[k];
  return true;
}

// Lowest eigenpair with the full eigenvector y (sign: largest |y_i| positive, reading R14).
inline bool tridiag_lowest_vec(int n, const double* alpha, const double* beta, double* theta, double* y) {
  std::vector<double> d(alpha, alpha + n), e(beta, beta + (n > 0 ? n - 1 : 0));
  std::vector<double> z((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) z[(size_t)i * n + i] = 1.0;
  if (!tql_implicit(n, d, e, z.data(), n)) return false;
  int k = 0;
  for (int i = 1; i < n; ++i)
    if (d[i] < d[k]) k = i;
  *theta = d[k];
  int imax = 0;
  for (int i = 0; i < n; ++i) {
    y[i] = z[(size_t)i * n + k];
    if (std::fabs(y[i]) > std::fabs(y[imax])) imax = i;
  }
  if (y[imax] < 0)
    for (int i = 0; i < n; ++i) y[i] = -y[i];
  return true;
}

}  // namespace heff
