// tridiag.h -- host-side eigen-solver for the Lanczos tridiagonal T_j (j <= a few hundred).
// Implicit-shift QL (the EISPACK tql2 scheme, written out here): eigenvalues plus the
// rotations applied either to the full eigenvector matrix (final Ritz vector) or to the
// last row only (per-step residual estimate beta_j |y_j[last]|).  A different algorithm
// from the oracle's Sturm bisection, so the two cross-check.
#pragma once
#include <algorithm>
#include <cmath>
#include <utility>
#include <vector>

namespace heff {

// sqrt(a^2 + b^2) without overflow or underflow in the squares (std::hypot's extra-precise
// scaling costs ~10x more and dominated the per-step checks: 0.77 ms of host time for a
// 40-step fixed Lanczos run at C1)
inline double hyp2(double a, double b) {
  a = std::fabs(a);
  b = std::fabs(b);
  const double m = a > b ? a : b;
  if (m == 0.0) return 0.0;
  const double r = (a > b ? b : a) / m;
  return m * std::sqrt(1.0 + r * r);
}

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
        double r = hyp2(g, 1.0);
        g = d[m] - d[l] + e[l] / (g + (g >= 0.0 ? std::fabs(r) : -std::fabs(r)));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        bool underflow = false;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = hyp2(f, g);
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

// ---- per-step check in O(n): lowest eigenvalue by Sturm bisection, last eigenvector
// component by inverse iteration.  The QL solve below is O(n^2) per call; called after every
// Lanczos step it made the host checks O(j^3) per run (C1, 40 steps: 0.6 ms of host time, a
// third of the solve; in converge mode the GPU idles meanwhile).  The reported energy and
// Ritz vector still come from tridiag_lowest_vec (QL) at the end.

// number of eigenvalues of T below x (LDL^T inertia; a zero pivot is nudged off zero)
inline int sturm_below(int n, const double* a, const double* b, double x, double tiny) {
  int c = 0;
  double q = a[0] - x;
  if (q < 0.0) ++c;
  for (int i = 1; i < n; ++i) {
    if (std::fabs(q) < tiny) q = q < 0.0 ? -tiny : tiny;
    q = (a[i] - x) - b[i - 1] * b[i - 1] / q;
    if (q < 0.0) ++c;
  }
  return c;
}

inline bool tridiag_lowest_fast(int n, const double* a, const double* b, double* theta, double* ylast) {
  if (n == 1) {
    *theta = a[0];
    *ylast = 1.0;
    return true;
  }
  // Gershgorin interval
  double lo = a[0], hi = a[0], scale = 0.0;
  for (int i = 0; i < n; ++i) {
    const double r = (i > 0 ? std::fabs(b[i - 1]) : 0.0) + (i < n - 1 ? std::fabs(b[i]) : 0.0);
    lo = std::min(lo, a[i] - r);
    hi = std::max(hi, a[i] + r);
    scale = std::max(scale, std::fabs(a[i]) + r);
  }
  const double eps = 2.220446049250313e-16;
  const double tiny = std::max(1e-300, scale * eps * eps);
  // invariant: count(lo) == 0, count(hi) >= 1
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (!(mid > lo && mid < hi) || hi - lo <= 2.0 * eps * std::max(std::fabs(lo), std::fabs(hi))) break;
    if (sturm_below(n, a, b, mid, tiny) >= 1)
      hi = mid;
    else
      lo = mid;
  }
  *theta = 0.5 * (lo + hi);
  // two steps of inverse iteration (T - theta) z_new = z, Gaussian elimination with partial
  // pivoting on the tridiagonal (the matrix is nearly singular: z grows in the eigenvector)
  std::vector<double> dl(n), d(n), du(n), du2(n), z(n, 1.0);
  std::vector<char> piv(n);
  for (int i = 0; i < n; ++i) d[i] = a[i] - *theta;
  for (int i = 0; i < n - 1; ++i) dl[i] = du[i] = b[i];
  // LU factorisation (dgttrf scheme)
  for (int i = 0; i < n - 1; ++i) {
    du2[i] = 0.0;
    if (std::fabs(d[i]) >= std::fabs(dl[i])) {
      piv[i] = 0;
      if (d[i] == 0.0) d[i] = tiny;
      const double f = dl[i] / d[i];
      dl[i] = f;
      d[i + 1] -= f * du[i];
    } else {
      piv[i] = 1;
      const double f = d[i] / dl[i];
      d[i] = dl[i];
      dl[i] = f;
      const double t = du[i];
      du[i] = d[i + 1];
      d[i + 1] = t - f * d[i + 1];
      if (i < n - 2) {
        du2[i] = du[i + 1];
        du[i + 1] = -f * du[i + 1];
      }
    }
  }
  if (d[n - 1] == 0.0) d[n - 1] = tiny;
  for (int rep = 0; rep < 2; ++rep) {
    // solve L U z_new = P z
    for (int i = 0; i < n - 1; ++i) {
      if (piv[i]) std::swap(z[i], z[i + 1]);
      z[i + 1] -= dl[i] * z[i];
    }
    z[n - 1] /= d[n - 1];
    if (n > 1) z[n - 2] = (z[n - 2] - du[n - 2] * z[n - 1]) / d[n - 2];
    for (int i = n - 3; i >= 0; --i) z[i] = (z[i] - du[i] * z[i + 1] - du2[i] * z[i + 2]) / d[i];
    double nrm = 0.0;
    for (int i = 0; i < n; ++i) nrm = std::max(nrm, std::fabs(z[i]));
    if (!(nrm > 0.0) || !std::isfinite(nrm)) return false;
    for (int i = 0; i < n; ++i) z[i] /= nrm;
  }
  double s2 = 0.0;
  for (int i = 0; i < n; ++i) s2 += z[i] * z[i];
  *ylast = z[n - 1] / std::sqrt(s2);
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
