/*
 * heff_oracle.c -- CPU ORACLE for the two-site DMRG effective-Hamiltonian matvec and
 * its Lanczos ground-state solver.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with the CUDA path (paper_2007_14822_b200/csrc) and never
 * includes or links anything from it.
 *
 * Plain, slow, obviously correct: nested loops in fp64, no BLAS, no blocking, no
 * fusion.  FMA contraction by the compiler is allowed (reading R15); no
 * -ffast-math.  OpenMP is used only to split the outermost independent loop.
 *
 * What it computes (paper citations are lines of /root/reference/PAPER.md):
 *
 *  The paper's DMRG computes "dominant eigenvectors of very large Hermitian linear
 *  operators" (Sec. 6.2).  At a two-site window the operator is the
 *  effective Hamiltonian formed with the ITensor `*` product, which contracts all
 *  matching indices (Sec. 4), priming keeping the output legs apart
 *  (Sec. 2.6).  Written out with the leg names of BASELINE.json's
 *  north_star:
 *
 *    out[a',s1',s2',b'] = sum_{a,w,s1,w1,s2,w2,b}
 *          L[a',w,a] W1[w,s1',s1,w1] W2[w1,s2',s2,w2] R[b',w2,b] psi[a,s1,s2,b]      (D)
 *
 *  All arrays are dense, row-major (last index fastest), fp64 (`Dense{Float64}`,
 *  PAPER.md:583).  The output is returned un-primed in psi's layout.
 *
 *  ref_heff_direct   -- (D) literally, one 7-fold sum per output element.
 *  ref_heff_apply_A  -- (D) re-associated as the north_star's four steps
 *                       L*psi -> *W1 -> *W2 -> *R, for an a' range.  This is the
 *                       pairwise `*` contraction sequence of PAPER.md:363-375; no
 *                       reordering beyond the association itself.
 *  ref_heff_apply_B  -- the mirror association R*psi -> *W2 -> *W1 -> *L, for a b'
 *                       range (reading R17: the per-shard order).
 *  ref_lanczos       -- Lanczos with full (two-pass classical Gram-Schmidt)
 *                       reorthogonalisation, the textbook algorithm for the local
 *                       eigensolver (SPEC.md:756-764 gives pre/post only; DESIGN.md
 *                       readings R11-R14 fix reorthogonalisation, stop rule,
 *                       breakdown and sign).
 *  ref_tridiag_lowest -- lowest eigenpair of the symmetric tridiagonal T_j by
 *                       Sturm-sequence bisection + inverse iteration.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  int64_t mL, d1, d2, mR, kL, kM, kR;
} oracle_dims;

void oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Row-major index helpers (explicit, so each access can be read against (D)). */
#define IDX3(i, j, k, J, K) ((((int64_t)(i)) * (J) + (j)) * (K) + (k))
#define IDX4(i, j, k, l, J, K, L_) (((((int64_t)(i)) * (J) + (j)) * (K) + (k)) * (L_) + (l))

/* (D) written out: for every output element, the full 7-fold sum.  O(m^4 d^4 k^3). */
void ref_heff_direct(const oracle_dims* D, const double* L, const double* W1, const double* W2,
                     const double* R, const double* psi, double* out) {
  const int64_t mL = D->mL, d1 = D->d1, d2 = D->d2, mR = D->mR, kL = D->kL, kM = D->kM, kR = D->kR;
#pragma omp parallel for schedule(static)
  for (int64_t ap = 0; ap < mL; ++ap)
    for (int64_t s1p = 0; s1p < d1; ++s1p)
      for (int64_t s2p = 0; s2p < d2; ++s2p)
        for (int64_t bp = 0; bp < mR; ++bp) {
          double acc = 0.0;
          for (int64_t a = 0; a < mL; ++a)
            for (int64_t w = 0; w < kL; ++w)
              for (int64_t s1 = 0; s1 < d1; ++s1)
                for (int64_t w1 = 0; w1 < kM; ++w1)
                  for (int64_t s2 = 0; s2 < d2; ++s2)
                    for (int64_t w2 = 0; w2 < kR; ++w2)
                      for (int64_t b = 0; b < mR; ++b)
                        acc += L[IDX3(ap, w, a, kL, mL)] * W1[IDX4(w, s1p, s1, w1, d1, d1, kM)] *
                               W2[IDX4(w1, s2p, s2, w2, d2, d2, kR)] * R[IDX3(bp, w2, b, kR, mR)] *
                               psi[IDX4(a, s1, s2, b, d1, d2, mR)];
          out[IDX4(ap, s1p, s2p, bp, d1, d2, mR)] = acc;
        }
}

/*
 * Order A (north_star: "L*psi -> *W1 -> *W2 -> *R"), rows a' in [a_lo, a_hi).
 * out_rows holds (a_hi-a_lo) rows of out, each [d1][d2][mR].
 *   T1[w,s1,s2,b]     = sum_a       L[a',w,a]          psi[a,s1,s2,b]
 *   T2[s1',w1,s2,b]   = sum_{w,s1}  W1[w,s1',s1,w1]    T1[w,s1,s2,b]
 *   T3[s1',s2',w2,b]  = sum_{w1,s2} W2[w1,s2',s2,w2]   T2[s1',w1,s2,b]
 *   out[a',s1',s2',b']= sum_{w2,b}  T3[s1',s2',w2,b]   R[b',w2,b]
 */
int ref_heff_apply_A(const oracle_dims* D, const double* L, const double* W1, const double* W2,
                     const double* R, const double* psi, int64_t a_lo, int64_t a_hi, double* out_rows) {
  const int64_t mL = D->mL, d1 = D->d1, d2 = D->d2, mR = D->mR, kL = D->kL, kM = D->kM, kR = D->kR;
  if (a_lo < 0 || a_hi > mL || a_lo > a_hi) return -1;
  int err = 0;
#pragma omp parallel
  {
    double* T1 = (double*)malloc(sizeof(double) * kL * d1 * d2 * mR);
    double* T2 = (double*)malloc(sizeof(double) * d1 * kM * d2 * mR);
    double* T3 = (double*)malloc(sizeof(double) * d1 * d2 * kR * mR);
    if (!T1 || !T2 || !T3) {
#pragma omp atomic write
      err = -2;
    } else {
#pragma omp for schedule(dynamic, 1)
      for (int64_t ap = a_lo; ap < a_hi; ++ap) {
        /* step 1: T1 = L[a',:,:] * psi */
        memset(T1, 0, sizeof(double) * kL * d1 * d2 * mR);
        for (int64_t w = 0; w < kL; ++w)
          for (int64_t a = 0; a < mL; ++a) {
            const double l = L[IDX3(ap, w, a, kL, mL)];
            double* t = T1 + w * d1 * d2 * mR;
            const double* p = psi + a * d1 * d2 * mR;
            for (int64_t x = 0; x < d1 * d2 * mR; ++x) t[x] += l * p[x]; /* x = (s1,s2,b) */
          }
        /* step 2: T2 = W1 * T1 */
        memset(T2, 0, sizeof(double) * d1 * kM * d2 * mR);
        for (int64_t s1p = 0; s1p < d1; ++s1p)
          for (int64_t w1 = 0; w1 < kM; ++w1)
            for (int64_t w = 0; w < kL; ++w)
              for (int64_t s1 = 0; s1 < d1; ++s1) {
                const double c = W1[IDX4(w, s1p, s1, w1, d1, d1, kM)];
                double* t2 = T2 + IDX3(s1p, w1, 0, kM, d2 * mR);
                const double* t1 = T1 + IDX3(w, s1, 0, d1, d2 * mR);
                for (int64_t x = 0; x < d2 * mR; ++x) t2[x] += c * t1[x]; /* x = (s2,b) */
              }
        /* step 3: T3 = W2 * T2 */
        memset(T3, 0, sizeof(double) * d1 * d2 * kR * mR);
        for (int64_t s1p = 0; s1p < d1; ++s1p)
          for (int64_t s2p = 0; s2p < d2; ++s2p)
            for (int64_t w2 = 0; w2 < kR; ++w2)
              for (int64_t w1 = 0; w1 < kM; ++w1)
                for (int64_t s2 = 0; s2 < d2; ++s2) {
                  const double c = W2[IDX4(w1, s2p, s2, w2, d2, d2, kR)];
                  double* t3 = T3 + IDX4(s1p, s2p, w2, 0, d2, kR, mR);
                  const double* t2 = T2 + IDX4(s1p, w1, s2, 0, kM, d2, mR);
                  for (int64_t b = 0; b < mR; ++b) t3[b] += c * t2[b];
                }
        /* step 4: out = T3 * R^T over (w2,b) */
        double* o = out_rows + (ap - a_lo) * d1 * d2 * mR;
        for (int64_t s = 0; s < d1 * d2; ++s) /* s = (s1',s2') */
          for (int64_t bp = 0; bp < mR; ++bp) {
            double acc = 0.0;
            const double* t3 = T3 + s * kR * mR;
            const double* r = R + bp * kR * mR;
            for (int64_t x = 0; x < kR * mR; ++x) acc += t3[x] * r[x]; /* x = (w2,b) */
            o[s * mR + bp] = acc;
          }
      }
    }
    free(T1);
    free(T2);
    free(T3);
  }
  return err;
}

/*
 * Order B (R*psi -> *W2 -> *W1 -> *L), columns b' in [b_lo, b_hi).  out_cols is laid
 * out as the b'-shard [mL][d1][d2][b_hi-b_lo].
 *   V1[a,s1,s2,w2]   = sum_b       psi[a,s1,s2,b]   R[b',w2,b]
 *   V2[a,s1,w1,s2']  = sum_{s2,w2} W2[w1,s2',s2,w2] V1[a,s1,s2,w2]
 *   V3[w,a,s1',s2']  = sum_{s1,w1} W1[w,s1',s1,w1] V2[a,s1,w1,s2']
 *   out[a',s1',s2',b'] = sum_{w,a} L[a',w,a]        V3[w,a,s1',s2']
 */
int ref_heff_apply_B(const oracle_dims* D, const double* L, const double* W1, const double* W2,
                     const double* R, const double* psi, int64_t b_lo, int64_t b_hi, double* out_cols) {
  const int64_t mL = D->mL, d1 = D->d1, d2 = D->d2, mR = D->mR, kL = D->kL, kM = D->kM, kR = D->kR;
  const int64_t nb = b_hi - b_lo;
  if (b_lo < 0 || b_hi > mR || b_lo > b_hi) return -1;
  int err = 0;
#pragma omp parallel
  {
    double* V1 = (double*)malloc(sizeof(double) * mL * d1 * d2 * kR);
    double* V2 = (double*)malloc(sizeof(double) * mL * d1 * kM * d2);
    double* V3 = (double*)malloc(sizeof(double) * kL * mL * d1 * d2);
    if (!V1 || !V2 || !V3) {
#pragma omp atomic write
      err = -2;
    } else {
#pragma omp for schedule(dynamic, 1)
      for (int64_t bp = b_lo; bp < b_hi; ++bp) {
        for (int64_t x = 0; x < mL * d1 * d2; ++x) /* x = (a,s1,s2) */
          for (int64_t w2 = 0; w2 < kR; ++w2) {
            double acc = 0.0;
            const double* p = psi + x * mR;
            const double* r = R + IDX3(bp, w2, 0, kR, mR);
            for (int64_t b = 0; b < mR; ++b) acc += p[b] * r[b];
            V1[x * kR + w2] = acc;
          }
        memset(V2, 0, sizeof(double) * mL * d1 * kM * d2);
        for (int64_t a = 0; a < mL; ++a)
          for (int64_t s1 = 0; s1 < d1; ++s1)
            for (int64_t w1 = 0; w1 < kM; ++w1)
              for (int64_t s2p = 0; s2p < d2; ++s2p) {
                double acc = 0.0;
                for (int64_t s2 = 0; s2 < d2; ++s2)
                  for (int64_t w2 = 0; w2 < kR; ++w2)
                    acc += W2[IDX4(w1, s2p, s2, w2, d2, d2, kR)] * V1[IDX4(a, s1, s2, w2, d1, d2, kR)];
                V2[IDX4(a, s1, w1, s2p, d1, kM, d2)] = acc;
              }
        for (int64_t w = 0; w < kL; ++w)
          for (int64_t a = 0; a < mL; ++a)
            for (int64_t s1p = 0; s1p < d1; ++s1p)
              for (int64_t s2p = 0; s2p < d2; ++s2p) {
                double acc = 0.0;
                for (int64_t s1 = 0; s1 < d1; ++s1)
                  for (int64_t w1 = 0; w1 < kM; ++w1)
                    acc += W1[IDX4(w, s1p, s1, w1, d1, d1, kM)] * V2[IDX4(a, s1, w1, s2p, d1, kM, d2)];
                V3[IDX4(w, a, s1p, s2p, mL, d1, d2)] = acc;
              }
        for (int64_t ap = 0; ap < mL; ++ap)
          for (int64_t s = 0; s < d1 * d2; ++s) { /* s = (s1',s2') */
            double acc = 0.0;
            for (int64_t w = 0; w < kL; ++w)
              for (int64_t a = 0; a < mL; ++a)
                acc += L[IDX3(ap, w, a, kL, mL)] * V3[IDX3(w, a, s, mL, d1 * d2)];
            out_cols[(ap * d1 * d2 + s) * nb + (bp - b_lo)] = acc;
          }
      }
    }
    free(V1);
    free(V2);
    free(V3);
  }
  return err;
}

/* ---------------------------------------------------------------------------------
 * Symmetric tridiagonal T (diagonal alpha[0..j), off-diagonal beta[0..j-1)).
 * Lowest eigenvalue by Sturm-sequence bisection; eigenvector by inverse iteration
 * with a partially pivoted tridiagonal LU.  (Textbook; reading R14 fixes
 * the sign: the largest-magnitude component of y is made positive.)
 * ------------------------------------------------------------------------------- */

/* number of eigenvalues of T strictly below x (Sturm count via the LDL^T pivots) */
static int sturm_count(int j, const double* alpha, const double* beta, double x) {
  int cnt = 0;
  double d = 1.0;
  for (int i = 0; i < j; ++i) {
    const double b2 = (i > 0) ? beta[i - 1] * beta[i - 1] : 0.0;
    d = alpha[i] - x - ((i > 0) ? b2 / d : 0.0);
    if (d == 0.0) d = -1e-300; /* x is an eigenvalue of a leading block: count it as below */
    if (d < 0.0) ++cnt;
  }
  return cnt;
}

/* solve (T - sigma I) y = rhs in place by Gaussian elimination with partial pivoting */
static void tridiag_shift_solve(int j, const double* alpha, const double* beta, double sigma, double* y) {
  /* rows i: sub c[i-1], diag dd[i], super e[i], second super f[i] (fill-in from pivoting) */
  double* dd = (double*)malloc(sizeof(double) * j);
  double* e = (double*)malloc(sizeof(double) * j);
  double* f = (double*)malloc(sizeof(double) * j);
  double* c = (double*)malloc(sizeof(double) * j);
  for (int i = 0; i < j; ++i) {
    dd[i] = alpha[i] - sigma;
    e[i] = (i + 1 < j) ? beta[i] : 0.0;
    c[i] = (i + 1 < j) ? beta[i] : 0.0; /* c[i] = T[i+1][i] */
    f[i] = 0.0;
  }
  double tiny = 0.0;
  for (int i = 0; i < j; ++i) tiny = fmax(tiny, fabs(alpha[i]) + ((i + 1 < j) ? fabs(beta[i]) : 0.0));
  tiny = (tiny > 0.0 ? tiny : 1.0) * 1e-20; /* relative guard for an exactly singular pivot */
  for (int i = 0; i + 1 < j; ++i) {
    /* rows i and i+1; row i: [dd[i], e[i], f[i]] at cols i,i+1,i+2; row i+1: [c[i], dd[i+1], e[i+1]] */
    if (fabs(c[i]) > fabs(dd[i])) { /* swap rows i and i+1 */
      double t;
      t = dd[i]; dd[i] = c[i]; c[i] = t;
      t = e[i]; e[i] = dd[i + 1]; dd[i + 1] = t;
      t = f[i]; f[i] = e[i + 1]; e[i + 1] = t;
      t = y[i]; y[i] = y[i + 1]; y[i + 1] = t;
    }
    if (dd[i] == 0.0) dd[i] = tiny;
    const double l = c[i] / dd[i];
    dd[i + 1] -= l * e[i];
    e[i + 1] -= l * f[i];
    y[i + 1] -= l * y[i];
    c[i] = 0.0;
  }
  if (dd[j - 1] == 0.0) dd[j - 1] = tiny;
  for (int i = j - 1; i >= 0; --i) {
    double s = y[i];
    if (i + 1 < j) s -= e[i] * y[i + 1];
    if (i + 2 < j) s -= f[i] * y[i + 2];
    y[i] = s / dd[i];
  }
  free(dd); free(e); free(f); free(c);
}

int ref_tridiag_lowest(int j, const double* alpha, const double* beta, double* theta, double* y) {
  if (j <= 0) return -1;
  /* Gershgorin interval */
  double lo = 0.0, hi = 0.0;
  for (int i = 0; i < j; ++i) {
    const double r = ((i > 0) ? fabs(beta[i - 1]) : 0.0) + ((i + 1 < j) ? fabs(beta[i]) : 0.0);
    const double a = alpha[i] - r, b = alpha[i] + r;
    if (i == 0 || a < lo) lo = a;
    if (i == 0 || b > hi) hi = b;
  }
  /* bisection for the smallest x with count(x) >= 1 */
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (sturm_count(j, alpha, beta, mid) >= 1) hi = mid; else lo = mid;
  }
  const double th = 0.5 * (lo + hi);
  *theta = th;
  if (y) {
    double scale = 0.0;
    for (int i = 0; i < j; ++i) scale = fmax(scale, fabs(alpha[i]) + ((i + 1 < j) ? fabs(beta[i]) : 0.0));
    if (scale == 0.0) scale = 1.0;
    const double sigma = th - 4.0 * 2.220446049250313e-16 * scale; /* just below theta */
    for (int i = 0; i < j; ++i) y[i] = 1.0 / sqrt((double)j);
    for (int rep = 0; rep < 3; ++rep) {
      tridiag_shift_solve(j, alpha, beta, sigma, y);
      double n2 = 0.0;
      for (int i = 0; i < j; ++i) n2 += y[i] * y[i];
      const double inv = 1.0 / sqrt(n2);
      for (int i = 0; i < j; ++i) y[i] *= inv;
    }
    int imax = 0;
    for (int i = 1; i < j; ++i) if (fabs(y[i]) > fabs(y[imax])) imax = i;
    if (y[imax] < 0.0)
      for (int i = 0; i < j; ++i) y[i] = -y[i];
  }
  return 0;
}

/* ---------------------------------------------------------------------------------
 * Lanczos with full reorthogonalisation (textbook order).
 *   v_1 = x0/||x0||                      (error -5 if ||x0|| = 0)
 *   for j = 1..:
 *     w = H v_j ; alpha_j = v_j . w ; w -= alpha_j v_j + beta_{j-1} v_{j-1}
 *     two passes of  w -= V_j (V_j^T w)   (CGS2, reading R11)
 *     beta_j = ||w|| ; theta_j, y_j = lowest eigenpair of T_j
 *     hnorm_j = max_i (|alpha_i| + beta_{i-1} + beta_i)   (||H|| estimate)
 *     breakdown: beta_j <= 1e-12 hnorm_j  -> stop (reading R13)
 *     mode 0 (fixed steps): stop at j = max_iter
 *     mode 1 (converge):    stop when beta_j |y_j[j]| <= tol hnorm_j, or j = max_iter (R12)
 *     v_{j+1} = w / beta_j
 *   x = V_j y_j / ||V_j y_j||
 * matvec(ctx, in, out) computes out = H in for vectors of length n.
 * ------------------------------------------------------------------------------- */
typedef void (*oracle_matvec_fn)(void* ctx, const double* in, double* out);

static double dotp(int64_t n, const double* x, const double* y) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += x[i] * y[i];
  return s;
}

int ref_lanczos(oracle_matvec_fn matvec, void* ctx, int64_t n, const double* x0, int max_iter, double tol,
                int mode, double* energy, double* x_out, int* iters_done, double* alpha_out, double* beta_out,
                double* theta_hist) {
  if (n <= 0 || max_iter <= 0) return -1;
  double nrm = sqrt(dotp(n, x0, x0));
  if (!(nrm > 0.0)) return -5;
  double* V = (double*)malloc(sizeof(double) * n * (size_t)(max_iter + 1));
  double* w = (double*)malloc(sizeof(double) * n);
  double* alpha = (double*)calloc(max_iter + 1, sizeof(double));
  double* beta = (double*)calloc(max_iter + 1, sizeof(double));
  double* y = (double*)calloc(max_iter + 1, sizeof(double));
  double* c = (double*)calloc(max_iter + 1, sizeof(double));
  if (!V || !w || !alpha || !beta || !y || !c) {
    free(V); free(w); free(alpha); free(beta); free(y); free(c);
    return -2;
  }
  for (int64_t i = 0; i < n; ++i) V[i] = x0[i] / nrm;
  double hnorm = 0.0, theta = 0.0;
  int j = 0;
  for (j = 1; j <= max_iter; ++j) {
    const double* vj = V + (int64_t)(j - 1) * n;
    matvec(ctx, vj, w);
    alpha[j - 1] = dotp(n, vj, w);
    for (int64_t i = 0; i < n; ++i) w[i] -= alpha[j - 1] * vj[i];
    if (j > 1) {
      const double* vjm = V + (int64_t)(j - 2) * n;
      for (int64_t i = 0; i < n; ++i) w[i] -= beta[j - 2] * vjm[i];
    }
    for (int pass = 0; pass < 2; ++pass) {
      for (int q = 0; q < j; ++q) c[q] = dotp(n, V + (int64_t)q * n, w);
      for (int q = 0; q < j; ++q) {
        const double* vq = V + (int64_t)q * n;
        for (int64_t i = 0; i < n; ++i) w[i] -= c[q] * vq[i];
      }
    }
    beta[j - 1] = sqrt(dotp(n, w, w));
    ref_tridiag_lowest(j, alpha, beta, &theta, y);
    if (theta_hist) theta_hist[j - 1] = theta;
    for (int i = 0; i < j; ++i) {
      const double g = fabs(alpha[i]) + ((i > 0) ? beta[i - 1] : 0.0) + beta[i];
      if (g > hnorm) hnorm = g;
    }
    if (beta[j - 1] <= 1e-12 * hnorm) break;                       /* breakdown: invariant subspace */
    if (mode == 1 && beta[j - 1] * fabs(y[j - 1]) <= tol * hnorm) break; /* converged */
    if (j == max_iter) break;
    double* vn = V + (int64_t)j * n;
    for (int64_t i = 0; i < n; ++i) vn[i] = w[i] / beta[j - 1];
  }
  if (j > max_iter) j = max_iter;
  /* Ritz vector */
  if (x_out) {
    for (int64_t i = 0; i < n; ++i) x_out[i] = 0.0;
    for (int q = 0; q < j; ++q) {
      const double* vq = V + (int64_t)q * n;
      for (int64_t i = 0; i < n; ++i) x_out[i] += y[q] * vq[i];
    }
    double xn = sqrt(dotp(n, x_out, x_out));
    for (int64_t i = 0; i < n; ++i) x_out[i] /= xn;
  }
  *energy = theta;
  *iters_done = j;
  if (alpha_out) memcpy(alpha_out, alpha, sizeof(double) * j);
  if (beta_out) memcpy(beta_out, beta, sizeof(double) * j);
  free(V); free(w); free(alpha); free(beta); free(y); free(c);
  return 0;
}

/* matvec adaptor: H = H_eff (order A over all rows) for use with ref_lanczos */
typedef struct {
  oracle_dims dims;
  const double *L, *W1, *W2, *R;
} oracle_heff_ctx;

void oracle_heff_matvec(void* vctx, const double* in, double* out) {
  oracle_heff_ctx* c = (oracle_heff_ctx*)vctx;
  ref_heff_apply_A(&c->dims, c->L, c->W1, c->W2, c->R, in, 0, c->dims.mL, out);
}

int ref_lanczos_heff(const oracle_dims* D, const double* L, const double* W1, const double* W2,
                     const double* R, const double* x0, int max_iter, double tol, int mode, double* energy,
                     double* x_out, int* iters_done, double* alpha_out, double* beta_out, double* theta_hist) {
  oracle_heff_ctx c;
  c.dims = *D;
  c.L = L; c.W1 = W1; c.W2 = W2; c.R = R;
  const int64_t n = D->mL * D->d1 * D->d2 * D->mR;
  return ref_lanczos(oracle_heff_matvec, &c, n, x0, max_iter, tol, mode, energy, x_out, iters_done, alpha_out,
                     beta_out, theta_hist);
}

/* ---------------------------------------------------------------------------------
 * Environment update.  SPEC's ProjMPO keeps "L[j] equals
 * contraction of psi-dag.H.psi over sites 1..j" (projmpo_position
 * S:747-755); DMRG moves it one site per bond step (Sec. 6.2):
 *   Lout[a',w',a] = sum_{x',s',w,s,x} A[x',s',a'] L[x',w,x] W[w,s',s,w'] A[x,s,a]
 *   Rout[b',w,b]  = sum_{y',s',w',s,y} B[b',s',y'] R[y',w',y] W[w,s',s,w'] B[b,s,y]
 * evaluated as the pairwise `*` chain L*A -> *W -> *A-dagger (and mirrored for R).
 * Shapes: L [mi][kl][mi], A [mi][d][mo], W [kl][d][d][kr] -> Lout [mo][kr][mo];
 *         R [mi][kr][mi], B [mo][d][mi], W [kl][d][d][kr] -> Rout [mo][kl][mo].
 * ------------------------------------------------------------------------------- */
int ref_env_left(int64_t mi, int64_t d, int64_t mo, int64_t kl, int64_t kr, const double* L, const double* A,
                 const double* W, double* Lout) {
  double* X = (double*)calloc((size_t)(mi * kl * d * mo), sizeof(double)); /* [x'][w][s][a]  */
  double* Y = (double*)calloc((size_t)(mi * d * kr * mo), sizeof(double)); /* [x'][s'][w'][a] */
  if (!X || !Y) { free(X); free(Y); return -2; }
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t xp = 0; xp < mi; ++xp) {
    for (int64_t w = 0; w < kl; ++w)
      for (int64_t x = 0; x < mi; ++x) {
        const double l = L[IDX3(xp, w, x, kl, mi)];
        double* xr = X + IDX3(xp, w, 0, kl, d * mo);
        const double* ar = A + x * d * mo;
        for (int64_t sa = 0; sa < d * mo; ++sa) xr[sa] += l * ar[sa]; /* sa = (s,a) */
      }
    for (int64_t sp = 0; sp < d; ++sp)
      for (int64_t wp = 0; wp < kr; ++wp)
        for (int64_t w = 0; w < kl; ++w)
          for (int64_t s = 0; s < d; ++s) {
            const double c = W[IDX4(w, sp, s, wp, d, d, kr)];
            double* yr = Y + IDX4(xp, sp, wp, 0, d, kr, mo);
            const double* xr = X + IDX4(xp, w, s, 0, kl, d, mo);
            for (int64_t a = 0; a < mo; ++a) yr[a] += c * xr[a];
          }
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t ap = 0; ap < mo; ++ap)
    for (int64_t wp = 0; wp < kr; ++wp) {
      double* o = Lout + IDX3(ap, wp, 0, kr, mo);
      for (int64_t a = 0; a < mo; ++a) o[a] = 0.0;
      for (int64_t xp = 0; xp < mi; ++xp)
        for (int64_t sp = 0; sp < d; ++sp) {
          const double c = A[IDX3(xp, sp, ap, d, mo)];
          const double* yr = Y + IDX4(xp, sp, wp, 0, d, kr, mo);
          for (int64_t a = 0; a < mo; ++a) o[a] += c * yr[a];
        }
    }
  free(X);
  free(Y);
  return 0;
}

int ref_env_right(int64_t mi, int64_t d, int64_t mo, int64_t kl, int64_t kr, const double* R, const double* B,
                  const double* W, double* Rout) {
  double* X = (double*)calloc((size_t)(mo * d * kr * mi), sizeof(double)); /* [b'][s'][w'][y] */
  double* Y = (double*)calloc((size_t)(mo * kl * d * mi), sizeof(double)); /* [b'][w][s][y]   */
  if (!X || !Y) { free(X); free(Y); return -2; }
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t bp = 0; bp < mo; ++bp) {
    for (int64_t sp = 0; sp < d; ++sp)
      for (int64_t yp = 0; yp < mi; ++yp) {
        const double b = B[IDX3(bp, sp, yp, d, mi)];
        double* xr = X + IDX3(bp, sp, 0, d, kr * mi);
        const double* rr = R + yp * kr * mi;
        for (int64_t wy = 0; wy < kr * mi; ++wy) xr[wy] += b * rr[wy]; /* wy = (w',y) */
      }
    for (int64_t w = 0; w < kl; ++w)
      for (int64_t s = 0; s < d; ++s)
        for (int64_t sp = 0; sp < d; ++sp)
          for (int64_t wp = 0; wp < kr; ++wp) {
            const double c = W[IDX4(w, sp, s, wp, d, d, kr)];
            double* yr = Y + IDX4(bp, w, s, 0, kl, d, mi);
            const double* xr = X + IDX4(bp, sp, wp, 0, d, kr, mi);
            for (int64_t y = 0; y < mi; ++y) yr[y] += c * xr[y];
          }
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t bp = 0; bp < mo; ++bp)
    for (int64_t w = 0; w < kl; ++w)
      for (int64_t b = 0; b < mo; ++b) {
        double acc = 0.0;
        const double* yr = Y + IDX3(bp, w, 0, kl, d * mi);
        const double* br = B + b * d * mi;
        for (int64_t sy = 0; sy < d * mi; ++sy) acc += yr[sy] * br[sy]; /* sy = (s,y) */
        Rout[IDX3(bp, w, b, kl, mo)] = acc;
      }
  free(X);
  free(Y);
  return 0;
}

/* ---------------------------------------------------------------------------------
 * Complex variant (ITensor's Dense{ComplexF64} storage and zgemm,
 * PAPER.md:583).  (D) is unchanged -- no conjugation inside the
 * contraction; Hermiticity comes from environments built with the bra tensors
 * conjugated.  Arrays are interleaved complex (double _Complex).  Order A, a' range.
 * ------------------------------------------------------------------------------- */
#include <complex.h>

int ref_heff_apply_A_z(const oracle_dims* D, const double _Complex* L, const double _Complex* W1,
                       const double _Complex* W2, const double _Complex* R, const double _Complex* psi, int64_t a_lo,
                       int64_t a_hi, double _Complex* out_rows) {
  const int64_t mL = D->mL, d1 = D->d1, d2 = D->d2, mR = D->mR, kL = D->kL, kM = D->kM, kR = D->kR;
  if (a_lo < 0 || a_hi > mL || a_lo > a_hi) return -1;
  int err = 0;
#pragma omp parallel
  {
    double _Complex* T1 = (double _Complex*)malloc(sizeof(double _Complex) * kL * d1 * d2 * mR);
    double _Complex* T2 = (double _Complex*)malloc(sizeof(double _Complex) * d1 * kM * d2 * mR);
    double _Complex* T3 = (double _Complex*)malloc(sizeof(double _Complex) * d1 * d2 * kR * mR);
    if (!T1 || !T2 || !T3) {
#pragma omp atomic write
      err = -2;
    } else {
#pragma omp for schedule(dynamic, 1)
      for (int64_t ap = a_lo; ap < a_hi; ++ap) {
        for (int64_t x = 0; x < kL * d1 * d2 * mR; ++x) T1[x] = 0;
        for (int64_t w = 0; w < kL; ++w)
          for (int64_t a = 0; a < mL; ++a) {
            const double _Complex l = L[IDX3(ap, w, a, kL, mL)];
            double _Complex* t = T1 + w * d1 * d2 * mR;
            const double _Complex* p = psi + a * d1 * d2 * mR;
            for (int64_t x = 0; x < d1 * d2 * mR; ++x) t[x] += l * p[x];
          }
        for (int64_t x = 0; x < d1 * kM * d2 * mR; ++x) T2[x] = 0;
        for (int64_t s1p = 0; s1p < d1; ++s1p)
          for (int64_t w1 = 0; w1 < kM; ++w1)
            for (int64_t w = 0; w < kL; ++w)
              for (int64_t s1 = 0; s1 < d1; ++s1) {
                const double _Complex c = W1[IDX4(w, s1p, s1, w1, d1, d1, kM)];
                double _Complex* t2 = T2 + IDX3(s1p, w1, 0, kM, d2 * mR);
                const double _Complex* t1 = T1 + IDX3(w, s1, 0, d1, d2 * mR);
                for (int64_t x = 0; x < d2 * mR; ++x) t2[x] += c * t1[x];
              }
        for (int64_t x = 0; x < d1 * d2 * kR * mR; ++x) T3[x] = 0;
        for (int64_t s1p = 0; s1p < d1; ++s1p)
          for (int64_t s2p = 0; s2p < d2; ++s2p)
            for (int64_t w2 = 0; w2 < kR; ++w2)
              for (int64_t w1 = 0; w1 < kM; ++w1)
                for (int64_t s2 = 0; s2 < d2; ++s2) {
                  const double _Complex c = W2[IDX4(w1, s2p, s2, w2, d2, d2, kR)];
                  double _Complex* t3 = T3 + IDX4(s1p, s2p, w2, 0, d2, kR, mR);
                  const double _Complex* t2 = T2 + IDX4(s1p, w1, s2, 0, kM, d2, mR);
                  for (int64_t b = 0; b < mR; ++b) t3[b] += c * t2[b];
                }
        double _Complex* o = out_rows + (ap - a_lo) * d1 * d2 * mR;
        for (int64_t s = 0; s < d1 * d2; ++s)
          for (int64_t bp = 0; bp < mR; ++bp) {
            double _Complex acc = 0;
            const double _Complex* t3 = T3 + s * kR * mR;
            const double _Complex* r = R + bp * kR * mR;
            for (int64_t x = 0; x < kR * mR; ++x) acc += t3[x] * r[x];
            o[s * mR + bp] = acc;
          }
      }
    }
    free(T1);
    free(T2);
    free(T3);
  }
  return err;
}

/* Hermitian Lanczos with CGS2 (same readings as ref_lanczos; <v,w> = sum conj(v) w).
 * matvec(ctx, in, out) on interleaved complex vectors of n complex entries. */
typedef void (*oracle_zmatvec_fn)(void* ctx, const double _Complex* in, double _Complex* out);

static double _Complex zdotc(int64_t n, const double _Complex* x, const double _Complex* y) {
  double _Complex s = 0;
  for (int64_t i = 0; i < n; ++i) s += conj(x[i]) * y[i];
  return s;
}

int ref_lanczos_z(oracle_zmatvec_fn matvec, void* ctx, int64_t n, const double _Complex* x0, int max_iter, double tol,
                  int mode, double* energy, double _Complex* x_out, int* iters_done, double* alpha_out,
                  double* beta_out, double* theta_hist) {
  if (n <= 0 || max_iter <= 0) return -1;
  double nrm = sqrt(creal(zdotc(n, x0, x0)));
  if (!(nrm > 0.0)) return -5;
  double _Complex* V = (double _Complex*)malloc(sizeof(double _Complex) * n * (size_t)(max_iter + 1));
  double _Complex* w = (double _Complex*)malloc(sizeof(double _Complex) * n);
  double* alpha = (double*)calloc(max_iter + 1, sizeof(double));
  double* beta = (double*)calloc(max_iter + 1, sizeof(double));
  double* y = (double*)calloc(max_iter + 1, sizeof(double));
  double _Complex* c = (double _Complex*)calloc(max_iter + 1, sizeof(double _Complex));
  if (!V || !w || !alpha || !beta || !y || !c) {
    free(V); free(w); free(alpha); free(beta); free(y); free(c);
    return -2;
  }
  for (int64_t i = 0; i < n; ++i) V[i] = x0[i] / nrm;
  double hnorm = 0.0, theta = 0.0;
  int j = 0;
  for (j = 1; j <= max_iter; ++j) {
    const double _Complex* vj = V + (int64_t)(j - 1) * n;
    matvec(ctx, vj, w);
    alpha[j - 1] = creal(zdotc(n, vj, w));
    for (int64_t i = 0; i < n; ++i) w[i] -= alpha[j - 1] * vj[i];
    if (j > 1) {
      const double _Complex* vjm = V + (int64_t)(j - 2) * n;
      for (int64_t i = 0; i < n; ++i) w[i] -= beta[j - 2] * vjm[i];
    }
    for (int pass = 0; pass < 2; ++pass) {
      for (int q = 0; q < j; ++q) c[q] = zdotc(n, V + (int64_t)q * n, w);
      for (int q = 0; q < j; ++q) {
        const double _Complex* vq = V + (int64_t)q * n;
        for (int64_t i = 0; i < n; ++i) w[i] -= c[q] * vq[i];
      }
    }
    beta[j - 1] = sqrt(creal(zdotc(n, w, w)));
    ref_tridiag_lowest(j, alpha, beta, &theta, y);
    if (theta_hist) theta_hist[j - 1] = theta;
    for (int i = 0; i < j; ++i) {
      const double g = fabs(alpha[i]) + ((i > 0) ? beta[i - 1] : 0.0) + beta[i];
      if (g > hnorm) hnorm = g;
    }
    if (beta[j - 1] <= 1e-12 * hnorm) break;
    if (mode == 1 && beta[j - 1] * fabs(y[j - 1]) <= tol * hnorm) break;
    if (j == max_iter) break;
    double _Complex* vn = V + (int64_t)j * n;
    for (int64_t i = 0; i < n; ++i) vn[i] = w[i] / beta[j - 1];
  }
  if (j > max_iter) j = max_iter;
  if (x_out) {
    for (int64_t i = 0; i < n; ++i) x_out[i] = 0;
    for (int q = 0; q < j; ++q) {
      const double _Complex* vq = V + (int64_t)q * n;
      for (int64_t i = 0; i < n; ++i) x_out[i] += y[q] * vq[i];
    }
    const double xn = sqrt(creal(zdotc(n, x_out, x_out)));
    for (int64_t i = 0; i < n; ++i) x_out[i] /= xn;
  }
  *energy = theta;
  *iters_done = j;
  if (alpha_out) memcpy(alpha_out, alpha, sizeof(double) * j);
  if (beta_out) memcpy(beta_out, beta, sizeof(double) * j);
  free(V); free(w); free(alpha); free(beta); free(y); free(c);
  return 0;
}

typedef struct {
  oracle_dims dims;
  const double _Complex *L, *W1, *W2, *R;
} oracle_heff_z_ctx;

void oracle_heff_matvec_z(void* vctx, const double _Complex* in, double _Complex* out) {
  oracle_heff_z_ctx* c = (oracle_heff_z_ctx*)vctx;
  ref_heff_apply_A_z(&c->dims, c->L, c->W1, c->W2, c->R, in, 0, c->dims.mL, out);
}

int ref_lanczos_heff_z(const oracle_dims* D, const double _Complex* L, const double _Complex* W1,
                       const double _Complex* W2, const double _Complex* R, const double _Complex* x0, int max_iter,
                       double tol, int mode, double* energy, double _Complex* x_out, int* iters_done,
                       double* alpha_out, double* beta_out, double* theta_hist) {
  oracle_heff_z_ctx c;
  c.dims = *D;
  c.L = L; c.W1 = W1; c.W2 = W2; c.R = R;
  const int64_t n = D->mL * D->d1 * D->d2 * D->mR;
  return ref_lanczos_z(oracle_heff_matvec_z, &c, n, x0, max_iter, tol, mode, energy, x_out, iters_done, alpha_out,
                       beta_out, theta_hist);
}
