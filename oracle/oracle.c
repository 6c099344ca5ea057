/* oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h). Plain loops, explicit re/im arithmetic,
 * fixed-order reductions. Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, R<k> = the
 * reading listed in DESIGN.md section 3. */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define RE(p, i) (p)[2 * (i)]
#define IM(p, i) (p)[2 * (i) + 1]

/* ------------------------------------------------------------------------------------------------ */
/* Chebyshev polynomials, eq:polydef and its sign rule for t < -1 (C_m(-t) = (-1)^m C_m(t)) */
long double ora_cheb(int32_t m, long double t) {
  if (m == 0) return 1.0L;
  if (t >= 1.0L) return coshl((long double)m * acoshl(t));
  if (t <= -1.0L) {
    long double v = coshl((long double)m * acoshl(-t));
    return (m % 2) ? -v : v;
  }
  return cosl((long double)m * acosl(t));
}

/* p_m(lam) = C_m(t)/C_m(t1), t = (lam-c)/e, t1 = (lambda1-c)/e */
long double ora_filter_gain(int32_t m, long double lam, long double lambda1, long double c,
                            long double e) {
  return ora_cheb(m, (lam - c) / e) / ora_cheb(m, (lambda1 - c) / e);
}

/* Alg 2 line 2 and line 6 */
void ora_sigma(int32_t mmax, double lambda1, double c, double e, double* sigma) {
  if (mmax < 1) return;
  sigma[0] = e / (lambda1 - c);
  for (int32_t i = 1; i < mmax; ++i) sigma[i] = 1.0 / (2.0 / sigma[0] - sigma[i - 1]);
}

/* ------------------------------------------------------------------------------------------------ */
/* (H~ Y)[:, j] = (H y_j - c y_j)/e for the columns j0..j1-1 of a block, naive loops. For
 * Hermitian H, (H y)[r] = sum_q conj(H[q,r]) y[q] (R13): row r of H is the conjugate of the
 * contiguous column r, so the loop runs down column r once and reuses it for every column of y. */
static void hshift_block(int64_t n, const double* H, int64_t ldh, const double* Y, int64_t ldy,
                         int64_t j0, int64_t j1, double c, double e, double* out, int64_t ldo) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) {
    const double* h = H + 2 * r * ldh;
    for (int64_t j = j0; j < j1; ++j) {
      const double* y = Y + 2 * j * ldy;
      double sr = 0.0, si = 0.0;
      for (int64_t q = 0; q < n; ++q) {
        double hr = h[2 * q], hi = -h[2 * q + 1];
        sr += hr * y[2 * q] - hi * y[2 * q + 1];
        si += hr * y[2 * q + 1] + hi * y[2 * q];
      }
      out[2 * (j * ldo + r)] = (sr - c * y[2 * r]) / e;
      out[2 * (j * ldo + r) + 1] = (si - c * y[2 * r + 1]) / e;
    }
  }
}

/* Algorithm 2, step by step, with readings R1 (Y_{i-1} in line 8), R2 (columns to k),
 * R3 (s = first column with m_j > i). The block is processed as Alg 2 states: all k columns at
 * i = 0 (lines 2-3), then for i = 1..m_k-1 only the columns s..k-1 (line 8), the columns before s
 * carried forward unchanged (line 7). */
int32_t ora_filter(int64_t n, const double* H, int64_t ldh, double* Y, int64_t ldy, int64_t k,
                   const int32_t* deg, double lambda1, double c, double e, int64_t* matvecs) {
  if (n < 1 || k < 0 || ldh < n || ldy < n || !(e > 0.0)) return 1;
  if (k == 0) return 0;
  for (int64_t j = 0; j < k; ++j) {
    if (deg[j] < 1) return 1;
    if (j > 0 && deg[j] < deg[j - 1]) return 1;
  }
  const int32_t mk = deg[k - 1];
  double* sigma = (double*)malloc(sizeof(double) * (size_t)(mk + 1));
  ora_sigma(mk, lambda1, c, e, sigma);
  size_t blk = (size_t)2 * n * k;
  double* Yprev = (double*)malloc(sizeof(double) * blk); /* Y_{i-1} */
  double* Ycur = (double*)malloc(sizeof(double) * blk);  /* Y_i */
  double* Ynext = (double*)malloc(sizeof(double) * blk); /* Y_{i+1} */
  double* hy = (double*)malloc(sizeof(double) * blk); /* H~ Y_i */
  for (int64_t j = 0; j < k; ++j) memcpy(Yprev + 2 * j * n, Y + 2 * j * ldy, sizeof(double) * 2 * n);
  /* line 3: Y_1 = sigma_1 H~ Y_0 (all columns) */
  hshift_block(n, H, ldh, Yprev, n, 0, k, c, e, hy, n);
  for (int64_t j = 0; j < k; ++j)
    for (int64_t r = 0; r < n; ++r) {
      Ycur[2 * (j * n + r)] = sigma[0] * hy[2 * (j * n + r)];
      Ycur[2 * (j * n + r) + 1] = sigma[0] * hy[2 * (j * n + r) + 1];
    }
  int64_t mv = k;
  /* line 4: s = first column whose degree is not 1 */
  int64_t s = 0;
  while (s < k && deg[s] <= 1) ++s;
  for (int32_t i = 1; i <= mk - 1; ++i) {
    const double sig_next = sigma[i], sig_i = sigma[i - 1]; /* sigma_{i+1}, sigma_i */
    /* line 7: finished columns carried forward */
    for (int64_t j = 0; j < s; ++j) memcpy(Ynext + 2 * j * n, Ycur + 2 * j * n, sizeof(double) * 2 * n);
    /* line 8 (R1): Y_{i+1} = 2 sigma_{i+1} H~ Y_i - sigma_{i+1} sigma_i Y_{i-1} */
    hshift_block(n, H, ldh, Ycur, n, s, k, c, e, hy, n);
    for (int64_t j = s; j < k; ++j) {
      for (int64_t r = 0; r < n; ++r) {
        double a = 2.0 * sig_next, b = sig_next * sig_i;
        Ynext[2 * (j * n + r)] = a * hy[2 * (j * n + r)] - b * Yprev[2 * (j * n + r)];
        Ynext[2 * (j * n + r) + 1] = a * hy[2 * (j * n + r) + 1] - b * Yprev[2 * (j * n + r) + 1];
      }
      ++mv;
    }
    /* line 9: s <- first column whose degree is not i+1 (and beyond the finished ones) */
    while (s < k && deg[s] <= i + 1) ++s;
    double* t = Yprev;
    Yprev = Ycur;
    Ycur = Ynext;
    Ynext = t;
  }
  int32_t status = 0;
  for (int64_t j = 0; j < k; ++j)
    for (int64_t r = 0; r < 2 * n; ++r) {
      double v = Ycur[2 * j * n + r];
      if (!isfinite(v)) status = 2;
      Y[2 * j * ldy + r] = v;
    }
  if (matvecs) *matvecs += mv;
  free(sigma);
  free(Yprev);
  free(Ycur);
  free(Ynext);
  free(hy);
  return status;
}

/* App. A: column j after m_j steps equals p_{m_j}(H) y_j exactly; for diagonal H that is an
 * entrywise scaling by p_{m_j}(d_r), evaluated by eq:polydef in long double. */
void ora_filter_diag_closed(int64_t n, const double* d, double* Y, int64_t ldy, int64_t k,
                            const int32_t* deg, double lambda1, double c, double e) {
  for (int64_t j = 0; j < k; ++j)
    for (int64_t r = 0; r < n; ++r) {
      long double g = ora_filter_gain(deg[j], d[r], lambda1, c, e);
      Y[2 * (j * ldy + r)] = (double)(g * (long double)Y[2 * (j * ldy + r)]);
      Y[2 * (j * ldy + r) + 1] = (double)(g * (long double)Y[2 * (j * ldy + r) + 1]);
    }
}

/* Q = I - V T V^H. apply_Q(adj=0): x <- Q x; adj=1: x <- Q^H x = (I - V T^H V^H) x. */
static void apply_wy(int64_t n, const double* V, const double* T, int adj, double* x) {
  const int R = 8;
  double w[16], u[16];
  for (int a = 0; a < R; ++a) { /* w = V^H x */
    double sr = 0.0, si = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double vr = V[2 * (a * n + i)], vi = V[2 * (a * n + i) + 1];
      sr += vr * x[2 * i] + vi * x[2 * i + 1];
      si += vr * x[2 * i + 1] - vi * x[2 * i];
    }
    w[2 * a] = sr;
    w[2 * a + 1] = si;
  }
  for (int a = 0; a < R; ++a) { /* u = T w or T^H w */
    double sr = 0.0, si = 0.0;
    for (int b = 0; b < R; ++b) {
      double tr, ti;
      if (!adj) {
        tr = T[2 * (b * R + a)];
        ti = T[2 * (b * R + a) + 1];
      } else {
        tr = T[2 * (a * R + b)];
        ti = -T[2 * (a * R + b) + 1];
      }
      sr += tr * w[2 * b] - ti * w[2 * b + 1];
      si += tr * w[2 * b + 1] + ti * w[2 * b];
    }
    u[2 * a] = sr;
    u[2 * a + 1] = si;
  }
  for (int64_t i = 0; i < n; ++i) { /* x -= V u */
    double sr = 0.0, si = 0.0;
    for (int a = 0; a < R; ++a) {
      double vr = V[2 * (a * n + i)], vi = V[2 * (a * n + i) + 1];
      sr += vr * u[2 * a] - vi * u[2 * a + 1];
      si += vr * u[2 * a + 1] + vi * u[2 * a];
    }
    x[2 * i] -= sr;
    x[2 * i + 1] -= si;
  }
}

void ora_filter_wy_closed(int64_t n, const double* lam, const double* V, const double* T,
                          double* Y, int64_t ldy, int64_t k, const int32_t* deg, double lambda1,
                          double c, double e) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t j = 0; j < k; ++j) {
    double* y = Y + 2 * j * ldy;
    apply_wy(n, V, T, 1, y); /* Q^H y */
    for (int64_t r = 0; r < n; ++r) {
      long double g = ora_filter_gain(deg[j], lam[r], lambda1, c, e);
      y[2 * r] = (double)(g * (long double)y[2 * r]);
      y[2 * r + 1] = (double)(g * (long double)y[2 * r + 1]);
    }
    apply_wy(n, V, T, 0, y); /* Q (...) */
  }
}

/* ------------------------------------------------------------------------------------------------ */
void ora_zgemm(char ta, char tb, int64_t m, int64_t n, int64_t kk, const double* A, int64_t lda,
               const double* B, int64_t ldb, double* C, int64_t ldc) {
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) {
      double sr = 0.0, si = 0.0;
      for (int64_t q = 0; q < kk; ++q) {
        double ar, ai, br, bi;
        if (ta == 'N') {
          ar = A[2 * (q * lda + i)];
          ai = A[2 * (q * lda + i) + 1];
        } else {
          ar = A[2 * (i * lda + q)];
          ai = -A[2 * (i * lda + q) + 1];
        }
        if (tb == 'N') {
          br = B[2 * (j * ldb + q)];
          bi = B[2 * (j * ldb + q) + 1];
        } else {
          br = B[2 * (q * ldb + j)];
          bi = -B[2 * (q * ldb + j) + 1];
        }
        sr += ar * br - ai * bi;
        si += ar * bi + ai * br;
      }
      C[2 * (j * ldc + i)] = sr;
      C[2 * (j * ldc + i) + 1] = si;
    }
}

/* Householder QR: reflector j maps x = A[j:n, j] to alpha e_1 with alpha = -(x_0/|x_0|) ||x||. */
int32_t ora_householder_qr(int64_t n, int64_t k, const double* A, int64_t lda, double* Q,
                           int64_t ldq, double* R, int64_t ldr) {
  double* W = (double*)malloc(sizeof(double) * 2 * (size_t)n * (size_t)k);
  double* vs = (double*)malloc(sizeof(double) * 2 * (size_t)n * (size_t)k); /* reflector vectors */
  double* alpha = (double*)malloc(sizeof(double) * 2 * (size_t)k);
  double* cnorm = (double*)malloc(sizeof(double) * (size_t)k);
  int32_t deficient = 0;
  for (int64_t j = 0; j < k; ++j) {
    memcpy(W + 2 * j * n, A + 2 * j * lda, sizeof(double) * 2 * n);
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += A[2 * (j * lda + i)] * A[2 * (j * lda + i)] + A[2 * (j * lda + i) + 1] * A[2 * (j * lda + i) + 1];
    cnorm[j] = sqrt(s);
  }
  memset(vs, 0, sizeof(double) * 2 * (size_t)n * (size_t)k);
  for (int64_t j = 0; j < k; ++j) {
    double* x = W + 2 * j * n;
    double nx = 0.0;
    for (int64_t i = j; i < n; ++i) nx += x[2 * i] * x[2 * i] + x[2 * i + 1] * x[2 * i + 1];
    nx = sqrt(nx);
    double x0r = x[2 * j], x0i = x[2 * j + 1];
    double ax0 = hypot(x0r, x0i);
    double pr = 1.0, pi = 0.0; /* phase of x_0 */
    if (ax0 > 0.0) {
      pr = x0r / ax0;
      pi = x0i / ax0;
    }
    double ar = -pr * nx, ai = -pi * nx;
    alpha[2 * j] = ar;
    alpha[2 * j + 1] = ai;
    double* v = vs + 2 * j * n;
    for (int64_t i = j; i < n; ++i) {
      v[2 * i] = x[2 * i];
      v[2 * i + 1] = x[2 * i + 1];
    }
    v[2 * j] -= ar;
    v[2 * j + 1] -= ai;
    double vv = 0.0;
    for (int64_t i = j; i < n; ++i) vv += v[2 * i] * v[2 * i] + v[2 * i + 1] * v[2 * i + 1];
    if (nx < 1e-12 * cnorm[j] || nx == 0.0) ++deficient;
    /* column j becomes alpha e_j above the diagonal part */
    x[2 * j] = ar;
    x[2 * j + 1] = ai;
    for (int64_t i = j + 1; i < n; ++i) x[2 * i] = x[2 * i + 1] = 0.0;
    if (vv == 0.0) continue;
    /* apply (I - 2 v v^H / vv) to columns j+1..k-1 */
#pragma omp parallel for schedule(static)
    for (int64_t l = j + 1; l < k; ++l) {
      double* y = W + 2 * l * n;
      double sr = 0.0, si = 0.0; /* v^H y */
      for (int64_t i = j; i < n; ++i) {
        sr += v[2 * i] * y[2 * i] + v[2 * i + 1] * y[2 * i + 1];
        si += v[2 * i] * y[2 * i + 1] - v[2 * i + 1] * y[2 * i];
      }
      double fr = 2.0 * sr / vv, fi = 2.0 * si / vv;
      for (int64_t i = j; i < n; ++i) {
        y[2 * i] -= v[2 * i] * fr - v[2 * i + 1] * fi;
        y[2 * i + 1] -= v[2 * i] * fi + v[2 * i + 1] * fr;
      }
    }
  }
  /* Q = H_0 H_1 ... H_{k-1} I[:, 0:k], accumulated backwards */
  for (int64_t l = 0; l < k; ++l) {
    double* q = Q + 2 * l * ldq;
    for (int64_t i = 0; i < n; ++i) q[2 * i] = q[2 * i + 1] = 0.0;
    q[2 * l] = 1.0;
  }
  for (int64_t j = k - 1; j >= 0; --j) {
    const double* v = vs + 2 * j * n;
    double vv = 0.0;
    for (int64_t i = j; i < n; ++i) vv += v[2 * i] * v[2 * i] + v[2 * i + 1] * v[2 * i + 1];
    if (vv == 0.0) continue;
#pragma omp parallel for schedule(static)
    for (int64_t l = 0; l < k; ++l) {
      double* y = Q + 2 * l * ldq;
      double sr = 0.0, si = 0.0;
      for (int64_t i = j; i < n; ++i) {
        sr += v[2 * i] * y[2 * i] + v[2 * i + 1] * y[2 * i + 1];
        si += v[2 * i] * y[2 * i + 1] - v[2 * i + 1] * y[2 * i];
      }
      double fr = 2.0 * sr / vv, fi = 2.0 * si / vv;
      for (int64_t i = j; i < n; ++i) {
        y[2 * i] -= v[2 * i] * fr - v[2 * i + 1] * fi;
        y[2 * i + 1] -= v[2 * i] * fi + v[2 * i + 1] * fr;
      }
    }
  }
  /* make diag(R) real positive: Q[:,j] *= phase(alpha_j), R[j,:] *= conj(phase(alpha_j)) */
  for (int64_t j = 0; j < k; ++j) {
    double ar = alpha[2 * j], ai = alpha[2 * j + 1];
    double aa = hypot(ar, ai);
    double pr = 1.0, pi = 0.0;
    if (aa > 0.0) {
      pr = ar / aa;
      pi = ai / aa;
    }
    double* q = Q + 2 * j * ldq;
    for (int64_t i = 0; i < n; ++i) {
      double qr = q[2 * i], qi = q[2 * i + 1];
      q[2 * i] = qr * pr - qi * pi;
      q[2 * i + 1] = qr * pi + qi * pr;
    }
    if (R) {
      for (int64_t l = 0; l < k; ++l) {
        double rr = 0.0, ri = 0.0;
        if (l >= j) {
          rr = W[2 * (l * n + j)];
          ri = W[2 * (l * n + j) + 1];
        }
        /* conj(p) * r */
        R[2 * (l * ldr + j)] = pr * rr + pi * ri;
        R[2 * (l * ldr + j) + 1] = pr * ri - pi * rr;
      }
    }
  }
  free(W);
  free(vs);
  free(alpha);
  free(cnorm);
  return deficient;
}

/* Cyclic complex Jacobi. For a pair (p,q) with b = a_pq = |b| e^{i phi}: D = diag(1, e^{-i phi})
 * makes the pair real, then the classical symmetric rotation (t = sgn(z)/(|z|+sqrt(1+z^2)),
 * z = (a_qq - a_pp)/(2|b|)) annihilates it. Combined G = D R applied as A <- G^H A G, V <- V G. */
int32_t ora_jacobi_eig(int64_t n, const double* Ain, int64_t lda, double* w, double* V,
                       int64_t ldv) {
  double* A = (double*)malloc(sizeof(double) * 2 * (size_t)n * (size_t)n);
  double* Z = (double*)malloc(sizeof(double) * 2 * (size_t)n * (size_t)n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) {
      /* hermitise (A + A^H)/2 */
      A[2 * (j * n + i)] = 0.5 * (Ain[2 * (j * lda + i)] + Ain[2 * (i * lda + j)]);
      A[2 * (j * n + i) + 1] = 0.5 * (Ain[2 * (j * lda + i) + 1] - Ain[2 * (i * lda + j) + 1]);
      Z[2 * (j * n + i)] = (i == j) ? 1.0 : 0.0;
      Z[2 * (j * n + i) + 1] = 0.0;
    }
  double fro = 0.0;
  for (int64_t t = 0; t < n * n; ++t) fro += A[2 * t] * A[2 * t] + A[2 * t + 1] * A[2 * t + 1];
  int32_t sweeps = -1;
  int64_t rotated_last = 1;
  for (int32_t sw = 1; sw <= 60; ++sw) {
    double off = 0.0;
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i)
        if (i != j) off += A[2 * (j * n + i)] * A[2 * (j * n + i)] + A[2 * (j * n + i) + 1] * A[2 * (j * n + i) + 1];
    if (off == 0.0 || rotated_last == 0) {
      sweeps = sw - 1;
      break;
    }
    rotated_last = 0;
    for (int64_t p = 0; p < n - 1; ++p)
      for (int64_t q = p + 1; q < n; ++q) {
        double br = A[2 * (q * n + p)], bi = A[2 * (q * n + p) + 1];
        double ab = hypot(br, bi);
        double app = A[2 * (p * n + p)], aqq = A[2 * (q * n + q)];
        /* skip negligible pairs: relative (Demmel-Veselic) and absolute thresholds */
        if (ab == 0.0) continue;
        if (ab <= 4e-16 * sqrt(fabs(app) * fabs(aqq)) || ab <= 1e-17 * sqrt(fro)) continue;
        ++rotated_last;
        double z = (aqq - app) / (2.0 * ab);
        double t = (z >= 0.0 ? 1.0 : -1.0) / (fabs(z) + sqrt(1.0 + z * z));
        double cs = 1.0 / sqrt(1.0 + t * t), sn = t * cs;
        double er = br / ab, ei = -bi / ab; /* e^{-i phi} */
        /* G = [[cs, sn], [-sn e, cs e]] with e = e^{-i phi}; columns p,q of A <- A G */
        for (int64_t i = 0; i < n; ++i) {
          double xr = A[2 * (p * n + i)], xi = A[2 * (p * n + i) + 1];
          double yr = A[2 * (q * n + i)], yi = A[2 * (q * n + i) + 1];
          double ye_r = yr * er - yi * ei, ye_i = yr * ei + yi * er; /* y e */
          A[2 * (p * n + i)] = cs * xr - sn * ye_r;
          A[2 * (p * n + i) + 1] = cs * xi - sn * ye_i;
          A[2 * (q * n + i)] = sn * xr + cs * ye_r;
          A[2 * (q * n + i) + 1] = sn * xi + cs * ye_i;
          double zr = Z[2 * (p * n + i)], zi = Z[2 * (p * n + i) + 1];
          double wr = Z[2 * (q * n + i)], wi = Z[2 * (q * n + i) + 1];
          double we_r = wr * er - wi * ei, we_i = wr * ei + wi * er;
          Z[2 * (p * n + i)] = cs * zr - sn * we_r;
          Z[2 * (p * n + i) + 1] = cs * zi - sn * we_i;
          Z[2 * (q * n + i)] = sn * zr + cs * we_r;
          Z[2 * (q * n + i) + 1] = sn * zi + cs * we_i;
        }
        /* rows p,q of A <- G^H A: row p' = cs row_p - sn conj(e) row_q; row q' = sn row_p + cs conj(e) row_q */
        for (int64_t l = 0; l < n; ++l) {
          double xr = A[2 * (l * n + p)], xi = A[2 * (l * n + p) + 1];
          double yr = A[2 * (l * n + q)], yi = A[2 * (l * n + q) + 1];
          double ye_r = yr * er + yi * ei, ye_i = yi * er - yr * ei; /* conj(e) y */
          A[2 * (l * n + p)] = cs * xr - sn * ye_r;
          A[2 * (l * n + p) + 1] = cs * xi - sn * ye_i;
          A[2 * (l * n + q)] = sn * xr + cs * ye_r;
          A[2 * (l * n + q) + 1] = sn * xi + cs * ye_i;
        }
        A[2 * (q * n + p)] = A[2 * (q * n + p) + 1] = 0.0;
        A[2 * (p * n + q)] = A[2 * (p * n + q) + 1] = 0.0;
        A[2 * (p * n + p) + 1] = 0.0;
        A[2 * (q * n + q) + 1] = 0.0;
      }
  }
  /* sort ascending, stable by index (insertion sort on an index array) */
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) idx[i] = i;
  for (int64_t i = 1; i < n; ++i) {
    int64_t t = idx[i];
    double v = A[2 * (t * n + t)];
    int64_t j = i - 1;
    while (j >= 0 && A[2 * (idx[j] * n + idx[j])] > v) {
      idx[j + 1] = idx[j];
      --j;
    }
    idx[j + 1] = t;
  }
  for (int64_t c = 0; c < n; ++c) {
    int64_t s = idx[c];
    w[c] = A[2 * (s * n + s)];
    const double* z = Z + 2 * s * n;
    /* phase: largest-|.| entry real positive, ties -> lowest row */
    int64_t im = 0;
    double best = -1.0;
    for (int64_t i = 0; i < n; ++i) {
      double a = z[2 * i] * z[2 * i] + z[2 * i + 1] * z[2 * i + 1];
      if (a > best) {
        best = a;
        im = i;
      }
    }
    double mr = z[2 * im], mi = z[2 * im + 1], mm = hypot(mr, mi);
    double pr = mm > 0 ? mr / mm : 1.0, pi = mm > 0 ? -mi / mm : 0.0; /* conj phase */
    for (int64_t i = 0; i < n; ++i) {
      double zr = z[2 * i], zi = z[2 * i + 1];
      V[2 * (c * ldv + i)] = zr * pr - zi * pi;
      V[2 * (c * ldv + i) + 1] = zr * pi + zi * pr;
    }
    V[2 * (c * ldv + im) + 1] = 0.0;
  }
  free(idx);
  free(A);
  free(Z);
  return sweeps;
}

/* ------------------------------------------------------------------------------------------------ */
static uint64_t ora_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

void ora_random_vector(int64_t n, uint64_t seed, uint64_t stream, double* x) {
  for (int64_t i = 0; i < n; ++i) {
    uint64_t h0 = ora_splitmix64(seed ^ (stream << 40) ^ (uint64_t)(2 * i));
    uint64_t h1 = ora_splitmix64(seed ^ (stream << 40) ^ (uint64_t)(2 * i + 1));
    double u0 = (double)(h0 >> 11) * (1.0 / 9007199254740992.0);
    double u1 = (double)(h1 >> 11) * (1.0 / 9007199254740992.0);
    x[2 * i] = 2.0 * u0 - 1.0;
    x[2 * i + 1] = 2.0 * u1 - 1.0;
  }
}

static double znrm2(int64_t n, const double* x) {
  double s = 0.0;
  for (int64_t i = 0; i < 2 * n; ++i) s += x[i] * x[i];
  return sqrt(s);
}

/* w = H v for Hermitian H, naive: w[r] = sum_q conj(H[q,r]) v[q] (R13) */
static void zhemv_naive(int64_t n, const double* H, int64_t ldh, const double* v, double* w) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) {
    const double* h = H + 2 * r * ldh;
    double sr = 0.0, si = 0.0;
    for (int64_t q = 0; q < n; ++q) {
      double hr = h[2 * q], hi = -h[2 * q + 1];
      sr += hr * v[2 * q] - hi * v[2 * q + 1];
      si += hr * v[2 * q + 1] + hi * v[2 * q];
    }
    w[2 * r] = sr;
    w[2 * r + 1] = si;
  }
}

/* eigenvalues of a real symmetric tridiagonal (alpha[0..m-1], beta[0..m-2]) by bisection
 * (Sturm counts), to full double accuracy */
static void tridiag_eig_extremes(int32_t m, const double* al, const double* be, double* tmin,
                                 double* tmax) {
  double lo = al[0], hi = al[0];
  for (int32_t i = 0; i < m; ++i) {
    double r = (i > 0 ? fabs(be[i - 1]) : 0.0) + (i < m - 1 ? fabs(be[i]) : 0.0);
    if (al[i] - r < lo) lo = al[i] - r;
    if (al[i] + r > hi) hi = al[i] + r;
  }
  for (int which = 0; which < 2; ++which) {
    /* count(x) = #eigenvalues < x */
    double a = lo, b = hi;
    int64_t target = which == 0 ? 1 : m; /* smallest: count >= 1; largest: count >= m */
    for (int it = 0; it < 200; ++it) {
      double x = 0.5 * (a + b);
      if (x == a || x == b) break;
      int64_t cnt = 0;
      double d = 1.0;
      for (int32_t i = 0; i < m; ++i) {
        double bb = i > 0 ? be[i - 1] * be[i - 1] : 0.0;
        d = (al[i] - x) - (i > 0 ? bb / d : 0.0);
        if (d == 0.0) d = -1e-300;
        if (d < 0) ++cnt;
      }
      if (cnt >= target) b = x;
      else a = x;
    }
    if (which == 0) *tmin = b;
    else *tmax = b;
  }
}

int32_t ora_lanczos(int64_t n, const double* H, int64_t ldh, int32_t steps, uint64_t seed,
                    double* theta_min, double* theta_max, double* beta_up) {
  if (steps < 1 || n < 1) return 1;
  if (steps > n) steps = (int32_t)n;
  double* Vb = (double*)malloc(sizeof(double) * 2 * (size_t)n * (size_t)(steps + 1));
  double* w = (double*)malloc(sizeof(double) * 2 * (size_t)n);
  double* al = (double*)malloc(sizeof(double) * (size_t)steps);
  double* be = (double*)malloc(sizeof(double) * (size_t)steps);
  int32_t status = 1;
  for (int restart = 0; restart <= 3; ++restart) {
    double* v0 = Vb;
    ora_random_vector(n, seed, ((uint64_t)4 << 16) | (uint64_t)restart, v0);
    double nv = znrm2(n, v0);
    for (int64_t i = 0; i < 2 * n; ++i) v0[i] /= nv;
    int32_t j;
    int broke = 0;
    double hest = 0.0;
    for (j = 0; j < steps; ++j) {
      double* vj = Vb + 2 * j * n;
      zhemv_naive(n, H, ldh, vj, w);
      double a = 0.0; /* Re(v^H w) */
      for (int64_t i = 0; i < n; ++i) a += vj[2 * i] * w[2 * i] + vj[2 * i + 1] * w[2 * i + 1];
      al[j] = a;
      for (int64_t i = 0; i < 2 * n; ++i) w[i] -= a * vj[i];
      if (j > 0) {
        double* vp = Vb + 2 * (j - 1) * n;
        for (int64_t i = 0; i < 2 * n; ++i) w[i] -= be[j - 1] * vp[i];
      }
      /* full reorthogonalisation, twice (classical Gram-Schmidt against v_0..v_j) */
      for (int pass = 0; pass < 2; ++pass)
        for (int32_t l = 0; l <= j; ++l) {
          double* vl = Vb + 2 * l * n;
          double sr = 0.0, si = 0.0;
          for (int64_t i = 0; i < n; ++i) {
            sr += vl[2 * i] * w[2 * i] + vl[2 * i + 1] * w[2 * i + 1];
            si += vl[2 * i] * w[2 * i + 1] - vl[2 * i + 1] * w[2 * i];
          }
          for (int64_t i = 0; i < n; ++i) {
            w[2 * i] -= vl[2 * i] * sr - vl[2 * i + 1] * si;
            w[2 * i + 1] -= vl[2 * i] * si + vl[2 * i + 1] * sr;
          }
        }
      double b = znrm2(n, w);
      be[j] = b;
      double m = fabs(a) + b + (j > 0 ? be[j - 1] : 0.0);
      if (m > hest) hest = m;
      if (j + 1 < steps) {
        if (b < 1e-14 * hest) {
          /* invariant subspace found: if the Krylov space is exhausted (j+1 == n) stop normally */
          if (j + 1 >= n) { ++j; break; }
          broke = 1;
          break;
        }
        double* vn = Vb + 2 * (j + 1) * n;
        for (int64_t i = 0; i < 2 * n; ++i) vn[i] = w[i] / b;
      }
    }
    if (broke) continue;
    int32_t m = j < steps ? j : steps;
    tridiag_eig_extremes(m, al, be, theta_min, theta_max);
    *beta_up = *theta_max + be[m - 1];
    status = 0;
    break;
  }
  free(Vb);
  free(w);
  free(al);
  free(be);
  return status;
}

int32_t ora_rayleigh_ritz(int64_t n, const double* H, int64_t ldh, double* Q, int64_t ldq,
                          int64_t k, double* ritz) {
  double* HQ = (double*)malloc(sizeof(double) * 2 * (size_t)n * (size_t)k);
  double* G = (double*)malloc(sizeof(double) * 2 * (size_t)k * (size_t)k);
  double* W = (double*)malloc(sizeof(double) * 2 * (size_t)k * (size_t)k);
  double* Y = (double*)malloc(sizeof(double) * 2 * (size_t)n * (size_t)k);
  ora_zgemm('N', 'N', n, k, n, H, ldh, Q, ldq, HQ, n);  /* H Q */
  ora_zgemm('C', 'N', k, k, n, Q, ldq, HQ, n, G, k);    /* Q^H (H Q) */
  int32_t sw = ora_jacobi_eig(k, G, k, ritz, W, k);    /* hermitised inside */
  ora_zgemm('N', 'N', n, k, k, Q, ldq, W, k, Y, n);     /* Q W */
  for (int64_t j = 0; j < k; ++j) memcpy(Q + 2 * j * ldq, Y + 2 * j * n, sizeof(double) * 2 * n);
  free(HQ);
  free(G);
  free(W);
  free(Y);
  return sw < 0 ? 1 : 0;
}

void ora_residuals(int64_t n, const double* H, int64_t ldh, const double* X, int64_t ldx, int64_t k,
                   const double* lam, double normH, double* resid) {
  double* w = (double*)malloc(sizeof(double) * 2 * (size_t)n);
  for (int64_t j = 0; j < k; ++j) {
    const double* x = X + 2 * j * ldx;
    zhemv_naive(n, H, ldh, x, w);
    double s = 0.0, xx = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double rr = w[2 * i] - lam[j] * x[2 * i], ri = w[2 * i + 1] - lam[j] * x[2 * i + 1];
      s += rr * rr + ri * ri;
      xx += x[2 * i] * x[2 * i] + x[2 * i + 1] * x[2 * i + 1];
    }
    resid[j] = sqrt(s) / (sqrt(xx) * normH);
  }
  free(w);
}

/* rho_j = Re(x_j^H H x_j) / (x_j^H x_j) (the Rayleigh quotient) and
 * resid_abs[j] = ||H x_j - rho_j x_j||_2 / ||x_j||_2, one naive mat-vec per column (R13). */
void ora_rayleigh_quotients(int64_t n, const double* H, int64_t ldh, const double* X, int64_t ldx, int64_t k,
                            double* rho, double* resid_abs) {
  double* w = (double*)malloc(sizeof(double) * 2 * (size_t)n);
  for (int64_t j = 0; j < k; ++j) {
    const double* x = X + 2 * j * ldx;
    zhemv_naive(n, H, ldh, x, w);
    double xhx = 0.0, xx = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      xhx += x[2 * i] * w[2 * i] + x[2 * i + 1] * w[2 * i + 1];
      xx += x[2 * i] * x[2 * i] + x[2 * i + 1] * x[2 * i + 1];
    }
    const double r = xhx / xx;
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double dr = w[2 * i] - r * x[2 * i], di = w[2 * i + 1] - r * x[2 * i + 1];
      s += dr * dr + di * di;
    }
    rho[j] = r;
    resid_abs[j] = sqrt(s) / sqrt(xx);
  }
  free(w);
}

double ora_rho(double t) {
  double a = fabs(t);
  if (a <= 1.0) return 1.0;
  return a + sqrt(a * a - 1.0);
}

int32_t ora_degree(double res, double tol, double t, int32_t cap) {
  double a = fabs(t);
  if (a <= 1.0) return cap;
  double ratio = res / tol;
  if (ratio < 1.0) ratio = 1.0;
  double m = ceil(acosh(ratio) / acosh(a));
  if (!(m >= 1.0)) m = 1.0;
  if (m > (double)cap) m = (double)cap;
  return (int32_t)m;
}

int32_t ora_degree_literal(double res, double tol, double rho, int32_t cap) {
  if (!(rho > 1.0)) return cap;
  double m = ceil(log(res / tol) / log(rho));
  if (!(m >= 1.0)) m = 1.0;
  if (m > (double)cap) m = (double)cap;
  return (int32_t)m;
}

/* ------------------------------------------------------------------------------------------------ */
/* Y (n x ka) <- Y - X (X^H Y), twice (CGS2 against the locked block, R15) */
static void cgs2(int64_t n, const double* X, int64_t nl, double* Y, int64_t ka) {
  if (nl == 0 || ka == 0) return;
  double* C = (double*)malloc(sizeof(double) * 2 * (size_t)nl * (size_t)ka);
  double* XC = (double*)malloc(sizeof(double) * 2 * (size_t)n * (size_t)ka);
  for (int pass = 0; pass < 2; ++pass) {
    ora_zgemm('C', 'N', nl, ka, n, X, n, Y, n, C, nl);
    ora_zgemm('N', 'N', n, ka, nl, X, n, C, nl, XC, n);
    for (int64_t t = 0; t < 2 * n * ka; ++t) Y[t] -= XC[t];
  }
  free(C);
  free(XC);
}

/* Alg 1 l6 with the rank-deficiency rule R23:
 *  nu_j = ||y_j|| (input);  repeat: Y <- CGS2(Y against X_L); Householder QR Y = Q R;
 *  D = {j : |R_jj| <= 1e-12 nu_j}; if D is empty, Y <- Q and stop; otherwise (at most 3 rounds)
 *  y_j <- x_j for j in D, x_j the R22 vector with seed `seed + round` and stream (6 << 16) | (nl + j),
 *  nu_j <- ||x_j||, and repeat on the whole block. */
int32_t ora_orthonormalize(int64_t n, const double* XL, int64_t nl, double* Y, int64_t ka, uint64_t seed,
                           int32_t* replaced) {
  if (replaced) *replaced = 0;
  if (ka == 0) return 0;
  const size_t colsz = sizeof(double) * 2 * (size_t)n;
  double* Q = (double*)malloc(colsz * (size_t)ka);
  double* R = (double*)malloc(sizeof(double) * 2 * (size_t)ka * (size_t)ka);
  double* nu = (double*)malloc(sizeof(double) * (size_t)ka);
  for (int64_t j = 0; j < ka; ++j) nu[j] = znrm2(n, Y + 2 * j * n);
  int32_t status = 4;
  for (int round = 0; round <= 3; ++round) {
    cgs2(n, XL, nl, Y, ka);
    ora_householder_qr(n, ka, Y, n, Q, n, R, ka);
    int32_t nd = 0;
    for (int64_t j = 0; j < ka; ++j) {
      const double rjj = hypot(R[2 * (j * ka + j)], R[2 * (j * ka + j) + 1]);
      if (!(rjj <= 1e-12 * nu[j])) continue;
      ++nd;
      if (round < 3) {
        ora_random_vector(n, seed + (uint64_t)round, ((uint64_t)6 << 16) | (uint64_t)(nl + j), Y + 2 * j * n);
        nu[j] = znrm2(n, Y + 2 * j * n);
      }
    }
    if (nd == 0) {
      memcpy(Y, Q, colsz * (size_t)ka);
      status = 0;
      break;
    }
    if (round == 3) break;
    if (replaced) *replaced += nd;
  }
  free(Q);
  free(R);
  free(nu);
  return status;
}

int32_t ora_chfsi_solve(int64_t n, const double* H, int64_t ldh, const ora_opts* o, double* X,
                        int64_t ldx, int32_t have_prev, double* lambda1, double* lambdak,
                        double* lam, double* resid, ora_report* rep) {
  const int64_t nev = o->nev, k = (int64_t)o->nev + o->nex;
  if (nev < 1 || o->nex < 0 || k > n || !(o->tol > 0) || o->deg0 < 1 || o->deg0 > o->deg_cap)
    return 1;
  memset(rep, 0, sizeof(*rep));
  /* Alg 1 l3: Lanczos upper bound (R17); ||H||_est (R8) */
  double tmin, tmax, beta;
  if (ora_lanczos(n, H, ldh, o->lanczos_steps, o->seed, &tmin, &tmax, &beta)) return 1;
  const size_t colsz = sizeof(double) * 2 * (size_t)n;
  double* XL = (double*)malloc(colsz * (size_t)k);   /* locked vectors, in locking order */
  double* lamL = (double*)malloc(sizeof(double) * (size_t)k);
  double* resL = (double*)malloc(sizeof(double) * (size_t)k);
  double* Ya = (double*)malloc(colsz * (size_t)k);   /* active block */
  double* Tmp = (double*)malloc(colsz * (size_t)k);
  double* mu = (double*)malloc(sizeof(double) * (size_t)k);
  double* res = (double*)malloc(sizeof(double) * (size_t)k);
  int32_t* m = (int32_t*)malloc(sizeof(int32_t) * (size_t)k);
  int32_t* ms = (int32_t*)malloc(sizeof(int32_t) * (size_t)k);
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
  for (int64_t j = 0; j < k; ++j) memcpy(Ya + 2 * j * n, X + 2 * j * ldx, colsz);

  double normH = fabs(tmin) > fabs(tmax) ? fabs(tmin) : fabs(tmax);
  rep->theta_min = tmin;
  rep->theta_max = tmax;
  rep->beta_up = beta;
  rep->normH = normH;
  rep->matvecs_total += o->lanczos_steps;

  double lam1 = *lambda1, alpha = *lambdak;
  int32_t status = 3;
  /* the previous problem's (lambda_1, lambda_k) must fit under this problem's bound; otherwise the
   * start block seeds them as for a first problem (R11) */
  if (have_prev && !(beta > alpha && lam1 < alpha)) have_prev = 0;
  if (!have_prev) {
    /* R11: random start -> QR -> RR seeds (lambda_1, alpha) */
    int32_t nrep = 0;
    if (ora_orthonormalize(n, NULL, 0, Ya, k, o->seed, &nrep)) status = 4;
    rep->qr_replaced += nrep;
    ora_rayleigh_ritz(n, H, ldh, Ya, n, k, mu);
    rep->matvecs_total += k;
    lam1 = mu[0];
    alpha = mu[k - 1];
  }
  /* Alg 1 l2 (R12): degrees start at deg0 */
  for (int64_t j = 0; j < k; ++j) m[j] = o->deg0;
  int64_t nl = 0; /* locked count */
  while (status == 3 && rep->loops < o->max_loops) {
    const int64_t ka = k - nl;
    double c = 0.5 * (alpha + beta), e = 0.5 * (beta - alpha);
    /* R6: stable ascending sort of the active columns by degree */
    for (int64_t j = 0; j < ka; ++j) perm[j] = j;
    for (int64_t i = 1; i < ka; ++i) {
      int64_t t = perm[i];
      int64_t j = i - 1;
      while (j >= 0 && m[perm[j]] > m[t]) {
        perm[j + 1] = perm[j];
        --j;
      }
      perm[j + 1] = t;
    }
    for (int64_t j = 0; j < ka; ++j) {
      memcpy(Tmp + 2 * j * n, Ya + 2 * perm[j] * n, colsz);
      ms[j] = m[perm[j]];
    }
    /* Alg 1 l5: Chebyshev filter (Alg 2) */
    int64_t mvf = 0;
    ora_filter(n, H, ldh, Tmp, n, ka, ms, lam1, c, e, &mvf);
    rep->matvecs_filter += mvf;
    rep->matvecs_total += mvf;
    /* Alg 1 l6: orthonormalise against the locked block (R15), then Householder QR (R14) */
    int32_t nrep = 0;
    if (ora_orthonormalize(n, XL, nl, Tmp, ka, o->seed, &nrep)) {
      status = 4;
      break;
    }
    rep->qr_replaced += nrep;
    memcpy(Ya, Tmp, colsz * (size_t)ka);
    /* Alg 1 l7-9: Rayleigh-Ritz on the active block (R16) */
    ora_rayleigh_ritz(n, H, ldh, Ya, n, ka, mu);
    rep->matvecs_total += ka;
    /* residuals (R8) */
    ora_residuals(n, H, ldh, Ya, n, ka, mu, normH, res);
    rep->matvecs_total += ka;
    rep->loops++;
    /* Alg 1 l10 (R7): lock wanted Ritz positions with r <= tol */
    const int64_t want = nev - nl;
    int64_t na = 0;
    for (int64_t j = 0; j < ka; ++j) {
      if (j < want && res[j] <= o->tol) {
        memcpy(XL + 2 * nl * n, Ya + 2 * j * n, colsz);
        lamL[nl] = mu[j];
        resL[nl] = res[j];
        ++nl;
      } else {
        if (na != j) {
          memmove(Ya + 2 * na * n, Ya + 2 * j * n, colsz);
          mu[na] = mu[j];
          res[na] = res[j];
        }
        ++na;
      }
    }
    /* R4: interval from the current k values (locked + active Ritz) */
    double vmin = HUGE_VAL, vmax = -HUGE_VAL;
    for (int64_t j = 0; j < na; ++j) {
      if (mu[j] < vmin) vmin = mu[j];
      if (mu[j] > vmax) vmax = mu[j];
    }
    for (int64_t j = 0; j < nl; ++j) {
      if (lamL[j] < vmin) vmin = lamL[j];
      if (lamL[j] > vmax) vmax = lamL[j];
    }
    lam1 = vmin;
    alpha = vmax;
    if (nl >= nev) {
      status = 0;
      break;
    }
    /* Alg 1 l11 (R21, R5, R9): degrees for the next filter */
    double c2 = 0.5 * (alpha + beta), e2 = 0.5 * (beta - alpha);
    const int64_t want2 = nev - nl;
    int32_t mmax = 1;
    for (int64_t j = 0; j < na; ++j) {
      if (j < want2) {
        m[j] = ora_degree(res[j], o->tol, (mu[j] - c2) / e2, o->deg_cap);
        if (m[j] == o->deg_cap) rep->capped++;
        if (m[j] > mmax) mmax = m[j];
      }
    }
    for (int64_t j = want2; j < na; ++j) m[j] = mmax;
  }
  rep->converged = (int32_t)nl;
  /* output: locked sorted ascending (stable), then the remaining active columns */
  int64_t* ord = perm;
  for (int64_t j = 0; j < nl; ++j) ord[j] = j;
  for (int64_t i = 1; i < nl; ++i) {
    int64_t t = ord[i];
    int64_t j = i - 1;
    while (j >= 0 && lamL[ord[j]] > lamL[t]) {
      ord[j + 1] = ord[j];
      --j;
    }
    ord[j + 1] = t;
  }
  for (int64_t j = 0; j < nl; ++j) {
    memcpy(X + 2 * j * ldx, XL + 2 * ord[j] * n, colsz);
    if (j < nev) {
      lam[j] = lamL[ord[j]];
      resid[j] = resL[ord[j]];
    }
  }
  const int64_t na_final = k - nl;
  for (int64_t j = 0; j < na_final; ++j) {
    memcpy(X + 2 * (nl + j) * ldx, Ya + 2 * j * n, colsz);
    if (nl + j < nev) { /* partial results (not converged) */
      lam[nl + j] = mu[j];
      resid[nl + j] = res[j];
    }
  }
  *lambda1 = lam1;
  *lambdak = alpha;
  free(XL);
  free(lamL);
  free(resL);
  free(Ya);
  free(Tmp);
  free(mu);
  free(res);
  free(m);
  free(ms);
  free(perm);
  return status;
}

/* ------------------------------------------------------------------------------------------------ */
/* Sylvester's law of inertia: H - sigma I = P L D L^H P^T has as many negative eigenvalues as the
 * block-diagonal D. D is produced by the Bunch-Kaufman symmetric pivoting strategy (1x1 and 2x2
 * pivots, alpha = (1 + sqrt 17)/8, the strategy of LAPACK's xHETF2), right-looking, on the lower
 * triangle of a copy. Only D is needed, so L is not kept and interchanges touch the trailing
 * matrix only. |.| is the complex modulus. */
#define LA(i, j) A[2 * ((j) * n + (i))]     /* Re A[i,j], i >= j (lower triangle) */
#define LAI(i, j) A[2 * ((j) * n + (i)) + 1] /* Im A[i,j] */

/* symmetric interchange of rows/columns p < r of the trailing matrix A[c0:, c0:] (lower storage,
 * c0 <= p): the entries of the columns c0..p-1 in rows p and r are exchanged as well */
static void bk_swap(int64_t n, double* A, int64_t c0, int64_t p, int64_t r) {
  if (r == p) return;
  double t;
  for (int64_t c = c0; c < p; ++c) {
    t = LA(p, c), LA(p, c) = LA(r, c), LA(r, c) = t;
    t = LAI(p, c), LAI(p, c) = LAI(r, c), LAI(r, c) = t;
  }
  t = LA(p, p), LA(p, p) = LA(r, r), LA(r, r) = t; /* diagonal entries (real) */
  for (int64_t i = r + 1; i < n; ++i) {           /* below both: A[i,p] <-> A[i,r] */
    t = LA(i, p), LA(i, p) = LA(i, r), LA(i, r) = t;
    t = LAI(i, p), LAI(i, p) = LAI(i, r), LAI(i, r) = t;
  }
  for (int64_t i = p + 1; i < r; ++i) { /* between: A[i,p] <-> conj(A[r,i]) */
    double xr = LA(i, p), xi = LAI(i, p);
    LA(i, p) = LA(r, i), LAI(i, p) = -LAI(r, i);
    LA(r, i) = xr, LAI(r, i) = -xi;
  }
  LAI(r, p) = -LAI(r, p); /* A[r,p] <- conj(A[r,p]) */
}

int64_t ora_count_below(int64_t n, const double* H, int64_t ldh, double sigma) {
  double* A = (double*)malloc(sizeof(double) * 2 * (size_t)n * (size_t)n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = j; i < n; ++i) {
      LA(i, j) = H[2 * (j * ldh + i)] - (i == j ? sigma : 0.0);
      LAI(i, j) = (i == j) ? 0.0 : H[2 * (j * ldh + i) + 1];
    }
  const double alpha = (1.0 + sqrt(17.0)) / 8.0;
  int64_t neg = 0;
  int64_t p = 0;
  while (p < n) {
    /* lambda = largest off-diagonal modulus in column p, at row r */
    double lam = 0.0;
    int64_t r = p;
    for (int64_t i = p + 1; i < n; ++i) {
      double a = hypot(LA(i, p), LAI(i, p));
      if (a > lam) lam = a, r = i;
    }
    const double app = fabs(LA(p, p));
    int size = 1;
    if (lam == 0.0) { /* column p already reduced: 1x1 pivot, no update */
      if (LA(p, p) < 0.0) ++neg;
      ++p;
      continue;
    }
    if (app < alpha * lam) {
      /* sigma_r = largest off-diagonal modulus in row/column r of the trailing matrix */
      double sr = 0.0;
      for (int64_t j = p; j < r; ++j) {
        double a = hypot(LA(r, j), LAI(r, j));
        if (a > sr) sr = a;
      }
      for (int64_t i = r + 1; i < n; ++i) {
        double a = hypot(LA(i, r), LAI(i, r));
        if (a > sr) sr = a;
      }
      if (app * sr >= alpha * lam * lam) {
        /* 1x1 pivot at p, no interchange */
      } else if (fabs(LA(r, r)) >= alpha * sr) {
        bk_swap(n, A, p, p, r); /* 1x1 pivot A[r,r] */
      } else {
        bk_swap(n, A, p, p + 1, r); /* 2x2 pivot on (p, r) */
        size = 2;
      }
    }
    if (size == 1) {
      const double d = LA(p, p);
      if (d < 0.0) ++neg;
      /* A[i,j] -= A[i,p] conj(A[j,p]) / d, i >= j > p */
#pragma omp parallel for schedule(dynamic, 16)
      for (int64_t j = p + 1; j < n; ++j) {
        const double xjr = LA(j, p), xji = LAI(j, p);
        for (int64_t i = j; i < n; ++i) {
          const double xir = LA(i, p), xii = LAI(i, p);
          LA(i, j) -= (xir * xjr + xii * xji) / d;
          LAI(i, j) -= (xii * xjr - xir * xji) / d;
        }
      }
      ++p;
    } else {
      /* D = [[a, conj(b)], [b, c]], a, c real, b = A[p+1,p]; inertia of D from det and trace */
      const double a = LA(p, p), c = LA(p + 1, p + 1), br = LA(p + 1, p), bi = LAI(p + 1, p);
      const double det = a * c - (br * br + bi * bi);
      if (det < 0.0) neg += 1;
      else if (det > 0.0) neg += (a + c < 0.0) ? 2 : 0;
      else neg += (a + c < 0.0) ? 1 : 0;
      /* A[i,j] -= u_i conj(x_j) + v_i conj(y_j), i >= j >= p+2, with x = A[:,p], y = A[:,p+1] and
       * [u_i v_i] = [x_i y_i] D^{-1} = [c x_i - b y_i, -conj(b) x_i + a y_i] / det */
#pragma omp parallel for schedule(dynamic, 16)
      for (int64_t j = p + 2; j < n; ++j) {
        const double xjr = LA(j, p), xji = LAI(j, p), yjr = LA(j, p + 1), yji = LAI(j, p + 1);
        for (int64_t i = j; i < n; ++i) {
          const double xr = LA(i, p), xi = LAI(i, p), yr = LA(i, p + 1), yi = LAI(i, p + 1);
          const double ur = (c * xr - (br * yr - bi * yi)) / det, ui = (c * xi - (br * yi + bi * yr)) / det;
          const double vr = (-(br * xr + bi * xi) + a * yr) / det, vi = (-(br * xi - bi * xr) + a * yi) / det;
          LA(i, j) -= (ur * xjr + ui * xji) + (vr * yjr + vi * yji);
          LAI(i, j) -= (ui * xjr - ur * xji) + (vi * yjr - vr * yji);
        }
      }
      p += 2;
    }
  }
  free(A);
  return neg;
}
#undef LA
#undef LAI

/* ------------------------------------------------------------------------------------------------ */
/* Cholesky, column by column (left-looking): L[j,j] = sqrt(B[j,j] - sum_p |L[j,p]|^2),
 * L[i,j] = (B[i,j] - sum_p L[i,p] conj(L[j,p])) / L[j,j] for i > j. */
int32_t ora_cholesky(int64_t n, const double* B, int64_t ldb, double* L, int64_t ldl) {
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) L[2 * (j * ldl + i)] = L[2 * (j * ldl + i) + 1] = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    double d = B[2 * (j * ldb + j)];
    for (int64_t p = 0; p < j; ++p) {
      double lr = L[2 * (p * ldl + j)], li = L[2 * (p * ldl + j) + 1];
      d -= lr * lr + li * li;
    }
    if (!(d > 0.0)) return (int32_t)(j + 1);
    d = sqrt(d);
    L[2 * (j * ldl + j)] = d;
#pragma omp parallel for schedule(static)
    for (int64_t i = j + 1; i < n; ++i) {
      double sr = B[2 * (j * ldb + i)], si = B[2 * (j * ldb + i) + 1];
      for (int64_t p = 0; p < j; ++p) {
        double ar = L[2 * (p * ldl + i)], ai = L[2 * (p * ldl + i) + 1]; /* L[i,p] */
        double br = L[2 * (p * ldl + j)], bi = -L[2 * (p * ldl + j) + 1]; /* conj(L[j,p]) */
        sr -= ar * br - ai * bi;
        si -= ar * bi + ai * br;
      }
      L[2 * (j * ldl + i)] = sr / d;
      L[2 * (j * ldl + i) + 1] = si / d;
    }
  }
  return 0;
}

void ora_trsm_lower(int64_t n, int64_t k, const double* L, int64_t ldl, double* X, int64_t ldx,
                    int32_t adjoint) {
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < k; ++c) {
    double* x = X + 2 * c * ldx;
    if (!adjoint) { /* forward: x_i = (x_i - sum_{p<i} L[i,p] x_p) / L[i,i] */
      for (int64_t i = 0; i < n; ++i) {
        double sr = x[2 * i], si = x[2 * i + 1];
        for (int64_t p = 0; p < i; ++p) {
          double lr = L[2 * (p * ldl + i)], li = L[2 * (p * ldl + i) + 1];
          sr -= lr * x[2 * p] - li * x[2 * p + 1];
          si -= lr * x[2 * p + 1] + li * x[2 * p];
        }
        double dr = L[2 * (i * ldl + i)], di = L[2 * (i * ldl + i) + 1];
        double den = dr * dr + di * di;
        x[2 * i] = (sr * dr + si * di) / den;
        x[2 * i + 1] = (si * dr - sr * di) / den;
      }
    } else { /* backward with L^H: x_i = (x_i - sum_{p>i} conj(L[p,i]) x_p) / conj(L[i,i]) */
      for (int64_t i = n - 1; i >= 0; --i) {
        double sr = x[2 * i], si = x[2 * i + 1];
        for (int64_t p = i + 1; p < n; ++p) {
          double lr = L[2 * (i * ldl + p)], li = -L[2 * (i * ldl + p) + 1];
          sr -= lr * x[2 * p] - li * x[2 * p + 1];
          si -= lr * x[2 * p + 1] + li * x[2 * p];
        }
        double dr = L[2 * (i * ldl + i)], di = -L[2 * (i * ldl + i) + 1];
        double den = dr * dr + di * di;
        x[2 * i] = (sr * dr + si * di) / den;
        x[2 * i + 1] = (si * dr - sr * di) / den;
      }
    }
  }
}

int32_t ora_reduce_generalized(int64_t n, const double* A, int64_t lda, const double* B, int64_t ldb,
                               double* H, int64_t ldh, double* L, int64_t ldl) {
  int32_t st = ora_cholesky(n, B, ldb, L, ldl);
  if (st) return st;
  double* W = (double*)malloc(sizeof(double) * 2 * (size_t)n * (size_t)n);
  for (int64_t j = 0; j < n; ++j) memcpy(W + 2 * j * n, A + 2 * j * lda, sizeof(double) * 2 * n);
  ora_trsm_lower(n, n, L, ldl, W, n, 0); /* W = L^{-1} A */
  for (int64_t j = 0; j < n; ++j)        /* H = W^H (= A L^{-H} for Hermitian A) */
    for (int64_t i = 0; i < n; ++i) {
      H[2 * (j * ldh + i)] = W[2 * (i * n + j)];
      H[2 * (j * ldh + i) + 1] = -W[2 * (i * n + j) + 1];
    }
  ora_trsm_lower(n, n, L, ldl, H, ldh, 0); /* H = L^{-1} A L^{-H} */
  for (int64_t j = 0; j < n; ++j)          /* hermitise */
    for (int64_t i = 0; i <= j; ++i) {
      double ur = 0.5 * (H[2 * (j * ldh + i)] + H[2 * (i * ldh + j)]);
      double ui = 0.5 * (H[2 * (j * ldh + i) + 1] - H[2 * (i * ldh + j) + 1]);
      if (i == j) ui = 0.0;
      H[2 * (j * ldh + i)] = ur;
      H[2 * (j * ldh + i) + 1] = ui;
      H[2 * (i * ldh + j)] = ur;
      H[2 * (i * ldh + j) + 1] = -ui;
    }
  free(W);
  return 0;
}
