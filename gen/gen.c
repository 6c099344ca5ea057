/* gen.c -- seeded synthetic input generator (see gen.h). Compiled with -O2 -fno-fast-math
 * -ffp-contract=off so every entry is a fixed sequence of IEEE binary64 operations. */
#include "gen.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

uint64_t gen_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

double gen_uniform(uint64_t seed, uint64_t stream, uint64_t idx) {
  uint64_t h = gen_splitmix64(seed ^ (stream << 40) ^ idx);
  return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

void gen_normal2(uint64_t seed, uint64_t stream, uint64_t idx, double* z0, double* z1) {
  double u1 = 1.0 - gen_uniform(seed, stream, 2 * idx); /* (0, 1] */
  double u2 = gen_uniform(seed, stream, 2 * idx + 1);
  double r = sqrt(-2.0 * log(u1));
  double th = 6.283185307179586476925 * u2;
  *z0 = r * cos(th);
  *z1 = r * sin(th);
}

void gen_spectrum(int64_t n, int64_t nd, double* lam) {
  for (int64_t i = 0; i < nd; ++i) {
    double x = (nd > 1) ? (double)i / (double)(nd - 1) : 0.0;
    lam[i] = -2.0 + 2.0 * log10(1.0 + 9.0 * x);
  }
  int64_t nt = n - nd;
  for (int64_t j = 0; j < nt; ++j) lam[nd + j] = 40.0 * (double)(j + 1) / (double)nt;
}

#define RE(p, i) (p)[2 * (i)]
#define IM(p, i) (p)[2 * (i) + 1]

void gen_wy(int64_t n, uint64_t seed, double* V, double* T) {
  const int R = GEN_NREF;
  for (int r = 0; r < R; ++r) {
    uint64_t st = GEN_STREAM(1, r);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      double x, y;
      gen_normal2(seed, st, (uint64_t)i, &x, &y);
      RE(V, r * n + i) = x;
      IM(V, r * n + i) = y;
    }
  }
  memset(T, 0, sizeof(double) * 2 * R * R);
  for (int r = 0; r < R; ++r) {
    const double* vr = V + 2 * r * n;
    double nrm2 = 0.0;
    for (int64_t i = 0; i < n; ++i) nrm2 += vr[2 * i] * vr[2 * i] + vr[2 * i + 1] * vr[2 * i + 1];
    double tau = 2.0 / nrm2;
    /* w = V[:,0:r]^H v_r */
    double w[2 * GEN_NREF];
    for (int a = 0; a < r; ++a) {
      const double* va = V + 2 * a * n;
      double sr = 0.0, si = 0.0;
      for (int64_t i = 0; i < n; ++i) {
        /* conj(va) * vr */
        sr += va[2 * i] * vr[2 * i] + va[2 * i + 1] * vr[2 * i + 1];
        si += va[2 * i] * vr[2 * i + 1] - va[2 * i + 1] * vr[2 * i];
      }
      w[2 * a] = sr;
      w[2 * a + 1] = si;
    }
    /* T[0:r, r] = -tau * T[0:r,0:r] w */
    for (int a = 0; a < r; ++a) {
      double sr = 0.0, si = 0.0;
      for (int b = a; b < r; ++b) {
        double tr = T[2 * (b * R + a)], ti = T[2 * (b * R + a) + 1];
        sr += tr * w[2 * b] - ti * w[2 * b + 1];
        si += tr * w[2 * b + 1] + ti * w[2 * b];
      }
      T[2 * (r * R + a)] = -tau * sr;
      T[2 * (r * R + a) + 1] = -tau * si;
    }
    T[2 * (r * R + r)] = tau;
    T[2 * (r * R + r) + 1] = 0.0;
  }
}

void gen_wy_aux(int64_t n, const double* lam, const double* V, const double* T, double* B,
                double* A, double* D) {
  const int R = GEN_NREF;
  /* B = V T, A = Lambda V */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    for (int b = 0; b < R; ++b) {
      double sr = 0.0, si = 0.0;
      for (int a = 0; a <= b; ++a) {
        double vr = V[2 * (a * n + i)], vi = V[2 * (a * n + i) + 1];
        double tr = T[2 * (b * R + a)], ti = T[2 * (b * R + a) + 1];
        sr += vr * tr - vi * ti;
        si += vr * ti + vi * tr;
      }
      B[2 * (b * n + i)] = sr;
      B[2 * (b * n + i) + 1] = si;
      A[2 * (b * n + i)] = lam[i] * V[2 * (b * n + i)];
      A[2 * (b * n + i) + 1] = lam[i] * V[2 * (b * n + i) + 1];
    }
  }
  /* M = V^H Lambda V = V^H A (8 x 8) */
  double M[2 * GEN_NREF * GEN_NREF];
  for (int a = 0; a < R; ++a)
    for (int b = 0; b < R; ++b) {
      double sr = 0.0, si = 0.0;
      for (int64_t i = 0; i < n; ++i) {
        double vr = V[2 * (a * n + i)], vi = V[2 * (a * n + i) + 1];
        double ar = A[2 * (b * n + i)], ai = A[2 * (b * n + i) + 1];
        sr += vr * ar + vi * ai;
        si += vr * ai - vi * ar;
      }
      M[2 * (b * R + a)] = sr;
      M[2 * (b * R + a) + 1] = si;
    }
  /* D = B M */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    for (int b = 0; b < R; ++b) {
      double sr = 0.0, si = 0.0;
      for (int a = 0; a < R; ++a) {
        double br = B[2 * (a * n + i)], bi = B[2 * (a * n + i) + 1];
        double mr = M[2 * (b * R + a)], mi = M[2 * (b * R + a) + 1];
        sr += br * mr - bi * mi;
        si += br * mi + bi * mr;
      }
      D[2 * (b * n + i)] = sr;
      D[2 * (b * n + i) + 1] = si;
    }
  }
}

/* f(r,c), r <= c: lam_r delta_rc - sum_a B[r,a] conj(A[c,a]) - sum_a A[r,a] conj(B[c,a])
 *                 + sum_a D[r,a] conj(B[c,a]) */
static void h1_entry(int64_t n, const double* lam, const double* B, const double* A,
                     const double* D, int64_t r, int64_t c, double* hr, double* hi) {
  const int R = GEN_NREF;
  double s1r = 0, s1i = 0, s2r = 0, s2i = 0, s3r = 0, s3i = 0;
  for (int a = 0; a < R; ++a) {
    double br = B[2 * (a * n + r)], bi = B[2 * (a * n + r) + 1];
    double ar = A[2 * (a * n + r)], ai = A[2 * (a * n + r) + 1];
    double dr = D[2 * (a * n + r)], di = D[2 * (a * n + r) + 1];
    double acr = A[2 * (a * n + c)], aci = -A[2 * (a * n + c) + 1];
    double bcr = B[2 * (a * n + c)], bci = -B[2 * (a * n + c) + 1];
    s1r += br * acr - bi * aci;
    s1i += br * aci + bi * acr;
    s2r += ar * bcr - ai * bci;
    s2i += ar * bci + ai * bcr;
    s3r += dr * bcr - di * bci;
    s3i += dr * bci + di * bcr;
  }
  double re = (r == c ? lam[r] : 0.0) - s1r - s2r + s3r;
  double im = 0.0 - s1i - s2i + s3i;
  if (r == c) im = 0.0;
  *hr = re;
  *hi = im;
}

void gen_h1_panel(int64_t n, const double* lam, const double* B, const double* A, const double* D,
                  int64_t c0, int64_t ncols, double* H, int64_t ldh) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < ncols; ++t) {
    int64_t c = c0 + t;
    double* col = H + 2 * t * ldh;
    for (int64_t r = 0; r < n; ++r) {
      double hr, hi;
      if (r <= c) {
        h1_entry(n, lam, B, A, D, r, c, &hr, &hi);
      } else {
        h1_entry(n, lam, B, A, D, c, r, &hr, &hi);
        hi = -hi;
      }
      col[2 * r] = hr;
      col[2 * r + 1] = hi;
    }
  }
}

void gen_eigvecs(int64_t n, const double* V, const double* B, const int64_t* idx, int64_t m,
                 double* X, int64_t ldx) {
  const int R = GEN_NREF;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < m; ++t) {
    int64_t i = idx[t];
    double* col = X + 2 * t * ldx;
    for (int64_t r = 0; r < n; ++r) {
      double sr = 0.0, si = 0.0;
      for (int a = 0; a < R; ++a) {
        double br = B[2 * (a * n + r)], bi = B[2 * (a * n + r) + 1];
        double vr = V[2 * (a * n + i)], vi = -V[2 * (a * n + i) + 1];
        sr += br * vr - bi * vi;
        si += br * vi + bi * vr;
      }
      col[2 * r] = (r == i ? 1.0 : 0.0) - sr;
      col[2 * r + 1] = 0.0 - si;
    }
  }
}

/* G[r,c] for r <= c */
static void gue_entry(int64_t n, uint64_t seed, uint64_t stream, int64_t r, int64_t c, double* gr,
                      double* gi) {
  double x, y;
  gen_normal2(seed, stream, (uint64_t)r * (uint64_t)n + (uint64_t)c, &x, &y);
  if (r == c) {
    *gr = x / sqrt((double)n);
    *gi = 0.0;
  } else {
    double s = sqrt(2.0 * (double)n);
    *gr = x / s;
    *gi = y / s;
  }
}

void gen_gue_panel(int64_t n, uint64_t seed, uint64_t stream, int64_t c0, int64_t ncols,
                   double* G, int64_t ldg) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < ncols; ++t) {
    int64_t c = c0 + t;
    double* col = G + 2 * t * ldg;
    for (int64_t r = 0; r < n; ++r) {
      double gr, gi;
      if (r <= c) {
        gue_entry(n, seed, stream, r, c, &gr, &gi);
      } else {
        gue_entry(n, seed, stream, c, r, &gr, &gi);
        gi = -gi;
      }
      col[2 * r] = gr;
      col[2 * r + 1] = gi;
    }
  }
}

void gen_perturb_panel(int64_t n, uint64_t seed, int32_t ell, double scale, int64_t c0,
                       int64_t ncols, double* H, int64_t ldh) {
  uint64_t stream = GEN_STREAM(2, ell);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < ncols; ++t) {
    int64_t c = c0 + t;
    double* col = H + 2 * t * ldh;
    for (int64_t r = 0; r < n; ++r) {
      double gr, gi;
      if (r <= c) {
        gue_entry(n, seed, stream, r, c, &gr, &gi);
      } else {
        gue_entry(n, seed, stream, c, r, &gr, &gi);
        gi = -gi;
      }
      double pr = scale * gr, pi = scale * gi;
      col[2 * r] = col[2 * r] + pr;
      col[2 * r + 1] = col[2 * r + 1] + pi;
    }
  }
}

void gen_start_basis(int64_t n, int64_t k, uint64_t seed, int64_t r0, int64_t nrows, double* Y,
                     int64_t ldy) {
  (void)n;
  uint64_t stream = GEN_STREAM(3, 0);
  const double s = sqrt(0.5);
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < k; ++j) {
    double* col = Y + 2 * j * ldy;
    for (int64_t t = 0; t < nrows; ++t) {
      int64_t r = r0 + t;
      double x, y;
      gen_normal2(seed, stream, (uint64_t)r * (uint64_t)k + (uint64_t)j, &x, &y);
      col[2 * t] = x * s;
      col[2 * t + 1] = y * s;
    }
  }
}

void gen_lower_factor(int64_t n, uint64_t seed, double scale, double* M, int64_t ldm) {
  uint64_t stream = GEN_STREAM(6, 0);
  const double s = scale / sqrt(2.0 * (double)n);
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t j = 0; j < n; ++j) {
    double* col = M + 2 * j * ldm;
    for (int64_t i = 0; i < n; ++i) {
      if (i < j) {
        col[2 * i] = col[2 * i + 1] = 0.0;
      } else if (i == j) {
        col[2 * i] = 1.0 + 0.5 * gen_uniform(seed, stream, (uint64_t)i * (uint64_t)n + (uint64_t)i);
        col[2 * i + 1] = 0.0;
      } else {
        double x, y;
        gen_normal2(seed, stream, (uint64_t)i * (uint64_t)n + (uint64_t)j, &x, &y);
        col[2 * i] = s * x;
        col[2 * i + 1] = s * y;
      }
    }
  }
}
