/* cartesian.c — ORACLE (test infrastructure only; see oracle.h). Plain FP64, no blocking.
 *
 * Cartesian Taylor expansions ("capability to switch to
 * Cartesian expansions ... key to achieving high performance for low-accuracy"). The paper
 * prints no formulas, so this follows the textbook Cartesian Taylor FMM (reading R17):
 *
 *   multi-index k = (kx, ky, kz), |k| = kx + ky + kz, k! = kx! ky! kz!, u^k = ux^kx uy^ky uz^kz,
 *   C(m, n) = prod_a binom(m_a, n_a),
 *   a_k(d) = (1/k!) d^k/dd^k (1/|d|)                                (normalised derivative tensor)
 *
 *   P2M  M_k    = sum_i q_i (y_i - c)^k                                    |k| <= p
 *   M2M  M_k(P) = sum_{j <= k} C(k, j) M_j(C) b^(k-j),       b = c_C - c_P  (exact)
 *   M2P  phi(x) = sum_k (-1)^|k| M_k a_k(x - c),  d_a phi = sum_k (-1)^|k| M_k (k_a + 1) a_{k+e_a}
 *   M2L  L_n    = sum_{|k| <= p - |n|} (-1)^|k| C(k + n, n) M_k a_{k+n}(c_t - c_s)   (total order p)
 *   L2L  L_n(C) = sum_{m >= n} C(m, n) L_m(P) e^(m-n),       e = c_C - c_P  (exact)
 *   L2P  phi(x) = sum_n L_n (x - c)^n,  d_a phi = sum_n L_n n_a (x - c)^(n - e_a)
 *
 * from 1/|x - y| = sum_k (-(y - c))^k / k! d^k(1/|.|)(x - c) (Taylor in the source point) and
 * L_n = (1/n!) d^n phi(c_t). The derivative tensor follows the recurrence (|n| >= 1)
 *   |n| |d|^2 a_n + (2|n| - 1) sum_a d_a a_{n - e_a} + (|n| - 1) sum_a a_{n - 2 e_a} = 0,
 * a_0 = 1/|d| (pinned against finite differences and closed forms in
 * tests/test_oracle_cartesian.py). Multi-indices are enumerated by order s = 0..P, then kx
 * descending, then ky descending.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

int orc_cart_count(int P) { return (P + 1) * (P + 2) * (P + 3) / 6; }

/* index of (kx, ky, kz) in the enumeration above */
int orc_cart_index(int kx, int ky, int kz) {
  const int s = kx + ky + kz;
  const int before = s * (s + 1) * (s + 2) / 6; /* multi-indices of order < s */
  const int rest = s - kx;                      /* ky + kz */
  /* within order s: kx descending (s .. 0), then ky descending (rest .. 0) */
  const int kx_before = (s - kx) * (s - kx + 1) / 2; /* indices with larger kx */
  return before + kx_before + (rest - ky);
}

void orc_cart_multi(int P, int *k3) {
  for (int s = 0; s <= P; ++s)
    for (int kx = s; kx >= 0; --kx)
      for (int ky = s - kx; ky >= 0; --ky) {
        const int i = orc_cart_index(kx, ky, s - kx - ky);
        k3[3 * i] = kx;
        k3[3 * i + 1] = ky;
        k3[3 * i + 2] = s - kx - ky;
      }
}

static double binom(int m, int n) {
  double b = 1.0;
  for (int i = 1; i <= n; ++i) b = b * (double)(m - n + i) / (double)i;
  return b;
}
static double ipow(double x, int e) {
  double r = 1.0;
  for (int i = 0; i < e; ++i) r *= x;
  return r;
}
static double mono(const double u[3], int kx, int ky, int kz) {
  return ipow(u[0], kx) * ipow(u[1], ky) * ipow(u[2], kz);
}

/* a_n(d) for |n| <= P, by the recurrence in the header */
void orc_cart_derivs(const double d[3], int P, double *a) {
  const double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
  a[0] = 1.0 / sqrt(r2);
  for (int s = 1; s <= P; ++s)
    for (int kx = s; kx >= 0; --kx)
      for (int ky = s - kx; ky >= 0; --ky) {
        const int kz = s - kx - ky;
        const int k[3] = {kx, ky, kz};
        double t1 = 0.0, t2 = 0.0;
        for (int ax = 0; ax < 3; ++ax) {
          int m[3] = {kx, ky, kz};
          if (k[ax] >= 1) {
            m[ax] -= 1;
            t1 += d[ax] * a[orc_cart_index(m[0], m[1], m[2])];
          }
          if (k[ax] >= 2) {
            m[ax] -= 1;
            t2 += a[orc_cart_index(m[0], m[1], m[2])];
          }
        }
        a[orc_cart_index(kx, ky, kz)] = -((2.0 * s - 1.0) * t1 + (s - 1.0) * t2) / (s * r2);
      }
}

void orc_cart_p2m(int p, const double c[3], int64_t n, const double *y, const double *q,
                  double *M) {
  const int nk = orc_cart_count(p);
  int *k3 = (int *)malloc(sizeof(int) * 3 * (size_t)nk);
  orc_cart_multi(p, k3);
  for (int64_t i = 0; i < n; ++i) {
    const double u[3] = {y[3 * i] - c[0], y[3 * i + 1] - c[1], y[3 * i + 2] - c[2]};
    for (int k = 0; k < nk; ++k) M[k] += q[i] * mono(u, k3[3 * k], k3[3 * k + 1], k3[3 * k + 2]);
  }
  free(k3);
}

void orc_cart_m2m(int p, const double *Mc, const double b[3], double *Mp) {
  const int nk = orc_cart_count(p);
  int *k3 = (int *)malloc(sizeof(int) * 3 * (size_t)nk);
  orc_cart_multi(p, k3);
  for (int k = 0; k < nk; ++k)
    for (int j = 0; j < nk; ++j) {
      const int *K = &k3[3 * k], *J = &k3[3 * j];
      if (J[0] > K[0] || J[1] > K[1] || J[2] > K[2]) continue;
      Mp[k] += binom(K[0], J[0]) * binom(K[1], J[1]) * binom(K[2], J[2]) * Mc[j] *
               mono(b, K[0] - J[0], K[1] - J[1], K[2] - J[2]);
    }
  free(k3);
}

void orc_cart_m2l(int p, const double *Ms, const double d[3], double *Lt) {
  const int nk = orc_cart_count(p);
  int *k3 = (int *)malloc(sizeof(int) * 3 * (size_t)nk);
  double *a = (double *)malloc(sizeof(double) * (size_t)nk);
  orc_cart_multi(p, k3);
  orc_cart_derivs(d, p, a);
  for (int n = 0; n < nk; ++n)
    for (int k = 0; k < nk; ++k) {
      const int *N = &k3[3 * n], *K = &k3[3 * k];
      const int sn = N[0] + N[1] + N[2], sk = K[0] + K[1] + K[2];
      if (sn + sk > p) continue;
      const double sg = (sk & 1) ? -1.0 : 1.0;
      Lt[n] += sg * binom(K[0] + N[0], N[0]) * binom(K[1] + N[1], N[1]) * binom(K[2] + N[2], N[2]) *
               Ms[k] * a[orc_cart_index(K[0] + N[0], K[1] + N[1], K[2] + N[2])];
    }
  free(a);
  free(k3);
}

void orc_cart_l2l(int p, const double *Lp, const double e[3], double *Lc) {
  const int nk = orc_cart_count(p);
  int *k3 = (int *)malloc(sizeof(int) * 3 * (size_t)nk);
  orc_cart_multi(p, k3);
  for (int n = 0; n < nk; ++n)
    for (int m = 0; m < nk; ++m) {
      const int *N = &k3[3 * n], *Mi = &k3[3 * m];
      if (Mi[0] < N[0] || Mi[1] < N[1] || Mi[2] < N[2]) continue;
      Lc[n] += binom(Mi[0], N[0]) * binom(Mi[1], N[1]) * binom(Mi[2], N[2]) * Lp[m] *
               mono(e, Mi[0] - N[0], Mi[1] - N[1], Mi[2] - N[2]);
    }
  free(k3);
}

void orc_cart_l2p(int p, const double *L, const double c[3], int64_t n, const double *x,
                  double *phi, double *grad) {
  const int nk = orc_cart_count(p);
  int *k3 = (int *)malloc(sizeof(int) * 3 * (size_t)nk);
  orc_cart_multi(p, k3);
  for (int64_t i = 0; i < n; ++i) {
    const double u[3] = {x[3 * i] - c[0], x[3 * i + 1] - c[1], x[3 * i + 2] - c[2]};
    for (int k = 0; k < nk; ++k) {
      const int *K = &k3[3 * k];
      phi[i] += L[k] * mono(u, K[0], K[1], K[2]);
      for (int ax = 0; ax < 3; ++ax) {
        if (K[ax] == 0) continue;
        int m[3] = {K[0], K[1], K[2]};
        m[ax] -= 1;
        grad[3 * i + ax] += L[k] * K[ax] * mono(u, m[0], m[1], m[2]);
      }
    }
  }
  free(k3);
}

void orc_cart_m2p(int p, const double *M, const double c[3], int64_t n, const double *x,
                  double *phi, double *grad) {
  const int nk = orc_cart_count(p), nk1 = orc_cart_count(p + 1);
  int *k3 = (int *)malloc(sizeof(int) * 3 * (size_t)nk);
  double *a = (double *)malloc(sizeof(double) * (size_t)nk1);
  orc_cart_multi(p, k3);
  for (int64_t i = 0; i < n; ++i) {
    const double d[3] = {x[3 * i] - c[0], x[3 * i + 1] - c[1], x[3 * i + 2] - c[2]};
    orc_cart_derivs(d, p + 1, a);
    for (int k = 0; k < nk; ++k) {
      const int *K = &k3[3 * k];
      const double sg = ((K[0] + K[1] + K[2]) & 1) ? -1.0 : 1.0;
      phi[i] += sg * M[k] * a[k];
      for (int ax = 0; ax < 3; ++ax) {
        int m[3] = {K[0], K[1], K[2]};
        m[ax] += 1;
        grad[3 * i + ax] += sg * M[k] * (K[ax] + 1) * a[orc_cart_index(m[0], m[1], m[2])];
      }
    }
  }
  free(a);
  free(k3);
}
