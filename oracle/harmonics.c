/* harmonics.c — ORACLE (test infrastructure only; see oracle.h). Plain FP64, no blocking.
 *
 * PAPER.md:60 says the kernels use "spherical harmonic expansions" and PAPER.md:205 says the
 * cell-cell kernel is O(p^4); the paper prints no formulas, so the oracle follows the convention
 * fixed in SURVEY.md §8(c) c6 (DESIGN.md §3 reading R1):
 *
 *   R_n^m(x) = r^n P_n^m(cos t) e^{i m f} / (n+m)!       (regular solid harmonic)
 *   I_n^m(x) = (n-m)! P_n^m(cos t) e^{i m f} / r^{n+1}   (irregular solid harmonic)
 *   1/|x-y|  = sum_{n,m} conj(R_n^m(y)) I_n^m(x),  |y| < |x|
 *
 * both evaluated with the trig-free recurrences of c6 (pinned against scipy's associated
 * Legendre functions in tests/test_oracle_harmonics.py).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* R_n^m for n = 0..P, m = -n..n (c6 recurrences, then R_n^{-m} = (-1)^m conj(R_n^m)). */
void orc_harm_R(const double x[3], int P, cplx *R) {
  const double r2 = x[0] * x[0] + x[1] * x[1] + x[2] * x[2];
  const cplx w = x[0] + I * x[1];
  const double z = x[2];
  memset(R, 0, sizeof(cplx) * (size_t)(P + 1) * (P + 1));
  for (int m = 0; m <= P; ++m) {
    if (m == 0)
      R[ORC_IDX(0, 0)] = 1.0;
    else
      R[ORC_IDX(m, m)] = -w / (2.0 * m) * R[ORC_IDX(m - 1, m - 1)];
    if (m + 1 <= P) R[ORC_IDX(m + 1, m)] = z * R[ORC_IDX(m, m)];
    for (int n = m + 2; n <= P; ++n)
      R[ORC_IDX(n, m)] = ((2.0 * n - 1.0) * z * R[ORC_IDX(n - 1, m)] - r2 * R[ORC_IDX(n - 2, m)]) /
                         ((double)(n - m) * (double)(n + m));
  }
  for (int n = 1; n <= P; ++n)
    for (int m = 1; m <= n; ++m) R[ORC_IDX(n, -m)] = ((m & 1) ? -1.0 : 1.0) * conj(R[ORC_IDX(n, m)]);
}

/* I_n^m for n = 0..P, m = -n..n (c6 recurrences, then I_n^{-m} = (-1)^m conj(I_n^m)). */
void orc_harm_I(const double x[3], int P, cplx *Iv) {
  const double r2 = x[0] * x[0] + x[1] * x[1] + x[2] * x[2];
  const double r = sqrt(r2);
  const cplx w = x[0] + I * x[1];
  const double z = x[2];
  memset(Iv, 0, sizeof(cplx) * (size_t)(P + 1) * (P + 1));
  for (int m = 0; m <= P; ++m) {
    if (m == 0)
      Iv[ORC_IDX(0, 0)] = 1.0 / r;
    else
      Iv[ORC_IDX(m, m)] = -(2.0 * m - 1.0) * w / r2 * Iv[ORC_IDX(m - 1, m - 1)];
    if (m + 1 <= P) Iv[ORC_IDX(m + 1, m)] = (2.0 * m + 1.0) * z / r2 * Iv[ORC_IDX(m, m)];
    for (int n = m + 2; n <= P; ++n)
      Iv[ORC_IDX(n, m)] = ((2.0 * n - 1.0) * z * Iv[ORC_IDX(n - 1, m)] -
                           (double)(n + m - 1) * (double)(n - m - 1) * Iv[ORC_IDX(n - 2, m)]) /
                          r2;
  }
  for (int n = 1; n <= P; ++n)
    for (int m = 1; m <= n; ++m)
      Iv[ORC_IDX(n, -m)] = ((m & 1) ? -1.0 : 1.0) * conj(Iv[ORC_IDX(n, m)]);
}

static cplx *scratch(int P) { return (cplx *)malloc(sizeof(cplx) * (size_t)(P + 1) * (P + 1)); }

/* P2M: M_n^m += sum_i q_i conj(R_n^m(y_i - c)). */
void orc_p2m(int p, const double c[3], int64_t n, const double *y, const double *q, cplx *M) {
  cplx *R = scratch(p);
  for (int64_t i = 0; i < n; ++i) {
    const double d[3] = {y[3 * i] - c[0], y[3 * i + 1] - c[1], y[3 * i + 2] - c[2]};
    orc_harm_R(d, p, R);
    for (int k = 0; k < (p + 1) * (p + 1); ++k) M[k] += q[i] * conj(R[k]);
  }
  free(R);
}

/* M2M: M_n^m(P) += sum_{j<=n,k} M_j^k(C) conj(R_{n-j}^{m-k}(b)),
 * b = c_child - c_parent.  (R addition theorem: exact.) */
void orc_m2m(int p, const cplx *Mc, const double b[3], cplx *Mp) {
  cplx *R = scratch(p);
  orc_harm_R(b, p, R);
  for (int n = 0; n <= p; ++n)
    for (int m = -n; m <= n; ++m) {
      cplx acc = 0;
      for (int j = 0; j <= n; ++j)
        for (int k = -j; k <= j; ++k) {
          const int dm = m - k;
          if (dm < -(n - j) || dm > n - j) continue;
          acc += Mc[ORC_IDX(j, k)] * conj(R[ORC_IDX(n - j, dm)]);
        }
      Mp[ORC_IDX(n, m)] += acc;
    }
  free(R);
}

/* M2L ("O(p^4) cell-cell kernel", SURVEY c6 and reading 3 = full truncation):
 * L_j^k += (-1)^{j+k} sum_{n<=p} sum_{|m|<=n} M_n^m I_{n+j}^{m-k}(d),  d = c_t - c_s. */
void orc_m2l(int p, const cplx *Ms, const double d[3], cplx *Lt) {
  cplx *Iv = scratch(2 * p);
  orc_harm_I(d, 2 * p, Iv);
  for (int j = 0; j <= p; ++j)
    for (int k = -j; k <= j; ++k) {
      cplx acc = 0;
      for (int n = 0; n <= p; ++n)
        for (int m = -n; m <= n; ++m) acc += Ms[ORC_IDX(n, m)] * Iv[ORC_IDX(n + j, m - k)];
      Lt[ORC_IDX(j, k)] += (((j + k) & 1) ? -1.0 : 1.0) * acc;
    }
  free(Iv);
}

/* L2L: L_n^m(C) += sum_{j>=n,k} L_j^k(P) R_{j-n}^{k-m}(e),
 * e = c_child - c_parent.  (Exact.) */
void orc_l2l(int p, const cplx *Lp, const double e[3], cplx *Lc) {
  cplx *R = scratch(p);
  orc_harm_R(e, p, R);
  for (int n = 0; n <= p; ++n)
    for (int m = -n; m <= n; ++m) {
      cplx acc = 0;
      for (int j = n; j <= p; ++j)
        for (int k = -j; k <= j; ++k) {
          const int dm = k - m;
          if (dm < -(j - n) || dm > j - n) continue;
          acc += Lp[ORC_IDX(j, k)] * R[ORC_IDX(j - n, dm)];
        }
      Lc[ORC_IDX(n, m)] += acc;
    }
  free(R);
}

/* L2P: phi += sum L_n^m R_n^m(x - c); gradient from the c6 identities
 * d/dz R_n^m = R_{n-1}^m and (d/dx + i d/dy) R_n^m = R_{n-1}^{m+1}. Accumulates (+=). */
void orc_l2p(int p, const cplx *L, const double c[3], int64_t n, const double *x, double *phi,
             double *grad) {
  cplx *R = scratch(p);
  for (int64_t i = 0; i < n; ++i) {
    const double d[3] = {x[3 * i] - c[0], x[3 * i + 1] - c[1], x[3 * i + 2] - c[2]};
    orc_harm_R(d, p, R);
    cplx ph = 0, gz = 0, gxy = 0;
    for (int nn = 0; nn <= p; ++nn)
      for (int m = -nn; m <= nn; ++m) {
        const cplx l = L[ORC_IDX(nn, m)];
        ph += l * R[ORC_IDX(nn, m)];
        if (nn >= 1) {
          if (m >= -(nn - 1) && m <= nn - 1) gz += l * R[ORC_IDX(nn - 1, m)];
          if (m + 1 >= -(nn - 1) && m + 1 <= nn - 1) gxy += l * R[ORC_IDX(nn - 1, m + 1)];
        }
      }
    phi[i] += creal(ph);
    grad[3 * i + 0] += creal(gxy);
    grad[3 * i + 1] += cimag(gxy);
    grad[3 * i + 2] += creal(gz);
  }
  free(R);
}

/* M2P: phi += sum M_n^m I_n^m(x - c); gradient from
 * d/dz I_n^m = -I_{n+1}^m and (d/dx + i d/dy) I_n^m = I_{n+1}^{m+1}. Accumulates (+=). */
void orc_m2p(int p, const cplx *M, const double c[3], int64_t n, const double *x, double *phi,
             double *grad) {
  cplx *Iv = scratch(p + 1);
  for (int64_t i = 0; i < n; ++i) {
    const double d[3] = {x[3 * i] - c[0], x[3 * i + 1] - c[1], x[3 * i + 2] - c[2]};
    orc_harm_I(d, p + 1, Iv);
    cplx ph = 0, gz = 0, gxy = 0;
    for (int nn = 0; nn <= p; ++nn)
      for (int m = -nn; m <= nn; ++m) {
        const cplx mm = M[ORC_IDX(nn, m)];
        ph += mm * Iv[ORC_IDX(nn, m)];
        gz -= mm * Iv[ORC_IDX(nn + 1, m)];
        gxy += mm * Iv[ORC_IDX(nn + 1, m + 1)];
      }
    phi[i] += creal(ph);
    grad[3 * i + 0] += creal(gxy);
    grad[3 * i + 1] += cimag(gxy);
    grad[3 * i + 2] += creal(gz);
  }
  free(Iv);
}

/* P2P ("direct summation"): phi_i += sum_j q_j/r_ij,
 * grad_i += -sum_j q_j (x_i - y_j)/r_ij^3; pairs with r = 0 contribute nothing (reading 13). */
void orc_p2p(int64_t nt, const double *xt, int64_t ns, const double *ys, const double *qs,
             double *phi, double *grad) {
  for (int64_t i = 0; i < nt; ++i) {
    double ph = 0, gx = 0, gy = 0, gz = 0;
    for (int64_t j = 0; j < ns; ++j) {
      const double dx = xt[3 * i] - ys[3 * j], dy = xt[3 * i + 1] - ys[3 * j + 1],
                   dz = xt[3 * i + 2] - ys[3 * j + 2];
      const double r2 = dx * dx + dy * dy + dz * dz;
      if (r2 == 0.0) continue;
      const double r = sqrt(r2);
      ph += qs[j] / r;
      const double f = qs[j] / (r2 * r);
      gx -= f * dx;
      gy -= f * dy;
      gz -= f * dz;
    }
    phi[i] += ph;
    grad[3 * i] += gx;
    grad[3 * i + 1] += gy;
    grad[3 * i + 2] += gz;
  }
}
