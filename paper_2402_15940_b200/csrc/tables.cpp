// tables.cpp -- 1D Gauss-Lobatto-Legendre basis and quadrature tables (SURVEY.md
// §8(a) row a2; SPEC.md:111-164 for the conventions: reference interval [0,1],
// B[k][i] = l_i(t_k), G[k][i] = l_i'(t_k)).  Host code, long double, written
// independently of the oracle: GLL nodes by Newton on P_{p+1} - P_{p-1}
// (whose roots are +-1 and the roots of P_p'), Gauss points by Newton on P_Q,
// and the Lagrange basis in barycentric form.
#include <math.h>
#include <string.h>

#include "internal.h"

namespace hofem {

namespace {

const long double kPi = 3.141592653589793238462643383279502884L;

// P_n(x) and P_n'(x) for n >= 0 by the Bonnet recurrence on (value, derivative).
void legendre_pd(int n, long double x, long double* P, long double* dP) {
  long double p0 = 1.0L, p1 = x, d0 = 0.0L, d1 = 1.0L;
  if (n == 0) { *P = 1.0L; *dP = 0.0L; return; }
  for (int k = 2; k <= n; ++k) {
    long double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
    long double d2 = d0 + (2 * k - 1) * p1;  // P_k' = P_{k-2}' + (2k-1) P_{k-1}
    p0 = p1; p1 = p2; d0 = d1; d1 = d2;
  }
  *P = p1; *dP = d1;
}

long double legendre(int n, long double x) {
  long double P, dP;
  legendre_pd(n, x, &P, &dP);
  return P;
}

}  // namespace

void gll_nodes_weights(int p, double* xo, double* wo) {
  long double x[kMaxQ + 1];
  for (int i = 0; i <= p; ++i) {
    // Newton on f = P_{p+1} - P_{p-1}, f' = (2p+1) P_p; start from Chebyshev-Lobatto.
    long double s = -cosl(kPi * i / p);
    if (i > 0 && i < p) {
      for (int it = 0; it < 60; ++it) {
        long double f = legendre(p + 1, s) - legendre(p - 1, s);
        long double df = (2 * p + 1) * legendre(p, s);
        long double ds = f / df;
        s -= ds;
        if (fabsl(ds) <= 1e-20L) break;
      }
    }
    x[i] = s;
  }
  for (int i = 0; i <= p; ++i) {
    long double Pp = legendre(p, x[i]);
    xo[i] = (double)(0.5L * (x[i] + 1.0L));
    wo[i] = (double)(1.0L / (p * (p + 1.0L) * Pp * Pp));  // 2/(p(p+1)P^2) halved for [0,1]
  }
  xo[0] = 0.0;
  xo[p] = 1.0;
}

static void gauss_points_weights(int q, double* xo, double* wo) {
  for (int i = 0; i < q; ++i) {
    long double s = cosl(kPi * (4.0L * (q - 1 - i) + 3.0L) / (4.0L * q + 2.0L));
    long double P = 0, dP = 1;
    for (int it = 0; it < 60; ++it) {
      legendre_pd(q, s, &P, &dP);
      long double ds = P / dP;
      s -= ds;
      if (fabsl(ds) <= 1e-20L) break;
    }
    legendre_pd(q, s, &P, &dP);
    xo[i] = (double)(0.5L * (s + 1.0L));
    wo[i] = (double)(1.0L / ((1.0L - s * s) * dP * dP));
  }
}

int build_tables(int p, int Q, int rule, Tables1D* T) {
  if (p < 1 || p > kMaxP || Q < 1 || Q > kMaxQ) return 1;
  memset(T, 0, sizeof(*T));
  T->p = p; T->Q = Q; T->rule = rule;
  double wn[kMaxQ + 1];
  gll_nodes_weights(p, T->xi, wn);
  if (rule == HOFEM_GAUSS) {
    gauss_points_weights(Q, T->t, T->w);
  } else if (rule == HOFEM_GLL) {
    if (Q < 2) return 1;
    gll_nodes_weights(Q - 1, T->t, T->w);
  } else {
    return 1;
  }
  const int P1 = p + 1;
  // barycentric weights lambda_i = 1 / prod_{j != i} (xi_i - xi_j)
  long double lam[kMaxP + 1];
  for (int i = 0; i < P1; ++i) {
    long double d = 1.0L;
    for (int j = 0; j < P1; ++j)
      if (j != i) d *= (long double)T->xi[i] - (long double)T->xi[j];
    lam[i] = 1.0L / d;
  }
  for (int k = 0; k < Q; ++k) {
    long double t = T->t[k];
    int hit = -1;
    for (int i = 0; i < P1; ++i)
      if (t == (long double)T->xi[i]) hit = i;
    if (hit >= 0) {
      // t is node k': l_i = delta, l_i' = (lam_i/lam_k')/(xi_k' - xi_i), diagonal by row-sum zero
      long double diag = 0.0L;
      for (int i = 0; i < P1; ++i) {
        T->B[k * P1 + i] = (i == hit) ? 1.0 : 0.0;
        if (i != hit) {
          long double v = (lam[i] / lam[hit]) / ((long double)T->xi[hit] - (long double)T->xi[i]);
          T->G[k * P1 + i] = (double)v;
          diag -= v;
        }
      }
      T->G[k * P1 + hit] = (double)diag;
    } else {
      long double den = 0.0L, s1 = 0.0L;
      long double li[kMaxP + 1];
      for (int i = 0; i < P1; ++i) {
        long double c = lam[i] / (t - (long double)T->xi[i]);
        li[i] = c;
        den += c;
      }
      for (int i = 0; i < P1; ++i) li[i] /= den;  // l_i(t)
      // l_i'(t) = l_i(t) * (sum_{j != i} 1/(t - xi_j))
      for (int j = 0; j < P1; ++j) s1 += 1.0L / (t - (long double)T->xi[j]);
      for (int i = 0; i < P1; ++i) {
        T->B[k * P1 + i] = (double)li[i];
        T->G[k * P1 + i] = (double)(li[i] * (s1 - 1.0L / (t - (long double)T->xi[i])));
      }
    }
  }
  return 0;
}

// DG (L2) basis of §8(f) f4 (reading R16): Lagrange polynomials on the p+1
// Gauss-Legendre points, evaluated at the Q Gauss quadrature points:
// B[k*P1+i] = psi_i(t_k) (barycentric form; psi_i(t_k) = delta when the point sets
// coincide, Q = P1).
int build_dg_table(int p, int Q, double* B) {
  if (p < 1 || p > kMaxP || Q < 1 || Q > kMaxQ) return 1;
  const int P1 = p + 1;
  double g[kMaxP + 1], gw[kMaxP + 1], t[kMaxQ], w[kMaxQ];
  gauss_points_weights(P1, g, gw);
  gauss_points_weights(Q, t, w);
  long double lam[kMaxP + 1];
  for (int i = 0; i < P1; ++i) {
    long double d = 1.0L;
    for (int j = 0; j < P1; ++j)
      if (j != i) d *= (long double)g[i] - (long double)g[j];
    lam[i] = 1.0L / d;
  }
  for (int k = 0; k < Q; ++k) {
    int hit = -1;
    for (int i = 0; i < P1; ++i)
      if (t[k] == g[i]) hit = i;
    long double den = 0.0L, li[kMaxP + 1];
    for (int i = 0; i < P1; ++i) {
      li[i] = hit >= 0 ? (i == hit ? 1.0L : 0.0L) : lam[i] / ((long double)t[k] - (long double)g[i]);
      den += li[i];
    }
    for (int i = 0; i < P1; ++i) B[k * P1 + i] = (double)(li[i] / den);
  }
  return 0;
}

}  // namespace hofem
