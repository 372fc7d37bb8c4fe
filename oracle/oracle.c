/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct FP64 CPU reference for the hot path of
 * arXiv 2402.15940 ("High-performance finite elements with MFEM"): the CEED
 * bake-off mass (BP1) and diffusion (BP3/BP5) operator actions on structured
 * curvilinear high-order hex meshes, and the CG solve built on them.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  The product (CUDA) path never
 * includes, links or calls anything here, and this file includes nothing from
 * the product: no shared headers, tables or helpers.
 *
 * What it computes, and the passage it follows:
 *   - The operator decomposition A = P^T G^T B^T D B G P (fig_feod,
 *     §3.5) is evaluated in its "Element Assembly" form (§2.2):
 *     every element matrix A_e is built by brute-force quadrature over the full
 *     tensor-product rule (sum over every quadrature point of products of full 3D
 *     basis functions), and y = sum_e R_e^T A_e R_e x.  No sum factorization
 *     anywhere.  Partial assembly computes exactly this operator
 *     up to rounding order, so this is the plain definition the GPU path must hit.
 *   - A second plain form, y_e = B_e^T D_e B_e x_e with B_e the DENSE (Q^3 x P1^3)
 *     basis-evaluation matrix, is used only where A_e would be
 *     too expensive to form (sampled parity at scale, p >= 6).  It is pinned to
 *     the EA form by tests/test_oracle_pins.py.
 *   - CG: textbook unpreconditioned Hestenes-Stiefel (§2.1 "Krylov
 *     subspace method").
 *   - §8(f) f4, DG (L2) mass: element matrices
 *     M_e = sum_q W detJ psi_a psi_b with the Gauss-Legendre-nodal basis (reading
 *     R16) by brute-force quadrature; the operator is block diagonal.
 *   - §8(f) f2, p-multigrid pieces: the assembled
 *     diagonal sum_e R_e^T diag(A_e), prolongation by evaluating the coarse
 *     element function at the fine nodes (owner element, product formula),
 *     restriction as its exact transpose, Chebyshev acceleration of Jacobi step
 *     by step (Saad, Alg. 12.1) and power iteration (readings R17-R18); the
 *     V-cycle and PCG are composed in oracle/__init__.py in the algorithm's order.
 *   - Readings for everything the paper leaves open (reference element [0,1]^3,
 *     quadrature rules, ordering, the deformation Phi, BCs, RHS) are SURVEY.md
 *     §8(c) R1-R14, restated in DESIGN.md §3.
 *
 * Rounding: FP64 round-to-nearest, compiled with -ffp-contract=off (no FMA
 * contraction, reading R10).  The 1D node/weight computation uses
 * long double Newton iterations.
 *
 * Parity pins: every exported function is pinned by a -m "not gpu" test in
 * tests/test_oracle_pins.py (closed forms, Kronecker structure, volume, K*1=0,
 * X_i^T K X_j identity, polynomial exactness, symmetry, CG closed forms,
 * O(h^{p+1}) convergence).  Nothing is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_MASS 1
#define ORC_DIFFUSION 2
#define ORC_GAUSS 1
#define ORC_GLL 2

#define ORC_MAXP1 17 /* p <= 16 */
#define ORC_MAXQ 24

static const long double PI_L = 3.141592653589793238462643383279502884L;

/* ------------------------------------------------------------------------- */
/* Mesh description (readings R1, R3, R4, R9).                      */
/* A window of a structured nx*ny*nz hex mesh of [0,Lx]x[0,Ly]x[0,Lz]: the     */
/* elements with ez in [z0, z0+nzl).  z0=0, nzl=nz is the whole mesh.          */
/* ------------------------------------------------------------------------- */
typedef struct {
  int nx, ny, nz, p;
  double L[3];
  double alpha; /* deformation amplitude of Phi, 0 => affine box */
  int z0, nzl;  /* element-layer window in z */
} orc_mesh;

/* ------------------------------------------------------------------------- */
/* 1D Legendre polynomials by the three-term recurrence, long double.         */
/* ------------------------------------------------------------------------- */
static void legendre(int n, long double s, long double *Pn, long double *Pnm1) {
  long double p0 = 1.0L, p1 = s;
  if (n == 0) { *Pn = 1.0L; *Pnm1 = 0.0L; return; }
  for (int k = 1; k < n; ++k) {
    long double p2 = ((2.0L * k + 1.0L) * s * p1 - (long double)k * p0) / (k + 1.0L);
    p0 = p1; p1 = p2;
  }
  *Pn = p1; *Pnm1 = p0;
}

/* GLL nodes/weights of degree p on [0,1]: endpoints plus the
 * roots of P_p' mapped from [-1,1]; weights 2/(p(p+1)P_p(s)^2), halved for [0,1]. */
int orc_gll(int p, double *nodes, double *weights) {
  if (p < 1 || p > ORC_MAXP1 - 1) return 1;
  long double s[ORC_MAXP1];
  s[0] = -1.0L; s[p] = 1.0L;
  for (int i = 1; i < p; ++i) {
    long double x = -cosl(PI_L * i / p); /* Chebyshev-Gauss-Lobatto guess */
    for (int it = 0; it < 100; ++it) {
      long double Pn, Pnm1;
      legendre(p, x, &Pn, &Pnm1);
      long double dP = p * (x * Pn - Pnm1) / (x * x - 1.0L);           /* P_p'  */
      long double d2P = (2.0L * x * dP - p * (p + 1.0L) * Pn) / (1.0L - x * x); /* P_p'' */
      long double dx = dP / d2P;
      x -= dx;
      if (fabsl(dx) < 1e-19L) break;
    }
    s[i] = x;
  }
  for (int i = 0; i <= p; ++i) {
    long double Pn, Pnm1;
    legendre(p, s[i], &Pn, &Pnm1);
    long double w = 2.0L / (p * (p + 1.0L) * Pn * Pn);
    nodes[i] = (double)((s[i] + 1.0L) / 2.0L);
    weights[i] = (double)(w / 2.0L);
  }
  nodes[0] = 0.0; nodes[p] = 1.0; /* exact endpoints (R4) */
  return 0;
}

/* Gauss-Legendre rule with q points on [0,1]: roots of P_q,
 * weights 2/((1-s^2) P_q'(s)^2), halved for [0,1]. */
int orc_gauss(int q, double *pts, double *wts) {
  if (q < 1 || q > ORC_MAXQ) return 1;
  for (int i = 0; i < q; ++i) {
    long double x = -cosl(PI_L * (i + 0.75L) / (q + 0.5L)); /* ascending guess */
    long double dP = 1.0L;
    for (int it = 0; it < 100; ++it) {
      long double Pn, Pnm1;
      legendre(q, x, &Pn, &Pnm1);
      dP = q * (x * Pn - Pnm1) / (x * x - 1.0L);
      long double dx = Pn / dP;
      x -= dx;
      if (fabsl(dx) < 1e-19L) break;
    }
    long double Pn, Pnm1;
    legendre(q, x, &Pn, &Pnm1);
    dP = q * (x * Pn - Pnm1) / (x * x - 1.0L);
    pts[i] = (double)((x + 1.0L) / 2.0L);
    wts[i] = (double)(1.0L / ((1.0L - x * x) * dP * dP));
  }
  return 0;
}

/* Lagrange basis on the GLL nodes xi[0..p], by the product formula. */
static double lagrange(int p, const double *xi, int i, double t) {
  double v = 1.0;
  for (int j = 0; j <= p; ++j)
    if (j != i) v *= (t - xi[j]) / (xi[i] - xi[j]);
  return v;
}
/* Its derivative: sum over the dropped factor k of the remaining product. */
static double lagrange_d(int p, const double *xi, int i, double t) {
  double s = 0.0;
  for (int k = 0; k <= p; ++k) {
    if (k == i) continue;
    double v = 1.0 / (xi[i] - xi[k]);
    for (int j = 0; j <= p; ++j)
      if (j != i && j != k) v *= (t - xi[j]) / (xi[i] - xi[j]);
    s += v;
  }
  return s;
}

/* 1D quadrature rule of the operator (reading R2): Gauss with Q points, or GLL
 * with Q points (Q = p+1 is collocated with the nodes). */
static int rule_1d(int rule, int Q, double *t, double *w) {
  if (rule == ORC_GAUSS) return orc_gauss(Q, t, w);
  if (rule == ORC_GLL) return Q >= 2 ? orc_gll(Q - 1, t, w) : 1;
  return 1;
}

/* B1d[k][i] = l_i(t_k), G1d[k][i] = l_i'(t_k), Q x (p+1). */
int orc_tabulate(int p, int Q, int rule, double *B, double *G) {
  double xi[ORC_MAXP1], wn[ORC_MAXP1], t[ORC_MAXQ], w[ORC_MAXQ];
  if (orc_gll(p, xi, wn) || rule_1d(rule, Q, t, w)) return 1;
  for (int k = 0; k < Q; ++k)
    for (int i = 0; i <= p; ++i) {
      B[k * (p + 1) + i] = lagrange(p, xi, i, t[k]);
      G[k * (p + 1) + i] = lagrange_d(p, xi, i, t[k]);
    }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Geometry: lattice points and the deformation Phi (reading R4).             */
/* ------------------------------------------------------------------------- */
static long long lat_n(const orc_mesh *m, int axis) {
  int n = axis == 0 ? m->nx : axis == 1 ? m->ny : m->nz;
  return (long long)m->p * n + 1;
}

/* Reference-cube coordinate of global lattice index I on an axis with n elements:
 * element e = floor(I/p), local node a = I mod p (the last lattice point is node p
 * of element n-1), u = (e + xi_a)/n. */
static double lattice_u(int I, int p, int n, const double *xi) {
  int e = I / p, a = I % p;
  if (e == n) { e = n - 1; a = p; }
  return ((double)e + xi[a]) / (double)n;
}

/* Phi(u)_i = u_i + alpha * s(u) * cos(pi u_{(i+1) mod 3}),
 * s(u) = sin(pi u_0) sin(pi u_1) sin(pi u_2); physical X_i = L_i * Phi(u)_i. */
static void phi_map(const orc_mesh *m, const double u[3], double X[3]) {
  const double pi = 3.14159265358979323846;
  double s = sin(pi * u[0]) * sin(pi * u[1]) * sin(pi * u[2]);
  for (int i = 0; i < 3; ++i)
    X[i] = m->L[i] * (u[i] + m->alpha * s * cos(pi * u[(i + 1) % 3]));
}

static void lattice_point(const orc_mesh *m, const double *xi, long long I, long long J,
                          long long K, double X[3]) {
  double u[3] = {lattice_u((int)I, m->p, m->nx, xi), lattice_u((int)J, m->p, m->ny, xi),
                 lattice_u((int)K, m->p, m->nz, xi)};
  phi_map(m, u, X);
}

/* Local (window) lattice sizes: planes K in [p*z0, p*(z0+nzl)]. */
static void local_dims(const orc_mesh *m, long long *Nx, long long *Ny, long long *Nz) {
  *Nx = lat_n(m, 0); *Ny = lat_n(m, 1); *Nz = (long long)m->p * m->nzl + 1;
}

long long orc_num_dofs(const orc_mesh *m) {
  long long Nx, Ny, Nz; local_dims(m, &Nx, &Ny, &Nz);
  return Nx * Ny * Nz;
}
long long orc_num_elems(const orc_mesh *m) { return (long long)m->nx * m->ny * m->nzl; }

/* Nodal coordinates of the window's L-vector, by component: xyz[c*N + l]. */
int orc_mesh_coords(const orc_mesh *m, double *xyz) {
  double xi[ORC_MAXP1], wn[ORC_MAXP1];
  if (orc_gll(m->p, xi, wn)) return 1;
  long long Nx, Ny, Nz; local_dims(m, &Nx, &Ny, &Nz);
  long long N = Nx * Ny * Nz;
  for (long long K = 0; K < Nz; ++K)
    for (long long J = 0; J < Ny; ++J)
      for (long long I = 0; I < Nx; ++I) {
        double X[3];
        lattice_point(m, xi, I, J, K + (long long)m->p * m->z0, X);
        long long l = I + Nx * (J + Ny * K);
        xyz[l] = X[0]; xyz[N + l] = X[1]; xyz[2 * N + l] = X[2];
      }
  return 0;
}

/* Element restriction R_e ("G" there): local dof
 * alpha=(a,b,c) (a fastest) of element e=(ex,ey,ez) -> window L-index. */
static long long l_index(const orc_mesh *m, long long e, int a, int b, int c) {
  long long Nx = lat_n(m, 0), Ny = lat_n(m, 1);
  long long ex = e % m->nx, ey = (e / m->nx) % m->ny, ez = e / ((long long)m->nx * m->ny);
  long long I = (long long)m->p * ex + a, J = (long long)m->p * ey + b,
            K = (long long)m->p * ez + c;
  return I + Nx * (J + Ny * K);
}

/* Essential (Dirichlet) dofs: the boundary of the GLOBAL lattice (reading R6). */
int orc_boundary_mask(const orc_mesh *m, uint8_t *mask) {
  long long Nx, Ny, Nz; local_dims(m, &Nx, &Ny, &Nz);
  long long NzG = lat_n(m, 2);
  for (long long K = 0; K < Nz; ++K)
    for (long long J = 0; J < Ny; ++J)
      for (long long I = 0; I < Nx; ++I) {
        long long KG = K + (long long)m->p * m->z0;
        mask[I + Nx * (J + Ny * K)] =
            (I == 0 || I == Nx - 1 || J == 0 || J == Ny - 1 || KG == 0 || KG == NzG - 1);
      }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Per-element quadrature data.                                               */
/* ------------------------------------------------------------------------- */
typedef struct {
  int p, P1, Q, nd, nq; /* nd = P1^3 element dofs, nq = Q^3 points */
  double xi[ORC_MAXP1];
  double t[ORC_MAXQ], w[ORC_MAXQ];
  double *phi;  /* [nq][nd] phi_alpha(xi_q) */
  double *dphi; /* [nq][3][nd] reference gradient of phi_alpha at xi_q */
} orc_basis;

/* Full 3D basis phi_alpha(xi) = l_a(xi_1) l_b(xi_2) l_c(xi_3) and its reference
 * gradient, evaluated at every quadrature point directly from the Lagrange
 * product formula (no tensor contraction of any kind). */
static int basis_build(orc_basis *bs, int p, int rule, int Q) {
  double wn[ORC_MAXP1];
  if (p < 1 || p >= ORC_MAXP1 || Q < 1 || Q > ORC_MAXQ) return 1;
  bs->p = p; bs->P1 = p + 1; bs->Q = Q;
  bs->nd = bs->P1 * bs->P1 * bs->P1; bs->nq = Q * Q * Q;
  if (orc_gll(p, bs->xi, wn) || rule_1d(rule, Q, bs->t, bs->w)) return 1;
  bs->phi = (double *)malloc(sizeof(double) * bs->nq * bs->nd);
  bs->dphi = (double *)malloc(sizeof(double) * bs->nq * 3 * bs->nd);
  if (!bs->phi || !bs->dphi) return 1;
  for (int qz = 0; qz < Q; ++qz)
    for (int qy = 0; qy < Q; ++qy)
      for (int qx = 0; qx < Q; ++qx) {
        int q = qx + Q * (qy + Q * qz);
        for (int c = 0; c <= p; ++c)
          for (int b = 0; b <= p; ++b)
            for (int a = 0; a <= p; ++a) {
              int al = a + bs->P1 * (b + bs->P1 * c);
              double la = lagrange(p, bs->xi, a, bs->t[qx]);
              double lb = lagrange(p, bs->xi, b, bs->t[qy]);
              double lc = lagrange(p, bs->xi, c, bs->t[qz]);
              double da = lagrange_d(p, bs->xi, a, bs->t[qx]);
              double db = lagrange_d(p, bs->xi, b, bs->t[qy]);
              double dc = lagrange_d(p, bs->xi, c, bs->t[qz]);
              bs->phi[(long long)q * bs->nd + al] = la * lb * lc;
              bs->dphi[((long long)q * 3 + 0) * bs->nd + al] = da * lb * lc;
              bs->dphi[((long long)q * 3 + 1) * bs->nd + al] = la * db * lc;
              bs->dphi[((long long)q * 3 + 2) * bs->nd + al] = la * lb * dc;
            }
      }
  return 0;
}
static void basis_free(orc_basis *bs) { free(bs->phi); free(bs->dphi); }

/* Nodal coordinates X_alpha of element e (isoparametric, geom order p). */
static void element_nodes(const orc_mesh *m, const orc_basis *bs, long long e, double *X) {
  long long ex = e % m->nx, ey = (e / m->nx) % m->ny, ez = e / ((long long)m->nx * m->ny);
  int P1 = bs->P1;
  for (int c = 0; c <= m->p; ++c)
    for (int b = 0; b <= m->p; ++b)
      for (int a = 0; a <= m->p; ++a) {
        int al = a + P1 * (b + P1 * c);
        double Xp[3];
        lattice_point(m, bs->xi, (long long)m->p * ex + a, (long long)m->p * ey + b,
                      (long long)m->p * (ez + m->z0) + c, Xp);
        X[3 * al + 0] = Xp[0]; X[3 * al + 1] = Xp[1]; X[3 * al + 2] = Xp[2];
      }
}

/* J_ij(xi_q) = d x_i / d xi_j = sum_alpha X_alpha,i * d phi_alpha / d xi_j. */
static void jacobian(const orc_basis *bs, const double *X, int q, double J[3][3]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int al = 0; al < bs->nd; ++al)
        s += X[3 * al + i] * bs->dphi[((long long)q * 3 + j) * bs->nd + al];
      J[i][j] = s;
    }
}

/* Pointwise D at one quadrature point ("D"; "essential
 * data at quadrature points"): mass W*detJ; diffusion the symmetric
 * W * adj(J) adj(J)^T / detJ, entries [00,01,02,11,12,22] (reading R3).
 * Returns detJ. */
static double point_data(const orc_basis *bs, const double *X, int q, int kind, double *D) {
  double J[3][3];
  jacobian(bs, X, q, J);
  /* adj(J) = cofactor^T: adj[i][j] = C[j][i], C = cofactor matrix */
  double adj[3][3];
  adj[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  adj[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
  adj[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
  adj[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  adj[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
  adj[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
  adj[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  adj[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
  adj[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  double det = J[0][0] * adj[0][0] + J[0][1] * adj[1][0] + J[0][2] * adj[2][0];
  int Q = bs->Q;
  int qx = q % Q, qy = (q / Q) % Q, qz = q / (Q * Q);
  double W = bs->w[qx] * bs->w[qy] * bs->w[qz];
  if (kind == ORC_MASS) {
    D[0] = W * det;
  } else {
    double M[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double s = 0.0;
        for (int k = 0; k < 3; ++k) s += adj[i][k] * adj[j][k];
        M[i][j] = W * s / det;
      }
    D[0] = M[0][0]; D[1] = M[0][1]; D[2] = M[0][2];
    D[3] = M[1][1]; D[4] = M[1][2]; D[5] = M[2][2];
  }
  return det;
}

static int ncomp(int kind) { return kind == ORC_MASS ? 1 : 6; }

/* qdata of the whole window, layout [E][n_c][Q^3] (reading R3).  Returns 2 if
 * detJ <= 0 anywhere. */
int orc_qdata(const orc_mesh *m, int kind, int rule, int Q, double *qd) {
  orc_basis bs;
  if (basis_build(&bs, m->p, rule, Q)) return 1;
  long long E = orc_num_elems(m);
  int nc = ncomp(kind), bad = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
  for (long long e = 0; e < E; ++e) {
    double *X = (double *)malloc(sizeof(double) * 3 * bs.nd);
    element_nodes(m, &bs, e, X);
    for (int q = 0; q < bs.nq; ++q) {
      double D[6];
      if (point_data(&bs, X, q, kind, D) <= 0.0) bad = 1;
      for (int c = 0; c < nc; ++c) qd[(e * nc + c) * bs.nq + q] = D[c];
    }
    free(X);
  }
  basis_free(&bs);
  return bad ? 2 : 0;
}

/* Element matrix by brute-force quadrature ("Element Assembly"):
 *   mass:      A[al][be] = sum_q W_q detJ_q phi_al(xi_q) phi_be(xi_q)
 *   diffusion: A[al][be] = sum_q gradphi_al(xi_q)^T D_q gradphi_be(xi_q)      */
static int element_matrix(const orc_mesh *m, const orc_basis *bs, int kind, long long e,
                          double *A) {
  int nd = bs->nd, bad = 0;
  double *X = (double *)malloc(sizeof(double) * 3 * nd);
  double *h = (double *)malloc(sizeof(double) * 3 * nd);
  element_nodes(m, bs, e, X);
  memset(A, 0, sizeof(double) * nd * nd);
  for (int q = 0; q < bs->nq; ++q) {
    double D[6];
    if (point_data(bs, X, q, kind, D) <= 0.0) bad = 1;
    if (kind == ORC_MASS) {
      const double *ph = bs->phi + (long long)q * nd;
      for (int al = 0; al < nd; ++al)
        for (int be = 0; be < nd; ++be) A[(long long)al * nd + be] += D[0] * ph[al] * ph[be];
    } else {
      const double *g = bs->dphi + (long long)q * 3 * nd;
      const double Dm[3][3] = {{D[0], D[1], D[2]}, {D[1], D[3], D[4]}, {D[2], D[4], D[5]}};
      for (int be = 0; be < nd; ++be) /* h_be = D grad phi_be */
        for (int i = 0; i < 3; ++i)
          h[i * nd + be] = Dm[i][0] * g[be] + Dm[i][1] * g[nd + be] + Dm[i][2] * g[2 * nd + be];
      for (int al = 0; al < nd; ++al)
        for (int be = 0; be < nd; ++be)
          A[(long long)al * nd + be] +=
              g[al] * h[be] + g[nd + al] * h[nd + be] + g[2 * nd + al] * h[2 * nd + be];
    }
  }
  free(X); free(h);
  return bad;
}

/* All element matrices of the window: Ae[E][nd][nd]. */
int orc_element_matrices(const orc_mesh *m, int kind, int rule, int Q, double *Ae) {
  orc_basis bs;
  if (basis_build(&bs, m->p, rule, Q)) return 1;
  long long E = orc_num_elems(m);
  long long nd2 = (long long)bs.nd * bs.nd;
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
  for (long long e = 0; e < E; ++e) bad |= element_matrix(m, &bs, kind, e, Ae + e * nd2);
  basis_free(&bs);
  return bad ? 2 : 0;
}

/* Dirichlet convention (reading R6): z = x; z[ess] = 0;
 * y = A z; y[ess] = x[ess]. */
static void bc_pre(const orc_mesh *m, int bc, const double *x, double *z) {
  long long N = orc_num_dofs(m);
  memcpy(z, x, sizeof(double) * N);
  if (!bc) return;
  uint8_t *mask = (uint8_t *)malloc(N);
  orc_boundary_mask(m, mask);
  for (long long l = 0; l < N; ++l) if (mask[l]) z[l] = 0.0;
  free(mask);
}
static void bc_post(const orc_mesh *m, int bc, const double *x, double *y) {
  if (!bc) return;
  long long N = orc_num_dofs(m);
  uint8_t *mask = (uint8_t *)malloc(N);
  orc_boundary_mask(m, mask);
  for (long long l = 0; l < N; ++l) if (mask[l]) y[l] = x[l];
  free(mask);
}

/* y_e = A_e R_e z per element (parallel), then y = sum_e R_e^T y_e in ascending
 * (e, alpha) order (serial, deterministic). */
static void scatter_fixed_order(const orc_mesh *m, int nd, const double *ye, double *y) {
  long long E = orc_num_elems(m), N = orc_num_dofs(m);
  int P1 = m->p + 1;
  memset(y, 0, sizeof(double) * N);
  for (long long e = 0; e < E; ++e)
    for (int c = 0; c < P1; ++c)
      for (int b = 0; b < P1; ++b)
        for (int a = 0; a < P1; ++a) {
          int al = a + P1 * (b + P1 * c);
          y[l_index(m, e, a, b, c)] += ye[e * nd + al];
        }
  (void)nd;
}

/* y = sum_e R_e^T A_e R_e x (with optional Dirichlet convention). */
int orc_apply_ea(const orc_mesh *m, const double *Ae, int bc, const double *x, double *y) {
  long long E = orc_num_elems(m), N = orc_num_dofs(m);
  int P1 = m->p + 1, nd = P1 * P1 * P1;
  long long nd2 = (long long)nd * nd;
  double *z = (double *)malloc(sizeof(double) * N);
  double *ye = (double *)malloc(sizeof(double) * E * nd);
  bc_pre(m, bc, x, z);
#pragma omp parallel for schedule(static)
  for (long long e = 0; e < E; ++e) {
    double xe[ORC_MAXP1 * ORC_MAXP1 * ORC_MAXP1];
    for (int c = 0; c < P1; ++c)
      for (int b = 0; b < P1; ++b)
        for (int a = 0; a < P1; ++a) xe[a + P1 * (b + P1 * c)] = z[l_index(m, e, a, b, c)];
    const double *A = Ae + e * nd2;
    for (int al = 0; al < nd; ++al) {
      double s = 0.0;
      for (int be = 0; be < nd; ++be) s += A[al * nd + be] * xe[be];
      ye[e * nd + al] = s;
    }
  }
  scatter_fixed_order(m, nd, ye, y);
  bc_post(m, bc, x, y);
  free(z); free(ye);
  return 0;
}

/* Dense-B form for one element: y_e = B_e^T (D_e (B_e x_e)), with B_e the dense
 * Q^3 x P1^3 basis-evaluation matrix (values for mass, reference gradients for
 * diffusion) -- the "B^T D B" of PAPER.md:595 with B written out as a dense
 * matrix (no tensor-product factorization). */
static int element_apply_dense(const orc_mesh *m, const orc_basis *bs, int kind, long long e,
                               const double *xe, double *ye) {
  int nd = bs->nd, bad = 0;
  double *X = (double *)malloc(sizeof(double) * 3 * nd);
  element_nodes(m, bs, e, X);
  for (int al = 0; al < nd; ++al) ye[al] = 0.0;
  for (int q = 0; q < bs->nq; ++q) {
    double D[6];
    if (point_data(bs, X, q, kind, D) <= 0.0) bad = 1;
    if (kind == ORC_MASS) {
      const double *ph = bs->phi + (long long)q * nd;
      double u = 0.0;
      for (int be = 0; be < nd; ++be) u += ph[be] * xe[be];
      double v = D[0] * u;
      for (int al = 0; al < nd; ++al) ye[al] += ph[al] * v;
    } else {
      const double *g = bs->dphi + (long long)q * 3 * nd;
      double gu[3] = {0.0, 0.0, 0.0};
      for (int be = 0; be < nd; ++be)
        for (int i = 0; i < 3; ++i) gu[i] += g[i * nd + be] * xe[be];
      double w0 = D[0] * gu[0] + D[1] * gu[1] + D[2] * gu[2];
      double w1 = D[1] * gu[0] + D[3] * gu[1] + D[4] * gu[2];
      double w2 = D[2] * gu[0] + D[4] * gu[1] + D[5] * gu[2];
      for (int al = 0; al < nd; ++al) ye[al] += g[al] * w0 + g[nd + al] * w1 + g[2 * nd + al] * w2;
    }
  }
  free(X);
  return bad;
}

/* y = sum_e R_e^T B_e^T D_e B_e R_e x, whole window (dense-B form). */
int orc_apply_dense(const orc_mesh *m, int kind, int rule, int Q, int bc, const double *x,
                    double *y) {
  orc_basis bs;
  if (basis_build(&bs, m->p, rule, Q)) return 1;
  long long E = orc_num_elems(m), N = orc_num_dofs(m);
  int P1 = m->p + 1, nd = bs.nd, bad = 0;
  double *z = (double *)malloc(sizeof(double) * N);
  double *ye = (double *)malloc(sizeof(double) * E * nd);
  bc_pre(m, bc, x, z);
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
  for (long long e = 0; e < E; ++e) {
    double xe[ORC_MAXP1 * ORC_MAXP1 * ORC_MAXP1];
    for (int c = 0; c < P1; ++c)
      for (int b = 0; b < P1; ++b)
        for (int a = 0; a < P1; ++a) xe[a + P1 * (b + P1 * c)] = z[l_index(m, e, a, b, c)];
    bad |= element_apply_dense(m, &bs, kind, e, xe, ye + e * nd);
  }
  scatter_fixed_order(m, nd, ye, y);
  bc_post(m, bc, x, y);
  free(z); free(ye); basis_free(&bs);
  return bad ? 2 : 0;
}

/* Sampled parity at scale (SURVEY.md §8(c) "Parity at scale"): for each listed
 * element e, y_e = B_e^T D_e B_e R_e x (no Dirichlet; x is the window L-vector).
 * Output ye[k][nd]. */
int orc_element_apply_sample(const orc_mesh *m, int kind, int rule, int Q, const double *x,
                             long long n, const long long *elems, double *ye) {
  orc_basis bs;
  if (basis_build(&bs, m->p, rule, Q)) return 1;
  int P1 = m->p + 1, nd = bs.nd, bad = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
  for (long long k = 0; k < n; ++k) {
    double xe[ORC_MAXP1 * ORC_MAXP1 * ORC_MAXP1];
    long long e = elems[k];
    for (int c = 0; c < P1; ++c)
      for (int b = 0; b < P1; ++b)
        for (int a = 0; a < P1; ++a) xe[a + P1 * (b + P1 * c)] = x[l_index(m, e, a, b, c)];
    bad |= element_apply_dense(m, &bs, kind, e, xe, ye + k * nd);
  }
  basis_free(&bs);
  return bad ? 2 : 0;
}

/* Dense global matrix A = sum_e R_e^T A_e R_e (tiny meshes only; the "Sparse
 * Matrix Assembly" level of PAPER.md:148 stored densely, used as a pin). */
int orc_assemble_dense(const orc_mesh *m, const double *Ae, double *A) {
  long long E = orc_num_elems(m), N = orc_num_dofs(m);
  int P1 = m->p + 1, nd = P1 * P1 * P1;
  long long idx[ORC_MAXP1 * ORC_MAXP1 * ORC_MAXP1];
  memset(A, 0, sizeof(double) * N * N);
  for (long long e = 0; e < E; ++e) {
    for (int c = 0; c < P1; ++c)
      for (int b = 0; b < P1; ++b)
        for (int a = 0; a < P1; ++a) idx[a + P1 * (b + P1 * c)] = l_index(m, e, a, b, c);
    for (int al = 0; al < nd; ++al)
      for (int be = 0; be < nd; ++be)
        A[idx[al] * N + idx[be]] += Ae[(e * nd + al) * nd + be];
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Right-hand side and error (reading R11).                                   */
/* ------------------------------------------------------------------------- */
static double u_exact(const double X[3]) {
  const double pi = 3.14159265358979323846;
  return sin(pi * X[0]) * sin(pi * X[1]) * sin(pi * X[2]);
}

/* b_i = sum_e sum_q W_q detJ f(x(xi_q)) phi_i(xi_q), x(xi) = sum_al X_al phi_al(xi).
 * BP3/BP5 (kind=DIFFUSION): f = 3 pi^2 u, BP1 (MASS): f = u.  bc=1 zeroes b[ess]. */
int orc_rhs(const orc_mesh *m, int kind, int rule, int Q, int bc, double *b) {
  const double pi = 3.14159265358979323846;
  orc_basis bs;
  if (basis_build(&bs, m->p, rule, Q)) return 1;
  long long E = orc_num_elems(m), N = orc_num_dofs(m);
  int nd = bs.nd, P1 = bs.P1;
  double *be = (double *)malloc(sizeof(double) * E * nd);
#pragma omp parallel for schedule(dynamic, 1)
  for (long long e = 0; e < E; ++e) {
    double *X = (double *)malloc(sizeof(double) * 3 * nd);
    element_nodes(m, &bs, e, X);
    for (int al = 0; al < nd; ++al) be[e * nd + al] = 0.0;
    for (int q = 0; q < bs.nq; ++q) {
      double D[6];
      point_data(&bs, X, q, ORC_MASS, D); /* W * detJ */
      const double *ph = bs.phi + (long long)q * nd;
      double xq[3] = {0.0, 0.0, 0.0};
      for (int al = 0; al < nd; ++al)
        for (int i = 0; i < 3; ++i) xq[i] += X[3 * al + i] * ph[al];
      double f = u_exact(xq);
      if (kind == ORC_DIFFUSION) f *= 3.0 * pi * pi;
      for (int al = 0; al < nd; ++al) be[e * nd + al] += D[0] * f * ph[al];
    }
    free(X);
  }
  scatter_fixed_order(m, nd, be, b);
  if (bc) {
    uint8_t *mask = (uint8_t *)malloc(N);
    orc_boundary_mask(m, mask);
    for (long long l = 0; l < N; ++l) if (mask[l]) b[l] = 0.0;
    free(mask);
  }
  free(be); basis_free(&bs);
  (void)P1;
  return 0;
}

/* || u_h - u ||_{L2(Omega)} with an over-integrated Gauss rule of Qover points. */
double orc_l2_error(const orc_mesh *m, const double *uh, int Qover) {
  orc_basis bs;
  if (basis_build(&bs, m->p, ORC_GAUSS, Qover)) return -1.0;
  long long E = orc_num_elems(m);
  int P1 = bs.P1, nd = bs.nd;
  double total = 0.0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : total)
  for (long long e = 0; e < E; ++e) {
    double *X = (double *)malloc(sizeof(double) * 3 * nd);
    double ue[ORC_MAXP1 * ORC_MAXP1 * ORC_MAXP1];
    element_nodes(m, &bs, e, X);
    for (int c = 0; c < P1; ++c)
      for (int b = 0; b < P1; ++b)
        for (int a = 0; a < P1; ++a) ue[a + P1 * (b + P1 * c)] = uh[l_index(m, e, a, b, c)];
    double s = 0.0;
    for (int q = 0; q < bs.nq; ++q) {
      double D[6];
      point_data(&bs, X, q, ORC_MASS, D);
      const double *ph = bs.phi + (long long)q * nd;
      double xq[3] = {0.0, 0.0, 0.0}, v = 0.0;
      for (int al = 0; al < nd; ++al) {
        for (int i = 0; i < 3; ++i) xq[i] += X[3 * al + i] * ph[al];
        v += ue[al] * ph[al];
      }
      double d = v - u_exact(xq);
      s += D[0] * d * d;
    }
    total += s;
    free(X);
  }
  basis_free(&bs);
  return sqrt(total);
}

/* ------------------------------------------------------------------------- */
/* DG (L2) mass, SURVEY.md §8(f) f4 (§2.4.1 "matrix-free    */
/* discontinuous Galerkin"; fig:dgpa-perf "DG mass operators").               */
/* Space: discontinuous Q_p per element with the nodal basis at the p+1 Gauss- */
/* Legendre points (reading R16: MFEM's default L2 basis); geometry = the H1   */
/* mesh's isoparametric map (element_nodes).  No inter-element coupling, so   */
/* the operator is block diagonal: y_e = M_e x_e with                          */
/*   M_e[al][be] = sum_q W_q detJ_q psi_al(xi_q) psi_be(xi_q)                  */
/* by brute-force quadrature (Gauss Q points, reading R2).  DG vectors are    */
/* element-major [E][P1^3], x fastest inside an element (reading R16).         */
/* ------------------------------------------------------------------------- */
/* psi[q][al] = psi_a(t_qx) psi_b(t_qy) psi_c(t_qz), psi = Lagrange on the P1
 * Gauss-Legendre points (product formula). */
static double *dg_basis(const orc_basis *bs) {
  int p = bs->p, P1 = bs->P1, nd = bs->nd, Q = bs->Q;
  double gn[ORC_MAXP1], gw[ORC_MAXP1];
  if (orc_gauss(P1, gn, gw)) return NULL;
  double *psi = (double *)malloc(sizeof(double) * bs->nq * nd);
  for (int qz = 0; qz < Q; ++qz)
    for (int qy = 0; qy < Q; ++qy)
      for (int qx = 0; qx < Q; ++qx) {
        int q = qx + Q * (qy + Q * qz);
        for (int c = 0; c <= p; ++c)
          for (int b = 0; b <= p; ++b)
            for (int a = 0; a <= p; ++a)
              psi[(long long)q * nd + a + P1 * (b + P1 * c)] =
                  lagrange(p, gn, a, bs->t[qx]) * lagrange(p, gn, b, bs->t[qy]) *
                  lagrange(p, gn, c, bs->t[qz]);
      }
  return psi;
}

/* M_e[al][be] = sum_q W_q detJ_q psi_al psi_be (brute force). */
static int dg_element_matrix(const orc_mesh *m, const orc_basis *bs, const double *psi,
                             long long e, double *A) {
  int nd = bs->nd, bad = 0;
  double *X = (double *)malloc(sizeof(double) * 3 * nd);
  element_nodes(m, bs, e, X);
  memset(A, 0, sizeof(double) * nd * nd);
  for (int q = 0; q < bs->nq; ++q) {
    double D[6];
    if (point_data(bs, X, q, ORC_MASS, D) <= 0.0) bad = 1;
    const double *ps = psi + (long long)q * nd;
    for (int al = 0; al < nd; ++al)
      for (int be = 0; be < nd; ++be) A[(long long)al * nd + be] += D[0] * ps[al] * ps[be];
  }
  free(X);
  return bad;
}

int orc_dg_mass_matrices(const orc_mesh *m, int Q, double *Me) {
  orc_basis bs; /* geometry (GLL nodes) and the quadrature rule */
  if (basis_build(&bs, m->p, ORC_GAUSS, Q)) return 1;
  double *psi = dg_basis(&bs);
  if (!psi) { basis_free(&bs); return 1; }
  long long E = orc_num_elems(m), nd2 = (long long)bs.nd * bs.nd;
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
  for (long long e = 0; e < E; ++e) bad |= dg_element_matrix(m, &bs, psi, e, Me + e * nd2);
  free(psi);
  basis_free(&bs);
  return bad ? 2 : 0;
}

/* Sampled DG parity at scale: y_e = M_e x_e for the listed elements only
 * (x is the whole E-vector; ye[k] holds element elems[k]). */
int orc_dg_apply_sample(const orc_mesh *m, int Q, const double *x, long long nel,
                        const long long *elems, double *ye) {
  orc_basis bs;
  if (basis_build(&bs, m->p, ORC_GAUSS, Q)) return 1;
  double *psi = dg_basis(&bs);
  if (!psi) { basis_free(&bs); return 1; }
  int nd = bs.nd, bad = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
  for (long long k = 0; k < nel; ++k) {
    double *A = (double *)malloc(sizeof(double) * nd * nd);
    long long e = elems[k];
    bad |= dg_element_matrix(m, &bs, psi, e, A);
    for (int al = 0; al < nd; ++al) {
      double s = 0.0;
      for (int be = 0; be < nd; ++be) s += A[(long long)al * nd + be] * x[e * nd + be];
      ye[k * nd + al] = s;
    }
    free(A);
  }
  free(psi);
  basis_free(&bs);
  return bad ? 2 : 0;
}

/* y_e = M_e x_e for every element (block-diagonal DG operator). */
int orc_dg_apply(const orc_mesh *m, const double *Me, const double *x, double *y) {
  long long E = orc_num_elems(m);
  int P1 = m->p + 1, nd = P1 * P1 * P1;
#pragma omp parallel for schedule(static)
  for (long long e = 0; e < E; ++e) {
    const double *A = Me + e * (long long)nd * nd;
    for (int al = 0; al < nd; ++al) {
      double s = 0.0;
      for (int be = 0; be < nd; ++be) s += A[(long long)al * nd + be] * x[e * nd + be];
      y[e * nd + al] = s;
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* CG (reading R7).                             */
/* ------------------------------------------------------------------------- */
static double dot(long long n, const double *a, const double *b) {
  double s = 0.0;
  for (long long i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* Operator = EA matvec (Ae != NULL) or a dense N x N matrix (Adense != NULL).
 * Returns 0 converged, 6 breakdown (p^T A p <= 0), 7 max_iter reached.
 * x: in x0, out solution.  rr_hist (len max_iter+1) and x_hist (len
 * (max_iter+1)*N) are optional; *iters = number of iterations performed. */
int orc_cg(const orc_mesh *m, const double *Ae, int bc, const double *Adense, long long N,
           const double *b, double *x, double rel_tol, int max_iter, int fixed_iters,
           double *rr_hist, double *x_hist, int *iters) {
  if (m) N = orc_num_dofs(m);
  double *r = (double *)malloc(sizeof(double) * N);
  double *pv = (double *)malloc(sizeof(double) * N);
  double *Ap = (double *)malloc(sizeof(double) * N);
#define APPLY(in, out)                                                          \
  do {                                                                          \
    if (Adense) {                                                               \
      for (long long i_ = 0; i_ < N; ++i_) (out)[i_] = dot(N, Adense + i_ * N, (in)); \
    } else {                                                                    \
      orc_apply_ea(m, Ae, bc, (in), (out));                                     \
    }                                                                           \
  } while (0)
  APPLY(x, Ap);
  for (long long i = 0; i < N; ++i) { r[i] = b[i] - Ap[i]; pv[i] = r[i]; }
  double rr = dot(N, r, r), rr0 = rr;
  if (rr_hist) rr_hist[0] = rr;
  if (x_hist) memcpy(x_hist, x, sizeof(double) * N);
  int k = 0, status = 7;
  if (rr == 0.0) status = 0;
  while (status == 7 && k < max_iter) {
    APPLY(pv, Ap);
    double pAp = dot(N, pv, Ap);
    if (pAp <= 0.0) { status = 6; break; }
    double alpha = rr / pAp;
    for (long long i = 0; i < N; ++i) { x[i] += alpha * pv[i]; r[i] -= alpha * Ap[i]; }
    double rrn = dot(N, r, r);
    ++k;
    if (rr_hist) rr_hist[k] = rrn;
    if (x_hist) memcpy(x_hist + (long long)k * N, x, sizeof(double) * N);
    if (!fixed_iters && (rrn == 0.0 || sqrt(rrn) <= rel_tol * sqrt(rr0))) { status = 0; break; }
    double beta = rrn / rr;
    for (long long i = 0; i < N; ++i) pv[i] = r[i] + beta * pv[i];
    rr = rrn;
  }
#undef APPLY
  if (fixed_iters && status == 7 && k == max_iter) status = 0;
  *iters = k;
  free(r); free(pv); free(Ap);
  return status;
}

/* ------------------------------------------------------------------------- */
/* p-multigrid preconditioned CG pieces, SURVEY.md §8(f) f2 (*/
/* §2.1: "p-multigrid ... restriction and prolongation operators ... smoothers */
/* based only on the diagonal of the matrix ... Chebyshev acceleration";       */
/* PAPER.md:156 BPS3).  Readings R17-R18.                       */
/* ------------------------------------------------------------------------- */

/* diag(A) = sum_e R_e^T diag(A_e) (ascending e); Dirichlet rows of the
 * identity-row convention (reading R6) get 1. */
int orc_diagonal(const orc_mesh *m, const double *Ae, int bc, double *d) {
  long long E = orc_num_elems(m), N = orc_num_dofs(m);
  int P1 = m->p + 1, nd = P1 * P1 * P1;
  memset(d, 0, sizeof(double) * N);
  for (long long e = 0; e < E; ++e)
    for (int c = 0; c < P1; ++c)
      for (int b = 0; b < P1; ++b)
        for (int a = 0; a < P1; ++a) {
          int al = a + P1 * (b + P1 * c);
          d[l_index(m, e, a, b, c)] += Ae[e * (long long)nd * nd + (long long)al * nd + al];
        }
  if (bc) {
    uint8_t *mask = (uint8_t *)malloc(N);
    orc_boundary_mask(m, mask);
    for (long long l = 0; l < N; ++l) if (mask[l]) d[l] = 1.0;
    free(mask);
  }
  return 0;
}

/* Owner element of a lattice index along one axis (lowest element containing it)
 * and the local node index there. */
static void owner_axis(long long I, int p, int n, long long *e, int *a) {
  long long q = I / p;
  if (q > n - 1) q = n - 1;
  *e = q;
  *a = (int)(I - (long long)p * q);
}

/* Coarse-to-fine interpolation weights of fine lattice point (I,J,K): its owner
 * element e and the values phi^c_alpha(xi) of the coarse element basis at the
 * fine node's reference coordinate (GLL nodes of both orders, product formula). */
static long long transfer_weights(const orc_mesh *mf, const orc_mesh *mc, long long I, long long J,
                                  long long K, double *w) {
  double xf[ORC_MAXP1], xc[ORC_MAXP1], wt[ORC_MAXP1];
  orc_gll(mf->p, xf, wt);
  orc_gll(mc->p, xc, wt);
  long long ex, ey, ez;
  int a, b, c;
  owner_axis(I, mf->p, mf->nx, &ex, &a);
  owner_axis(J, mf->p, mf->ny, &ey, &b);
  owner_axis(K, mf->p, mf->nzl, &ez, &c);
  int P1c = mc->p + 1;
  for (int gc = 0; gc < P1c; ++gc)
    for (int gb = 0; gb < P1c; ++gb)
      for (int ga = 0; ga < P1c; ++ga)
        w[ga + P1c * (gb + P1c * gc)] = lagrange(mc->p, xc, ga, xf[a]) *
                                        lagrange(mc->p, xc, gb, xf[b]) *
                                        lagrange(mc->p, xc, gc, xf[c]);
  return ex + (long long)mf->nx * (ey + (long long)mf->ny * ez);
}

/* Prolongation P (order mc->p -> mf->p, same elements): the fine nodal value is
 * the coarse finite-element function evaluated at the fine node (the natural
 * injection of the nested spaces). */
int orc_prolong(const orc_mesh *mf, const orc_mesh *mc, const double *xc, double *xf) {
  long long Nx, Ny, Nz;
  local_dims(mf, &Nx, &Ny, &Nz);
  int P1c = mc->p + 1;
  double w[ORC_MAXP1 * ORC_MAXP1 * ORC_MAXP1];
  for (long long K = 0; K < Nz; ++K)
    for (long long J = 0; J < Ny; ++J)
      for (long long I = 0; I < Nx; ++I) {
        long long e = transfer_weights(mf, mc, I, J, K, w);
        double s = 0.0;
        for (int gc = 0; gc < P1c; ++gc)
          for (int gb = 0; gb < P1c; ++gb)
            for (int ga = 0; ga < P1c; ++ga)
              s += w[ga + P1c * (gb + P1c * gc)] * xc[l_index(mc, e, ga, gb, gc)];
        xf[I + Nx * (J + Ny * K)] = s;
      }
  return 0;
}

/* Restriction R = P^T: rc[j] = sum_i P_ij rf[i], looping over fine points i with
 * the same owner element and weights as orc_prolong (so R is exactly P^T). */
int orc_restrict(const orc_mesh *mf, const orc_mesh *mc, const double *rf, double *rc) {
  long long Nx, Ny, Nz;
  local_dims(mf, &Nx, &Ny, &Nz);
  int P1c = mc->p + 1;
  memset(rc, 0, sizeof(double) * orc_num_dofs(mc));
  double w[ORC_MAXP1 * ORC_MAXP1 * ORC_MAXP1];
  for (long long K = 0; K < Nz; ++K)
    for (long long J = 0; J < Ny; ++J)
      for (long long I = 0; I < Nx; ++I) {
        long long e = transfer_weights(mf, mc, I, J, K, w);
        double v = rf[I + Nx * (J + Ny * K)];
        for (int gc = 0; gc < P1c; ++gc)
          for (int gb = 0; gb < P1c; ++gb)
            for (int ga = 0; ga < P1c; ++ga)
              rc[l_index(mc, e, ga, gb, gc)] += w[ga + P1c * (gb + P1c * gc)] * v;
      }
  return 0;
}

/* Largest eigenvalue estimate of D^{-1}A by power iteration (reading R17):
 * v = v0/|v0|; iters times: w = D^{-1} A v, lambda = |w|, v = w/lambda. */
double orc_power_lmax(const orc_mesh *m, const double *Ae, int bc, const double *dinv,
                      const double *v0, int iters) {
  long long N = orc_num_dofs(m);
  double *v = (double *)malloc(sizeof(double) * N), *w = (double *)malloc(sizeof(double) * N);
  double nv = sqrt(dot(N, v0, v0)), lam = 0.0;
  for (long long i = 0; i < N; ++i) v[i] = v0[i] / nv;
  for (int k = 0; k < iters; ++k) {
    orc_apply_ea(m, Ae, bc, v, w);
    for (long long i = 0; i < N; ++i) w[i] *= dinv[i];
    lam = sqrt(dot(N, w, w));
    for (long long i = 0; i < N; ++i) v[i] = w[i] / lam;
  }
  free(v); free(w);
  return lam;
}

/* Chebyshev acceleration of Jacobi (Saad, "Iterative Methods for Sparse Linear
 * Systems", Algorithm 12.1, preconditioner D = diag(A)), `degree` >= 1 steps on
 * the interval [lmin, lmax] of D^{-1}A, starting from x (updated in place):
 *   r = b - A x; theta = (lmax+lmin)/2; delta = (lmax-lmin)/2; sigma = theta/delta
 *   rho = 1/sigma; d = D^{-1} r / theta
 *   for k = 1..degree: x += d; if k < degree: r -= A d;
 *       rho' = 1/(2 sigma - rho); d = rho' rho d + (2 rho'/delta) D^{-1} r; rho = rho' */
int orc_cheb(const orc_mesh *m, const double *Ae, int bc, const double *dinv, double lmin,
             double lmax, int degree, const double *b, double *x) {
  long long N = orc_num_dofs(m);
  double *r = (double *)malloc(sizeof(double) * N), *d = (double *)malloc(sizeof(double) * N);
  double *Ad = (double *)malloc(sizeof(double) * N);
  orc_apply_ea(m, Ae, bc, x, Ad);
  for (long long i = 0; i < N; ++i) r[i] = b[i] - Ad[i];
  double theta = 0.5 * (lmax + lmin), delta = 0.5 * (lmax - lmin), sigma = theta / delta;
  double rho = 1.0 / sigma;
  for (long long i = 0; i < N; ++i) d[i] = dinv[i] * r[i] / theta;
  for (int k = 1; k <= degree; ++k) {
    for (long long i = 0; i < N; ++i) x[i] += d[i];
    if (k == degree) break;
    orc_apply_ea(m, Ae, bc, d, Ad);
    for (long long i = 0; i < N; ++i) r[i] -= Ad[i];
    double rn = 1.0 / (2.0 * sigma - rho);
    for (long long i = 0; i < N; ++i) d[i] = rn * rho * d[i] + (2.0 * rn / delta) * dinv[i] * r[i];
    rho = rn;
  }
  free(r); free(d); free(Ad);
  return 0;
}

void orc_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n > 0 ? n : 1);
#else
  (void)n;
#endif
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
