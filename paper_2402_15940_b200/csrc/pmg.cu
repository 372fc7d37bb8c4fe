// pmg.cu -- p-multigrid preconditioned CG, SURVEY.md §8(f) f2 (PAPER.md:103-111,
// §2.1: "p-multigrid ... restriction and prolongation operators ... computed
// efficiently on the GPU using sum-factorization techniques ... smoothers based
// only on the diagonal of the matrix; sum-factorization techniques provide
// algorithms to efficiently compute the diagonal ... Chebyshev acceleration";
// PAPER.md:156 BPS3).  Readings R17 (hierarchy, smoother, eigen estimate) and R18
// (PCG), DESIGN.md §3.
//
//   diagonal   per element, sum-factorized over squared 1D tables:
//              diag_e[a,b,c] = sum_t coef_t sum_qz Z_t[qz][c] sum_qy Y_t[qy][b]
//                              sum_qx X_t[qx][a] D_t[qx,qy,qz]
//              (t over D00 (GG,BB,BB), D11, D22, 2 D01 (GB,GB,BB), 2 D02, 2 D12;
//              mass: D (BB,BB,BB)), then the deterministic transposed-offset
//              scatter; Dirichlet rows 1 (identity-row convention, reading R6).
//   transfers  prolongation = nodal interpolation of the coarse finite-element
//              function (1D table I[f][c] = l^{pc}_c(xi^{pf}_f), three tensor
//              contractions per element, each fine node written once by its owner
//              element); restriction = its transpose (per element: fine values
//              divided by their multiplicity, transposed contractions, transposed-
//              offset scatter onto the coarse lattice; coarse Dirichlet rows 0).
//   smoother   Chebyshev acceleration of Jacobi (Saad Alg. 12.1) on
//              [0.3 * 1.2 lam, 1.2 lam], lam from power iteration on D^-1 A.
//   V-cycle    pre-smooth, residual, restrict, recurse, prolong-correct,
//              post-smooth; the coarsest level (p = 1) is smoothed twice.
//   PCG        Hestenes-Stiefel PCG with one V-cycle as the preconditioner.
// Single rank.  Every level applies its operator with the fused brick kernel.
#include <math.h>
#include <string.h>

#include <vector>

#include "internal.h"

namespace hofem {

namespace {

inline unsigned grid_for(long long n, int bs) { return (unsigned)((n + bs - 1) / bs); }

// ---------------------------------------------------------------- diagonal
__device__ __forceinline__ double tab1(const double* B, const double* G, int kind, int idx) {
  const double b = B[idx], g = G[idx];
  return kind == 0 ? b * b : (kind == 1 ? g * g : g * b);  // 0 BB, 1 GG, 2 GB
}

__global__ void diag_elem_kernel(int P1, int Q, int mass, const double* __restrict__ qdata,
                                 const double* __restrict__ dB, const double* __restrict__ dG,
                                 double* __restrict__ ediag) {
  extern __shared__ double sm[];
  const int nq = Q * Q * Q, nd = P1 * P1 * P1, nc = mass ? 1 : 6;
  double* B = sm;
  double* G = B + Q * P1;
  double* D = G + Q * P1;     // nc * Q^3
  double* U = D + nc * nq;    // [a][qy][qz]
  double* V = U + P1 * Q * Q; // [a][b][qz]
  double* acc = V + P1 * P1 * Q;
  const long long e = blockIdx.x;
  for (int i = threadIdx.x; i < Q * P1; i += blockDim.x) { B[i] = dB[i]; G[i] = dG[i]; }
  for (int i = threadIdx.x; i < nc * nq; i += blockDim.x) D[i] = qdata[e * nc * nq + i];
  for (int i = threadIdx.x; i < nd; i += blockDim.x) acc[i] = 0.0;
  __syncthreads();
  // terms: D component, X / Y / Z table kinds, coefficient
  const int comp[6] = {0, 3, 5, 1, 2, 4};
  const int kx[6] = {1, 0, 0, 2, 2, 0}, ky[6] = {0, 1, 0, 2, 0, 2}, kz[6] = {0, 0, 1, 0, 2, 2};
  const double coef[6] = {1.0, 1.0, 1.0, 2.0, 2.0, 2.0};
  const int nterms = mass ? 1 : 6;
  for (int t = 0; t < nterms; ++t) {
    const double* Dt = D + (mass ? 0 : comp[t]) * nq;
    const int X = mass ? 0 : kx[t], Y = mass ? 0 : ky[t], Z = mass ? 0 : kz[t];
    for (int i = threadIdx.x; i < P1 * Q * Q; i += blockDim.x) {
      const int a = i / (Q * Q), r = i % (Q * Q);  // r = qy + Q qz
      double s = 0.0;
      for (int qx = 0; qx < Q; ++qx) s += tab1(B, G, X, qx * P1 + a) * Dt[qx + Q * r];
      U[i] = s;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < P1 * P1 * Q; i += blockDim.x) {
      const int a = i / (P1 * Q), b = (i / Q) % P1, qz = i % Q;
      double s = 0.0;
      for (int qy = 0; qy < Q; ++qy) s += tab1(B, G, Y, qy * P1 + b) * U[a * Q * Q + qy + Q * qz];
      V[i] = s;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nd; i += blockDim.x) {
      const int a = i % P1, b = (i / P1) % P1, c = i / (P1 * P1);
      double s = 0.0;
      for (int qz = 0; qz < Q; ++qz) s += tab1(B, G, Z, qz * P1 + c) * V[(a * P1 + b) * Q + qz];
      acc[i] += coef[t] * s;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < nd; i += blockDim.x) ediag[e * nd + i] = acc[i];
}

__global__ void recip_kernel(long long n, const double* __restrict__ d, double* __restrict__ di) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) di[i] = 1.0 / d[i];
}

// ---------------------------------------------------------------- transfers
struct XferGeo {
  int nx, ny, nz;           // elements
  int pf, pc;               // orders
  long long Nxf, Nyf, Nzf;  // fine lattice
  long long Nxc, Nyc;       // coarse lattice
};

// xf += P xc (owner-element writes; deterministic, race-free)
__global__ void prolong_add_kernel(XferGeo g, const double* __restrict__ I1,
                                   const double* __restrict__ xc, double* __restrict__ xf) {
  extern __shared__ double sm[];
  const int Pf = g.pf + 1, Pc = g.pc + 1;
  double* I = sm;                 // [f][c]
  double* ce = I + Pf * Pc;       // [gc][gb][ga]
  double* T1 = ce + Pc * Pc * Pc; // [gc][gb][a]
  double* T2 = T1 + Pc * Pc * Pf; // [gc][b][a]
  const long long e = blockIdx.x;
  const int ex = (int)(e % g.nx), ey = (int)((e / g.nx) % g.ny), ez = (int)(e / ((long long)g.nx * g.ny));
  for (int i = threadIdx.x; i < Pf * Pc; i += blockDim.x) I[i] = I1[i];
  for (int i = threadIdx.x; i < Pc * Pc * Pc; i += blockDim.x) {
    const int ga = i % Pc, gb = (i / Pc) % Pc, gc = i / (Pc * Pc);
    ce[i] = xc[(long long)(g.pc * ex + ga) +
               g.Nxc * ((long long)(g.pc * ey + gb) + g.Nyc * (long long)(g.pc * ez + gc))];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < Pc * Pc * Pf; i += blockDim.x) {
    const int a = i % Pf, r = i / Pf;  // r = gb + Pc gc
    double s = 0.0;
    for (int ga = 0; ga < Pc; ++ga) s += I[a * Pc + ga] * ce[ga + Pc * r];
    T1[i] = s;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < Pc * Pf * Pf; i += blockDim.x) {
    const int a = i % Pf, b = (i / Pf) % Pf, gc = i / (Pf * Pf);
    double s = 0.0;
    for (int gb = 0; gb < Pc; ++gb) s += I[b * Pc + gb] * T1[a + Pf * (gb + Pc * gc)];
    T2[i] = s;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < Pf * Pf * Pf; i += blockDim.x) {
    const int a = i % Pf, b = (i / Pf) % Pf, c = i / (Pf * Pf);
    const bool own = (a < g.pf || ex == g.nx - 1) && (b < g.pf || ey == g.ny - 1) &&
                     (c < g.pf || ez == g.nz - 1);
    if (!own) continue;
    double s = 0.0;
    for (int gc = 0; gc < Pc; ++gc) s += I[c * Pc + gc] * T2[a + Pf * (b + Pf * gc)];
    xf[(long long)(g.pf * ex + a) +
       g.Nxf * ((long long)(g.pf * ey + b) + g.Nyf * (long long)(g.pf * ez + c))] += s;
  }
}

__device__ __forceinline__ int mult(long long I, int p, long long N) {
  return (I % p == 0 && I > 0 && I < N - 1) ? 2 : 1;
}

// ec[e] = I^T (rf_e / multiplicity) per element (coarse E-vector)
__global__ void restrict_elem_kernel(XferGeo g, const double* __restrict__ I1,
                                     const double* __restrict__ rf, double* __restrict__ ec) {
  extern __shared__ double sm[];
  const int Pf = g.pf + 1, Pc = g.pc + 1;
  double* I = sm;
  double* fe = I + Pf * Pc;       // [c][b][a]
  double* T1 = fe + Pf * Pf * Pf; // [c][b][ga]
  double* T2 = T1 + Pf * Pf * Pc; // [c][gb][ga]
  const long long e = blockIdx.x;
  const int ex = (int)(e % g.nx), ey = (int)((e / g.nx) % g.ny), ez = (int)(e / ((long long)g.nx * g.ny));
  for (int i = threadIdx.x; i < Pf * Pc; i += blockDim.x) I[i] = I1[i];
  for (int i = threadIdx.x; i < Pf * Pf * Pf; i += blockDim.x) {
    const int a = i % Pf, b = (i / Pf) % Pf, c = i / (Pf * Pf);
    const long long Ig = g.pf * ex + a, Jg = g.pf * ey + b, Kg = g.pf * ez + c;
    const int m = mult(Ig, g.pf, g.Nxf) * mult(Jg, g.pf, g.Nyf) * mult(Kg, g.pf, g.Nzf);
    fe[i] = rf[Ig + g.Nxf * (Jg + g.Nyf * Kg)] / (double)m;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < Pf * Pf * Pc; i += blockDim.x) {
    const int ga = i % Pc, r = i / Pc;  // r = b + Pf c
    double s = 0.0;
    for (int a = 0; a < Pf; ++a) s += I[a * Pc + ga] * fe[a + Pf * r];
    T1[i] = s;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < Pf * Pc * Pc; i += blockDim.x) {
    const int ga = i % Pc, gb = (i / Pc) % Pc, c = i / (Pc * Pc);
    double s = 0.0;
    for (int b = 0; b < Pf; ++b) s += I[b * Pc + gb] * T1[ga + Pc * (b + Pf * c)];
    T2[i] = s;
  }
  __syncthreads();
  const int ndc = Pc * Pc * Pc;
  for (int i = threadIdx.x; i < ndc; i += blockDim.x) {
    const int ga = i % Pc, gb = (i / Pc) % Pc, gc = i / (Pc * Pc);
    double s = 0.0;
    for (int c = 0; c < Pf; ++c) s += I[c * Pc + gc] * T2[ga + Pc * (gb + Pc * c)];
    ec[e * ndc + i] = s;
  }
}

// ---------------------------------------------------------------- vector kernels
// r = b - Ax (Ax may be null: x = 0); d = dinv r / theta
__global__ void cheb_init_kernel(long long n, const double* __restrict__ b,
                                 const double* __restrict__ Ax, const double* __restrict__ dinv,
                                 double* __restrict__ r, double* __restrict__ d, double inv_theta) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double ri = Ax ? b[i] - Ax[i] : b[i];
  r[i] = ri;
  d[i] = dinv[i] * ri * inv_theta;
}
// x += d; r -= Ad; d = c1 d + c2 dinv r
__global__ void cheb_step_kernel(long long n, double* __restrict__ x, double* __restrict__ r,
                                 double* __restrict__ d, const double* __restrict__ Ad,
                                 const double* __restrict__ dinv, double c1, double c2) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double di = d[i];
  x[i] += di;
  const double ri = r[i] - Ad[i];
  r[i] = ri;
  d[i] = c1 * di + c2 * dinv[i] * ri;
}
__global__ void axpy_kernel(long long n, double a, const double* __restrict__ x,
                            double* __restrict__ y) {  // y += a x
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) y[i] += a * x[i];
}
__global__ void scale_kernel(long long n, double a, const double* __restrict__ x,
                             double* __restrict__ y) {  // y = a x
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) y[i] = a * x[i];
}
__global__ void mul_kernel(long long n, const double* __restrict__ a, double* __restrict__ y) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) y[i] *= a[i];
}
__global__ void sub_kernel(long long n, const double* __restrict__ b, const double* __restrict__ a,
                           double* __restrict__ r) {  // r = b - a
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) r[i] = b[i] - a[i];
}
// x += alpha p; r -= alpha Ap
__global__ void pcg_update_kernel(long long n, double alpha, const double* __restrict__ p,
                                  const double* __restrict__ Ap, double* __restrict__ x,
                                  double* __restrict__ r) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  x[i] += alpha * p[i];
  r[i] -= alpha * Ap[i];
}
// p = z + beta p
__global__ void xpby_kernel(long long n, const double* __restrict__ z, double beta,
                            double* __restrict__ p) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) p[i] = z[i] + beta * p[i];
}

constexpr int kBS = 256;

}  // namespace

hofem_status apply_any(Op* op, const double* x, double* y, cudaStream_t s);

hofem_status op_diagonal(Op* op, double* d, cudaStream_t s) {
  Mesh* m = op->mesh;
  // (collocated BP5 qdata has the same [E][6][Q^3] layout, with B = I)
  const int P1 = m->P1, Q = op->Q, nd = P1 * P1 * P1, nc = op->nc;
  const long long ent = m->elems * nd;
  double* ed = nullptr;
  HOFEM_CUDA(cudaMallocAsync(&ed, sizeof(double) * (ent + 1), s));
  const size_t smem = sizeof(double) * (2 * Q * P1 + nc * Q * Q * Q + P1 * Q * Q + P1 * P1 * Q + nd);
  static size_t smem_set = 0;  // set once per size class, not per call
  if (smem > 48 * 1024 && smem > smem_set) {
    HOFEM_CUDA(cudaFuncSetAttribute(diag_elem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
    smem_set = smem;
  }
  if (m->elems > 0) {
    diag_elem_kernel<<<(unsigned)m->elems, 128, smem, s>>>(P1, Q, op->kind == HOFEM_MASS,
                                                           op->d_qdata, op->d_B, op->d_G, ed);
    HOFEM_LAUNCHED();
  }
  HOFEM_TRY(scatter_evector_bc(op, ed, d, op->bc ? 3 : 0, nullptr, s));
  HOFEM_TRY(exchange_planes_bc(op, nullptr, d, op->bc ? 3 : 0, s));
  HOFEM_CUDA(cudaFreeAsync(ed, s));
  return HOFEM_OK;
}

// ---------------------------------------------------------------- the hierarchy
struct PMGLevel {
  Mesh* mesh = nullptr;
  Op* op = nullptr;
  double* dinv = nullptr;
  double *b = nullptr, *x = nullptr, *r = nullptr, *d = nullptr, *t = nullptr;
  double* I1 = nullptr;  // interpolation from the NEXT (coarser) level: [P1 this][P1 coarse]
  double* ec = nullptr;  // coarse E-vector scratch of the restriction (next level)
  double lam = 0.0;
  long long n = 0;
};

struct PMG {
  Mesh* fine = nullptr;
  int degree = 3, power_iters = 10;
  unsigned long long seed = 1;
  std::vector<PMGLevel> L;  // L[0] finest
  double* pcg = nullptr;    // PCG vectors: r, z, p, Ap (4 * n0)
};

namespace {

double cheb_hi() { return 1.2; }
double cheb_lo() { return 0.3; }

hofem_status dot_host(Mesh* m, const double* a, const double* b, double* out, cudaStream_t s) {
  HOFEM_TRY(dot_device(m, a, b, m->d_scalars, s));
  return d2h(m, out, m->d_scalars, sizeof(double), s);
}

XferGeo xgeo(const PMGLevel& f, const PMGLevel& c) {
  XferGeo g;
  g.nx = f.mesh->nx; g.ny = f.mesh->ny; g.nz = f.mesh->nzl;
  g.pf = f.mesh->p; g.pc = c.mesh->p;
  g.Nxf = f.mesh->Nx; g.Nyf = f.mesh->Ny; g.Nzf = f.mesh->Nzl;
  g.Nxc = c.mesh->Nx; g.Nyc = c.mesh->Ny;
  return g;
}

// 1D interpolation table I[f][c] = l^{pc}_c(xi^{pf}_f) on the GLL nodes of both
// orders (barycentric form; exact 0/1 where the nodes coincide).
void interp_table(int pf, int pc, double* I) {
  double xf[kMaxP + 1], xc[kMaxP + 1], w[kMaxP + 1];
  gll_nodes_weights(pf, xf, w);
  gll_nodes_weights(pc, xc, w);
  long double lam[kMaxP + 1];
  for (int i = 0; i <= pc; ++i) {
    long double d = 1.0L;
    for (int j = 0; j <= pc; ++j)
      if (j != i) d *= (long double)xc[i] - (long double)xc[j];
    lam[i] = 1.0L / d;
  }
  for (int f = 0; f <= pf; ++f) {
    int hit = -1;
    for (int i = 0; i <= pc; ++i)
      if (xf[f] == xc[i]) hit = i;
    long double li[kMaxP + 1], den = 0.0L;
    for (int i = 0; i <= pc; ++i) {
      li[i] = hit >= 0 ? (i == hit ? 1.0L : 0.0L) : lam[i] / ((long double)xf[f] - (long double)xc[i]);
      den += li[i];
    }
    for (int i = 0; i <= pc; ++i) I[f * (pc + 1) + i] = (double)(li[i] / den);
  }
}

}  // namespace

hofem_status pmg_prolong_add(PMG* P, int k, const double* xc, double* xf, cudaStream_t s) {
  const PMGLevel &F = P->L[k], &C = P->L[k + 1];
  const XferGeo g = xgeo(F, C);
  const int Pf = g.pf + 1, Pc = g.pc + 1;
  const size_t smem = sizeof(double) * (Pf * Pc + Pc * Pc * Pc + Pc * Pc * Pf + Pc * Pf * Pf);
  prolong_add_kernel<<<(unsigned)F.mesh->elems, 128, smem, s>>>(g, F.I1, xc, xf);
  HOFEM_LAUNCHED();
  return HOFEM_OK;
}

hofem_status pmg_restrict(PMG* P, int k, const double* rf, double* rc, cudaStream_t s) {
  PMGLevel &F = P->L[k], &C = P->L[k + 1];
  const XferGeo g = xgeo(F, C);
  const int Pf = g.pf + 1, Pc = g.pc + 1;
  const size_t smem = sizeof(double) * (Pf * Pc + Pf * Pf * Pf + Pf * Pf * Pc + Pf * Pc * Pc);
  restrict_elem_kernel<<<(unsigned)F.mesh->elems, 128, smem, s>>>(g, F.I1, rf, F.ec);
  HOFEM_LAUNCHED();
  // coarse Dirichlet rows of the restricted residual are zero (reading R17)
  return scatter_evector_bc(C.op, F.ec, rc, 2, nullptr, s);
}

// One Chebyshev-Jacobi smoothing pass at level k: x <- x + p(D^-1 A) D^-1 (b - A x)
// (Saad Alg. 12.1, `degree` steps).  x_zero: x is known to be 0 (skips A x).
hofem_status pmg_smooth(PMG* P, int k, const double* b, double* x, bool x_zero, cudaStream_t s) {
  PMGLevel& V = P->L[k];
  const long long n = V.n;
  const double lmax = cheb_hi() * V.lam, lmin = cheb_lo() * lmax;
  const double theta = 0.5 * (lmax + lmin), delta = 0.5 * (lmax - lmin), sigma = theta / delta;
  double rho = 1.0 / sigma;
  if (!x_zero) HOFEM_TRY(apply_any(V.op, x, V.t, s));
  cheb_init_kernel<<<grid_for(n, kBS), kBS, 0, s>>>(n, b, x_zero ? nullptr : V.t, V.dinv, V.r, V.d,
                                                    1.0 / theta);
  HOFEM_LAUNCHED();
  for (int step = 1; step < P->degree; ++step) {
    HOFEM_TRY(apply_any(V.op, V.d, V.t, s));
    const double rn = 1.0 / (2.0 * sigma - rho);
    cheb_step_kernel<<<grid_for(n, kBS), kBS, 0, s>>>(n, x, V.r, V.d, V.t, V.dinv, rn * rho,
                                                      2.0 * rn / delta);
    HOFEM_LAUNCHED();
    rho = rn;
  }
  axpy_kernel<<<grid_for(n, kBS), kBS, 0, s>>>(n, 1.0, V.d, x);
  HOFEM_LAUNCHED();
  return HOFEM_OK;
}

// z = V-cycle(b) at level k (z overwritten)
hofem_status pmg_vcycle_level(PMG* P, int k, const double* b, double* z, cudaStream_t s) {
  PMGLevel& V = P->L[k];
  HOFEM_CUDA(cudaMemsetAsync(z, 0, sizeof(double) * V.n, s));
  HOFEM_TRY(pmg_smooth(P, k, b, z, true, s));
  if (k + 1 < (int)P->L.size()) {
    PMGLevel& C = P->L[k + 1];
    HOFEM_TRY(apply_any(V.op, z, V.t, s));
    sub_kernel<<<grid_for(V.n, kBS), kBS, 0, s>>>(V.n, b, V.t, V.r);
    HOFEM_LAUNCHED();
    HOFEM_TRY(pmg_restrict(P, k, V.r, C.b, s));
    HOFEM_TRY(pmg_vcycle_level(P, k + 1, C.b, C.x, s));
    HOFEM_TRY(pmg_prolong_add(P, k, C.x, z, s));
  }
  return pmg_smooth(P, k, b, z, false, s);
}

void pmg_destroy(PMG* P) {
  if (!P) return;
  for (size_t k = 0; k < P->L.size(); ++k) {
    PMGLevel& V = P->L[k];
    cudaFree(V.dinv); cudaFree(V.b); cudaFree(V.x); cudaFree(V.r); cudaFree(V.d); cudaFree(V.t);
    cudaFree(V.I1); cudaFree(V.ec);
    op_free(V.op);
    if (k > 0) mesh_free(V.mesh);  // level 0's mesh is the caller's
  }
  cudaFree(P->pcg);
  delete P;
}

hofem_status pmg_estimate(PMG* P, int k, cudaStream_t s) {
  PMGLevel& V = P->L[k];
  const long long n = V.n;
  // v = R12 random vector of the level (seed), normalized
  HOFEM_TRY(fill_random_range(P->seed, 0, n, V.x, s));
  double nv = 0.0;
  HOFEM_TRY(dot_host(V.mesh, V.x, V.x, &nv, s));
  scale_kernel<<<grid_for(n, kBS), kBS, 0, s>>>(n, 1.0 / sqrt(nv), V.x, V.x);
  HOFEM_LAUNCHED();
  double lam = 0.0;
  for (int it = 0; it < P->power_iters; ++it) {
    HOFEM_TRY(apply_any(V.op, V.x, V.t, s));
    mul_kernel<<<grid_for(n, kBS), kBS, 0, s>>>(n, V.dinv, V.t);
    HOFEM_LAUNCHED();
    double ww = 0.0;
    HOFEM_TRY(dot_host(V.mesh, V.t, V.t, &ww, s));
    lam = sqrt(ww);
    scale_kernel<<<grid_for(n, kBS), kBS, 0, s>>>(n, 1.0 / lam, V.t, V.x);
    HOFEM_LAUNCHED();
  }
  V.lam = lam;
  return HOFEM_OK;
}

hofem_status pmg_create(Mesh* fine, int degree, int power_iters, unsigned long long seed,
                        cudaStream_t s, PMG** out) {
  if (fine->nranks != 1) {
    set_error("hofem_pmg_create: single rank only");
    return HOFEM_ERR_ARG;
  }
  if (degree < 1 || power_iters < 1) {
    set_error("hofem_pmg_create: need degree >= 1 and power_iters >= 1");
    return HOFEM_ERR_ARG;
  }
  auto* P = new PMG();
  P->fine = fine;
  P->degree = degree;
  P->power_iters = power_iters;
  P->seed = seed;
  // orders p, p/2, ..., 1 (reading R17)
  std::vector<int> orders{fine->p};
  while (orders.back() > 1) orders.push_back(orders.back() / 2 > 1 ? orders.back() / 2 : 1);
  hofem_status st = HOFEM_OK;
#define CK(x) do { st = (x); if (st != HOFEM_OK) { pmg_destroy(P); return st; } } while (0)
  for (size_t k = 0; k < orders.size(); ++k) {
    PMGLevel V;
    if (k == 0) {
      V.mesh = fine;
    } else {
      hofem_mesh_desc d = fine->desc;
      d.p = orders[k];
      CK(mesh_new(&d, nullptr, s, &V.mesh));
    }
    P->L.push_back(V);
    PMGLevel& W = P->L.back();
    CK(op_new(W.mesh, HOFEM_DIFFUSION, HOFEM_GAUSS, 0, HOFEM_BC_DIRICHLET, s, &W.op));
    W.n = W.mesh->n_local;
    double** vecs[6] = {&W.dinv, &W.b, &W.x, &W.r, &W.d, &W.t};
    for (double** v : vecs)
      CK(cuda_status(cudaMalloc(v, sizeof(double) * (W.n + 1)), "pmg vectors"));
    CK(op_diagonal(W.op, W.t, s));
    recip_kernel<<<grid_for(W.n, kBS), kBS, 0, s>>>(W.n, W.t, W.dinv);
    CK(cuda_status(cudaPeekAtLastError(), "recip"));
    count_launch();
  }
  for (size_t k = 0; k + 1 < orders.size(); ++k) {
    PMGLevel &F = P->L[k], &C = P->L[k + 1];
    const int Pf = F.mesh->P1, Pc = C.mesh->P1;
    double I[(kMaxP + 1) * (kMaxP + 1)];
    interp_table(F.mesh->p, C.mesh->p, I);
    CK(cuda_status(cudaMalloc(&F.I1, sizeof(double) * Pf * Pc), "pmg tables"));
    CK(cuda_status(cudaMemcpyAsync(F.I1, I, sizeof(double) * Pf * Pc, cudaMemcpyHostToDevice, s),
                   "pmg tables"));
    CK(cuda_status(cudaMalloc(&F.ec, sizeof(double) * (F.mesh->elems * Pc * Pc * Pc + 1)),
                   "pmg scratch"));
  }
  for (size_t k = 0; k < orders.size(); ++k) CK(pmg_estimate(P, (int)k, s));
  CK(cuda_status(cudaMalloc(&P->pcg, sizeof(double) * 4 * (P->L[0].n + 1)), "pcg vectors"));
  CK(cuda_status(cudaStreamSynchronize(s), "pmg_create sync"));
#undef CK
  *out = P;
  return HOFEM_OK;
}

// Preconditioned CG (reading R18), one V-cycle per iteration.  SYNC.
hofem_status pmg_pcg(PMG* P, const double* b, double* x, double rel_tol, int max_iter,
                     double* rr_history, hofem_cg_stats* stats, cudaStream_t s) {
  PMGLevel& V = P->L[0];
  Mesh* m = V.mesh;
  const long long n = V.n;
  double *r = P->pcg, *z = r + (n + 1), *p = z + (n + 1), *Ap = p + (n + 1);
  // r = b - A x0
  HOFEM_TRY(apply_any(V.op, x, Ap, s));
  sub_kernel<<<grid_for(n, kBS), kBS, 0, s>>>(n, b, Ap, r);
  HOFEM_LAUNCHED();
  double rr0 = 0.0, rr = 0.0, rz = 0.0;
  HOFEM_TRY(dot_host(m, r, r, &rr0, s));
  rr = rr0;
  if (rr_history) rr_history[0] = rr0;
  int k = 0;
  hofem_status status = HOFEM_NOT_CONVERGED;
  if (rr0 == 0.0) status = HOFEM_OK;
  if (status != HOFEM_OK) {
    HOFEM_TRY(pmg_vcycle_level(P, 0, r, z, s));
    HOFEM_CUDA(cudaMemcpyAsync(p, z, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    HOFEM_TRY(dot_host(m, r, z, &rz, s));
  }
  while (status != HOFEM_OK && k < max_iter) {
    HOFEM_TRY(apply_any(V.op, p, Ap, s));
    double pAp = 0.0;
    HOFEM_TRY(dot_host(m, p, Ap, &pAp, s));
    if (!(pAp > 0.0)) { status = HOFEM_ERR_BREAKDOWN; break; }
    const double alpha = rz / pAp;
    pcg_update_kernel<<<grid_for(n, kBS), kBS, 0, s>>>(n, alpha, p, Ap, x, r);
    HOFEM_LAUNCHED();
    ++k;
    HOFEM_TRY(dot_host(m, r, r, &rr, s));
    if (rr_history) rr_history[k] = rr;
    if (rr == 0.0 || sqrt(rr) <= rel_tol * sqrt(rr0)) { status = HOFEM_OK; break; }
    HOFEM_TRY(pmg_vcycle_level(P, 0, r, z, s));
    double rzn = 0.0;
    HOFEM_TRY(dot_host(m, r, z, &rzn, s));
    xpby_kernel<<<grid_for(n, kBS), kBS, 0, s>>>(n, z, rzn / rz, p);
    HOFEM_LAUNCHED();
    rz = rzn;
  }
  HOFEM_CUDA(cudaStreamSynchronize(s));
  if (stats) {
    stats->iterations = k;
    stats->converged = status == HOFEM_OK ? 1 : 0;
    stats->r0_norm = sqrt(rr0);
    stats->final_rel_res = rr0 > 0.0 ? sqrt(rr / rr0) : 0.0;
  }
  if (status == HOFEM_ERR_BREAKDOWN) set_error("hofem_pmg_pcg: breakdown at k=%d", k);
  if (status == HOFEM_NOT_CONVERGED) set_error("hofem_pmg_pcg: max_iter=%d reached", max_iter);
  return status;
}

int pmg_levels(const PMG* P) { return (int)P->L.size(); }
Mesh* pmg_level_mesh(PMG* P, int k) { return P->L[k].mesh; }
Op* pmg_level_op(PMG* P, int k) { return P->L[k].op; }
double pmg_level_lambda(const PMG* P, int k) { return P->L[k].lam; }
void pmg_set_lambda(PMG* P, int k, double lam) { P->L[k].lam = lam; }
int pmg_degree(const PMG* P) { return P->degree; }

}  // namespace hofem
