// qdata.cu -- quadrature-point geometric factors: the
// only stored operator data of partial assembly ("Only the essential
// data at quadrature points is precomputed and stored"; "D").
//   J_ij = d x_i / d xi_j at every point, from the element's nodal coordinates
//   through the 1D B1d/G1d tables; mass D = W detJ; diffusion
//   D = W adj(J) adj(J)^T / detJ (6 entries [00,01,02,11,12,22]), layout
//   [E][n_c][Q^3] with the point index qx + Q (qy + Q qz) (reading R3).
// Also the manufactured right-hand side of reading R11.  Setup only.
#include "internal.h"

namespace hofem {

hofem_status scatter_evector(Op* op, const double* ein, double* y, cudaStream_t s);

namespace {

constexpr int kQThreads = 128;

// Loads the element's nodal coordinates X[3][P1^3] (a fastest) into smem.
__device__ void load_element_coords(const Mesh* mm, long long e, int P1, int p, int nx, int ny,
                                    long long Nx, long long Ny, long long n,
                                    const double* __restrict__ xyz, double* X) {
  const int nd = P1 * P1 * P1;
  long long ex = e % nx, ey = (e / nx) % ny, ez = e / ((long long)nx * ny);
  for (int i = threadIdx.x; i < nd; i += blockDim.x) {
    int a = i % P1, b = (i / P1) % P1, c = i / (P1 * P1);
    long long l = (p * ex + a) + Nx * ((p * ey + b) + Ny * (p * ez + c));
    X[i] = xyz[l];
    X[nd + i] = xyz[n + l];
    X[2 * nd + i] = xyz[2 * n + l];
  }
  (void)mm;
}

struct Geo {
  int p, P1, Q, nx, ny;
  long long Nx, Ny, n, E;
};

// J at point (qx,qy,qz): J_ij = sum_{abc} X_i(abc) * d/dxi_j [l_a l_b l_c].
__device__ void jacobian_at(const Geo& g, const double* X, const double* B, const double* G,
                            int qx, int qy, int qz, double J[3][3]) {
  const int P1 = g.P1, nd = P1 * P1 * P1;
  for (int i = 0; i < 3; ++i) J[i][0] = J[i][1] = J[i][2] = 0.0;
  for (int c = 0; c < P1; ++c) {
    double bz = B[qz * P1 + c], gz = G[qz * P1 + c];
    for (int b = 0; b < P1; ++b) {
      double by = B[qy * P1 + b], gy = G[qy * P1 + b];
      for (int a = 0; a < P1; ++a) {
        double bx = B[qx * P1 + a], gx = G[qx * P1 + a];
        int al = a + P1 * (b + P1 * c);
        double d0 = gx * by * bz, d1 = bx * gy * bz, d2 = bx * by * gz;
        for (int i = 0; i < 3; ++i) {
          double Xi = X[i * nd + al];
          J[i][0] += Xi * d0;
          J[i][1] += Xi * d1;
          J[i][2] += Xi * d2;
        }
      }
    }
  }
}

__global__ void qdata_kernel(Geo g, int kind, const double* __restrict__ xyz,
                             const double* __restrict__ dB, const double* __restrict__ dG,
                             const double* __restrict__ dw, double* __restrict__ qd,
                             int* __restrict__ bad) {
  extern __shared__ double sm[];
  const int P1 = g.P1, Q = g.Q, nd = P1 * P1 * P1, nq = Q * Q * Q;
  double* X = sm;
  double* B = X + 3 * nd;
  double* G = B + Q * P1;
  double* w = G + Q * P1;
  for (int i = threadIdx.x; i < Q * P1; i += blockDim.x) { B[i] = dB[i]; G[i] = dG[i]; }
  for (int i = threadIdx.x; i < Q; i += blockDim.x) w[i] = dw[i];
  long long e = blockIdx.x;
  load_element_coords(nullptr, e, P1, g.p, g.nx, g.ny, g.Nx, g.Ny, g.n, xyz, X);
  __syncthreads();
  const int nc = kind == HOFEM_MASS ? 1 : 6;
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    int qx = q % Q, qy = (q / Q) % Q, qz = q / (Q * Q);
    double J[3][3];
    jacobian_at(g, X, B, G, qx, qy, qz, J);
    double A[3][3];  // adj(J)
    A[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    A[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
    A[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
    A[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    A[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
    A[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
    A[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    A[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
    A[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    double det = J[0][0] * A[0][0] + J[0][1] * A[1][0] + J[0][2] * A[2][0];
    if (!(det > 0.0)) atomicOr(bad, 1);
    double W = w[qx] * w[qy] * w[qz];
    double* out = qd + (e * nc) * nq + q;
    if (kind == HOFEM_MASS) {
      out[0] = W * det;
    } else {
      double f = W / det;
      out[0 * nq] = f * (A[0][0] * A[0][0] + A[0][1] * A[0][1] + A[0][2] * A[0][2]);
      out[1 * nq] = f * (A[0][0] * A[1][0] + A[0][1] * A[1][1] + A[0][2] * A[1][2]);
      out[2 * nq] = f * (A[0][0] * A[2][0] + A[0][1] * A[2][1] + A[0][2] * A[2][2]);
      out[3 * nq] = f * (A[1][0] * A[1][0] + A[1][1] * A[1][1] + A[1][2] * A[1][2]);
      out[4 * nq] = f * (A[1][0] * A[2][0] + A[1][1] * A[2][1] + A[1][2] * A[2][2]);
      out[5 * nq] = f * (A[2][0] * A[2][0] + A[2][1] * A[2][1] + A[2][2] * A[2][2]);
    }
  }
}

// E-vector of b_i = sum_q W detJ f(x_q) phi_i(xi_q) (reading R11).
__global__ void rhs_kernel(Geo g, int kind, const double* __restrict__ xyz,
                           const double* __restrict__ dB, const double* __restrict__ dG,
                           const double* __restrict__ dw, double* __restrict__ be) {
  extern __shared__ double sm[];
  const int P1 = g.P1, Q = g.Q, nd = P1 * P1 * P1, nq = Q * Q * Q;
  double* X = sm;
  double* B = X + 3 * nd;
  double* G = B + Q * P1;
  double* w = G + Q * P1;
  double* fq = w + Q;  // nq values: W detJ f at each point
  for (int i = threadIdx.x; i < Q * P1; i += blockDim.x) { B[i] = dB[i]; G[i] = dG[i]; }
  for (int i = threadIdx.x; i < Q; i += blockDim.x) w[i] = dw[i];
  long long e = blockIdx.x;
  load_element_coords(nullptr, e, P1, g.p, g.nx, g.ny, g.Nx, g.Ny, g.n, xyz, X);
  __syncthreads();
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    int qx = q % Q, qy = (q / Q) % Q, qz = q / (Q * Q);
    double J[3][3];
    jacobian_at(g, X, B, G, qx, qy, qz, J);
    double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                 J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                 J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    double xq[3] = {0.0, 0.0, 0.0};
    for (int c = 0; c < P1; ++c)
      for (int b = 0; b < P1; ++b)
        for (int a = 0; a < P1; ++a) {
          double ph = B[qx * P1 + a] * B[qy * P1 + b] * B[qz * P1 + c];
          int al = a + P1 * (b + P1 * c);
          xq[0] += X[al] * ph;
          xq[1] += X[nd + al] * ph;
          xq[2] += X[2 * nd + al] * ph;
        }
    double f = sinpi(xq[0]) * sinpi(xq[1]) * sinpi(xq[2]);
    if (kind == HOFEM_DIFFUSION) f *= 3.0 * M_PI * M_PI;
    fq[q] = w[qx] * w[qy] * w[qz] * det * f;
  }
  __syncthreads();
  for (int al = threadIdx.x; al < nd; al += blockDim.x) {
    int a = al % P1, b = (al / P1) % P1, c = al / (P1 * P1);
    double s = 0.0;
    for (int q = 0; q < nq; ++q) {
      int qx = q % Q, qy = (q / Q) % Q, qz = q / (Q * Q);
      s += fq[q] * B[qx * P1 + a] * B[qy * P1 + b] * B[qz * P1 + c];
    }
    be[e * nd + al] = s;
  }
}

Geo make_geo(const Op* op) {
  const Mesh* m = op->mesh;
  Geo g;
  g.p = m->p; g.P1 = m->P1; g.Q = op->Q; g.nx = m->nx; g.ny = m->ny;
  g.Nx = m->Nx; g.Ny = m->Ny; g.n = m->n_local; g.E = m->elems;
  return g;
}

}  // namespace

hofem_status build_qdata(Op* op, cudaStream_t s, int* bad_host) {
  Mesh* m = op->mesh;
  Geo g = make_geo(op);
  const int nd = m->P1 * m->P1 * m->P1;
  size_t smem = sizeof(double) * (3 * nd + 2 * op->Q * m->P1 + op->Q);
  double* dw = nullptr;
  int* dbad = nullptr;
  HOFEM_CUDA(cudaMallocAsync(&dw, sizeof(double) * op->Q, s));
  HOFEM_CUDA(cudaMallocAsync(&dbad, sizeof(int), s));
  HOFEM_CUDA(cudaMemcpyAsync(dw, op->tab.w, sizeof(double) * op->Q, cudaMemcpyHostToDevice, s));
  HOFEM_CUDA(cudaMemsetAsync(dbad, 0, sizeof(int), s));
  if (m->elems > 0) {
    qdata_kernel<<<(unsigned)m->elems, kQThreads, smem, s>>>(g, op->kind, m->d_coords, op->d_B,
                                                             op->d_G, dw, op->d_qdata, dbad);
    HOFEM_LAUNCHED();
  }
  HOFEM_TRY(d2h(m, bad_host, dbad, sizeof(int), s));
  HOFEM_CUDA(cudaFreeAsync(dw, s));
  HOFEM_CUDA(cudaFreeAsync(dbad, s));
  return HOFEM_OK;
}

hofem_status build_rhs(Op* op, double* b, cudaStream_t s) {
  Mesh* m = op->mesh;
  Geo g = make_geo(op);
  const int nd = m->P1 * m->P1 * m->P1, nq = op->Q * op->Q * op->Q;
  size_t smem = sizeof(double) * (3 * nd + 2 * op->Q * m->P1 + op->Q + nq);
  double *dw = nullptr, *be = nullptr;
  HOFEM_CUDA(cudaMallocAsync(&dw, sizeof(double) * op->Q, s));
  HOFEM_CUDA(cudaMallocAsync(&be, sizeof(double) * (m->elems * nd + 1), s));
  HOFEM_CUDA(cudaMemcpyAsync(dw, op->tab.w, sizeof(double) * op->Q, cudaMemcpyHostToDevice, s));
  if (smem > 48 * 1024)
    HOFEM_CUDA(cudaFuncSetAttribute(rhs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
  if (m->elems > 0) {
    rhs_kernel<<<(unsigned)m->elems, kQThreads, smem, s>>>(g, op->kind, m->d_coords, op->d_B,
                                                           op->d_G, dw, be);
    HOFEM_LAUNCHED();
  }
  HOFEM_TRY(scatter_evector(op, be, b, s));
  HOFEM_CUDA(cudaFreeAsync(dw, s));
  HOFEM_CUDA(cudaFreeAsync(be, s));
  return HOFEM_OK;
}

}  // namespace hofem
