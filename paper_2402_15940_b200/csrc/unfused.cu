// unfused.cu -- the unfused reference GPU path:
//   gather kernel (R: L->E through the l2e table)
//   -> element kernel (B, D, B^T applied by runtime-sized sum factorization)
//   -> deterministic scatter-add (R^T) through precomputed transposed offsets,
//      each dof summing its 1..8 element contributions in ascending (e, i) order.
// Supports any 1 <= p <= 8 and 1 <= Q <= 16.  Kept simple on purpose: it is the
// GPU-side cross-check of the fused kernels, not the product hot path.
#include "internal.h"

namespace hofem {

namespace {

struct EssInfo {
  long long Nx, Ny, Nzl, K0, NzG;
};

__device__ __forceinline__ bool ess_at(const EssInfo& s, long long l) {
  long long I = l % s.Nx, J = (l / s.Nx) % s.Ny, K = l / (s.Nx * s.Ny) + s.K0;
  return I == 0 || I == s.Nx - 1 || J == 0 || J == s.Ny - 1 || K == 0 || K == s.NzG - 1;
}

__global__ void gather_kernel(long long ent, const int* __restrict__ l2e,
                              const double* __restrict__ x, int bc, EssInfo es,
                              double* __restrict__ ein) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= ent) return;
  int l = l2e[t];
  ein[t] = (bc && ess_at(es, l)) ? 0.0 : x[l];
}

// bcmode: 0 none, 1 y[ess] = xbc[ess], 2 y[ess] = 0, 3 y[ess] = 1
__global__ void scatter_kernel(long long n, const long long* __restrict__ toff,
                               const int* __restrict__ tidx, const double* __restrict__ eout,
                               int bcmode, const double* __restrict__ xbc, EssInfo es,
                               double* __restrict__ y) {
  long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (l >= n) return;
  double s = 0.0;
  for (long long k = toff[l]; k < toff[l + 1]; ++k) s += eout[tidx[k]];
  if (bcmode && ess_at(es, l)) s = (bcmode == 1) ? xbc[l] : (bcmode == 3 ? 1.0 : 0.0);
  y[l] = s;
}

// One block per element; runtime P1, Q.  Layouts: xe[a + P1(b + P1 c)],
// T1[(qx) + Q(b + P1 c)], T2[qx + Q(qy + Q c)], T3[qx + Q(qy + Q qz)].
__global__ void element_kernel(int P1, int Q, int kind, long long E,
                               const double* __restrict__ dB, const double* __restrict__ dG,
                               const double* __restrict__ qdata, const double* __restrict__ ein,
                               double* __restrict__ eout) {
  extern __shared__ double sm[];
  const int nd = P1 * P1 * P1, nq = Q * Q * Q, n1 = Q * P1 * P1, n2 = Q * Q * P1;
  double* B = sm;
  double* G = B + Q * P1;
  double* xe = G + Q * P1;     // nd
  double* T1 = xe + nd;        // 2*n1
  double* T2 = T1 + 2 * n1;    // 3*n2
  double* T3 = T2 + 3 * n2;    // 3*nq
  const long long e = blockIdx.x;
  for (int i = threadIdx.x; i < Q * P1; i += blockDim.x) { B[i] = dB[i]; G[i] = dG[i]; }
  for (int i = threadIdx.x; i < nd; i += blockDim.x) xe[i] = ein[e * nd + i];
  __syncthreads();
  const bool diff = kind == HOFEM_DIFFUSION;
  const int nc = diff ? 6 : 1;
  const double* D = qdata + e * nc * nq;
  // x-contraction
  for (int t = threadIdx.x; t < n1; t += blockDim.x) {
    int qx = t % Q, bc = t / Q;
    double sb = 0.0, sg = 0.0;
    for (int a = 0; a < P1; ++a) {
      double v = xe[a + P1 * bc];
      sb += B[qx * P1 + a] * v;
      sg += G[qx * P1 + a] * v;
    }
    T1[t] = sb;
    T1[n1 + t] = sg;
  }
  __syncthreads();
  // y-contraction
  for (int t = threadIdx.x; t < n2; t += blockDim.x) {
    int qx = t % Q, qy = (t / Q) % Q, c = t / (Q * Q);
    double bb = 0.0, bg = 0.0, gb = 0.0;
    for (int b = 0; b < P1; ++b) {
      double vb = T1[qx + Q * (b + P1 * c)], vg = T1[n1 + qx + Q * (b + P1 * c)];
      bb += B[qy * P1 + b] * vb;
      bg += G[qy * P1 + b] * vb;
      gb += B[qy * P1 + b] * vg;
    }
    T2[t] = gb;          // G_x B_y
    T2[n2 + t] = bg;     // B_x G_y
    T2[2 * n2 + t] = bb; // B_x B_y
  }
  __syncthreads();
  // z-contraction + pointwise D
  for (int t = threadIdx.x; t < nq; t += blockDim.x) {
    int qxy = t % (Q * Q), qz = t / (Q * Q);
    double u0 = 0.0, u1 = 0.0, u2 = 0.0;
    for (int c = 0; c < P1; ++c) {
      double bz = B[qz * P1 + c], gz = G[qz * P1 + c];
      u0 += bz * T2[qxy + Q * Q * c];
      u1 += bz * T2[n2 + qxy + Q * Q * c];
      u2 += gz * T2[2 * n2 + qxy + Q * Q * c];
    }
    if (diff) {
      double d00 = D[t], d01 = D[nq + t], d02 = D[2 * nq + t], d11 = D[3 * nq + t],
             d12 = D[4 * nq + t], d22 = D[5 * nq + t];
      T3[t] = d00 * u0 + d01 * u1 + d02 * u2;
      T3[nq + t] = d01 * u0 + d11 * u1 + d12 * u2;
      T3[2 * nq + t] = d02 * u0 + d12 * u1 + d22 * u2;
    } else {
      // mass: only the B_x B_y B_z value is needed
      double u = 0.0;
      for (int c = 0; c < P1; ++c) u += B[qz * P1 + c] * T2[2 * n2 + qxy + Q * Q * c];
      T3[t] = D[t] * u;
    }
  }
  __syncthreads();
  // z-transpose
  for (int t = threadIdx.x; t < n2; t += blockDim.x) {
    int qxy = t % (Q * Q), c = t / (Q * Q);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int qz = 0; qz < Q; ++qz) {
      double bz = B[qz * P1 + c];
      if (diff) {
        s0 += bz * T3[qxy + Q * Q * qz];
        s1 += bz * T3[nq + qxy + Q * Q * qz];
        s2 += G[qz * P1 + c] * T3[2 * nq + qxy + Q * Q * qz];
      } else {
        s2 += bz * T3[qxy + Q * Q * qz];
      }
    }
    T2[t] = s0;
    T2[n2 + t] = s1;
    T2[2 * n2 + t] = s2;
  }
  __syncthreads();
  // y-transpose: RG (to be G_x^T'd) and RB (to be B_x^T'd)
  for (int t = threadIdx.x; t < n1; t += blockDim.x) {
    int qx = t % Q, b = (t / Q) % P1, c = t / (Q * P1);
    double rg = 0.0, rb = 0.0;
    for (int qy = 0; qy < Q; ++qy) {
      int i2 = qx + Q * (qy + Q * c);
      double by = B[qy * P1 + b];
      if (diff) {
        rg += by * T2[i2];
        rb += G[qy * P1 + b] * T2[n2 + i2] + by * T2[2 * n2 + i2];
      } else {
        rb += by * T2[2 * n2 + i2];
      }
    }
    T1[t] = rg;
    T1[n1 + t] = rb;
  }
  __syncthreads();
  // x-transpose
  for (int t = threadIdx.x; t < nd; t += blockDim.x) {
    int a = t % P1, bc = t / P1;
    double s = 0.0;
    for (int qx = 0; qx < Q; ++qx) {
      int i1 = qx + Q * bc;
      s += B[qx * P1 + a] * T1[n1 + i1];
      if (diff) s += G[qx * P1 + a] * T1[i1];
    }
    eout[e * nd + t] = s;
  }
}

inline unsigned grid_for(long long n, int bs) { return (unsigned)((n + bs - 1) / bs); }

EssInfo ess_info(const Mesh* m) {
  return EssInfo{m->Nx, m->Ny, m->Nzl, (long long)m->p * m->z0, m->NzG};
}

}  // namespace

hofem_status scatter_evector_bc(Op* op, const double* ein, double* y, int bcmode,
                                const double* xbc, cudaStream_t s) {
  Mesh* m = op->mesh;
  HOFEM_TRY(mesh_build_restriction(m, s));
  scatter_kernel<<<grid_for(m->n_local, 256), 256, 0, s>>>(m->n_local, m->d_toff, m->d_tidx, ein,
                                                           bcmode, xbc, ess_info(m), y);
  HOFEM_LAUNCHED();
  return HOFEM_OK;
}

hofem_status scatter_evector(Op* op, const double* ein, double* y, cudaStream_t s) {
  return scatter_evector_bc(op, ein, y, op->bc ? 2 : 0, nullptr, s);
}

hofem_status apply_unfused(Op* op, const double* x, double* y, cudaStream_t s) {
  Mesh* m = op->mesh;
  HOFEM_TRY(mesh_build_restriction(m, s));
  const int P1 = m->P1, Q = op->Q, nd = P1 * P1 * P1;
  const long long ent = m->elems * nd;
  if (!op->d_ein) {
    // stream-ordered (no device-wide synchronization between exchanges)
    if (cudaMallocAsync(&op->d_ein, sizeof(double) * (ent + 1), s) != cudaSuccess ||
        cudaMallocAsync(&op->d_eout, sizeof(double) * (ent + 1), s) != cudaSuccess) {
      cudaGetLastError();
      set_error("unfused path: out of device memory for E-vectors");
      return HOFEM_ERR_OOM;
    }
  }
  gather_kernel<<<grid_for(ent, 256), 256, 0, s>>>(ent, m->d_l2e, x, op->bc, ess_info(m),
                                                   op->d_ein);
  HOFEM_LAUNCHED();
  size_t smem = sizeof(double) *
                (2 * Q * P1 + nd + 2 * Q * P1 * P1 + 3 * Q * Q * P1 + 3 * Q * Q * Q);
  static size_t smem_set = 0;
  if (smem > 48 * 1024 && smem > smem_set) {
    HOFEM_CUDA(cudaFuncSetAttribute(element_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
    smem_set = smem;
  }
  if (m->elems > 0) {
    element_kernel<<<(unsigned)m->elems, 128, smem, s>>>(P1, Q, op->kind, m->elems, op->d_B,
                                                         op->d_G, op->d_qdata, op->d_ein,
                                                         op->d_eout);
    HOFEM_LAUNCHED();
  }
  HOFEM_TRY(scatter_evector_bc(op, op->d_eout, y, op->bc ? 1 : 0, x, s));
  return exchange_planes(op, x, y, s);
}

}  // namespace hofem
