// mesh.cu -- structured hex mesh + dof generator:
// nodal coordinates per lattice point (reading R4), the L->E restriction table
// l2e and its transposed offsets (reading R3; "G"), and the
// counter-based random L-vector of reading R12.
#include <cub/device/device_scan.cuh>

#include "internal.h"

namespace hofem {

namespace {

__device__ __forceinline__ double lattice_u(long long I, int p, int n, const double* xi) {
  long long e = I / p;
  int a = (int)(I - e * p);
  if (e == n) { e = n - 1; a = p; }
  return ((double)e + xi[a]) / (double)n;
}

// Phi(u)_i = u_i + alpha s(u) cos(pi u_{i+1}), s = prod sin(pi u_j); X_i = L_i Phi_i.
__global__ void coords_kernel(hofem_mesh_desc d, int z0, long long Nx, long long Ny,
                              long long n, const double* __restrict__ xi,
                              double* __restrict__ xyz) {
  long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (l >= n) return;
  long long I = l % Nx, J = (l / Nx) % Ny, K = l / (Nx * Ny) + (long long)d.p * z0;
  double u[3] = {lattice_u(I, d.p, d.nx, xi), lattice_u(J, d.p, d.ny, xi),
                 lattice_u(K, d.p, d.nz_global, xi)};
  double s = sinpi(u[0]) * sinpi(u[1]) * sinpi(u[2]);
#pragma unroll
  for (int i = 0; i < 3; ++i)
    xyz[i * n + l] = d.extent[i] * (u[i] + d.alpha * s * cospi(u[(i + 1) % 3]));
}

__global__ void l2e_kernel(int p, int nx, int ny, long long Nx, long long Ny, long long E,
                           int* __restrict__ l2e) {
  const int P1 = p + 1, nd = P1 * P1 * P1;
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= E * nd) return;
  long long e = t / nd;
  int i = (int)(t - e * nd);
  int a = i % P1, b = (i / P1) % P1, c = i / (P1 * P1);
  long long ex = e % nx, ey = (e / nx) % ny, ez = e / ((long long)nx * ny);
  l2e[t] = (int)((p * ex + a) + Nx * ((p * ey + b) + Ny * (p * ez + c)));
}

__device__ __forceinline__ int axis_count(long long I, int p, long long N) {
  return (I % p == 0 && I > 0 && I < N - 1) ? 2 : 1;
}

__global__ void tcount_kernel(int p, long long Nx, long long Ny, long long Nz,
                              long long* __restrict__ cnt) {
  long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long n = Nx * Ny * Nz;
  if (l > n) return;
  if (l == n) { cnt[l] = 0; return; }
  long long I = l % Nx, J = (l / Nx) % Ny, K = l / (Nx * Ny);
  cnt[l] = axis_count(I, p, Nx) * axis_count(J, p, Ny) * axis_count(K, p, Nz);
}

// Candidate elements along one axis containing lattice index I, ascending.
__device__ __forceinline__ int axis_elems(long long I, int p, int n, long long* e, int* a) {
  long long q = I / p;
  int r = (int)(I - q * p);
  int k = 0;
  if (r == 0 && q > 0) { e[k] = q - 1; a[k] = p; ++k; }
  if (q < n) { e[k] = q; a[k] = r; ++k; }
  return k;
}

__global__ void tfill_kernel(int p, int nx, int ny, int nz, long long Nx, long long Ny,
                             long long Nz, const long long* __restrict__ toff,
                             int* __restrict__ tidx) {
  long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (l >= Nx * Ny * Nz) return;
  const int P1 = p + 1, nd = P1 * P1 * P1;
  long long I = l % Nx, J = (l / Nx) % Ny, K = l / (Nx * Ny);
  long long ex[2], ey[2], ez[2];
  int ax[2], ay[2], az[2];
  int kx = axis_elems(I, p, nx, ex, ax), ky = axis_elems(J, p, ny, ey, ay),
      kz = axis_elems(K, p, nz, ez, az);
  long long o = toff[l];
  for (int c = 0; c < kz; ++c)      // ascending e = ex + nx (ey + ny ez)
    for (int b = 0; b < ky; ++b)
      for (int a = 0; a < kx; ++a) {
        long long e = ex[a] + (long long)nx * (ey[b] + (long long)ny * ez[c]);
        tidx[o++] = (int)(e * nd + ax[a] + P1 * (ay[b] + P1 * az[c]));
      }
}

// splitmix64 finalizer; reading R12.
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void random_kernel(unsigned long long seed, long long g0, long long n,
                              double* __restrict__ x) {
  long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (l >= n) return;
  unsigned long long g = (unsigned long long)(g0 + l);
  unsigned long long z = mix64(seed + (g + 1ULL) * 0x9E3779B97F4A7C15ULL);
  x[l] = 2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0;
}

inline unsigned grid_for(long long n, int bs) { return (unsigned)((n + bs - 1) / bs); }

}  // namespace

hofem_status mesh_build_coords(Mesh* m, cudaStream_t s) {
  coords_kernel<<<grid_for(m->n_local, 256), 256, 0, s>>>(m->desc, m->z0, m->Nx, m->Ny,
                                                          m->n_local, m->d_xi, m->d_coords);
  HOFEM_LAUNCHED();
  return HOFEM_OK;
}

hofem_status mesh_build_restriction(Mesh* m, cudaStream_t s) {
  if (m->d_l2e) return HOFEM_OK;
  const int P1 = m->P1, nd = P1 * P1 * P1;
  long long ent = m->elems * nd;
  if (m->n_local >= (1LL << 31) || ent >= (1LL << 31)) {
    set_error("unfused path: mesh too large for 32-bit restriction tables");
    return HOFEM_ERR_ARG;
  }
  // stream-ordered (no device-wide synchronization between exchanges)
  if (cudaMallocAsync(&m->d_l2e, sizeof(int) * ent, s) != cudaSuccess ||
      cudaMallocAsync(&m->d_toff, sizeof(long long) * (m->n_local + 1), s) != cudaSuccess ||
      cudaMallocAsync(&m->d_tidx, sizeof(int) * ent, s) != cudaSuccess) {
    cudaGetLastError();
    set_error("restriction tables: out of device memory");
    return HOFEM_ERR_OOM;
  }
  l2e_kernel<<<grid_for(ent, 256), 256, 0, s>>>(m->p, m->nx, m->ny, m->Nx, m->Ny, m->elems,
                                                m->d_l2e);
  HOFEM_LAUNCHED();
  long long* cnt = nullptr;
  HOFEM_CUDA(cudaMallocAsync(&cnt, sizeof(long long) * (m->n_local + 1), s));
  tcount_kernel<<<grid_for(m->n_local + 1, 256), 256, 0, s>>>(m->p, m->Nx, m->Ny, m->Nzl, cnt);
  HOFEM_LAUNCHED();
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, m->d_toff, m->n_local + 1, s);
  void* tmp = nullptr;
  HOFEM_CUDA(cudaMallocAsync(&tmp, tmp_bytes, s));
  HOFEM_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, m->d_toff, m->n_local + 1, s));
  count_launch();
  tfill_kernel<<<grid_for(m->n_local, 256), 256, 0, s>>>(m->p, m->nx, m->ny, m->nzl, m->Nx,
                                                         m->Ny, m->Nzl, m->d_toff, m->d_tidx);
  HOFEM_LAUNCHED();
  HOFEM_CUDA(cudaFreeAsync(tmp, s));
  HOFEM_CUDA(cudaFreeAsync(cnt, s));
  return HOFEM_OK;
}

hofem_status fill_random(const Mesh* m, unsigned long long seed, double* x, cudaStream_t s) {
  return fill_random_range(seed, m->plane * (long long)m->p * m->z0, m->n_local, x, s);
}

hofem_status fill_random_range(unsigned long long seed, long long g0, long long n, double* x,
                               cudaStream_t s) {
  if (n <= 0) return HOFEM_OK;
  random_kernel<<<grid_for(n, 256), 256, 0, s>>>(seed, g0, n, x);
  HOFEM_LAUNCHED();
  return HOFEM_OK;
}

}  // namespace hofem
