// cg.cu -- CG vector kernels and the CG driver (
// PAPER.md:89 "Krylov subspace method"; reading R7).
//
// Per iteration (single rank: 5 launches, no host sync):
//   Ap = A p                      fused brick kernel + brick fix-up (fused.cu)
//   pAp = p.Ap                    dot_kernel (owned dofs, last-block reduction)
//   alpha = rr/pAp; x += alpha p; r -= alpha Ap; rr' = r.r     update_kernel
//   beta = rr'/rr; p = r + beta p                               pupdate_kernel
// alpha and beta are recomputed by every thread from device scalars, so the
// host never waits.  Every reduction has a fixed grid and a fixed combination
// order: results are bitwise reproducible run to run.  Multi-rank: the scalar
// partials are ncclAllReduce'd on the same stream before use.
#include <math.h>

#include <vector>

#include "internal.h"

namespace hofem {

constexpr int kDotBlocks = 2 * kNumSMs;  // fixed grid => fixed reduction order
constexpr int kDotThreads = 512;

namespace {

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  return v;  // valid in thread 0
}

// Writes the block partial; the last block to finish sums all partials in
// block order and stores *out.  Deterministic.
__device__ __forceinline__ void finish_reduction(double v, double* partials,
                                                 unsigned int* counter, double* out) {
  __shared__ double sh[32];
  __shared__ bool last;
  v = block_sum(v, sh);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = v;
    __threadfence();
    unsigned int t = atomicAdd(counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double s = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x)
    s += ((volatile double*)partials)[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) {
    *out = s;
    *counter = 0u;
  }
}

__global__ void __launch_bounds__(kDotThreads) dot_kernel(long long n, const double* __restrict__ a,
                                                          const double* __restrict__ b,
                                                          double* partials, unsigned int* counter,
                                                          double* out) {
  double s = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
    s = fma(a[i], b[i], s);
  finish_reduction(s, partials, counter, out);
}

// r = b - Ax; p = r; rr0 = r.r (owned prefix)
__global__ void __launch_bounds__(kDotThreads) init_kernel(long long n, long long n_owned,
                                                           const double* __restrict__ b,
                                                           const double* __restrict__ Ax,
                                                           double* __restrict__ r,
                                                           double* __restrict__ p,
                                                           double* partials,
                                                           unsigned int* counter, double* out) {
  double s = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    double v = b[i] - Ax[i];
    r[i] = v;
    p[i] = v;
    if (i < n_owned) s = fma(v, v, s);
  }
  finish_reduction(s, partials, counter, out);
}

// alpha = rr/pAp; x += alpha p; r -= alpha Ap; rr' = r.r (owned prefix).
// sc[0] = rr_k, sc[1] = pAp, out = rr_{k+1}; flag set if pAp <= 0.
__global__ void __launch_bounds__(kDotThreads) update_kernel(
    long long n, long long n_owned, const double* __restrict__ p, const double* __restrict__ Ap,
    double* __restrict__ x, double* __restrict__ r, const double* sc_rr, const double* sc_pAp,
    double* partials, unsigned int* counter, double* out, double* flag) {
  const double pAp = *sc_pAp;
  double alpha = *sc_rr / pAp;
  if (!(pAp > 0.0)) {
    alpha = 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) *flag = 1.0;
  }
  double s = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    x[i] = fma(alpha, p[i], x[i]);
    double v = fma(-alpha, Ap[i], r[i]);
    r[i] = v;
    if (i < n_owned) s = fma(v, v, s);
  }
  finish_reduction(s, partials, counter, out);
}

// beta = rr_{k+1}/rr_k; p = r + beta p
__global__ void pupdate_kernel(long long n, const double* __restrict__ r, double* __restrict__ p,
                               const double* sc_new, const double* sc_old) {
  const double rn = *sc_new, ro = *sc_old;
  const double beta = ro > 0.0 ? rn / ro : 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
    p[i] = fma(beta, p[i], r[i]);
}

}  // namespace

hofem_status dot_device(Mesh* m, const double* a, const double* b, double* d_out,
                        cudaStream_t s) {
  dot_kernel<<<kDotBlocks, kDotThreads, 0, s>>>(m->n_owned, a, b, m->d_partials, m->d_counter,
                                                d_out);
  HOFEM_LAUNCHED();
  return allreduce_sum(m, d_out, 1, s);
}

hofem_status apply_any(Op* op, const double* x, double* y, cudaStream_t s);

hofem_status cg_solve(Op* op, const double* b, double* x, double rel_tol, int max_iter,
                      int fixed_iters, int check_every, double* rr_history,
                      hofem_cg_stats* stats, cudaStream_t s) {
  Mesh* m = op->mesh;
  const long long n = m->n_local, no = m->n_owned;
  if (max_iter < 0) { set_error("hofem_cg: max_iter < 0"); return HOFEM_ERR_ARG; }
  if (check_every < 1) check_every = 1;
  if (!op->d_r) {
    if (cudaMalloc(&op->d_r, sizeof(double) * n) != cudaSuccess ||
        cudaMalloc(&op->d_p, sizeof(double) * n) != cudaSuccess ||
        cudaMalloc(&op->d_Ap, sizeof(double) * n) != cudaSuccess) {
      cudaGetLastError();
      set_error("hofem_cg: out of device memory for work vectors");
      return HOFEM_ERR_OOM;
    }
  }
  if (op->cg_cap < max_iter + 1) {
    if (op->d_cg) cudaFree(op->d_cg);
    op->d_cg = nullptr;
    HOFEM_CUDA(cudaMalloc(&op->d_cg, sizeof(double) * (max_iter + 1 + 8)));
    op->cg_cap = max_iter + 1;
  }
  double* rr = op->d_cg;                  // rr[k], k = 0..max_iter
  double* pAp = op->d_cg + op->cg_cap;    // scratch
  double* flag = pAp + 1;
  HOFEM_CUDA(cudaMemsetAsync(flag, 0, sizeof(double), s));

  HOFEM_TRY(apply_any(op, x, op->d_Ap, s));
  init_kernel<<<kDotBlocks, kDotThreads, 0, s>>>(n, no, b, op->d_Ap, op->d_r, op->d_p,
                                                 m->d_partials, m->d_counter, rr);
  HOFEM_LAUNCHED();
  HOFEM_TRY(allreduce_sum(m, rr, 1, s));
  double rr0 = 0.0;
  HOFEM_CUDA(cudaMemcpyAsync(&rr0, rr, sizeof(double), cudaMemcpyDeviceToHost, s));
  HOFEM_CUDA(cudaStreamSynchronize(s));

  const unsigned vgrid = kDotBlocks;
  int k = 0;
  hofem_status status = fixed_iters ? HOFEM_OK : HOFEM_NOT_CONVERGED;
  double rr_last = rr0;
  bool done = (rr0 == 0.0 && !fixed_iters);
  if (done) status = HOFEM_OK;
  while (!done && k < max_iter) {
    HOFEM_TRY(apply_any(op, op->d_p, op->d_Ap, s));
    dot_kernel<<<kDotBlocks, kDotThreads, 0, s>>>(no, op->d_p, op->d_Ap, m->d_partials,
                                                  m->d_counter, pAp);
    HOFEM_LAUNCHED();
    HOFEM_TRY(allreduce_sum(m, pAp, 1, s));
    update_kernel<<<kDotBlocks, kDotThreads, 0, s>>>(n, no, op->d_p, op->d_Ap, x, op->d_r, rr + k,
                                                     pAp, m->d_partials, m->d_counter,
                                                     rr + k + 1, flag);
    HOFEM_LAUNCHED();
    HOFEM_TRY(allreduce_sum(m, rr + k + 1, 1, s));
    pupdate_kernel<<<vgrid, 256, 0, s>>>(n, op->d_r, op->d_p, rr + k + 1, rr + k);
    HOFEM_LAUNCHED();
    ++k;
    if ((!fixed_iters && k % check_every == 0) || k == max_iter) {
      double h[2];
      HOFEM_CUDA(cudaMemcpyAsync(&h[0], rr + k, sizeof(double), cudaMemcpyDeviceToHost, s));
      HOFEM_CUDA(cudaMemcpyAsync(&h[1], flag, sizeof(double), cudaMemcpyDeviceToHost, s));
      HOFEM_CUDA(cudaStreamSynchronize(s));
      rr_last = h[0];
      if (h[1] != 0.0) { status = HOFEM_ERR_BREAKDOWN; break; }
      if (!fixed_iters && (rr_last == 0.0 || sqrt(rr_last) <= rel_tol * sqrt(rr0))) {
        status = HOFEM_OK;
        done = true;
      }
    }
  }
  if (rr_history) {
    HOFEM_CUDA(cudaMemcpyAsync(rr_history, rr, sizeof(double) * (k + 1), cudaMemcpyDeviceToHost, s));
  }
  HOFEM_CUDA(cudaStreamSynchronize(s));
  if (stats) {
    stats->iterations = k;
    stats->converged = status == HOFEM_OK ? 1 : 0;
    stats->r0_norm = sqrt(rr0);
    stats->final_rel_res = rr0 > 0.0 ? sqrt(rr_last / rr0) : 0.0;
  }
  if (status == HOFEM_ERR_BREAKDOWN) set_error("hofem_cg: breakdown (p^T A p <= 0) at k=%d", k);
  if (status == HOFEM_NOT_CONVERGED) set_error("hofem_cg: max_iter=%d reached", max_iter);
  return status;
}

}  // namespace hofem
