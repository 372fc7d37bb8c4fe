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
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include <vector>

#include "internal.h"

namespace hofem {

constexpr int kDotBlocks = 4 * kNumSMs;  // fixed grid => fixed reduction order
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

// The vector kernels walk [0, n) in 16-byte pairs (torch allocations are
// 256-byte aligned), two pairs per thread per iteration for memory-level
// parallelism; an odd tail element is handled by the last pair's owner.  The
// traversal order of every thread is fixed, so reductions are deterministic.
struct Span {
  long long npair, stride, i0;
};
__device__ __forceinline__ Span span(long long n) {
  Span s;
  s.npair = n >> 1;
  s.stride = (long long)gridDim.x * blockDim.x;
  s.i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  return s;
}

__global__ void __launch_bounds__(kDotThreads) dot_kernel(long long n, const double* __restrict__ a,
                                                          const double* __restrict__ b,
                                                          double* partials, unsigned int* counter,
                                                          double* out) {
  const Span S = span(n);
  const double2* a2 = reinterpret_cast<const double2*>(a);
  const double2* b2 = reinterpret_cast<const double2*>(b);
  double s0 = 0.0, s1 = 0.0;
  for (long long i = S.i0; i < S.npair; i += 2 * S.stride) {
    const double2 x0 = a2[i], y0 = b2[i];
    s0 = fma(x0.x, y0.x, s0);
    s0 = fma(x0.y, y0.y, s0);
    if (i + S.stride < S.npair) {
      const double2 x1 = a2[i + S.stride], y1 = b2[i + S.stride];
      s1 = fma(x1.x, y1.x, s1);
      s1 = fma(x1.y, y1.y, s1);
    }
  }
  if ((n & 1) && S.i0 == 0) s0 = fma(a[n - 1], b[n - 1], s0);
  finish_reduction(s0 + s1, partials, counter, out);
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

// alpha = rr/pAp; r -= alpha Ap; rr' = r.r (owned prefix).  The x update is
// deferred to pupdate_kernel, which reads p anyway (one stream less per
// iteration; x_{k+1} = x_k + alpha p_k is the same fma either way).
__device__ __forceinline__ double cg_alpha(const double* sc_rr, const double* sc_pAp) {
  const double pAp = *sc_pAp;
  return pAp > 0.0 ? *sc_rr / pAp : 0.0;
}

__global__ void __launch_bounds__(kDotThreads) update_kernel(
    long long n, long long n_owned, const double* __restrict__ Ap, double* __restrict__ r,
    const double* sc_rr, const double* sc_pAp, double* partials, unsigned int* counter,
    double* out, double* flag) {
  if (!(*sc_pAp > 0.0) && blockIdx.x == 0 && threadIdx.x == 0) *flag = 1.0;
  const double alpha = cg_alpha(sc_rr, sc_pAp);
  const Span S = span(n);
  const double2* A2 = reinterpret_cast<const double2*>(Ap);
  double2* r2 = reinterpret_cast<double2*>(r);
  double s0 = 0.0, s1 = 0.0;
  for (long long i = S.i0; i < S.npair; i += 2 * S.stride) {
    const long long j = i + S.stride;
    const bool has1 = j < S.npair;
    const double2 aa = A2[i], ra = r2[i];
    double2 ab, rb;
    if (has1) { ab = A2[j]; rb = r2[j]; }
    double2 ro;
    ro.x = fma(-alpha, aa.x, ra.x); ro.y = fma(-alpha, aa.y, ra.y);
    r2[i] = ro;
    if (2 * i < n_owned) s0 = fma(ro.x, ro.x, s0);
    if (2 * i + 1 < n_owned) s0 = fma(ro.y, ro.y, s0);
    if (has1) {
      ro.x = fma(-alpha, ab.x, rb.x); ro.y = fma(-alpha, ab.y, rb.y);
      r2[j] = ro;
      if (2 * j < n_owned) s1 = fma(ro.x, ro.x, s1);
      if (2 * j + 1 < n_owned) s1 = fma(ro.y, ro.y, s1);
    }
  }
  if ((n & 1) && S.i0 == 0) {
    const long long i = n - 1;
    const double v = fma(-alpha, Ap[i], r[i]);
    r[i] = v;
    if (i < n_owned) s0 = fma(v, v, s0);
  }
  finish_reduction(s0 + s1, partials, counter, out);
}

// x += alpha_k p; beta = rr_{k+1}/rr_k; p = r + beta p
__global__ void __launch_bounds__(kDotThreads) pupdate_kernel(
    long long n, const double* __restrict__ r, double* __restrict__ p, double* __restrict__ x,
    const double* sc_new, const double* sc_old, const double* sc_pAp) {
  const double alpha = cg_alpha(sc_old, sc_pAp);
  const double rn = *sc_new, ro = *sc_old;
  const double beta = ro > 0.0 ? rn / ro : 0.0;
  const Span S = span(n);
  const double2* r2 = reinterpret_cast<const double2*>(r);
  double2* p2 = reinterpret_cast<double2*>(p);
  double2* x2 = reinterpret_cast<double2*>(x);
  for (long long i = S.i0; i < S.npair; i += 2 * S.stride) {
    const long long j = i + S.stride;
    const bool has1 = j < S.npair;
    const double2 ra = r2[i], pa = p2[i], xa = x2[i];
    double2 rb, pb, xb;
    if (has1) { rb = r2[j]; pb = p2[j]; xb = x2[j]; }
    double2 o;
    o.x = fma(alpha, pa.x, xa.x); o.y = fma(alpha, pa.y, xa.y);
    x2[i] = o;
    o.x = fma(beta, pa.x, ra.x); o.y = fma(beta, pa.y, ra.y);
    p2[i] = o;
    if (has1) {
      o.x = fma(alpha, pb.x, xb.x); o.y = fma(alpha, pb.y, xb.y);
      x2[j] = o;
      o.x = fma(beta, pb.x, rb.x); o.y = fma(beta, pb.y, rb.y);
      p2[j] = o;
    }
  }
  if ((n & 1) && S.i0 == 0) {
    const double pv = p[n - 1];
    x[n - 1] = fma(alpha, pv, x[n - 1]);
    p[n - 1] = fma(beta, pv, r[n - 1]);
  }
}

// Fixed-order sum of n partials into *out (fallback when the fused update
// cannot be launched after the operator left its p.Ap partials unsummed).
__global__ void __launch_bounds__(256) sum_partials_kernel(const double* part, long long n,
                                                           double* out) {
  __shared__ double sh[32];
  double v = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) v += part[i];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) *out = v;
}

// Small single-rank problems: update + p-update in ONE cooperative kernel
// (the first step of the fused CG iteration, §8(f) f1).  Phase 1: alpha =
// rr/pAp, r -= alpha Ap, block partials of r.r; grid barrier; every block sums
// the partials in block order (same value everywhere, deterministic), beta =
// rr'/rr; phase 2: x += alpha p, p = r + beta p.  Saves a launch and the
// last-block reduction per iteration.
__global__ void __launch_bounds__(kDotThreads) upd_fused_kernel(
    long long n, long long n_owned, const double* __restrict__ Ap, double* r, double* p,
    double* __restrict__ x, const double* sc_rr, double* sc_pAp, const double* pparts,
    long long npparts, double* partials, double* out, double* flag, GridBar* bar) {
  __shared__ double sh[32];
  __shared__ double pap_sh;
  double pAp;
  if (pparts) {
    // the operator kernel's per-CTA p.Ap partials, summed here in fixed order
    // (identical in every block) instead of by a separate launch
    double v = 0.0;
    for (long long i = threadIdx.x; i < npparts; i += blockDim.x) v += pparts[i];
    v = block_sum(v, sh);
    if (threadIdx.x == 0) {
      pap_sh = v;
      if (blockIdx.x == 0) *sc_pAp = v;
    }
    __syncthreads();
    pAp = pap_sh;
  } else {
    pAp = *sc_pAp;
  }
  if (!(pAp > 0.0) && blockIdx.x == 0 && threadIdx.x == 0) *flag = 1.0;
  const double alpha = pAp > 0.0 ? *sc_rr / pAp : 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double s = 0.0;
  for (long long i = t0; i < n; i += stride) {
    const double v = fma(-alpha, Ap[i], r[i]);
    r[i] = v;
    if (i < n_owned) s = fma(v, v, s);
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
  grid_barrier(bar);
  double rn = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) rn += __ldcg(partials + b);
  rn = block_sum(rn, sh);
  __shared__ double rn_sh;
  if (threadIdx.x == 0) {
    rn_sh = rn;
    if (blockIdx.x == 0) *out = rn;
  }
  __syncthreads();
  rn = rn_sh;
  const double ro = *sc_rr;
  const double beta = ro > 0.0 ? rn / ro : 0.0;
  for (long long i = t0; i < n; i += stride) {
    const double pv = p[i];
    x[i] = fma(alpha, pv, x[i]);
    p[i] = fma(beta, pv, r[i]);
  }
}

}  // namespace

hofem_status d2h(Mesh* m, void* dst, const void* src, size_t bytes, cudaStream_t s) {
  char* d = static_cast<char*>(dst);
  const char* sp = static_cast<const char*>(src);
  const size_t chunk = sizeof(double) * kPinDoubles;
  for (size_t off = 0; off < bytes; off += chunk) {
    const size_t nb = bytes - off < chunk ? bytes - off : chunk;
    HOFEM_CUDA(cudaMemcpyAsync(m->h_pin, sp + off, nb, cudaMemcpyDeviceToHost, s));
    HOFEM_CUDA(cudaStreamSynchronize(s));
    memcpy(d + off, m->h_pin, nb);
  }
  return HOFEM_OK;
}

hofem_status dot_local(Mesh* m, const double* a, const double* b, double* d_out,
                       cudaStream_t s) {
  dot_kernel<<<kDotBlocks, kDotThreads, 0, s>>>(m->n_owned, a, b, m->d_partials, m->d_counter,
                                                d_out);
  HOFEM_LAUNCHED();
  return HOFEM_OK;
}

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
  // stream-ordered allocations: no implicit device synchronization (a rank of
  // the loopback transport must never wait on another rank's pending kernels)
  if (!op->d_r) {
    if (cudaMallocAsync(&op->d_r, sizeof(double) * n, s) != cudaSuccess ||
        cudaMallocAsync(&op->d_p, sizeof(double) * n, s) != cudaSuccess ||
        cudaMallocAsync(&op->d_Ap, sizeof(double) * n, s) != cudaSuccess) {
      cudaGetLastError();
      set_error("hofem_cg: out of device memory for work vectors");
      return HOFEM_ERR_OOM;
    }
  }
  if (op->cg_cap < max_iter + 1) {
    if (op->d_cg) HOFEM_CUDA(cudaFreeAsync(op->d_cg, s));
    op->d_cg = nullptr;
    HOFEM_CUDA(cudaMallocAsync(&op->d_cg, sizeof(double) * (max_iter + 1 + 8), s));
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
  HOFEM_TRY(d2h(m, &rr0, rr, sizeof(double), s));

  const unsigned vgrid = kDotBlocks;
  // Whole solve in one persistent cooperative kernel (§8(f) f1): single rank,
  // fused operator; 2 = always; auto = local problems up to 256 Ki dofs, where
  // it measured fastest (gpurun_out/r2e, profiles/ab/r2_cg_modes.txt: BP3 p=5
  // 8^3 elements 31.4 vs 32.8 us/it); from ~0.5M dofs on, the per-iteration
  // kernels (fused cooperative update) win.  Convergence is tested every
  // iteration on the device (check_every does not apply).
  // (several ranks: with the kernel-initiated exchange, mesh mode 1 -- the
  // planes and both dot products are then exchanged inside the kernel)
  const bool persist = (m->nranks == 1 || m->xmode == 1) && fused_supported(op) &&
                       (op->opt_cg_persist == 2 || (op->opt_cg_persist == 1 && n <= (256LL << 10)));
  if (persist && !(rr0 == 0.0 && !fixed_iters)) {
    int* dres = reinterpret_cast<int*>(flag + 1);
    HOFEM_CUDA(cudaMemsetAsync(dres, 0, 4 * sizeof(int), s));
    hofem_status st = cg_persistent(op, x, op->d_r, op->d_p, op->d_Ap, rr, max_iter, fixed_iters,
                                    rel_tol, dres, s);
    if (st == HOFEM_OK) {
      int res[4] = {0, 0, 0, 0};
      HOFEM_TRY(d2h(m, res, dres, sizeof(res), s));
      const int k = res[0];
      m->xseq += (unsigned long long)res[2];  // the kernel's exchanges / chain reductions
      m->rseq += (unsigned long long)res[3];
      double rr_last = rr0;
      // stream-ordered copies only: a legacy-stream cudaMemcpy could wait on
      // another loopback rank's spinning kernel
      if (k > 0) HOFEM_TRY(d2h(m, &rr_last, rr + k, sizeof(double), s));
      hofem_status status = HOFEM_OK;
      if (res[1]) status = HOFEM_ERR_BREAKDOWN;
      else if (!fixed_iters && !(rr_last == 0.0 || sqrt(rr_last) <= rel_tol * sqrt(rr0)))
        status = HOFEM_NOT_CONVERGED;
      if (rr_history) HOFEM_TRY(d2h(m, rr_history, rr, sizeof(double) * (k + 1), s));
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
    if (op->opt_cg_persist == 2) return st;
    cudaGetLastError();  // e.g. grid not co-resident right now: per-iteration kernels
  }
  // fused update + p-update (one cooperative kernel) for small single-rank
  // problems; the grid is what the device holds co-resident (<= kDotBlocks)
  int ugrid = 0;
  if (op->opt_cg_fuse && m->nranks == 1 && (op->opt_cg_fuse == 2 || n <= (8LL << 20))) {
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, upd_fused_kernel, kDotThreads, 0) ==
            cudaSuccess &&
        per > 0) {
      ugrid = std::min(per * num_sms(), kDotBlocks);
      if (!op->d_bar) {
        if (cudaMallocAsync(&op->d_bar, sizeof(GridBar), s) != cudaSuccess ||
            cudaMemsetAsync(op->d_bar, 0, sizeof(GridBar), s) != cudaSuccess) {
          cudaGetLastError();
          op->d_bar = nullptr;
          ugrid = 0;
        }
      }
    } else {
      cudaGetLastError();
    }
  }
  int k = 0;
  hofem_status status = fixed_iters ? HOFEM_OK : HOFEM_NOT_CONVERGED;
  double rr_last = rr0;
  bool done = (rr0 == 0.0 && !fixed_iters);
  if (done) status = HOFEM_OK;
  while (!done && k < max_iter) {
    // Ap = A p and pAp = p.Ap: fused into the operator kernels when possible
    // (computed from the contributions they write), else a separate dot
    const double* pparts = nullptr;
    long long npparts = 0;
    if (fused_supported(op)) {
      if (ugrid > 0)
        HOFEM_TRY(apply_fused(op, op->d_p, op->d_Ap, s, pAp, &pparts, &npparts));
      else
        HOFEM_TRY(apply_fused(op, op->d_p, op->d_Ap, s, pAp));
    } else {
      HOFEM_TRY(apply_unfused(op, op->d_p, op->d_Ap, s));
      HOFEM_TRY(dot_local(m, op->d_p, op->d_Ap, pAp, s));
    }
    HOFEM_TRY(allreduce_sum(m, pAp, 1, s));
    bool fused_upd = false;
    if (ugrid > 0) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)ugrid);
      cfg.blockDim = dim3(kDotThreads);
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      const cudaError_t e =
          cudaLaunchKernelEx(&cfg, upd_fused_kernel, n, no, (const double*)op->d_Ap, op->d_r,
                             op->d_p, x, (const double*)(rr + k), pAp, pparts, npparts,
                             m->d_partials, rr + k + 1, flag, op->d_bar);
      if (e == cudaSuccess) {
        count_launch();
        fused_upd = true;
      } else {
        cudaGetLastError();  // e.g. grid no longer co-resident: separate kernels
        ugrid = 0;
      }
    }
    if (!fused_upd && pparts) {  // deferred p.Ap sum (fallback path)
      sum_partials_kernel<<<1, 256, 0, s>>>(pparts, npparts, pAp);
      HOFEM_LAUNCHED();
    }
    if (!fused_upd) {
      update_kernel<<<kDotBlocks, kDotThreads, 0, s>>>(n, no, op->d_Ap, op->d_r, rr + k, pAp,
                                                       m->d_partials, m->d_counter, rr + k + 1,
                                                       flag);
      HOFEM_LAUNCHED();
      HOFEM_TRY(allreduce_sum(m, rr + k + 1, 1, s));
      pupdate_kernel<<<vgrid, kDotThreads, 0, s>>>(n, op->d_r, op->d_p, x, rr + k + 1, rr + k,
                                                   pAp);
      HOFEM_LAUNCHED();
    }
    ++k;
    if ((!fixed_iters && k % check_every == 0) || k == max_iter) {
      double h[2];
      HOFEM_TRY(d2h(m, &h[0], rr + k, sizeof(double), s));
      HOFEM_TRY(d2h(m, &h[1], flag, sizeof(double), s));
      rr_last = h[0];
      if (h[1] != 0.0) { status = HOFEM_ERR_BREAKDOWN; break; }
      if (!fixed_iters && (rr_last == 0.0 || sqrt(rr_last) <= rel_tol * sqrt(rr0))) {
        status = HOFEM_OK;
        done = true;
      }
    }
  }
  if (rr_history) HOFEM_TRY(d2h(m, rr_history, rr, sizeof(double) * (k + 1), s));
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
