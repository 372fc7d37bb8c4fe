// fused_p.cu -- instantiation of the fused SIMT kernels for one P1 = p+1
// (compiled once per P1 with -DHOFEM_P1=<P1>, so the builds run in parallel):
// the operator kernel fused_elem_simt and the persistent CG kernel
// cg_persistent_simt, for mass (Gauss Q = P1+1, P1), diffusion (same) and
// collocated diffusion (GLL Q = P1).
#include <string.h>

#include "fused_impl.cuh"

#ifndef HOFEM_P1
#error "compile with -DHOFEM_P1=<p+1>"
#endif

namespace hofem {

namespace {

template <int KIND, int P1, int Q>
auto simt_kernel() {
  using S = ShapeSK<KIND, P1>;
  return fused_elem_simt<KIND, P1, Q, S::BX, S::BY, S::NT, S::MAXR, HOFEM_SIMT_EO != 0>;
}
template <int KIND, int P1, int Q>
auto cg_kernel() {
  using S = ShapeSK<KIND, P1>;
  return cg_persistent_simt<KIND, P1, Q, S::BX, S::BY, S::NT, cg_maxr(S::MAXR),
                            HOFEM_SIMT_EO != 0>;
}
template <int KIND, int P1, int Q>
constexpr int simt_smem() {
  using S = ShapeSK<KIND, P1>;
  return CfgS<KIND, P1, Q, S::BX, S::BY>::SMEM_BYTES;
}

template <class K, class... Args>
cudaError_t launch(K kern, int grid, int nt, int smem, bool coop, cudaStream_t s,
                   Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)nt);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = coop ? at : nullptr;
  cfg.numAttrs = coop ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <class K>
cudaError_t set_smem(K kern, int bytes) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

template <int KIND, int P1, int Q>
cudaError_t launch_simt(const double* B, const double* G, const ColArgs& A, int grid, bool coop,
                        cudaStream_t s) {
  using S = ShapeSK<KIND, P1>;
  constexpr int SMEM = simt_smem<KIND, P1, Q>();
  Tab<P1, Q> T;
  fill_tab(T, B, G);
  auto kern = simt_kernel<KIND, P1, Q>();
  static const cudaError_t attr = set_smem(kern, SMEM);
  if (attr != cudaSuccess) return attr;
  return launch(kern, grid, S::NT, SMEM, coop, s, T, A);
}

template <int KIND, int P1, int Q>
cudaError_t launch_cg(const double* B, const double* G, const ColArgs& A, const CGArgs& CG,
                      int grid, cudaStream_t s) {
  using S = ShapeSK<KIND, P1>;
  constexpr int SMEM = simt_smem<KIND, P1, Q>();
  Tab<P1, Q> T;
  fill_tab(T, B, G);
  auto kern = cg_kernel<KIND, P1, Q>();
  static const cudaError_t attr = set_smem(kern, SMEM);
  if (attr != cudaSuccess) return attr;
  return launch(kern, grid, S::NT, SMEM, true, s, T, A, CG);
}

// Resident CTAs per SM of a kernel (occupancy API; registers and shared memory
// both count), so the persistent grid never oversubscribes and a cooperative
// launch of that grid fits.
template <class K>
int occupancy(K kern, int threads, int smem, int fallback) {
  int v = 0;
  if (set_smem(kern, smem) == cudaSuccess &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, threads, smem) == cudaSuccess &&
      v > 0)
    return v;
  cudaGetLastError();
  return fallback;
}

template <int KIND, int P1, int Q>
int simt_ctas_per_sm() {
  using S = ShapeSK<KIND, P1>;
  static const int n =
      occupancy(simt_kernel<KIND, P1, Q>(), S::NT, simt_smem<KIND, P1, Q>(), S::CPS);
  return n;
}
template <int KIND, int P1, int Q>
int cg_ctas_per_sm() {
  using S = ShapeSK<KIND, P1>;
  static const int n = occupancy(cg_kernel<KIND, P1, Q>(), S::NT, simt_smem<KIND, P1, Q>(), 1);
  return n;
}

template <int KIND, int P1>
FusedLaunch shape_of(int Q) {
  constexpr int p = P1 - 1;
  using S = ShapeSK<KIND, P1>;
  const bool q1 = KIND == KIND_COLLOC || Q == P1;
  const int cps = q1 ? simt_ctas_per_sm<KIND, P1, P1>() : simt_ctas_per_sm<KIND, P1, P1 + 1>();
  const int cpc = q1 ? cg_ctas_per_sm<KIND, P1, P1>() : cg_ctas_per_sm<KIND, P1, P1 + 1>();
  return FusedLaunch{S::BX, S::BY, FaceLayout<p, p * S::BX + 1, p * S::BY + 1>::FB, cps, cpc};
}

}  // namespace

template <>
bool fused_launch<HOFEM_P1>(int kind, int Q, const double* B, const double* G, const ColArgs& A,
                            int grid, bool coop, cudaStream_t s, cudaError_t* err) {
  constexpr int P1 = HOFEM_P1;
  if (kind == KIND_COLLOC) {
    if (Q != P1) return false;
    *err = launch_simt<KIND_COLLOC, P1, P1>(B, G, A, grid, coop, s);
    return true;
  }
  if (Q == P1 + 1) {
    *err = kind == KIND_MASS ? launch_simt<KIND_MASS, P1, P1 + 1>(B, G, A, grid, coop, s)
                             : launch_simt<KIND_DIFF, P1, P1 + 1>(B, G, A, grid, coop, s);
    return true;
  }
  if (Q == P1) {
    *err = kind == KIND_MASS ? launch_simt<KIND_MASS, P1, P1>(B, G, A, grid, coop, s)
                             : launch_simt<KIND_DIFF, P1, P1>(B, G, A, grid, coop, s);
    return true;
  }
  return false;
}

template <>
bool cg_launch<HOFEM_P1>(int kind, int Q, const double* B, const double* G, const ColArgs& A,
                         const CGArgs& CG, int grid, cudaStream_t s, cudaError_t* err) {
  constexpr int P1 = HOFEM_P1;
  if (kind == KIND_COLLOC) {
    if (Q != P1) return false;
    *err = launch_cg<KIND_COLLOC, P1, P1>(B, G, A, CG, grid, s);
    return true;
  }
  if (Q == P1 + 1) {
    *err = kind == KIND_MASS ? launch_cg<KIND_MASS, P1, P1 + 1>(B, G, A, CG, grid, s)
                             : launch_cg<KIND_DIFF, P1, P1 + 1>(B, G, A, CG, grid, s);
    return true;
  }
  if (Q == P1) {
    *err = kind == KIND_MASS ? launch_cg<KIND_MASS, P1, P1>(B, G, A, CG, grid, s)
                             : launch_cg<KIND_DIFF, P1, P1>(B, G, A, CG, grid, s);
    return true;
  }
  return false;
}

template <>
FusedLaunch fused_shape<HOFEM_P1>(int kind, int Q) {
  constexpr int P1 = HOFEM_P1;
  if (kind == KIND_COLLOC) return shape_of<KIND_COLLOC, P1>(P1);
  if (kind == KIND_MASS) return shape_of<KIND_MASS, P1>(Q);
  return shape_of<KIND_DIFF, P1>(Q);
}

}  // namespace hofem
