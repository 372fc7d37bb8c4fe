// fused_p.cu -- instantiation of the fused column kernels for one P1 = p+1
// (compiled once per P1 with -DHOFEM_P1=<P1>, so the builds run in parallel).
#include <string.h>

#include "fused_impl.cuh"

#ifndef HOFEM_P1
#error "compile with -DHOFEM_P1=<p+1>"
#endif

namespace hofem {

namespace {

template <class K>
cudaError_t set_smem(K kern, int bytes, bool* done) {
  if (*done) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) *done = true;
  return e;
}

template <int KIND, int P1, int Q>
auto mma_kernel() {
  using S = ShapeE<P1>;
  return fused_elem_mma<KIND, P1, Q, S::BX, S::BY, S::MINB>;
}

template <int KIND, int P1, int Q>
cudaError_t launch_general(const double* B, const double* G, const ColArgs& A, int grid,
                           cudaStream_t s) {
  using S = ShapeE<P1>;
  constexpr int SMEM = smem_bytes_elem<KIND, P1, Q, S::BX, S::BY>();
  Tab<P1, Q> T;
  fill_tab(T, B, G);
  auto kern = mma_kernel<KIND, P1, Q>();
  static bool attr_done = false;
  cudaError_t e = set_smem(kern, SMEM, &attr_done);
  if (e != cudaSuccess) return e;
  kern<<<grid, S::BX * S::BY * 32, SMEM, s>>>(T, A);
  return cudaPeekAtLastError();
}

template <int KIND, int P1, int Q>
auto simt_kernel() {
  using S = ShapeSK<KIND, P1>;
  return fused_elem_simt<KIND, P1, Q, S::BX, S::BY, S::NT, S::MAXR, HOFEM_SIMT_EO != 0>;
}
template <int KIND, int P1, int Q>
constexpr int simt_smem() {
  using S = ShapeSK<KIND, P1>;
  return CfgS<KIND, P1, Q, S::BX, S::BY>::SMEM_BYTES;
}

template <int KIND, int P1, int Q>
cudaError_t launch_simt(const double* B, const double* G, const ColArgs& A, int grid,
                        cudaStream_t s) {
  using S = ShapeSK<KIND, P1>;
  constexpr int SMEM = simt_smem<KIND, P1, Q>();
  Tab<P1, Q> T;
  fill_tab(T, B, G);
  auto kern = simt_kernel<KIND, P1, Q>();
  static bool attr_done = false;
  cudaError_t e = set_smem(kern, SMEM, &attr_done);
  if (e != cudaSuccess) return e;
  if (!A.infix) {
    kern<<<grid, S::NT, SMEM, s>>>(T, A);
    return cudaPeekAtLastError();
  }
  // in-kernel fix-up behind a grid barrier: cooperative launch, so all CTAs
  // are guaranteed co-resident (or the launch fails instead of deadlocking)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(S::NT);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, T, A);
}

// Resident CTAs per SM of a kernel (occupancy API; registers and shared memory
// both count), so the persistent grid never oversubscribes.
template <class K>
int occupancy(K kern, int threads, int smem, int fallback) {
  int v = 0;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) ==
          cudaSuccess &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, threads, smem) == cudaSuccess &&
      v > 0)
    return v;
  cudaGetLastError();
  return fallback;
}

template <int KIND, int P1, int Q>
int mma_ctas_per_sm() {
  using S = ShapeE<P1>;
  static const int n = occupancy(mma_kernel<KIND, P1, Q>(), 32 * S::BX * S::BY,
                                 smem_bytes_elem<KIND, P1, Q, S::BX, S::BY>(), S::MINB);
  return n;
}

// Resident CTAs per SM of a SIMT instantiation (occupancy API; registers and
// shared memory both count), so the persistent grid never oversubscribes.
template <int KIND, int P1, int Q>
int simt_ctas_per_sm() {
  static int n = 0;
  if (n == 0) {
    auto kern = simt_kernel<KIND, P1, Q>();
    constexpr int SMEM = simt_smem<KIND, P1, Q>();
    int v = 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) ==
            cudaSuccess &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, ShapeSK<KIND, P1>::NT, SMEM) ==
            cudaSuccess &&
        v > 0)
      n = v;
    else {
      cudaGetLastError();
      n = ShapeSK<KIND, P1>::CPS;
    }
  }
  return n;
}

// Default fused variant per P1 (measured): 0 tensor-core, 1 SIMT.
// With even-odd contractions the SIMT kernel is faster at every p and kind
// (gpurun_out/e1: BP3 p=5 1.37 ms vs 1.62 ms DMMA; BP1 p=8 31.5 us vs 45 us).
constexpr int default_for(int) { return 1; }

int pick(int variant, int kind) { return variant < 0 ? default_for(kind) : variant; }

}  // namespace

template <>
int fused_default_variant<HOFEM_P1>(int kind) {
  return default_for(kind);
}

namespace {

template <int P1>
cudaError_t launch_colloc(const double* G, const ColArgs& A, int grid, cudaStream_t s) {
  using S = Shape<P1>;
  constexpr int SMEM = smem_bytes<KIND_COLLOC, P1, P1, S::BX, S::BY, S::NBUF>();
  Tab<P1, P1> T;
  fill_tab(T, nullptr, G);
  auto kern = fused_column_colloc<P1, S::BX, S::BY, S::NT, S::NBUF, S::MAXR>;
  static bool attr_done = false;
  cudaError_t e = set_smem(kern, SMEM, &attr_done);
  if (e != cudaSuccess) return e;
  kern<<<grid, S::NT, SMEM, s>>>(T, A);
  return cudaPeekAtLastError();
}

}  // namespace

template <>
bool fused_launch<HOFEM_P1>(int kind, int variant, int Q, const double* B, const double* G,
                            const ColArgs& A, int grid, cudaStream_t s, cudaError_t* err) {
  constexpr int P1 = HOFEM_P1;
  if (kind == KIND_COLLOC) {
    if (Q != P1) return false;
    *err = variant == 1 ? launch_simt<KIND_COLLOC, P1, P1>(B, G, A, grid, s)
                        : launch_colloc<P1>(G, A, grid, s);
    return true;
  }
  if (pick(variant, kind) == 1) {
    if (Q == P1 + 1) {
      *err = kind == KIND_MASS ? launch_simt<KIND_MASS, P1, P1 + 1>(B, G, A, grid, s)
                               : launch_simt<KIND_DIFF, P1, P1 + 1>(B, G, A, grid, s);
      return true;
    }
    if (Q == P1) {
      *err = kind == KIND_MASS ? launch_simt<KIND_MASS, P1, P1>(B, G, A, grid, s)
                               : launch_simt<KIND_DIFF, P1, P1>(B, G, A, grid, s);
      return true;
    }
    return false;
  }
  if (Q == P1 + 1) {
    *err = kind == KIND_MASS ? launch_general<KIND_MASS, P1, P1 + 1>(B, G, A, grid, s)
                             : launch_general<KIND_DIFF, P1, P1 + 1>(B, G, A, grid, s);
    return true;
  }
  if (Q == P1) {
    *err = kind == KIND_MASS ? launch_general<KIND_MASS, P1, P1>(B, G, A, grid, s)
                             : launch_general<KIND_DIFF, P1, P1>(B, G, A, grid, s);
    return true;
  }
  return false;
}

template <>
FusedLaunch fused_shape<HOFEM_P1>(int kind, int variant) {
  constexpr int p = HOFEM_P1 - 1;
  if (kind == KIND_COLLOC) {
    if (variant == 1) {
      using S = ShapeSC<HOFEM_P1>;
      return FusedLaunch{S::BX, S::BY, FaceLayout<p, p * S::BX + 1, p * S::BY + 1>::FB,
                         simt_ctas_per_sm<KIND_COLLOC, HOFEM_P1, HOFEM_P1>()};
    }
    using S = Shape<HOFEM_P1>;
    return FusedLaunch{S::BX, S::BY, FaceLayout<p, p * S::BX + 1, p * S::BY + 1>::FB, 1};
  }
  if (pick(variant, kind) == 1) {
    if (kind == KIND_MASS) {
      using S = ShapeSK<KIND_MASS, HOFEM_P1>;
      return FusedLaunch{S::BX, S::BY, FaceLayout<p, p * S::BX + 1, p * S::BY + 1>::FB,
                         simt_ctas_per_sm<KIND_MASS, HOFEM_P1, HOFEM_P1 + 1>()};
    }
    using S = ShapeS<HOFEM_P1>;
    return FusedLaunch{S::BX, S::BY, FaceLayout<p, p * S::BX + 1, p * S::BY + 1>::FB,
                       simt_ctas_per_sm<KIND_DIFF, HOFEM_P1, HOFEM_P1 + 1>()};
  }
  using S = ShapeE<HOFEM_P1>;
  const int cps = kind == KIND_MASS ? mma_ctas_per_sm<KIND_MASS, HOFEM_P1, HOFEM_P1 + 1>()
                                    : mma_ctas_per_sm<KIND_DIFF, HOFEM_P1, HOFEM_P1 + 1>();
  return FusedLaunch{S::BX, S::BY, FaceLayout<p, p * S::BX + 1, p * S::BY + 1>::FB, cps};
}

}  // namespace hofem
