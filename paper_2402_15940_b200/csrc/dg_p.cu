// dg_p.cu -- instantiation of the DG mass kernel (dg_impl.cuh) for one P1
// (compiled once per P1 with -DHOFEM_P1=<P1>, like fused_p.cu).
#include "dg_impl.cuh"

#ifndef HOFEM_P1
#error "compile with -DHOFEM_P1=<p+1>"
#endif

namespace hofem {

template <>
int dg_batch_elems<HOFEM_P1>() {
  return ShapeDG<HOFEM_P1>::NE;
}

template <>
cudaError_t dg_launch<HOFEM_P1>(int Q, const double* B, const DGArgs& A, int* grid_io,
                                cudaStream_t s) {
  constexpr int P1 = HOFEM_P1, QQ = HOFEM_P1 + 1;
  using S = ShapeDG<P1>;
  using C = CfgDG<P1, QQ, S::NE>;
  if (Q != QQ) return cudaErrorInvalidValue;
  auto kern = dg_mass_simt<P1, QQ, S::NE, S::NT>;
  static const int per_sm = [&] {
    int v = 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES) !=
            cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, S::NT, C::SMEM_BYTES) !=
            cudaSuccess ||
        v < 1) {
      cudaGetLastError();
      v = 1;
    }
    return v;
  }();
  Tab<P1, QQ> T;
  double G[QQ * P1] = {};
  fill_tab(T, B, G);
  const long long want = (long long)per_sm * num_sms();
  const int grid = (int)(A.nbatch < want ? A.nbatch : want);
  *grid_io = grid;
  if (grid < 1) return cudaSuccess;
  kern<<<grid, S::NT, C::SMEM_BYTES, s>>>(T, A);
  return cudaPeekAtLastError();
}

}  // namespace hofem
