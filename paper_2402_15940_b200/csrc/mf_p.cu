// mf_p.cu -- instantiation of the fully matrix-free diffusion kernel
// (mf_impl.cuh) for one P1 (compiled once per P1 with -DHOFEM_P1=<P1>).
#include "mf_impl.cuh"

#ifndef HOFEM_P1
#error "compile with -DHOFEM_P1=<p+1>"
#endif

namespace hofem {

template <>
int mf_batch_elems<HOFEM_P1>() {
  return ShapeMF<HOFEM_P1>::NE;
}

template <>
cudaError_t mf_launch<HOFEM_P1>(int Q, const double* B, const double* G, const double* w,
                                const MFArgs& A, int* grid_io, cudaStream_t s) {
  constexpr int P1 = HOFEM_P1, QQ = HOFEM_P1 + 1;
  using S = ShapeMF<P1>;
  using C = CfgMF<P1, QQ, S::NE>;
  if (Q != QQ) return cudaErrorInvalidValue;
  auto kern = mf_diffusion_simt<P1, QQ, S::NE, S::NT>;
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
  fill_tab(T, B, G);
  TabW<P1, QQ> TW;
  for (int i = 0; i < QQ; ++i) TW.w[i] = w[i];
  const long long want = (long long)per_sm * num_sms();
  const int grid = (int)(A.nbatch < want ? A.nbatch : want);
  *grid_io = grid;
  if (grid < 1) return cudaSuccess;
  kern<<<grid, S::NT, C::SMEM_BYTES, s>>>(T, TW, A);
  return cudaPeekAtLastError();
}

}  // namespace hofem
