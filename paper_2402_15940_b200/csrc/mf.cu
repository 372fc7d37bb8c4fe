// mf.cu -- host side of the fully matrix-free BP3 apply (
// PAPER.md:145): launches mf_diffusion_simt (mf_impl.cuh) into the operator's
// E-vector scratch, then the deterministic transposed-offset scatter with the
// Dirichlet rows y = x (reading R6) and, with > 1 rank, the interface exchange.
#include "mf_impl.cuh"

namespace hofem {

#define HOFEM_MF_FOR_P1(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9)
#define HOFEM_MF_DECL(P1)                                                                  \
  template <>                                                                              \
  cudaError_t mf_launch<P1>(int, const double*, const double*, const double*,             \
                            const MFArgs&, int*, cudaStream_t);                           \
  template <>                                                                              \
  int mf_batch_elems<P1>();
HOFEM_MF_FOR_P1(HOFEM_MF_DECL)
#undef HOFEM_MF_DECL

hofem_status apply_mf(Op* op, const double* x, double* y, cudaStream_t s) {
  Mesh* m = op->mesh;
  if (op->kind != HOFEM_DIFFUSION || op->rule != HOFEM_GAUSS || op->Q != m->P1 + 1) {
    set_error("fully matrix-free apply: BP3 diffusion with the Gauss rule Q = p+2 only");
    return HOFEM_ERR_ARG;
  }
  HOFEM_TRY(mesh_build_restriction(m, s));
  const long long ent = m->elems * m->P1 * m->P1 * m->P1;
  if (!op->d_eout) {
    // stream-ordered (no device-wide synchronization between exchanges)
    if (cudaMallocAsync(&op->d_ein, sizeof(double) * (ent + 1), s) != cudaSuccess ||
        cudaMallocAsync(&op->d_eout, sizeof(double) * (ent + 1), s) != cudaSuccess) {
      cudaGetLastError();
      set_error("fully matrix-free apply: out of device memory for the E-vector");
      return HOFEM_ERR_OOM;
    }
  }
  MFArgs A;
  A.x = x;
  A.coords = m->d_coords;
  A.ye = op->d_eout;
  A.nx = m->nx; A.ny = m->ny; A.nzl = m->nzl;
  A.Nx = m->Nx; A.Ny = m->Ny; A.n_local = m->n_local;
  A.K0 = (long long)m->p * m->z0; A.NzG = m->NzG;
  A.bc = op->bc;
  A.E = m->elems;
  int NE = 0;
  switch (m->P1) {
#define HOFEM_CASE(P) \
  case P:             \
    NE = mf_batch_elems<P>(); \
    break;
    HOFEM_MF_FOR_P1(HOFEM_CASE)
#undef HOFEM_CASE
  }
  if (NE <= 0) { set_error("fully matrix-free apply: unsupported p"); return HOFEM_ERR_ARG; }
  A.nbatch = (A.E + NE - 1) / NE;
  if (A.nbatch > 0) {
    cudaError_t e = cudaErrorInvalidValue;
    int grid = 0;
    switch (m->P1) {
#define HOFEM_CASE(P)                                                            \
  case P:                                                                        \
    e = mf_launch<P>(op->Q, op->tab.B, op->tab.G, op->tab.w, A, &grid, s); \
    break;
      HOFEM_MF_FOR_P1(HOFEM_CASE)
#undef HOFEM_CASE
    }
    if (e != cudaSuccess) return cuda_status(e, "fully matrix-free kernel launch");
    count_launch();
  }
  HOFEM_TRY(scatter_evector_bc(op, op->d_eout, y, op->bc ? 1 : 0, x, s));
  return exchange_planes(op, x, y, s);
}

}  // namespace hofem
