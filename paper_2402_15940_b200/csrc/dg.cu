// dg.cu -- host side of the DG (L2) mass operator (
// PAPER.md:205-211, §2.4.1): geometry qdata W*detJ from the mesh's isoparametric
// map (the BP1 qdata builder), the DG basis table (tables.cpp build_dg_table),
// and the launch of dg_mass_simt (dg_impl.cuh).
#include "dg_impl.cuh"

namespace hofem {

#define HOFEM_DG_FOR_P1(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9)
#define HOFEM_DG_DECL(P1)                                                                   \
  template <>                                                                               \
  cudaError_t dg_launch<P1>(int, const double*, const DGArgs&, int*, cudaStream_t);         \
  template <>                                                                               \
  int dg_batch_elems<P1>();
HOFEM_DG_FOR_P1(HOFEM_DG_DECL)
#undef HOFEM_DG_DECL

hofem_status dg_create(Mesh* m, int q_override, cudaStream_t s, DGOp** out) {
  const int Q = q_override ? q_override : m->p + 2;
  if (Q != m->P1 + 1) {
    set_error("hofem_dg_create: the DG kernel is instantiated for the Gauss rule Q = p+2 only");
    return HOFEM_ERR_ARG;
  }
  auto* dg = new DGOp();
  dg->mesh = m;
  dg->Q = Q;
  dg->nd = m->P1 * m->P1 * m->P1;
  dg->n_local = m->elems * dg->nd;
  if (build_dg_table(m->p, Q, dg->B)) {
    delete dg;
    set_error("hofem_dg_create: DG basis table failed");
    return HOFEM_ERR_ARG;
  }
  // the geometry of the DG operator: W*detJ at the Gauss points, exactly the BP1 qdata
  hofem_status st = op_new(m, HOFEM_MASS, HOFEM_GAUSS, Q, HOFEM_BC_NONE, s, &dg->geo);
  if (st != HOFEM_OK) {
    delete dg;
    return st;
  }
  *out = dg;
  return HOFEM_OK;
}

void dg_destroy(DGOp* dg) {
  if (!dg) return;
  op_free(dg->geo);
  delete dg;
}

hofem_status dg_apply(DGOp* dg, const double* x, double* y, cudaStream_t s) {
  Mesh* m = dg->mesh;
  DGArgs A;
  A.x = x;
  A.y = y;
  A.qd = dg->geo->d_qdata;
  A.E = m->elems;
  int NE = 0;
  switch (m->P1) {
#define HOFEM_CASE(P) \
  case P:             \
    NE = dg_batch_elems<P>(); \
    break;
    HOFEM_DG_FOR_P1(HOFEM_CASE)
#undef HOFEM_CASE
  }
  if (NE <= 0) { set_error("hofem_dg_apply: unsupported p"); return HOFEM_ERR_ARG; }
  A.nbatch = (A.E + NE - 1) / NE;
  if (A.nbatch == 0) return HOFEM_OK;
  cudaError_t e = cudaErrorInvalidValue;
  int grid = 0;
  switch (m->P1) {
#define HOFEM_CASE(P) \
  case P:             \
    e = dg_launch<P>(dg->Q, dg->B, A, &grid, s); \
    break;
    HOFEM_DG_FOR_P1(HOFEM_CASE)
#undef HOFEM_CASE
  }
  if (e != cudaSuccess) return cuda_status(e, "DG mass kernel launch");
  count_launch();
  dg->grid = grid;
  return HOFEM_OK;
}

hofem_status dg_fill_random(const DGOp* dg, unsigned long long seed, double* x, cudaStream_t s) {
  const Mesh* m = dg->mesh;
  // global DG index: (global element) * P1^3 + local node (reading R16)
  const long long g0 = (long long)m->z0 * m->nx * m->ny * dg->nd;
  return fill_random_range(seed, g0, dg->n_local, x, s);
}

}  // namespace hofem
