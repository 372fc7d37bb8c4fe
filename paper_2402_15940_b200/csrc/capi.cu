// capi.cu -- the C ABI declared in include/hofem.h: argument checking, handle
// lifetime, error reporting, and the host-side orchestration of the kernels.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <cstdint>

#include "internal.h"

namespace hofem {

namespace {
thread_local char g_err[512] = "no error";
std::atomic<long long> g_launches{0};
}  // namespace

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

hofem_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return HOFEM_OK;
  set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  if (e == cudaErrorMemoryAllocation) return HOFEM_ERR_OOM;
  return HOFEM_ERR_CUDA;
}

void count_launch(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

hofem_status profile_enable(int on);
hofem_status profile_read(hofem_profile_stats* out);

hofem_status cg_solve(Op* op, const double* b, double* x, double rel_tol, int max_iter,
                      int fixed_iters, int check_every, double* rr_history,
                      hofem_cg_stats* stats, cudaStream_t s);

hofem_status apply_any(Op* op, const double* x, double* y, cudaStream_t s) {
  if (fused_supported(op)) return apply_fused(op, x, y, s);
  return apply_unfused(op, x, y, s);
}

namespace {

template <class T>
hofem_status dalloc(T** p, long long n, const char* what) {
  if (cudaMalloc(p, sizeof(T) * (n > 0 ? n : 1)) != cudaSuccess) {
    cudaGetLastError();
    set_error("%s: out of device memory (%lld elements)", what, n);
    return HOFEM_ERR_OOM;
  }
  return HOFEM_OK;
}

void free_mesh(Mesh* m) {
  if (!m) return;
  mesh_release_exchange(m);
  cudaFree(m->d_xi); cudaFree(m->d_coords);
  cudaFree(m->d_l2e); cudaFree(m->d_toff); cudaFree(m->d_tidx);
  cudaFree(m->d_partials); cudaFree(m->d_counter); cudaFree(m->d_scalars);
  cudaFree(m->d_recv); cudaFree(m->d_send);
  if (m->h_pin) cudaFreeHost(m->h_pin);
  delete m;
}

void free_op(Op* op) {
  if (!op) return;
  cudaFree(op->d_B); cudaFree(op->d_G); cudaFree(op->d_qdata);
  cudaFree(op->d_ein); cudaFree(op->d_eout); cudaFree(op->d_bbuf);
  cudaFree(op->d_r); cudaFree(op->d_p); cudaFree(op->d_Ap); cudaFree(op->d_cg);
  cudaFree(op->d_dotp); cudaFree(op->d_bar); cudaFree(op->d_cgparts);
  delete op;
}

inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

// Vector arguments must be 16-byte aligned (the vector kernels use 16-byte
// loads); a misaligned pointer is an argument error, never a device fault.
inline bool aligned(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
#define HOFEM_ALIGNED(fn, ...)                                                       \
  do {                                                                               \
    const void* ps_[] = {__VA_ARGS__};                                               \
    for (const void* q_ : ps_)                                                       \
      if (!aligned(q_)) {                                                            \
        set_error("%s: vector pointer %p is not 16-byte aligned", fn, q_);           \
        return HOFEM_ERR_ARG;                                                        \
      }                                                                              \
  } while (0)

}  // namespace

void op_free(Op* op) { free_op(op); }
void mesh_free(Mesh* m) { free_mesh(m); }

// Build a mesh (hofem_mesh_create without the handle checks); SYNC.  Also used
// for the p-multigrid levels.
hofem_status mesh_new(const hofem_mesh_desc* d, Comm* c, cudaStream_t stream, Mesh** mesh_out) {
  if (d->p < 1 || d->p > kMaxP || d->nx < 1 || d->ny < 1 || d->nz_global < 1 ||
      !(d->extent[0] > 0) || !(d->extent[1] > 0) || !(d->extent[2] > 0)) {
    set_error("hofem_mesh_create: need 1<=p<=%d, n>=1, extents>0", kMaxP);
    return HOFEM_ERR_ARG;
  }
  const int R = c ? c->nranks : 1, r = c ? c->rank : 0;
  if (d->nz_global % R != 0) {
    set_error("hofem_mesh_create: nranks=%d must divide nz_global=%d", R, d->nz_global);
    return HOFEM_ERR_ARG;
  }
  int dev = 0;
  HOFEM_CUDA(cudaGetDevice(&dev));
  auto* m = new Mesh();
  m->desc = *d;
  m->comm = c;
  m->rank = r; m->nranks = R;
  m->p = d->p; m->P1 = d->p + 1;
  m->nx = d->nx; m->ny = d->ny; m->nzl = d->nz_global / R; m->z0 = r * m->nzl;
  m->Nx = (long long)d->p * d->nx + 1;
  m->Ny = (long long)d->p * d->ny + 1;
  m->Nzl = (long long)d->p * m->nzl + 1;
  m->NzG = (long long)d->p * d->nz_global + 1;
  m->plane = m->Nx * m->Ny;
  m->n_local = m->plane * m->Nzl;
  m->n_owned = (r == R - 1) ? m->n_local : m->n_local - m->plane;
  m->n_global = m->plane * m->NzG;
  m->elems = (long long)d->nx * d->ny * m->nzl;
  double xi[kMaxP + 1], w[kMaxP + 1];
  gll_nodes_weights(d->p, xi, w);
  hofem_status st = HOFEM_OK;
#define CK(x) do { st = (x); if (st != HOFEM_OK) { free_mesh(m); return st; } } while (0)
  CK(dalloc(&m->d_xi, m->P1, "mesh"));
  CK(dalloc(&m->d_coords, 3 * m->n_local, "mesh coords"));
  CK(dalloc(&m->d_partials, 4 * kNumSMs + 64, "mesh"));
  CK(dalloc(&m->d_counter, 4, "mesh"));
  CK(dalloc(&m->d_scalars, 16, "mesh"));
  if (R > 1) CK(dalloc(&m->d_recv, 2 * m->plane, "mesh planes"));
  CK(cuda_status(cudaHostAlloc(reinterpret_cast<void**>(&m->h_pin), sizeof(double) * kPinDoubles,
                               cudaHostAllocDefault), "mesh pinned staging"));
  CK(cuda_status(cudaMemcpyAsync(m->d_xi, xi, sizeof(double) * m->P1, cudaMemcpyHostToDevice,
                                 stream), "mesh upload"));
  CK(cuda_status(cudaMemsetAsync(m->d_counter, 0, 4 * sizeof(unsigned), stream), "memset"));
  CK(mesh_build_coords(m, stream));
  CK(cuda_status(cudaStreamSynchronize(stream), "mesh_create sync"));
#undef CK
  *mesh_out = m;
  return HOFEM_OK;
}


// Build a partially assembled operator (hofem_op_create without the handle
// checks); also used for the DG operator's geometry and the p-multigrid levels.
hofem_status op_new(Mesh* m, int kind, int rule, int q_override, int bc, cudaStream_t stream,
                    Op** op_out) {
  if ((kind != HOFEM_MASS && kind != HOFEM_DIFFUSION) || (rule != HOFEM_GAUSS && rule != HOFEM_GLL) ||
      (bc != HOFEM_BC_NONE && bc != HOFEM_BC_DIRICHLET) || q_override < 0 || q_override > kMaxQ) {
    set_error("hofem_op_create: bad kind/rule/bc/q_override");
    return HOFEM_ERR_ARG;
  }
  const int Q = q_override ? q_override : (rule == HOFEM_GAUSS ? m->p + 2 : m->p + 1);
  if (rule == HOFEM_GLL && Q < 2) { set_error("hofem_op_create: GLL needs Q>=2"); return HOFEM_ERR_ARG; }
  auto* op = new Op();
  op->mesh = m; op->kind = kind; op->rule = rule; op->Q = Q; op->bc = bc;
  op->nc = kind == HOFEM_MASS ? 1 : 6;
  if (build_tables(m->p, Q, rule, &op->tab)) {
    delete op;
    set_error("hofem_op_create: 1D tables failed");
    return HOFEM_ERR_ARG;
  }
  hofem_status st = HOFEM_OK;
#define CK(x) do { st = (x); if (st != HOFEM_OK) { free_op(op); return st; } } while (0)
  const int P1 = m->P1;
  op->qcount = m->elems * op->nc * (long long)Q * Q * Q;
  CK(dalloc(&op->d_B, Q * P1, "op tables"));
  CK(dalloc(&op->d_G, Q * P1, "op tables"));
  CK(dalloc(&op->d_qdata, op->qcount + 2, "qdata"));  // +16 B: widened L2 prefetch
  CK(cuda_status(cudaMemcpyAsync(op->d_B, op->tab.B, sizeof(double) * Q * P1,
                                 cudaMemcpyHostToDevice, stream), "upload B"));
  CK(cuda_status(cudaMemcpyAsync(op->d_G, op->tab.G, sizeof(double) * Q * P1,
                                 cudaMemcpyHostToDevice, stream), "upload G"));
  int bad = 0;
  CK(build_qdata(op, stream, &bad));
  if (bad) {
    free_op(op);
    set_error("hofem_op_create: detJ <= 0 at some quadrature point (invalid mesh)");
    return HOFEM_ERR_MESH;
  }
#undef CK
  *op_out = op;
  return HOFEM_OK;
}

}  // namespace hofem

using namespace hofem;

extern "C" {

const char* hofem_last_error(void) { return g_err; }

hofem_status hofem_profile_enable(int enable) { return profile_enable(enable); }
hofem_status hofem_profile_read(hofem_profile_stats* out) {
  if (!out) { set_error("hofem_profile_read: NULL"); return HOFEM_ERR_ARG; }
  return profile_read(out);
}

namespace {
int* option_slot(Op* op, int opt) {
  switch (opt) {
    case HOFEM_OPT_INFIX: return &op->opt_infix;
    case HOFEM_OPT_CG_FUSED_UPDATE: return &op->opt_cg_fuse;
    case HOFEM_OPT_CG_PERSISTENT: return &op->opt_cg_persist;
    case HOFEM_OPT_L2_PREFETCH: return &op->opt_l2pf;
  }
  return nullptr;
}
}  // namespace

hofem_status hofem_op_set_option(void* op, hofem_option opt, int value) {
  int* slot = op ? option_slot(static_cast<Op*>(op), opt) : nullptr;
  const int vmax = opt == HOFEM_OPT_L2_PREFETCH ? 1 : 2;
  if (!slot || value < 0 || value > vmax) {
    set_error("hofem_op_set_option: need op != NULL, a known option and 0 <= value <= %d", vmax);
    return HOFEM_ERR_ARG;
  }
  *slot = value;
  return HOFEM_OK;
}

hofem_status hofem_op_get_option(const void* op, hofem_option opt, int* value) {
  int* slot = op ? option_slot(const_cast<Op*>(static_cast<const Op*>(op)), opt) : nullptr;
  if (!slot || !value) {
    set_error("hofem_op_get_option: need op != NULL, a known option and value != NULL");
    return HOFEM_ERR_ARG;
  }
  *value = *slot;
  return HOFEM_OK;
}

hofem_status hofem_op_fused_info(const void* op, hofem_fused_info* out) {
  if (!op || !out) { set_error("hofem_op_fused_info: NULL"); return HOFEM_ERR_ARG; }
  return fused_info(static_cast<const Op*>(op), out);
}

long long hofem_launch_count(void) { return g_launches.load(); }
void hofem_launch_count_reset(void) { g_launches.store(0); }

hofem_status hofem_mesh_create(const hofem_mesh_desc* d, void* comm, void* stream,
                               void** mesh_out) {
  if (!d || !mesh_out) { set_error("hofem_mesh_create: NULL argument"); return HOFEM_ERR_ARG; }
  Mesh* m = nullptr;
  HOFEM_TRY(mesh_new(d, static_cast<Comm*>(comm), S(stream), &m));
  *mesh_out = m;
  return HOFEM_OK;
}

hofem_status hofem_mesh_info_get(const void* mesh, hofem_mesh_info* info) {
  const Mesh* m = static_cast<const Mesh*>(mesh);
  if (!m || !info) { set_error("hofem_mesh_info_get: NULL"); return HOFEM_ERR_ARG; }
  info->n_local = m->n_local; info->n_owned = m->n_owned; info->n_global = m->n_global;
  info->elems_local = m->elems; info->plane = m->plane;
  info->rank = m->rank; info->nranks = m->nranks; info->z0 = m->z0; info->nz_local = m->nzl;
  return HOFEM_OK;
}

hofem_status hofem_mesh_coords(const void* mesh, double* xyz, void* stream) {
  const Mesh* m = static_cast<const Mesh*>(mesh);
  if (!m || !xyz) { set_error("hofem_mesh_coords: NULL"); return HOFEM_ERR_ARG; }
  HOFEM_CUDA(cudaMemcpyAsync(xyz, m->d_coords, sizeof(double) * 3 * m->n_local,
                             cudaMemcpyDeviceToDevice, S(stream)));
  return HOFEM_OK;
}

void hofem_mesh_destroy(void* mesh) { free_mesh(static_cast<Mesh*>(mesh)); }

hofem_status hofem_op_create(void* mesh, hofem_kind kind, hofem_rule rule, int q_override,
                             hofem_bc bc, void* stream, void** op_out) {
  Mesh* m = static_cast<Mesh*>(mesh);
  if (!m || !op_out) { set_error("hofem_op_create: NULL"); return HOFEM_ERR_ARG; }
  Op* op = nullptr;
  HOFEM_TRY(op_new(m, kind, rule, q_override, bc, S(stream), &op));
  *op_out = op;
  return HOFEM_OK;
}

hofem_status hofem_op_apply(void* op_, const double* x, double* y, void* stream) {
  Op* op = static_cast<Op*>(op_);
  if (!op || !x || !y || x == y) { set_error("hofem_op_apply: NULL or aliased x/y"); return HOFEM_ERR_ARG; }
  HOFEM_ALIGNED("hofem_op_apply", x, y);
  return apply_any(op, x, y, S(stream));
}

hofem_status hofem_op_apply_dot(void* op_, const double* x, double* y, double* dot_host,
                                void* stream) {
  Op* op = static_cast<Op*>(op_);
  if (!op || !x || !y || x == y || !dot_host) {
    set_error("hofem_op_apply_dot: NULL or aliased x/y");
    return HOFEM_ERR_ARG;
  }
  HOFEM_ALIGNED("hofem_op_apply_dot", x, y);
  Mesh* m = op->mesh;
  if (fused_supported(op)) {
    HOFEM_TRY(apply_fused(op, x, y, S(stream), m->d_scalars));
  } else {
    HOFEM_TRY(apply_unfused(op, x, y, S(stream)));
    HOFEM_TRY(dot_local(m, x, y, m->d_scalars, S(stream)));
  }
  HOFEM_TRY(allreduce_sum(m, m->d_scalars, 1, S(stream)));
  return d2h(m, dot_host, m->d_scalars, sizeof(double), S(stream));
}

hofem_status hofem_op_apply_unfused(void* op_, const double* x, double* y, void* stream) {
  Op* op = static_cast<Op*>(op_);
  if (!op || !x || !y || x == y) { set_error("hofem_op_apply_unfused: NULL or aliased x/y"); return HOFEM_ERR_ARG; }
  HOFEM_ALIGNED("hofem_op_apply_unfused", x, y);
  return apply_unfused(op, x, y, S(stream));
}

hofem_status hofem_op_apply_mf(void* op_, const double* x, double* y, void* stream) {
  Op* op = static_cast<Op*>(op_);
  if (!op || !x || !y || x == y) { set_error("hofem_op_apply_mf: NULL or aliased x/y"); return HOFEM_ERR_ARG; }
  HOFEM_ALIGNED("hofem_op_apply_mf", x, y);
  return apply_mf(op, x, y, S(stream));
}

hofem_status hofem_op_qdata(const void* op_, const double** qdata, long long* count) {
  const Op* op = static_cast<const Op*>(op_);
  if (!op || !qdata || !count) { set_error("hofem_op_qdata: NULL"); return HOFEM_ERR_ARG; }
  *qdata = op->d_qdata;
  *count = op->qcount;
  return HOFEM_OK;
}

hofem_status hofem_op_nq1d(const void* op_, int* q) {
  const Op* op = static_cast<const Op*>(op_);
  if (!op || !q) { set_error("hofem_op_nq1d: NULL"); return HOFEM_ERR_ARG; }
  *q = op->Q;
  return HOFEM_OK;
}

hofem_status hofem_rhs_manufactured(void* op_, double* b, void* stream) {
  Op* op = static_cast<Op*>(op_);
  if (!op || !b) { set_error("hofem_rhs_manufactured: NULL"); return HOFEM_ERR_ARG; }
  HOFEM_ALIGNED("hofem_rhs_manufactured", b);
  HOFEM_TRY(build_rhs(op, b, S(stream)));
  return exchange_planes(op, nullptr, b, S(stream));
}

hofem_status hofem_fill_random(const void* mesh, unsigned long long seed, double* x, void* stream) {
  const Mesh* m = static_cast<const Mesh*>(mesh);
  if (!m || !x) { set_error("hofem_fill_random: NULL"); return HOFEM_ERR_ARG; }
  HOFEM_ALIGNED("hofem_fill_random", x);
  return fill_random(m, seed, x, S(stream));
}

void hofem_op_destroy(void* op) { free_op(static_cast<Op*>(op)); }

hofem_status hofem_cg(void* op_, const double* b, double* x, double rel_tol, int max_iter,
                      int fixed_iters, int check_every, double* rr_history,
                      hofem_cg_stats* stats, void* stream) {
  Op* op = static_cast<Op*>(op_);
  if (!op || !b || !x || b == x) { set_error("hofem_cg: NULL or aliased b/x"); return HOFEM_ERR_ARG; }
  HOFEM_ALIGNED("hofem_cg", b, x);
  return cg_solve(op, b, x, rel_tol, max_iter, fixed_iters, check_every, rr_history, stats,
                  S(stream));
}

hofem_status hofem_dg_create(void* mesh, int q_override, void* stream, void** dg_out) {
  Mesh* m = static_cast<Mesh*>(mesh);
  if (!m || !dg_out || q_override < 0) { set_error("hofem_dg_create: bad argument"); return HOFEM_ERR_ARG; }
  DGOp* dg = nullptr;
  HOFEM_TRY(dg_create(m, q_override, S(stream), &dg));
  hofem_status st = cuda_status(cudaStreamSynchronize(S(stream)), "hofem_dg_create sync");
  if (st != HOFEM_OK) { dg_destroy(dg); return st; }
  *dg_out = dg;
  return HOFEM_OK;
}

hofem_status hofem_dg_info_get(const void* dg_, hofem_dg_info* info) {
  const DGOp* dg = static_cast<const DGOp*>(dg_);
  if (!dg || !info) { set_error("hofem_dg_info_get: NULL"); return HOFEM_ERR_ARG; }
  const Mesh* m = dg->mesh;
  info->n_local = dg->n_local;
  info->n_global = (long long)m->desc.nx * m->desc.ny * m->desc.nz_global * dg->nd;
  info->elems_local = m->elems;
  info->p = m->p; info->Q = dg->Q; info->dofs_per_elem = dg->nd; info->grid = dg->grid;
  return HOFEM_OK;
}

hofem_status hofem_dg_apply(void* dg_, const double* x, double* y, void* stream) {
  DGOp* dg = static_cast<DGOp*>(dg_);
  if (!dg || !x || !y || x == y) { set_error("hofem_dg_apply: NULL or aliased x/y"); return HOFEM_ERR_ARG; }
  HOFEM_ALIGNED("hofem_dg_apply", x, y);
  return dg_apply(dg, x, y, S(stream));
}

hofem_status hofem_dg_fill_random(const void* dg_, unsigned long long seed, double* x, void* stream) {
  const DGOp* dg = static_cast<const DGOp*>(dg_);
  if (!dg || !x) { set_error("hofem_dg_fill_random: NULL"); return HOFEM_ERR_ARG; }
  HOFEM_ALIGNED("hofem_dg_fill_random", x);
  return dg_fill_random(dg, seed, x, S(stream));
}

void hofem_dg_destroy(void* dg) { dg_destroy(static_cast<DGOp*>(dg)); }

hofem_status hofem_op_diagonal(void* op_, double* d, void* stream) {
  Op* op = static_cast<Op*>(op_);
  if (!op || !d) { set_error("hofem_op_diagonal: NULL"); return HOFEM_ERR_ARG; }
  HOFEM_ALIGNED("hofem_op_diagonal", d);
  return op_diagonal(op, d, S(stream));
}

hofem_status hofem_pmg_create(void* mesh, int degree, int power_iters, unsigned long long seed,
                              void* stream, void** pmg_out) {
  Mesh* m = static_cast<Mesh*>(mesh);
  if (!m || !pmg_out) { set_error("hofem_pmg_create: NULL"); return HOFEM_ERR_ARG; }
  PMG* P = nullptr;
  HOFEM_TRY(pmg_create(m, degree, power_iters, seed, S(stream), &P));
  *pmg_out = P;
  return HOFEM_OK;
}

hofem_status hofem_pmg_info_get(const void* pmg, hofem_pmg_info* info) {
  const PMG* P = static_cast<const PMG*>(pmg);
  if (!P || !info) { set_error("hofem_pmg_info_get: NULL"); return HOFEM_ERR_ARG; }
  memset(info, 0, sizeof(*info));
  info->levels = pmg_levels(P);
  for (int k = 0; k < info->levels && k < 8; ++k) {
    info->orders[k] = pmg_level_mesh(const_cast<PMG*>(P), k)->p;
    info->lambda[k] = pmg_level_lambda(P, k);
  }
  info->degree = pmg_degree(P);
  return HOFEM_OK;
}

hofem_status hofem_pmg_set_lambda(void* pmg, int level, double lambda) {
  PMG* P = static_cast<PMG*>(pmg);
  if (!P || level < 0 || level >= pmg_levels(P) || !(lambda > 0)) {
    set_error("hofem_pmg_set_lambda: bad level or lambda");
    return HOFEM_ERR_ARG;
  }
  pmg_set_lambda(P, level, lambda);
  return HOFEM_OK;
}

hofem_status hofem_pmg_level(void* pmg, int level, void** mesh_out, void** op_out) {
  PMG* P = static_cast<PMG*>(pmg);
  if (!P || level < 0 || level >= pmg_levels(P)) { set_error("hofem_pmg_level: bad level"); return HOFEM_ERR_ARG; }
  if (mesh_out) *mesh_out = pmg_level_mesh(P, level);
  if (op_out) *op_out = pmg_level_op(P, level);
  return HOFEM_OK;
}

hofem_status hofem_pmg_vcycle(void* pmg, const double* r, double* z, void* stream) {
  PMG* P = static_cast<PMG*>(pmg);
  if (!P || !r || !z || r == z) { set_error("hofem_pmg_vcycle: NULL or aliased"); return HOFEM_ERR_ARG; }
  HOFEM_ALIGNED("hofem_pmg_vcycle", r, z);
  return pmg_vcycle_level(P, 0, r, z, S(stream));
}

hofem_status hofem_pmg_smooth(void* pmg, int level, const double* b, double* x, void* stream) {
  PMG* P = static_cast<PMG*>(pmg);
  if (!P || !b || !x || b == x || level < 0 || level >= pmg_levels(P)) {
    set_error("hofem_pmg_smooth: bad arguments");
    return HOFEM_ERR_ARG;
  }
  HOFEM_ALIGNED("hofem_pmg_smooth", b, x);
  return pmg_smooth(P, level, b, x, false, S(stream));
}

hofem_status hofem_pmg_transfer(void* pmg, int level, int dir, const double* in, double* out,
                                void* stream) {
  PMG* P = static_cast<PMG*>(pmg);
  if (!P || !in || !out || in == out || level < 0 || level + 1 >= pmg_levels(P) ||
      (dir != 0 && dir != 1)) {
    set_error("hofem_pmg_transfer: bad arguments");
    return HOFEM_ERR_ARG;
  }
  HOFEM_ALIGNED("hofem_pmg_transfer", in, out);
  return dir == 0 ? pmg_prolong_add(P, level, in, out, S(stream))
                  : pmg_restrict(P, level, in, out, S(stream));
}

hofem_status hofem_pmg_pcg(void* pmg, const double* b, double* x, double rel_tol, int max_iter,
                           double* rr_history, hofem_cg_stats* stats, void* stream) {
  PMG* P = static_cast<PMG*>(pmg);
  if (!P || !b || !x || b == x || max_iter < 0) { set_error("hofem_pmg_pcg: bad arguments"); return HOFEM_ERR_ARG; }
  HOFEM_ALIGNED("hofem_pmg_pcg", b, x);
  return pmg_pcg(P, b, x, rel_tol, max_iter, rr_history, stats, S(stream));
}

void hofem_pmg_destroy(void* pmg) { pmg_destroy(static_cast<PMG*>(pmg)); }

hofem_status hofem_dot(const void* mesh, const double* a, const double* b, double* out_host,
                       void* stream) {
  Mesh* m = const_cast<Mesh*>(static_cast<const Mesh*>(mesh));
  if (!m || !a || !b || !out_host) { set_error("hofem_dot: NULL"); return HOFEM_ERR_ARG; }
  HOFEM_ALIGNED("hofem_dot", a, b);
  HOFEM_TRY(dot_device(m, a, b, m->d_scalars, S(stream)));
  return d2h(m, out_host, m->d_scalars, sizeof(double), S(stream));
}

}  // extern "C"
