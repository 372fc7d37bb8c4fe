// internal.h -- shared internals of libhofem (the product CUDA path).
// Nothing here is shared with oracle/ (see DESIGN.md §2 "independence").
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <string>

#include "../../include/hofem.h"

namespace hofem {

constexpr int kMaxP = 8;    // p <= 8 (P1 <= 9)
constexpr int kMaxQ = 16;   // 1D quadrature points
constexpr int kNumSMs = 148;

void set_error(const char* fmt, ...);
hofem_status cuda_status(cudaError_t e, const char* what);
void count_launch(long long n = 1);
int num_sms();  // SM count of the current device (fused.cu)

#define HOFEM_CUDA(call)                                                   \
  do {                                                                     \
    cudaError_t e_ = (call);                                               \
    if (e_ != cudaSuccess) return ::hofem::cuda_status(e_, #call);          \
  } while (0)
#define HOFEM_LAUNCHED()                                                   \
  do {                                                                     \
    ::hofem::count_launch();                                               \
    cudaError_t e_ = cudaPeekAtLastError();                                \
    if (e_ != cudaSuccess) return ::hofem::cuda_status(e_, "kernel launch"); \
  } while (0)
#define HOFEM_TRY(call)                                                    \
  do {                                                                     \
    hofem_status s_ = (call);                                              \
    if (s_ != HOFEM_OK) return s_;                                         \
  } while (0)

// In-process loopback transport (comm.cu): ranks are host threads of one
// process on one device; plane exchange by device copies ordered with CUDA
// events behind host barriers, allreduce by a fixed rank-order sum.  Exercises
// the whole multi-rank data path (partition, exchange, Dirichlet re-imposition,
// owned-dof dot products) on a single GPU.
struct LoopGroup;

struct Comm {
  int rank = 0, nranks = 1, device = 0;
  ncclComm_t nccl = nullptr;
  LoopGroup* loop = nullptr;  // non-null: loopback transport instead of NCCL
};

// 1D tables (independent host implementation, long double Newton).
struct Tables1D {
  int p = 0, Q = 0, rule = 0;
  double xi[kMaxP + 1];            // GLL nodes on [0,1]
  double t[kMaxQ], w[kMaxQ];       // quadrature points / weights on [0,1]
  double B[kMaxQ * (kMaxP + 1)];   // B[k*P1+i] = l_i(t_k)
  double G[kMaxQ * (kMaxP + 1)];   // G[k*P1+i] = l_i'(t_k)
};
int build_tables(int p, int Q, int rule, Tables1D* out);  // 0 ok
void gll_nodes_weights(int p, double* x, double* w);
int build_dg_table(int p, int Q, double* B);  // DG basis (Gauss-Legendre nodes) at Gauss points

struct Mesh {
  hofem_mesh_desc desc{};
  Comm* comm = nullptr;
  int rank = 0, nranks = 1;
  int p = 1, P1 = 2;
  int nx = 1, ny = 1, nzl = 1, z0 = 0;     // local element counts, first layer
  long long Nx = 0, Ny = 0, Nzl = 0;       // local lattice sizes
  long long NzG = 0;                        // global lattice planes
  long long n_local = 0, n_owned = 0, n_global = 0, elems = 0, plane = 0;
  double* d_xi = nullptr;                   // GLL nodes (device)
  double* d_coords = nullptr;               // 3*n_local
  // lazily built for the unfused path
  int* d_l2e = nullptr;                     // [E][P1^3]
  long long* d_toff = nullptr;              // [n_local+1]
  int* d_tidx = nullptr;                    // [E*P1^3] entries e*P1^3+i
  // reductions
  double* d_partials = nullptr;             // [kDotBlocks]
  unsigned int* d_counter = nullptr;        // last-block counters
  double* d_scalars = nullptr;              // scratch scalars
  double* d_recv = nullptr;                 // 2 planes for the interface exchange
  double* d_send = nullptr;                 // 2 planes staging (copies of own planes)
  // kernel-initiated exchange (hofem_mesh_set_exchange, comm.cu): the
  // neighbours write their planes straight into d_xrecv (2 parities x [lo|hi])
  // and raise d_xflag[lo|hi]; d_xflag[2] counts the exchanges this rank has
  // consumed (read by the neighbours before reusing a parity slot)
  int xmode = 0;                            // 0 collective (NCCL / loopback copies), 1 peer puts
  double* d_xrecv = nullptr;                // 4 planes
  unsigned long long* d_xflag = nullptr;    // [lo filled, hi filled, consumed, -, chain up, chain down, put-kernel barrier x2]
  double* peer_recv[2] = {nullptr, nullptr};               // lower / upper neighbour's d_xrecv
  unsigned long long* peer_flag[2] = {nullptr, nullptr};   // lower / upper neighbour's d_xflag
  bool peer_ipc[2] = {false, false};        // opened with cudaIpcOpenMemHandle
  unsigned long long xseq = 0;              // exchanges issued
  unsigned long long rseq = 0;              // in-kernel chain allreduces (persistent CG)
  // pinned host staging for the library's device->host reads (dot results, CG
  // scalars): a copy into pageable memory may wait on the whole device, which
  // deadlocks against a loopback neighbour's spinning kernel
  double* h_pin = nullptr;                  // kPinDoubles doubles (cudaHostAlloc)
};

// Grid-wide barrier state of a cooperative launch: arrival count and
// generation word (zeroed once at allocation; self-resetting, no host state).
struct GridBar {
  unsigned int count;
  unsigned int gen;
};

struct Op {
  Mesh* mesh = nullptr;
  int kind = HOFEM_DIFFUSION, rule = HOFEM_GAUSS, Q = 0, nc = 6, bc = 0;
  Tables1D tab{};
  double* d_B = nullptr;    // Q*P1
  double* d_G = nullptr;    // Q*P1
  double* d_qdata = nullptr;
  long long qcount = 0;
  // unfused scratch (lazy)
  double* d_ein = nullptr;
  double* d_eout = nullptr;
  // fused brick scratch (boundary partials)
  double* d_bbuf = nullptr;
  long long bbuf_len = 0;
  double* d_dotp = nullptr; // per-CTA partials of the fused x.y (CG)
  long long dotp_len = 0;
  GridBar* d_bar = nullptr; // self-resetting grid barrier (cooperative launches)
  double* d_cgparts = nullptr;  // persistent CG: 2 x grid partials
  long long cgparts_len = 0;
  // per-operator schedule options (hofem_op_set_option); 0 never, 1 auto (size
  // threshold, the measured default), 2 always
  int opt_infix = 1;        // HOFEM_OPT_INFIX: edge-line fix-up inside the brick kernel
  int opt_cg_fuse = 1;      // HOFEM_OPT_CG_FUSED_UPDATE: one cooperative update kernel
  int opt_cg_persist = 1;   // HOFEM_OPT_CG_PERSISTENT: whole CG solve in one kernel
  int opt_l2pf = 1;         // HOFEM_OPT_L2_PREFETCH: bulk-prefetch next brick's qdata
  // CG scratch
  double *d_r = nullptr, *d_p = nullptr, *d_Ap = nullptr;
  double* d_cg = nullptr;   // device CG scalars / history
  int cg_cap = 0;
};

// fully matrix-free BP3 apply (mf.cu, mf_impl.cuh; §8(f) f3)
hofem_status apply_mf(Op* op, const double* x, double* y, cudaStream_t s);

// p-multigrid (pmg.cu; §8(f) f2)
struct PMG;
hofem_status op_diagonal(Op* op, double* d, cudaStream_t s);
hofem_status pmg_create(Mesh* fine, int degree, int power_iters, unsigned long long seed,
                        cudaStream_t s, PMG** out);
void pmg_destroy(PMG* P);
hofem_status pmg_vcycle_level(PMG* P, int k, const double* b, double* z, cudaStream_t s);
hofem_status pmg_smooth(PMG* P, int k, const double* b, double* x, bool x_zero, cudaStream_t s);
hofem_status pmg_prolong_add(PMG* P, int k, const double* xc, double* xf, cudaStream_t s);
hofem_status pmg_restrict(PMG* P, int k, const double* rf, double* rc, cudaStream_t s);
hofem_status pmg_pcg(PMG* P, const double* b, double* x, double rel_tol, int max_iter,
                     double* rr_history, hofem_cg_stats* stats, cudaStream_t s);
int pmg_levels(const PMG* P);
Mesh* pmg_level_mesh(PMG* P, int k);
Op* pmg_level_op(PMG* P, int k);
double pmg_level_lambda(const PMG* P, int k);
void pmg_set_lambda(PMG* P, int k, double lam);
int pmg_degree(const PMG* P);

// Operator construction / destruction (capi.cu): qdata, tables; SYNC.
hofem_status op_new(Mesh* m, int kind, int rule, int q_override, int bc, cudaStream_t s,
                    Op** out);
void op_free(Op* op);
hofem_status mesh_new(const hofem_mesh_desc* d, Comm* comm, cudaStream_t s, Mesh** out);
void mesh_free(Mesh* m);
// E-vector -> L-vector deterministic scatter through the transposed offsets
// (unfused.cu).  bcmode: 0 none, 1 y[ess] = xbc[ess], 2 y[ess] = 0, 3 y[ess] = 1.
hofem_status scatter_evector_bc(Op* op, const double* ein, double* y, int bcmode,
                                const double* xbc, cudaStream_t s);

// DG (L2) mass operator (dg.cu, dg_impl.cuh; §8(f) f4)
struct DGOp {
  Mesh* mesh = nullptr;
  Op* geo = nullptr;            // W*detJ qdata at the Gauss points (BP1 layout)
  int Q = 0, nd = 0, grid = 0;
  long long n_local = 0;        // E * P1^3
  double B[kMaxQ * (kMaxP + 1)];  // B[k*P1+i] = psi_i(t_k), psi on Gauss-Legendre nodes
};
hofem_status dg_create(Mesh* m, int q_override, cudaStream_t s, DGOp** out);
hofem_status dg_apply(DGOp* dg, const double* x, double* y, cudaStream_t s);
hofem_status dg_fill_random(const DGOp* dg, unsigned long long seed, double* x, cudaStream_t s);
void dg_destroy(DGOp* dg);

// ---- mesh / setup kernels (mesh.cu)
hofem_status mesh_build_coords(Mesh* m, cudaStream_t s);
hofem_status mesh_build_restriction(Mesh* m, cudaStream_t s);
hofem_status fill_random(const Mesh* m, unsigned long long seed, double* x, cudaStream_t s);
// x[l] = R12 random value of global index g0 + l, l < n
hofem_status fill_random_range(unsigned long long seed, long long g0, long long n, double* x,
                               cudaStream_t s);

// ---- qdata / rhs (qdata.cu)
hofem_status build_qdata(Op* op, cudaStream_t s, int* bad_host);
hofem_status build_rhs(Op* op, double* b, cudaStream_t s);

// Device -> host read of `bytes` through the mesh's pinned staging buffer
// (chunked), ordered on stream s: synchronizes s only.
constexpr int kPinDoubles = 512;
hofem_status d2h(Mesh* m, void* dst, const void* src, size_t bytes, cudaStream_t s);

// ---- operator apply paths
hofem_status apply_unfused(Op* op, const double* x, double* y, cudaStream_t s);
// dot_out (device scalar, optional): the rank-local owned x.y, computed inside
// the fused kernels from the contributions they write (deterministic); the
// caller allreduces it.
// With dot_parts non-null (and dot_out non-null) the final fixed-order sum of
// the per-CTA x.y partials is left to the caller: *dot_parts / *dot_nparts
// name the partial array (single rank only; used by the fused CG update).
hofem_status apply_fused(Op* op, const double* x, double* y, cudaStream_t s,
                         double* dot_out = nullptr, const double** dot_parts = nullptr,
                         long long* dot_nparts = nullptr);
// Rank-local a.b over owned dofs into *d_out (device), deterministic; no allreduce.
hofem_status dot_local(Mesh* m, const double* a, const double* b, double* d_out, cudaStream_t s);
hofem_status fused_info(const Op* op, hofem_fused_info* out);
// The whole CG solve (r, p, rr[0] initialised by the caller) in one cooperative
// kernel (fused.cu / fused_impl.cuh cg_persistent_simt); d_result[0] =
// iterations, d_result[1] = breakdown flag.  Returns HOFEM_ERR_CUDA with
// cudaErrorCooperativeLaunchTooLarge if the grid cannot be co-resident.
hofem_status cg_persistent(Op* op, double* x, double* r, double* p, double* Ap, double* rr,
                           int max_iter, int fixed, double rel_tol, int* d_result,
                           cudaStream_t s);
bool fused_supported(const Op* op);

// ---- comm (comm.cu): sum duplicated interface planes, fix BC there
hofem_status exchange_planes(Op* op, const double* x, double* y, cudaStream_t s);
hofem_status exchange_planes_bc(Op* op, const double* x, double* y, int bcmode, cudaStream_t s);
// switch a multi-rank mesh to the kernel-initiated exchange (collective: every
// rank of the mesh calls it); comm.cu
hofem_status mesh_set_exchange(Mesh* m, int mode, cudaStream_t s);
void mesh_release_exchange(Mesh* m);
hofem_status allreduce_sum(Mesh* m, double* d_val, int count, cudaStream_t s);

// ---- vector kernels (cg.cu)
hofem_status dot_device(Mesh* m, const double* a, const double* b, double* d_out, cudaStream_t s);

// ---- host helpers
inline bool is_ess(const Mesh* m, long long I, long long J, long long Kglob) {
  return I == 0 || I == m->Nx - 1 || J == 0 || J == m->Ny - 1 || Kglob == 0 ||
         Kglob == m->NzG - 1;
}

#ifdef __CUDACC__
// Grid-wide barrier of a cooperative (co-resident) launch.  Self-resetting: each
// CTA reads the generation word, then arrives on the counter; the last CTA to
// arrive zeroes the counter and publishes generation + 1, which releases the
// others.  No host-side state, so a launch may be captured into a CUDA graph and
// replayed.  The wait is bounded by %globaltimer (20 s): a barrier that cannot
// complete traps instead of hanging the GPU.
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void grid_barrier(GridBar* bar) {
  // thread 0 carries the CTA: bar.sync orders the CTA's memory operations, the
  // acq_rel arrival releases them to / acquires the other CTAs' at gpu scope,
  // and the generation flip is a release store read with acquire loads -- no
  // separate fences (measured: 3.07 -> 2.14 us per barrier at 444 CTAs,
  // scratch microbenchmark, DESIGN.md §4 CG)
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int g;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(&bar->gen) : "memory");
    unsigned int arrived;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(arrived)
                 : "l"(&bar->count)
                 : "memory");
    if (arrived == gridDim.x - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(&bar->count) : "memory");
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&bar->gen), "r"(g + 1u) : "memory");
    } else {
      const unsigned long long t0 = global_ns();
      unsigned int v;
      unsigned spins = 0;
      while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&bar->gen) : "memory");
        if (v != g) break;
        if ((++spins & 1023u) == 0u && global_ns() - t0 > 20000000000ull) __trap();
        __nanosleep(32);
      }
    }
  }
  __syncthreads();
}

#endif

}  // namespace hofem
