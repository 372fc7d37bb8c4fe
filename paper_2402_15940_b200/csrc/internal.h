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

struct Comm {
  int rank = 0, nranks = 1, device = 0;
  ncclComm_t nccl = nullptr;
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
  int fused_variant = -1;   // -1: HOFEM_FUSED env / per-p default; 0 DMMA; 1 SIMT
  double* d_dotp = nullptr; // per-CTA partials of the fused x.y (CG)
  long long dotp_len = 0;
  unsigned long long* d_bar = nullptr;  // grid-barrier counter of the in-kernel fix-up
  unsigned long long bar_count = 0;     // CTAs launched against it so far
  // CG scratch
  double *d_r = nullptr, *d_p = nullptr, *d_Ap = nullptr;
  double* d_cg = nullptr;   // device CG scalars / history
  int cg_cap = 0;
};

// ---- mesh / setup kernels (mesh.cu)
hofem_status mesh_build_coords(Mesh* m, cudaStream_t s);
hofem_status mesh_build_restriction(Mesh* m, cudaStream_t s);
hofem_status fill_random(const Mesh* m, unsigned long long seed, double* x, cudaStream_t s);

// ---- qdata / rhs (qdata.cu)
hofem_status build_qdata(Op* op, cudaStream_t s, int* bad_host);
hofem_status build_rhs(Op* op, double* b, cudaStream_t s);

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
bool fused_supported(const Op* op);

// ---- comm (comm.cu): sum duplicated interface planes, fix BC there
hofem_status exchange_planes(Op* op, const double* x, double* y, cudaStream_t s);
hofem_status allreduce_sum(Mesh* m, double* d_val, int count, cudaStream_t s);

// ---- vector kernels (cg.cu)
hofem_status dot_device(Mesh* m, const double* a, const double* b, double* d_out, cudaStream_t s);

// ---- host helpers
inline bool is_ess(const Mesh* m, long long I, long long J, long long Kglob) {
  return I == 0 || I == m->Nx - 1 || J == 0 || J == m->Ny - 1 || Kglob == 0 ||
         Kglob == m->NzG - 1;
}

#ifdef __CUDACC__
// Grid-wide barrier of a cooperative (co-resident) launch on a monotonic
// 64-bit counter: every CTA adds 1 and waits for `target` (the host keeps the
// running total of launched CTAs, so the counter is never reset).  Bounded
// spin: a barrier that cannot complete traps (launch error) instead of
// hanging the GPU.
__device__ __forceinline__ void grid_barrier(unsigned long long* bar, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1ull);
    unsigned long long v;
    unsigned spins = 0;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
      if (v >= target) break;
      __nanosleep(100);
    } while (++spins < (1u << 25));
    if (v < target) __trap();
    __threadfence();
  }
  __syncthreads();
}

#endif

}  // namespace hofem
