/*
 * hofem.h -- C ABI of the B200-native matrix-free high-order FEM hot path of
 * arXiv 2402.15940 ("High-performance finite elements with MFEM"):
 * partial-assembly (PA) sum-factorization operator actions on structured
 * curvilinear high-order hexahedral meshes -- the CEED bake-off mass (BP1) and
 * diffusion (BP3, BP5) actions y = R^T B^T D B R x -- and the CG solve built on
 * them, slab-partitioned over up to 8 GPUs with NCCL.
 *
 * Citations are PAPER.md line numbers (section in parentheses) and the
 * DESIGN.md readings R1-R14 (= SURVEY.md §8(c)) for everything the paper leaves
 * open.  Operator decomposition: A = P^T G^T B^T D B G P (PAPER.md:595,
 * fig_feod, §3.5); this library calls the paper's element restriction "G" R, and
 * its P is the z-slab interface exchange.
 *
 * Conventions (all entry points):
 *  - Every vector argument is a DEVICE pointer to contiguous FP64 owned by the
 *    caller (e.g. a torch.float64 CUDA tensor's data_ptr()).  Vectors are
 *    rank-local L-vectors of length n_local, lexicographic with x fastest:
 *    l = I + Nx*(J + Ny*K) (reading R3).  The two z-interface planes are
 *    duplicated on both neighbouring ranks and kept bitwise identical (R9).
 *  - Vector pointers must be 16-byte aligned (the vector kernels use 16-byte
 *    accesses); a misaligned pointer returns HOFEM_ERR_ARG.  Lengths are not
 *    passed: every vector holds n_local doubles of its mesh (hofem_mesh_info);
 *    the caller guarantees that (the Python binding checks it).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Everything is stream-ordered and asynchronous, except the calls marked
 *    SYNC, which synchronize `stream` before returning.  Stream-ordered calls
 *    (hofem_op_apply included) may be captured into a CUDA graph and replayed:
 *    the in-kernel grid barriers reset themselves and keep no host state.
 *  - Single-stream handles: an operator (and the mesh it was built on) owns
 *    scratch buffers (brick partials, reduction partials, the grid barrier) that
 *    every call reuses, so calls on one operator or mesh must be ordered on ONE
 *    stream (or otherwise serialised by the caller).  Concurrent calls on the
 *    same handle from two streams race.  Distinct operators on distinct meshes
 *    are independent.
 *  - Opaque handles are owned by the library; each destroy frees exactly what
 *    the matching create allocated.  The library never frees caller buffers.
 *  - x and y must not alias; y is fully overwritten.
 *  - On error the outputs are unspecified; handles stay valid except after
 *    HOFEM_ERR_CUDA / HOFEM_ERR_NCCL.  hofem_last_error() gives a message.
 *  - There is no CPU fallback: every step of every call runs in this library's
 *    CUDA kernels (sm_100a).  Without a usable CUDA device, calls that touch the
 *    device return HOFEM_ERR_CUDA.
 */
#ifndef HOFEM_H
#define HOFEM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HOFEM_OK = 0,
  HOFEM_ERR_ARG = 1,       /* precondition violated: p<1 or p>8, n<1, NULL, x==y, bad rule/kind */
  HOFEM_ERR_MESH = 2,      /* detJ <= 0 at some quadrature point */
  HOFEM_ERR_CUDA = 3,      /* CUDA runtime error (message in hofem_last_error) */
  HOFEM_ERR_NCCL = 4,      /* NCCL error */
  HOFEM_ERR_OOM = 5,       /* device allocation failed */
  HOFEM_ERR_BREAKDOWN = 6, /* CG: p^T A p <= 0 */
  HOFEM_NOT_CONVERGED = 7  /* CG: max_iter reached, outputs valid */
} hofem_status;

/* Thread-local message describing the last non-OK status (never NULL). */
const char* hofem_last_error(void);

/* ---------------------------------------------------------------- comm (P) */
/* NCCL communicator for the z-slab partition (§2.3: the
 * parallel operator P^T A P).  hofem_comm_unique_id writes the
 * 128-byte ncclUniqueId on rank 0; the caller broadcasts it (torch.distributed)
 * and every rank calls hofem_comm_init with its rank and CUDA device. */
hofem_status hofem_comm_unique_id(void* nccl_id_out /* 128 bytes, host */);
hofem_status hofem_comm_init(const void* nccl_id /* 128 B host */, int rank, int nranks,
                             int device, void** comm_out);
void hofem_comm_destroy(void* comm);
/* In-process loopback transport (testing the multi-rank data path on ONE GPU):
 * a group of nranks "ranks" that are host threads of this process sharing the
 * current device.  Every rank's thread calls hofem_comm_init_loopback with its
 * rank and then drives its own mesh / operator on its own stream exactly as
 * with NCCL; the interface exchange becomes device-to-device plane copies
 * ordered by CUDA events behind host barriers, the allreduce a fixed rank-order
 * sum (bitwise identical on every rank).  All ranks must make the same sequence
 * of collective calls (apply, dot, CG, ...), like NCCL.  Cooperative in-kernel
 * grid barriers are not used on a loopback multi-rank mesh (several ranks'
 * kernels share the device).  The group must outlive its comms. */
hofem_status hofem_loopback_group_create(int nranks, void** group_out);
hofem_status hofem_comm_init_loopback(void* group, int rank, void** comm_out);
void hofem_loopback_group_destroy(void* group);

/* ---------------------------------------------------------------- mesh (a1) */
/* Structured nx*ny*nz_global hex mesh of [0,extent0]x[0,extent1]x[0,extent2],
 * isoparametric degree p (geometry order = p), nodes at GLL
 * points mapped by the smooth deformation Phi of reading R4 with amplitude
 * alpha (0 = affine box).  With comm != NULL, rank r gets the element layers
 * ez in [r*nz/R, (r+1)*nz/R) (R must divide nz_global) and its L-vector covers
 * lattice planes K in [p*z0, p*z1] (reading R9). 1 <= p <= 8. */
typedef struct {
  int nx, ny, nz_global, p;
  double extent[3];
  double alpha;
} hofem_mesh_desc;

typedef struct {
  long long n_local;    /* L-vector length on this rank = Nx*Ny*Nz_local */
  long long n_owned;    /* dofs this rank owns (dot products / counting, R8-R9) */
  long long n_global;   /* global dof count (p*nx+1)(p*ny+1)(p*nz+1) */
  long long elems_local;
  long long plane;      /* Nx*Ny, the size of one z lattice plane */
  int rank, nranks, z0, nz_local;
} hofem_mesh_info;

hofem_status hofem_mesh_create(const hofem_mesh_desc* desc, void* comm /* NULL => 1 rank */,
                               void* stream, void** mesh_out);
hofem_status hofem_mesh_info_get(const void* mesh, hofem_mesh_info* info_out);
/* Nodal coordinates: xyz[c*n_local + l], c = 0,1,2 (device, 3*n_local FP64). */
hofem_status hofem_mesh_coords(const void* mesh, double* xyz, void* stream);
void hofem_mesh_destroy(void* mesh);
/* Interface-exchange transport of a multi-rank mesh (no-op on one rank).
 * mode 0: the communicator's collective (NCCL grouped send/recv, or the
 * loopback copies).  mode 1: kernel-initiated puts (§2.3
 * "GPU-initiated communication"; §8(f) f1): one small cooperative kernel per
 * exchange writes this rank's boundary planes straight into the z neighbours'
 * receive slots through peer pointers (CUDA IPC handles swapped over NCCL and
 * opened with cudaIpcOpenMemHandle -- NVLink stores between GPUs; plain
 * pointers in the loopback transport), raises their "filled" flags with a
 * system-scope release, waits for its own, adds the received planes
 * (Dirichlet rows re-imposed) and publishes "consumed" (double-buffered slots:
 * a rank runs at most one exchange ahead of its neighbours).  Collective: every
 * rank of the mesh calls it with the same mode.  Not graph-capturable (the
 * exchange counter lives on the host).  With the loopback transport (all ranks
 * on ONE device) a rank's thread must not synchronize the whole device
 * (cudaDeviceSynchronize, cudaFree, torch.cuda.synchronize) between exchanges:
 * it would wait on a neighbour's put kernel that waits on this rank -- use
 * stream synchronization.  Calls on existing handles allocate stream-ordered
 * (cudaMallocAsync); creating a handle (mesh, operator, DG, p-MG) and
 * allocating caller buffers (cudaMalloc, a torch caching-allocator miss) may
 * synchronize the device, so on a loopback mesh create every object and
 * buffer before switching mode 1 on -- and load the kernel modules eagerly
 * (CUDA_MODULE_LOADING=EAGER): a kernel's first, lazy load may synchronize the
 * context as well; so may a device-to-host copy into PAGEABLE memory, so read
 * results back after the ranks' last exchange (the library's own reads --
 * dots, CG scalars -- go through pinned staging).  With mode 1, hofem_cg's persistent schedule
 * (HOFEM_OPT_CG_PERSISTENT) also runs on several ranks: the planes and both
 * dot products are then exchanged inside the one kernel per rank. */
hofem_status hofem_mesh_set_exchange(void* mesh, int mode, void* stream);

/* ---------------------------------------------------------- operator (a2-a9) */
typedef enum { HOFEM_MASS = 1, HOFEM_DIFFUSION = 2 } hofem_kind;
/* Quadrature (reading R2): GAUSS Q = p+2 (BP1, BP3); GLL Q = p+1 collocated with
 * the nodes, so B1d = I (BP5).  q_override != 0 selects another Q in [1, 16]
 * (Q = p+1 with GAUSS, Q = p+2 with GLL also use the fused kernels). */
typedef enum { HOFEM_GAUSS = 1, HOFEM_GLL = 2 } hofem_rule;
typedef enum { HOFEM_BC_NONE = 0, HOFEM_BC_DIRICHLET = 1 } hofem_bc;

/* SYNC.  Build the partially assembled operator: only the quadrature-point data
 * D is stored (§2.2 "Partial Assembly"): mass W*detJ, diffusion
 * the symmetric W adj(J) adj(J)^T / detJ (6 entries [00,01,02,11,12,22]),
 * layout [E][n_c][Q^3] (R3).  Returns HOFEM_ERR_MESH if detJ <= 0 anywhere.
 * bc = DIRICHLET applies the homogeneous whole-boundary convention of R6:
 * z = x; z[ess] = 0; y = A z; y[ess] = x[ess]. */
hofem_status hofem_op_create(void* mesh, hofem_kind kind, hofem_rule rule, int q_override,
                             hofem_bc bc, void* stream, void** op_out);

/* y = P^T R^T B^T D B R P x: the fused path.  One sm_100a kernel
 * per element brick does gather (R), the 1D B/G contractions dimension by
 * dimension, the pointwise D, the transposed contractions and the in-brick
 * deterministic sum; a fix-up kernel sums brick-interface dofs in fixed order;
 * with >1 rank the interface planes are then exchanged over NCCL (P).
 * Bitwise deterministic run to run. */
hofem_status hofem_op_apply(void* op, const double* x, double* y, void* stream);

/* Same operator, unfused reference path: gather kernel (R through the l2e
 * table) -> element kernel -> deterministic scatter through precomputed
 * transposed offsets (R^T, ascending (e, i) order). */
hofem_status hofem_op_apply_unfused(void* op, const double* x, double* y, void* stream);
/* y = A x, "Fully Matrix-Free" assembly level (§2.2; §8(f) f3):
 * the same operator as hofem_op_apply, but the quadrature data is NOT read --
 * every call recomputes J = dX/dxi at the quadrature points from the nodal
 * coordinates by sum factorization, then adj(J), detJ and
 * D = W adj(J)adj(J)^T / detJ pointwise, in the kernel.  One persistent kernel
 * per apply writes element results to an E-vector, then the deterministic
 * transposed-offset scatter (ascending (e, i)) assembles y; Dirichlet rows
 * y = x.  BP3 only (DIFFUSION, Gauss Q = p+2), else HOFEM_ERR_ARG. */
hofem_status hofem_op_apply_mf(void* op, const double* x, double* y, void* stream);

/* SYNC.  y = A x (as hofem_op_apply) and *dot_host = x.y over owned dofs,
 * allreduced -- the x^T A x energy that CG needs as p^T A p.  On the fused
 * path the product is accumulated inside the operator kernels from the values
 * they write (each element contribution times x at its dof, Dirichlet rows
 * once), in a fixed order: deterministic, and equal to hofem_dot(x, y) up to
 * rounding (the order of the sum differs). */
hofem_status hofem_op_apply_dot(void* op, const double* x, double* y, double* dot_host,
                                void* stream);

/* Device pointer to the stored qdata (owned by op) and its length E*n_c*Q^3. */
hofem_status hofem_op_qdata(const void* op, const double** qdata, long long* count);
/* Q (1D quadrature points) actually used by op. */
hofem_status hofem_op_nq1d(const void* op, int* q_out);

/* b_i = sum_e sum_q W_q detJ f(x(xi_q)) phi_i(xi_q) (reading R11): diffusion
 * f = 3 pi^2 prod sin(pi x_j), mass f = prod sin(pi x_j); b[ess] = 0 when op has
 * Dirichlet BCs.  Interface planes are summed across ranks. */
hofem_status hofem_rhs_manufactured(void* op, double* b, void* stream);

/* Counter-based random L-vector of reading R12, indexed by the GLOBAL dof:
 * x_g = 2*((splitmix64(seed + (g+1)*0x9E3779B97F4A7C15) >> 11) * 2^-53) - 1. */
hofem_status hofem_fill_random(const void* mesh, unsigned long long seed, double* x, void* stream);

void hofem_op_destroy(void* op);

/* ------------------------------------------------- DG (L2) mass (§8(f) f4) */
/* Matrix-free discontinuous Galerkin mass operator on the same hex mesh
 * (§2.4.1 "matrix-free discontinuous Galerkin"; fig:dgpa-perf
 * "DG mass operators").  Space: discontinuous Q_p per element with the nodal
 * basis at the p+1 Gauss-Legendre points (reading R16).  Vectors are
 * element-major E-vectors of n_local = elems_local * (p+1)^3 doubles: entry
 * e*(p+1)^3 + a + (p+1)(b + (p+1)c), elements lexicographic (x fastest), local
 * element e of rank r is global element e + z0*nx*ny.  The operator is block
 * diagonal, y_e = B^T D_e B x_e, D_e = W detJ at the Gauss points (the BP1
 * qdata): no inter-element coupling, hence no scatter and no communication.
 * Geometry: the mesh's isoparametric map.  Only the Gauss rule Q = p+2 is
 * instantiated (q_override 0 or p+2, else HOFEM_ERR_ARG). */
typedef struct {
  long long n_local;    /* E-vector length on this rank */
  long long n_global;   /* all ranks */
  long long elems_local;
  int p, Q, dofs_per_elem;
  int grid;             /* CTAs of the last apply (0 before the first) */
} hofem_dg_info;
/* SYNC.  Builds the DG operator (qdata, tables); HOFEM_ERR_MESH if detJ <= 0. */
hofem_status hofem_dg_create(void* mesh, int q_override, void* stream, void** dg_out);
hofem_status hofem_dg_info_get(const void* dg, hofem_dg_info* info_out);
/* y = M_DG x (one persistent kernel: asynchronous copies of x, one bulk (TMA)
 * copy of D per element batch, sum factorization, coalesced stores of y). */
hofem_status hofem_dg_apply(void* dg, const double* x, double* y, void* stream);
/* R12 random E-vector indexed by the GLOBAL DG dof (global element * (p+1)^3 + node). */
hofem_status hofem_dg_fill_random(const void* dg, unsigned long long seed, double* x, void* stream);
void hofem_dg_destroy(void* dg);

/* -------------------------------------------------------------------- CG (a10) */
typedef struct {
  int iterations;        /* iterations performed */
  int converged;         /* 1 if ||r_k|| <= rel_tol ||r_0|| (or fixed count done) */
  double r0_norm;        /* ||r_0||_2 over owned dofs, all ranks */
  double final_rel_res;  /* ||r_k|| / ||r_0|| */
} hofem_cg_stats;

/* SYNC.  Unpreconditioned CG (§2.1; reading R7):
 * r0 = b - A x0, p = r0; per iteration Ap = A p (fused apply), pAp = p.Ap
 * (owned dofs, NCCL allreduce), alpha = rr/pAp, x += alpha p, r -= alpha Ap,
 * rr' = r.r (fused with the update), beta = rr'/rr, p = r + beta p.  alpha and
 * beta stay on the device.  Stops when ||r|| <= rel_tol ||r0|| (tested every
 * check_every iterations: the only device->host copy), or runs exactly max_iter
 * iterations when fixed_iters = 1.  x: in x0, out the iterate.
 * rr_history (host, nullable, length max_iter+1) receives r_k.r_k.
 * Small single-rank problems run the whole solve in one persistent kernel
 * (HOFEM_OPT_CG_PERSISTENT), which tests convergence every iteration.
 * Returns HOFEM_NOT_CONVERGED if max_iter was hit in tolerance mode,
 * HOFEM_ERR_BREAKDOWN if pAp <= 0. */
hofem_status hofem_cg(void* op, const double* b, double* x, double rel_tol, int max_iter,
                      int fixed_iters, int check_every, double* rr_history,
                      hofem_cg_stats* stats, void* stream);

/* SYNC.  out = sum over owned dofs of a_l*b_l, allreduced over ranks; the
 * reduction order is fixed (deterministic). */
hofem_status hofem_dot(const void* mesh, const double* a, const double* b, double* out_host,
                       void* stream);

/* ---------------------------------- p-multigrid preconditioned CG (§8(f) f2) */
/* Matrix-free preconditioning of the BP3 problem, CEED BPS3 (PAPER.md:103-111,
 * §2.1 "p-multigrid ... Chebyshev acceleration").  Readings R17-R18
 * (DESIGN.md §3): levels of orders p, p/2, ..., 1 on the same element grid
 * (each a BP3 Gauss Q = p_k + 2 Dirichlet operator on its own isoparametric mesh
 * of order p_k), prolongation = nodal interpolation of the coarse function,
 * restriction = its transpose (coarse Dirichlet rows zeroed), smoother =
 * Chebyshev acceleration of Jacobi (Saad Alg. 12.1, `degree` steps) on
 * [0.3 lam_hi, lam_hi], lam_hi = 1.2 x the power-iteration estimate (power_iters
 * iterations from the R12 random vector `seed`) of lambda_max(D^-1 A); V-cycle
 * pre-smooth / residual / restrict / recurse / prolong-correct / post-smooth, the
 * coarsest level smoothed twice (no AMG coarse solve: hypre is out of scope).
 * Single rank only (HOFEM_ERR_ARG otherwise). */

/* diag(A) of a partially assembled operator by sum factorization over squared
 * 1D tables (no assembly), interface planes summed across ranks, Dirichlet rows
 * 1 (identity-row convention R6).  d: n_local doubles. */
hofem_status hofem_op_diagonal(void* op, double* d, void* stream);

typedef struct {
  int levels;          /* number of levels (level 0 = the finest, order p) */
  int orders[8];       /* polynomial order of each level */
  double lambda[8];    /* power-iteration estimate of lambda_max(D^-1 A) per level */
  int degree;          /* Chebyshev steps per smoothing pass */
} hofem_pmg_info;
/* SYNC.  Builds the hierarchy on `mesh` (borrowed: it must outlive the handle). */
hofem_status hofem_pmg_create(void* mesh, int degree, int power_iters, unsigned long long seed,
                              void* stream, void** pmg_out);
hofem_status hofem_pmg_info_get(const void* pmg, hofem_pmg_info* info_out);
/* Override level k's eigenvalue estimate (parity testing against the oracle's). */
hofem_status hofem_pmg_set_lambda(void* pmg, int level, double lambda);
/* Borrowed handles of level k (its mesh: vector lengths via hofem_mesh_info_get;
 * its operator: hofem_op_apply etc.).  Owned by the pmg handle. */
hofem_status hofem_pmg_level(void* pmg, int level, void** mesh_out, void** op_out);
/* z = V-cycle(r) on level 0 (r, z: level-0 vectors, must not alias). */
hofem_status hofem_pmg_vcycle(void* pmg, const double* r, double* z, void* stream);
/* One smoothing pass on level k: x <- x + p(D^-1 A) D^-1 (b - A x). */
hofem_status hofem_pmg_smooth(void* pmg, int level, const double* b, double* x, void* stream);
/* Transfers between level k (fine) and k+1 (coarse): dir = 0 prolongation
 * (fine += P coarse: `in` is coarse, `out` fine, accumulated), dir = 1
 * restriction (coarse = R fine, coarse Dirichlet rows 0: `in` fine, `out` coarse). */
hofem_status hofem_pmg_transfer(void* pmg, int level, int dir, const double* in, double* out,
                                void* stream);
/* SYNC.  Preconditioned CG (reading R18) on level 0 with one V-cycle per
 * iteration: x in x0 / out, stop at ||r|| <= rel_tol ||r0||; rr_history (host,
 * nullable, length max_iter+1) receives r_k.r_k.  Status as hofem_cg. */
hofem_status hofem_pmg_pcg(void* pmg, const double* b, double* x, double rel_tol, int max_iter,
                           double* rr_history, hofem_cg_stats* stats, void* stream);
void hofem_pmg_destroy(void* pmg);

/* Kernel timing hooks for the bench's roofline figure.  When enabled, the
 * library records CUDA events on the launching stream around every fused brick
 * kernel and every brick fix-up kernel; hofem_profile_read synchronizes on
 * those events, returns the summed device durations and clears the record. */
typedef struct {
  long long brick_launches;
  double brick_ms;
  long long fixup_launches;
  double fixup_ms;
} hofem_profile_stats;
hofem_status hofem_profile_enable(int enable);
hofem_status hofem_profile_read(hofem_profile_stats* out);

/* How hofem_op_apply runs this operator (for the bench's roofline figure):
 * fused kernel variant (1 = the SIMT thread-per-line brick kernel, incl. its
 * collocated BP5 form; -1 the operator has no fused kernel and apply uses the
 * unfused path), brick shape, work-unit z chunking, and the number of local
 * lattice points the fused kernel completes itself (interior points, and
 * single-face points by two order-independent reductions) vs. through the
 * fix-up (edge lines of the brick grid).  Host-only, no device work. */
typedef struct {
  int variant;
  int bx, by;            /* elements per brick in x, y (one element layer in z) */
  int zc, nchunks;       /* element layers per work unit; units per column */
  int grid;              /* persistent CTAs launched */
  long long direct_points, fixup_points;
} hofem_fused_info;
hofem_status hofem_op_fused_info(const void* op, hofem_fused_info* out);
/* Per-operator schedule options.  Every setting computes the same operator /
 * the same CG recurrence (parity-tested); only the kernel schedule differs.
 * Values: 0 = never, 1 = auto (the measured default: a size threshold),
 * 2 = always (L2_PREFETCH: 0 / 1).  HOFEM_ERR_ARG for an unknown option or value.
 *  INFIX          edge-line fix-up (and the zeroing of y) inside the brick kernel
 *                 behind a grid barrier (cooperative launch) instead of a memset +
 *                 separate fix-up kernel; auto = local meshes <= 8 Mi points.
 *  CG_FUSED_UPDATE  per-iteration CG: r/x/p updates and both dot products in one
 *                 cooperative kernel; auto = single rank, <= 8 Mi dofs.
 *  CG_PERSISTENT  hofem_cg runs the whole solve in ONE cooperative kernel (brick
 *                 pass, fix-up, p.Ap, updates, r.r, stop test, all behind grid
 *                 barriers; §2.3); a single rank, or several
 *                 ranks with the kernel-initiated exchange (otherwise the
 *                 per-iteration kernels run even with "always"; mesh mode 1: the
 *                 interface planes are put into the neighbours' slots and p.Ap /
 *                 r.r allreduced by a chain over the ranks inside the kernel,
 *                 PAPER.md:197); auto = <= 256 Ki local dofs (measured crossover).
 *                 Convergence is then tested every iteration.
 *  L2_PREFETCH    bulk-prefetch the next brick's qdata into L2. */
typedef enum {
  HOFEM_OPT_INFIX = 1,
  HOFEM_OPT_CG_FUSED_UPDATE = 2,
  HOFEM_OPT_CG_PERSISTENT = 3,
  HOFEM_OPT_L2_PREFETCH = 4
} hofem_option;
hofem_status hofem_op_set_option(void* op, hofem_option opt, int value);
hofem_status hofem_op_get_option(const void* op, hofem_option opt, int* value);

/* Number of kernel launches the library issued since the last reset (for the
 * bench's gpu_launches claim); counts every <<<>>> launch of this library. */
long long hofem_launch_count(void);
void hofem_launch_count_reset(void);

#ifdef __cplusplus
}
#endif
#endif /* HOFEM_H */
