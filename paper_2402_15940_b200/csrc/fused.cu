// fused.cu -- dispatch of the fused column kernels (fused_impl.cuh) and the
// brick-interface fix-up kernel that completes the deterministic R^T
// (SURVEY.md §8(a) row a8): every lattice point on an interior x/y brick face or
// a work-unit boundary plane sums the partials of its 2, 4 or 8 bricks in
// ascending brick order.
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "fused_impl.cuh"

namespace hofem {

#define HOFEM_FOR_P1(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9)
#define HOFEM_DECL(P1)                                                                      \
  template <>                                                                               \
  bool fused_launch<P1>(int, int, const double*, const double*, const ColArgs&, int, bool,  \
                        cudaStream_t, cudaError_t*);                                        \
  template <>                                                                               \
  bool cg_launch<P1>(int, int, const double*, const double*, const ColArgs&, const CGArgs&, \
                     int, cudaStream_t, cudaError_t*);                                      \
  template <>                                                                               \
  FusedLaunch fused_shape<P1>(int, int);
HOFEM_FOR_P1(HOFEM_DECL)
#undef HOFEM_DECL

namespace {

// Edge-line fix-up as its own kernel (one thread per edge point, flat
// enumeration: fixup_flat in fused_impl.cuh).
__global__ void __launch_bounds__(256) fixup_kernel(FixArgs F) {
  __shared__ double red[256];
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const double d = g < fixup_count(F) ? fixup_flat(F, g) : 0.0;
  if (F.dotp) block_sum_store(d, F.dotp + blockIdx.x, red);
}

// Sums the x.y partials of the fused kernel and the fix-up in index order.
__global__ void __launch_bounds__(256) dot_partials_kernel(const double* part, long long n,
                                                           double* out) {
  __shared__ double red[256];
  double v = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) v += part[i];
  block_sum_store(v, out, red);
}

FusedLaunch shape_for(int P1, int kind, int Q) {
  switch (P1) {
#define HOFEM_CASE(P) \
  case P:             \
    return fused_shape<P>(kind, Q);
    HOFEM_FOR_P1(HOFEM_CASE)
#undef HOFEM_CASE
  }
  return FusedLaunch{0, 0, 0, 1, 1};
}

int fused_kind(const Op* op) {
  if (op->kind == HOFEM_MASS) return KIND_MASS;
  if (op->rule == HOFEM_GLL && op->Q == op->mesh->P1) return KIND_COLLOC;
  return KIND_DIFF;
}

struct ProfState {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> brick, fixup;
  std::vector<cudaEvent_t> pool;
};
ProfState g_prof;

cudaEvent_t prof_event() {
  if (!g_prof.pool.empty()) {
    cudaEvent_t e = g_prof.pool.back();
    g_prof.pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

}  // namespace

hofem_status profile_enable(int on) {
  g_prof.on = on != 0;
  return HOFEM_OK;
}

hofem_status profile_read(hofem_profile_stats* out) {
  out->brick_launches = (long long)g_prof.brick.size();
  out->fixup_launches = (long long)g_prof.fixup.size();
  out->brick_ms = out->fixup_ms = 0.0;
  for (int which = 0; which < 2; ++which) {
    auto& v = which == 0 ? g_prof.brick : g_prof.fixup;
    for (auto& pr : v) {
      HOFEM_CUDA(cudaEventSynchronize(pr.second));
      float ms = 0.f;
      HOFEM_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
      (which == 0 ? out->brick_ms : out->fixup_ms) += ms;
      g_prof.pool.push_back(pr.first);
      g_prof.pool.push_back(pr.second);
    }
    v.clear();
  }
  return HOFEM_OK;
}

bool fused_supported(const Op* op) {
  const int P1 = op->mesh->P1;
  if (P1 < 2 || P1 > kMaxP + 1) return false;
  if (fused_kind(op) == KIND_COLLOC) return true;
  return op->Q == P1 || op->Q == P1 + 1;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = kNumSMs;
  }
  return n;
}

// Split each column into chunks so that the units fill the persistent grid in
// as few, as full, rounds as possible (fewer chunks on ties: each chunk boundary
// is a plane the fix-up kernel has to sum).
#ifndef HOFEM_CHUNKS_MIN
#define HOFEM_CHUNKS_MIN 1  // tuning knob: at least this many z chunks per column
#endif
void choose_chunks(long long ncol, int nzl, int G, int* zc_out, int* nchunks_out) {
  double best = -1.0;
  int bz = nzl, bn = 1;
  for (int want = HOFEM_CHUNKS_MIN < nzl ? HOFEM_CHUNKS_MIN : nzl; want <= 16 && want <= nzl;
       ++want) {
    const int zc = (nzl + want - 1) / want, nch = (nzl + zc - 1) / zc;
    const long long units = ncol * nch;
    const long long rounds = (units + G - 1) / G;
    const double eff = (double)units / (double)(rounds * G) - 0.002 * nch;
    if (eff > best + 1e-12) { best = eff; bz = zc; bn = nch; }
  }
  *zc_out = bz;
  *nchunks_out = bn;
}

// Dirichlet points of the local slab (the fix-up's boundary pass; same count
// as bnd_count in fused_impl.cuh)
long long boundary_points(const Mesh* m) {
  const long long K0 = (long long)m->p * m->z0;
  const bool bot = K0 == 0, top = K0 + m->Nzl - 1 == m->NzG - 1;
  const long long kz0 = bot ? 1 : 0, kz1 = m->Nzl - (top ? 1 : 0);
  const long long nk = kz1 > kz0 ? kz1 - kz0 : 0;
  return m->Nx * m->Ny * ((bot ? 1 : 0) + (top ? 1 : 0)) + 2 * m->Nx * nk + 2 * (m->Ny - 2) * nk;
}


namespace {
struct Plan {
  int kind;
  FusedLaunch L;
  int nbx, nby, zc, nchunks, grid;
  long long ncol, nbricks, nunits;
};
Plan make_plan(const Op* op, bool for_cg = false) {
  const Mesh* m = op->mesh;
  Plan P;
  P.kind = fused_kind(op);
  P.L = shape_for(m->P1, P.kind, op->Q);
  if (for_cg) P.L.ctas_per_sm = P.L.ctas_per_sm_cg;
  P.nbx = (m->nx + P.L.BX - 1) / P.L.BX;
  P.nby = (m->ny + P.L.BY - 1) / P.L.BY;
  P.ncol = (long long)P.nbx * P.nby;
  P.nbricks = P.ncol * m->nzl;
  const int G0 = num_sms() * P.L.ctas_per_sm;
  P.zc = 1;
  P.nchunks = 1;
  choose_chunks(P.ncol, m->nzl, G0, &P.zc, &P.nchunks);
  P.nunits = P.ncol * P.nchunks;
  P.grid = (int)(P.nunits < G0 ? P.nunits : G0);
  return P;
}

// Everything one launch of the fused kernels needs (ColArgs incl. the fix-up's
// FixArgs), with the operator's scratch buffers sized for it.
struct Prepared {
  Plan PL;
  ColArgs A;
  long long nfixp = 0, nfixb = 0, npts = 0;
  bool need_fix = false, zero_y = false;
};

// Stream-ordered (re)allocation of operator scratch: no implicit device
// synchronization, so a rank of the loopback transport never waits on another
// rank's pending kernels.
template <class T>
hofem_status grow(T** p, long long* len, long long need, const char* what, cudaStream_t s) {
  if (*len >= need) return HOFEM_OK;
  if (*p) cudaFreeAsync(*p, s);
  *p = nullptr;
  *len = 0;
  if (cudaMallocAsync(p, sizeof(T) * need, s) != cudaSuccess) {
    cudaGetLastError();
    set_error("fused apply: out of device memory for %s", what);
    return HOFEM_ERR_OOM;
  }
  *len = need;
  return HOFEM_OK;
}

hofem_status ensure_bar(Op* op, cudaStream_t s) {
  if (op->d_bar) return HOFEM_OK;
  if (cudaMallocAsync(&op->d_bar, sizeof(GridBar), s) != cudaSuccess ||
      cudaMemsetAsync(op->d_bar, 0, sizeof(GridBar), s) != cudaSuccess) {
    cudaGetLastError();
    op->d_bar = nullptr;
    set_error("fused apply: out of device memory for the grid barrier");
    return HOFEM_ERR_OOM;
  }
  return HOFEM_OK;
}

hofem_status prepare(Op* op, const double* x, double* y, bool fdot, Prepared* out,
                     cudaStream_t s, bool for_cg = false) {
  Mesh* m = op->mesh;
  const int p = m->p;
  Prepared& R = *out;
  R.PL = make_plan(op, for_cg);
  const Plan& PL = R.PL;
  const FusedLaunch L = PL.L;
  HOFEM_TRY(grow(&op->d_bbuf, &op->bbuf_len, PL.nbricks * L.face_block,
                 "the brick-interface buffer", s));
  ColArgs& A = R.A;
  A = ColArgs{};
  A.x = x; A.y = y; A.qd = op->d_qdata; A.bbuf = op->d_bbuf;
  A.nx = m->nx; A.ny = m->ny; A.nzl = m->nzl;
  A.nbx = PL.nbx; A.nby = PL.nby; A.zc = PL.zc; A.nunits = (int)PL.nunits;
  A.Nx = m->Nx; A.Ny = m->Ny; A.Nzl = m->Nzl;
  A.K0 = (long long)p * m->z0; A.NzG = m->NzG;
  A.bc = op->bc;
  A.l2pf = op->opt_l2pf ? 1 : 0;
  // fix-up work: edge-line points, plus the Dirichlet boundary points
  // (fixup_bnd; same count as bnd_count in fused_impl.cuh)
  R.nfixp = (long long)(PL.nbx - 1) * (PL.nby - 1) * m->Nzl +
            (long long)(PL.nbx - 1) * (PL.nchunks - 1) * m->Ny +
            (long long)(PL.nby - 1) * (PL.nchunks - 1) * m->Nx;
  if (op->bc) R.nfixp += boundary_points(m);
  if (R.nfixp >= (1LL << 31)) {  // the fix-up indexes its points in 32 bits
    set_error("fused apply: %lld fix-up points exceed the 32-bit index range", R.nfixp);
    return HOFEM_ERR_ARG;
  }
  R.need_fix = R.nfixp > 0;
  R.nfixb = R.need_fix ? (R.nfixp + 255) / 256 : 0;
  if (fdot) HOFEM_TRY(grow(&op->d_dotp, &op->dotp_len, PL.grid + R.nfixb, "the dot partials", s));
  A.dotp = fdot ? op->d_dotp : nullptr;
  A.kown = m->n_owned / (m->Nx * m->Ny);
  FixArgs F;
  F.x = x; F.y = y; F.bbuf = op->d_bbuf;
  F.Nx = (int)m->Nx; F.Ny = (int)m->Ny; F.Nzl = (int)m->Nzl; F.K0 = A.K0; F.NzG = m->NzG;
  F.p = p; F.PX = p * L.BX; F.PY = p * L.BY; F.PZU = p * PL.zc;
  F.LX = F.PX + 1; F.LY = F.PY + 1;
  F.nbx = PL.nbx; F.nby = PL.nby; F.nzl = m->nzl; F.bc = op->bc;
  F.FYS = 2 * (p + 1); F.OY = 0; F.OZ = 2 * F.FYS;  // FaceLayout<>
  F.FZS = F.LX * F.LY; F.FB = F.OZ + 2 * F.FZS;
  if (F.FB != L.face_block) {
    set_error("fused apply: face-block layout mismatch (%d vs %d)", F.FB, L.face_block);
    return HOFEM_ERR_ARG;
  }
  F.nplZ = PL.nchunks - 1; F.nplY = PL.nby - 1; F.nplX = PL.nbx - 1;
  F.dotp = fdot ? op->d_dotp + PL.grid : nullptr;
  F.kown = (int)A.kown;
  A.fx = F;
  R.npts = m->Nx * m->Ny * m->Nzl;
  R.zero_y = PL.nbx > 1 || PL.nby > 1 || PL.nchunks > 1;  // face points are reduced into y
  A.infix = 0;
  A.zero_n = 0;
  A.bar = nullptr;
  return HOFEM_OK;
}

bool launch_p1(int P1, int kind, const Op* op, const ColArgs& A, int grid, bool coop,
               cudaStream_t s, cudaError_t* err) {
  switch (P1) {
#define HOFEM_CASE(P) \
  case P:             \
    return fused_launch<P>(kind, op->Q, op->tab.B, op->tab.G, A, grid, coop, s, err);
    HOFEM_FOR_P1(HOFEM_CASE)
#undef HOFEM_CASE
  }
  return false;
}
}  // namespace

hofem_status fused_info(const Op* op, hofem_fused_info* out) {
  if (!fused_supported(op)) {
    *out = hofem_fused_info{-1, 0, 0, 0, 0, 0, 0, 0};
    return HOFEM_OK;
  }
  const Mesh* m = op->mesh;
  const Plan P = make_plan(op);
  out->variant = 1;
  out->bx = P.L.BX; out->by = P.L.BY; out->zc = P.zc; out->nchunks = P.nchunks;
  out->grid = P.grid;
  // points on >= 2 interior brick planes (edge lines) go through the fix-up
  const long long N = m->Nx * m->Ny * m->Nzl;
  const long long ax = P.nbx - 1, ay = P.nby - 1, az = P.nchunks - 1;
  out->fixup_points = ax * ay * m->Nzl + ax * az * m->Ny + ay * az * m->Nx - 2 * ax * ay * az;
  out->direct_points = N - out->fixup_points;  // (Dirichlet points: boundary pass)
  return HOFEM_OK;
}

hofem_status apply_fused(Op* op, const double* x, double* y, cudaStream_t s,
                         double* dot_out, const double** dot_parts, long long* dot_nparts) {
  Mesh* m = op->mesh;
  const bool fdot = dot_out != nullptr;
  Prepared R;
  HOFEM_TRY(prepare(op, x, y, fdot, &R, s));
  const Plan& PL = R.PL;
  if (PL.nbricks == 0) return HOFEM_OK;
  ColArgs& A = R.A;
  // in-kernel fix-up (cooperative launch, grid barrier).  Measured (gpurun_out/
  // e15, e16): pays for small (launch/latency-bound) problems, neutral or
  // slower at ~30M dofs -- hence the size threshold of the auto setting.
  // (not on a loopback multi-rank mesh: several ranks' grids share one device)
  const bool loopback = m->nranks > 1 && m->comm && m->comm->loop;
  bool infix = R.need_fix && !loopback &&
               (op->opt_infix == 2 || (op->opt_infix == 1 && R.npts <= (8LL << 20)));
  if (infix) HOFEM_TRY(ensure_bar(op, s));
  A.infix = infix ? 1 : 0;
  A.bar = op->d_bar;
  // with infix the zeroing of y moves into the kernel too (first barrier)
  A.zero_n = infix && R.zero_y ? R.npts : 0;
  if (R.zero_y && A.zero_n == 0) {
    // single-face points are completed by two-term reductions onto zero
    HOFEM_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * R.npts, s));
  }
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  if (g_prof.on) {
    ev = {prof_event(), prof_event()};
    cudaEventRecord(ev.first, s);
  }
  cudaError_t err = cudaSuccess;
  bool ok = launch_p1(m->P1, PL.kind, op, A, PL.grid, infix, s, &err);
  if (ok && infix && err == cudaErrorCooperativeLaunchTooLarge) {
    // the device cannot hold the whole grid right now (e.g. shared by another
    // context): memset + plain launch, fix-up as its own kernel
    cudaGetLastError();
    infix = false;
    A.infix = 0;
    if (A.zero_n > 0) {
      A.zero_n = 0;
      HOFEM_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * R.npts, s));
    }
    ok = launch_p1(m->P1, PL.kind, op, A, PL.grid, false, s, &err);
  }
  if (!ok) {
    set_error("fused apply: no fused kernel for p=%d Q=%d", m->p, op->Q);
    return HOFEM_ERR_ARG;
  }
  count_launch();
  if (err != cudaSuccess) return cuda_status(err, "fused brick kernel launch");
  if (g_prof.on) {
    cudaEventRecord(ev.second, s);
    g_prof.brick.push_back(ev);
  }
  if (R.need_fix && !infix) {
    if (g_prof.on) {
      ev = {prof_event(), prof_event()};
      cudaEventRecord(ev.first, s);
    }
    fixup_kernel<<<(unsigned)R.nfixb, 256, 0, s>>>(A.fx);
    HOFEM_LAUNCHED();
    if (g_prof.on) {
      cudaEventRecord(ev.second, s);
      g_prof.fixup.push_back(ev);
    }
  }
  if (fdot) {
    const long long nparts = PL.grid + (R.need_fix && !infix ? R.nfixb : 0);
    if (dot_parts && dot_nparts) {
      *dot_parts = op->d_dotp;  // summed by the caller's kernel, same fixed order
      *dot_nparts = nparts;
    } else {
      dot_partials_kernel<<<1, 256, 0, s>>>(op->d_dotp, nparts, dot_out);
      HOFEM_LAUNCHED();
    }
  }
  return exchange_planes(op, x, y, s);
}

hofem_status cg_persistent(Op* op, double* x, double* r, double* p, double* Ap, double* rr,
                           int max_iter, int fixed, double rel_tol, int* d_result,
                           cudaStream_t s) {
  Mesh* m = op->mesh;
  const bool multi = m->nranks > 1;
  if (!fused_supported(op) || (multi && m->xmode != 1)) {
    set_error("persistent CG: fused operator; several ranks need the kernel-initiated "
              "exchange (hofem_mesh_set_exchange mode 1)");
    return HOFEM_ERR_ARG;
  }
  Prepared R;
  HOFEM_TRY(prepare(op, p, Ap, false, &R, s, true));
  Plan& PL = R.PL;
  // loopback: all ranks' grids share one device and must be co-resident; 1/(R+1)
  // of the device each leaves room for the other ranks' put kernels and the
  // waves of their (non-cooperative) brick kernels
  if (multi && m->comm && m->comm->loop) PL.grid = std::max(1, PL.grid / (m->nranks + 1));
  HOFEM_TRY(ensure_bar(op, s));
  HOFEM_TRY(grow(&op->d_cgparts, &op->cgparts_len, 2LL * PL.grid + 2, "the CG partials", s));
  ColArgs& A = R.A;
  A.infix = 1;
  A.zero_n = 0;  // the CG kernel zeroes Ap itself
  A.bar = op->d_bar;
  // the brick epilogue accumulates x.y terms only when dotp is non-null; the
  // CG kernel stores its own per-CTA sums (G.parts), never A.dotp
  A.dotp = op->d_cgparts;
  A.fx.dotp = nullptr;
  CGArgs G;
  G.n = m->n_local;
  G.n_owned = m->n_owned;
  G.x = x; G.r = r; G.p = p; G.Ap = Ap; G.rr = rr;
  G.parts = op->d_cgparts;
  G.parts2 = op->d_cgparts + PL.grid;
  G.result = d_result;
  G.max_iter = max_iter;
  G.fixed = fixed;
  G.rel_tol = rel_tol;
  G.zero_ap = R.zero_y ? 1 : 0;
  G.multi = multi ? 1 : 0;
  G.X = XArgs{};
  if (multi) {
    XArgs& X = G.X;
    X.R = m->nranks;
    X.rank = m->rank;
    X.plane = m->plane;
    X.Nx = m->Nx; X.Ny = m->Ny; X.NzG = m->NzG;
    X.Klo = (long long)m->p * m->z0;
    X.Khi = X.Klo + m->Nzl - 1;
    X.peer_lo = m->peer_recv[0];
    X.peer_hi = m->peer_recv[1];
    X.pflag_lo = m->peer_flag[0];
    X.pflag_hi = m->peer_flag[1];
    X.recv = m->d_xrecv;
    X.my = m->d_xflag;
    X.seq0 = m->xseq;
    X.rseq0 = m->rseq;
    X.scratch = op->d_cgparts + 2 * PL.grid;
    X.bcmode = op->bc ? 1 : 0;
  }
  cudaError_t err = cudaSuccess;
  bool ok = false;
  switch (m->P1) {
#define HOFEM_CASE(P)                                                                   \
  case P:                                                                               \
    ok = cg_launch<P>(PL.kind, op->Q, op->tab.B, op->tab.G, A, G, PL.grid, s, &err); \
    break;
    HOFEM_FOR_P1(HOFEM_CASE)
#undef HOFEM_CASE
  }
  if (!ok) {
    set_error("persistent CG: no fused kernel for p=%d Q=%d", m->p, op->Q);
    return HOFEM_ERR_ARG;
  }
  if (err != cudaSuccess) {
    cudaGetLastError();
    return cuda_status(err, "persistent CG kernel launch");
  }
  count_launch();
  return HOFEM_OK;
}

}  // namespace hofem
