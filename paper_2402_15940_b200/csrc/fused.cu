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
#define HOFEM_DECL(P1)                                                                     \
  template <>                                                                              \
  bool fused_launch<P1>(int, int, int, const double*, const double*, const ColArgs&, int,  \
                        cudaStream_t, cudaError_t*);                                       \
  template <>                                                                              \
  FusedLaunch fused_shape<P1>(int, int);                                                   \
  template <>                                                                              \
  int fused_default_variant<P1>(int);
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

// Tuning knob HOFEM_FUSED = "mma" | "simt" overrides the per-p default kernel.
int fused_variant() {
  static const int v = [] {
    const char* e = getenv("HOFEM_FUSED");
    if (!e) return -1;
    if (!strcmp(e, "mma")) return 0;
    if (!strcmp(e, "simt")) return 1;
    return -1;
  }();
  return v;
}

int default_variant(int P1, int kind) {
  switch (P1) {
#define HOFEM_CASE(P) \
  case P:             \
    return fused_default_variant<P>(kind);
    HOFEM_FOR_P1(HOFEM_CASE)
#undef HOFEM_CASE
  }
  return 0;
}

FusedLaunch shape_for(int P1, int kind, int variant) {
  switch (P1) {
#define HOFEM_CASE(P) \
  case P:             \
    return fused_shape<P>(kind, variant);
    HOFEM_FOR_P1(HOFEM_CASE)
#undef HOFEM_CASE
  }
  return FusedLaunch{0, 0, 0, 1};
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
void choose_chunks(long long ncol, int nzl, int G, int* zc_out, int* nchunks_out) {
  double best = -1.0;
  int bz = nzl, bn = 1;
  for (int want = 1; want <= 16 && want <= nzl; ++want) {
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
  int variant, kind;
  FusedLaunch L;
  int nbx, nby, zc, nchunks, grid;
  long long ncol, nbricks, nunits;
};
Plan make_plan(const Op* op) {
  const Mesh* m = op->mesh;
  Plan P;
  P.kind = fused_kind(op);
  const int v = op->fused_variant >= 0 ? op->fused_variant : fused_variant();
  // variant: 0 DMMA, 1 SIMT (mass / diffusion / collocated), 2 the older
  // collocated column kernel (requested as 0 for a collocated operator)
  if (P.kind == KIND_COLLOC)
    P.variant = (v < 0 || v == 1) ? 1 : 2;
  else
    P.variant = v < 0 ? default_variant(m->P1, P.kind) : v;
  P.L = shape_for(m->P1, P.kind, P.variant == 2 ? 0 : P.variant);
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
}  // namespace

hofem_status fused_info(const Op* op, hofem_fused_info* out) {
  if (!fused_supported(op)) {
    *out = hofem_fused_info{-1, 0, 0, 0, 0, 0, 0, 0};
    return HOFEM_OK;
  }
  const Mesh* m = op->mesh;
  const Plan P = make_plan(op);
  out->variant = P.variant;
  out->bx = P.L.BX; out->by = P.L.BY; out->zc = P.zc; out->nchunks = P.nchunks;
  out->grid = P.grid;
  // points on >= 2 interior brick planes (edge lines) go through fixup_kernel
  const long long N = m->Nx * m->Ny * m->Nzl;
  const long long ax = P.nbx - 1, ay = P.nby - 1, az = P.nchunks - 1;
  out->fixup_points = ax * ay * m->Nzl + ax * az * m->Ny + ay * az * m->Nx - 2 * ax * ay * az;
  out->direct_points = N - out->fixup_points;  // (Dirichlet points: boundary pass)
  return HOFEM_OK;
}

hofem_status apply_fused(Op* op, const double* x, double* y, cudaStream_t s,
                         double* dot_out, const double** dot_parts, long long* dot_nparts) {
  Mesh* m = op->mesh;
  const int P1 = m->P1, p = m->p;
  const Plan PL = make_plan(op);
  const int kind = PL.kind, variant = PL.variant == 2 ? 0 : PL.variant;
  const FusedLaunch L = PL.L;
  const int nbx = PL.nbx, nby = PL.nby, zc = PL.zc, nchunks = PL.nchunks, grid = PL.grid;
  const long long nbricks = PL.nbricks, nunits = PL.nunits;
  if (nbricks == 0) return HOFEM_OK;
  const long long need = nbricks * L.face_block;
  if (op->bbuf_len < need) {
    if (op->d_bbuf) cudaFree(op->d_bbuf);
    op->d_bbuf = nullptr;
    op->bbuf_len = 0;
    if (cudaMalloc(&op->d_bbuf, sizeof(double) * need) != cudaSuccess) {
      cudaGetLastError();
      set_error("fused apply: out of device memory for the brick-interface buffer");
      return HOFEM_ERR_OOM;
    }
    op->bbuf_len = need;
  }
  ColArgs A;
  A.x = x; A.y = y; A.qd = op->d_qdata; A.bbuf = op->d_bbuf;
  A.nx = m->nx; A.ny = m->ny; A.nzl = m->nzl;
  A.nbx = nbx; A.nby = nby; A.zc = zc; A.nunits = (int)nunits;
  A.Nx = m->Nx; A.Ny = m->Ny; A.Nzl = m->Nzl;
  A.K0 = (long long)p * m->z0; A.NzG = m->NzG;
  A.bc = op->bc;
  static const int l2pf = [] {
    const char* e = getenv("HOFEM_L2PF");  // tuning knob: 0 disables the L2 bulk prefetch
    return e ? atoi(e) : 1;
  }();
  A.l2pf = l2pf;
  // fused x.y: per-CTA partials of the brick kernel, then one per fix-up block
  const bool fdot = dot_out != nullptr && PL.variant != 2;
  // fix-up work: edge-line points, plus the Dirichlet boundary points
  // (fixup_bnd; same count as bnd_count in fused_impl.cuh)
  long long nfixp = (long long)(nbx - 1) * (nby - 1) * m->Nzl +
                    (long long)(nbx - 1) * (nchunks - 1) * m->Ny +
                    (long long)(nby - 1) * (nchunks - 1) * m->Nx;
  if (op->bc) nfixp += boundary_points(m);
  if (nfixp >= (1LL << 31)) {  // the fix-up indexes its points in 32 bits
    set_error("fused apply: %lld fix-up points exceed the 32-bit index range", nfixp);
    return HOFEM_ERR_ARG;
  }
  const bool need_fix = nfixp > 0;
  const long long nfixb = need_fix ? (nfixp + 255) / 256 : 0;
  if (fdot && op->dotp_len < grid + nfixb) {
    if (op->d_dotp) cudaFree(op->d_dotp);
    op->d_dotp = nullptr;
    op->dotp_len = 0;
    if (cudaMalloc(&op->d_dotp, sizeof(double) * (grid + nfixb)) != cudaSuccess) {
      cudaGetLastError();
      set_error("fused apply: out of device memory for the dot partials");
      return HOFEM_ERR_OOM;
    }
    op->dotp_len = grid + nfixb;
  }
  A.dotp = fdot ? op->d_dotp : nullptr;
  A.kown = m->n_owned / (m->Nx * m->Ny);
  FixArgs F;
  F.x = x; F.y = y; F.bbuf = op->d_bbuf;
  F.Nx = (int)m->Nx; F.Ny = (int)m->Ny; F.Nzl = (int)m->Nzl; F.K0 = A.K0; F.NzG = m->NzG;
  F.p = p; F.PX = p * L.BX; F.PY = p * L.BY; F.PZU = p * zc;
  F.LX = F.PX + 1; F.LY = F.PY + 1;
  F.nbx = nbx; F.nby = nby; F.nzl = m->nzl; F.bc = op->bc;
  F.FYS = 2 * (p + 1); F.OY = 0; F.OZ = 2 * F.FYS;  // FaceLayout<>
  F.FZS = F.LX * F.LY; F.FB = F.OZ + 2 * F.FZS;
  if (F.FB != L.face_block) {
    set_error("fused apply: face-block layout mismatch (%d vs %d)", F.FB, L.face_block);
    return HOFEM_ERR_ARG;
  }
  F.nplZ = nchunks - 1; F.nplY = nby - 1; F.nplX = nbx - 1;
  F.dotp = fdot ? op->d_dotp + grid : nullptr;
  F.kown = (int)A.kown;
  // in-kernel fix-up (SIMT kernel; cooperative launch with a grid barrier)
  static const int infix_env = [] {
    // tuning knob: 0 = always the separate fixup_kernel, 2 = always in-kernel,
    // 1 (default) = in-kernel for local meshes up to 8 Mi lattice points
    const char* e = getenv("HOFEM_INFIX");
    return e ? atoi(e) : 1;
  }();
  // measured (gpurun_out/e15, e16): pays for small (launch/latency-bound)
  // problems, neutral or slower at ~30M dofs
  const long long npts = m->Nx * m->Ny * m->Nzl;
  bool infix = (infix_env == 1 ? npts <= (8LL << 20) : infix_env == 2) &&
               PL.variant == 1 && need_fix && grid <= nunits;
  if (infix && !op->d_bar) {
    if (cudaMalloc(&op->d_bar, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMemset(op->d_bar, 0, sizeof(unsigned long long)) != cudaSuccess) {
      cudaGetLastError();
      set_error("fused apply: out of device memory for the grid barrier");
      return HOFEM_ERR_OOM;
    }
    op->bar_count = 0;
  }
  const bool zero_y = nbx > 1 || nby > 1 || nchunks > 1;  // face points are reduced into y
  A.infix = infix ? 1 : 0;
  A.bar = op->d_bar;
  // with infix the zeroing of y moves into the kernel too (first barrier)
  A.zero_n = infix && zero_y ? m->Nx * m->Ny * m->Nzl : 0;
  const unsigned long long nbar = infix ? (A.zero_n > 0 ? 2ULL : 1ULL) : 0ULL;
  A.bar_target0 = op->bar_count + (unsigned long long)grid;
  A.bar_target = op->bar_count + nbar * (unsigned long long)grid;
  A.fx = F;
  cudaError_t err = cudaSuccess;
  bool ok = false;
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  if (zero_y && A.zero_n == 0) {
    // single-face points are completed by two-term reductions onto zero
    HOFEM_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * m->Nx * m->Ny * m->Nzl, s));
  }
  if (g_prof.on) {
    ev = {prof_event(), prof_event()};
    cudaEventRecord(ev.first, s);
  }
  auto launch = [&]() {
    switch (P1) {
#define HOFEM_CASE(P)                                                                     \
  case P:                                                                                 \
    ok = fused_launch<P>(kind, variant, op->Q, op->tab.B, op->tab.G, A, grid, s, &err); \
    break;
      HOFEM_FOR_P1(HOFEM_CASE)
#undef HOFEM_CASE
    }
  };
  launch();
  if (ok && infix && err == cudaErrorCooperativeLaunchTooLarge) {
    // the device cannot hold the whole grid right now (e.g. shared by another
    // context): memset + plain launch, fix-up as its own kernel
    cudaGetLastError();
    infix = false;
    A.infix = 0;
    err = cudaSuccess;
    if (A.zero_n > 0) {
      A.zero_n = 0;
      HOFEM_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * m->Nx * m->Ny * m->Nzl, s));
    }
    launch();
  }
  if (!ok) {
    set_error("fused apply: no fused kernel for p=%d Q=%d", p, op->Q);
    return HOFEM_ERR_ARG;
  }
  count_launch();
  if (err != cudaSuccess) return cuda_status(err, "fused column kernel launch");
  if (infix) op->bar_count = A.bar_target;  // every CTA arrived at each barrier
  if (g_prof.on) {
    cudaEventRecord(ev.second, s);
    g_prof.brick.push_back(ev);
  }
  if (need_fix && !infix) {
    if (g_prof.on) {
      ev = {prof_event(), prof_event()};
      cudaEventRecord(ev.first, s);
    }
    fixup_kernel<<<(unsigned)nfixb, 256, 0, s>>>(F);
    HOFEM_LAUNCHED();
    if (g_prof.on) {
      cudaEventRecord(ev.second, s);
      g_prof.fixup.push_back(ev);
    }
  }
  if (fdot) {
    const long long nparts = grid + (need_fix && !infix ? nfixb : 0);
    if (dot_parts && dot_nparts) {
      *dot_parts = op->d_dotp;  // summed by the caller's kernel, same fixed order
      *dot_nparts = nparts;
    } else {
      dot_partials_kernel<<<1, 256, 0, s>>>(op->d_dotp, nparts, dot_out);
      HOFEM_LAUNCHED();
    }
  }
  HOFEM_TRY(exchange_planes(op, x, y, s));
  if (dot_out && !fdot) return dot_local(m, x, y, dot_out, s);  // owned dofs, after exchange
  return HOFEM_OK;
}

}  // namespace hofem
