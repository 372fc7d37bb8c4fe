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

struct FixArgs {
  const double* x;
  double* y;
  const double* bbuf;
  long long K0, NzG;
  int Nx, Ny, Nzl;
  int p, PX, PY, PZU, LX, LY, nbx, nby, nzl, bc;
  int FB, OY, OZ, FYS, FZS;  // FaceLayout<> of the launched kernel
  int nplZ, nplY, nplX;      // interior brick-boundary planes per axis
  double* dotp;              // non-null: one x.y partial per block (flat block index)
  int kown;                  // local planes K < kown are owned
};

__device__ __forceinline__ bool on_plane(int I, int P, int N) {
  return I % P == 0 && I > 0 && I < N - 1;
}

__device__ __forceinline__ int axis_bricks(int I, int P, int nb, int L, bool split, int* br,
                                           int* loc) {
  if (split) {
    br[0] = I / P - 1; loc[0] = L - 1;
    br[1] = I / P;     loc[1] = 0;
    return 2;
  }
  int b = I / P;
  if (b > nb - 1) b = nb - 1;
  br[0] = b;
  loc[0] = I - P * b;
  return 1;
}

// z: bricks are single element layers; only work-unit boundary planes (every
// PZU = p*zc lattice planes) are split between two bricks -- element faces
// inside a unit were summed through the in-kernel carry into the upper brick.
__device__ __forceinline__ int axis_bricks_z(int K, int p, int nzl, bool split, int* br,
                                             int* loc) {
  if (split) {
    br[0] = K / p - 1; loc[0] = p;
    br[1] = K / p;     loc[1] = 0;
    return 2;
  }
  int b = K / p;
  if (b > nzl - 1) b = nzl - 1;
  br[0] = b;
  loc[0] = K - p * b;
  return 1;
}

// The edge lines of the brick grid: lattice points on two or three interior
// brick-boundary planes (4 or 8 contributions).  grid (ceil(line length/256),
// line count, 3): blockIdx.z = 0 x-y lines (along z), 1 x-z lines (along y,
// skipping y planes), 2 y-z lines (along x, skipping x planes).  Each point sums
// its partials in ascending brick order (deterministic).  Points on a single
// plane were completed in the fused kernel by two-term reductions.
__device__ __forceinline__ double fixup_point(const FixArgs& F, int type, int line, int r);
// Flat launch: thread g enumerates the edge points type by type (n0 x-y line
// points, then n1 x-z, then n2 y-z), so no thread idles on a short line type.
__global__ void __launch_bounds__(256) fixup_kernel(FixArgs F) {
  __shared__ double red[256];
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n0 = (long long)F.nplX * F.nplY * F.Nzl, n1 = (long long)F.nplX * F.nplZ * F.Ny,
                  n2 = (long long)F.nplY * F.nplZ * F.Nx;
  double d = 0.0;
  if (g < n0)
    d = fixup_point(F, 0, (int)(g / F.Nzl), (int)(g % F.Nzl));
  else if (g < n0 + n1)
    d = fixup_point(F, 1, (int)((g - n0) / F.Ny), (int)((g - n0) % F.Ny));
  else if (g < n0 + n1 + n2)
    d = fixup_point(F, 2, (int)((g - n0 - n1) / F.Nx), (int)((g - n0 - n1) % F.Nx));
  if (F.dotp) block_sum_store(d, F.dotp + blockIdx.x, red);
}

// One edge-line point (see fixup_kernel); returns its x.y term (0 if none).
__device__ __forceinline__ double fixup_point(const FixArgs& F, int type, int line, int r) {
  int I, J, K;
  if (type == 0) {
    if (line >= F.nplX * F.nplY || r >= F.Nzl) return 0.0;
    I = (line % F.nplX + 1) * F.PX; J = (line / F.nplX + 1) * F.PY; K = r;
  } else if (type == 1) {
    if (line >= F.nplX * F.nplZ || r >= F.Ny) return 0.0;
    I = (line % F.nplX + 1) * F.PX; K = (line / F.nplX + 1) * F.PZU; J = r;
    if (on_plane(J, F.PY, F.Ny)) return 0.0;
  } else {
    if (line >= F.nplY * F.nplZ || r >= F.Nx) return 0.0;
    J = (line % F.nplY + 1) * F.PY; K = (line / F.nplY + 1) * F.PZU; I = r;
    if (on_plane(I, F.PX, F.Nx)) return 0.0;
  }
  const bool zs = on_plane(K, F.PZU, F.Nzl), ys = on_plane(J, F.PY, F.Ny),
             xs = on_plane(I, F.PX, F.Nx);
  int bx[2], ix[2], by[2], iy[2], bz[2], iz[2];
  const int nbxl = axis_bricks(I, F.PX, F.nbx, F.LX, xs, bx, ix);
  const int nbyl = axis_bricks(J, F.PY, F.nby, F.LY, ys, by, iy);
  const int nbzl = axis_bricks_z(K, F.p, F.nzl, zs, bz, iz);
  double s = 0.0;
  for (int c = 0; c < nbzl; ++c)
    for (int b = 0; b < nbyl; ++b)
      for (int a = 0; a < nbxl; ++a) {
        const long long brick = bx[a] + (long long)F.nbx * (by[b] + (long long)F.nby * bz[c]);
        const int off = zs ? F.OZ + (c == 0) * F.FZS + iy[b] * F.LX + ix[a]
                           : F.OY + (b == 0) * F.FYS + (ix[a] == 0 ? 0 : F.p + 1) + iz[c];
        s += F.bbuf[brick * F.FB + off];
      }
  const long long l = I + (long long)F.Nx * (J + (long long)F.Ny * K);
  const double xl = F.x[l];
  if (F.bc) {
    const long long Kg = K + F.K0;
    if (I == 0 || I == F.Nx - 1 || J == 0 || J == F.Ny - 1 || Kg == 0 || Kg == F.NzG - 1) {
      F.y[l] = xl;
      return K < F.kown ? xl * xl : 0.0;  // Dirichlet value: counted by the owner
    }
  }
  F.y[l] = s;
  return xl * s;
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
  out->direct_points = N - out->fixup_points;
  return HOFEM_OK;
}

hofem_status apply_fused(Op* op, const double* x, double* y, cudaStream_t s,
                         double* dot_out) {
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
  const long long nfixp = (long long)(nbx - 1) * (nby - 1) * m->Nzl +
                          (long long)(nbx - 1) * (nchunks - 1) * m->Ny +
                          (long long)(nby - 1) * (nchunks - 1) * m->Nx;
  const int nlines0 = std::max((nbx - 1) * (nby - 1),
                               std::max((nbx - 1) * (nchunks - 1), (nby - 1) * (nchunks - 1)));
  const long long nfixb = nlines0 > 0 ? (nfixp + 255) / 256 : 0;
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
  cudaError_t err = cudaSuccess;
  bool ok = false;
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  if (nbx > 1 || nby > 1 || nchunks > 1) {
    // single-face points are completed by two-term reductions onto zero
    HOFEM_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * m->Nx * m->Ny * m->Nzl, s));
  }
  if (g_prof.on) {
    ev = {prof_event(), prof_event()};
    cudaEventRecord(ev.first, s);
  }
  switch (P1) {
#define HOFEM_CASE(P)                                                            \
  case P:                                                                        \
    ok = fused_launch<P>(kind, variant, op->Q, op->tab.B, op->tab.G, A, grid, s, &err); \
    break;
    HOFEM_FOR_P1(HOFEM_CASE)
#undef HOFEM_CASE
  }
  if (!ok) {
    set_error("fused apply: no fused kernel for p=%d Q=%d", p, op->Q);
    return HOFEM_ERR_ARG;
  }
  count_launch();
  if (err != cudaSuccess) return cuda_status(err, "fused column kernel launch");
  if (g_prof.on) {
    cudaEventRecord(ev.second, s);
    g_prof.brick.push_back(ev);
  }
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
  const int nlines = std::max(F.nplX * F.nplY, std::max(F.nplX * F.nplZ, F.nplY * F.nplZ));
  if (nlines > 0) {
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
    dot_partials_kernel<<<1, 256, 0, s>>>(op->d_dotp, grid + (nlines > 0 ? nfixb : 0), dot_out);
    HOFEM_LAUNCHED();
  }
  HOFEM_TRY(exchange_planes(op, x, y, s));
  if (dot_out && !fdot) return dot_local(m, x, y, dot_out, s);  // owned dofs, after exchange
  return HOFEM_OK;
}

}  // namespace hofem
