// fused.cu -- dispatch of the fused column kernels (fused_impl.cuh) and the
// brick-interface fix-up kernel that completes the deterministic R^T
// (SURVEY.md §8(a) row a8): every lattice point on an interior x/y brick face or
// a work-unit boundary plane sums the partials of its 2, 4 or 8 bricks in
// ascending brick order.
#include <stdlib.h>

#include <vector>

#include "fused_impl.cuh"

namespace hofem {

#define HOFEM_FOR_P1(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9)
#define HOFEM_DECL(P1)                                                                     \
  template <>                                                                              \
  bool fused_launch<P1>(int, int, const double*, const double*, const ColArgs&, int,       \
                        cudaStream_t, cudaError_t*);                                       \
  template <>                                                                              \
  FusedLaunch fused_shape<P1>(int);
HOFEM_FOR_P1(HOFEM_DECL)
#undef HOFEM_DECL

namespace {

struct FixArgs {
  const double* x;
  double* y;
  const double* bbuf;
  long long Nx, Ny, Nzl, K0, NzG;
  int p, PX, PY, PZU, LX, LY, nbx, nby, nzl, bc;
  long long BLAT, nZ, nY, nX;
};

__device__ __forceinline__ bool on_plane(long long I, int P, long long N) {
  return I % P == 0 && I > 0 && I < N - 1;
}

__device__ __forceinline__ int axis_bricks(long long I, int P, int nb, long long N, int L,
                                           int* br, int* loc) {
  if (on_plane(I, P, N)) {
    br[0] = (int)(I / P) - 1; loc[0] = L - 1;
    br[1] = (int)(I / P);     loc[1] = 0;
    return 2;
  }
  int b = (int)(I / P);
  if (b > nb - 1) b = nb - 1;
  br[0] = b;
  loc[0] = (int)(I - (long long)P * b);
  return 1;
}

// z: bricks are single element layers; only work-unit boundary planes (every
// PZU = p*zc lattice planes) are split between two bricks -- element faces
// inside a unit were summed through the in-kernel carry into the upper brick.
__device__ __forceinline__ int axis_bricks_z(long long K, int p, int PZU, int nzl, long long N,
                                             int* br, int* loc) {
  if (on_plane(K, PZU, N)) {
    br[0] = (int)(K / p) - 1; loc[0] = p;
    br[1] = (int)(K / p);     loc[1] = 0;
    return 2;
  }
  int b = (int)(K / p);
  if (b > nzl - 1) b = nzl - 1;
  br[0] = b;
  loc[0] = (int)(K - (long long)p * b);
  return 1;
}

__global__ void fixup_kernel(FixArgs F) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long I, J, K;
  if (t < F.nZ) {
    long long m = t / (F.Nx * F.Ny) + 1, r = t % (F.Nx * F.Ny);
    K = m * F.PZU; I = r % F.Nx; J = r / F.Nx;
  } else if ((t -= F.nZ) < F.nY) {
    long long m = t / (F.Nx * F.Nzl) + 1, r = t % (F.Nx * F.Nzl);
    J = m * F.PY; I = r % F.Nx; K = r / F.Nx;
    if (on_plane(K, F.PZU, F.Nzl)) return;
  } else if ((t -= F.nY) < F.nX) {
    long long m = t / (F.Ny * F.Nzl) + 1, r = t % (F.Ny * F.Nzl);
    I = m * F.PX; J = r % F.Ny; K = r / F.Ny;
    if (on_plane(J, F.PY, F.Ny) || on_plane(K, F.PZU, F.Nzl)) return;
  } else {
    return;
  }
  int bx[2], ix[2], by[2], iy[2], bz[2], iz[2];
  int nbxl = axis_bricks(I, F.PX, F.nbx, F.Nx, F.LX, bx, ix);
  int nbyl = axis_bricks(J, F.PY, F.nby, F.Ny, F.LY, by, iy);
  int nbzl = axis_bricks_z(K, F.p, F.PZU, F.nzl, F.Nzl, bz, iz);
  double s = 0.0;
  for (int c = 0; c < nbzl; ++c)
    for (int b = 0; b < nbyl; ++b)
      for (int a = 0; a < nbxl; ++a) {
        long long brick = bx[a] + (long long)F.nbx * (by[b] + (long long)F.nby * bz[c]);
        s += F.bbuf[brick * F.BLAT + ix[a] + F.LX * (iy[b] + (long long)F.LY * iz[c])];
      }
  long long l = I + F.Nx * (J + F.Ny * K);
  if (F.bc) {
    long long Kg = K + F.K0;
    if (I == 0 || I == F.Nx - 1 || J == 0 || J == F.Ny - 1 || Kg == 0 || Kg == F.NzG - 1)
      s = F.x[l];
  }
  F.y[l] = s;
}

FusedLaunch shape_for(int P1, int kind) {
  switch (P1) {
#define HOFEM_CASE(P) \
  case P:             \
    return fused_shape<P>(kind);
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

hofem_status apply_fused(Op* op, const double* x, double* y, cudaStream_t s) {
  Mesh* m = op->mesh;
  const int P1 = m->P1, p = m->p, kind = fused_kind(op);
  FusedLaunch L = shape_for(P1, kind);
  const int nbx = (m->nx + L.BX - 1) / L.BX, nby = (m->ny + L.BY - 1) / L.BY;
  const long long ncol = (long long)nbx * nby;
  const long long nbricks = ncol * m->nzl;
  if (nbricks == 0) return HOFEM_OK;
  const int G0 = num_sms() * L.ctas_per_sm;
  int zc = 1, nchunks = 1;
  choose_chunks(ncol, m->nzl, G0, &zc, &nchunks);
  const long long nunits = ncol * nchunks;
  const int grid = (int)(nunits < G0 ? nunits : G0);
  const long long need = nbricks * L.blat;
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
  cudaError_t err = cudaSuccess;
  bool ok = false;
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  if (g_prof.on) {
    ev = {prof_event(), prof_event()};
    cudaEventRecord(ev.first, s);
  }
  switch (P1) {
#define HOFEM_CASE(P)                                                            \
  case P:                                                                        \
    ok = fused_launch<P>(kind, op->Q, op->tab.B, op->tab.G, A, grid, s, &err);   \
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
  F.Nx = m->Nx; F.Ny = m->Ny; F.Nzl = m->Nzl; F.K0 = A.K0; F.NzG = m->NzG;
  F.p = p; F.PX = p * L.BX; F.PY = p * L.BY; F.PZU = p * zc;
  F.LX = F.PX + 1; F.LY = F.PY + 1;
  F.nbx = nbx; F.nby = nby; F.nzl = m->nzl; F.bc = op->bc;
  F.BLAT = L.blat;
  F.nZ = (long long)(nchunks - 1) * m->Nx * m->Ny;
  F.nY = (long long)(nby - 1) * m->Nx * m->Nzl;
  F.nX = (long long)(nbx - 1) * m->Ny * m->Nzl;
  const long long nt = F.nZ + F.nY + F.nX;
  if (nt > 0) {
    if (g_prof.on) {
      ev = {prof_event(), prof_event()};
      cudaEventRecord(ev.first, s);
    }
    fixup_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, s>>>(F);
    HOFEM_LAUNCHED();
    if (g_prof.on) {
      cudaEventRecord(ev.second, s);
      g_prof.fixup.push_back(ev);
    }
  }
  return exchange_planes(op, x, y, s);
}

}  // namespace hofem
