// fused_impl.cuh -- the fused sm_100a operator kernels (SURVEY.md §8(a) rows
// a4-a9; north star "one fused sm_100a kernel per operator").
//
// Persistent "column" kernel: a grid of SMs x (resident CTAs per SM) CTAs (the
// residency from the occupancy API).  A work unit is a column of bricks --
// BX*BY elements in x,y by one element layer in z -- over a chunk of zc element
// layers; the CTA streams the column bottom to top.  Per brick it does:
//   a4  gather R: the brick's (p*BX+1)(p*BY+1)(p+1) lattice of x, read with
//       asynchronous 8-byte copies into a double-buffered shared-memory lattice
//       (the NEXT brick's lattice is in flight while this one computes);
//       Dirichlet dofs and out-of-mesh points are zero-filled (reading R6);
//   a5  B: the 1D B1d/G1d contractions dimension by dimension (x, then y in
//       shared memory; z in registers, one thread per (qx,qy) quadrature column);
//   a6  D: the pointwise qdata, streamed from L2 into registers inside stage 3
//       (the next point pairs' loads in flight while a pair computes); the
//       brick's qdata was bulk-prefetched into L2 one brick ahead, so the
//       dominant HBM stream runs ahead of the math without shared memory (D is
//       staged in shared memory by bulk copies only at P1 = 9);
//   a7  B^T: the transposed contractions (z in registers, then y, x in smem);
//   a8  R^T: a deterministic in-brick sum -- every brick lattice point sums its
//       1..4 element contributions in ascending element order; the top lattice
//       plane is carried in shared memory and added (in fixed order) to the
//       bottom plane of the next brick of the column, so z-faces inside a unit
//       never leave the SM.  Points on exactly one shared brick face are added to
//       the zeroed y by two order-independent reductions; points on two or three
//       (the brick grid's edge lines) go to a per-brick partial buffer that the
//       fix-up sums in ascending brick order; all others are stored to y.
//   a9  y[ess] = x[ess] (the fix-up's boundary pass).
// The 1D tables (even-odd halves) live in the kernel-parameter constant bank and
// are read as uniform constant loads (no shared-memory traffic for B/G).
//
// Shared-memory layouts keep consecutive lanes on consecutive or odd-strided
// doubles (conflict-free 64-bit accesses): see DESIGN.md §4.
#pragma once

#include <type_traits>

#include "internal.h"
#include "simt_layout.h"

#ifndef HOFEM_SIMT_DSMEM
#define HOFEM_SIMT_DSMEM -1  // SIMT: D staged in smem (1), from L2 in registers (0), per p (-1)
#endif
#ifndef HOFEM_SIMT_EO
#define HOFEM_SIMT_EO 1  // SIMT: even-odd (symmetry-halved) 1D contractions
#endif
#ifndef HOFEM_EO_DLA
#define HOFEM_EO_DLA 0  // SIMT-EO stage 3: point pairs of D loads in flight (0: per p)
#endif
#ifndef HOFEM_EO_PRE
#define HOFEM_EO_PRE -1  // SIMT-EO: stage-3 D loads of the first round issued before stage 2
                          // (1: into registers, 2: L1 prefetch, 0: no, -1: per p)
#endif
#ifndef HOFEM_EO_ZO
#define HOFEM_EO_ZO 1  // table offsets through a loop-variant zero (no hoisting)
#endif
#ifndef HOFEM_L2PF_AHEAD
#define HOFEM_L2PF_AHEAD 1  // SIMT: qdata L2 bulk prefetch this many bricks ahead
#endif
#ifndef HOFEM_EO_DPOL
#define HOFEM_EO_DPOL -1  // SIMT-EO: L2 policy of the stage-3 D loads (see ld_dp; -1 per p)
#endif
#ifndef HOFEM_L2PF_POL
#define HOFEM_L2PF_POL -1  // 1: the qdata L2 prefetch marks its lines evict_last (-1: per P1)
#endif
#ifndef HOFEM_SIMT_T2QX
#define HOFEM_SIMT_T2QX -1  // SIMT: 1 = T2 [m][qy][c][qx] with qx-fastest stage-2 items
                            // (simt_layout.h), 0 = T2 [m][qy][qx][c], -1 = per P1 (measured)
#endif
#ifndef HOFEM_LAT_KF
#define HOFEM_LAT_KF 0  // lattice copies / epilogue rows with k (z) fastest across lanes
                        // (measured r2h: no gain for BP3, -5 % for BP5 at p = 5)
#endif
#ifndef HOFEM_SIMT_ENDBAR
#define HOFEM_SIMT_ENDBAR -1  // SIMT: 1 = barrier at the end of every brick, 0 = folded (see
                               // kernel), -1 = per kind (measured, gpurun_out/e17)
#endif

namespace hofem {

// CTA barrier.  __syncthreads() is `bar.sync` (.aligned): every thread of a
// warp must reach it convergently.  compute-sanitizer synccheck caught warps
// arriving diverged (lanes of one warp still in a different compile-time
// epilogue segment), which gave layout-dependent wrong answers; the item
// loops (FOR_ITEMS) and the warp-uniform epilogue segments below remove the
// divergence, and the explicit __syncwarp documents the requirement.
__device__ __forceinline__ void cta_sync() {
  __syncwarp();
  __syncthreads();
}

// Item loop with a warp-uniform trip count: for it = first, first+NT, ... < N.
// The per-lane bound is an `if` inside each round, so every lane leaves the
// loop together and divergence stays inside structured if-bodies (a per-lane
// trip count left warps diverged at the next CTA barrier, see cta_sync).
#define FOR_ITEMS(it, N, NT, first)                                  \
  for (int it##_base = 0; it##_base < (N); it##_base += (NT))        \
    if (const int it = it##_base + (first); it < (N))

// 1D tables.  B/G [q][i] row-major; BE/BO/GE/GO are their even-odd halves
// (fill_tab): the GLL nodes and the Gauss/GLL points are symmetric about 1/2,
// so B[Q-1-q][P-1-i] = B[q][i] and G[Q-1-q][P-1-i] = -G[q][i], and
//   ME[t][i] = (M[t][i] + M[t][P-1-i]) / 2   (i < P/2;  ME[t][P/2] = M[t][P/2] for odd P)
//   MO[t][i] = (M[t][i] - M[t][P-1-i]) / 2   (i < P/2)
// for rows t < ceil(Q/2).  A contraction of length P -> Q then costs about
// half the multiply-adds (even-odd decomposition of symmetric 1D operators).
template <int P1, int Q>
struct Tab {
  static constexpr int H = (P1 + 1) / 2, PH = P1 / 2, HQ = (Q + 1) / 2;
  double B[Q * P1];
  double G[Q * P1];
  double BE[HQ * H], BO[HQ * PH], GE[HQ * H], GO[HQ * PH];
};

template <int P1, int Q>
inline void fill_tab(Tab<P1, Q>& T, const double* B, const double* G) {
  using TT = Tab<P1, Q>;
  for (int i = 0; i < Q * P1; ++i) {
    T.B[i] = B ? B[i] : 0.0;
    T.G[i] = G[i];
  }
  for (int t = 0; t < TT::HQ; ++t) {
    for (int i = 0; i < TT::PH; ++i) {
      const int j = P1 - 1 - i;
      T.BE[t * TT::H + i] = 0.5 * (T.B[t * P1 + i] + T.B[t * P1 + j]);
      T.BO[t * TT::PH + i] = 0.5 * (T.B[t * P1 + i] - T.B[t * P1 + j]);
      T.GE[t * TT::H + i] = 0.5 * (T.G[t * P1 + i] + T.G[t * P1 + j]);
      T.GO[t * TT::PH + i] = 0.5 * (T.G[t * P1 + i] - T.G[t * P1 + j]);
    }
    if (P1 & 1) {
      T.BE[t * TT::H + TT::PH] = T.B[t * P1 + TT::PH];
      T.GE[t * TT::H + TT::PH] = T.G[t * P1 + TT::PH];
    }
  }
}

// ---------------------------------------------------------------------------
// Edge-line fix-up (a8): lattice points on two or three interior brick-boundary
// planes (4 or 8 contributions) sum their partials in ascending brick order
// (deterministic).  Points on a single plane were completed in the fused kernel
// by two-term reductions.  Run either as fixup_kernel (fused.cu) after the
// brick kernel or inside the SIMT kernel after a grid barrier (ColArgs::infix).
// ---------------------------------------------------------------------------
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
        s += __ldcg(F.bbuf + brick * F.FB + off);  // written by other CTAs
      }
  const long long l = I + (long long)F.Nx * (J + (long long)F.Ny * K);
  if (F.bc) {
    const long long Kg = K + F.K0;
    if (I == 0 || I == F.Nx - 1 || J == 0 || J == F.Ny - 1 || Kg == 0 || Kg == F.NzG - 1)
      return 0.0;  // Dirichlet point: written by the boundary pass (fixup_bnd)
  }
  F.y[l] = s;
  return F.x[l] * s;
}

// a9 boundary pass: y = x at every Dirichlet point of the local slab (global
// boundary I, J or Kg in {0, max}), x.x counted by the owning rank.  The brick
// kernels skip these points, so their x loads leave the brick epilogue.
// Enumeration: global-bottom / global-top planes, then the two y faces, then
// the two x faces (without the rows already covered).
struct BndCount {
  long long nz, ny, nx;
  int kz0, nk;
  bool bot, top;
};
__device__ __forceinline__ BndCount bnd_count(const FixArgs& F) {
  BndCount b;
  b.bot = F.K0 == 0;
  b.top = F.K0 + F.Nzl - 1 == F.NzG - 1;
  const long long plane = (long long)F.Nx * F.Ny;
  b.kz0 = b.bot ? 1 : 0;
  const int kz1 = F.Nzl - (b.top ? 1 : 0);
  b.nk = kz1 > b.kz0 ? kz1 - b.kz0 : 0;
  b.nz = F.bc ? plane * ((b.bot ? 1 : 0) + (b.top ? 1 : 0)) : 0;
  b.ny = F.bc ? 2LL * F.Nx * b.nk : 0;
  b.nx = F.bc ? 2LL * (F.Ny - 2) * b.nk : 0;
  return b;
}
__device__ __forceinline__ double fixup_bnd(const FixArgs& F, const BndCount& b, long long g64) {
  // 32-bit index arithmetic (the boundary of one slab has < 2^31 points)
  unsigned g = (unsigned)g64;
  const unsigned Nx = (unsigned)F.Nx, Ny = (unsigned)F.Ny, plane = Nx * Ny;
  const unsigned nz = (unsigned)b.nz, ny = (unsigned)b.ny;
  int I, J, K;
  if (g < nz) {
    K = (b.bot && g < plane) ? 0 : F.Nzl - 1;
    const unsigned r = g < plane ? g : g - plane;
    I = (int)(r % Nx);
    J = (int)(r / Nx);
  } else if ((g -= nz) < ny) {
    const unsigned face = Nx * (unsigned)b.nk;
    const unsigned r = g < face ? g : g - face;
    J = g < face ? 0 : F.Ny - 1;
    I = (int)(r % Nx);
    K = b.kz0 + (int)(r / Nx);
  } else {
    g -= ny;
    const unsigned face = (Ny - 2) * (unsigned)b.nk;
    const unsigned r = g < face ? g : g - face;
    I = g < face ? 0 : F.Nx - 1;
    J = 1 + (int)(r % (Ny - 2));
    K = b.kz0 + (int)(r / (Ny - 2));
  }
  const long long l = I + (long long)F.Nx * (J + (long long)F.Ny * K);
  const double xl = F.x[l];
  F.y[l] = xl;
  return K < F.kown ? xl * xl : 0.0;
}

// Flat enumeration of the edge points, type by type: n0 x-y line points (along
// z), then n1 x-z (along y, skipping y planes), then n2 y-z (along x).
// (then, with Dirichlet conditions, the boundary points: fixup_bnd)
__device__ __forceinline__ long long fixup_edges(const FixArgs& F) {
  return (long long)F.nplX * F.nplY * F.Nzl + (long long)F.nplX * F.nplZ * F.Ny +
         (long long)F.nplY * F.nplZ * F.Nx;
}
__device__ __forceinline__ long long fixup_count(const FixArgs& F) {
  const BndCount b = bnd_count(F);
  return fixup_edges(F) + b.nz + b.ny + b.nx;
}
__device__ __forceinline__ double fixup_flat(const FixArgs& F, long long g64) {
  const long long ne = fixup_edges(F);
  if (g64 >= ne) return fixup_bnd(F, bnd_count(F), g64 - ne);
  // 32-bit index arithmetic (< 2^31 edge points per slab)
  const unsigned g = (unsigned)g64;
  const unsigned n0 = (unsigned)F.nplX * F.nplY * F.Nzl, n1 = (unsigned)F.nplX * F.nplZ * F.Ny;
  if (g < n0) return fixup_point(F, 0, (int)(g / (unsigned)F.Nzl), (int)(g % (unsigned)F.Nzl));
  if (g < n0 + n1)
    return fixup_point(F, 1, (int)((g - n0) / (unsigned)F.Ny), (int)((g - n0) % (unsigned)F.Ny));
  return fixup_point(F, 2, (int)((g - n0 - n1) / (unsigned)F.Nx),
                     (int)((g - n0 - n1) % (unsigned)F.Nx));
}

struct ColArgs {
  const double* x;
  double* y;
  const double* qd;
  double* bbuf;
  int nx, ny, nzl;        // local element counts
  int nbx, nby;           // bricks per axis in x, y (a brick is BX x BY x 1 elements)
  int zc, nunits;         // element layers per work unit; units = nbx*nby*chunks
  long long Nx, Ny, Nzl;  // local lattice sizes
  long long K0, NzG;      // global index of local plane 0; global plane count
  int bc;
  int l2pf;               // 1: bulk-prefetch the next brick's qdata into L2
  double* dotp;           // non-null: per-CTA partials of x.y over owned dofs (CG's pAp)
  long long kown;         // local planes K < kown are owned by this rank
  // in-kernel fix-up (SIMT kernel, cooperative launch): after all bricks, a grid
  // barrier, then the edge points of fx
  int infix;
  GridBar* bar;           // self-resetting grid barrier (internal.h)
  FixArgs fx;
  // with infix: y (zero_n doubles) zeroed in-kernel before a first grid barrier
  // instead of a cudaMemsetAsync
  long long zero_n;
};

// Fixed-order block sum; thread 0 stores it to *out.  All threads must call.
// `red` is blockDim.x doubles of free shared scratch.
__device__ __forceinline__ void block_sum_store(double v, double* out, double* red) {
  // every thread's value through shared memory, summed in thread order by
  // warp 0 (lane l adds threads l, l+32, ...), then across lanes in order
  cta_sync();
  red[threadIdx.x] = v;
  cta_sync();
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int i = threadIdx.x; i < (int)blockDim.x; i += 32) s += red[i];
    red[threadIdx.x] = s;
  }
  cta_sync();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < 32 && i < (int)blockDim.x; ++i) s += red[i];
    *out = s;
  }
}

enum { KIND_MASS = 0, KIND_DIFF = 1, KIND_COLLOC = 2 };


__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int n = valid ? 8 : 0;  // src-size 0 => zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(n)
               : "memory");
}
// threadIdx.x through a volatile read: per-brick index arithmetic is then
// recomputed inside the persistent loop instead of being hoisted into
// long-lived registers (which starves the contraction stages).
__device__ __forceinline__ int vtid() {
  int t;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
  return t;
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
}


// ---------------------------------------------------------------------------
// a4: items are (lattice row (j,k), element column s): a thread loads the row's
// points i = p s .. p s + p - 1 (plus i = p BX for the last column) with
// asynchronous 8-byte copies; the inner loop is unrolled so each point is a
// compile-time offset from the row base.  Bricks that touch neither the mesh
// boundary nor a ragged edge take a predicate-free path.
// ---------------------------------------------------------------------------
template <class C, int NT, int BX>
__device__ __forceinline__ void issue_lattice(const ColArgs& A, double* L, long long I0,
                                              long long J0, long long K0l) {
  constexpr int LX = C::LX, LY = C::LY, LZ = C::LZ, p = C::p;
  const long long nvx = A.Nx - I0;  // lattice points of this brick inside the mesh along x
  const long long Kg0 = K0l + A.K0;
  const bool interior = I0 > 0 && I0 + LX < A.Nx && J0 > 0 && J0 + LY < A.Ny &&
                        (!A.bc || (Kg0 > 0 && Kg0 + LZ < A.NzG));
  FOR_ITEMS(it, LY * LZ * BX, NT, vtid()) {
    const int sx = it % BX, r = it / BX;
    const int j = HOFEM_LAT_KF ? r / LZ : r % LY, k = HOFEM_LAT_KF ? r % LZ : r / LY;
    const long long J = J0 + j, K = K0l + k;
    double* dst = L + C::lat(p * sx, j, k);
    if (interior) {
      const double* src = A.x + I0 + p * sx + A.Nx * (J + A.Ny * K);
#pragma unroll
      for (int ii = 0; ii < p; ++ii) cp_async8(dst + C::LXS * ii, src + ii, true);
      if (sx == BX - 1) cp_async8(dst + C::LXS * p, src + p, true);
    } else {
      const long long Kg = K + A.K0;
      const bool rin = J < A.Ny;
      const bool ress = A.bc && (J == 0 || J == A.Ny - 1 || Kg == 0 || Kg == A.NzG - 1);
      const double* src = A.x + (rin ? I0 + A.Nx * (J + A.Ny * K) : 0);
#pragma unroll
      for (int ii = 0; ii <= p; ++ii) {
        if (ii < p || sx == BX - 1) {
          const long long i = p * sx + ii;
          const bool valid = rin && !ress && i < nvx &&
                             !(A.bc && ((I0 + i) == 0 || (I0 + i) == A.Nx - 1));
          cp_async8(dst + C::LXS * ii, valid ? src + i : A.x, valid);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// a8 + a9 for one brick (element layer ez of a column).  Items are (lattice
// row (j,k), element column sx); sx is dispatched to a compile-time template
// argument so that, per point, which elements contribute and whether the point
// lies on an x face of the brick are compile-time facts.  Along x and y a
// lattice index has a "lower" contribution (element q-1, local node p) on an
// element face and a "primary" one (element q, node i - p q); along z there is
// one element layer (node k).  Ascending element order: y outer, x inner.
// k == 0 adds the carried top plane of the previous brick first; k == p goes to
// the carry unless the brick ends the unit.
// ---------------------------------------------------------------------------
// Interior brick faces.  A lattice point on exactly ONE shared face (x, y or
// z-unit plane) has exactly two contributions, a (this brick) and b (the
// neighbour); y is zeroed before the kernel and both bricks add with an FP64
// reduction: 0 + a + b == 0 + b + a bitwise (IEEE addition is commutative and
// 0 + a is exact), so the result is deterministic in any order.  Points on two
// or three shared faces (the edge lines of the brick grid) have 4 or 8
// contributions; they go to the brick's face block in the partial buffer and
// fixup_kernel (fused.cu) sums them in ascending brick order.  Face block: y
// faces [ys][k][i], z-unit faces [zs][j][i]; a point on a z-unit face is stored
// in the z face, otherwise in the y face (x-only points never get here).
template <int p, int LX, int LY>
struct FaceLayout {
  static constexpr int P1 = p + 1;
  static constexpr int OY = 0;                  // y faces
  // a y face only ever holds its two x-end columns (the z lines of the brick
  // grid): [ys][x end][k], k fastest, so the fix-up reads a z line contiguously
  static constexpr int FYS = 2 * P1;
  static constexpr int OZ = OY + 2 * FYS;       // z faces
  static constexpr int FZS = LX * LY;
  static constexpr int FB = OZ + 2 * FZS;       // doubles per brick
  __device__ __forceinline__ static int yf(int ys, int k) { return OY + ys * FYS + k; }
  __device__ __forceinline__ static int zf(int zs, int j) { return OZ + zs * FZS + j * LX; }
};

__device__ __forceinline__ void red_add(double* p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

struct EpiRow {
  const double* cin;
  double* cout;
  double* bb;   // shared-face row (z-unit or y face) in the brick's face block
  long long gl;
  int base0, base1;  // y-element offsets of the lower / primary contributions
  bool vy0, vy1, to_carry, from_carry, row_sh, row_multi, row_ess, yface;
  // fused x.y (CG's pAp): lattice row of x, owned row (Dirichlet terms), lower side of the
  // row's shared y/z face (a Dirichlet point on one shared face is written by
  // both bricks and counted by the lower one only)
  const double* lx;
  bool dot, own, face_lo;
};

template <class C, int BX, bool NATURAL, int ESTRIDE, int SX>
__device__ __forceinline__ void epi_segment(const ColArgs& A, const double* RA, const EpiRow& R,
                                            long long I0, long long nvx, long long iess,
                                            bool exok_lo, bool exok, bool xlo_sh, bool xhi_sh,
                                            bool xlo_ess, double& dsum) {
  constexpr int p = C::p, LX = C::LX;
  // x.y by contributions: every contribution this brick writes counts (also on
  // the non-owned top plane: the neighbour rank counts ITS contributions there);
  // a Dirichlet value y = x counts once, on the owning rank.
  const bool acc = R.dot;
  constexpr int NPT = (SX == BX - 1) ? p + 1 : p;  // the last column also owns i = p*BX
  double v[NPT];
#pragma unroll
  for (int ii = 0; ii < NPT; ++ii) {
    double s = R.from_carry ? R.cin[p * SX + ii] : 0.0;
#pragma unroll
    for (int cy = 0; cy < 2; ++cy) {
      const bool vy = cy ? R.vy1 : R.vy0;
      const int base = cy ? R.base1 : R.base0;
      if (ii == 0 && SX > 0) {  // lower contribution: element SX-1, node p
        if (vy && exok_lo) s += RA[base + (SX - 1) * ESTRIDE + (NATURAL ? p : C::SA * p)];
      }
      if (ii < p) {
        if (vy && exok) s += RA[base + SX * ESTRIDE + (NATURAL ? ii : C::SA * ii)];
      } else {
        if (vy && exok) s += RA[base + SX * ESTRIDE + (NATURAL ? p : C::SA * p)];
      }
    }
    v[ii] = s;
  }
  // Destinations: row-uniform cases first (carry, partial buffer), then the
  // common interior case with compile-time x-face handling; the rare rows that
  // touch the Dirichlet boundary or a ragged mesh edge take the general path.
  const int nv = (int)(nvx < LX ? nvx : LX);
  if (R.to_carry) {
#pragma unroll
    for (int ii = 0; ii < NPT; ++ii)
      if (p * SX + ii < nv) R.cout[p * SX + ii] = v[ii];
    return;
  }
  const int ie = (int)(iess >= 0 && iess < LX ? iess : -1);
  if (R.row_sh) {  // row on a y face or a z-unit face
#pragma unroll
    for (int ii = 0; ii < NPT; ++ii) {
      const int i = p * SX + ii;
      if (i >= nv) continue;
      const bool lo = (SX == 0 && ii == 0), hi = (SX == BX - 1 && ii == p);
      if (R.row_multi || (lo && xlo_sh) || (hi && xhi_sh)) {
        R.bb[R.yface ? (i == 0 ? 0 : p + 1) : i] = v[ii];  // edge line: partial buffer
      } else if (R.row_ess || (lo && xlo_ess) || i == ie) {
        // Dirichlet point: y = x and its x.y term come from the fix-up pass
      } else {
        red_add(A.y + R.gl + i, v[ii]);
        if (acc) dsum = fma(R.lx[C::LXS * i], v[ii], dsum);
      }
    }
    return;
  }
  if (!R.row_ess && nv == LX && ie < 0 && !xlo_ess) {
#pragma unroll
    for (int ii = 0; ii < NPT; ++ii) {
      const bool lo = (SX == 0 && ii == 0), hi = (SX == BX - 1 && ii == p);
      if ((lo && xlo_sh) || (hi && xhi_sh))
        red_add(A.y + R.gl + p * SX + ii, v[ii]);
      else
        A.y[R.gl + p * SX + ii] = v[ii];
      if (acc) dsum = fma(R.lx[C::LXS * (p * SX + ii)], v[ii], dsum);
    }
    return;
  }
#pragma unroll
  for (int ii = 0; ii < NPT; ++ii) {
    const int i = p * SX + ii;
    if (i >= nv) continue;
    const bool lo = (SX == 0 && ii == 0), hi = (SX == BX - 1 && ii == p);
    const bool ess = R.row_ess || (lo && xlo_ess) || (i == ie);
    if (!ess) {  // Dirichlet points: y = x and x.y in the fix-up pass
      if ((lo && xlo_sh) || (hi && xhi_sh))
        red_add(A.y + R.gl + i, v[ii]);
      else
        A.y[R.gl + i] = v[ii];
      if (acc) dsum = fma(R.lx[C::LXS * i], v[ii], dsum);
    }
  }
}

template <class C, int BX, bool NATURAL, int ESTRIDE, int SX>
__device__ __forceinline__ void epi_dispatch(int sx, const ColArgs& A, const double* RA,
                                             const EpiRow& R, long long I0, long long nvx,
                                             long long iess, const bool* exok, bool xlo_sh,
                                             bool xhi_sh, bool xlo_ess, double& dsum) {
  if constexpr (SX < BX) {
    if (sx == SX)
      epi_segment<C, BX, NATURAL, ESTRIDE, SX>(A, RA, R, I0, nvx, iess,
                                               SX > 0 ? exok[SX > 0 ? SX - 1 : 0] : false,
                                               exok[SX], xlo_sh, xhi_sh, xlo_ess, dsum);
    else
      epi_dispatch<C, BX, NATURAL, ESTRIDE, SX + 1>(sx, A, RA, R, I0, nvx, iess, exok, xlo_sh,
                                                    xhi_sh, xlo_ess, dsum);
  }
}

template <class C, int NT, int BX, int BY, bool NATURAL, int ESTRIDE = C::YEN, int EOFF = 0>
__device__ __forceinline__ void brick_epilogue(const ColArgs& A, const double* RA,
                                               const double* carry_in, double* carry_out,
                                               long long brick, int ex0, int ey0, long long I0,
                                               long long J0, long long K0l, bool first,
                                               bool last, const double* Lx, double& dsum) {
  constexpr int p = C::p, P1 = p + 1, LX = C::LX, LY = C::LY;
  RA += EOFF;
  const long long nvx = A.Nx - I0;
  const bool xlo_sh = I0 > 0, xhi_sh = I0 + LX - 1 < A.Nx - 1;
  const bool xlo_ess = A.bc && I0 == 0;
  const long long iess = A.bc ? A.Nx - 1 - I0 : -1;
  bool exok[BX];
#pragma unroll
  for (int q = 0; q < BX; ++q) exok[q] = ex0 + q < A.nx;
  // items (element column sx, row r): the rows of one column are padded to a
  // multiple of 32 so every warp runs a single compile-time segment SX
  constexpr int ROWS = LY * P1, RPS = (ROWS + 31) / 32 * 32;
  FOR_ITEMS(it, RPS * BX, NT, threadIdx.x) {
    const int sx = it / RPS, r = it % RPS;
    const int j = HOFEM_LAT_KF ? r / P1 : r % LY, k = HOFEM_LAT_KF ? r % P1 : r / LY;
    if (r >= ROWS) continue;
    const long long J = J0 + j, K = K0l + k, Kg = K + A.K0;
    if (J >= A.Ny) continue;
    const int qj = j / p, rj = j - qj * p;
    EpiRow R;
    R.vy0 = rj == 0 && qj > 0 && ey0 + qj - 1 < A.ny;
    R.vy1 = qj < BY && ey0 + qj < A.ny;
    R.base0 = BX * (qj - 1) * ESTRIDE + (NATURAL ? P1 * (p + P1 * k) : k + P1 * p);
    R.base1 = BX * qj * ESTRIDE + (NATURAL ? P1 * (rj + P1 * k) : k + P1 * rj);
    R.to_carry = (k == p) && !last;
    R.from_carry = (k == 0) && !first;
    const bool ysh = (j == 0 && J > 0) || (j == LY - 1 && J < A.Ny - 1);
    const bool zsh = (k == 0 && first && K > 0) || (k == p && last && K < A.Nzl - 1);
    R.row_sh = ysh || zsh;
    R.row_multi = ysh && zsh;
    R.row_ess = A.bc && (J == 0 || J == A.Ny - 1 || Kg == 0 || Kg == A.NzG - 1);
    R.gl = I0 + A.Nx * (J + A.Ny * K);
    {
      using FL = FaceLayout<p, LX, LY>;
      double* fb = A.bbuf + brick * FL::FB;
      R.bb = zsh ? fb + FL::zf(k == 0 ? 0 : 1, j) : fb + FL::yf(j == 0 ? 0 : 1, k);
      R.yface = !zsh;
    }
    R.cin = carry_in + LX * j;
    R.cout = carry_out + LX * j;
    R.dot = A.dotp != nullptr;
    R.own = K < A.kown;
    R.face_lo = ysh ? j == 0 : k == 0;
    R.lx = Lx + C::lat(0, j, k);
    epi_dispatch<C, BX, NATURAL, ESTRIDE, 0>(sx, A, RA, R, I0, nvx, iess, exok, xlo_sh, xhi_sh,
                                             xlo_ess, dsum);
  }
}

// ---------------------------------------------------------------------------
// The CTA's brick sequence: units u = blockIdx.x, blockIdx.x + G, ...; within a
// unit the element layers z0 .. z1-1 of one column.  Pipelining crosses unit
// boundaries (the next brick may start a new unit).
// ---------------------------------------------------------------------------
struct Brick {
  int u, bx, by, z0, z1, ez;  // u >= nunits => past the end
};
__device__ __forceinline__ Brick unit_first(const ColArgs& A, int u) {
  Brick b;
  b.u = u;
  if (u >= A.nunits) { b.bx = b.by = b.z0 = b.z1 = b.ez = 0; return b; }
  const int ncol = A.nbx * A.nby, col = u % ncol, chunk = u / ncol;
  b.bx = col % A.nbx;
  b.by = col / A.nbx;
  b.z0 = chunk * A.zc;
  b.z1 = min(A.nzl, b.z0 + A.zc);
  b.ez = b.z0;
  return b;
}
__device__ __forceinline__ Brick brick_next(const ColArgs& A, Brick b) {
  if (b.ez + 1 < b.z1) { ++b.ez; return b; }
  return unit_first(A, b.u + gridDim.x);
}

// mbarrier / bulk-copy (TMA) helpers.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{ .reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra LAB_WAIT;\n"
      "}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// qdata staging slot per element: NC*NQ^3 doubles, widened to 16-byte
// boundaries (+2 doubles) because bulk copies move 16-byte granules.
template <class C>
struct Stage {
  static constexpr int PER = C::NC * C::NQ1 * C::NQ1 * C::NQ1;  // doubles per element
  static constexpr int SLOT = ((PER + 2) + 1) / 2 * 2;
};

// Thread 0: one bulk copy per element of brick b into staging buffer qs;
// arms the buffer's mbarrier with the byte count.  Elements outside the mesh
// are skipped.
template <class C, int BX, int BY>
__device__ __forceinline__ void issue_qdata(const ColArgs& A, const Brick& b, double* qs,
                                            unsigned long long* bar) {
  if (threadIdx.x != 0 || b.u >= A.nunits) return;
  constexpr long long per = (long long)Stage<C>::PER * 8;
  unsigned total = 0;
  long long lo[BX * BY], hi[BX * BY];
#pragma unroll
  for (int el = 0; el < BX * BY; ++el) {
    const int ex = b.bx * BX + el % BX, ey = b.by * BY + el / BX;
    lo[el] = hi[el] = 0;
    if (ex < A.nx && ey < A.ny) {
      const long long e = ex + (long long)A.nx * (ey + (long long)A.ny * b.ez);
      lo[el] = (e * per) & ~15LL;
      hi[el] = ((e + 1) * per + 15) & ~15LL;
      total += (unsigned)(hi[el] - lo[el]);
    }
  }
  fence_proxy_async();
  mbar_expect_tx(bar, total);
  const char* base = reinterpret_cast<const char*>(A.qd);
#pragma unroll
  for (int el = 0; el < BX * BY; ++el)
    if (hi[el] > lo[el])
      bulk_g2s(qs + el * Stage<C>::SLOT, base + lo[el], (unsigned)(hi[el] - lo[el]), bar);
}

// Offset (0 or 1 double) of element (ex,ey,ez)'s data inside its staging slot.
template <class C>
__device__ __forceinline__ int stage_off(const ColArgs& A, int ex, int ey, int ez) {
  constexpr long long per = (long long)Stage<C>::PER * 8;
  if (per % 16 == 0) return 0;
  const long long e = ex + (long long)A.nx * (ey + (long long)A.ny * ez);
  return (int)(((e * per) & 15LL) >> 3);
}

// Thread 0: warm L2 with brick b's qdata (one bulk prefetch per element).
template <class C, int BX, int BY>
__device__ __forceinline__ void prefetch_qdata_l2(const ColArgs& A, const Brick& b) {
  if (threadIdx.x != 0 || b.u >= A.nunits || !A.l2pf) return;
  constexpr long long per = (long long)C::NC * C::NQ1 * C::NQ1 * C::NQ1 * 8;
  const char* base = reinterpret_cast<const char*>(A.qd);
#pragma unroll
  for (int el = 0; el < BX * BY; ++el) {
    const int ex = b.bx * BX + el % BX, ey = b.by * BY + el / BX;
    if (ex < A.nx && ey < A.ny) {
      const long long e = ex + (long long)A.nx * (ey + (long long)A.ny * b.ez);
      const long long lo = (e * per) & ~15LL, hi = ((e + 1) * per + 15) & ~15LL;
      // evict_last: measured -1.1 % on the config-5 slab, neutral at 62^3, for the
      // P1 = 6 1x3 brick (profiles/ab/r2v_ab_p6knobs3.txt); off elsewhere (round 2)
      if (HOFEM_L2PF_POL >= 0 ? HOFEM_L2PF_POL != 0 : C::P == 6 && C::KINDV == KIND_DIFF) {
        unsigned long long pol;
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(base + lo),
                     "r"((unsigned)(hi - lo)), "l"(pol)
                     : "memory");
      } else {
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + lo),
                     "r"((unsigned)(hi - lo))
                     : "memory");
      }
    }
  }
}

// ---------------------------------------------------------------------------
// SIMT kernel (mass / diffusion): thread-per-line sum factorization.
//
// Every 1D contraction is an item = one line of the element tensor held in
// registers: a thread loads the line's P (or Q) inputs and produces all Q (or P)
// outputs of every product at once, so the FP64 FMA chains are independent
// (ILP 7..21) and the table operands are compile-time constant-bank entries
// (uniform-register DFMA operands; no shared traffic for B/G).  Items of all
// NE elements of the brick are spread over the CTA's threads; stages are
// separated by __syncthreads.  Stage 3 (z, pointwise D, z back) runs entirely
// in registers with D read straight from L2 (prefetched one brick ahead).
//   S1  item (b,c):  T1[m][qx][b][c]   m: 0 = B_x x, 1 = G_x x
//   S2  item (qx,c): T2[m][qy][qx][c]  m: 0 = G_x B_y, 1 = B_x G_y, 2 = B_x B_y
//   S3  item (qx,qy): in place in T2: z contraction, D, z back-contraction
//   S2T item (qx,c): T1[0] = B_y^T (.. y,z parts), T1[1] = B_y^T (x part)
//   S1T item (b,c):  y_e[a][b][c] (aliases T2)
// Strides: S1 == P (mod 16) and c-fastest S2 items make S2/S2T's T1 accesses
// conflict-free; SP (the T2 point stride) is odd so S3 is conflict-free
// (scripts/simt_layout.py checks the layouts).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Volatile read-only load: stays in program order w.r.t. the other volatile
// loads, so a register pipeline written in the source is kept.
__device__ __forceinline__ double ld_nc_v(const double* ptr) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(ptr));
  return v;
}

template <bool SMEM>
__device__ __forceinline__ double ld_d(const double* ptr) {
  if constexpr (SMEM)
    return *ptr;
  else
    return ld_nc_v(ptr);
}
// stage-3 D load with an L2 policy (HOFEM_EO_DPOL: 1 = evict_first hint,
// 2 = evict_first + no L1 allocation; 0 = plain ld_d)
// measured (gpurun_out/e7): evict_first + no L1 allocation is 6 % faster at p = 6,
// slower at p = 4, 5
template <int P1>
constexpr int eo_dpol() {
  return HOFEM_EO_DPOL >= 0 ? HOFEM_EO_DPOL : (P1 == 7 ? 2 : 0);
}
template <bool SMEM, int DPOL>
__device__ __forceinline__ double ld_dp(const double* ptr, unsigned long long pol) {
  if constexpr (SMEM || DPOL == 0) {
    (void)pol;
    return ld_d<SMEM>(ptr);
  } else {
    double v;
    if (DPOL == 1)
      asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(ptr), "l"(pol));
    else
      asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                   : "=d"(v)
                   : "l"(ptr), "l"(pol));
    return v;
  }
}

// Per-P1 stage layout (HOFEM_SIMT_T2QX = -1).  Measured (gpurun_out/r2h, r2i;
// profiles/ab/r2h_ab_layout.txt, r2i_ab_layout2.txt; brick-kernel ms at 30M
// dofs): qx-fastest T2 wins at P1 = 2 (BP3 -2.7 %), 3 (BP3 -4 %, BP5 -6 %),
// 4 (BP3 -5 %), 6 (p=5: BP3 -2.7 %, BP5 -5 %) and 8 (p=7: BP3 -12 %, BP5 -6 %);
// loses at P1 = 5 (BP3 +2.5 %, BP5 +8 %); at P1 = 7 BP3 even, BP5 -1.3 % (r2m);
// ~neutral at P1 = 9 (old kept).
template <int P1>
constexpr bool simt_t2qx() {
  return HOFEM_SIMT_T2QX >= 0 ? HOFEM_SIMT_T2QX != 0
                              : (P1 == 2 || P1 == 3 || P1 == 4 || P1 == 6 || P1 == 7 || P1 == 8);
}

template <int KIND, int P1, int Q, int BX, int BY>
struct CfgS {
  static constexpr int p = P1 - 1, P = P1, NE = BX * BY, KINDV = KIND;
  static constexpr int LX = p * BX + 1, LY = p * BY + 1, LZ = P1;
  static constexpr int LXS = ((LY * LZ) % 2 == 0) ? LY * LZ + 1 : LY * LZ;
  static constexpr int LAT = LXS * LX;
  static constexpr int cmax(int a, int b) { return a > b ? a : b; }
  static constexpr int NA = (KIND == KIND_MASS) ? 1 : 2;
  static constexpr int NB = (KIND == KIND_MASS) ? 1 : 3;
  static constexpr int NC = (KIND == KIND_MASS) ? 1 : 6;
  static constexpr int SA = ((P * P) % 2 == 0) ? P * P + 1 : P * P;
  static constexpr int YEN = SA * P;
  // T1 [m][qx][b*P+c]: qx stride S1.  QXF: T2 [m][qy][c][qx] (qy stride TY,
  // c stride TC = Q), stage-2 items qx fastest, strides from the generated
  // conflict search (simt_layout.h; every kind keeps the diffusion block's
  // residue mod 16).  Otherwise T2 [m][qy][qx][c] with odd point stride SP and
  // c-fastest stage-2 items.
  static constexpr bool QXF = simt_t2qx<P1>();
  using LYT = LayoutS<P1, Q, NE>;
  static constexpr int SPO = (P % 2) ? P : P + 1;
  static constexpr int S1 = QXF ? LYT::S1 : P * P + (((P - P * P) % 16) + 16) % 16;
  static constexpr int SP = QXF ? P : SPO;
  static constexpr int TY = QXF ? LYT::RS : Q * SPO, TX = QXF ? 1 : SPO, TC = QXF ? Q : 1;
  static constexpr int T1M = Q * S1, T1SZ = NA * T1M;
  static constexpr int T2M = Q * TY;
  static constexpr int EB0 = T1SZ + cmax(NB * T2M, YEN);
  static constexpr int EBD = 2 * Q * S1 + cmax(3 * T2M, YEN) + LYT::EBPAD;
  static constexpr int EB = QXF ? EB0 + ((EBD - EB0) % 16 + 16) % 16
                                : EB0 + ((7 - EB0) % 16 + 16) % 16;  // old: == 7 (mod 16)
  static constexpr int CARRY = LX * LY;
  static constexpr int TOFF0 = NE * EB + 2 * LAT + 2 * CARRY;
  static constexpr int TOFF = TOFF0 + (TOFF0 & 1);  // 16-byte aligned
  // D staged in shared memory (one buffer, bulk-copied one brick ahead) or
  // loaded from L2 into registers inside stage 3.
  static constexpr bool DSM =
      HOFEM_SIMT_DSMEM >= 0 ? HOFEM_SIMT_DSMEM != 0 : (P1 == 9);  // measured
  static constexpr int QOFF = TOFF;  // D stage (DSM), 16-byte aligned
  static constexpr int QSLOT = ((NC * Q * Q * Q + 2) + 1) / 2 * 2;
  static constexpr int SMEM_DOUBLES = QOFF + (DSM ? NE * QSLOT : 0);
  static constexpr int SMEM_BYTES = SMEM_DOUBLES * 8;
  static constexpr int NQ1 = Q;
  __device__ static constexpr int lat(int i, int j, int k) { return k + LZ * j + LXS * i; }
};

template <class C, int NT, int BX, int BY>
__device__ __forceinline__ void simt_epilogue(const ColArgs& A, double* smem, double* CY,
                                              const Brick& b, const double* L, double& dsum) {
  constexpr int p = C::p;
  const int ex0 = b.bx * BX, ey0 = b.by * BY, ez = b.ez;
  const long long brick = b.bx + (long long)A.nbx * (b.by + (long long)A.nby * ez);
  brick_epilogue<C, NT, BX, BY, false, C::EB, C::T1SZ>(
      A, smem, CY + ((ez + 1) & 1) * C::CARRY, CY + (ez & 1) * C::CARRY, brick, ex0, ey0,
      (long long)p * ex0, (long long)p * ey0, (long long)p * ez, ez == b.z0, ez + 1 == b.z1, L, dsum);
}

// ---- even-odd contractions (tables BE/BO/GE/GO of Tab, constant bank).  S is
// the symmetry sign of the 1D matrix: +1 for B, -1 for G.
template <int P>
struct EOn {
  static constexpr int H = (P + 1) / 2, PH = P / 2;
};
// v[P] -> e[i] = v[i] + v[P-1-i], o[i] = v[i] - v[P-1-i] (i < P/2); e[P/2] = v[P/2] (odd P)
template <int P>
__device__ __forceinline__ void eo_split(const double (&v)[P], double (&e)[EOn<P>::H],
                                         double (&o)[EOn<P>::PH]) {
#pragma unroll
  for (int i = 0; i < P / 2; ++i) {
    e[i] = v[i] + v[P - 1 - i];
    o[i] = v[i] - v[P - 1 - i];
  }
  if (P & 1) e[P / 2] = v[P / 2];
}
// row . v over N entries (table row from the constant bank, zo = loop-variant 0)
template <int N>
__device__ __forceinline__ double cdot(const double* row, int zo, const double (&v)[N]) {
  double s = row[zo] * v[0];
#pragma unroll
  for (int i = 1; i < N; ++i) s = fma(row[i + zo], v[i], s);
  return s;
}
// forward pair t < Q/2: outputs at q = t (lo) and q = Q-1-t (hi)
template <int S, int P>
__device__ __forceinline__ void eo_fwd(const double* ME, const double* MO, int t, int zo,
                                       const double (&e)[EOn<P>::H],
                                       const double (&o)[EOn<P>::PH], double& lo, double& hi) {
  constexpr int H = EOn<P>::H, PH = EOn<P>::PH;
  const double E = cdot<H>(ME + t * H, zo, e), O = cdot<PH>(MO + t * PH, zo, o);
  lo = E + O;
  hi = S > 0 ? E - O : O - E;
}
// forward middle row (odd Q): B rows are even (O = 0), G rows odd (E = 0)
template <int S, int P>
__device__ __forceinline__ double eo_fwd_mid(const double* ME, const double* MO, int t, int zo,
                                             const double (&e)[EOn<P>::H],
                                             const double (&o)[EOn<P>::PH]) {
  constexpr int H = EOn<P>::H, PH = EOn<P>::PH;
  return S > 0 ? cdot<H>(ME + t * H, zo, e) : cdot<PH>(MO + t * PH, zo, o);
}
// transposed accumulate of the pair (w at q = t, w at q = Q-1-t) into SE/SO
template <int S, int P>
__device__ __forceinline__ void eo_acc(const double* ME, const double* MO, int t, int zo,
                                       double wlo, double whi, double (&SE)[EOn<P>::H],
                                       double (&SO)[EOn<P>::PH]) {
  constexpr int H = EOn<P>::H, PH = EOn<P>::PH;
  const double we = S > 0 ? wlo + whi : wlo - whi;
  const double wo = S > 0 ? wlo - whi : wlo + whi;
#pragma unroll
  for (int i = 0; i < H; ++i) SE[i] = fma(ME[t * H + i + zo], we, SE[i]);
#pragma unroll
  for (int i = 0; i < PH; ++i) SO[i] = fma(MO[t * PH + i + zo], wo, SO[i]);
}
template <int S, int P>
__device__ __forceinline__ void eo_acc_mid(const double* ME, const double* MO, int t, int zo,
                                           double w, double (&SE)[EOn<P>::H],
                                           double (&SO)[EOn<P>::PH]) {
  constexpr int H = EOn<P>::H, PH = EOn<P>::PH;
  if (S > 0) {
#pragma unroll
    for (int i = 0; i < H; ++i) SE[i] = fma(ME[t * H + i + zo], w, SE[i]);
  } else {
#pragma unroll
    for (int i = 0; i < PH; ++i) SO[i] = fma(MO[t * PH + i + zo], w, SO[i]);
  }
}
// r[i] = SE[i] + SO[i], r[P-1-i] = SE[i] - SO[i]; r[P/2] = SE[P/2] (odd P)
template <int P>
__device__ __forceinline__ void eo_join(const double (&SE)[EOn<P>::H],
                                        const double (&SO)[EOn<P>::PH], double (&r)[P]) {
#pragma unroll
  for (int i = 0; i < P / 2; ++i) {
    r[i] = SE[i] + SO[i];
    r[P - 1 - i] = SE[i] - SO[i];
  }
  if (P & 1) r[P / 2] = SE[P / 2];
}
template <int N>
__device__ __forceinline__ void zero(double (&v)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = 0.0;
}

// D of the point pair t of a z line (qz = t and Q-1-t; the middle point alone)
template <bool SMEM, int NCD, int Q, int DPOL>
__device__ __forceinline__ void eo_ldpair(const double* qde, int t, double (&d)[2][NCD],
                                          unsigned long long pol) {
  constexpr int Q2 = Q * Q, Q3 = Q * Q * Q;
  const bool mid = (Q & 1) && t == Q / 2;
#pragma unroll
  for (int m = 0; m < NCD; ++m) {
    d[0][m] = ld_dp<SMEM, DPOL>(qde + m * Q3 + t * Q2, pol);
    d[1][m] = mid ? 0.0 : ld_dp<SMEM, DPOL>(qde + m * Q3 + (Q - 1 - t) * Q2, pol);
  }
}


// One pass of the brick pipeline over all of this CTA's work units: y = A x
// (A.x -> A.y) for the CTA's bricks, edge-line partials to A.bbuf, x.y terms of
// the values written into dsum.  Shared memory must have been set up by
// simt_prologue; qbar / qphase carry the D-staging mbarrier state (DSM) across
// passes.  A CTA without a work unit returns at once.
template <int KIND, int P1, int Q, int BX, int BY, int NT, int MAXR, bool EO>
__device__ __forceinline__ void simt_pass(const Tab<P1, Q>& T, const ColArgs& A,
                                          unsigned long long* qbar, unsigned& qphase,
                                          double& dsum) {
  using C = CfgS<KIND, P1, Q, BX, BY>;
  constexpr int P = P1, p = P1 - 1, NE = C::NE;
  constexpr int Q2 = Q * Q, Q3 = Q * Q * Q;
  constexpr int H = (P + 1) / 2, PH = P / 2, QH = Q / 2;  // even-odd sizes (EO)
  (void)H; (void)PH; (void)QH;
  // EO stage 3: D of LA point pairs in flight; EOPRE: the first round's are
  // issued before stage 2 (registers live across S2 and the barrier)
  constexpr int HQ = (Q + 1) / 2, NCD = KIND == KIND_MASS ? 1 : 6;
  // measured (gpurun_out/e4, e5, e8): register hoist helps at p = 6, 7 (3-4 %), costs
  // at p = 4, 5 (register cap 128); deeper rings and L1 prefetch do not help
  // measured (gpurun_out/r2m, r2n; profiles/ab/r2m_ab_knobs.txt, r2n_ab_p6.txt):
  // two pairs in flight at P1 = 6 (BP3 -1.8 %, BP5 -3.1 %); the first-pair hoist
  // pays more for collocated BP5 at P1 = 6 (-6.4 %) but not with two pairs in
  // flight (+5.6 %), and not for BP3 (+14 %)
  constexpr int LA0 =
      HOFEM_EO_DLA > 0 ? HOFEM_EO_DLA : (P1 == 6 && KIND != KIND_COLLOC ? 2 : 1);
  constexpr int LA = LA0 < HQ ? LA0 : HQ;
  // (P1 = 8: the hoist won with round 1's layout; with the searched layout it
  // costs BP3 p=7 6.3 % and BP5 1.5 %, r2o -- off)
  constexpr int PRE = HOFEM_EO_PRE >= 0
                          ? HOFEM_EO_PRE
                          : (P1 == 7 || (P1 == 6 && KIND == KIND_COLLOC) ? 1 : 0);
  constexpr bool EOPRE = EO && !C::DSM && PRE == 1;
  // COLLOC (BP5): GLL points = nodes, so B = I; every B contraction is the
  // identity and is skipped (diffusion structure otherwise).
  constexpr bool COL = KIND == KIND_COLLOC;
  constexpr bool DIFF = KIND == KIND_DIFF || COL;
  // folded end-of-brick barrier: +1-2 % for BP1/BP3, -1.5 % for BP5
  constexpr bool ENDBAR = HOFEM_SIMT_ENDBAR >= 0 ? HOFEM_SIMT_ENDBAR != 0 : COL;
  constexpr int EB = C::EB, S1 = C::S1, T1M = C::T1M, T1SZ = C::T1SZ, SP = C::SP,
                T2M = C::T2M, TY = C::TY, TX = C::TX, TC = C::TC;
  (void)SP;
  extern __shared__ __align__(16) double smem[];
  double* LB = smem + NE * EB;
  double* CY = LB + 2 * C::LAT;
  double* QS = smem + C::QOFF;  // staged D of the current brick (DSM)
  (void)QS; (void)CY;
  Brick cur = unit_first(A, blockIdx.x);
  if (cur.u >= A.nunits) return;  // no work unit for this CTA
  if (C::DSM) {
    issue_qdata<C, BX, BY>(A, cur, QS, qbar);
  } else {
    prefetch_qdata_l2<C, BX, BY>(A, cur);
    if (HOFEM_L2PF_AHEAD > 1) prefetch_qdata_l2<C, BX, BY>(A, brick_next(A, cur));
  }
  issue_lattice<C, NT, BX>(A, LB, (long long)p * cur.bx * BX, (long long)p * cur.by * BY,
                           (long long)p * cur.ez);
  cp_async_wait_all();
  cta_sync();
  constexpr int DPOL = eo_dpol<P1>();
  unsigned long long dpol = 0;
  if (DPOL) dpol = evict_first_policy();
  for (int kb = 0; cur.u < A.nunits; ++kb) {
    const int tid = vtid();
#if HOFEM_EO_ZO
    const int zo = cur.ez >> 30;  // == 0, loop-variant (see eo_fwd / cdot)
#else
    constexpr int zo = 0;  // EO tables: direct constant-bank operands
#endif
    (void)zo;
    const Brick nxt = brick_next(A, cur);
    const int ex0 = cur.bx * BX, ey0 = cur.by * BY, ez = cur.ez;
    const double* L = LB + (kb & 1) * C::LAT;
    if (nxt.u < A.nunits) {
      if (ENDBAR)
        issue_lattice<C, NT, BX>(A, LB + ((kb + 1) & 1) * C::LAT, (long long)p * nxt.bx * BX,
                                 (long long)p * nxt.by * BY, (long long)p * nxt.ez);
      if (HOFEM_L2PF_AHEAD > 1)
        prefetch_qdata_l2<C, BX, BY>(A, brick_next(A, nxt));
      else
        prefetch_qdata_l2<C, BX, BY>(A, nxt);
    }

    // ---- S1: contract x.  item (el, b, c), c fastest.
    FOR_ITEMS(it, NE * P * P, NT, tid) {
      const int el = it / (P * P), r = it % (P * P), b = r / P, c = r % P;
      const double* xl = L + C::lat(p * (el % BX), p * (el / BX) + b, c);
      double xa[P];
#pragma unroll
      for (int a = 0; a < P; ++a) xa[a] = xl[C::LXS * a];
      double* t1 = smem + el * EB + r;
      {
        double e[H], o[PH];
        eo_split<P>(xa, e, o);
#pragma unroll
        for (int t = 0; t < QH; ++t) {
          double lo, hi;
          if (COL) {
            lo = xa[t];
            hi = xa[Q - 1 - t];
          } else {
            eo_fwd<1, P>(T.BE, T.BO, t, zo, e, o, lo, hi);
          }
          t1[t * S1] = lo;
          t1[(Q - 1 - t) * S1] = hi;
          if (DIFF) {
            eo_fwd<-1, P>(T.GE, T.GO, t, zo, e, o, lo, hi);
            t1[T1M + t * S1] = lo;
            t1[T1M + (Q - 1 - t) * S1] = hi;
          }
        }
        if (Q & 1) {
          t1[QH * S1] = COL ? xa[QH] : eo_fwd_mid<1, P>(T.BE, T.BO, QH, zo, e, o);
          if (DIFF) t1[T1M + QH * S1] = eo_fwd_mid<-1, P>(T.GE, T.GO, QH, zo, e, o);
        }
      }
    }
    cta_sync();
    // (no end-of-brick barrier) the previous brick's epilogue read the lattice
    // buffer the next brick's copies target; every thread is past it here
    if (!ENDBAR && nxt.u < A.nunits)
      issue_lattice<C, NT, BX>(A, LB + ((kb + 1) & 1) * C::LAT, (long long)p * nxt.bx * BX,
                               (long long)p * nxt.by * BY, (long long)p * nxt.ez);

    double dpre[LA][2][NCD];
    if constexpr (EOPRE) {
      if (tid < NE * Q2) {
        const int el = tid / Q2, pt = tid % Q2;
        const int ex = ex0 + el % BX, ey = ey0 + el / BX;
        if (ex < A.nx && ey < A.ny) {
          const double* qde = A.qd + (ex + (long long)A.nx * (ey + (long long)A.ny * ez)) *
                                         (long long)(C::NC * Q3) + pt;
#pragma unroll
          for (int k = 0; k < LA; ++k) eo_ldpair<false, NCD, Q, DPOL>(qde, k, dpre[k], dpol);
        }
      }
    }
    // ---- S2: contract y.  item (el, qx, c), c fastest.
    FOR_ITEMS(it, NE * Q * P, NT, tid) {
      const int el = it / (Q * P), r = it % (Q * P);
      const int qx = C::QXF ? r % Q : r / P, c = C::QXF ? r / Q : r % P;
      const double* t1 = smem + el * EB + qx * S1 + c;
      double vb[P], vg[P];
#pragma unroll
      for (int b = 0; b < P; ++b) {
        vb[b] = t1[b * P];
        vg[b] = DIFF ? t1[T1M + b * P] : 0.0;
      }
      double* t2 = smem + el * EB + T1SZ + qx * TX + c * TC;
      {
        double eb[H], ob[PH], eg[H], og[PH];
        eo_split<P>(vb, eb, ob);
        if (DIFF && !COL) eo_split<P>(vg, eg, og);
        auto put = [&](int qy, double bb, double gb, double bg) {
          if (DIFF) {
            t2[qy * TY] = gb;            // G_x B_y  (-> u_x)
            t2[T2M + qy * TY] = bg;      // B_x G_y  (-> u_y)
            t2[2 * T2M + qy * TY] = bb;  // B_x B_y  (-> u_z)
          } else {
            t2[qy * TY] = bb;
          }
        };
#pragma unroll
        for (int t = 0; t < QH; ++t) {
          double bbl, bbh, gbl = 0.0, gbh = 0.0, bgl = 0.0, bgh = 0.0;
          if (COL) {
            bbl = vb[t]; bbh = vb[Q - 1 - t];
            gbl = vg[t]; gbh = vg[Q - 1 - t];
          } else {
            eo_fwd<1, P>(T.BE, T.BO, t, zo, eb, ob, bbl, bbh);
            if (DIFF) eo_fwd<1, P>(T.BE, T.BO, t, zo, eg, og, gbl, gbh);
          }
          if (DIFF) eo_fwd<-1, P>(T.GE, T.GO, t, zo, eb, ob, bgl, bgh);
          put(t, bbl, gbl, bgl);
          put(Q - 1 - t, bbh, gbh, bgh);
        }
        if (Q & 1) {
          double bb, gb = 0.0, bg = 0.0;
          if (COL) {
            bb = vb[QH]; gb = vg[QH];
          } else {
            bb = eo_fwd_mid<1, P>(T.BE, T.BO, QH, zo, eb, ob);
            if (DIFF) gb = eo_fwd_mid<1, P>(T.BE, T.BO, QH, zo, eg, og);
          }
          if (DIFF) bg = eo_fwd_mid<-1, P>(T.GE, T.GO, QH, zo, eb, ob);
          put(QH, bb, gb, bg);
        }
      }
    }
    cta_sync();

    // ---- S3: z contraction, pointwise D, z back-contraction; item (el, pt).
    //      Streamed over qz: u(qz) -> w(qz) = D u -> s += B/G(qz) w.  D(qz+1)
    //      is loaded (volatile, in program order) while qz computes.
    if (C::DSM) {
      mbar_wait(qbar, qphase);
      qphase ^= 1u;
    }
    FOR_ITEMS(it, NE * Q2, NT, tid) {
      const int el = it / Q2, pt = it % Q2;
      const int ex = ex0 + el % BX, ey = ey0 + el / BX;
      if (ex >= A.nx || ey >= A.ny) continue;
      const double* qde =
          C::DSM ? QS + el * C::QSLOT + stage_off<C>(A, ex, ey, ez) + pt
                 : A.qd + (ex + (long long)A.nx * (ey + (long long)A.ny * ez)) *
                              (long long)(C::NC * Q3) + pt;
      double* t2 = smem + el * EB + T1SZ + (pt / Q) * TY + (pt % Q) * TX;
      {
        // pairs (qz = t, Q-1-t), then the middle point (odd Q); the next pair's
        // D values are loaded while this pair computes
        double dr[LA][2][NCD];
        if (EOPRE && it_base == 0) {
#pragma unroll
          for (int k = 0; k < LA; ++k)
#pragma unroll
            for (int m = 0; m < NCD; ++m) {
              dr[k][0][m] = dpre[k][0][m];
              dr[k][1][m] = dpre[k][1][m];
            }
        } else {
#pragma unroll
          for (int k = 0; k < LA; ++k) eo_ldpair<C::DSM, NCD, Q, DPOL>(qde, k, dr[k], dpol);
        }
        if (DIFF) {
          double g0[P], g1[P], g2[P];
#pragma unroll
          for (int c = 0; c < P; ++c) {
            g0[c] = t2[c * TC];
            g1[c] = t2[T2M + c * TC];
            g2[c] = t2[2 * T2M + c * TC];
          }
          double e0[H], o0[PH], e1[H], o1[PH], e2[H], o2[PH];
          if (!COL) {
            eo_split<P>(g0, e0, o0);
            eo_split<P>(g1, e1, o1);
          }
          eo_split<P>(g2, e2, o2);
          double SE0[H], SO0[PH], SE1[H], SO1[PH], SE2[H], SO2[PH];
          zero(SE0); zero(SO0); zero(SE1); zero(SO1); zero(SE2); zero(SO2);
#pragma unroll
          for (int t = 0; t < HQ; ++t) {
            const bool mid = (Q & 1) && t == QH;
            double dl[NCD], dh[NCD];
#pragma unroll
            for (int m = 0; m < NCD; ++m) {
              dl[m] = dr[t % LA][0][m];
              dh[m] = dr[t % LA][1][m];
            }
            if (t + LA < HQ) eo_ldpair<C::DSM, NCD, Q, DPOL>(qde, t + LA, dr[t % LA], dpol);
            double u0l, u0h = 0.0, u1l, u1h = 0.0, u2l, u2h = 0.0;
            if (mid) {
              u0l = COL ? g0[t] : eo_fwd_mid<1, P>(T.BE, T.BO, t, zo, e0, o0);
              u1l = COL ? g1[t] : eo_fwd_mid<1, P>(T.BE, T.BO, t, zo, e1, o1);
              u2l = eo_fwd_mid<-1, P>(T.GE, T.GO, t, zo, e2, o2);
            } else {
              if (COL) {
                u0l = g0[t]; u0h = g0[Q - 1 - t];
                u1l = g1[t]; u1h = g1[Q - 1 - t];
              } else {
                eo_fwd<1, P>(T.BE, T.BO, t, zo, e0, o0, u0l, u0h);
                eo_fwd<1, P>(T.BE, T.BO, t, zo, e1, o1, u1l, u1h);
              }
              eo_fwd<-1, P>(T.GE, T.GO, t, zo, e2, o2, u2l, u2h);
            }
            const double w0l = dl[0] * u0l + dl[1] * u1l + dl[2] * u2l;
            const double w1l = dl[1] * u0l + dl[3] * u1l + dl[4] * u2l;
            const double w2l = dl[2] * u0l + dl[4] * u1l + dl[5] * u2l;
            if (mid) {
              if (COL) {
                t2[t * TC] = w0l;  // written after all loads of g0 (registers)
                t2[T2M + t * TC] = w1l;
              } else {
                eo_acc_mid<1, P>(T.BE, T.BO, t, zo, w0l, SE0, SO0);
                eo_acc_mid<1, P>(T.BE, T.BO, t, zo, w1l, SE1, SO1);
              }
              eo_acc_mid<-1, P>(T.GE, T.GO, t, zo, w2l, SE2, SO2);
            } else {
              const double w0h = dh[0] * u0h + dh[1] * u1h + dh[2] * u2h;
              const double w1h = dh[1] * u0h + dh[3] * u1h + dh[4] * u2h;
              const double w2h = dh[2] * u0h + dh[4] * u1h + dh[5] * u2h;
              if (COL) {
                t2[t * TC] = w0l; t2[(Q - 1 - t) * TC] = w0h;
                t2[T2M + t * TC] = w1l; t2[T2M + (Q - 1 - t) * TC] = w1h;
              } else {
                eo_acc<1, P>(T.BE, T.BO, t, zo, w0l, w0h, SE0, SO0);
                eo_acc<1, P>(T.BE, T.BO, t, zo, w1l, w1h, SE1, SO1);
              }
              eo_acc<-1, P>(T.GE, T.GO, t, zo, w2l, w2h, SE2, SO2);
            }
          }
          double s[P];
          if (!COL) {
            eo_join<P>(SE0, SO0, s);
#pragma unroll
            for (int c = 0; c < P; ++c) t2[c * TC] = s[c];
            eo_join<P>(SE1, SO1, s);
#pragma unroll
            for (int c = 0; c < P; ++c) t2[T2M + c * TC] = s[c];
          }
          eo_join<P>(SE2, SO2, s);
#pragma unroll
          for (int c = 0; c < P; ++c) t2[2 * T2M + c * TC] = s[c];
        } else {
          double g[P];
#pragma unroll
          for (int c = 0; c < P; ++c) g[c] = t2[c * TC];
          double e[H], o[PH], SE[H], SO[PH];
          eo_split<P>(g, e, o);
          zero(SE); zero(SO);
#pragma unroll
          for (int t = 0; t < HQ; ++t) {
            const bool mid = (Q & 1) && t == QH;
            double dl[1] = {dr[t % LA][0][0]}, dh[1] = {dr[t % LA][1][0]};
            if (t + LA < HQ) eo_ldpair<C::DSM, NCD, Q, DPOL>(qde, t + LA, dr[t % LA], dpol);
            if (mid) {
              const double u = eo_fwd_mid<1, P>(T.BE, T.BO, t, zo, e, o);
              eo_acc_mid<1, P>(T.BE, T.BO, t, zo, dl[0] * u, SE, SO);
            } else {
              double ul, uh;
              eo_fwd<1, P>(T.BE, T.BO, t, zo, e, o, ul, uh);
              eo_acc<1, P>(T.BE, T.BO, t, zo, dl[0] * ul, dh[0] * uh, SE, SO);
            }
          }
          double s[P];
          eo_join<P>(SE, SO, s);
#pragma unroll
          for (int c = 0; c < P; ++c) t2[c * TC] = s[c];
        }
      }
    }
    cta_sync();
    if (C::DSM) issue_qdata<C, BX, BY>(A, nxt, QS, qbar);  // D(k) consumed

    // ---- S2T: contract qy.  item (el, qx, c), c fastest.
    FOR_ITEMS(it, NE * Q * P, NT, tid) {
      const int el = it / (Q * P), r = it % (Q * P);
      const int qx = C::QXF ? r % Q : r / P, c = C::QXF ? r / Q : r % P;
      const double* t2 = smem + el * EB + T1SZ + qx * TX + c * TC;
      double* t1 = smem + el * EB + qx * S1 + c;
      {
        // rg = B_y^T v0 (x part), rb = G_y^T v1 + B_y^T v2 (y, z parts); mass: rb = B_y^T v0
        double SEg[H], SOg[PH], SEb[H], SOb[PH];
        zero(SEg); zero(SOg); zero(SEb); zero(SOb);
        double rg[P] = {}, rb[P];
        constexpr int QS = TY;
#pragma unroll
        for (int t = 0; t < (Q + 1) / 2; ++t) {
          const int th = Q - 1 - t;
          if ((Q & 1) && t == QH) {
            const double v0 = t2[t * QS];
            if (!DIFF) {
              eo_acc_mid<1, P>(T.BE, T.BO, t, zo, v0, SEb, SOb);
              continue;
            }
            const double v1 = t2[T2M + t * QS], v2 = t2[2 * T2M + t * QS];
            if (COL) {
              rg[t] = v0;
            } else {
              eo_acc_mid<1, P>(T.BE, T.BO, t, zo, v0, SEg, SOg);
              eo_acc_mid<1, P>(T.BE, T.BO, t, zo, v2, SEb, SOb);
            }
            eo_acc_mid<-1, P>(T.GE, T.GO, t, zo, v1, SEb, SOb);
            continue;
          }
          const double v0l = t2[t * QS], v0h = t2[th * QS];
          if (!DIFF) {
            eo_acc<1, P>(T.BE, T.BO, t, zo, v0l, v0h, SEb, SOb);
            continue;
          }
          const double v1l = t2[T2M + t * QS], v1h = t2[T2M + th * QS];
          const double v2l = t2[2 * T2M + t * QS], v2h = t2[2 * T2M + th * QS];
          if (COL) {
            rg[t] = v0l;
            rg[th] = v0h;
          } else {
            eo_acc<1, P>(T.BE, T.BO, t, zo, v0l, v0h, SEg, SOg);
            eo_acc<1, P>(T.BE, T.BO, t, zo, v2l, v2h, SEb, SOb);
          }
          eo_acc<-1, P>(T.GE, T.GO, t, zo, v1l, v1h, SEb, SOb);
        }
        eo_join<P>(SEb, SOb, rb);
        if (DIFF && !COL) eo_join<P>(SEg, SOg, rg);
        if (COL) {
          // collocated: the z part is B_y^T v2 = v2 (identity), added after G_y^T v1
#pragma unroll
          for (int b = 0; b < P; ++b) rb[b] += t2[2 * T2M + b * QS];
        }
#pragma unroll
        for (int b = 0; b < P; ++b) {
          t1[b * P] = rb[b];
          if (DIFF) t1[T1M + b * P] = rg[b];
        }
      }
    }
    cta_sync();

    // ---- S1T: contract qx.  item (el, b, c) -> y_e[a][b][c] (aliases T2).
    FOR_ITEMS(it, NE * P * P, NT, tid) {
      const int el = it / (P * P), r = it % (P * P);
      const double* t1 = smem + el * EB + r;
      double ye[P];
      {
        // ye = B_x^T vb + G_x^T vg (collocated: vb + G_x^T vg; mass: B_x^T vb)
        double SE[H], SO[PH];
        zero(SE); zero(SO);
#pragma unroll
        for (int t = 0; t < (Q + 1) / 2; ++t) {
          const int th = Q - 1 - t;
          if ((Q & 1) && t == QH) {
            if (!COL) eo_acc_mid<1, P>(T.BE, T.BO, t, zo, t1[t * S1], SE, SO);
            if (DIFF) eo_acc_mid<-1, P>(T.GE, T.GO, t, zo, t1[T1M + t * S1], SE, SO);
            continue;
          }
          if (!COL) eo_acc<1, P>(T.BE, T.BO, t, zo, t1[t * S1], t1[th * S1], SE, SO);
          if (DIFF) eo_acc<-1, P>(T.GE, T.GO, t, zo, t1[T1M + t * S1], t1[T1M + th * S1], SE, SO);
        }
        eo_join<P>(SE, SO, ye);
        if (COL) {
#pragma unroll
          for (int a = 0; a < P; ++a) ye[a] += t1[a * S1];
        }
      }
      double* yo = smem + el * EB + T1SZ + r;
#pragma unroll
      for (int a = 0; a < P; ++a) yo[C::SA * a] = ye[a];
    }

    if (ENDBAR) {
      cta_sync();
      simt_epilogue<C, NT, BX, BY>(A, smem, CY, cur, L, dsum);
      cp_async_wait_all();
      cta_sync();
    } else {
      // the next brick's lattice (issued after S1) lands before this barrier,
      // which also publishes y_e to the epilogue; the next brick's first
      // shared-memory writes (T1 in S1) do not touch what the epilogue reads
      cp_async_wait_all();
      cta_sync();
      simt_epilogue<C, NT, BX, BY>(A, smem, CY, cur, L, dsum);
    }
    cur = nxt;
  }
}

// Per-launch shared-memory setup: zero everything (padding included) and
// initialise the D-staging mbarrier.  (The 1D tables are kernel-parameter
// constant-bank operands, never copied to shared memory.)
template <int KIND, int P1, int Q, int BX, int BY, int NT, int MAXR, bool EO>
__device__ __forceinline__ void simt_prologue(const Tab<P1, Q>& T, unsigned long long* qbar) {
  using C = CfgS<KIND, P1, Q, BX, BY>;
  (void)T;
  extern __shared__ __align__(16) double smem[];
  if (C::DSM && threadIdx.x == 0) {
    mbar_init(qbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  FOR_ITEMS(i, C::SMEM_DOUBLES, NT, threadIdx.x) smem[i] = 0.0;
  cta_sync();
}

// The fused operator kernel: y = A x over the whole local mesh (persistent
// grid), then -- with A.infix, in a cooperative launch -- the edge-line fix-up
// behind a grid barrier; A.zero_n > 0 zeroes y in-kernel first.
template <int KIND, int P1, int Q, int BX, int BY, int NT, int MAXR, bool EO>
__global__ void __maxnreg__(MAXR)
    fused_elem_simt(const __grid_constant__ Tab<P1, Q> T, const __grid_constant__ ColArgs A) {
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) unsigned long long qbar;
  simt_prologue<KIND, P1, Q, BX, BY, NT, MAXR, EO>(T, &qbar);
  if (A.zero_n > 0) {
    // y = 0 before any brick adds into it (small problems: no separate memset)
    const long long st = (long long)gridDim.x * NT;
    for (long long i = (long long)blockIdx.x * NT + threadIdx.x; i < A.zero_n; i += st)
      A.y[i] = 0.0;
    grid_barrier(A.bar);
  }
  unsigned qphase = 0;
  double dsum = 0.0;  // this thread's share of x.y (A.dotp)
  simt_pass<KIND, P1, Q, BX, BY, NT, MAXR, EO>(T, A, &qbar, qphase, dsum);
  if (A.infix) {
    // all bricks' partials and face reductions are in memory: the edge points
    grid_barrier(A.bar);
    const long long nfx = fixup_count(A.fx);
    for (long long g = (long long)blockIdx.x * NT + threadIdx.x; g < nfx;
         g += (long long)gridDim.x * NT)
      dsum += fixup_flat(A.fx, g);
  }
  if (A.dotp) block_sum_store(dsum, A.dotp + blockIdx.x, smem);
}

// ---------------------------------------------------------------------------
// Persistent CG (§2.3: "fused ... BP
// kernels" with Cooperative Groups grid synchronisation): the WHOLE
// unpreconditioned CG solve of reading R7 in one cooperative launch.  Per
// iteration k, with rr_k known to every CTA:
//   pass:  Ap = A p (brick pipeline, y = Ap pre-zeroed), p.Ap terms  | barrier
//   fix-up of the edge-line / Dirichlet points, p.Ap terms -> parts[cta] | barrier
//   pAp = sum parts (every CTA, same fixed order); alpha = rr_k / pAp
//   r -= alpha Ap; r.r terms -> parts2[cta]                           | barrier
//   rr_{k+1} = sum parts2; beta = rr_{k+1} / rr_k
//   x += alpha p; p = r + beta p; Ap = 0 (for the next pass)           | barrier
// Every CTA computes the scalars from the same partials in the same order, so
// they agree bitwise and take the same stop decision (tolerance, breakdown) --
// no host round trip, no launch gaps.  Deterministic run to run.
// ---------------------------------------------------------------------------
// Multi-rank persistent CG (kernel-initiated communication, PAPER.md:197,
// §2.3): the interface planes of Ap go straight into the z neighbours' receive
// slots through peer pointers (the hofem_mesh_set_exchange(mode 1) buffers and
// flag protocol), and p.Ap / r.r are allreduced inside the kernel by a chain
// over the z neighbours -- up: s_r = s_{r-1} + v_r (fixed rank order), down:
// the top rank's total back to every rank -- so every rank gets bitwise the same
// scalar without leaving the kernel.
struct XArgs {
  int R, rank;
  long long plane, Nx, Ny, NzG, Klo, Khi;
  double* peer_lo;                   // lower neighbour's receive buffer (null at rank 0)
  double* peer_hi;                   // upper neighbour's receive buffer (null at the top)
  unsigned long long* pflag_lo;      // lower / upper neighbour's flags
  unsigned long long* pflag_hi;
  double* recv;                      // my receive buffer: 2 parities x [lo | hi] planes, then
                                     // [4P] = up slot, [4P+1] = down slot
  unsigned long long* my;            // my flags: [0] lo filled, [1] hi filled, [2] consumed,
                                     // [4] up value ready, [5] down value ready
  unsigned long long seq0, rseq0;    // exchanges / chain reductions done before this launch
  double* scratch;                   // my device scalar for the reduced value
  int bcmode;                        // Dirichlet rows of the summed planes: 1 y = x
};

struct CGArgs {
  long long n;           // local vector length
  long long n_owned;     // local dofs this rank owns (dot products, R8-R9)
  double* x;
  double* r;
  double* p;             // == ColArgs::x
  double* Ap;            // == ColArgs::y
  double* rr;            // rr[0] (input, r0.r0) .. rr[k] (output)
  double* parts;         // [gridDim.x] p.Ap partials
  double* parts2;        // [gridDim.x] r.r partials
  int* result;           // [0] iterations done, [1] 1 = breakdown (p.Ap <= 0),
                         // [2] exchanges, [3] chain reductions performed (multi-rank)
  int max_iter, fixed;
  double rel_tol;
  int zero_ap;           // Ap must be zero before each pass (face reductions)
  int multi;             // 1: multi-rank (X below)
  XArgs X;
};

// Fixed-order sum of gridDim.x partials; every thread of every CTA gets the same
// value.  `red` = blockDim.x doubles of shared scratch.
template <int NT>
__device__ __forceinline__ double grid_sum(const double* parts, double* red) {
  double v = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += NT) v += __ldcg(parts + i);
  __shared__ double total;
  block_sum_store(v, &total, red);
  cta_sync();
  return total;
}

// Vector phases of the persistent CG as separate (not inlined) functions: their
// 16-byte, CGU-deep load batches would otherwise raise the register pressure of
// the inlined brick pass (spills); a call per phase per iteration is free.
// Grid-stride over 16-byte pairs (vectors are 16-byte aligned, hofem.h); the
// traversal order is fixed, so the returned partial is deterministic.
constexpr int CGU = 2;

// r -= alpha Ap; returns this thread's share of r.r
static __device__ __noinline__ double cg_r_update(long long n, long long no, double alpha,
                                                  const double* Ap, double* r) {
  const long long st = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long np = n >> 1;
  const double2* A2 = reinterpret_cast<const double2*>(Ap);
  double2* r2 = reinterpret_cast<double2*>(r);
  double s = 0.0;
  for (long long i0 = t0; i0 < np; i0 += (long long)CGU * st) {
    double2 a[CGU], v[CGU];
#pragma unroll
    for (int u = 0; u < CGU; ++u) {
      const long long i = i0 + u * st;
      if (i < np) { a[u] = __ldcg(A2 + i); v[u] = r2[i]; }
    }
#pragma unroll
    for (int u = 0; u < CGU; ++u) {
      const long long i = i0 + u * st;
      if (i < np) {
        v[u].x = fma(-alpha, a[u].x, v[u].x);
        v[u].y = fma(-alpha, a[u].y, v[u].y);
        r2[i] = v[u];
        if (2 * i < no) s = fma(v[u].x, v[u].x, s);  // owned dofs only (R8-R9)
        if (2 * i + 1 < no) s = fma(v[u].y, v[u].y, s);
      }
    }
  }
  if ((n & 1) && t0 == 0) {
    const double v = fma(-alpha, __ldcg(Ap + n - 1), r[n - 1]);
    r[n - 1] = v;
    if (n - 1 < no) s = fma(v, v, s);
  }
  return s;
}

// x += alpha p; p = r + beta p; Ap = 0 (for the next pass) if zero_ap
static __device__ __noinline__ void cg_xp_update(long long n, double alpha, double beta, double* x,
                                          double* p, const double* r, double* Ap, int zero_ap) {
  const long long st = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long np = n >> 1;
  double2* x2 = reinterpret_cast<double2*>(x);
  double2* p2 = reinterpret_cast<double2*>(p);
  const double2* r2 = reinterpret_cast<const double2*>(r);
  double2* A2 = reinterpret_cast<double2*>(Ap);
  for (long long i0 = t0; i0 < np; i0 += (long long)CGU * st) {
    double2 pv[CGU], xv[CGU], rv[CGU];
#pragma unroll
    for (int u = 0; u < CGU; ++u) {
      const long long i = i0 + u * st;
      if (i < np) { pv[u] = p2[i]; xv[u] = x2[i]; rv[u] = r2[i]; }
    }
#pragma unroll
    for (int u = 0; u < CGU; ++u) {
      const long long i = i0 + u * st;
      if (i < np) {
        xv[u].x = fma(alpha, pv[u].x, xv[u].x);
        xv[u].y = fma(alpha, pv[u].y, xv[u].y);
        x2[i] = xv[u];
        rv[u].x = fma(beta, pv[u].x, rv[u].x);
        rv[u].y = fma(beta, pv[u].y, rv[u].y);
        p2[i] = rv[u];
        if (zero_ap) A2[i] = make_double2(0.0, 0.0);
      }
    }
  }
  if ((n & 1) && t0 == 0) {
    const long long i = n - 1;
    const double pv = p[i];
    x[i] = fma(alpha, pv, x[i]);
    p[i] = fma(beta, pv, r[i]);
    if (zero_ap) Ap[i] = 0.0;
  }
}

__device__ __forceinline__ unsigned long long px_ld_acq(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void px_st_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void px_spin(const unsigned long long* p, unsigned long long v) {
  const unsigned long long t0 = global_ns();
  unsigned spins = 0;
  while (px_ld_acq(p) < v) {
    if ((++spins & 1023u) == 0u && global_ns() - t0 > 20000000000ull) __trap();  // 20 s
    __nanosleep(64);
  }
}

// In-kernel interface exchange of y's boundary planes (all CTAs; mirrors
// plane_put_kernel in comm.cu, same slots, flags and sequence numbers): wait
// until the neighbours consumed this parity's previous use, put my planes into
// their slots, raise their "filled" flags, wait for mine, add the received
// planes (Dirichlet rows re-imposed, y = x), publish "consumed".
static __device__ __noinline__ void px_exchange(const XArgs& X, double* y, const double* x,
                                         unsigned long long seq, GridBar* bar) {
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  const long long P = X.plane;
  const long long par = (long long)(seq & 1ull) * 2 * P;
  if (lead) {
    if (X.peer_lo && seq > 2) px_spin(X.pflag_lo + 2, seq - 2);
    if (X.peer_hi && seq > 2) px_spin(X.pflag_hi + 2, seq - 2);
  }
  grid_barrier(bar);
  double* ylo = y;
  double* yhi = y + (X.Khi - X.Klo) * P;
  const long long st = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long i = t0; i < P; i += st) {
    if (X.peer_lo) X.peer_lo[par + P + i] = ylo[i];  // the lower rank's "hi" slot
    if (X.peer_hi) X.peer_hi[par + i] = yhi[i];      // the upper rank's "lo" slot
  }
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
  grid_barrier(bar);
  if (lead) {
    __threadfence_system();
    if (X.peer_lo) px_st_rel(X.pflag_lo + 1, seq);
    if (X.peer_hi) px_st_rel(X.pflag_hi + 0, seq);
    if (X.peer_lo) px_spin(X.my + 0, seq);
    if (X.peer_hi) px_spin(X.my + 1, seq);
  }
  grid_barrier(bar);
  const double* xlo = x;
  const double* xhi = x + (X.Khi - X.Klo) * P;
  for (long long i = t0; i < P; i += st) {
    const long long I = i % X.Nx, J = i / X.Nx;
    const bool side = I == 0 || I == X.Nx - 1 || J == 0 || J == X.Ny - 1;
    if (X.peer_lo) {
      double v = ylo[i] + __ldcv(X.recv + par + i);
      if (X.bcmode == 1 && (side || X.Klo == 0 || X.Klo == X.NzG - 1)) v = xlo[i];
      ylo[i] = v;
    }
    if (X.peer_hi) {
      double v = yhi[i] + __ldcv(X.recv + par + P + i);
      if (X.bcmode == 1 && (side || X.Khi == 0 || X.Khi == X.NzG - 1)) v = xhi[i];
      yhi[i] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
  grid_barrier(bar);
  if (lead) px_st_rel(X.my + 2, seq);  // consumed
}

// In-kernel allreduce of v (the same value in every thread of this rank) over
// the ranks: chain up (s_r = s_{r-1} + v_r), the top rank's total back down;
// the leader runs the chain, every thread returns the total after a grid barrier.
static __device__ __noinline__ double px_allreduce(const XArgs& X, double v, unsigned long long c,
                                            GridBar* bar) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const long long P = X.plane;
    double s = v;
    if (X.peer_lo) {
      px_spin(X.my + 4, c);
      s = __ldcv(X.recv + 4 * P) + v;  // lower ranks first: fixed order
    }
    double t;
    if (X.peer_hi) {
      X.peer_hi[4 * P] = s;            // the upper rank's up slot
      __threadfence_system();
      px_st_rel(X.pflag_hi + 4, c);
      px_spin(X.my + 5, c);
      t = __ldcv(X.recv + 4 * P + 1);
    } else {
      t = s;                           // the top rank holds the total
    }
    if (X.peer_lo) {
      X.peer_lo[4 * P + 1] = t;        // the lower rank's down slot
      __threadfence_system();
      px_st_rel(X.pflag_lo + 5, c);
    }
    *X.scratch = t;
    __threadfence();
  }
  grid_barrier(bar);
  return __ldcg(X.scratch);
}

template <int KIND, int P1, int Q, int BX, int BY, int NT, int MAXR, bool EO>
__global__ void __maxnreg__(MAXR)
    cg_persistent_simt(const __grid_constant__ Tab<P1, Q> T, const __grid_constant__ ColArgs A,
                       const __grid_constant__ CGArgs G) {
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) unsigned long long qbar;
  simt_prologue<KIND, P1, Q, BX, BY, NT, MAXR, EO>(T, &qbar);
  unsigned qphase = 0;
  // CG state (identical in every thread of every CTA) lives in shared memory
  // across the brick pass: registers held over simt_pass made it spill
  __shared__ double s_rr0, s_rr;
  __shared__ int s_k, s_brk, s_nx, s_nr;  // iterations, breakdown, exchanges, reductions
  {
    const long long st = (long long)gridDim.x * NT;
    const long long t0 = (long long)blockIdx.x * NT + threadIdx.x;
    if (G.zero_ap)
      for (long long i = t0; i < G.n; i += st) G.Ap[i] = 0.0;
  }
  if (threadIdx.x == 0) {
    s_rr0 = s_rr = __ldcg(G.rr);
    s_k = 0;
    s_brk = 0;
    s_nx = 0;
    s_nr = 0;
  }
  grid_barrier(A.bar);  // (also orders the shared stores for the CTA)
  for (;;) {
    if ((!G.fixed && s_rr0 == 0.0) || s_k >= G.max_iter) break;
    double dsum = 0.0;
    simt_pass<KIND, P1, Q, BX, BY, NT, MAXR, EO>(T, A, &qbar, qphase, dsum);
    grid_barrier(A.bar);
    const long long st = (long long)gridDim.x * NT;
    const long long t0 = (long long)blockIdx.x * NT + threadIdx.x;
    const long long nfx = fixup_count(A.fx);
    for (long long g = t0; g < nfx; g += st) dsum += fixup_flat(A.fx, g);
    if (G.multi) {  // Ap's interface planes: neighbours' contributions added in-kernel
      px_exchange(G.X, G.Ap, G.p, G.X.seq0 + (unsigned long long)s_nx + 1, A.bar);
      __syncthreads();
      if (threadIdx.x == 0) ++s_nx;
    }
    block_sum_store(dsum, G.parts + blockIdx.x, smem);
    grid_barrier(A.bar);
    double pAp = grid_sum<NT>(G.parts, smem);
    if (G.multi) {
      pAp = px_allreduce(G.X, pAp, G.X.rseq0 + (unsigned long long)s_nr + 1, A.bar);
      __syncthreads();
      if (threadIdx.x == 0) ++s_nr;
    }
    if (!(pAp > 0.0)) {  // same value in every CTA (and rank): all stop here
      if (threadIdx.x == 0) s_brk = 1;
      break;
    }
    const double rr = s_rr;
    const double alpha = rr / pAp;
    const double sr = cg_r_update(G.n, G.n_owned, alpha, G.Ap, G.r);
    block_sum_store(sr, G.parts2 + blockIdx.x, smem);
    grid_barrier(A.bar);
    double rn = grid_sum<NT>(G.parts2, smem);  // every thread has read s_rr
    if (G.multi) {
      rn = px_allreduce(G.X, rn, G.X.rseq0 + (unsigned long long)s_nr + 1, A.bar);
      __syncthreads();
      if (threadIdx.x == 0) ++s_nr;
    }
    const double beta = rr > 0.0 ? rn / rr : 0.0;
    cg_xp_update(G.n, alpha, beta, G.x, G.p, G.r, G.Ap, G.zero_ap);
    const int k = s_k + 1;
    const bool stop = !G.fixed && (rn == 0.0 || sqrt(rn) <= G.rel_tol * sqrt(s_rr0));
    cta_sync();  // every thread has read s_k / s_rr0 of this iteration
    if (threadIdx.x == 0) {
      s_rr = rn;
      s_k = k;
      if (blockIdx.x == 0) G.rr[k] = rn;
    }
    if (stop) break;
    grid_barrier(A.bar);
  }
  cta_sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    G.result[0] = s_k;
    G.result[1] = s_brk;
    G.result[2] = s_nx;
    G.result[3] = s_nr;
  }
}

// SIMT kernel shapes: brick BX x BY elements, NT threads (>= the stage-3 item
// count NE*Q^2 for Gauss Q where possible, so every stage is one round),
// register cap, CTAs per SM.
template <int P1>
struct ShapeSD;
//                                     BX BY  NT  MAXR  CTAs/SM
template <> struct ShapeSD<2> { static constexpr int BX = 4, BY = 4, NT = 160, MAXR = 96, CPS = 4; };
template <> struct ShapeSD<3> { static constexpr int BX = 4, BY = 2, NT = 128, MAXR = 128, CPS = 4; };
template <> struct ShapeSD<4> { static constexpr int BX = 3, BY = 2, NT = 160, MAXR = 102, CPS = 4; };
template <> struct ShapeSD<5> { static constexpr int BX = 3, BY = 1, NT = 128, MAXR = 102, CPS = 5; };
// P1 = 6: 1x3 bricks with 160 threads (S1 / S2 / S3 fill 108 / 126 / 147 of them,
// epilogue 96 rows; 3 CTAs/SM at 128 registers) beat round 2's 1x2 / 128 threads
// (72 / 84 / 98 items: the fourth warp idled in most stages): BP3 p=5 brick kernel
// 4.94 -> 4.70 ms on the config-5 slab, 1.015 -> 0.979 ms at 60^3, 1.120 -> 1.110 ms
// at 62^3 (profiles/ab/r2v_ab_shapes2.txt); BP1 p=5 (~1M dofs) 45.5 -> 43.5 us
// (r2v_ab_p6x3.txt, which also re-checked DLA, T2QX, PRE, ENDBAR on this shape)
template <> struct ShapeSD<6> { static constexpr int BX = 1, BY = 3, NT = 160, MAXR = 128, CPS = 3; };
template <> struct ShapeSD<7> { static constexpr int BX = 1, BY = 1, NT = 64, MAXR = 168, CPS = 6; };
template <> struct ShapeSD<8> { static constexpr int BX = 1, BY = 1, NT = 96, MAXR = 168, CPS = 4; };
template <> struct ShapeSD<9> { static constexpr int BX = 1, BY = 1, NT = 128, MAXR = 232, CPS = 2; };

// Tuning override (scripts/build_variant.py): -DHOFEM_SS_P1=6 -DHOFEM_SS_BX=2
// -DHOFEM_SS_BY=2 -DHOFEM_SS_NT=224 -DHOFEM_SS_MAXR=144 -DHOFEM_SS_CPS=2.
#ifdef HOFEM_SS_P1
struct ShapeSOverride {
  static constexpr int BX = HOFEM_SS_BX, BY = HOFEM_SS_BY, NT = HOFEM_SS_NT,
                       MAXR = HOFEM_SS_MAXR, CPS = HOFEM_SS_CPS;
};
template <int P1>
struct ShapeS : std::conditional_t<P1 == HOFEM_SS_P1, ShapeSOverride, ShapeSD<P1>> {};
#else
template <int P1>
struct ShapeS : ShapeSD<P1> {};
#endif

// Collocated (BP5) SIMT shapes: every stage has NE*P1^2 items.
template <int P1>
struct ShapeSCD : ShapeS<P1> {};
//                                      BX BY  NT  MAXR  CTAs/SM  (measured, BP5)
// collocated (BP5) shapes, measured (gpurun_out/e10)
template <> struct ShapeSCD<4> { static constexpr int BX = 2, BY = 2, NT = 128, MAXR = 144, CPS = 3; };
template <> struct ShapeSCD<5> { static constexpr int BX = 3, BY = 2, NT = 160, MAXR = 102, CPS = 4; };
template <> struct ShapeSCD<6> { static constexpr int BX = 2, BY = 2, NT = 160, MAXR = 128, CPS = 3; };
template <> struct ShapeSCD<7> { static constexpr int BX = 2, BY = 1, NT = 128, MAXR = 128, CPS = 4; };
template <> struct ShapeSCD<8> { static constexpr int BX = 2, BY = 1, NT = 128, MAXR = 128, CPS = 4; };
template <> struct ShapeSCD<9> { static constexpr int BX = 1, BY = 1, NT = 96, MAXR = 128, CPS = 5; };
// Tuning override: -DHOFEM_SC_P1=6 -DHOFEM_SC_BX=.. (same fields as HOFEM_SS_*).
#ifdef HOFEM_SC_P1
struct ShapeSCOverride {
  static constexpr int BX = HOFEM_SC_BX, BY = HOFEM_SC_BY, NT = HOFEM_SC_NT,
                       MAXR = HOFEM_SC_MAXR, CPS = HOFEM_SC_CPS;
};
template <int P1>
struct ShapeSC : std::conditional_t<P1 == HOFEM_SC_P1, ShapeSCOverride, ShapeSCD<P1>> {};
#else
template <int P1>
struct ShapeSC : ShapeSCD<P1> {};
#endif
// mass (BP1) shapes: the diffusion ones unless measured otherwise
template <int P1>
struct ShapeSMD : ShapeS<P1> {};
// measured (BP1 at ~1M dofs, whole apply incl. memset and fix-up; gpurun_out/e12,
// f5): single-element bricks pay off at p = 8 only (more edge lines elsewhere)
// register caps (r2v, profiles/ab/r2v_ab_massregs.txt, BP1 ~1M dofs): the mass kernels fit
// in 64-80 registers without spills; a lower cap (more CTAs per SM) pays at P1 = 2 (64: -7 %),
// 5 (80: -9 %), 6 (80: -6.5 %), 9 (64: -2 %) and loses elsewhere (the inherited caps stay)
template <> struct ShapeSMD<2> { static constexpr int BX = 4, BY = 4, NT = 160, MAXR = 64, CPS = 6; };
template <> struct ShapeSMD<5> { static constexpr int BX = 2, BY = 2, NT = 160, MAXR = 80, CPS = 5; };
template <> struct ShapeSMD<6> { static constexpr int BX = 1, BY = 3, NT = 160, MAXR = 80, CPS = 5; };
template <> struct ShapeSMD<9> { static constexpr int BX = 1, BY = 1, NT = 128, MAXR = 64, CPS = 8; };
#ifdef HOFEM_SM_P1
struct ShapeSMOverride {
  static constexpr int BX = HOFEM_SM_BX, BY = HOFEM_SM_BY, NT = HOFEM_SM_NT,
                       MAXR = HOFEM_SM_MAXR, CPS = HOFEM_SM_CPS;
};
template <int P1>
struct ShapeSM : std::conditional_t<P1 == HOFEM_SM_P1, ShapeSMOverride, ShapeSMD<P1>> {};
#else
template <int P1>
struct ShapeSM : ShapeSMD<P1> {};
#endif
template <int KIND, int P1>
using ShapeSK = std::conditional_t<KIND == KIND_COLLOC, ShapeSC<P1>,
                                   std::conditional_t<KIND == KIND_MASS, ShapeSM<P1>, ShapeS<P1>>>;

struct FusedLaunch {
  int BX, BY, face_block, ctas_per_sm;  // face_block = FaceLayout<>::FB
  int ctas_per_sm_cg;                   // the persistent CG kernel (own register cap)
};

// Register cap of the persistent CG kernel.  Measured (gpurun_out/r2e vs r2c):
// 32 more registers than the apply kernel remove most spills but cost resident
// CTAs and are slower overall; the apply kernel's cap is kept.
constexpr int cg_maxr(int maxr) { return maxr; }

// Defined per P1 in fused_p.cu: kind in {KIND_MASS, KIND_DIFF, KIND_COLLOC},
// Q in {P1, P1+1} for MASS/DIFF and Q == P1 for COLLOC.  Return false if the
// combination is not instantiated.  cooperative: launch with
// cudaLaunchAttributeCooperative (all CTAs co-resident or the launch fails).
template <int P1>
bool fused_launch(int kind, int Q, const double* B, const double* G, const ColArgs& A, int grid,
                  bool cooperative, cudaStream_t s, cudaError_t* err);
template <int P1>
bool cg_launch(int kind, int Q, const double* B, const double* G, const ColArgs& A,
               const CGArgs& CG, int grid, cudaStream_t s, cudaError_t* err);
template <int P1>
FusedLaunch fused_shape(int kind, int Q);

}  // namespace hofem
