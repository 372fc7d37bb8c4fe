// fused_impl.cuh -- the fused sm_100a operator kernels (SURVEY.md §8(a) rows
// a4-a9; north star "one fused sm_100a kernel per operator").
//
// One CTA owns a brick of BX*BY*BZ elements and does, for all of them:
//   a4  gather R: the brick's (p*BX+1)(p*BY+1)(p*BZ+1) lattice of x is read once
//       from HBM (rows coalesced along x) into shared memory, Dirichlet dofs
//       zeroed (reading R6);
//   a5  B: the 1D B1d/G1d contractions dimension by dimension (x, then y in
//       shared memory; z in registers, one thread per (qx,qy) quadrature column);
//   a6  D: the pointwise qdata (streamed from HBM, coalesced, L2 evict-first);
//   a7  B^T: the transposed contractions (z in registers, then y, x in smem);
//   a8  R^T: a deterministic in-brick sum -- every brick lattice point sums its
//       1..8 element contributions in ascending element order.  Points strictly
//       inside the brick (and on the domain boundary) are written to y directly;
//       points on an interior brick face go to a per-brick partial buffer that
//       fixup_kernel (fused.cu) sums in ascending brick order.
//   a9  y[ess] = x[ess].
// The 1D tables live in the kernel-parameter constant bank (every index is a
// compile-time constant after unrolling, so DFMA takes them as uniform-register
// operands: no shared-memory traffic for B/G).
//
// Shared-memory layouts are chosen so that consecutive lanes touch consecutive
// or odd-strided doubles (conflict-free 64-bit accesses): see DESIGN.md §4.
#pragma once

#include "internal.h"

namespace hofem {

template <int P1, int Q>
struct Tab {
  double B[Q * P1];
  double G[Q * P1];
};

struct FusedArgs {
  const double* x;
  double* y;
  const double* qd;
  double* bbuf;
  int nx, ny, nzl;       // local element counts
  int nbx, nby, nbz;     // bricks per axis
  long long Nx, Ny, Nzl; // local lattice sizes
  long long K0, NzG;     // global index of local plane 0; global plane count
  int bc;
};

enum { KIND_MASS = 0, KIND_DIFF = 1, KIND_COLLOC = 2 };

__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile(
      "{ .reg .b64 pol; createpolicy.fractional.L2::evict_first.b64 pol, 1.0;"
      " ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], pol; }"
      : "=d"(v)
      : "l"(p));
  return v;
}

__device__ __forceinline__ bool ess_point(const FusedArgs& A, long long I, long long J,
                                          long long K) {
  long long Kg = K + A.K0;
  return I == 0 || I == A.Nx - 1 || J == 0 || J == A.Ny - 1 || Kg == 0 || Kg == A.NzG - 1;
}

template <int KIND, int P1, int Q, int BX, int BY, int BZ>
struct Cfg {
  static constexpr int p = P1 - 1;
  static constexpr int NE = BX * BY * BZ;
  static constexpr int LX = p * BX + 1, LY = p * BY + 1, LZ = p * BZ + 1;
  static constexpr int BLAT = LX * LY * LZ;                 // dense brick lattice
  static constexpr int PS = ((LX * LY) % 2 == 0) ? LX * LY + 1 : LX * LY;  // odd plane stride
  static constexpr int LAT = PS * LZ;
  static constexpr int Qp = (Q % 2 == 0) ? Q + 1 : Q;        // odd c-stride in T1
  static constexpr int S2 = Qp * P1;                         // b-stride in T1
  static constexpr int NT1 = (KIND == KIND_MASS) ? 1 : 2;
  static constexpr int NT2 = (KIND == KIND_MASS) ? 1 : 3;
  static constexpr int T1N = NT1 * S2 * P1;
  static constexpr int QQP = Q * Q * P1;
  static constexpr int T2N = NT2 * QQP;
  static constexpr int SA = ((P1 * P1) % 2 == 0) ? P1 * P1 + 1 : P1 * P1;  // a-stride of y_e
  static constexpr int YEN = (KIND == KIND_COLLOC) ? P1 * P1 * P1 : SA * P1;
  static constexpr int WN = 3 * P1 * P1 * P1;                // collocated: w per element
  static constexpr int cmax(int a, int b) { return a > b ? a : b; }
  static constexpr int REGA =
      (KIND == KIND_COLLOC) ? cmax(LAT, NE * YEN) : cmax(LAT, cmax(NE * T2N, NE * YEN));
  static constexpr int REGB = (KIND == KIND_COLLOC) ? NE * WN : NE * T1N;
  static constexpr int SMEM_BYTES = (REGA + REGB) * 8;
  static constexpr int NC = (KIND == KIND_MASS) ? 1 : 6;
};

// ---------------------------------------------------------------------------
// Shared prologue / epilogue.
// ---------------------------------------------------------------------------
template <class C, int NT>
__device__ __forceinline__ void load_brick_lattice(const FusedArgs& A, double* RA,
                                                   long long I0, long long J0, long long K0l) {
  for (int t = threadIdx.x; t < C::BLAT; t += NT) {
    int i = t % C::LX, j = (t / C::LX) % C::LY, k = t / (C::LX * C::LY);
    long long I = I0 + i, J = J0 + j, K = K0l + k;
    double v = 0.0;
    if (I < A.Nx && J < A.Ny && K < A.Nzl) {
      v = A.x[I + A.Nx * (J + A.Ny * K)];
      if (A.bc && ess_point(A, I, J, K)) v = 0.0;
    }
    RA[i + C::LX * j + C::PS * k] = v;
  }
}

// Contributing local elements along one brick axis for brick-lattice index i.
template <int p, int BN>
__device__ __forceinline__ int local_elems(int i, int e0, int n, int* el, int* a) {
  int q = i / p, r = i - q * p, k = 0;
  if (r == 0 && q > 0 && e0 + q - 1 < n) { el[k] = q - 1; a[k] = p; ++k; }
  if (q < BN && e0 + q < n) { el[k] = q; a[k] = r; ++k; }
  return k;
}

// a8 + a9: in-brick deterministic sum; direct write or partial buffer.
template <class C, int NT, int BX, int BY, int BZ, bool NATURAL>
__device__ __forceinline__ void brick_sum_store(const FusedArgs& A, const double* RA, int brick,
                                                int ex0, int ey0, int ez0, long long I0,
                                                long long J0, long long K0l) {
  constexpr int p = C::p, P1 = p + 1;
  for (int t = threadIdx.x; t < C::BLAT; t += NT) {
    int i = t % C::LX, j = (t / C::LX) % C::LY, k = t / (C::LX * C::LY);
    long long I = I0 + i, J = J0 + j, K = K0l + k;
    if (I >= A.Nx || J >= A.Ny || K >= A.Nzl) continue;
    int exl[2], ax[2], eyl[2], ay[2], ezl[2], az[2];
    int nxl = local_elems<p, BX>(i, ex0, A.nx, exl, ax);
    int nyl = local_elems<p, BY>(j, ey0, A.ny, eyl, ay);
    int nzl = local_elems<p, BZ>(k, ez0, A.nzl, ezl, az);
    double s = 0.0;
    for (int c = 0; c < nzl; ++c)
      for (int b = 0; b < nyl; ++b)
        for (int a = 0; a < nxl; ++a) {
          int el = exl[a] + BX * (eyl[b] + BY * ezl[c]);
          int off = NATURAL ? ax[a] + P1 * (ay[b] + P1 * az[c])
                            : az[c] + P1 * ay[b] + C::SA * ax[a];
          s += RA[el * C::YEN + off];
        }
    bool shared = (i == 0 && I > 0) || (i == C::LX - 1 && I < A.Nx - 1) ||
                  (j == 0 && J > 0) || (j == C::LY - 1 && J < A.Ny - 1) ||
                  (k == 0 && K > 0) || (k == C::LZ - 1 && K < A.Nzl - 1);
    long long l = I + A.Nx * (J + A.Ny * K);
    if (shared) {
      A.bbuf[(long long)brick * C::BLAT + t] = s;
    } else {
      if (A.bc && ess_point(A, I, J, K)) s = A.x[l];
      A.y[l] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// General kernel: mass (BP1) and diffusion (BP3) with any (P1, Q) tables.
// ---------------------------------------------------------------------------
template <int KIND, int P1, int Q, int BX, int BY, int BZ, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) fused_brick(const Tab<P1, Q> T, FusedArgs A) {
  using C = Cfg<KIND, P1, Q, BX, BY, BZ>;
  constexpr int p = P1 - 1, NE = C::NE, Qp = C::Qp, S2 = C::S2, QQP = C::QQP;
  constexpr bool DIFF = KIND == KIND_DIFF;
  extern __shared__ double smem[];
  double* RA = smem;
  double* RB = smem + C::REGA;
  const int tid = threadIdx.x;
  const int brick = blockIdx.x;
  const int ex0 = (brick % A.nbx) * BX;
  const int ey0 = ((brick / A.nbx) % A.nby) * BY;
  const int ez0 = (brick / (A.nbx * A.nby)) * BZ;
  const long long I0 = (long long)p * ex0, J0 = (long long)p * ey0, K0l = (long long)p * ez0;

  load_brick_lattice<C, NT>(A, RA, I0, J0, K0l);
  __syncthreads();

  // ---- stage 1: contract x.  item (el, b, c), c fastest.
  for (int it = tid; it < NE * P1 * P1; it += NT) {
    const int el = it / (P1 * P1), r = it % (P1 * P1), c = r % P1, b = r / P1;
    const int exl = el % BX, eyl = (el / BX) % BY, ezl = el / (BX * BY);
    const double* xl = RA + p * exl + C::LX * (p * eyl + b) + C::PS * (p * ezl + c);
    double xa[P1];
#pragma unroll
    for (int a = 0; a < P1; ++a) xa[a] = xl[a];
    double* t1 = RB + el * C::T1N + Qp * c + S2 * b;
#pragma unroll
    for (int qx = 0; qx < Q; ++qx) {
      double sb = 0.0, sg = 0.0;
#pragma unroll
      for (int a = 0; a < P1; ++a) {
        sb = fma(T.B[qx * P1 + a], xa[a], sb);
        if (DIFF) sg = fma(T.G[qx * P1 + a], xa[a], sg);
      }
      t1[qx] = sb;                       // B_x x
      if (DIFF) t1[S2 * P1 + qx] = sg;   // G_x x
    }
  }
  __syncthreads();

  // ---- stage 2: contract y.  item (el, qx, c), qx fastest.
  for (int it = tid; it < NE * Q * P1; it += NT) {
    const int el = it / (Q * P1), r = it % (Q * P1), qx = r % Q, c = r / Q;
    const double* t1 = RB + el * C::T1N + qx + Qp * c;
    double vb[P1], vg[P1];
#pragma unroll
    for (int b = 0; b < P1; ++b) {
      vb[b] = t1[S2 * b];
      if (DIFF) vg[b] = t1[S2 * P1 + S2 * b];
    }
    double* t2 = RA + el * C::T2N + qx + Q * Q * c;
#pragma unroll
    for (int qy = 0; qy < Q; ++qy) {
      double bb = 0.0, gb = 0.0, bg = 0.0;
#pragma unroll
      for (int b = 0; b < P1; ++b) {
        bb = fma(T.B[qy * P1 + b], vb[b], bb);
        if (DIFF) {
          gb = fma(T.B[qy * P1 + b], vg[b], gb);
          bg = fma(T.G[qy * P1 + b], vb[b], bg);
        }
      }
      if (DIFF) {
        t2[Q * qy] = gb;            // G_x B_y
        t2[QQP + Q * qy] = bg;      // B_x G_y
        t2[2 * QQP + Q * qy] = bb;  // B_x B_y
      } else {
        t2[Q * qy] = bb;
      }
    }
  }
  __syncthreads();

  // ---- stage 3: contract z in registers, pointwise D, z-transpose.
  //      item (el, qx, qy), qx fastest: qdata reads are coalesced.
  for (int it = tid; it < NE * Q * Q; it += NT) {
    const int el = it / (Q * Q), i3 = it % (Q * Q);
    const int exl = el % BX, eyl = (el / BX) % BY, ezl = el / (BX * BY);
    const int ex = ex0 + exl, ey = ey0 + eyl, ez = ez0 + ezl;
    if (ex >= A.nx || ey >= A.ny || ez >= A.nzl) continue;
    const long long e = ex + (long long)A.nx * (ey + (long long)A.ny * ez);
    const double* qd = A.qd + e * (C::NC * Q * Q * Q) + i3;
    double* t2 = RA + el * C::T2N + i3;
    if (DIFF) {
      double g0[P1], g1[P1], g2[P1], s0[P1], s1[P1], s2[P1];
#pragma unroll
      for (int c = 0; c < P1; ++c) {
        g0[c] = t2[Q * Q * c];
        g1[c] = t2[QQP + Q * Q * c];
        g2[c] = t2[2 * QQP + Q * Q * c];
        s0[c] = s1[c] = s2[c] = 0.0;
      }
#pragma unroll
      for (int qz = 0; qz < Q; ++qz) {
        const double* d = qd + qz * Q * Q;
        const double d00 = ld_stream(d), d01 = ld_stream(d + Q * Q * Q),
                     d02 = ld_stream(d + 2 * Q * Q * Q), d11 = ld_stream(d + 3 * Q * Q * Q),
                     d12 = ld_stream(d + 4 * Q * Q * Q), d22 = ld_stream(d + 5 * Q * Q * Q);
        double u0 = 0.0, u1 = 0.0, u2 = 0.0;
#pragma unroll
        for (int c = 0; c < P1; ++c) {
          u0 = fma(T.B[qz * P1 + c], g0[c], u0);
          u1 = fma(T.B[qz * P1 + c], g1[c], u1);
          u2 = fma(T.G[qz * P1 + c], g2[c], u2);
        }
        const double w0 = d00 * u0 + d01 * u1 + d02 * u2;
        const double w1 = d01 * u0 + d11 * u1 + d12 * u2;
        const double w2 = d02 * u0 + d12 * u1 + d22 * u2;
#pragma unroll
        for (int c = 0; c < P1; ++c) {
          s0[c] = fma(T.B[qz * P1 + c], w0, s0[c]);
          s1[c] = fma(T.B[qz * P1 + c], w1, s1[c]);
          s2[c] = fma(T.G[qz * P1 + c], w2, s2[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < P1; ++c) {
        t2[Q * Q * c] = s0[c];
        t2[QQP + Q * Q * c] = s1[c];
        t2[2 * QQP + Q * Q * c] = s2[c];
      }
    } else {
      double g[P1], s[P1];
#pragma unroll
      for (int c = 0; c < P1; ++c) { g[c] = t2[Q * Q * c]; s[c] = 0.0; }
#pragma unroll
      for (int qz = 0; qz < Q; ++qz) {
        const double d = ld_stream(qd + qz * Q * Q);
        double u = 0.0;
#pragma unroll
        for (int c = 0; c < P1; ++c) u = fma(T.B[qz * P1 + c], g[c], u);
        const double v = d * u;
#pragma unroll
        for (int c = 0; c < P1; ++c) s[c] = fma(T.B[qz * P1 + c], v, s[c]);
      }
#pragma unroll
      for (int c = 0; c < P1; ++c) t2[Q * Q * c] = s[c];
    }
  }
  __syncthreads();

  // ---- stage 2^T: contract qy.  item (el, qx, c), qx fastest.
  for (int it = tid; it < NE * Q * P1; it += NT) {
    const int el = it / (Q * P1), r = it % (Q * P1), qx = r % Q, c = r / Q;
    const double* t2 = RA + el * C::T2N + qx + Q * Q * c;
    double* t1 = RB + el * C::T1N + qx + Qp * c;
    if (DIFF) {
      double v0[Q], v1[Q], v2[Q];
#pragma unroll
      for (int qy = 0; qy < Q; ++qy) {
        v0[qy] = t2[Q * qy];
        v1[qy] = t2[QQP + Q * qy];
        v2[qy] = t2[2 * QQP + Q * qy];
      }
#pragma unroll
      for (int b = 0; b < P1; ++b) {
        double rg = 0.0, rb = 0.0;
#pragma unroll
        for (int qy = 0; qy < Q; ++qy) {
          rg = fma(T.B[qy * P1 + b], v0[qy], rg);
          rb = fma(T.G[qy * P1 + b], v1[qy], rb);
          rb = fma(T.B[qy * P1 + b], v2[qy], rb);
        }
        t1[S2 * b] = rg;            // -> G_x^T
        t1[S2 * P1 + S2 * b] = rb;  // -> B_x^T
      }
    } else {
      double v[Q];
#pragma unroll
      for (int qy = 0; qy < Q; ++qy) v[qy] = t2[Q * qy];
#pragma unroll
      for (int b = 0; b < P1; ++b) {
        double rb = 0.0;
#pragma unroll
        for (int qy = 0; qy < Q; ++qy) rb = fma(T.B[qy * P1 + b], v[qy], rb);
        t1[S2 * b] = rb;
      }
    }
  }
  __syncthreads();

  // ---- stage 1^T: contract qx.  item (el, b, c), c fastest -> y_e[a][b][c].
  for (int it = tid; it < NE * P1 * P1; it += NT) {
    const int el = it / (P1 * P1), r = it % (P1 * P1), c = r % P1, b = r / P1;
    const double* t1 = RB + el * C::T1N + Qp * c + S2 * b;
    double rg[Q], rb[Q];
#pragma unroll
    for (int qx = 0; qx < Q; ++qx) {
      if (DIFF) {
        rg[qx] = t1[qx];
        rb[qx] = t1[S2 * P1 + qx];
      } else {
        rb[qx] = t1[qx];
      }
    }
    double* ye = RA + el * C::YEN + c + P1 * b;
#pragma unroll
    for (int a = 0; a < P1; ++a) {
      double s = 0.0;
#pragma unroll
      for (int qx = 0; qx < Q; ++qx) {
        s = fma(T.B[qx * P1 + a], rb[qx], s);
        if (DIFF) s = fma(T.G[qx * P1 + a], rg[qx], s);
      }
      ye[C::SA * a] = s;
    }
  }
  __syncthreads();

  brick_sum_store<C, NT, BX, BY, BZ, false>(A, RA, brick, ex0, ey0, ez0, I0, J0, K0l);
}

// ---------------------------------------------------------------------------
// Collocated diffusion kernel (BP5: GLL points = nodes, B1d = I, Q = P1).
// u_x = G_x x, u_y = G_y x, u_z = G_z x; w = D u; y = G_x^T w_x + G_y^T w_y + G_z^T w_z.
// ---------------------------------------------------------------------------
template <int P1, int BX, int BY, int BZ, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) fused_brick_colloc(const Tab<P1, P1> T, FusedArgs A) {
  using C = Cfg<KIND_COLLOC, P1, P1, BX, BY, BZ>;
  constexpr int p = P1 - 1, NE = C::NE, N2 = P1 * P1, N3 = P1 * P1 * P1;
  extern __shared__ double smem[];
  double* RA = smem;
  double* RB = smem + C::REGA;
  const int tid = threadIdx.x;
  const int brick = blockIdx.x;
  const int ex0 = (brick % A.nbx) * BX;
  const int ey0 = ((brick / A.nbx) % A.nby) * BY;
  const int ez0 = (brick / (A.nbx * A.nby)) * BZ;
  const long long I0 = (long long)p * ex0, J0 = (long long)p * ey0, K0l = (long long)p * ez0;

  load_brick_lattice<C, NT>(A, RA, I0, J0, K0l);
  __syncthreads();

  // ---- forward: item (el, i, j), i fastest; z-column k in registers.
  for (int it = tid; it < NE * N2; it += NT) {
    const int el = it / N2, item = it % N2, i = item % P1, j = item / P1;
    const int exl = el % BX, eyl = (el / BX) % BY, ezl = el / (BX * BY);
    const int ex = ex0 + exl, ey = ey0 + eyl, ez = ez0 + ezl;
    if (ex >= A.nx || ey >= A.ny || ez >= A.nzl) continue;
    const long long e = ex + (long long)A.nx * (ey + (long long)A.ny * ez);
    const double* qd = A.qd + e * (6 * N3) + item;
    const double* xl = RA + p * exl + C::LX * (p * eyl) + C::PS * (p * ezl);
    double Gi[P1], Gj[P1], xz[P1];
#pragma unroll
    for (int a = 0; a < P1; ++a) {
      Gi[a] = T.G[i * P1 + a];
      Gj[a] = T.G[j * P1 + a];
      xz[a] = xl[i + C::LX * j + C::PS * a];
    }
    double* w = RB + el * C::WN + item;
#pragma unroll
    for (int k = 0; k < P1; ++k) {
      double ux = 0.0, uy = 0.0, uz = 0.0;
#pragma unroll
      for (int a = 0; a < P1; ++a) {
        ux = fma(Gi[a], xl[a + C::LX * j + C::PS * k], ux);
        uy = fma(Gj[a], xl[i + C::LX * a + C::PS * k], uy);
        uz = fma(T.G[k * P1 + a], xz[a], uz);
      }
      const double* d = qd + k * N2;
      const double d00 = ld_stream(d), d01 = ld_stream(d + N3), d02 = ld_stream(d + 2 * N3),
                   d11 = ld_stream(d + 3 * N3), d12 = ld_stream(d + 4 * N3),
                   d22 = ld_stream(d + 5 * N3);
      w[N2 * k] = d00 * ux + d01 * uy + d02 * uz;
      w[N3 + N2 * k] = d01 * ux + d11 * uy + d12 * uz;
      w[2 * N3 + N2 * k] = d02 * ux + d12 * uy + d22 * uz;
    }
  }
  __syncthreads();

  // ---- transpose: item (el, a, b) -> y_e[a + P1 b + P1^2 c] for all c.
  for (int it = tid; it < NE * N2; it += NT) {
    const int el = it / N2, item = it % N2, a = item % P1, b = item / P1;
    const double* w = RB + el * C::WN;
    double Ga[P1], Gb[P1], wz[P1];
#pragma unroll
    for (int k = 0; k < P1; ++k) {
      Ga[k] = T.G[k * P1 + a];
      Gb[k] = T.G[k * P1 + b];
      wz[k] = w[2 * N3 + item + N2 * k];
    }
    double* ye = RA + el * C::YEN + item;
#pragma unroll
    for (int c = 0; c < P1; ++c) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < P1; ++k) {
        s = fma(Ga[k], w[k + P1 * b + N2 * c], s);          // G_x^T w_x
        s = fma(Gb[k], w[N3 + a + P1 * k + N2 * c], s);      // G_y^T w_y
        s = fma(T.G[k * P1 + c], wz[k], s);                  // G_z^T w_z
      }
      ye[N2 * c] = s;
    }
  }
  __syncthreads();

  brick_sum_store<C, NT, BX, BY, BZ, true>(A, RA, brick, ex0, ey0, ez0, I0, J0, K0l);
}

// ---------------------------------------------------------------------------
// Per-P1 launch configurations (brick shape, threads per CTA, min CTAs/SM).
// ---------------------------------------------------------------------------
template <int P1>
struct Shape;
//                                   BX BY BZ  NT  MINB
template <> struct Shape<2> { static constexpr int BX = 8, BY = 4, BZ = 4, NT = 384, MINB = 1; };
template <> struct Shape<3> { static constexpr int BX = 4, BY = 4, BZ = 2, NT = 512, MINB = 1; };
template <> struct Shape<4> { static constexpr int BX = 4, BY = 2, BZ = 2, NT = 416, MINB = 1; };
template <> struct Shape<5> { static constexpr int BX = 2, BY = 2, BZ = 2, NT = 288, MINB = 1; };
template <> struct Shape<6> { static constexpr int BX = 2, BY = 2, BZ = 2, NT = 416, MINB = 1; };
template <> struct Shape<7> { static constexpr int BX = 2, BY = 2, BZ = 1, NT = 256, MINB = 1; };
template <> struct Shape<8> { static constexpr int BX = 2, BY = 2, BZ = 1, NT = 352, MINB = 1; };
template <> struct Shape<9> { static constexpr int BX = 2, BY = 1, BZ = 1, NT = 224, MINB = 1; };

struct FusedLaunch {
  int BX, BY, BZ, blat;
};

// Defined per P1 in fused_p*.cu: kind in {KIND_MASS, KIND_DIFF, KIND_COLLOC},
// Q in {P1, P1+1} for MASS/DIFF and Q == P1 for COLLOC.  Returns false if the
// combination is not instantiated.
template <int P1>
bool fused_launch(int kind, int Q, const double* B, const double* G, const FusedArgs& A,
                  int nbricks, cudaStream_t s, cudaError_t* err);
template <int P1>
FusedLaunch fused_shape(int kind);

}  // namespace hofem
