// dg_impl.cuh -- matrix-free DG (L2) mass operator, SURVEY.md §8(f) f4
// (§2.4.1 "matrix-free discontinuous Galerkin"; fig:dgpa-perf
// "DG mass operators").
//
// Space: discontinuous Q_p per element, nodal basis at the p+1 Gauss-Legendre
// points (reading R16); vectors are element-major E-vectors [E][P1^3] (x fastest
// inside an element).  The operator is block diagonal: y_e = B^T D_e B x_e with
// D_e = W detJ at the Q^3 Gauss points (the BP1 qdata) and B the 1D basis table
// applied dimension by dimension -- no gather, no scatter, no fix-up.
//
// Persistent kernel, one CTA per (SM x occupancy), batches of NE elements.
// x and y stay in their natural element-contiguous layout end to end:
//   - x and D of the NEXT batch arrive by two bulk copies (cp.async.bulk, the
//     TMA engine) into a double-buffered stage, completing on one mbarrier;
//   - the five thread-per-line stages contract z first (lines along the slowest
//     index, so lanes run over contiguous (a, b) and read the dense x without
//     bank conflicts), then y, then x with the pointwise D, and back (x^T, y^T,
//     z^T) -- even-odd contractions, tables from the kernel-parameter constant
//     bank, padded strides from a bank-conflict search (dg_layout below);
//   - z^T writes y densely into the batch's x stage, which ONE bulk store
//     (cp.async.bulk global <- shared) sends to HBM.
// No per-dof index arithmetic is left outside the contraction stages.
// Bound: HBM (16 + 8 Q^3/P1^3 B/DOF; flop/B < 3.1 even at p = 8).
#pragma once

#include "fused_impl.cuh"

namespace hofem {

struct DGArgs {
  const double* x;
  double* y;
  const double* qd;  // [E][Q^3] W*detJ (allocated with 2 doubles of slack)
  long long E;       // local elements
  long long nbatch;  // ceil(E / NE)
};

// Work-area strides per element: T1 [qz][b][a] (qz stride R1), T2 [qz][qy][a]
// (qz stride R2, qy stride PP), element block EB = Q R1 + Q R2 + PAD.
template <int P1, int NE>
struct LayoutDG {  // generic fallback (odd row strides)
  static constexpr int Q = P1 + 1;
  static constexpr int R1 = P1 * P1, PP = (P1 % 2) ? P1 : P1 + 1, R2 = Q * PP, PAD = 0;
};

// Searched (fewest 64-bit shared-memory bank conflicts over the stage access
// patterns, 16-lane phases; at most 2-way) for the default batch sizes:
template <> struct LayoutDG<2, 16> { static constexpr int Q = 3, R1 = 10, PP = 3, R2 = 10, PAD = 2; };
template <> struct LayoutDG<3, 8> { static constexpr int Q = 4, R1 = 19, PP = 4, R2 = 19, PAD = 4; };
template <> struct LayoutDG<4, 4> { static constexpr int Q = 5, R1 = 28, PP = 5, R2 = 28, PAD = 4; };
template <> struct LayoutDG<5, 4> { static constexpr int Q = 6, R1 = 37, PP = 6, R2 = 37, PAD = 2; };
template <> struct LayoutDG<6, 2> { static constexpr int Q = 7, R1 = 38, PP = 7, R2 = 54, PAD = 6; };
template <> struct LayoutDG<7, 2> { static constexpr int Q = 8, R1 = 55, PP = 10, R2 = 87, PAD = 8; };
template <> struct LayoutDG<8, 2> { static constexpr int Q = 9, R1 = 72, PP = 9, R2 = 88, PAD = 8; };
template <> struct LayoutDG<9, 2> { static constexpr int Q = 10, R1 = 89, PP = 10, R2 = 105, PAD = 6; };

template <int P1, int Q, int NE>
struct CfgDG {
  using L = LayoutDG<P1, NE>;
  static constexpr int P = P1, P2 = P1 * P1, P3 = P2 * P1, Q2 = Q * Q, Q3 = Q2 * Q;
  static constexpr int R1 = L::R1, PP = L::PP, R2 = L::R2;
  static constexpr int T2OFF = Q * R1;
  static constexpr int EB = Q * R1 + Q * R2 + L::PAD;
  static constexpr int XB = ((NE * P3) + 1) / 2 * 2;             // x in / y out stage (even)
  static constexpr int QSL = ((NE * Q3 + 2) + 1) / 2 * 2;        // D stage (even)
  static constexpr int OFF_X = 0;
  static constexpr int OFF_Q = 2 * XB;
  static constexpr int OFF_W = OFF_Q + 2 * QSL;
  static constexpr int SMEM_DOUBLES = OFF_W + NE * EB;
  static constexpr int SMEM_BYTES = SMEM_DOUBLES * 8;
};

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Thread 0: x and D of batch bk into stage (xs, qs), completing on `bar`.  An
// odd-length x tail (last batch only) loads its final double directly (the
// bulk size must be a multiple of 16 B and x has no slack); D has 16 B of slack.
template <int P1, int Q, int NE>
__device__ __forceinline__ void dg_issue(const DGArgs& A, double* xs, double* qs,
                                         unsigned long long* bar, long long bk) {
  using C = CfgDG<P1, Q, NE>;
  const long long e0 = bk * NE;
  const long long cnt = A.E - e0 < NE ? A.E - e0 : NE;
  const long long nx = cnt * C::P3;
  const unsigned xbytes = (unsigned)((nx & ~1LL) * 8);
  const unsigned qbytes = (unsigned)((cnt * C::Q3 * 8 + 15) & ~15LL);
  if (nx & 1) xs[nx - 1] = A.x[e0 * C::P3 + nx - 1];
  fence_proxy_async();
  mbar_expect_tx(bar, xbytes + qbytes);
  if (xbytes) bulk_g2s(xs, A.x + e0 * C::P3, xbytes, bar);
  bulk_g2s(qs, A.qd + e0 * C::Q3, qbytes, bar);
}

template <int P1, int Q, int NE, int NT>
__global__ void __launch_bounds__(NT) dg_mass_simt(const __grid_constant__ Tab<P1, Q> T,
                                                   const __grid_constant__ DGArgs A) {
  using C = CfgDG<P1, Q, NE>;
  constexpr int P = P1, H = (P + 1) / 2, PH = P / 2, QH = Q / 2, HQ = (Q + 1) / 2;
  constexpr int P2 = C::P2, P3 = C::P3, Q2 = C::Q2, Q3 = C::Q3, R1 = C::R1, R2 = C::R2,
                PP = C::PP, EB = C::EB, T2O = C::T2OFF;
  (void)H; (void)PH;
  extern __shared__ __align__(16) double smem[];
  double* XS0 = smem + C::OFF_X;
  double* QS0 = smem + C::OFF_Q;
  double* W = smem + C::OFF_W;
  __shared__ __align__(8) unsigned long long qbar[2];
  if (threadIdx.x == 0) {
    mbar_init(&qbar[0], 1);
    mbar_init(&qbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long bk = blockIdx.x;
  if (bk >= A.nbatch) return;
  if (threadIdx.x == 0) dg_issue<P1, Q, NE>(A, XS0, QS0, &qbar[0], bk);
  unsigned phase = 0;  // bit j: parity of qbar[j]
  for (int k = 0; bk < A.nbatch; ++k, bk += gridDim.x) {
    const int buf = k & 1;
    const long long nb = bk + gridDim.x;
    const int tid = vtid();
    const int zo = (int)(bk >> 40);  // == 0, loop-variant (see cdot in fused_impl.cuh)
    double* X = XS0 + buf * C::XB;
    const double* QD = QS0 + buf * C::QSL;
    if (threadIdx.x == 0 && nb < A.nbatch) {
      bulk_wait_read();  // the previous batch's y store has read stage buf^1
      dg_issue<P1, Q, NE>(A, XS0 + (buf ^ 1) * C::XB, QS0 + (buf ^ 1) * C::QSL, &qbar[buf ^ 1],
                          nb);
    }
    mbar_wait(&qbar[buf], (phase >> buf) & 1u);
    phase ^= 1u << buf;
    cta_sync();  // (the odd tail double of x is a generic store by thread 0)

    // ---- S1: z lines (items (b, a), a fastest) -> T1[qz][b][a]
    FOR_ITEMS(it, NE * P2, NT, tid) {
      const int el = it / P2, r = it % P2;
      const double* xl = X + el * P3 + r;
      double v[P];
#pragma unroll
      for (int c = 0; c < P; ++c) v[c] = xl[c * P2];
      double e[H], o[PH];
      eo_split<P>(v, e, o);
      double* t1 = W + el * EB + r;
#pragma unroll
      for (int t = 0; t < QH; ++t) {
        double lo, hi;
        eo_fwd<1, P>(T.BE, T.BO, t, zo, e, o, lo, hi);
        t1[t * R1] = lo;
        t1[(Q - 1 - t) * R1] = hi;
      }
      if (Q & 1) t1[QH * R1] = eo_fwd_mid<1, P>(T.BE, T.BO, QH, zo, e, o);
    }
    cta_sync();
    // ---- S2: y lines (items (qz, a), a fastest) -> T2[qz][qy][a]
    FOR_ITEMS(it, NE * Q * P, NT, tid) {
      const int el = it / (Q * P), r = it % (Q * P), qz = r / P, a = r % P;
      const double* t1 = W + el * EB + qz * R1 + a;
      double v[P];
#pragma unroll
      for (int b = 0; b < P; ++b) v[b] = t1[b * P];
      double e[H], o[PH];
      eo_split<P>(v, e, o);
      double* t2 = W + el * EB + T2O + qz * R2 + a;
#pragma unroll
      for (int t = 0; t < QH; ++t) {
        double lo, hi;
        eo_fwd<1, P>(T.BE, T.BO, t, zo, e, o, lo, hi);
        t2[t * PP] = lo;
        t2[(Q - 1 - t) * PP] = hi;
      }
      if (Q & 1) t2[QH * PP] = eo_fwd_mid<1, P>(T.BE, T.BO, QH, zo, e, o);
    }
    cta_sync();
    // ---- S3: x lines (items (qz, qy), qy fastest): x contraction, D, x back
    FOR_ITEMS(it, NE * Q2, NT, tid) {
      const int el = it / Q2, r = it % Q2, qz = r / Q, qy = r % Q;
      double* t2 = W + el * EB + T2O + qz * R2 + qy * PP;
      const double* qde = QD + el * Q3 + qz * Q2 + qy * Q;
      double g[P];
#pragma unroll
      for (int a = 0; a < P; ++a) g[a] = t2[a];
      double e[H], o[PH], SE[H], SO[PH];
      eo_split<P>(g, e, o);
      zero(SE);
      zero(SO);
#pragma unroll
      for (int t = 0; t < HQ; ++t) {
        if ((Q & 1) && t == QH) {
          const double u = eo_fwd_mid<1, P>(T.BE, T.BO, t, zo, e, o);
          eo_acc_mid<1, P>(T.BE, T.BO, t, zo, qde[t] * u, SE, SO);
        } else {
          double ul, uh;
          eo_fwd<1, P>(T.BE, T.BO, t, zo, e, o, ul, uh);
          eo_acc<1, P>(T.BE, T.BO, t, zo, qde[t] * ul, qde[Q - 1 - t] * uh, SE, SO);
        }
      }
      double s[P];
      eo_join<P>(SE, SO, s);
#pragma unroll
      for (int a = 0; a < P; ++a) t2[a] = s[a];
    }
    cta_sync();
    // ---- S2T: y back (items (qz, a)) -> T1[qz][b][a]
    FOR_ITEMS(it, NE * Q * P, NT, tid) {
      const int el = it / (Q * P), r = it % (Q * P), qz = r / P, a = r % P;
      const double* t2 = W + el * EB + T2O + qz * R2 + a;
      double* t1 = W + el * EB + qz * R1 + a;
      double SE[H], SO[PH], rb[P];
      zero(SE);
      zero(SO);
#pragma unroll
      for (int t = 0; t < HQ; ++t) {
        if ((Q & 1) && t == QH)
          eo_acc_mid<1, P>(T.BE, T.BO, t, zo, t2[t * PP], SE, SO);
        else
          eo_acc<1, P>(T.BE, T.BO, t, zo, t2[t * PP], t2[(Q - 1 - t) * PP], SE, SO);
      }
      eo_join<P>(SE, SO, rb);
#pragma unroll
      for (int b = 0; b < P; ++b) t1[b * P] = rb[b];
    }
    cta_sync();
    // ---- S1T: z back (items (b, a)) -> y[c][b][a] into the x stage (dense)
    FOR_ITEMS(it, NE * P2, NT, tid) {
      const int el = it / P2, r = it % P2;
      const double* t1 = W + el * EB + r;
      double SE[H], SO[PH], y[P];
      zero(SE);
      zero(SO);
#pragma unroll
      for (int t = 0; t < HQ; ++t) {
        if ((Q & 1) && t == QH)
          eo_acc_mid<1, P>(T.BE, T.BO, t, zo, t1[t * R1], SE, SO);
        else
          eo_acc<1, P>(T.BE, T.BO, t, zo, t1[t * R1], t1[(Q - 1 - t) * R1], SE, SO);
      }
      eo_join<P>(SE, SO, y);
      double* yo = X + el * P3 + r;
#pragma unroll
      for (int c = 0; c < P; ++c) yo[c * P2] = y[c];
    }
    cta_sync();
    // ---- y: one bulk store of the batch's contiguous E-vector range
    if (threadIdx.x == 0) {
      const long long e0 = bk * NE;
      const long long ny = (A.E - e0 < NE ? A.E - e0 : NE) * P3;
      if (ny & 1) A.y[e0 * P3 + ny - 1] = X[ny - 1];
      fence_proxy_async();
      if (ny > 1) bulk_s2g(A.y + e0 * P3, X, (unsigned)((ny & ~1LL) * 8));
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

// Per-P1 batch shapes (elements per batch, threads): stage-3 items NE*Q^2 <= NT,
// shared memory small enough for several CTAs per SM (bytes in flight and
// barrier-latency hiding).  -DHOFEM_DG_NE=.. -DHOFEM_DG_NT=.. overrides the
// shape of the P1 being compiled (tuning builds, scripts/build_pvariant.py).
template <int P1>
struct ShapeDGD;
template <> struct ShapeDGD<2> { static constexpr int NE = 16, NT = 160; };
template <> struct ShapeDGD<3> { static constexpr int NE = 8, NT = 128; };
template <> struct ShapeDGD<4> { static constexpr int NE = 4, NT = 128; };
template <> struct ShapeDGD<5> { static constexpr int NE = 4, NT = 160; };
template <> struct ShapeDGD<6> { static constexpr int NE = 2, NT = 128; };
template <> struct ShapeDGD<7> { static constexpr int NE = 2, NT = 128; };
template <> struct ShapeDGD<8> { static constexpr int NE = 2, NT = 192; };
template <> struct ShapeDGD<9> { static constexpr int NE = 2, NT = 224; };
#if defined(HOFEM_DG_NE) && defined(HOFEM_DG_NT)
template <int P1>
struct ShapeDG {
  static constexpr int NE = HOFEM_DG_NE, NT = HOFEM_DG_NT;
};
#else
template <int P1>
struct ShapeDG : ShapeDGD<P1> {};
#endif

// Defined per P1 in dg_p.cu (Q = P1 + 1, the Gauss rule of reading R2).
template <int P1>
cudaError_t dg_launch(int Q, const double* B, const DGArgs& A, int* grid_io, cudaStream_t s);
template <int P1>
int dg_batch_elems();

}  // namespace hofem
