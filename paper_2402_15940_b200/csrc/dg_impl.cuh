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
// Persistent kernel, one CTA per (SM x occupancy), batches of NE elements:
//   - x of the NEXT batch arrives by asynchronous 8-byte copies (coalesced global
//     reads) into a padded, a-slowest shared-memory stage (odd strides: bank-
//     conflict-free stage-1 reads), double-buffered;
//   - D of the next batch (contiguous NE*Q^3 doubles) by ONE bulk copy
//     (cp.async.bulk, the TMA engine) into a second double-buffered stage,
//     completion on an mbarrier;
//   - the five thread-per-line stages of the SIMT brick kernel (even-odd
//     contractions, tables from the kernel-parameter constant bank): x, y, z+D+z^T,
//     y^T, x^T;
//   - y written back with coalesced stores.
// Bound: HBM (16 + 8 Q^3/P1^3 B/DOF; flop/B < 3.1 even at p = 8).
#pragma once

#include "fused_impl.cuh"

namespace hofem {

struct DGArgs {
  const double* x;
  double* y;
  const double* qd;  // [E][Q^3] W*detJ
  long long E;       // local elements
  long long nbatch;  // ceil(E / NE)
};

template <int P1, int Q, int NE>
struct CfgDG {
  static constexpr int P = P1, P2 = P1 * P1, P3 = P2 * P1, Q2 = Q * Q, Q3 = Q2 * Q;
  static constexpr int XS = (P2 % 2) ? P2 : P2 + 1;  // a-stride of x / y staging (odd)
  static constexpr int XE = P * XS;                  // doubles per element
  static constexpr int S1 = P2 + (((P - P2) % 16) + 16) % 16;
  static constexpr int T1M = Q * S1;
  static constexpr int SP = (P % 2) ? P : P + 1;
  static constexpr int T2M = Q2 * SP;
  static constexpr int EB0 = T1M + (T2M > XE ? T2M : XE);
  static constexpr int EB = EB0 + ((7 - EB0) % 16 + 16) % 16;  // == 7 (mod 16)
  static constexpr int XB = NE * XE;                             // one x stage
  static constexpr int QSL = ((NE * Q3 + 2) + 1) / 2 * 2;        // one D stage (even)
  static constexpr int OFF_X = 0;
  static constexpr int OFF_Q = ((2 * XB) + 1) / 2 * 2;           // 16-byte aligned
  static constexpr int OFF_W = OFF_Q + 2 * QSL;
  static constexpr int SMEM_DOUBLES = OFF_W + NE * EB;
  static constexpr int SMEM_BYTES = SMEM_DOUBLES * 8;
  static_assert(T2M >= XE, "y staging aliases T2");
};

template <int P1, int Q, int NE, int NT>
__device__ __forceinline__ void dg_issue_x(const DGArgs& A, double* xs, long long bk) {
  using C = CfgDG<P1, Q, NE>;
  constexpr int P = P1;
  const long long e0 = bk * NE;
  for (int i = threadIdx.x; i < NE * C::P3; i += NT) {
    const int el = i / C::P3, g = i - el * C::P3;
    const int a = g % P, b = (g / P) % P, c = g / C::P2;
    const bool valid = e0 + el < A.E;
    cp_async8(xs + el * C::XE + a * C::XS + b * P + c, valid ? A.x + (e0 * C::P3 + i) : A.x,
              valid);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int P1, int Q, int NE>
__device__ __forceinline__ void dg_issue_q(const DGArgs& A, double* qs, unsigned long long* bar,
                                           long long bk) {
  using C = CfgDG<P1, Q, NE>;
  if (threadIdx.x != 0) return;
  const long long e0 = bk * NE;
  const long long cnt = A.E - e0 < NE ? A.E - e0 : NE;
  const unsigned bytes = (unsigned)((cnt * C::Q3 * 8 + 15) & ~15LL);  // qdata has 16 B of slack
  fence_proxy_async();
  mbar_expect_tx(bar, bytes);
  bulk_g2s(qs, A.qd + e0 * C::Q3, bytes, bar);
}

template <int P1, int Q, int NE, int NT>
__global__ void __launch_bounds__(NT) dg_mass_simt(const __grid_constant__ Tab<P1, Q> T,
                                                   const __grid_constant__ DGArgs A) {
  using C = CfgDG<P1, Q, NE>;
  constexpr int P = P1, H = (P + 1) / 2, PH = P / 2, QH = Q / 2, HQ = (Q + 1) / 2;
  constexpr int Q2 = C::Q2, S1 = C::S1, T1M = C::T1M, SP = C::SP, EB = C::EB, XS = C::XS;
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
  dg_issue_x<P1, Q, NE, NT>(A, XS0, bk);
  dg_issue_q<P1, Q, NE>(A, QS0, &qbar[0], bk);
  unsigned phase = 0;  // bit j: parity of qbar[j]
  for (int k = 0; bk < A.nbatch; ++k, bk += gridDim.x) {
    const int buf = k & 1;
    const long long nb = bk + gridDim.x;
    const int tid = vtid();
    const int zo = (int)(bk >> 40);  // == 0, loop-variant (see cb_row in fused_impl.cuh)
    if (nb < A.nbatch) {
      dg_issue_x<P1, Q, NE, NT>(A, XS0 + (buf ^ 1) * C::XB, nb);
      dg_issue_q<P1, Q, NE>(A, QS0 + (buf ^ 1) * C::QSL, &qbar[buf ^ 1], nb);
    } else {
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    cta_sync();
    const double* X = XS0 + buf * C::XB;

    // ---- S1: x lines (items (b, c), c fastest) -> T1[qx][b][c]
    FOR_ITEMS(it, NE * P * P, NT, tid) {
      const int el = it / (P * P), r = it % (P * P);
      const double* xl = X + el * C::XE + r;
      double xa[P];
#pragma unroll
      for (int a = 0; a < P; ++a) xa[a] = xl[XS * a];
      double e[H], o[PH];
      eo_split<P>(xa, e, o);
      double* t1 = W + el * EB + r;
#pragma unroll
      for (int t = 0; t < QH; ++t) {
        double lo, hi;
        eo_fwd<1, P>(T.BE, T.BO, t, zo, e, o, lo, hi);
        t1[t * S1] = lo;
        t1[(Q - 1 - t) * S1] = hi;
      }
      if (Q & 1) t1[QH * S1] = eo_fwd_mid<1, P>(T.BE, T.BO, QH, zo, e, o);
    }
    cta_sync();
    // ---- S2: y lines (items (qx, c), c fastest) -> T2[qy][qx][c]
    FOR_ITEMS(it, NE * Q * P, NT, tid) {
      const int el = it / (Q * P), r = it % (Q * P), qx = r / P, c = r % P;
      const double* t1 = W + el * EB + qx * S1 + c;
      double vb[P];
#pragma unroll
      for (int b = 0; b < P; ++b) vb[b] = t1[b * P];
      double eb[H], ob[PH];
      eo_split<P>(vb, eb, ob);
      double* t2 = W + el * EB + T1M + qx * SP + c;
#pragma unroll
      for (int t = 0; t < QH; ++t) {
        double lo, hi;
        eo_fwd<1, P>(T.BE, T.BO, t, zo, eb, ob, lo, hi);
        t2[t * Q * SP] = lo;
        t2[(Q - 1 - t) * Q * SP] = hi;
      }
      if (Q & 1) t2[QH * Q * SP] = eo_fwd_mid<1, P>(T.BE, T.BO, QH, zo, eb, ob);
    }
    cta_sync();
    // ---- S3: z lines (items (qx, qy)): z contraction, D, z back-contraction
    mbar_wait(&qbar[buf], (phase >> buf) & 1u);
    phase ^= 1u << buf;
    {
      const double* QD = QS0 + buf * C::QSL;
      FOR_ITEMS(it, NE * Q2, NT, tid) {
        const int el = it / Q2, pt = it % Q2;
        const double* qde = QD + el * C::Q3 + pt;
        double* t2 = W + el * EB + T1M + pt * SP;
        double g[P];
#pragma unroll
        for (int c = 0; c < P; ++c) g[c] = t2[c];
        double e[H], o[PH], SE[H], SO[PH];
        eo_split<P>(g, e, o);
        zero(SE);
        zero(SO);
#pragma unroll
        for (int t = 0; t < HQ; ++t) {
          if ((Q & 1) && t == QH) {
            const double u = eo_fwd_mid<1, P>(T.BE, T.BO, t, zo, e, o);
            eo_acc_mid<1, P>(T.BE, T.BO, t, zo, qde[t * Q2] * u, SE, SO);
          } else {
            double ul, uh;
            eo_fwd<1, P>(T.BE, T.BO, t, zo, e, o, ul, uh);
            eo_acc<1, P>(T.BE, T.BO, t, zo, qde[t * Q2] * ul, qde[(Q - 1 - t) * Q2] * uh, SE,
                         SO);
          }
        }
        double s[P];
        eo_join<P>(SE, SO, s);
#pragma unroll
        for (int c = 0; c < P; ++c) t2[c] = s[c];
      }
    }
    cta_sync();
    // ---- S2T: y back (items (qx, c)) -> T1[qx][b][c]
    FOR_ITEMS(it, NE * Q * P, NT, tid) {
      const int el = it / (Q * P), r = it % (Q * P), qx = r / P, c = r % P;
      const double* t2 = W + el * EB + T1M + qx * SP + c;
      double* t1 = W + el * EB + qx * S1 + c;
      double SE[H], SO[PH], rb[P];
      zero(SE);
      zero(SO);
      constexpr int QS = Q * SP;
#pragma unroll
      for (int t = 0; t < HQ; ++t) {
        if ((Q & 1) && t == QH)
          eo_acc_mid<1, P>(T.BE, T.BO, t, zo, t2[t * QS], SE, SO);
        else
          eo_acc<1, P>(T.BE, T.BO, t, zo, t2[t * QS], t2[(Q - 1 - t) * QS], SE, SO);
      }
      eo_join<P>(SE, SO, rb);
#pragma unroll
      for (int b = 0; b < P; ++b) t1[b * P] = rb[b];
    }
    cta_sync();
    // ---- S1T: x back (items (b, c)) -> y staging [a][b][c] (aliases T2)
    FOR_ITEMS(it, NE * P * P, NT, tid) {
      const int el = it / (P * P), r = it % (P * P);
      const double* t1 = W + el * EB + r;
      double SE[H], SO[PH], ye[P];
      zero(SE);
      zero(SO);
#pragma unroll
      for (int t = 0; t < HQ; ++t) {
        if ((Q & 1) && t == QH)
          eo_acc_mid<1, P>(T.BE, T.BO, t, zo, t1[t * S1], SE, SO);
        else
          eo_acc<1, P>(T.BE, T.BO, t, zo, t1[t * S1], t1[(Q - 1 - t) * S1], SE, SO);
      }
      eo_join<P>(SE, SO, ye);
      double* yo = W + el * EB + T1M + r;
#pragma unroll
      for (int a = 0; a < P; ++a) yo[XS * a] = ye[a];
    }
    cta_sync();
    // ---- y: coalesced stores of the batch's contiguous E-vector range
    {
      const long long e0 = bk * NE;
      const long long lim = (A.E - e0 < NE ? A.E - e0 : NE) * C::P3;
      for (int i = tid; i < lim; i += NT) {
        const int el = i / C::P3, g = i - el * C::P3;
        const int a = g % P, b = (g / P) % P, c = g / C::P2;
        A.y[e0 * C::P3 + i] = W[el * EB + T1M + a * XS + b * P + c];
      }
    }
  }
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
