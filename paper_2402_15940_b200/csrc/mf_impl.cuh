// mf_impl.cuh -- fully matrix-free BP3 diffusion apply, SURVEY.md §8(f) f3
// (§2.2 "Fully Matrix-Free. All necessary data needed for operator
// evaluation is computed on the fly, minimizing storage and memory
// requirements, at the cost of potentially recomputing data").
//
// Same operator as the PA path (reading R3-R6: y = R^T B^T D B R x with
// D = W adj(J) adj(J)^T / detJ), but D is never stored: every apply recomputes
// J = dX/dxi at the quadrature points from the element's nodal coordinates by
// the same sum factorization as the gradient of u (the mesh is isoparametric,
// so each coordinate field is just another degree-p field), then adj(J), detJ
// and D pointwise.  HBM stream per apply: x and the 3 coordinate fields
// (gathered from L-vectors, 32 B/DOF) and the E-vector round trip of the
// deterministic scatter, instead of the 8*6*Q^3/P1^3 B/DOF of the qdata.
//
// Persistent kernel over batches of NE elements; per batch:
//   gather   x (Dirichlet points zero-filled, reading R6) and X, Y, Z of the
//            batch's elements into padded a-slowest stages (asynchronous 8-byte
//            copies: the next batch's gather overlaps this batch's math);
//   geometry for each coordinate field f: x / y / z contractions (even-odd, the
//            forward half of the u pipeline) -> J[f][0..2] at every point; after
//            field 2, D = W adj(J) adj(J)^T / detJ in place (6 values per point);
//   apply    the five thread-per-line stages of the PA kernel with D from shared
//            memory;
//   output   y_e to the E-vector (coalesced); the host then runs the
//            transposed-offset scatter (ascending (e, i): deterministic) with
//            y[ess] = x[ess].
#pragma once

#include "fused_impl.cuh"

namespace hofem {

struct MFArgs {
  const double* x;
  const double* coords;  // 3 x n_local (x, y, z components)
  double* ye;            // E-vector [E][P1^3]
  int nx, ny, nzl;
  long long Nx, Ny, n_local, K0, NzG;
  int bc;
  long long E, nbatch;
};

template <int P1, int Q, int NE>
struct CfgMF {
  static constexpr int P = P1, P2 = P1 * P1, P3 = P2 * P1, Q2 = Q * Q, Q3 = Q2 * Q;
  static constexpr int XS = (P2 % 2) ? P2 : P2 + 1;  // a-stride of the gathered stages (odd)
  static constexpr int XE = P * XS;
  static constexpr int S1 = P2 + (((P - P2) % 16) + 16) % 16;
  static constexpr int T1M = Q * S1, T1SZ = 2 * T1M;
  static constexpr int SP = (P % 2) ? P : P + 1;
  static constexpr int T2M = Q2 * SP;
  static constexpr int EB0 = T1SZ + (3 * T2M > XE ? 3 * T2M : XE);
  static constexpr int EB = EB0 + ((7 - EB0) % 16 + 16) % 16;  // == 7 (mod 16)
  static constexpr int DQ = 6 * Q3 + 1;                          // D (and J of fields 0, 1)
  static constexpr int GS = 4 * NE * XE;                         // one gather stage: x, X, Y, Z
  static constexpr int OFF_G = 0;
  static constexpr int OFF_D = 2 * GS;
  static constexpr int OFF_W = OFF_D + NE * DQ;
  static constexpr int SMEM_DOUBLES = OFF_W + NE * EB;
  static constexpr int SMEM_BYTES = SMEM_DOUBLES * 8;
};

template <int P1, int Q>
struct TabW {
  double w[Q];  // 1D Gauss weights on [0,1]
};

template <int P1, int Q, int NE, int NT>
__device__ __forceinline__ void mf_issue(const MFArgs& A, double* gs, long long bk) {
  using C = CfgMF<P1, Q, NE>;
  constexpr int P = P1, p = P1 - 1;
  const long long e0 = bk * NE;
  for (int i = threadIdx.x; i < NE * C::P3; i += NT) {
    const int el = i / C::P3, g = i - el * C::P3;
    const int a = g % P, b = (g / P) % P, c = g / C::P2;
    const long long e = e0 + el;
    const bool ve = e < A.E;
    long long l = 0;
    bool ess = false;
    if (ve) {
      const long long ex = e % A.nx, ey = (e / A.nx) % A.ny, ez = e / ((long long)A.nx * A.ny);
      const long long I = p * ex + a, J = p * ey + b, K = p * ez + c;
      l = I + A.Nx * (J + A.Ny * K);
      const long long Kg = K + A.K0;
      ess = A.bc && (I == 0 || I == A.Nx - 1 || J == 0 || J == A.Ny - 1 || Kg == 0 || Kg == A.NzG - 1);
    }
    const int off = el * C::XE + a * C::XS + b * P + c;
    cp_async8(gs + off, ve && !ess ? A.x + l : A.x, ve && !ess);
#pragma unroll
    for (int f = 0; f < 3; ++f)
      cp_async8(gs + (f + 1) * NE * C::XE + off, ve ? A.coords + f * A.n_local + l : A.coords, ve);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// S1 (x lines, items (b, c)) of one field: T1[0] = B_x F, T1[1] = G_x F
template <int P1, int Q, int NE, int NT>
__device__ __forceinline__ void mf_s1(const Tab<P1, Q>& T, const double* F, double* W, int tid,
                                      int zo) {
  using C = CfgMF<P1, Q, NE>;
  constexpr int P = P1, H = (P + 1) / 2, PH = P / 2, QH = Q / 2;
  FOR_ITEMS(it, NE * P * P, NT, tid) {
    const int el = it / (P * P), r = it % (P * P);
    const double* xl = F + el * C::XE + r;
    double xa[P];
#pragma unroll
    for (int a = 0; a < P; ++a) xa[a] = xl[C::XS * a];
    double e[H], o[PH];
    eo_split<P>(xa, e, o);
    double* t1 = W + el * C::EB + r;
#pragma unroll
    for (int t = 0; t < QH; ++t) {
      double lo, hi;
      eo_fwd<1, P>(T.BE, T.BO, t, zo, e, o, lo, hi);
      t1[t * C::S1] = lo;
      t1[(Q - 1 - t) * C::S1] = hi;
      eo_fwd<-1, P>(T.GE, T.GO, t, zo, e, o, lo, hi);
      t1[C::T1M + t * C::S1] = lo;
      t1[C::T1M + (Q - 1 - t) * C::S1] = hi;
    }
    if (Q & 1) {
      t1[QH * C::S1] = eo_fwd_mid<1, P>(T.BE, T.BO, QH, zo, e, o);
      t1[C::T1M + QH * C::S1] = eo_fwd_mid<-1, P>(T.GE, T.GO, QH, zo, e, o);
    }
  }
}

// S2 (y lines, items (qx, c)): T2[0] = G_x B_y, T2[1] = B_x G_y, T2[2] = B_x B_y
template <int P1, int Q, int NE, int NT>
__device__ __forceinline__ void mf_s2(const Tab<P1, Q>& T, double* W, int tid, int zo) {
  using C = CfgMF<P1, Q, NE>;
  constexpr int P = P1, H = (P + 1) / 2, PH = P / 2, QH = Q / 2, SP = C::SP, T2M = C::T2M;
  FOR_ITEMS(it, NE * Q * P, NT, tid) {
    const int el = it / (Q * P), r = it % (Q * P), qx = r / P, c = r % P;
    const double* t1 = W + el * C::EB + qx * C::S1 + c;
    double vb[P], vg[P];
#pragma unroll
    for (int b = 0; b < P; ++b) {
      vb[b] = t1[b * P];
      vg[b] = t1[C::T1M + b * P];
    }
    double eb[H], ob[PH], eg[H], og[PH];
    eo_split<P>(vb, eb, ob);
    eo_split<P>(vg, eg, og);
    double* t2 = W + el * C::EB + C::T1SZ + qx * SP + c;
    auto put = [&](int qy, double bb, double gb, double bg) {
      t2[qy * Q * SP] = gb;
      t2[T2M + qy * Q * SP] = bg;
      t2[2 * T2M + qy * Q * SP] = bb;
    };
#pragma unroll
    for (int t = 0; t < QH; ++t) {
      double bbl, bbh, gbl, gbh, bgl, bgh;
      eo_fwd<1, P>(T.BE, T.BO, t, zo, eb, ob, bbl, bbh);
      eo_fwd<1, P>(T.BE, T.BO, t, zo, eg, og, gbl, gbh);
      eo_fwd<-1, P>(T.GE, T.GO, t, zo, eb, ob, bgl, bgh);
      put(t, bbl, gbl, bgl);
      put(Q - 1 - t, bbh, gbh, bgh);
    }
    if (Q & 1) {
      put(QH, eo_fwd_mid<1, P>(T.BE, T.BO, QH, zo, eb, ob),
          eo_fwd_mid<1, P>(T.BE, T.BO, QH, zo, eg, og),
          eo_fwd_mid<-1, P>(T.GE, T.GO, QH, zo, eb, ob));
    }
  }
}

// D = W adj(J) adj(J)^T / detJ, entries [00,01,02,11,12,22] (reading R3);
// J[i][j] = d x_i / d xi_j.
__device__ __forceinline__ void geo_d(const double (&J)[3][3], double W, double (&D)[6]) {
  const double a00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  const double a01 = J[0][2] * J[2][1] - J[0][1] * J[2][2];
  const double a02 = J[0][1] * J[1][2] - J[0][2] * J[1][1];
  const double a10 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  const double a11 = J[0][0] * J[2][2] - J[0][2] * J[2][0];
  const double a12 = J[0][2] * J[1][0] - J[0][0] * J[1][2];
  const double a20 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  const double a21 = J[0][1] * J[2][0] - J[0][0] * J[2][1];
  const double a22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  const double det = J[0][0] * a00 + J[0][1] * a10 + J[0][2] * a20;
  const double s = W / det;
  D[0] = s * (a00 * a00 + a01 * a01 + a02 * a02);
  D[1] = s * (a00 * a10 + a01 * a11 + a02 * a12);
  D[2] = s * (a00 * a20 + a01 * a21 + a02 * a22);
  D[3] = s * (a10 * a10 + a11 * a11 + a12 * a12);
  D[4] = s * (a10 * a20 + a11 * a21 + a12 * a22);
  D[5] = s * (a20 * a20 + a21 * a21 + a22 * a22);
}

template <int P1, int Q, int NE, int NT>
__global__ void __launch_bounds__(NT) mf_diffusion_simt(const __grid_constant__ Tab<P1, Q> T,
                                                        const __grid_constant__ TabW<P1, Q> TW,
                                                        const __grid_constant__ MFArgs A) {
  using C = CfgMF<P1, Q, NE>;
  constexpr int P = P1, H = (P + 1) / 2, PH = P / 2, QH = Q / 2, HQ = (Q + 1) / 2;
  constexpr int Q2 = C::Q2, Q3 = C::Q3, S1 = C::S1, T1M = C::T1M, T1SZ = C::T1SZ, SP = C::SP,
                T2M = C::T2M, EB = C::EB, XS = C::XS;
  (void)H; (void)PH;
  extern __shared__ __align__(16) double smem[];
  double* GS0 = smem + C::OFF_G;
  double* DQ = smem + C::OFF_D;
  double* W = smem + C::OFF_W;
  long long bk = blockIdx.x;
  if (bk >= A.nbatch) return;
  mf_issue<P1, Q, NE, NT>(A, GS0, bk);
  for (int k = 0; bk < A.nbatch; ++k, bk += gridDim.x) {
    const int buf = k & 1;
    const long long nb = bk + gridDim.x;
    const int tid = vtid();
    const int zo = (int)(bk >> 40);  // == 0, loop-variant (see cdot in fused_impl.cuh)
    if (nb < A.nbatch)
      mf_issue<P1, Q, NE, NT>(A, GS0 + (buf ^ 1) * C::GS, nb);
    else
      asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    cta_sync();
    const double* G = GS0 + buf * C::GS;

    // ---- geometry: J[f][j] for the three coordinate fields, then D in place
#pragma unroll 1
    for (int f = 0; f < 3; ++f) {
      mf_s1<P1, Q, NE, NT>(T, G + (f + 1) * NE * C::XE, W, tid, zo);
      cta_sync();
      mf_s2<P1, Q, NE, NT>(T, W, tid, zo);
      cta_sync();
      FOR_ITEMS(it, NE * Q2, NT, tid) {
        const int el = it / Q2, pt = it % Q2;
        const double* t2 = W + el * EB + T1SZ + pt * SP;
        double* dq = DQ + el * C::DQ + pt;
        double g0[P], g1[P], g2[P];
#pragma unroll
        for (int c = 0; c < P; ++c) {
          g0[c] = t2[c];
          g1[c] = t2[T2M + c];
          g2[c] = t2[2 * T2M + c];
        }
        double e0[H], o0[PH], e1[H], o1[PH], e2[H], o2[PH];
        eo_split<P>(g0, e0, o0);
        eo_split<P>(g1, e1, o1);
        eo_split<P>(g2, e2, o2);
        const int qx = pt % Q, qy = pt / Q;
        const double wxy = TW.w[qx] * TW.w[qy];
#pragma unroll
        for (int t = 0; t < HQ; ++t) {
          const bool mid = (Q & 1) && t == QH;
          double j0[2], j1[2], j2[2];
          if (mid) {
            j0[0] = eo_fwd_mid<1, P>(T.BE, T.BO, t, zo, e0, o0);
            j1[0] = eo_fwd_mid<1, P>(T.BE, T.BO, t, zo, e1, o1);
            j2[0] = eo_fwd_mid<-1, P>(T.GE, T.GO, t, zo, e2, o2);
          } else {
            eo_fwd<1, P>(T.BE, T.BO, t, zo, e0, o0, j0[0], j0[1]);
            eo_fwd<1, P>(T.BE, T.BO, t, zo, e1, o1, j1[0], j1[1]);
            eo_fwd<-1, P>(T.GE, T.GO, t, zo, e2, o2, j2[0], j2[1]);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (mid && h) continue;
            const int qz = h ? Q - 1 - t : t;
            double* d = dq + qz * Q2;
            if (f < 2) {  // J row f (field f): d x_f / d xi_{0,1,2}
              d[(3 * f + 0) * Q3] = j0[h];
              d[(3 * f + 1) * Q3] = j1[h];
              d[(3 * f + 2) * Q3] = j2[h];
            } else {      // all three rows known: D in place of J rows 0, 1
              const double J[3][3] = {{d[0], d[Q3], d[2 * Q3]},
                                      {d[3 * Q3], d[4 * Q3], d[5 * Q3]},
                                      {j0[h], j1[h], j2[h]}};
              double Dv[6];
              geo_d(J, wxy * TW.w[qz], Dv);
#pragma unroll
              for (int m = 0; m < 6; ++m) d[m * Q3] = Dv[m];
            }
          }
        }
      }
      cta_sync();
    }

    // ---- u: S1, S2 (gradient to the points), S3 (z, D, z back), S2T, S1T
    mf_s1<P1, Q, NE, NT>(T, G, W, tid, zo);
    cta_sync();
    mf_s2<P1, Q, NE, NT>(T, W, tid, zo);
    cta_sync();
    FOR_ITEMS(it, NE * Q2, NT, tid) {
      const int el = it / Q2, pt = it % Q2;
      const double* qde = DQ + el * C::DQ + pt;
      double* t2 = W + el * EB + T1SZ + pt * SP;
      double g0[P], g1[P], g2[P];
#pragma unroll
      for (int c = 0; c < P; ++c) {
        g0[c] = t2[c];
        g1[c] = t2[T2M + c];
        g2[c] = t2[2 * T2M + c];
      }
      double e0[H], o0[PH], e1[H], o1[PH], e2[H], o2[PH];
      eo_split<P>(g0, e0, o0);
      eo_split<P>(g1, e1, o1);
      eo_split<P>(g2, e2, o2);
      double SE0[H], SO0[PH], SE1[H], SO1[PH], SE2[H], SO2[PH];
      zero(SE0); zero(SO0); zero(SE1); zero(SO1); zero(SE2); zero(SO2);
#pragma unroll
      for (int t = 0; t < HQ; ++t) {
        const bool mid = (Q & 1) && t == QH;
        double dl[6], dh[6];
#pragma unroll
        for (int m = 0; m < 6; ++m) {
          dl[m] = qde[m * Q3 + t * Q2];
          dh[m] = mid ? 0.0 : qde[m * Q3 + (Q - 1 - t) * Q2];
        }
        double u0l, u0h = 0.0, u1l, u1h = 0.0, u2l, u2h = 0.0;
        if (mid) {
          u0l = eo_fwd_mid<1, P>(T.BE, T.BO, t, zo, e0, o0);
          u1l = eo_fwd_mid<1, P>(T.BE, T.BO, t, zo, e1, o1);
          u2l = eo_fwd_mid<-1, P>(T.GE, T.GO, t, zo, e2, o2);
        } else {
          eo_fwd<1, P>(T.BE, T.BO, t, zo, e0, o0, u0l, u0h);
          eo_fwd<1, P>(T.BE, T.BO, t, zo, e1, o1, u1l, u1h);
          eo_fwd<-1, P>(T.GE, T.GO, t, zo, e2, o2, u2l, u2h);
        }
        const double w0l = dl[0] * u0l + dl[1] * u1l + dl[2] * u2l;
        const double w1l = dl[1] * u0l + dl[3] * u1l + dl[4] * u2l;
        const double w2l = dl[2] * u0l + dl[4] * u1l + dl[5] * u2l;
        if (mid) {
          eo_acc_mid<1, P>(T.BE, T.BO, t, zo, w0l, SE0, SO0);
          eo_acc_mid<1, P>(T.BE, T.BO, t, zo, w1l, SE1, SO1);
          eo_acc_mid<-1, P>(T.GE, T.GO, t, zo, w2l, SE2, SO2);
        } else {
          const double w0h = dh[0] * u0h + dh[1] * u1h + dh[2] * u2h;
          const double w1h = dh[1] * u0h + dh[3] * u1h + dh[4] * u2h;
          const double w2h = dh[2] * u0h + dh[4] * u1h + dh[5] * u2h;
          eo_acc<1, P>(T.BE, T.BO, t, zo, w0l, w0h, SE0, SO0);
          eo_acc<1, P>(T.BE, T.BO, t, zo, w1l, w1h, SE1, SO1);
          eo_acc<-1, P>(T.GE, T.GO, t, zo, w2l, w2h, SE2, SO2);
        }
      }
      double s[P];
      eo_join<P>(SE0, SO0, s);
#pragma unroll
      for (int c = 0; c < P; ++c) t2[c] = s[c];
      eo_join<P>(SE1, SO1, s);
#pragma unroll
      for (int c = 0; c < P; ++c) t2[T2M + c] = s[c];
      eo_join<P>(SE2, SO2, s);
#pragma unroll
      for (int c = 0; c < P; ++c) t2[2 * T2M + c] = s[c];
    }
    cta_sync();
    // S2T: rg = B_y^T v0 (x part), rb = G_y^T v1 + B_y^T v2 (y, z parts)
    FOR_ITEMS(it, NE * Q * P, NT, tid) {
      const int el = it / (Q * P), r = it % (Q * P), qx = r / P, c = r % P;
      const double* t2 = W + el * EB + T1SZ + qx * SP + c;
      double* t1 = W + el * EB + qx * S1 + c;
      double SEg[H], SOg[PH], SEb[H], SOb[PH], rg[P], rb[P];
      zero(SEg); zero(SOg); zero(SEb); zero(SOb);
      constexpr int QS = Q * SP;
#pragma unroll
      for (int t = 0; t < HQ; ++t) {
        if ((Q & 1) && t == QH) {
          eo_acc_mid<1, P>(T.BE, T.BO, t, zo, t2[t * QS], SEg, SOg);
          eo_acc_mid<1, P>(T.BE, T.BO, t, zo, t2[2 * T2M + t * QS], SEb, SOb);
          eo_acc_mid<-1, P>(T.GE, T.GO, t, zo, t2[T2M + t * QS], SEb, SOb);
          continue;
        }
        const int th = Q - 1 - t;
        eo_acc<1, P>(T.BE, T.BO, t, zo, t2[t * QS], t2[th * QS], SEg, SOg);
        eo_acc<1, P>(T.BE, T.BO, t, zo, t2[2 * T2M + t * QS], t2[2 * T2M + th * QS], SEb, SOb);
        eo_acc<-1, P>(T.GE, T.GO, t, zo, t2[T2M + t * QS], t2[T2M + th * QS], SEb, SOb);
      }
      eo_join<P>(SEb, SOb, rb);
      eo_join<P>(SEg, SOg, rg);
#pragma unroll
      for (int b = 0; b < P; ++b) {
        t1[b * P] = rb[b];
        t1[T1M + b * P] = rg[b];
      }
    }
    cta_sync();
    // S1T: ye = B_x^T vb + G_x^T vg -> staging [a][b][c] (aliases T2)
    FOR_ITEMS(it, NE * P * P, NT, tid) {
      const int el = it / (P * P), r = it % (P * P);
      const double* t1 = W + el * EB + r;
      double SE[H], SO[PH], ye[P];
      zero(SE); zero(SO);
#pragma unroll
      for (int t = 0; t < HQ; ++t) {
        if ((Q & 1) && t == QH) {
          eo_acc_mid<1, P>(T.BE, T.BO, t, zo, t1[t * S1], SE, SO);
          eo_acc_mid<-1, P>(T.GE, T.GO, t, zo, t1[T1M + t * S1], SE, SO);
          continue;
        }
        const int th = Q - 1 - t;
        eo_acc<1, P>(T.BE, T.BO, t, zo, t1[t * S1], t1[th * S1], SE, SO);
        eo_acc<-1, P>(T.GE, T.GO, t, zo, t1[T1M + t * S1], t1[T1M + th * S1], SE, SO);
      }
      eo_join<P>(SE, SO, ye);
      double* yo = W + el * EB + T1SZ + r;
#pragma unroll
      for (int a = 0; a < P; ++a) yo[XS * a] = ye[a];
    }
    cta_sync();
    {
      const long long e0 = bk * NE;
      const long long lim = (A.E - e0 < NE ? A.E - e0 : NE) * C::P3;
      for (int i = tid; i < lim; i += NT) {
        const int el = i / C::P3, g = i - el * C::P3;
        const int a = g % P, b = (g / P) % P, c = g / C::P2;
        A.ye[e0 * C::P3 + i] = W[el * EB + T1SZ + a * XS + b * P + c];
      }
    }
  }
}

// Per-P1 batch shapes (elements per batch, threads).
template <int P1>
struct ShapeMFD;
template <> struct ShapeMFD<2> { static constexpr int NE = 8, NT = 96; };
template <> struct ShapeMFD<3> { static constexpr int NE = 4, NT = 64; };
template <> struct ShapeMFD<4> { static constexpr int NE = 4, NT = 128; };  // r2q: -3.6 %
template <> struct ShapeMFD<5> { static constexpr int NE = 2, NT = 96; };
template <> struct ShapeMFD<6> { static constexpr int NE = 1, NT = 64; };
template <> struct ShapeMFD<7> { static constexpr int NE = 1, NT = 64; };
template <> struct ShapeMFD<8> { static constexpr int NE = 1, NT = 96; };
template <> struct ShapeMFD<9> { static constexpr int NE = 1, NT = 128; };
#if defined(HOFEM_MF_NE) && defined(HOFEM_MF_NT)
template <int P1>
struct ShapeMF {
  static constexpr int NE = HOFEM_MF_NE, NT = HOFEM_MF_NT;
};
#else
template <int P1>
struct ShapeMF : ShapeMFD<P1> {};
#endif

// Defined per P1 in mf_p.cu (Gauss Q = P1 + 1).
template <int P1>
cudaError_t mf_launch(int Q, const double* B, const double* G, const double* w,
                      const MFArgs& A, int* grid_io, cudaStream_t s);
template <int P1>
int mf_batch_elems();

}  // namespace hofem
