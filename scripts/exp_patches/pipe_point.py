"""Experiment: point-granular rolling register prefetch of the apply's coefficient loads."""
import sys
p = sys.argv[1]
s = open(p).read()
a = s.index("#pragma unroll 1\n  for (int qx = 0; qx < 4; ++qx) {\n    double xB[3][2], xG[3][2];")
b = s.index("    accp[0] -= wxT * dv0;")
new = r'''  double cur[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) cur[k] = (k >= 1 && k <= 3 && !HG) ? 0.0 : __ldg(cp + (k * 4) * JNT);
#pragma unroll 1
  for (int qx = 0; qx < 4; ++qx) {
    double xB[3][2], xG[3][2];
#pragma unroll
    for (int jy = 0; jy < 3; ++jy)
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        const double f0 = XM.at(d, r0 + jy, c0), f1 = XM.at(d, r0 + jy, c0 + 1), f2 = XM.at(d, r0 + jy, c0 + 2);
        xB[jy][d] = T.B[qx][0] * f0 + T.B[qx][1] * f1 + T.B[qx][2] * f2;
        xG[jy][d] = T.Gx[qx][0] * f0 + T.Gx[qx][1] * f1 + T.Gx[qx][2] * f2;
      }
    double Pa[3][2] = {{0, 0}, {0, 0}, {0, 0}}, Qa[3][2] = {{0, 0}, {0, 0}, {0, 0}};
    const double wxT = T.w[qx] * WT;
    // pressure along the column: dp(qy) = w_qy pA + wyh_qy pB
    const double pA = wxT * (P[0] + P[1] * T.xh[qx]), pB = wxT * P[2];
    double dv0 = 0.0, dv1 = 0.0;
    const int qxn = qx < 3 ? qx + 1 : 3;
#pragma unroll
    for (int qy = 0; qy < 4; ++qy) {
      // the next point's coefficients fly while this point is evaluated
      double nxt[6];
      const double* np = qy < 3 ? cp + (qx * 24 + qy + 1) * JNT : cp + (qxn * 24) * JNT;
#pragma unroll
      for (int k = 0; k < 6; ++k) nxt[k] = (k >= 1 && k <= 3 && !HG) ? 0.0 : __ldg(np + (k * 4) * JNT);
      if ((qy & 1) == 0) apc_prefetch_l2(cp, 2 * qx + (qy >> 1) + PDST_PF_AHEAD, HG);
      {
        double u[2], ux[2], uy[2];
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          u[d] = T.B[qy][0] * xB[0][d] + T.B[qy][1] * xB[1][d] + T.B[qy][2] * xB[2][d];
          ux[d] = T.B[qy][0] * xG[0][d] + T.B[qy][1] * xG[1][d] + T.B[qy][2] * xG[2][d];
          uy[d] = T.Gy[qy][0] * xB[0][d] + T.Gy[qy][1] * xB[1][d] + T.Gy[qy][2] * xB[2][d];
        }
        const double ce = cur[0], ca0 = cur[1], ca1 = cur[2], ca2 = cur[3], cv0 = cur[4], cv1 = cur[5];
        // wq T(B) with B = sym grad u (b0, b1, b2 = cc / 2)
        const double b0 = ux[0], b1 = uy[1], cc = uy[0] + ux[1];
        const double t = ca0 * b0 + ca1 * b1 + ca2 * cc;
        double F00 = ce * b0 - t * ca0;
        double F11 = ce * b1 - t * ca1;
        double F01 = ce * (0.5 * cc) - t * ca2;
        // - wq (u (x) v + v (x) u)
        F00 -= 2.0 * u[0] * cv0;
        F11 -= 2.0 * u[1] * cv1;
        F01 -= u[1] * cv0 + u[0] * cv1;
        if (ds.pressure) {
          const double dp = T.w[qy] * pA + T.wyh[qy] * pB;
          F00 -= dp;
          F11 -= dp;
          const double div = ux[0] + uy[1];
          dv0 = fma(T.w[qy], div, dv0);
          dv1 = fma(T.wyh[qy], div, dv1);
        }
#pragma unroll
        for (int jy = 0; jy < 3; ++jy) {
          Pa[jy][0] = fma(F00, T.B[qy][jy], Pa[jy][0]);
          Pa[jy][1] = fma(F01, T.B[qy][jy], Pa[jy][1]);
          Qa[jy][0] = fma(F01, T.Gy[qy][jy], Qa[jy][0]);
          Qa[jy][1] = fma(F11, T.Gy[qy][jy], Qa[jy][1]);
        }
      }
#pragma unroll
      for (int k = 0; k < 6; ++k) cur[k] = nxt[k];
    }
'''
s = s[:a] + new + s[b:]
open(p, "w").write(s)
