// Compact pair-block records (PB_STRIDE doubles per active pair):
//   [0, 24)  gradient g24 in the reference's 24 affine DOFs (two bodies x 12)
//   [24]     type: 0 = contact, 5 columns   H24 = Q M5 Q^T, Q = [ch (x) e_a | fq0 | fq1]
//                  1 = contact, 9 columns   H24 = (Qx (x) I3) M9 (Qx (x) I3)^T   (mollified EE)
//                  2 = friction             H24 = G^T Hu G, G = [G0; G1] (2 x 24), Hu 2x2
//   [25, ..) payload  type 0: ch[8] | fq0[24] | fq1[24] | M5[5][5]
//                     type 1: Qx[8][3] | M9[9][9]
//                     type 2: G0[24] | G1[24] | h00 h01 h11  (kinematic-side columns zero)
// Entries are evaluated on demand (system reduction, dense readout) with the same
// operation order as the dense expansion they replace (abd_contact.cuh,
// abd_misc.cuh friction_blocks_dev), 3.4x fewer bytes written and re-read.
#pragma once
#include "abd_math.cuh"

namespace abd {

// reference DOF d (0..11) of a body -> 24-space index in the affine ordering
// sj * 3 + a (sj = 4 side + j, j = 0 translation / 1..3 rest coordinate)
ABD_D int pb_rho(int side, int d) {
  const int j = d < 3 ? 0 : 1 + (d - 3) % 3;
  const int a = d < 3 ? d : (d - 3) / 3;
  return (4 * side + j) * 3 + a;
}

// H24 entry at reference indices R = 12 side_r + d_r, C = 12 side_c + d_c
ABD_D double pb_entry(const double* __restrict__ rec, int R, int C) {
  const int type = (int)rec[24];
  if (type == 2) {
    const double* G0 = rec + 25;
    const double* G1 = rec + 49;
    const double h00 = rec[73], h01 = rec[74], h11 = rec[75];
    const double t0 = h00 * G0[R] + h01 * G1[R];
    const double t1 = h01 * G0[R] + h11 * G1[R];
    return t0 * G0[C] + t1 * G1[C];
  }
  int rho = pb_rho(R / 12, R % 12), sg = pb_rho(C / 12, C % 12);
  if (sg < rho) {
    const int t = rho;
    rho = sg;
    sg = t;
  }
  const int sj = rho / 3, a = rho % 3, tl = sg / 3, b = sg % 3;
  if (type == 0) {
    const double* ch = rec + 25;
    const double* f0 = rec + 33;
    const double* f1 = rec + 57;
    const double* M = rec + 81;
    const double ub = ch[sj] * M[5 * a + b] + f0[rho] * M[15 + b] + f1[rho] * M[20 + b];
    const double u3 = ch[sj] * M[5 * a + 3] + f0[rho] * M[15 + 3] + f1[rho] * M[20 + 3];
    const double u4 = ch[sj] * M[5 * a + 4] + f0[rho] * M[15 + 4] + f1[rho] * M[20 + 4];
    return ub * ch[tl] + u3 * f0[sg] + u4 * f1[sg];
  }
  const double* Q = rec + 25;
  const double* M = rec + 49;
  double u[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int c = 3 * k + b;
    u[k] = Q[3 * sj] * M[9 * a + c] + Q[3 * sj + 1] * M[9 * (3 + a) + c] + Q[3 * sj + 2] * M[9 * (6 + a) + c];
  }
  return u[0] * Q[3 * tl] + u[1] * Q[3 * tl + 1] + u[2] * Q[3 * tl + 2];
}

}  // namespace abd
