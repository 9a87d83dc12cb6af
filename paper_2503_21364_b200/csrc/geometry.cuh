// fp64 projection geometry shared by K1 (preprocess.cu) and the backward
// (backward.cu).  Both translation units are compiled with -fmad=false, so
// every operation rounds exactly where the reference's torch ops do: the
// products torch hands to MKL dgemm (means @ r_wc.T, j @ r_wc) are written as
// the FMA chain MKL evaluates, the bmm products as plain sequential sums.
#pragma once

#include "lmgs_internal.cuh"

namespace lmgs {

__device__ __forceinline__ double mkl_dot3(double a0, double b0, double a1, double b1, double a2,
                                           double b2) {
  return fma(a2, b2, fma(a1, b1, a0 * b0));
}
__device__ __forceinline__ double bmm_dot3(double a0, double b0, double a1, double b1, double a2,
                                           double b2) {
  return (a0 * b0 + a1 * b1) + a2 * b2;
}

// The world-space covariance of a Gaussian, view-independent: quat_to_rotmat
// (93-102) and covariance_3d (105-117) op for op.  S = {S00, S01, S02, S11,
// S12, S22}: the bmm's S10 / S20 / S21 are the same products in the same
// order as S01 / S02 / S12 (fp64 multiplication commutes), so equal bits.
__device__ __forceinline__ void covariance_3d(float4 q, double s0, double s1, double s2,
                                              double S[6]) {
  // quat_to_rotmat (93-102)
  const double qw = q.x, qx = q.y, qy = q.z, qz = q.w;
  const double nr = sqrt(((qw * qw + qx * qx) + qy * qy) + qz * qz);
  const double w = qw / nr, X = qx / nr, Y = qy / nr, Z = qz / nr;
  const double r00 = 1 - 2 * (Y * Y + Z * Z), r01 = 2 * (X * Y - w * Z),
               r02 = 2 * (X * Z + w * Y);
  const double r10 = 2 * (X * Y + w * Z), r11 = 1 - 2 * (X * X + Z * Z),
               r12 = 2 * (Y * Z - w * X);
  const double r20 = 2 * (X * Z - w * Y), r21 = 2 * (Y * Z + w * X),
               r22 = 1 - 2 * (X * X + Y * Y);
  // covariance_3d (105-117): M = R * s[None,:], Sigma = M M^T
  const double M00 = r00 * s0, M01 = r01 * s1, M02 = r02 * s2;
  const double M10 = r10 * s0, M11 = r11 * s1, M12 = r12 * s2;
  const double M20 = r20 * s0, M21 = r21 * s1, M22 = r22 * s2;
  S[0] = bmm_dot3(M00, M00, M01, M01, M02, M02);
  S[1] = bmm_dot3(M00, M10, M01, M11, M02, M12);
  S[2] = bmm_dot3(M00, M20, M01, M21, M02, M22);
  S[3] = bmm_dot3(M10, M10, M11, M11, M12, M12);
  S[4] = bmm_dot3(M10, M20, M11, M21, M12, M22);
  S[5] = bmm_dot3(M20, M20, M21, M21, M22, M22);
}

// Camera-space point (x, y, z) of a near-kept Gaussian and its world
// covariance -> mean2d, cov2d (incl. the 0.3 floor) and radius, in fp64, op
// for op as the reference (project_splats 199-225).
__device__ __forceinline__ void splat_projection(const CamArgs& cam, double x, double y, double z,
                                                 const double S[6], double* mx, double* my,
                                                 double* ca_out, double* cb_out, double* cc_out,
                                                 double* radius) {
  *mx = cam.fx * x / z + cam.cx;  // 201
  *my = cam.fy * y / z + cam.cy;
  const double S00 = S[0], S01 = S[1], S02 = S[2], S11 = S[3], S12 = S[4], S22 = S[5];
  const double S10 = S01, S20 = S02, S21 = S12;
  // clamped Jacobian (205-218); `fx / z` is torch's reciprocal(z) * fx
  const double tx = fmin(fmax(x / z, -cam.lim_x), cam.lim_x) * z;
  const double ty = fmin(fmax(y / z, -cam.lim_y), cam.lim_y) * z;
  const double rz = 1.0 / z;
  const double zz = z * z;
  const double J00 = rz * cam.fx, J02 = -cam.fx * tx / zz;
  const double J11 = rz * cam.fy, J12 = -cam.fy * ty / zz;
  // jw = j @ r_wc (219): MKL FMA chain over (J0k, 0, J2k) rows incl. the zeros
  const double W00 = mkl_dot3(J00, cam.r[0], 0.0, cam.r[3], J02, cam.r[6]);
  const double W01 = mkl_dot3(J00, cam.r[1], 0.0, cam.r[4], J02, cam.r[7]);
  const double W02 = mkl_dot3(J00, cam.r[2], 0.0, cam.r[5], J02, cam.r[8]);
  const double W10 = mkl_dot3(0.0, cam.r[0], J11, cam.r[3], J12, cam.r[6]);
  const double W11 = mkl_dot3(0.0, cam.r[1], J11, cam.r[4], J12, cam.r[7]);
  const double W12 = mkl_dot3(0.0, cam.r[2], J11, cam.r[5], J12, cam.r[8]);
  // cov2d = (jw @ cov3d) @ jw^T + 0.3 I (220-221)
  const double T00 = bmm_dot3(W00, S00, W01, S10, W02, S20);
  const double T01 = bmm_dot3(W00, S01, W01, S11, W02, S21);
  const double T02 = bmm_dot3(W00, S02, W01, S12, W02, S22);
  const double T10 = bmm_dot3(W10, S00, W11, S10, W12, S20);
  const double T11 = bmm_dot3(W10, S01, W11, S11, W12, S21);
  const double T12 = bmm_dot3(W10, S02, W11, S12, W12, S22);
  const double ca = bmm_dot3(T00, W00, T01, W01, T02, W02) + kCov2dReg;
  const double cb = bmm_dot3(T00, W10, T01, W11, T02, W12);  // cov2d[0,1]
  const double cc = bmm_dot3(T10, W10, T11, W11, T12, W12) + kCov2dReg;
  *ca_out = ca;
  *cb_out = cb;
  *cc_out = cc;
  // lam_max / radius (223-225)
  const double h = 0.5 * (ca - cc);
  const double lam = 0.5 * (ca + cc) + sqrt(h * h + cb * cb);
  *radius = 3.0 * sqrt(lam);
}

// Both of the above (K1 and the exact replays share these bit-identical values).
__device__ __forceinline__ void splat_geometry(const CamArgs& cam, double x, double y, double z,
                                               float4 q, double s0, double s1, double s2,
                                               double* mx, double* my, double* ca_out,
                                               double* cb_out, double* cc_out, double* radius) {
  double S[6];
  covariance_3d(q, s0, s1, s2, S);
  splat_projection(cam, x, y, z, S, mx, my, ca_out, cb_out, cc_out, radius);
}

}  // namespace lmgs
