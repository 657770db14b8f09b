// numerics.cuh -- the arithmetic contract shared by the host symbolic phase and
// every sm_100a kernel.  Compiled with --fmad=false (device) and
// -ffp-contract=off (host) so that only the fma() calls written here fuse; the
// oracle (oracle/oracle.c) restates the same operation sequences, which makes
// GPU and CPU results bit-identical rather than merely close.
#pragma once

#include <cmath>

#ifdef __CUDACC__
#define GB_HD __host__ __device__ __forceinline__
#else
#define GB_HD inline
#endif

namespace gbnr {

// sin/cos by Cody-Waite reduction with a 3-part pi/2 and the fdlibm minimax
// kernels on [-pi/4, pi/4] (Horner in explicit fma).
GB_HD void gb_sincos(double x, double* s_out, double* c_out) {
    const double two_over_pi = 6.36619772367581382433e-01;
    const double p1 = 1.57079632679489655800e+00;
    const double p2 = 6.12323399573676603587e-17;
    const double p3 = -1.49738490485916983248e-33;
    double q = rint(x * two_over_pi);
    double r = fma(-q, p1, x);
    r = fma(-q, p2, r);
    r = fma(-q, p3, r);
    double z = r * r;
    double ps = fma(z, 1.58969099521155010221e-10, -2.50507602534068634195e-08);
    ps = fma(z, ps, 2.75573137070700676789e-06);
    ps = fma(z, ps, -1.98412698298579493134e-04);
    ps = fma(z, ps, 8.33333333332248946124e-03);
    ps = fma(z, ps, -1.66666666666666324348e-01);
    double sn = fma(r * z, ps, r);
    double pc = fma(z, -1.13596475577881948265e-11, 2.08757232129817482790e-09);
    pc = fma(z, pc, -2.75573143513906633035e-07);
    pc = fma(z, pc, 2.48015872894767294178e-05);
    pc = fma(z, pc, -1.38888888888741095749e-03);
    pc = fma(z, pc, 4.16666666666666019037e-02);
    double cs = fma(z * z, pc, fma(-0.5, z, 1.0));
    double qm = q - 4.0 * floor(q * 0.25);
    if (qm == 0.0) {
        *s_out = sn; *c_out = cs;
    } else if (qm == 1.0) {
        *s_out = cs; *c_out = -sn;
    } else if (qm == 2.0) {
        *s_out = -sn; *c_out = -cs;
    } else if (qm == 3.0) {
        *s_out = -cs; *c_out = sn;
    } else {
        *s_out = x - x; *c_out = x - x;
    }
}

// One Ybus term of the current injection: I += Y_rk * V_k.
GB_HD void acc_current(double g, double b, double vre, double vim, double& ire, double& iim) {
    ire = fma(g, vre, ire);
    ire = fma(-b, vim, ire);
    iim = fma(g, vim, iim);
    iim = fma(b, vre, iim);
}

// Calculated injection S = V conj(I).
GB_HD void injection(double vre, double vim, double ire, double iim, double& P, double& Q) {
    P = fma(vre, ire, vim * iim);
    Q = fma(vim, ire, -(vre * iim));
}

// Z = V_r conj(Y_rk e^{j th_k}); dS/d|V_k| = Z, dS/dth_k = -j |V_k| ... (App. B).
GB_HD void jac_z(double g, double b, double vre_r, double vim_r, double ck, double sk,
                 double& zre, double& zim) {
    double yer = fma(g, ck, -(b * sk));
    double yei = fma(g, sk, b * ck);
    zre = fma(vre_r, yer, vim_r * yei);
    zim = fma(vim_r, yer, -(vre_r * yei));
}

// The four Jacobian entries of Ybus slot (r, k): {dP/dth_k, dP/d|V_k|, dQ/dth_k, dQ/d|V_k|}.
GB_HD void jac_entries(bool diag, double zre, double zim, double vmk, double ck, double sk,
                       double ire, double iim, double P, double Q, double* j) {
    if (!diag) {
        j[0] = vmk * zim;
        j[1] = zre;
        j[2] = -(vmk * zre);
        j[3] = zim;
    } else {
        j[0] = fma(vmk, zim, -Q);
        j[1] = zre + fma(ire, ck, iim * sk);
        j[2] = fma(-vmk, zre, P);
        j[3] = zim + fma(ire, sk, -(iim * ck));
    }
}

// Branch flow S = V_a conj(Y_a V_f + Y_b V_t) of one branch end.
GB_HD void branch_end_flow(double ar, double ai, double br, double bi, double vfr, double vfi, double vtr,
                           double vti, double var, double vai, double& P, double& Q) {
    double ire = 0.0, iim = 0.0;
    acc_current(ar, ai, vfr, vfi, ire, iim);
    acc_current(br, bi, vtr, vti, ire, iim);
    injection(var, vai, ire, iim, P, Q);
}

}  // namespace gbnr
