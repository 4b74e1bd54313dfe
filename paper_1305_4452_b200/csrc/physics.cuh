// physics.cuh -- pointwise integrands of the four built-in physics,
// written as residual coefficients r_(k,i) and Jacobian coefficients D_(k,i),(k2,j) over
// SPATIAL basis kinds k in {N, dN/dx_0..dN/dx_{d-1}, lap N}:
//
//     R_(A,i)        = sum_q sum_k     B_k(A,q) r_(k,i)(q)            dV_q
//     J_(A,i),(B,j)  = sum_q sum_{k,k2} B_k(A,q) D_(k,i),(k2,j)(q) B_k2(B,q)  dV_q
//
// with J = a dR/dUdot + b dR/dU (A-16).  The paper leaves the integrand to the user
// (P:576-579); these are this build's closed set.  This is the GPU side's own derivation: the
// coefficient form below is NOT how the oracle computes its entries (it linearises per (A,B)).
//
// Each physics provides
//   NK<DIM>            number of spatial kinds it uses (1+DIM, or 2+DIM with the Laplacian)
//   HESS               whether the Laplacian kind is used (needs Hessians)
//   dmask(k,i,k2,j)    constexpr structural nonzero pattern of D (zeros are never stored)
//   rmask(k,i)         constexpr structural nonzero pattern of r
//   prepare(...)       per-point state from the fields
//   residual(st, r)    r_(k,i)
//   dcol(st, k2, j, a, b, col)  the column D_(:,:),(k2,j)
#pragma once
#include <cmath>

namespace iga {

template <int DIM, int M>
struct Fields {
    double u[M], gu[M][DIM], lu[M], ut[M];   // u, grad u, lap u, udot at the point
    double x[DIM];                            // physical point
    double dxi[DIM][DIM];                     // xi_{alpha,i}
    double hpar[DIM];                         // parametric element lengths
};

// ------------------------------------------------------------------------------------------
// LAPLACE (configs 1, 2):  R_A = kappa gradN.grad u + sigma N u - N f;  J = b(kappa gradN.gradN + sigma N N)
// ------------------------------------------------------------------------------------------
struct PhysLaplace {
    static constexpr int M = 1;
    static constexpr bool HESS = false;
    static constexpr bool UDOT = false;       // residual depends on the time derivative
    template <int DIM> static constexpr int NK() { return 1 + DIM; }
    template <int DIM> static constexpr bool dmask(int k, int i, int k2, int j) { return k == k2 && i == 0 && j == 0; }
    static constexpr bool rmask(int k, int i) { return i == 0; }
    template <int DIM>
    struct State { double kap, sig, f, u, gu[DIM]; };
    template <int DIM>
    __device__ static inline void prepare(const double *p, const Fields<DIM, 1> &F, State<DIM> &s) {
        s.kap = p[0];
        s.sig = p[1];
        s.f = 0.0;
        if (p[2] == 1.0 && DIM >= 2) {
            const double pi = 3.14159265358979323846;
            s.f = 2.0 * pi * pi * sin(pi * F.x[0]) * sin(pi * F.x[DIM >= 2 ? 1 : 0]);
        }
        s.u = F.u[0];
#pragma unroll
        for (int i = 0; i < DIM; i++) s.gu[i] = F.gu[0][i];
    }
    template <int DIM>
    __device__ static inline void residual(const State<DIM> &s, double *r) {
        r[0] = s.sig * s.u - s.f;
#pragma unroll
        for (int i = 0; i < DIM; i++) r[1 + i] = s.kap * s.gu[i];
    }
    template <int DIM>
    __device__ static inline void dcol(const State<DIM> &s, int k2, int j, double a, double b, double *col) {
#pragma unroll
        for (int k = 0; k < 1 + DIM; k++) col[k] = 0.0;
        col[k2] = b * (k2 == 0 ? s.sig : s.kap);
    }
};

// ------------------------------------------------------------------------------------------
// CAHN_HILLIARD (config 3), readings A-10/A-11:  M = c(1-c), mu' = 3 alpha (1/(2 theta c(1-c)) - 2)
//   R_A = N cdot + (M mu' + M' lap c) gradN.grad c + M lap c lapN
// kinds: 0 = N, 1..DIM = d/dx_i, DIM+1 = lap
// ------------------------------------------------------------------------------------------
struct PhysCahnHilliard {
    static constexpr int M = 1;
    static constexpr bool HESS = true;
    static constexpr bool UDOT = true;       // residual depends on the time derivative
    template <int DIM> static constexpr int NK() { return 2 + DIM; }
    // structural D for DIM up to 3 (kinds: 0 N, 1..3 grad, last lap); lap index passed as L
    static constexpr bool dmask_d(int k, int k2, int L) {
        const bool kN = k == 0, kG = k >= 1 && k < L, kL = k == L;
        const bool sN = k2 == 0, sG = k2 >= 1 && k2 < L, sL = k2 == L;
        return (kN && sN) || (kG && sN) || (kL && sN) || (kG && sG && k == k2) || (kG && sL) || (kL && sL);
    }
    template <int DIM> static constexpr bool dmask(int k, int i, int k2, int j) { return dmask_d(k, k2, 1 + DIM); }
    static constexpr bool rmask(int k, int i) { return true; }
    template <int DIM>
    struct State { double a, M, Mp, Mpp, mup, mupp, lc, gc[DIM], ut; };
    template <int DIM>
    __device__ static inline void prepare(const double *p, const Fields<DIM, 1> &F, State<DIM> &s) {
        const double th = p[0], al = p[1];
        const double c = F.u[0];
        const double omc = 1.0 - c;
        s.M = c * omc;
        s.Mp = 1.0 - 2.0 * c;
        s.Mpp = -2.0;
        const double inv = 1.0 / (2.0 * th * s.M);
        s.mup = 3.0 * al * (inv - 2.0);
        s.mupp = -3.0 * al * s.Mp * inv / s.M;      // 3 alpha (2c-1) / (2 theta c^2 (1-c)^2)
        s.lc = F.lu[0];
#pragma unroll
        for (int i = 0; i < DIM; i++) s.gc[i] = F.gu[0][i];
        s.ut = F.ut[0];
    }
    template <int DIM>
    __device__ static inline void residual(const State<DIM> &s, double *r) {
        r[0] = s.ut;
        const double g = s.M * s.mup + s.Mp * s.lc;
#pragma unroll
        for (int i = 0; i < DIM; i++) r[1 + i] = g * s.gc[i];
        r[1 + DIM] = s.M * s.lc;
    }
    template <int DIM>
    __device__ static inline void dcol(const State<DIM> &s, int k2, int j, double a, double b, double *col) {
#pragma unroll
        for (int k = 0; k < 2 + DIM; k++) col[k] = 0.0;
        if (k2 == 0) {                      // trial kind N
            col[0] = a;
            const double g = b * (s.Mp * s.mup + s.M * s.mupp + s.Mpp * s.lc);
#pragma unroll
            for (int i = 0; i < DIM; i++) col[1 + i] = g * s.gc[i];
            col[1 + DIM] = b * s.Mp * s.lc;
        } else if (k2 <= DIM) {             // trial kind d/dx_l
            col[k2] = b * (s.M * s.mup + s.Mp * s.lc);
        } else {                            // trial kind lap
#pragma unroll
            for (int i = 0; i < DIM; i++) col[1 + i] = b * s.Mp * s.gc[i];
            col[1 + DIM] = b * s.M;
        }
    }
};

// ------------------------------------------------------------------------------------------
// NEOHOOKE (config 4), readings A-12/A-13, total Lagrangian on the parametric cube.
//   P = lambda/2 (J^2-1) F^{-T} + mu (F - F^{-T})
//   AA_aIbJ = delta_ab S_IJ + lambda J^2 Fi_Ia Fi_Jb + c2 (delta_ab Ci_IJ + Fi_Ja Fi_Ib),
//   c2 = mu - lambda (J^2-1)/2,  Fi = F^{-1},  Ci = Fi Fi^T   (the push of C_IJKL through F)
// kinds: 0 = N (unused), 1..3 = d/dX_I;  components a = 0..2
// ------------------------------------------------------------------------------------------
struct PhysNeoHooke {
    static constexpr int M = 3;
    static constexpr bool HESS = false;
    static constexpr bool UDOT = false;       // residual depends on the time derivative
    template <int DIM> static constexpr int NK() { return 1 + DIM; }
    template <int DIM> static constexpr bool dmask(int k, int i, int k2, int j) { return k >= 1 && k2 >= 1; }
    static constexpr bool rmask(int k, int i) { return k >= 1; }
    template <int DIM>
    struct State { double P[3][3], S[3][3], Fi[3][3], Ci[3][3], lJ2, c2; };
    template <int DIM>
    __device__ static inline void prepare(const double *p, const Fields<DIM, 3> &F, State<DIM> &s) {
        static_assert(DIM == 3, "NEOHOOKE is 3D");
        const double lam = p[0], mu = p[1];
        double Fm[3][3];
#pragma unroll
        for (int a = 0; a < 3; a++)
#pragma unroll
            for (int I = 0; I < 3; I++) Fm[a][I] = (a == I ? 1.0 : 0.0) + F.gu[a][I];
        const double c00 = Fm[1][1] * Fm[2][2] - Fm[1][2] * Fm[2][1];
        const double c01 = Fm[1][2] * Fm[2][0] - Fm[1][0] * Fm[2][2];
        const double c02 = Fm[1][0] * Fm[2][1] - Fm[1][1] * Fm[2][0];
        const double J = Fm[0][0] * c00 + Fm[0][1] * c01 + Fm[0][2] * c02;
        const double iJ = 1.0 / J;
        // Fi = adj(F)/J, Fi[I][a]
        s.Fi[0][0] = c00 * iJ;
        s.Fi[1][0] = c01 * iJ;
        s.Fi[2][0] = c02 * iJ;
        s.Fi[0][1] = (Fm[0][2] * Fm[2][1] - Fm[0][1] * Fm[2][2]) * iJ;
        s.Fi[1][1] = (Fm[0][0] * Fm[2][2] - Fm[0][2] * Fm[2][0]) * iJ;
        s.Fi[2][1] = (Fm[0][1] * Fm[2][0] - Fm[0][0] * Fm[2][1]) * iJ;
        s.Fi[0][2] = (Fm[0][1] * Fm[1][2] - Fm[0][2] * Fm[1][1]) * iJ;
        s.Fi[1][2] = (Fm[0][2] * Fm[1][0] - Fm[0][0] * Fm[1][2]) * iJ;
        s.Fi[2][2] = (Fm[0][0] * Fm[1][1] - Fm[0][1] * Fm[1][0]) * iJ;
#pragma unroll
        for (int I = 0; I < 3; I++)
#pragma unroll
            for (int J2 = 0; J2 < 3; J2++)
                s.Ci[I][J2] = s.Fi[I][0] * s.Fi[J2][0] + s.Fi[I][1] * s.Fi[J2][1] + s.Fi[I][2] * s.Fi[J2][2];
        const double h = 0.5 * lam * (J * J - 1.0);
        s.lJ2 = lam * J * J;
        s.c2 = mu - h;
#pragma unroll
        for (int I = 0; I < 3; I++)
#pragma unroll
            for (int J2 = 0; J2 < 3; J2++) s.S[I][J2] = h * s.Ci[I][J2] + mu * ((I == J2 ? 1.0 : 0.0) - s.Ci[I][J2]);
#pragma unroll
        for (int a = 0; a < 3; a++)
#pragma unroll
            for (int I = 0; I < 3; I++) s.P[a][I] = h * s.Fi[I][a] + mu * (Fm[a][I] - s.Fi[I][a]);
    }
    template <int DIM>
    __device__ static inline void residual(const State<DIM> &s, double *r) {
        // r[(k)*M + a]: k = 0 (N) unused, k = 1+I
#pragma unroll
        for (int a = 0; a < 3; a++) r[a] = 0.0;
#pragma unroll
        for (int I = 0; I < 3; I++)
#pragma unroll
            for (int a = 0; a < 3; a++) r[(1 + I) * 3 + a] = s.P[a][I];
    }
    template <int DIM>
    __device__ static inline void dcol(const State<DIM> &s, int k2, int bb, double a, double b, double *col) {
#pragma unroll
        for (int t = 0; t < 12; t++) col[t] = 0.0;
        if (k2 == 0) return;
        const int J = k2 - 1;
#pragma unroll
        for (int I = 0; I < 3; I++)
#pragma unroll
            for (int aa = 0; aa < 3; aa++) {
                double v = s.lJ2 * s.Fi[I][aa] * s.Fi[J][bb] + s.c2 * s.Fi[J][aa] * s.Fi[I][bb];
                if (aa == bb) v += s.S[I][J] + s.c2 * s.Ci[I][J];
                col[(1 + I) * 3 + aa] = b * v;
            }
    }
};

// ------------------------------------------------------------------------------------------
// NS_VMS (config 5), residual-based VMS (readings A-14/A-15), parametric geometry.
//   r_M = udot + (u.grad) u + grad p - nu lap u,  r_C = div u,  u' = -tau_M r_M,  p' = -tau_C r_C
//   R^M_(A,i) = N [udot_i + u'_k u_i,k] + N_,k [-u_k u_i + nu(u_i,k + u_k,i) - d_ik (p + p')
//                                                - u_k u'_i - u'_i u'_k]
//   R^C_A     = N div u - N_,k u'_k
// Jacobian with tau frozen: the column (k2, j) is the derivative of r along the trial direction
// "kind k2 of component j", weighted a for the Udot part and b for the U part.
// kinds: 0 = N, 1..3 = d/dx_k, 4 = lap;  components 0..2 velocity, 3 pressure.
// ------------------------------------------------------------------------------------------
struct PhysNSVMS {
    static constexpr int M = 4;
    static constexpr bool HESS = true;
    static constexpr bool UDOT = true;       // residual depends on the time derivative
    template <int DIM> static constexpr int NK() { return 5; }
    // exact structural pattern (derived in DESIGN.md; 192 entries)
    template <int DIM> static constexpr bool dmask(int k, int i, int k2, int j) {
        if (k == 4) return false;                       // no lap test kind
        const bool tN = k == 0;
        const int kk = k - 1;                           // test derivative direction (if !tN)
        if (j < 3) {
            if (k2 == 0) {                              // velocity N (udot and u directions)
                if (i < 3) return true;                 // N,i and d_k,i
                return !tN;                             // d_k,3 = -du'_k ; N,3 = 0
            }
            if (k2 == 4) {                              // velocity lap
                if (i < 3) return tN ? true : (i == j || kk == j);
                return !tN && kk == j;
            }
            const int l = k2 - 1;                       // velocity d_l
            if (i < 3) {
                if (tN) return true;
                return i == j || kk == j || (l == j && i == kk);
            }
            return tN ? (l == j) : (kk == j);
        }
        // pressure trial
        if (k2 == 0) return !tN && i < 3 && kk == i;    // -d_ik dp
        if (k2 == 4) return false;
        const int l = k2 - 1;
        if (i < 3) return tN ? true : (i == l || kk == l);
        return !tN && kk == l;
    }
    static constexpr bool rmask(int k, int i) { return k < 4; }
    template <int DIM>
    struct State {
        double u[3], gu[3][3], up[3], tauM, tauC, nu;   // read by dcol (the first JSTATE doubles)
        double rN[4], rG[3][4];                          // residual coefficients only
    };
    static constexpr int JSTATE = 18;
    template <int DIM>
    __device__ static inline void prepare(const double *p, const Fields<DIM, 4> &F, State<DIM> &s) {
        static_assert(DIM == 3, "NS_VMS is 3D");
        const double nu = p[0], dt = p[1], Ct = p[2], CI = p[3];
        s.nu = nu;
        // metric of the parent-element map: dxihat_k/dx_i = (2/h_k) xi_{k,i}
        double Dm[3][3];
#pragma unroll
        for (int k = 0; k < 3; k++)
#pragma unroll
            for (int i = 0; i < 3; i++) Dm[k][i] = 2.0 / F.hpar[k] * F.dxi[k][i];
        double G[3][3], g[3];
#pragma unroll
        for (int i = 0; i < 3; i++) {
            g[i] = Dm[0][i] + Dm[1][i] + Dm[2][i];
#pragma unroll
            for (int j = 0; j < 3; j++) G[i][j] = Dm[0][i] * Dm[0][j] + Dm[1][i] * Dm[1][j] + Dm[2][i] * Dm[2][j];
        }
        double uGu = 0.0, GG = 0.0;
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
            for (int j = 0; j < 3; j++) {
                uGu += F.u[i] * G[i][j] * F.u[j];
                GG += G[i][j] * G[i][j];
            }
        const double gg = g[0] * g[0] + g[1] * g[1] + g[2] * g[2];
        s.tauM = rsqrt(Ct / (dt * dt) + uGu + CI * nu * nu * GG);
        s.tauC = 1.0 / (s.tauM * gg);
#pragma unroll
        for (int i = 0; i < 3; i++) {
            s.u[i] = F.u[i];
#pragma unroll
            for (int k = 0; k < 3; k++) s.gu[i][k] = F.gu[i][k];
        }
        double rM[3];
#pragma unroll
        for (int i = 0; i < 3; i++)
            rM[i] = F.ut[i] + F.u[0] * F.gu[i][0] + F.u[1] * F.gu[i][1] + F.u[2] * F.gu[i][2] + F.gu[3][i] - nu * F.lu[i];
        const double rC = F.gu[0][0] + F.gu[1][1] + F.gu[2][2];
#pragma unroll
        for (int i = 0; i < 3; i++) s.up[i] = -s.tauM * rM[i];
        const double pp = -s.tauC * rC;
        // residual coefficients
#pragma unroll
        for (int i = 0; i < 3; i++) {
            s.rN[i] = F.ut[i] + s.up[0] * F.gu[i][0] + s.up[1] * F.gu[i][1] + s.up[2] * F.gu[i][2];
#pragma unroll
            for (int k = 0; k < 3; k++) {
                double v = -F.u[k] * F.u[i] + nu * (F.gu[i][k] + F.gu[k][i]) - F.u[k] * s.up[i] - s.up[i] * s.up[k];
                if (i == k) v -= F.u[3] + pp;
                s.rG[k][i] = v;
            }
        }
        s.rN[3] = rC;
#pragma unroll
        for (int k = 0; k < 3; k++) s.rG[k][3] = -s.up[k];
    }
    template <int DIM>
    __device__ static inline void residual(const State<DIM> &s, double *r) {
#pragma unroll
        for (int i = 0; i < 4; i++) r[i] = s.rN[i];
#pragma unroll
        for (int k = 0; k < 3; k++)
#pragma unroll
            for (int i = 0; i < 4; i++) r[(1 + k) * 4 + i] = s.rG[k][i];
#pragma unroll
        for (int i = 0; i < 4; i++) r[16 + i] = 0.0;
    }
    template <int DIM>
    __device__ static inline void dcol(const State<DIM> &s, int k2, int j, double a, double b, double *col) {
        // trial direction
        double dut[3] = {0, 0, 0}, du[3] = {0, 0, 0}, dgu[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        double dlu[3] = {0, 0, 0}, dp = 0.0, dgp[3] = {0, 0, 0};
        if (j < 3) {
            if (k2 == 0) { dut[j] = a; du[j] = b; }
            else if (k2 <= 3) dgu[j][k2 - 1] = b;
            else dlu[j] = b;
        } else {
            if (k2 == 0) dp = b;
            else if (k2 <= 3) dgp[k2 - 1] = b;
        }
        dcol_dir<DIM>(s, dut, du, dgu, dlu, dp, dgp, col);
    }
    // the same column for a compile-time trial kind K2 and a run-time (warp-uniform) component j:
    // the direction is built with selects (no dynamically indexed register arrays), so one code copy
    // serves the four components (the FS kernel's phase 4, fused3d.cu)
    template <int DIM, int K2>
    __device__ static inline void dcol_j(const State<DIM> &s, int j, double a, double b, double *col) {
        double dut[3], du[3], dgu[3][3], dlu[3], dgp[3];
#pragma unroll
        for (int x = 0; x < 3; x++) {
            dut[x] = (K2 == 0 && j == x) ? a : 0.0;
            du[x] = (K2 == 0 && j == x) ? b : 0.0;
            dlu[x] = (K2 == 4 && j == x) ? b : 0.0;
            dgp[x] = (K2 == 1 + x && j == 3) ? b : 0.0;
#pragma unroll
            for (int y = 0; y < 3; y++) dgu[x][y] = (K2 == 1 + y && j == x) ? b : 0.0;
        }
        const double dp = (K2 == 0 && j == 3) ? b : 0.0;
        dcol_dir<DIM>(s, dut, du, dgu, dlu, dp, dgp, col);
    }
    template <int DIM>
    __device__ static inline void dcol_dir(const State<DIM> &s, const double (&dut)[3], const double (&du)[3],
                                           const double (&dgu)[3][3], const double (&dlu)[3], double dp,
                                           const double (&dgp)[3], double *col) {
        double drM[3];
#pragma unroll
        for (int i = 0; i < 3; i++)
            drM[i] = dut[i] + du[0] * s.gu[i][0] + du[1] * s.gu[i][1] + du[2] * s.gu[i][2]
                   + s.u[0] * dgu[i][0] + s.u[1] * dgu[i][1] + s.u[2] * dgu[i][2] + dgp[i] - s.nu * dlu[i];
        const double drC = dgu[0][0] + dgu[1][1] + dgu[2][2];
        double dup[3];
#pragma unroll
        for (int i = 0; i < 3; i++) dup[i] = -s.tauM * drM[i];
        const double dpp = -s.tauC * drC;
#pragma unroll
        for (int i = 0; i < 3; i++) {
            double v = dut[i];
#pragma unroll
            for (int k = 0; k < 3; k++) v += dup[k] * s.gu[i][k] + s.up[k] * dgu[i][k];
            col[i] = v;
#pragma unroll
            for (int k = 0; k < 3; k++) {
                double w = -du[k] * s.u[i] - s.u[k] * du[i] + s.nu * (dgu[i][k] + dgu[k][i])
                         - du[k] * s.up[i] - s.u[k] * dup[i] - dup[i] * s.up[k] - s.up[i] * dup[k];
                if (i == k) w -= dp + dpp;
                col[(1 + k) * 4 + i] = w;
            }
        }
        col[3] = drC;
#pragma unroll
        for (int k = 0; k < 3; k++) col[(1 + k) * 4 + 3] = -dup[k];
#pragma unroll
        for (int i = 0; i < 4; i++) col[16 + i] = 0.0;
    }
};

// ------------------------------------------------------------------------------------------
// NAVIER-STOKES-KORTEWEG (P:774-801 strong form, readings A-25..A-27):
// unknowns (rho, u_1, u_2) per node, 2D.  p = [a, b, R, theta, mu_bar, lambda_bar, lambda].
//   r_(N,0)   = rho_t                         r_(d_l,0)   = -rho u_l
//   r_(N,1+i) = rho_t u_i + rho u_{i,t}       r_(d_l,1+i) = -rho u_i u_l - p d_il + tau_il + zeta_il
//   tau  = mu_bar (grad u + grad u^T) + lambda_bar div u I,
//   zeta = lambda (rho lap rho + |grad rho|^2/2) I - lambda grad rho (x) grad rho,
//   p = R b rho theta/(b - rho) - a rho^2 (van der Waals)
// kinds: 0 = N, 1..2 = d/dx_l, 3 = lap
// ------------------------------------------------------------------------------------------
struct PhysNSK {
    static constexpr int M = 3;
    static constexpr bool HESS = true;
    static constexpr bool UDOT = true;       // residual depends on the time derivative
    template <int DIM> static constexpr int NK() { return 2 + DIM; }
    template <int DIM> static constexpr bool dmask(int k, int i, int k2, int j) {
        const int L = 1 + DIM;                       // Laplacian kind
        if (k == L) return false;                    // no Laplacian test kind
        if (k == 0) return i == 0 ? (k2 == 0 && j == 0) : (k2 == 0 && (j == 0 || j == i));
        const int l = k - 1;                         // test direction
        if (i == 0) return k2 == 0 && (j == 0 || j == 1 + l);
        const int ii = i - 1;
        if (j == 0) {                                // density trial: value, gradient, Laplacian
            if (k2 == 0) return true;
            if (k2 == L) return ii == l;
            const int m = k2 - 1;
            return ii == l || m == ii || m == l;
        }
        const int n = j - 1;                         // velocity trial
        if (k2 == 0) return n == ii || n == l;
        if (k2 == L) return false;
        const int m = k2 - 1;
        return (n == ii && m == l) || (n == l && m == ii) || (n == m && ii == l);
    }
    static constexpr bool rmask(int k, int i) { return k < 3; }
    template <int DIM>
    struct State { double rho, rt, u[2], ut[2], gr[2], gu[2][2], lr, p, dp, mub, lamb, lam; };
    template <int DIM>
    __device__ static inline void prepare(const double *p, const Fields<DIM, 3> &F, State<DIM> &s) {
        static_assert(DIM == 2, "NSK is 2D in this build");
        const double av = p[0], bv = p[1], Rg = p[2], th = p[3];
        s.mub = p[4];
        s.lamb = p[5];
        s.lam = p[6];
        s.rho = F.u[0];
        s.rt = F.ut[0];
        s.lr = F.lu[0];
#pragma unroll
        for (int i = 0; i < 2; i++) {
            s.u[i] = F.u[1 + i];
            s.ut[i] = F.ut[1 + i];
            s.gr[i] = F.gu[0][i];
#pragma unroll
            for (int l = 0; l < 2; l++) s.gu[i][l] = F.gu[1 + i][l];
        }
        const double ib = 1.0 / (bv - s.rho);
        s.p = Rg * bv * th * s.rho * ib - av * s.rho * s.rho;
        s.dp = Rg * bv * bv * th * ib * ib - 2.0 * av * s.rho;
    }
    template <int DIM>
    __device__ static inline void residual(const State<DIM> &s, double *r) {
        // r[kind * 3 + component]
        r[0] = s.rt;
#pragma unroll
        for (int i = 0; i < 2; i++) r[1 + i] = s.rt * s.u[i] + s.rho * s.ut[i];
        const double div = s.gu[0][0] + s.gu[1][1];
        const double iso = s.lam * (s.rho * s.lr + 0.5 * (s.gr[0] * s.gr[0] + s.gr[1] * s.gr[1])) - s.p + s.lamb * div;
#pragma unroll
        for (int l = 0; l < 2; l++) {
            r[(1 + l) * 3] = -s.rho * s.u[l];
#pragma unroll
            for (int i = 0; i < 2; i++)
                r[(1 + l) * 3 + 1 + i] = -s.rho * s.u[i] * s.u[l] + s.mub * (s.gu[i][l] + s.gu[l][i])
                                         - s.lam * s.gr[i] * s.gr[l] + (i == l ? iso : 0.0);
        }
#pragma unroll
        for (int i = 0; i < 3; i++) r[9 + i] = 0.0;
    }
    // column D_(:,:),(k2,j) = a d r/d(trial_t) + b d r/d(trial); trial kind k2, component j
    template <int DIM>
    __device__ static inline void dcol(const State<DIM> &s, int k2, int j, double a, double b, double *col) {
#pragma unroll
        for (int k = 0; k < 12; k++) col[k] = 0.0;
        if (j == 0) {                                          // density
            if (k2 == 0) {
                col[0] = a;                                    // d rho_t
#pragma unroll
                for (int i = 0; i < 2; i++) col[1 + i] = a * s.u[i] + b * s.ut[i];
#pragma unroll
                for (int l = 0; l < 2; l++) {
                    col[(1 + l) * 3] = -b * s.u[l];
#pragma unroll
                    for (int i = 0; i < 2; i++)
                        col[(1 + l) * 3 + 1 + i] = b * (-s.u[i] * s.u[l] + (i == l ? s.lam * s.lr - s.dp : 0.0));
                }
            } else if (k2 <= 2) {                              // d grad rho, direction m
                const int m = k2 - 1;
#pragma unroll
                for (int l = 0; l < 2; l++)
#pragma unroll
                    for (int i = 0; i < 2; i++) {
                        double v = -s.lam * ((i == m ? s.gr[l] : 0.0) + (l == m ? s.gr[i] : 0.0));
                        if (i == l) v += s.lam * s.gr[m];
                        col[(1 + l) * 3 + 1 + i] = b * v;
                    }
            } else {                                           // d lap rho
#pragma unroll
                for (int l = 0; l < 2; l++) col[(1 + l) * 3 + 1 + l] = b * s.lam * s.rho;
            }
        } else {                                               // velocity component n
            const int n = j - 1;
            if (k2 == 0) {
                col[1 + n] = a * s.rho + b * s.rt;
#pragma unroll
                for (int l = 0; l < 2; l++) {
                    if (l == n) col[(1 + l) * 3] = -b * s.rho;
#pragma unroll
                    for (int i = 0; i < 2; i++) {
                        double v = 0.0;
                        if (i == n) v -= s.rho * s.u[l];
                        if (l == n) v -= s.rho * s.u[i];
                        col[(1 + l) * 3 + 1 + i] = b * v;
                    }
                }
            } else if (k2 <= 2) {                              // d (u_n)_{,m}
                const int m = k2 - 1;
#pragma unroll
                for (int l = 0; l < 2; l++)
#pragma unroll
                    for (int i = 0; i < 2; i++) {
                        double v = 0.0;
                        if (i == n && l == m) v += s.mub;
                        if (l == n && i == m) v += s.mub;
                        if (i == l && n == m) v += s.lamb;
                        col[(1 + l) * 3 + 1 + i] = b * v;
                    }
            }
        }
    }
};

}  // namespace iga
