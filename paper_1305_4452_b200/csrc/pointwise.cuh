// pointwise.cuh -- one quadrature point of Alg. 4: tensor-product kinds from the
// 1D tables, rational basis (eqs. rational/drational/ddrational P:211-247),
// isoparametric map, its inverse and second derivatives, fields from U_e, the
// physics coefficients, and the compact lists r~ (NR) and D~ (NE) times detJ*w_q.
// Shared by the split kernels (assemble.cu) and the fused kernels (fused2d.cu, fused3d.cu).
#pragma once
#include "kinds.cuh"
#include "physics.cuh"

namespace iga {

struct Prm { double p[8]; };

__host__ __device__ constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }

// value of separable contraction kind C of local function (a0,a1,a2) from 1D tables v[d][k][a]
template <class KS, int DIM, int C, int NP1, class V>
__device__ __forceinline__ double kind_value(const V &v, const int *aa) {
    double s = 0.0;
    static_for<KS::nterms(C)>([&](auto T) {
        constexpr int t = decltype(T)::value;
        double prod = 1.0;
        static_for<DIM>([&](auto D) {
            constexpr int d = decltype(D)::value;
            prod *= v[d][KS::ord(C, t, d)][aa[d]];
        });
        s += prod;
    });
    return s;
}

// Nodes: accessor with u(A,m), ud(A,m), has_ud(), w(A), x(A,i) for the element's local functions;
// Nodes::PREMUL = the accessor returns w_A u, w_A udot, w_A x (homogeneous coordinates, staged once).
// Returns error bits (1: detJ <= 0, 2: non-finite).
// PRE: the caller already formed the homogeneous sums of the point (fused2d: sum factorised over
// the element's lane group) and passes them in `pre` = [W: NC][X: DIM x NC][Phi: M x NC][Phit: M];
// the per-function loop is skipped.
template <int DIM, int P, class PH, int MODE, bool JAC, class Nodes, bool UNROLL_A = false, bool PRE = false>
__device__ __forceinline__ int pointwise_qp(const SpaceDev &s, const Prm &prm, double a, double b,
                                            const double (&v)[DIM][3][P + 1], double wq, const double (&xq)[DIM],
                                            const double (&hp)[DIM], const Nodes &nodes, double *__restrict__ Dt,
                                            long long dstr, double *__restrict__ Rt, long long rstr,
                                            const double *pre = nullptr) {
    using L = Lists<PH, DIM, MODE>;
    using KS = typename L::KS;
    constexpr int M = PH::M, NP1 = P + 1;
    constexpr int NKS = KS::NKS, NC = KS::NC;
    constexpr bool HESS = PH::HESS;
    double Phi[M][NC], Phit[M], W[NC], X[DIM][NC];
#pragma unroll
    for (int c = 0; c < NC; c++) {
        W[c] = 0.0;
#pragma unroll
        for (int m = 0; m < M; m++) Phi[m][c] = 0.0;
#pragma unroll
        for (int i = 0; i < DIM; i++) X[i][c] = 0.0;
    }
#pragma unroll
    for (int m = 0; m < M; m++) Phit[m] = 0.0;
    const bool nurbs_geom = (MODE == MODE_NURBS) && s.geom == IGA_GEOM_NURBS;

    constexpr int NEN = ipow(NP1, DIM);
    auto body = [&](int A) {
        int aa[3] = {0, 0, 0};
        {
            int r = A;
#pragma unroll
            for (int d = DIM - 1; d >= 0; d--) { aa[d] = r % NP1; r /= NP1; }
        }
        double Pc[NC];
        static_for<NC>([&](auto C) {
            constexpr int c = decltype(C)::value;
            Pc[c] = kind_value<KS, DIM, c, NP1>(v, aa);
        });
        double wA = 1.0;
        if (MODE == MODE_NURBS) {
            wA = nodes.w(A);
#pragma unroll
            for (int c = 0; c < NC; c++) W[c] += wA * Pc[c];
            if (nurbs_geom) {
#pragma unroll
                for (int i = 0; i < DIM; i++) {
                    const double xA = Nodes::PREMUL ? nodes.x(A, i) : wA * nodes.x(A, i);
#pragma unroll
                    for (int c = 0; c < NC; c++) X[i][c] += xA * Pc[c];
                }
            }
        }
#pragma unroll
        for (int m = 0; m < M; m++) {
            const double uA = (MODE == MODE_NURBS && Nodes::PREMUL) ? nodes.u(A, m) : wA * nodes.u(A, m);
#pragma unroll
            for (int c = 0; c < NC; c++) Phi[m][c] += uA * Pc[c];
            if (PH::UDOT && nodes.has_ud())
                Phit[m] += ((MODE == MODE_NURBS && Nodes::PREMUL) ? nodes.ud(A, m) : wA * nodes.ud(A, m)) * Pc[0];
        }
    };
    if constexpr (PRE) {
#pragma unroll
        for (int c = 0; c < NC; c++) {
            W[c] = pre[c];
#pragma unroll
            for (int i = 0; i < DIM; i++) X[i][c] = pre[NC + i * NC + c];
#pragma unroll
            for (int m = 0; m < M; m++) Phi[m][c] = pre[NC + DIM * NC + m * NC + c];
        }
#pragma unroll
        for (int m = 0; m < M; m++) Phit[m] = pre[NC + DIM * NC + M * NC + m];
    } else if constexpr (UNROLL_A) {
        static_for<NEN>([&](auto AA) { body(decltype(AA)::value); });
    } else {
#pragma unroll 1
        for (int A = 0; A < NEN; A++) body(A);
    }

    Fields<DIM, M> F;
    double T[NKS][NC];
    double dV;
    bool bad = false;
    if (MODE == MODE_PARAM) {
#pragma unroll
        for (int m = 0; m < M; m++) {
            F.u[m] = Phi[m][0];
#pragma unroll
            for (int i = 0; i < DIM; i++) F.gu[m][i] = Phi[m][1 + i];
            F.lu[m] = HESS ? Phi[m][NKS - 1] : 0.0;
            F.ut[m] = Phit[m];
        }
#pragma unroll
        for (int i = 0; i < DIM; i++) {
            F.x[i] = xq[i];
            F.hpar[i] = hp[i];
#pragma unroll
            for (int j = 0; j < DIM; j++) F.dxi[i][j] = (i == j) ? 1.0 : 0.0;
        }
        dV = wq;
#pragma unroll
        for (int k = 0; k < NKS; k++)
#pragma unroll
            for (int c = 0; c < NC; c++) T[k][c] = (k == c) ? 1.0 : 0.0;
    } else {
        // rational kinds as combinations of parametric kinds (drational P:234, ddrational P:245)
        const double w = W[0], iw = 1.0 / w;
        double rR[NC], rA[DIM][NC], rAB[HESS ? KS::NH : 1][NC];
#pragma unroll
        for (int c = 0; c < NC; c++) {
            rR[c] = (c == 0 ? 1.0 : 0.0) * iw;
#pragma unroll
            for (int al = 0; al < DIM; al++) rA[al][c] = ((c == 1 + al ? 1.0 : 0.0) - W[1 + al] * rR[c]) * iw;
        }
        if (HESS) {
#pragma unroll
            for (int h = 0; h < KS::NH; h++) {
                const int al = KS::hal(h), be = KS::hbe(h);
#pragma unroll
                for (int c = 0; c < NC; c++)
                    rAB[h][c] = ((c == 1 + DIM + h ? 1.0 : 0.0) - W[1 + DIM + h] * rR[c] - W[1 + al] * rA[be][c]
                                 - W[1 + be] * rA[al][c]) * iw;
            }
        }
        // isoparametric map by the quotient rule on the homogeneous sums
        double x[DIM], xa[DIM][DIM], xab[DIM][HESS ? KS::NH : 1];
#pragma unroll
        for (int i = 0; i < DIM; i++) {
            if (nurbs_geom) {
                x[i] = X[i][0] * iw;
#pragma unroll
                for (int al = 0; al < DIM; al++) xa[i][al] = (X[i][1 + al] - x[i] * W[1 + al]) * iw;
                if (HESS) {
#pragma unroll
                    for (int h = 0; h < KS::NH; h++) {
                        const int al = KS::hal(h), be = KS::hbe(h);
                        xab[i][h] = (X[i][1 + DIM + h] - x[i] * W[1 + DIM + h] - xa[i][be] * W[1 + al]
                                     - xa[i][al] * W[1 + be]) * iw;
                    }
                }
            } else {
                x[i] = xq[i];
#pragma unroll
                for (int al = 0; al < DIM; al++) xa[i][al] = (i == al) ? 1.0 : 0.0;
#pragma unroll
                for (int h = 0; h < (HESS ? KS::NH : 1); h++) xab[i][h] = 0.0;
            }
        }
        // inverse map xi_{alpha,i} (identity P:287, derividentity P:292 as a matrix inverse)
        double det, Xi[DIM][DIM];
        if constexpr (DIM == 2) {
            det = xa[0][0] * xa[1][1] - xa[0][1] * xa[1][0];
            const double id = 1.0 / det;
            Xi[0][0] = xa[1][1] * id;
            Xi[0][1] = -xa[0][1] * id;
            Xi[1][0] = -xa[1][0] * id;
            Xi[1][1] = xa[0][0] * id;
        } else {
            const double c00 = xa[1][1] * xa[2][2] - xa[1][2] * xa[2][1];
            const double c01 = xa[1][2] * xa[2][0] - xa[1][0] * xa[2][2];
            const double c02 = xa[1][0] * xa[2][1] - xa[1][1] * xa[2][0];
            det = xa[0][0] * c00 + xa[0][1] * c01 + xa[0][2] * c02;
            const double id = 1.0 / det;
            // Xi = adj(xa) / det, Xi[alpha][i]
            Xi[0][0] = c00 * id;
            Xi[1][0] = c01 * id;
            Xi[2][0] = c02 * id;
            Xi[0][1] = (xa[0][2] * xa[2][1] - xa[0][1] * xa[2][2]) * id;
            Xi[1][1] = (xa[0][0] * xa[2][2] - xa[0][2] * xa[2][0]) * id;
            Xi[2][1] = (xa[0][1] * xa[2][0] - xa[0][0] * xa[2][1]) * id;
            Xi[0][2] = (xa[0][1] * xa[1][2] - xa[0][2] * xa[1][1]) * id;
            Xi[1][2] = (xa[0][2] * xa[1][0] - xa[0][0] * xa[1][2]) * id;
            Xi[2][2] = (xa[0][0] * xa[1][1] - xa[0][1] * xa[1][0]) * id;
        }
        if (!(det > 0.0)) bad = true;
        // T rows: spatial kinds from rational kinds (dspatial P:309, ddspatial P:310)
#pragma unroll
        for (int c = 0; c < NC; c++) {
            T[0][c] = rR[c];
#pragma unroll
            for (int i = 0; i < DIM; i++) {
                double sum = 0.0;
#pragma unroll
                for (int al = 0; al < DIM; al++) sum += Xi[al][i] * rA[al][c];
                T[1 + i][c] = sum;
            }
        }
        if (HESS) {
            // xi_{nu,nl} = - x_{m,eps mu} xi_{eps,n} xi_{mu,l} xi_{nu,m}, only n = l needed
            double Xi2d[DIM][DIM];   // [nu][n] = xi_{nu,nn}
#pragma unroll
            for (int nu_ = 0; nu_ < DIM; nu_++)
#pragma unroll
                for (int n = 0; n < DIM; n++) {
                    double sum = 0.0;
#pragma unroll
                    for (int m = 0; m < DIM; m++)
#pragma unroll
                        for (int ep = 0; ep < DIM; ep++)
#pragma unroll
                            for (int mu = 0; mu < DIM; mu++)
                                sum -= xab[m][KS::hidx(ep, mu)] * Xi[ep][n] * Xi[mu][n] * Xi[nu_][m];
                    Xi2d[nu_][n] = sum;
                }
#pragma unroll
            for (int c = 0; c < NC; c++) {
                double sum = 0.0;
#pragma unroll
                for (int i = 0; i < DIM; i++) {
#pragma unroll
                    for (int al = 0; al < DIM; al++) {
#pragma unroll
                        for (int be = 0; be < DIM; be++) sum += Xi[al][i] * Xi[be][i] * rAB[KS::hidx(al, be)][c];
                        sum += Xi2d[al][i] * rA[al][c];
                    }
                }
                T[NKS - 1][c] = sum;
            }
        }
#pragma unroll
        for (int m = 0; m < M; m++) {
            double u0 = 0.0, l0 = 0.0;
            double gg[DIM];
#pragma unroll
            for (int i = 0; i < DIM; i++) gg[i] = 0.0;
#pragma unroll
            for (int c = 0; c < NC; c++) {
                u0 += T[0][c] * Phi[m][c];
#pragma unroll
                for (int i = 0; i < DIM; i++) gg[i] += T[1 + i][c] * Phi[m][c];
                if (HESS) l0 += T[NKS - 1][c] * Phi[m][c];
            }
            F.u[m] = u0;
            F.lu[m] = l0;
            F.ut[m] = Phit[m] * iw;
#pragma unroll
            for (int i = 0; i < DIM; i++) F.gu[m][i] = gg[i];
        }
#pragma unroll
        for (int i = 0; i < DIM; i++) {
            F.x[i] = x[i];
            F.hpar[i] = hp[i];
#pragma unroll
            for (int j = 0; j < DIM; j++) F.dxi[i][j] = Xi[i][j];
        }
        dV = det * wq;
    }

    typename PH::template State<DIM> st;
    PH::template prepare<DIM>(prm.p, F, st);
    double chk = 0.0;
    if (Rt) {
        double r[NKS * M];
        PH::template residual<DIM>(st, r);
        static_for<L::NR>([&](auto RR) {
            constexpr int rr = decltype(RR)::value;
            constexpr int c = L::R.c[rr], i = L::R.i[rr];
            double val = 0.0;
            static_for<NKS>([&](auto K) {
                constexpr int k = decltype(K)::value;
                if constexpr (KS::tmask(k, c) && PH::rmask(k, i)) val += T[k][c] * r[k * M + i];
            });
            val *= dV;
            chk += val;
            Rt[rr * rstr] = val;
        });
    }
    if constexpr (JAC) {
        if constexpr (MODE == MODE_PARAM) {
            static_for<NKS>([&](auto K2) {
                constexpr int k2 = decltype(K2)::value;
                static_for<M>([&](auto J) {
                    constexpr int j = decltype(J)::value;
                    double col[NKS * M];
                    PH::template dcol<DIM>(st, k2, j, a, b, col);
                    static_for<L::NE>([&](auto E) {
                        constexpr int ee = decltype(E)::value;
                        constexpr int c = L::E.c[ee], i = L::E.i[ee];
                        if constexpr (L::E.c2[ee] == k2 && L::E.j[ee] == j) {
                            const double val = col[c * M + i] * dV;
                            chk += val;
                            Dt[ee * dstr] = val;
                        }
                    });
                });
            });
        } else {
            double acc[L::NE];
#pragma unroll
            for (int ee = 0; ee < L::NE; ee++) acc[ee] = 0.0;
            static_for<NKS>([&](auto K2) {
                constexpr int k2 = decltype(K2)::value;
                static_for<M>([&](auto J) {
                    constexpr int j = decltype(J)::value;
                    double col[NKS * M];
                    PH::template dcol<DIM>(st, k2, j, a, b, col);
                    static_for<L::NE>([&](auto E) {
                        constexpr int ee = decltype(E)::value;
                        constexpr int c = L::E.c[ee], i = L::E.i[ee], c2 = L::E.c2[ee];
                        if constexpr (L::E.j[ee] == j && KS::tmask(k2, c2)) {
                            double sum = 0.0;
                            static_for<NKS>([&](auto K) {
                                constexpr int k = decltype(K)::value;
                                if constexpr (KS::tmask(k, c) && PH::template dmask<DIM>(k, i, k2, j))
                                    sum += T[k][c] * col[k * M + i];
                            });
                            acc[ee] += T[k2][c2] * sum;
                        }
                    });
                });
            });
#pragma unroll
            for (int ee = 0; ee < L::NE; ee++) {
                const double val = acc[ee] * dV;
                chk += val;
                Dt[ee * dstr] = val;
            }
        }
    }
    if (!isfinite(chk)) bad = true;
    if (!bad) return 0;
    return (MODE == MODE_NURBS && !(dV > 0.0)) ? 1 : 2;
}

}  // namespace iga
