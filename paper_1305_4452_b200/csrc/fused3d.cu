// fused3d.cu -- K3/K4 for 3D parametric spaces (configs 4, 5): one fused kernel per call.
//
// Persistent CTAs walk the element grid; per element the CTA runs Alg. 4 in phases
// separated by __syncthreads, everything staged in shared memory:
//   1. stage U_e, the element's 1D tables (3 axes), Gauss weights, CSR row starts and the
//      per-element column-offset table colOff[A][B] (closed form from the Alg. 3 tables);
//   2. field kinds at every point  Phi[q][m][k] = sum_A U_Am P_k(A,q)  (thread per (q, m)) and the
//      trial-kind values P_c(B,q) of every function (thread per (c, q, B));
//   3. per point: physics state + residual coefficients r~ (thread per q);
//   4. Jacobian coefficients: warp-uniform trial column (k2, j), lane = q -> dense per-(i,j)
//      blocks D[q][i,j][test kind][trial kind];
//   5. test-side sum factorisation, warp = component pair (i, j), lane = trial function B:
//      H(q) = D_(i,j)(q) P(B,q), then contraction over q2, q1, q0 with the 1D tables
//      (729 FMA per column for p = 2 instead of 19683 for the rank form); the block goes to a
//      shared staging array in CSR-segment order [A][i][B][j];
//   6. F_e: warp = component i, lane = A, same kinds / tables;
//   7. emission: warp = row (A, i), lanes = consecutive (B, j) -> red.global.add.f64 into the CSR
//      values (runs of p+1 nodes x m dofs are contiguous in CSR), F likewise.
#include <cstdio>

#include "iga_host.h"
#include "pointwise.cuh"

namespace iga {

template <int P, class PH>
struct F3 {
    static constexpr int M = PH::M;
    static constexpr int NP1 = P + 1, NQ1 = P + 1, NQ = NQ1 * NQ1 * NQ1, NEN = NP1 * NP1 * NP1;
    static constexpr int NCOMBO = M * M;
    static constexpr int NWARP = NCOMBO % 9 == 0 ? 9 : 8;       // m=3: 9 pairs, m=4: 2 per warp
    static constexpr int NT = 32 * NWARP;
    using L = Lists<PH, 3, MODE_PARAM>;
    using KS = typename L::KS;
    static constexpr int NKS = KS::NKS, NC = KS::NC, NR = L::NR, NTK = L::NTK, NQK = L::NQK;
    static constexpr int DB = NTK * NQK;                      // dense block per (i, j)
    using State = typename PH::template State<3>;
    static constexpr int STD = (sizeof(State) + 7) / 8;      // doubles per state
    // shared-memory carve-up (in doubles)
    static constexpr int O_U = 0;                            // [NEN][M]
    static constexpr int O_UD = O_U + NEN * M;               // [NEN][M]
    static constexpr int O_TAB = O_UD + NEN * M;             // [3][NQ1][3][NP1]
    static constexpr int O_QW = O_TAB + 3 * NQ1 * 3 * NP1;   // [3][NQ1]
    static constexpr int O_QX = O_QW + 3 * NQ1;              // [3][NQ1]
    static constexpr int O_HP = O_QX + 3 * NQ1;              // [4]
    static constexpr int O_PHI = O_HP + 4;                   // [NQ][M][NKS+1]  (+1: udot)
    static constexpr int O_ST = O_PHI + NQ * M * (NKS + 1);  // [NQ][STD]
    static constexpr int O_DV = O_ST + NQ * STD;             // [NQ]
    static constexpr int O_PB = O_DV + NQ;                   // [NQK][NQ][NEN]  trial kind values
    static constexpr int O_R = O_PB + NQK * NQ * NEN;        // [NR][NQ]
    static constexpr int O_D = O_R + NR * NQ;                // [NQ][M*M][NTK][NQK]
    static constexpr int O_KE = O_D + NQ * NCOMBO * DB;      // [NEN][M][NEN][M]
    static constexpr int O_FE = O_KE + NEN * M * NEN * M;    // [NEN][M]
    static constexpr int O_RS = O_FE + NEN * M;              // long long [NEN*M] row starts
    static constexpr int O_ND = O_RS + NEN * M;              // long long [NEN] nodes
    static constexpr int O_CO = O_ND + NEN;                  // int [NEN][NEN] column offsets (in nodes)
    static constexpr size_t SMEM = (size_t)O_CO * sizeof(double) + (size_t)NEN * NEN * sizeof(int);
};

// test-side sum factorisation in 3D of one column: trial function B, component pair ij.
//   Kc[A] = sum_q sum_{tk,qk} P_tk(A,q) D[q][ij][tk][qk] P_qk(B,q)
template <class F>
__device__ __forceinline__ void tsf_column_3d(double (&Kc)[F::NEN], const double *__restrict__ Dsm, int ij,
                                              const double *__restrict__ Pb, int B, const double *__restrict__ tab) {
    using L = typename F::L;
    using KS = typename F::KS;
    constexpr int NP1 = F::NP1, NQ1 = F::NQ1, NEN = F::NEN, NTK = F::NTK, NQK = F::NQK, DB = F::DB;
    auto T = [&](int d, int q, int k, int a) -> double { return tab[((d * NQ1 + q) * 3 + k) * NP1 + a]; };
    // which stage tracks exist (test kinds' separable terms)
    constexpr auto used01 = [](int o0, int o1) {
        for (int t = 0; t < NTK; t++) {
            const int c = L::tk(t);
            for (int s = 0; s < KS::nterms(c); s++)
                if (KS::ord(c, s, 0) == o0 && KS::ord(c, s, 1) == o1) return true;
        }
        return false;
    };
    constexpr auto used0 = [](int o0) {
        for (int t = 0; t < NTK; t++) {
            const int c = L::tk(t);
            for (int s = 0; s < KS::nterms(c); s++)
                if (KS::ord(c, s, 0) == o0) return true;
        }
        return false;
    };
#pragma unroll
    for (int A = 0; A < NEN; A++) Kc[A] = 0.0;
#pragma unroll 1
    for (int q0 = 0; q0 < NQ1; q0++) {
        double Tt[3][NP1][NP1];
#pragma unroll
        for (int o = 0; o < 3; o++)
#pragma unroll
            for (int x = 0; x < NP1; x++)
#pragma unroll
                for (int y = 0; y < NP1; y++) Tt[o][x][y] = 0.0;
#pragma unroll 1
        for (int q1 = 0; q1 < NQ1; q1++) {
            double S[3][3][NP1];
#pragma unroll
            for (int o = 0; o < 3; o++)
#pragma unroll
                for (int o2 = 0; o2 < 3; o2++)
#pragma unroll
                    for (int x = 0; x < NP1; x++) S[o][o2][x] = 0.0;
#pragma unroll
            for (int q2 = 0; q2 < NQ1; q2++) {
                const int q = (q0 * NQ1 + q1) * NQ1 + q2;
                double pb[NQK];
#pragma unroll
                for (int k = 0; k < NQK; k++) pb[k] = Pb[(k * F::NQ + q) * NEN + B];
                const double *Dq = Dsm + (q * F::NCOMBO + ij) * DB;
                double H[NTK];
#pragma unroll
                for (int t = 0; t < NTK; t++) {
                    double h = 0.0;
#pragma unroll
                    for (int k = 0; k < NQK; k++) h += Dq[t * NQK + k] * pb[k];
                    H[t] = h;
                }
                static_for<NTK>([&](auto TK) {
                    constexpr int t = decltype(TK)::value;
                    constexpr int c = L::tk(t);
                    static_for<KS::nterms(c)>([&](auto TT) {
                        constexpr int s = decltype(TT)::value;
                        constexpr int o0 = KS::ord(c, s, 0), o1 = KS::ord(c, s, 1), o2 = KS::ord(c, s, 2);
#pragma unroll
                        for (int a2 = 0; a2 < NP1; a2++) S[o0][o1][a2] += H[t] * T(2, q2, o2, a2);
                    });
                });
            }
            static_for<3>([&](auto O0) {
                constexpr int o0 = decltype(O0)::value;
                static_for<3>([&](auto O1) {
                    constexpr int o1 = decltype(O1)::value;
                    if constexpr (used01(o0, o1)) {
#pragma unroll
                        for (int a1 = 0; a1 < NP1; a1++) {
                            const double n1 = T(1, q1, o1, a1);
#pragma unroll
                            for (int a2 = 0; a2 < NP1; a2++) Tt[o0][a1][a2] += n1 * S[o0][o1][a2];
                        }
                    }
                });
            });
        }
        static_for<3>([&](auto O0) {
            constexpr int o0 = decltype(O0)::value;
            if constexpr (used0(o0)) {
#pragma unroll
                for (int a0 = 0; a0 < NP1; a0++) {
                    const double n0 = T(0, q0, o0, a0);
#pragma unroll
                    for (int a1 = 0; a1 < NP1; a1++)
#pragma unroll
                        for (int a2 = 0; a2 < NP1; a2++) Kc[(a0 * NP1 + a1) * NP1 + a2] += n0 * Tt[o0][a1][a2];
                }
            }
        });
    }
}

template <int P, class PH, bool JAC>
__global__ void __launch_bounds__(F3<P, PH>::NT, 1)
k_fused3d(SpaceDev s, Prm prm, double a, double b, const double *__restrict__ U, const double *__restrict__ Ud,
          double *__restrict__ val, double *__restrict__ Fout, long long nelem) {
    using F = F3<P, PH>;
    using L = typename F::L;
    using KS = typename F::KS;
    using State = typename F::State;
    constexpr int M = F::M, NP1 = F::NP1, NQ1 = F::NQ1, NQ = F::NQ, NEN = F::NEN;
    constexpr int NKS = F::NKS, NR = F::NR, NTK = F::NTK, NQK = F::NQK, DB = F::DB;
    extern __shared__ __align__(16) double sm[];
    double *sU = sm + F::O_U, *sUd = sm + F::O_UD, *sTab = sm + F::O_TAB, *sQW = sm + F::O_QW, *sQX = sm + F::O_QX;
    double *sHP = sm + F::O_HP, *sPhi = sm + F::O_PHI, *sDV = sm + F::O_DV, *sPb = sm + F::O_PB, *sR = sm + F::O_R;
    double *sD = sm + F::O_D, *sKe = sm + F::O_KE, *sFe = sm + F::O_FE;
    State *sSt = reinterpret_cast<State *>(sm + F::O_ST);
    long long *sRS = reinterpret_cast<long long *>(sm + F::O_RS);   // [NEN*M] CSR start of row (A, i)
    long long *sNode = reinterpret_cast<long long *>(sm + F::O_ND); // [NEN]
    int *sCO = reinterpret_cast<int *>(sm + F::O_CO);               // [NEN][NEN] column offset (nodes)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    int errbits = 0;
    const int n1 = s.ax[1].el_hi - s.ax[1].el_lo, n2 = s.ax[2].el_hi - s.ax[2].el_lo;
    auto TB = [&](int d, int q, int k, int aa) -> double { return sTab[((d * NQ1 + q) * 3 + k) * NP1 + aa]; };

    for (long long el = blockIdx.x; el < nelem; el += gridDim.x) {
        int e[3];
        {
            long long r = el;
            e[2] = s.ax[2].el_lo + (int)(r % n2); r /= n2;
            e[1] = s.ax[1].el_lo + (int)(r % n1); r /= n1;
            e[0] = s.ax[0].el_lo + (int)r;
        }
        // ---- 1. stage ----
        for (int i = tid; i < 3 * NQ1 * 3 * NP1; i += F::NT) {
            const int d = i / (NQ1 * 3 * NP1), r = i % (NQ1 * 3 * NP1);
            sTab[i] = s.ax[d].tab[(size_t)e[d] * NQ1 * 3 * NP1 + r];
        }
        for (int i = tid; i < 3 * NQ1; i += F::NT) {
            const int d = i / NQ1, q = i % NQ1;
            sQW[i] = s.ax[d].qw[(size_t)e[d] * NQ1 + q];
            sQX[i] = s.ax[d].qx[(size_t)e[d] * NQ1 + q];
        }
        if (tid < 3) sHP[tid] = s.ax[tid].hpar[e[tid]];
        for (int A = tid; A < NEN; A += F::NT) {
            int g[3], W[3];
            long long S[3], T[3];
            int rr = A;
            for (int d = 2; d >= 0; d--) {
                const int aa = rr % NP1;
                rr /= NP1;
                g[d] = s.ax[d].first[e[d]] + aa;
                if (g[d] >= s.ax[d].nu) g[d] -= s.ax[d].nu;
                W[d] = s.ax[d].rowW[g[d]];
                S[d] = s.ax[d].rowS[g[d]];
                T[d] = s.ax[d].T;
            }
            const long long node = ((long long)g[0] * s.ax[1].nu + g[1]) * s.ax[2].nu + g[2];
            sNode[A] = node;
            const long long base = (long long)M * M * (S[0] * T[1] * T[2] + W[0] * S[1] * T[2] + (long long)W[0] * W[1] * S[2]);
            const long long Wn = (long long)W[0] * W[1] * W[2];
            for (int i = 0; i < M; i++) sRS[A * M + i] = base + i * Wn * M;
            // column offsets (in nodes) of every B in row A: ((pos0 W1 + pos1) W2 + pos2)
            const int a0 = A / (NP1 * NP1), a1 = (A / NP1) % NP1, a2 = A % NP1;
            const int *p0 = s.ax[0].pos + (size_t)e[0] * NP1 * NP1 + a0 * NP1;
            const int *p1 = s.ax[1].pos + (size_t)e[1] * NP1 * NP1 + a1 * NP1;
            const int *p2 = s.ax[2].pos + (size_t)e[2] * NP1 * NP1 + a2 * NP1;
            for (int B = 0; B < NEN; B++) {
                const int b0 = B / (NP1 * NP1), b1 = (B / NP1) % NP1, b2 = B % NP1;
                sCO[A * NEN + B] = (p0[b0] * W[1] + p1[b1]) * W[2] + p2[b2];
            }
        }
        __syncthreads();
        for (int i = tid; i < NEN * M; i += F::NT) {
            const long long node = sNode[i / M];
            sU[i] = U[node * M + i % M];
            sUd[i] = Ud ? Ud[node * M + i % M] : 0.0;
        }
        __syncthreads();

        // ---- 2. field kinds per (q, m) and trial-kind values per (k, q, B) ----
        for (int task = tid; task < NQ * M; task += F::NT) {
            const int q = task / M, m = task % M;
            const int q0 = q / (NQ1 * NQ1), q1 = (q / NQ1) % NQ1, q2 = q % NQ1;
            double acc[NKS + 1];
#pragma unroll
            for (int k = 0; k <= NKS; k++) acc[k] = 0.0;
#pragma unroll
            for (int A = 0; A < NEN; A++) {
                const int a0 = A / (NP1 * NP1), a1 = (A / NP1) % NP1, a2 = A % NP1;
                double v[3][3];
#pragma unroll
                for (int k = 0; k < 3; k++) {
                    v[0][k] = TB(0, q0, k, a0);
                    v[1][k] = TB(1, q1, k, a1);
                    v[2][k] = TB(2, q2, k, a2);
                }
                const double uA = sU[A * M + m];
                static_for<NKS>([&](auto K) {
                    constexpr int k = decltype(K)::value;
                    double pv = 0.0;
                    static_for<KS::nterms(k)>([&](auto TT) {
                        constexpr int t = decltype(TT)::value;
                        pv += v[0][KS::ord(k, t, 0)] * v[1][KS::ord(k, t, 1)] * v[2][KS::ord(k, t, 2)];
                    });
                    acc[k] += uA * pv;
                });
                acc[NKS] += sUd[A * M + m] * v[0][0] * v[1][0] * v[2][0];
            }
#pragma unroll
            for (int k = 0; k <= NKS; k++) sPhi[(q * M + m) * (NKS + 1) + k] = acc[k];
        }
        if (JAC)
            for (int task = tid; task < NQK * NQ * NEN; task += F::NT) {
                const int kk = task / (NQ * NEN), q = (task / NEN) % NQ, B = task % NEN;
                const int q0 = q / (NQ1 * NQ1), q1 = (q / NQ1) % NQ1, q2 = q % NQ1;
                const int b0 = B / (NP1 * NP1), b1 = (B / NP1) % NP1, b2 = B % NP1;
                double pv = 0.0;
                static_for<NQK>([&](auto K) {
                    constexpr int kq = decltype(K)::value;
                    constexpr int cc = L::qk(kq);
                    if (kk == kq) {
                        static_for<KS::nterms(cc)>([&](auto TT) {
                            constexpr int t = decltype(TT)::value;
                            pv += TB(0, q0, KS::ord(cc, t, 0), b0) * TB(1, q1, KS::ord(cc, t, 1), b1)
                                  * TB(2, q2, KS::ord(cc, t, 2), b2);
                        });
                    }
                });
                sPb[task] = pv;
            }
        __syncthreads();

        // ---- 3. per-point state + residual coefficients ----
        if (tid < NQ) {
            const int q = tid;
            const int q0 = q / (NQ1 * NQ1), q1 = (q / NQ1) % NQ1, q2 = q % NQ1;
            Fields<3, M> Fq;
#pragma unroll
            for (int m = 0; m < M; m++) {
                const double *ph = sPhi + (q * M + m) * (NKS + 1);
                Fq.u[m] = ph[0];
#pragma unroll
                for (int i = 0; i < 3; i++) Fq.gu[m][i] = ph[1 + i];
                Fq.lu[m] = PH::HESS ? ph[NKS - 1] : 0.0;
                Fq.ut[m] = ph[NKS];
            }
            const int qq[3] = {q0, q1, q2};
#pragma unroll
            for (int i = 0; i < 3; i++) {
                Fq.x[i] = sQX[i * NQ1 + qq[i]];
                Fq.hpar[i] = sHP[i];
#pragma unroll
                for (int j = 0; j < 3; j++) Fq.dxi[i][j] = (i == j) ? 1.0 : 0.0;
            }
            const double dV = sQW[q0] * sQW[NQ1 + q1] * sQW[2 * NQ1 + q2];
            State st;
            PH::template prepare<3>(prm.p, Fq, st);
            sSt[q] = st;
            sDV[q] = dV;
            if (Fout) {
                double r[NKS * M];
                PH::template residual<3>(st, r);
                double chk = 0.0;
                static_for<NR>([&](auto RR) {
                    constexpr int rr = decltype(RR)::value;
                    constexpr int c = L::R.c[rr], i = L::R.i[rr];
                    const double v = r[c * M + i] * dV;
                    chk += v;
                    sR[rr * NQ + q] = v;
                });
                if (!isfinite(chk)) errbits |= 2;
            }
        }
        __syncthreads();

        // ---- 4. Jacobian coefficients: warp-uniform trial column (k2 = qk(kq), j), lane = q ----
        if constexpr (JAC) {
            for (int kj = warp; kj < NQK * M; kj += F::NWARP) {
                if (lane < NQ) {
                    const int q = lane;
                    const State st = sSt[q];
                    const double dV = sDV[q];
                    double chk = 0.0;
                    static_for<NQK * M>([&](auto KJ) {
                        constexpr int kq = decltype(KJ)::value / M, j = decltype(KJ)::value % M;
                        constexpr int k2 = L::qk(kq);
                        if (kj == decltype(KJ)::value) {
                            double col[NKS * M];
                            PH::template dcol<3>(st, k2, j, a, b, col);
#pragma unroll
                            for (int i = 0; i < M; i++) {
                                double *dst = sD + (q * F::NCOMBO + i * M + j) * DB + kq;
                                static_for<NTK>([&](auto TK) {
                                    constexpr int t = decltype(TK)::value;
                                    const double v = col[L::tk(t) * M + i] * dV;
                                    chk += v;
                                    dst[t * NQK] = v;
                                });
                            }
                        }
                    });
                    if (!isfinite(chk)) errbits |= 2;
                }
            }
            __syncthreads();

            // ---- 5. test-side sum factorisation, warp = (i, j) pairs, lane = B ----
            for (int combo = warp; combo < F::NCOMBO; combo += F::NWARP) {
                if (lane < NEN) {
                    double Kc[NEN];
                    tsf_column_3d<F>(Kc, sD, combo, sPb, lane, sTab);
                    const int I = combo / M, J = combo % M, B = lane;
#pragma unroll
                    for (int A = 0; A < NEN; A++) sKe[((A * M + I) * NEN + B) * M + J] = Kc[A];
                }
            }
        }
        // ---- 6. residual F_e[A, i]: warp = i, lane = A ----
        if (Fout && warp < M && lane < NEN) {
            const int A = lane;
            const int a0 = A / (NP1 * NP1), a1 = (A / NP1) % NP1, a2 = A % NP1;
            static_for<M>([&](auto II) {
                constexpr int I = decltype(II)::value;
                if (warp == I) {
                    double acc = 0.0;
#pragma unroll 1
                    for (int q = 0; q < NQ; q++) {
                        const int q0 = q / (NQ1 * NQ1), q1 = (q / NQ1) % NQ1, q2 = q % NQ1;
                        double v[3][3];
#pragma unroll
                        for (int k = 0; k < 3; k++) {
                            v[0][k] = TB(0, q0, k, a0);
                            v[1][k] = TB(1, q1, k, a1);
                            v[2][k] = TB(2, q2, k, a2);
                        }
                        static_for<NR>([&](auto RR) {
                            constexpr int rr = decltype(RR)::value;
                            constexpr int c = L::R.c[rr];
                            if constexpr (L::R.i[rr] == I) {
                                double pv = 0.0;
                                static_for<KS::nterms(c)>([&](auto TT) {
                                    constexpr int t = decltype(TT)::value;
                                    pv += v[0][KS::ord(c, t, 0)] * v[1][KS::ord(c, t, 1)] * v[2][KS::ord(c, t, 2)];
                                });
                                acc += pv * sR[rr * NQ + q];
                            }
                        });
                    }
                    sFe[A * M + I] = acc;
                }
            });
        }
        __syncthreads();

        // ---- 7. emission: warp = row (A, i), lanes = consecutive (B, j) ----
        if constexpr (JAC) {
            for (int row = warp; row < NEN * M; row += F::NWARP) {
                const int A = row / M;
                const long long rs = sRS[row];
                const double *src = sKe + (size_t)row * NEN * M;
                const int *co = sCO + A * NEN;
                for (int t = lane; t < NEN * M; t += 32) {
                    const int B = t / M, j = t - B * M;
                    atomicAdd(val + rs + (long long)co[B] * M + j, src[t]);
                }
            }
        }
        if (Fout)
            for (int task = tid; task < NEN * M; task += F::NT) atomicAdd(Fout + sNode[task / M] * M + task % M, sFe[task]);
        __syncthreads();
    }
    if (errbits) atomicOr(s.errflag, errbits);
}

template <int P, class PH>
static iga_status run_fused3d(iga_space_s *s, const iga_phys *phys, double a, double b, const double *U,
                              const double *Ud, double *val, double *F, cudaStream_t st, int nsm) {
    using FF = F3<P, PH>;
    Prm prm;
    for (int i = 0; i < 8; i++) prm.p[i] = phys->p[i];
    const bool jac = val != nullptr;
    const size_t smem = FF::SMEM;
    static bool attr[2] = {false, false};
    if (!attr[jac]) {
        cudaError_t ce = jac ? cudaFuncSetAttribute(k_fused3d<P, PH, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                             : cudaFuncSetAttribute(k_fused3d<P, PH, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ce != cudaSuccess) { set_error(std::string("fused3d smem: ") + cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
        attr[jac] = true;
    }
    int occ = 1;
    if (jac) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fused3d<P, PH, true>, FF::NT, smem);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fused3d<P, PH, false>, FF::NT, smem);
    occ = std::max(occ, 1);
    const long long nel = s->nel_local;
    const int grid = (int)std::min<long long>(nel, (long long)nsm * occ);
    int launches = 0;
    if (jac) { ProfScope ps(s, "k_zero", st); k_zero_vec(val, s->nnz_owned, st, nsm); launches++; }
    if (F) { ProfScope ps(s, "k_zero", st); k_zero_vec(F, s->nrows_owned, st, nsm); launches++; }
    {
        ProfScope ps(s, "k_fused3d", st);
        if (jac) k_fused3d<P, PH, true><<<grid, FF::NT, smem, st>>>(s->dev, prm, a, b, U, Ud, val, F, nel);
        else k_fused3d<P, PH, false><<<grid, FF::NT, smem, st>>>(s->dev, prm, a, b, U, Ud, val, F, nel);
        launches++;
    }
    s->last_launches = launches;
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) { set_error(std::string("fused3d launch: ") + cudaGetErrorString(ce)); return IGA_ERR_CUDA; }
    return IGA_OK;
}

iga_status launch_fused3d(iga_space_s *s, const iga_phys *ph, double a, double b, const double *U,
                          const double *Ud, double *val, double *F, cudaStream_t st, int nsm) {
    if (s->dim != 3 || s->mode != MODE_PARAM || s->nranks != 1) return IGA_ERR_STATE;
    if (s->p[0] != 2 || s->p[1] != 2 || s->p[2] != 2) return IGA_ERR_STATE;
    if (ph->kind == IGA_PHYS_NS_VMS && s->dof == 4) return run_fused3d<2, PhysNSVMS>(s, ph, a, b, U, Ud, val, F, st, nsm);
    if (ph->kind == IGA_PHYS_NEOHOOKE && s->dof == 3) return run_fused3d<2, PhysNeoHooke>(s, ph, a, b, U, Ud, val, F, st, nsm);
    return IGA_ERR_STATE;
}

}  // namespace iga
